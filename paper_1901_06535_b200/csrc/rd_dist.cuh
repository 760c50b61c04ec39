// rd_dist.cuh — multi-GPU row slabs inside the library (SURVEY.md §8(b)
// rd_dist_unique_id / rd_create_dist, §8(e)).
//
// PRODUCT CODE, part of the rd_runtime.cu translation unit (it uses the
// runtime's launch machinery directly). The paper has no multi-device path
// (one tablet); the decomposition is BASELINE.json
// north_star's "row-slab domain decomposition across the 8 GPUs of one box,
// with halo exchange by NCCL send/recv or CUDA P2P over NVLink overlapped
// with interior compute".
//
// One handle per rank (one process per GPU, or one host thread per rank in
// one process). Rank r of G owns global rows [row0(r), row0(r) + rows(r)),
// the first H % G ranks one row more, with halo = K ghost rows above and
// below (K = the temporal-blocking depth). rd_step(n) on a dist handle runs
// the whole super-step here:
//   1. checkpoint;
//   2. blocks of k <= K steps. Each block: the compute stream grants the
//      neighbours write access to its ghost rows, and launches the interior
//      rows (they read owned rows only); meanwhile the exchange stream waits
//      for the neighbours' grants, copies this rank's send rows straight into
//      their ghost rows with cudaMemcpyAsync over the peer mapping -- copy
//      engines, no SMs, so the transfer runs under the interior launch that
//      fills every SM -- signals "landed" to them and waits for their rows to
//      land here; the compute stream waits for the exchange stream (an event)
//      and launches the two edge bands. Across processes the grants / landed
//      signals are stream-ordered 32-bit counters in the arenas (written with
//      cuStreamWriteValue32, waited on with cuStreamWaitValue32 on the
//      exchange stream only); between host threads of one process they are
//      CUDA events (local_publish). Transport fallback (no peer mapping, or
//      RD_DIST_TRANSPORT=nccl): grouped ncclSend/ncclRecv on the exchange
//      stream;
//   3. one fault / division-guard flag read, OR-reduced over the ranks
//      (ncclAllReduce MAX, or the in-process group's host reduction) together
//      with a digest of the control state (stimuli, probes, timelapse,
//      parameters, step) that must agree on every rank;
//   4. if any rank saw a non-finite cell or a tripped guard: every rank
//      restores and replays step by step in PRECISE mode (one exchange per
//      step), all stopping at the first failing step with the global first
//      cell (MIN over ranks of the row-major key).
// Counters are monotone across rd_step calls (the block sequence is the same
// on every rank), so they never need resetting.

#include <dlfcn.h>
#include <fcntl.h>
#include <nccl.h>  // types and enums only; the library is opened with dlopen
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <chrono>

#include <condition_variable>
#include <memory>
#include <random>

namespace {

// ---- NCCL, opened at run time (librd loads without it; RD_ENCCL if absent) --
struct NcclApi {
  bool ok = false;
  std::string why;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

const NcclApi& nccl_api() {
  static NcclApi api = [] {
    NcclApi a;
    // 1. a copy this process already loaded (e.g. torch's): the soname is
    //    taken, so any other copy would clash with it;
    // 2. RD_NCCL_LIB (the binding points it at the NCCL torch ships, so that a
    //    later `import torch` finds the copy it links against);
    // 3. the system's libnccl.so.2 (plain C callers).
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h)
      if (const char* p = getenv("RD_NCCL_LIB"))
        if (*p) h = dlopen(p, RTLD_NOW | RTLD_LOCAL);
    for (const char* name : {"libnccl.so.2", "libnccl.so"})
      if (!h) h = dlopen(name, RTLD_NOW | RTLD_LOCAL);
    if (!h) {
      a.why = std::string("NCCL not found (dlopen libnccl.so.2): ") + (dlerror() ? dlerror() : "");
      return a;
    }
    auto sym = [&](const char* n) { return dlsym(h, n); };
    a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(sym("ncclGetUniqueId"));
    a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(sym("ncclCommInitRank"));
    a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(sym("ncclCommDestroy"));
    a.AllReduce = reinterpret_cast<decltype(a.AllReduce)>(sym("ncclAllReduce"));
    a.AllGather = reinterpret_cast<decltype(a.AllGather)>(sym("ncclAllGather"));
    a.Send = reinterpret_cast<decltype(a.Send)>(sym("ncclSend"));
    a.Recv = reinterpret_cast<decltype(a.Recv)>(sym("ncclRecv"));
    a.GroupStart = reinterpret_cast<decltype(a.GroupStart)>(sym("ncclGroupStart"));
    a.GroupEnd = reinterpret_cast<decltype(a.GroupEnd)>(sym("ncclGroupEnd"));
    a.GetErrorString = reinterpret_cast<decltype(a.GetErrorString)>(sym("ncclGetErrorString"));
    a.ok = a.GetUniqueId && a.CommInitRank && a.CommDestroy && a.AllReduce && a.AllGather && a.Send && a.Recv &&
           a.GroupStart && a.GroupEnd && a.GetErrorString;
    if (!a.ok) a.why = "NCCL library lacks a required symbol";
    return a;
  }();
  return api;
}

#define RD_NCCL(sim, call)                                                                              \
  do {                                                                                                  \
    ncclResult_t r_ = (call);                                                                           \
    if (r_ != ncclSuccess)                                                                              \
      return set_err((sim), RD_ENCCL, "%s: %s (%s:%d)", #call, nccl_api().GetErrorString(r_), __FILE__, \
                     __LINE__);                                                                         \
  } while (0)

// ---- in-process groups (one host thread per rank; rd_dist_local_id) --------
constexpr char kLocalMagic[8] = {'R', 'D', 'L', 'O', 'C', 'A', 'L', '1'};

struct LocalGroup {
  std::mutex mu;
  std::condition_variable cv;
  int world = 0;
  std::vector<rd_sim*> members;
  int joined = 0, left = 0;
  uint64_t round = 0;  // completed reductions
  int arrived = 0;
  std::vector<uint64_t> acc, result;
  // per rank: the last block whose grant / landed event it has recorded
  std::vector<uint32_t> granted, landed;
};

std::mutex g_local_mu;
std::map<uint64_t, std::shared_ptr<LocalGroup>> g_local;

// In-process ranks order their halo copies with CUDA events instead of
// device-side counters: ranks on one device share its hardware queues, and a
// stream-memory wait queued ahead of the write it waits for (another host
// thread's, submitted later) would block that queue for good. An event wait
// only ever waits for work already submitted, so the order is deadlock-free
// by construction. The host thread waits until the neighbour has RECORDED
// the block's event (publish / await below), then waits on it on the stream.
// Two events per kind suffice: a rank re-records slot e % 2 at block e + 2
// only after it has seen the neighbour's block-(e + 1) publication, which the
// neighbour makes after its wait on the block-e event.
void local_publish(LocalGroup& g, std::vector<uint32_t>& what, int rank, uint32_t e) {
  std::lock_guard<std::mutex> lk(g.mu);
  what[(size_t)rank] = e;
  g.cv.notify_all();
}

void local_await(LocalGroup& g, std::vector<uint32_t>& what, int rank, uint32_t e) {
  std::unique_lock<std::mutex> lk(g.mu);
  g.cv.wait(lk, [&] { return what[(size_t)rank] >= e; });
}

// Element-wise MAX over the ranks of v (every rank calls with the same size).
void local_allmax(LocalGroup& g, std::vector<uint64_t>& v) {
  std::unique_lock<std::mutex> lk(g.mu);
  const uint64_t my_round = g.round;
  if (g.arrived == 0)
    g.acc = v;
  else
    for (size_t i = 0; i < v.size(); ++i) g.acc[i] = std::max(g.acc[i], v[i]);
  if (++g.arrived == g.world) {
    g.result = g.acc;
    g.arrived = 0;
    ++g.round;
    g.cv.notify_all();
  } else {
    g.cv.wait(lk, [&] { return g.round != my_round; });
  }
  v = g.result;
}

// ---- one-node process groups without NCCL (rd_dist_shm_id) -----------------
// Ranks are processes of one box (one per GPU, or several sharing a GPU to
// test the cross-process protocol on one device). The control plane -- the
// record all-gather of the rendezvous and the per-rd_step flag reduction --
// lives in a POSIX shared-memory segment; the data plane is the same copy-
// engine push over CUDA IPC mappings as with NCCL (there is no send/recv
// fallback here: a failed mapping is an error).
constexpr char kShmMagic[8] = {'R', 'D', 'S', 'H', 'M', '0', '0', '1'};
constexpr int kShmMaxWorld = 64, kShmWords = 64;

struct ShmSeg {
  std::atomic<uint32_t> world;    // set by the first rank to join
  std::atomic<uint32_t> joined;   // ranks that have mapped the segment
  std::atomic<uint32_t> left;     // ranks that have destroyed their handle
  std::atomic<uint32_t> failed;   // a rank gave up (timeout): every waiter returns
  std::atomic<uint64_t> arrived;  // monotone barrier counter: world per round
  uint64_t slot[2][kShmMaxWorld][kShmWords];  // a rank's contribution, by round parity
  unsigned char rec[kShmMaxWorld][256];       // the DistRec of every rank
};

struct ShmGroup {
  ShmSeg* seg = nullptr;
  std::string name;
  int rank = 0, world = 1;
  uint64_t round = 0;  // reductions this rank has completed
};

double shm_timeout_s() {
  const char* e = getenv("RD_DIST_TIMEOUT_S");
  const double t = e && *e ? atof(e) : 0.0;
  return t > 0 ? t : 300.0;
}

std::string shm_name(const uint8_t id[128]) {
  uint64_t tok;
  std::memcpy(&tok, id + 8, 8);
  char buf[64];
  snprintf(buf, sizeof buf, "/rd_dist_%016llx", (unsigned long long)tok);
  return buf;
}

// All ranks have arrived `round + 1` times. false on timeout or when another
// rank failed (a dead peer must not hang the rest for good).
bool shm_barrier(ShmGroup& g) {
  ShmSeg& m = *g.seg;
  const uint64_t target = (uint64_t)g.world * (g.round + 1);
  m.arrived.fetch_add(1, std::memory_order_acq_rel);
  const auto t0 = std::chrono::steady_clock::now();
  const double limit = shm_timeout_s();
  for (unsigned spins = 0; m.arrived.load(std::memory_order_acquire) < target; ++spins) {
    if (m.failed.load(std::memory_order_acquire)) return false;
    if (spins > 2000) usleep(50);
    if ((spins & 1023) == 1023 &&
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > limit) {
      m.failed.store(1, std::memory_order_release);
      return false;
    }
  }
  ++g.round;
  return true;
}

// Element-wise MAX over the ranks. A rank writes its slot of parity
// round % 2, all meet, each reduces all slots. A slot is rewritten two
// rounds later, i.e. after a barrier every reader of this round has passed.
bool shm_allmax(ShmGroup& g, std::vector<uint64_t>& v) {
  ShmSeg& m = *g.seg;
  const int par = (int)(g.round & 1);
  for (size_t i = 0; i < v.size(); ++i) m.slot[par][g.rank][i] = v[i];
  if (!shm_barrier(g)) return false;
  for (size_t i = 0; i < v.size(); ++i) {
    uint64_t x = 0;
    for (int r = 0; r < g.world; ++r) x = std::max(x, m.slot[par][r][i]);
    v[i] = x;
  }
  return true;
}

// word indices in each arena's 256-byte tail (words 0/1 belong to the
// low-level RD_BLOCK_PUSH protocol, rd_flag_ptr): 4 + side = blocks the
// neighbour on `side` allowed me to write into its ghost rows ("ready"),
// 6 + side = blocks whose rows that neighbour delivered into mine ("landed")
// 8 + side = the create-time self-test of the flag transport (dist_flag_selftest)
constexpr int kWordReady = 4, kWordLanded = 6, kWordTest = 8;

// What a rank publishes about its planes (NCCL rendezvous: all-gathered).
struct DistRec {
  cudaIpcMemHandle_t ipc;
  uint64_t base;  // arena base in the owner's address space
  uint64_t u[2], v[2], phi;
  int64_t rows, stride_bytes, pitch, W, B, arena_bytes;
  int32_t esz, halo;
  int32_t ipc_ok;
  int32_t pad;
};
static_assert(sizeof(DistRec) <= 256, "DistRec");

struct DistState {
  int rank = 0, world = 1;
  bool local = false;
  std::shared_ptr<LocalGroup> lg;
  ShmGroup* sg = nullptr;  // processes of one box without NCCL (rd_dist_shm_id)
  ncclComm_t comm = nullptr;
  bool p2p = true;  // copy-engine push into peer memory; false: NCCL send/recv
  bool flush = false;
  cudaStream_t xs = nullptr;  // exchange stream
  cudaEvent_t ev_start = nullptr, ev_x = nullptr;
  // in-process groups: per-block grant / landed events (ring of 2, see
  // local_sync), recorded by this rank and waited on by its neighbours
  cudaEvent_t ev_grant[2] = {nullptr, nullptr}, ev_land[2] = {nullptr, nullptr};
  uint32_t epoch = 0;  // blocks exchanged (identical on every rank)
  int nb[2] = {-1, -1};  // rank above (side 0) / below (side 1)
  // neighbour planes as pointers valid here (peer mapping)
  struct Nb {
    char* u[2] = {nullptr, nullptr};
    char* v[2] = {nullptr, nullptr};
    char* phi = nullptr;
    uint32_t* words = nullptr;
    int64_t rows = 0, stride_bytes = 0;
  } peer[2];
  std::vector<void*> ipc;  // mappings to close
  uint64_t* d_red = nullptr;  // NCCL reduction scratch (64 x u64)
  int dev = 0;
  int64_t exchanges = 0;
  int selftest = 0;  // dist_flag_selftest: 0 not run (world 1, in-process), 1 passed, -1 failed (NCCL transport)
};

uint32_t* my_words(rd_sim* s) {
  return reinterpret_cast<uint32_t*>(static_cast<char*>(s->arena) + s->arena_bytes - 256);
}

int stream_write32(rd_sim* s, cudaStream_t st, void* flag, uint32_t value) {
  auto fn = reinterpret_cast<PFN_cuStreamWriteValue32_v11070>(driver_entry("cuStreamWriteValue32"));
  if (!fn) return set_err(s, RD_ECUDA, "cuStreamWriteValue32 entry point unavailable");
  if (fn(reinterpret_cast<CUstream>(st), reinterpret_cast<CUdeviceptr>(flag), value, 0) != CUDA_SUCCESS)
    return set_err(s, RD_ECUDA, "cuStreamWriteValue32 failed");
  return RD_OK;
}

int stream_wait32(rd_sim* s, cudaStream_t st, void* flag, uint32_t value, bool flush) {
  auto fn = reinterpret_cast<PFN_cuStreamWaitValue32_v11070>(driver_entry("cuStreamWaitValue32"));
  if (!fn) return set_err(s, RD_ECUDA, "cuStreamWaitValue32 entry point unavailable");
  const unsigned fl = CU_STREAM_WAIT_VALUE_GEQ | (flush ? CU_STREAM_WAIT_VALUE_FLUSH : 0);
  if (fn(reinterpret_cast<CUstream>(st), reinterpret_cast<CUdeviceptr>(flag), value, fl) != CUDA_SUCCESS)
    return set_err(s, RD_ECUDA, "cuStreamWaitValue32 failed");
  return RD_OK;
}

// Element-wise MAX of v over the ranks (collective). MIN of x is ~MAX(~x).
int dist_allmax(rd_sim* s, std::vector<uint64_t>& v) {
  DistState* d = s->dist;
  Range r_("rd_dist.allreduce");
  if (d->local) {
    local_allmax(*d->lg, v);
    return RD_OK;
  }
  if (v.size() > 64) return set_err(s, RD_EINVAL, "reduction too large");
  if (d->sg) {
    if (!shm_allmax(*d->sg, v))
      return set_err(s, RD_ENCCL, "shared-memory group: a rank failed or did not arrive within %.0f s (RD_DIST_TIMEOUT_S)",
                     shm_timeout_s());
    return RD_OK;
  }
  RD_CUDA(s, cudaMemcpyAsync(d->d_red, v.data(), v.size() * 8, cudaMemcpyHostToDevice, s->stream));
  RD_NCCL(s, nccl_api().AllReduce(d->d_red, d->d_red, v.size(), ncclUint64, ncclMax, d->comm, s->stream));
  RD_CUDA(s, cudaMemcpyAsync(v.data(), d->d_red, v.size() * 8, cudaMemcpyDeviceToHost, s->stream));
  RD_CUDA(s, cudaStreamSynchronize(s->stream));
  return RD_OK;
}

int dist_barrier(rd_sim* s) {
  std::vector<uint64_t> v{0};
  return dist_allmax(s, v);
}

// FNV-1a over the control state that decides the launch sequence (and so the
// buffer parity every rank relies on): pending stimuli, latched probes,
// timelapse stride, parameters, depth, step and buffer. Must agree on all
// ranks: stimuli, probes, timelapse and parameters are collective settings.
uint64_t control_digest(const rd_sim* s) {
  uint64_t h = 1469598103934665603ull;
  auto mix = [&](const void* p, size_t n) {
    const unsigned char* c = static_cast<const unsigned char*>(p);
    for (size_t i = 0; i < n; ++i) h = (h ^ c[i]) * 1099511628211ull;
  };
  auto mixv = [&](auto x) { mix(&x, sizeof x); };
  mixv(s->step), mixv(s->cur), mixv(s->K), mixv(s->tl_stride);
  for (const auto& e : s->events) {
    mixv(e.b), mixv(e.at), mixv(e.value), mixv(e.mask_phi);
    mixv(e.shape.kind), mixv(e.shape.dir), mixv(e.shape.cy2), mixv(e.shape.cx2), mixv(e.shape.r);
    mixv(e.shape.y0), mixv(e.shape.x0), mixv(e.shape.y1), mixv(e.shape.x1), mixv(e.shape.mask);
  }
  for (const auto& q : s->probes) mixv(q.b), mixv(q.rect), mixv(q.threshold), mixv(q.stride);
  mixv(s->p);
  for (const auto& p : s->pinst) mixv(p);
  return h;
}

// Whether the block of k steps from the current step is one plain launch:
// k <= depth, no stimulus due in [step, step + k), no probe or timelapse
// sample strictly inside (the rd_step_begin rule).
bool block_plain(const rd_sim* s, int64_t k) {
  if (k > s->K) return false;
  for (const auto& ev : s->events)
    if (ev.at >= s->step && ev.at < s->step + k) return false;
  for (int64_t t = s->step + 1; t < s->step + k; ++t) {
    if (probe_due(s, t)) return false;
    if (s->tl_stride > 0 && t % s->tl_stride == 0) return false;
  }
  return true;
}

// Copies of this rank's send rows (row storage, mirrored columns included)
// of u and v of the current buffer, per instance and side, into the
// neighbour's ghost rows (p2p), or the matching NCCL send/recv group.
int exchange_rows(rd_sim* s, cudaStream_t st) {
  DistState* d = s->dist;
  const size_t row_bytes = (size_t)s->pitch * s->esz, col = (size_t)s->col_off * s->esz;
  const size_t bytes = (size_t)s->halo * row_bytes;
  if (d->p2p) {
    for (int side = 0; side < 2; ++side) {
      if (d->nb[side] < 0) continue;
      const auto& p = d->peer[side];
      const int64_t my_row = side == 0 ? 0 : s->H - s->halo;
      const int64_t its_row = side == 0 ? p.rows : -s->halo;
      for (int64_t b = 0; b < s->B; ++b)
        for (int pl = 0; pl < 2; ++pl) {
          const char* src = plane_ptr(s, pl == 0 ? s->u[s->cur] : s->v[s->cur], b, my_row) - col;
          char* dst = (pl == 0 ? p.u[s->cur] : p.v[s->cur]) + b * p.stride_bytes + its_row * (int64_t)row_bytes -
                      (int64_t)col;
          RD_CUDA(s, cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, st));
        }
    }
    return RD_OK;
  }
  const auto& N = nccl_api();
  RD_NCCL(s, N.GroupStart());
  for (int side = 0; side < 2; ++side) {
    if (d->nb[side] < 0) continue;
    const int64_t send_row = side == 0 ? 0 : s->H - s->halo;
    const int64_t recv_row = side == 0 ? -s->halo : s->H;
    for (int64_t b = 0; b < s->B; ++b)
      for (int pl = 0; pl < 2; ++pl) {
        void* plane = pl == 0 ? s->u[s->cur] : s->v[s->cur];
        RD_NCCL(s, N.Send(plane_ptr(s, plane, b, send_row) - col, bytes, ncclUint8, d->nb[side], d->comm, st));
        RD_NCCL(s, N.Recv(plane_ptr(s, plane, b, recv_row) - col, bytes, ncclUint8, d->nb[side], d->comm, st));
      }
  }
  RD_NCCL(s, N.GroupEnd());
  return RD_OK;
}

// One block of k steps with its halo exchange overlapped with the interior
// rows (header comment, step 2).
// check: the block's launches run the health check (the block precedes a
// stamp or the flag read), else the lean tb_kernel variant.
int dist_block(rd_sim* s, int64_t k, bool check) {
  DistState* d = s->dist;
  s->ghost_valid = (int32_t)s->halo;
  const uint32_t e = ++d->epoch;
  const bool plain = block_plain(s, k);
  const int32_t a = s->top_edge ? 0 : (int32_t)k;
  const int32_t b = (int32_t)s->H - (s->bot_edge ? 0 : (int32_t)k);
  int rc = RD_OK;
  LocalGroup* lg = d->local ? d->lg.get() : nullptr;
  // grant: my current buffer's ghost rows may be overwritten from now on (the
  // launches before this point on my stream -- the previous block, a restore
  // -- are the last to touch them)
  if (lg) {
    RD_CUDA(s, cudaEventRecord(d->ev_grant[e & 1], s->stream));
    local_publish(*lg, lg->granted, d->rank, e);
  } else if (d->p2p) {
    for (int side = 0; side < 2; ++side)
      if (d->nb[side] >= 0 && (rc = stream_write32(s, s->stream, d->peer[side].words + kWordReady + (1 - side), e)))
        return rc;
  }
  RD_CUDA(s, cudaEventRecord(d->ev_start, s->stream));
  s->lean_launch = !check;
  if (plain && a < b && (rc = launch_rows(s, (int)k, s->cur, s->cur ^ 1, a, b))) {
    s->lean_launch = false;
    return rc;
  }
  s->lean_launch = false;
  {
    // the exchange and every wait on another rank live on the exchange
    // stream; the compute stream only waits for its event below
    Range r_("rd_dist.halo_exchange");
    RD_CUDA(s, cudaStreamWaitEvent(d->xs, d->ev_start, 0));
    for (int side = 0; side < 2; ++side) {
      if (d->nb[side] < 0) continue;
      if (lg) {
        local_await(*lg, lg->granted, d->nb[side], e);
        RD_CUDA(s, cudaStreamWaitEvent(d->xs, lg->members[d->nb[side]]->dist->ev_grant[e & 1], 0));
      } else if (d->p2p && (rc = stream_wait32(s, d->xs, my_words(s) + kWordReady + side, e, false))) {
        return rc;
      }
    }
    if ((rc = exchange_rows(s, d->xs))) return rc;
    if (lg) {
      RD_CUDA(s, cudaEventRecord(d->ev_land[e & 1], d->xs));
      local_publish(*lg, lg->landed, d->rank, e);
    } else if (d->p2p) {
      for (int side = 0; side < 2; ++side)
        if (d->nb[side] >= 0 &&
            (rc = stream_write32(s, d->xs, d->peer[side].words + kWordLanded + (1 - side), e)))
          return rc;
    }
    for (int side = 0; side < 2; ++side) {
      if (d->nb[side] < 0) continue;
      if (lg) {
        local_await(*lg, lg->landed, d->nb[side], e);
        RD_CUDA(s, cudaStreamWaitEvent(d->xs, lg->members[d->nb[side]]->dist->ev_land[e & 1], 0));
      } else if (d->p2p && (rc = stream_wait32(s, d->xs, my_words(s) + kWordLanded + side, e, d->flush))) {
        return rc;
      }
    }
    RD_CUDA(s, cudaEventRecord(d->ev_x, d->xs));
    ++d->exchanges;
  }
  // the neighbours' rows have landed in my ghost rows, and my send rows have
  // been read before any later launch overwrites them
  RD_CUDA(s, cudaStreamWaitEvent(s->stream, d->ev_x, 0));
  if (!plain) return run_range(s, s->step + k, s->K);
  int32_t lo, hi;
  block_rows(s, (int)k, &lo, &hi);
  s->lean_launch = !check;
  if (a < b) {
    if (lo < a) rc = launch_rows(s, (int)k, s->cur, s->cur ^ 1, lo, a);
    if (rc == RD_OK && b < hi) rc = launch_rows(s, (int)k, s->cur, s->cur ^ 1, b, hi);
  } else {
    rc = launch_rows(s, (int)k, s->cur, s->cur ^ 1, lo, hi);
  }
  s->lean_launch = false;
  if (rc) return rc;
  if ((rc = end_block(s, (int)k, lo, hi))) return rc;
  s->step += k;
  if (!s->defer_samples && probe_due(s, s->step)) return launch_probes(s, s->step);
  return RD_OK;
}

int dist_run(rd_sim* s, int64_t n) {
  if (int rc = sync_probes(s)) return rc;
  const int64_t end = s->step + n;
  while (s->step < end) {
    const int64_t k = next_k(end - s->step, (int)s->halo);
    bool check = s->step + k >= end;  // the last block before the flag read
    for (const auto& ev : s->events) check = check || ev.at == s->step + k;  // ... or before a stamp
    if (int rc = dist_block(s, k, check)) return rc;
  }
  return RD_OK;
}

// rd_step on a dist handle (header comment, steps 1-4).
int dist_step(rd_sim* s, int64_t n) {
  Range r_("rd_step(dist)");
  const bool ckpt = !(s->g.flags & RD_NO_CHECKPOINT);
  const int64_t step0 = s->step;
  int rc = sync_probes(s);
  if (rc) return rc;
  const uint64_t digest = control_digest(s);
  if (ckpt && (rc = save_checkpoint(s))) return rc;
  if ((rc = dist_run(s, n))) return rc;
  unsigned long long key = ~0ull;
  int precise_hit = 0;
  if ((rc = read_fault(s, &key, &precise_hit))) return rc;
  std::vector<uint64_t> v{(key != ~0ull || precise_hit) ? 1ull : 0ull, digest, ~digest, ~(uint64_t)key};
  if ((rc = dist_allmax(s, v))) return rc;
  if (v[1] != ~v[2])
    return set_err(s, RD_EINVAL,
                   "dist ranks disagree on the control state (stimuli, probes, timelapse, parameters or step must "
                   "be set identically on every rank)");
  if (!v[0]) return RD_OK;
  unsigned long long gkey = ~v[3];
  if (ckpt) {
    Range rr_("rd_step.precise_replay(dist)");
    if ((rc = restore_checkpoint(s))) return rc;
    s->precise_mode = true;
    s->defer_samples = true;
    s->st.replays++;
    gkey = ~0ull;
    while (s->step < step0 + n) {
      if ((rc = dist_run(s, 1)) || (rc = read_fault(s, &key, nullptr))) break;
      std::vector<uint64_t> f{~(uint64_t)key};
      if ((rc = dist_allmax(s, f))) break;
      gkey = ~f[0];  // MIN over ranks: the first non-finite cell in global row-major order
      if (gkey != ~0ull) break;
      if ((rc = sample_step(s))) break;
    }
    s->precise_mode = false;
    s->defer_samples = false;
    if (rc) return rc;
    if (gkey == ~0ull) return RD_OK;
  } else if (gkey == ~0ull) {
    return RD_OK;  // only the division guard tripped: PRECISE kernels already ran
  }
  const unsigned long long W = (unsigned long long)s->W, Hg = (unsigned long long)s->Hg;
  s->fault.step = s->step;
  s->fault.b = (int32_t)(gkey / (W * Hg));
  s->fault.i = (int64_t)((gkey / W) % Hg);
  s->fault.j = (int64_t)(gkey % W);
  reset_fault(s);
  return set_err(s, RD_ENONFINITE, "non-finite value at instance %d, cell (%lld, %lld) after step %lld (dist)",
                 s->fault.b, (long long)s->fault.i, (long long)s->fault.j, (long long)s->fault.step);
}

// Latched probe result over all ranks (collective): the first firing step.
int dist_probe_result(rd_sim* s, int64_t local, int64_t* out) {
  std::vector<uint64_t> v{~(uint64_t)(local < 0 ? INT64_MAX : local)};
  if (int rc = dist_allmax(s, v)) return rc;
  const int64_t m = (int64_t)~v[0];
  *out = m == INT64_MAX ? -1 : m;
  return RD_OK;
}

// Order-preserving map of a double (no NaN) to uint64 for MAX reductions.
uint64_t dbl_key(double x) {
  uint64_t u;
  std::memcpy(&u, &x, 8);
  return (u >> 63) ? ~u : (u | (1ull << 63));
}
double key_dbl(uint64_t k) {
  const uint64_t u = (k >> 63) ? (k & ~(1ull << 63)) : ~k;
  double x;
  std::memcpy(&x, &u, 8);
  return x;
}

// Phi ghost rows once at create (the host map holds owned rows only): the
// same transport as the field exchange, then a barrier.
int exchange_phi(rd_sim* s) {
  DistState* d = s->dist;
  const size_t row_bytes = (size_t)s->pitch * s->esz, col = (size_t)s->col_off * s->esz;
  const size_t bytes = (size_t)s->halo * row_bytes;
  if (d->p2p) {
    for (int side = 0; side < 2; ++side) {
      if (d->nb[side] < 0) continue;
      const auto& p = d->peer[side];
      const int64_t my_row = side == 0 ? 0 : s->H - s->halo;
      const int64_t its_row = side == 0 ? p.rows : -s->halo;
      for (int64_t b = 0; b < s->B; ++b)
        RD_CUDA(s, cudaMemcpyAsync(p.phi + b * p.stride_bytes + its_row * (int64_t)row_bytes - (int64_t)col,
                                   plane_ptr(s, s->phi, b, my_row) - col, bytes, cudaMemcpyDeviceToDevice,
                                   s->stream));
    }
  } else {
    const auto& N = nccl_api();
    RD_NCCL(s, N.GroupStart());
    for (int side = 0; side < 2; ++side) {
      if (d->nb[side] < 0) continue;
      const int64_t send_row = side == 0 ? 0 : s->H - s->halo;
      const int64_t recv_row = side == 0 ? -s->halo : s->H;
      for (int64_t b = 0; b < s->B; ++b) {
        RD_NCCL(s, N.Send(plane_ptr(s, s->phi, b, send_row) - col, bytes, ncclUint8, d->nb[side], d->comm, s->stream));
        RD_NCCL(s, N.Recv(plane_ptr(s, s->phi, b, recv_row) - col, bytes, ncclUint8, d->nb[side], d->comm, s->stream));
      }
    }
    RD_NCCL(s, N.GroupEnd());
  }
  RD_CUDA(s, cudaStreamSynchronize(s->stream));
  if (int rc = dist_barrier(s)) return rc;  // every rank's ghosts have landed
  return launch_mirror(s, s->phi, nullptr, nullptr, s->r_lo, s->r_hi);
}

DistRec make_rec(rd_sim* s, bool ipc) {
  DistRec r;
  std::memset(&r, 0, sizeof r);
  r.ipc_ok = ipc && cudaIpcGetMemHandle(&r.ipc, s->arena) == cudaSuccess;
  if (ipc && !r.ipc_ok) cudaGetLastError();
  r.base = (uint64_t)(uintptr_t)s->arena;
  auto org = [&](void* plane) { return (uint64_t)(uintptr_t)plane_ptr(s, plane, 0, 0); };
  r.u[0] = org(s->u[0]), r.u[1] = org(s->u[1]), r.v[0] = org(s->v[0]), r.v[1] = org(s->v[1]);
  r.phi = org(s->phi);
  r.rows = s->H, r.stride_bytes = s->plane_stride * (int64_t)s->esz, r.pitch = s->pitch, r.W = s->W, r.B = s->B;
  r.esz = (int32_t)s->esz, r.halo = (int32_t)s->halo;
  r.arena_bytes = (int64_t)s->arena_bytes;
  return r;
}

// Register neighbour `side` from its record, with its pointers translated by
// `delta` (mapped base - its base; 0 in one process).
void set_neighbour(DistState* d, int side, const DistRec& r, int64_t delta) {
  auto rel = [&](uint64_t p) { return reinterpret_cast<char*>((int64_t)p + delta); };
  auto& p = d->peer[side];
  p.u[0] = rel(r.u[0]), p.u[1] = rel(r.u[1]), p.v[0] = rel(r.v[0]), p.v[1] = rel(r.v[1]), p.phi = rel(r.phi);
  p.rows = r.rows;
  p.stride_bytes = r.stride_bytes;
  p.words = nullptr;  // set by the caller: the neighbour's arena tail
}

// The block protocol of dist_block rests on two things that only ranks in
// different processes exercise: a stream-ordered 32-bit write into the
// neighbour's IPC-mapped arena, and a stream wait on a word that another
// process (another device) writes. Try both once at create, on words of their
// own, so that a platform without them falls back to NCCL send/recv here
// instead of failing -- or hanging -- inside rd_step. A wait that is not
// satisfied within RD_DIST_SELFTEST_MS (default 5000) is released by writing
// the words from this rank itself.
bool dist_flag_selftest(rd_sim* s) {
  DistState* d = s->dist;
  bool ok = true;
  for (int side = 0; side < 2; ++side)
    if (d->nb[side] >= 0 && ok)
      ok = stream_write32(s, d->xs, d->peer[side].words + kWordTest + (1 - side), 1) == RD_OK;
  for (int side = 0; side < 2; ++side)
    if (d->nb[side] >= 0 && ok) ok = stream_wait32(s, d->xs, my_words(s) + kWordTest + side, 1, d->flush) == RD_OK;
  const char* e = getenv("RD_DIST_SELFTEST_MS");
  const double limit = (e && *e && atof(e) > 0 ? atof(e) : 5000.0) * 1e-3;
  const auto t0 = std::chrono::steady_clock::now();
  cudaError_t q;
  while ((q = cudaStreamQuery(d->xs)) == cudaErrorNotReady &&
         std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() < limit)
    usleep(200);
  if (q == cudaErrorNotReady) {
    ok = false;
    static const uint32_t one = 1;
    for (int side = 0; side < 2; ++side)
      cudaMemcpyAsync(my_words(s) + kWordTest + side, &one, 4, cudaMemcpyHostToDevice, s->stream);
    cudaStreamSynchronize(s->stream);
    q = cudaStreamSynchronize(d->xs);
  }
  if (q != cudaSuccess) {
    cudaGetLastError();
    ok = false;
  }
  if (!ok) s->err.clear();
  return ok;
}

int dist_rendezvous(rd_sim* s) {
  DistState* d = s->dist;
  // (each neighbour's word block sits at the end of ITS arena, whose size
  // follows its own row count)
  bool p2p_ok = true;
  if (d->local) {
    LocalGroup& g = *d->lg;
    {
      std::unique_lock<std::mutex> lk(g.mu);
      g.members[d->rank] = s;
      if (++g.joined == g.world) g.cv.notify_all();
      g.cv.wait(lk, [&] { return g.joined >= g.world; });
    }
    for (int side = 0; side < 2; ++side) {
      if (d->nb[side] < 0) continue;
      rd_sim* o = g.members[d->nb[side]];
      int odev = o->dist->dev;
      if (odev != d->dev) {
        int can = 0;
        cudaDeviceCanAccessPeer(&can, d->dev, odev);
        if (!can) return set_err(s, RD_EINVAL, "in-process dist ranks on devices %d and %d without peer access", d->dev, odev);
        cudaError_t e = cudaDeviceEnablePeerAccess(odev, 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
          return set_err(s, RD_ECUDA, "cudaDeviceEnablePeerAccess: %s", cudaGetErrorString(e));
        cudaGetLastError();
      }
      set_neighbour(d, side, make_rec(o, false), 0);
      d->peer[side].words = my_words(o);
    }
    return RD_OK;
  }
  // all-gather every rank's record (NCCL, or the shared segment), map the
  // neighbours' arenas by IPC
  DistRec mine = make_rec(s, true);
  std::vector<unsigned char> all((size_t)256 * d->world);
  int rc = RD_OK;
  if (d->sg) {
    RD_CUDA(s, cudaStreamSynchronize(s->stream));  // the arena's zero fill, before anyone can write into it
    std::memcpy(d->sg->seg->rec[d->rank], &mine, sizeof mine);
    if ((rc = dist_barrier(s))) return rc;
    std::memcpy(all.data(), d->sg->seg->rec, all.size());
  } else {
    const auto& N = nccl_api();
    void* d_all = nullptr;
    RD_CUDA(s, cudaMalloc(&d_all, (size_t)256 * (d->world + 1)));
    std::vector<unsigned char> tmp(256, 0);
    std::memcpy(tmp.data(), &mine, sizeof mine);
    cudaError_t ce = cudaMemcpyAsync(static_cast<char*>(d_all) + 256 * d->world, tmp.data(), 256,
                                     cudaMemcpyHostToDevice, s->stream);
    ncclResult_t nr = ncclSuccess;
    if (ce == cudaSuccess)
      nr = N.AllGather(static_cast<char*>(d_all) + 256 * d->world, d_all, 256, ncclUint8, d->comm, s->stream);
    if (ce == cudaSuccess && nr == ncclSuccess)
      ce = cudaMemcpyAsync(all.data(), d_all, all.size(), cudaMemcpyDeviceToHost, s->stream);
    if (ce == cudaSuccess) ce = cudaStreamSynchronize(s->stream);
    cudaFree(d_all);
    if (ce != cudaSuccess) return set_err(s, RD_ECUDA, "dist rendezvous: %s", cudaGetErrorString(ce));
    if (nr != ncclSuccess) return set_err(s, RD_ENCCL, "dist rendezvous all-gather: %s", N.GetErrorString(nr));
  }
  const char* tr = getenv("RD_DIST_TRANSPORT");
  if (tr && std::string(tr) == "nccl") p2p_ok = false;
  for (int side = 0; side < 2 && p2p_ok; ++side) {
    if (d->nb[side] < 0) continue;
    DistRec r;
    std::memcpy(&r, all.data() + 256 * d->nb[side], sizeof r);
    void* mapped = nullptr;
    if (!r.ipc_ok || cudaIpcOpenMemHandle(&mapped, r.ipc, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
      cudaGetLastError();
      p2p_ok = false;
      break;
    }
    d->ipc.push_back(mapped);
    set_neighbour(d, side, r, (int64_t)(uintptr_t)mapped - (int64_t)r.base);
    d->peer[side].words = reinterpret_cast<uint32_t*>(static_cast<char*>(mapped) + r.arena_bytes - 256);
  }
  // every rank must use the same transport: first whether all mapped their
  // neighbours, then whether the flag words work between them
  std::vector<uint64_t> v{p2p_ok ? 0ull : 1ull};
  if ((rc = dist_allmax(s, v))) return rc;
  p2p_ok = v[0] == 0;
  if (p2p_ok && d->world > 1) {
    v[0] = dist_flag_selftest(s) ? 0ull : 1ull;
    if ((rc = dist_allmax(s, v))) return rc;
    p2p_ok = v[0] == 0;
    d->selftest = p2p_ok ? 1 : -1;
  }
  d->p2p = p2p_ok;
  if (!d->p2p) {
    for (void* m : d->ipc) cudaIpcCloseMemHandle(m);
    d->ipc.clear();
    if (d->sg)
      return set_err(s, RD_ECUDA,
                     "shared-memory dist group: the peer mapping or its flag words are unavailable (CUDA IPC, "
                     "cuStreamWriteValue32 / cuStreamWaitValue32 across processes) and this group has no NCCL "
                     "fallback; use rd_dist_unique_id");
  }
  return RD_OK;
}

int dist_create(const rd_grid* global, const rd_params* params, const void* phi_rows, int32_t rank, int32_t world,
                const uint8_t id[128], rd_sim** out) {
  if (!out) return set_err(nullptr, RD_EINVAL, "out is NULL");
  *out = nullptr;
  if (!global || !params || !id) return set_err(nullptr, RD_EINVAL, "grid, params and id are required");
  if (world < 1 || rank < 0 || rank >= world) return set_err(nullptr, RD_EINVAL, "rank %d of world %d", rank, world);
  if (global->height < 3 || global->height < world)
    return set_err(nullptr, RD_EINVAL, "height must be >= 3 and >= world (SPEC.md:32)");
  const bool local = std::memcmp(id, kLocalMagic, 8) == 0;
  const bool shm = std::memcmp(id, kShmMagic, 8) == 0;
  if (shm && world > kShmMaxWorld)
    return set_err(nullptr, RD_EINVAL, "a shared-memory group holds at most %d ranks", kShmMaxWorld);
  std::shared_ptr<LocalGroup> lg;
  if (local) {
    uint64_t tok;
    std::memcpy(&tok, id + 8, 8);
    std::lock_guard<std::mutex> lk(g_local_mu);
    auto it = g_local.find(tok);
    if (it == g_local.end()) return set_err(nullptr, RD_EINVAL, "unknown in-process dist id (rd_dist_local_id)");
    lg = it->second;
    std::lock_guard<std::mutex> lk2(lg->mu);
    if (lg->world == 0) {
      lg->world = world;
      lg->members.assign((size_t)world, nullptr);
      lg->granted.assign((size_t)world, 0);
      lg->landed.assign((size_t)world, 0);
    }
    if (lg->world != world) return set_err(nullptr, RD_EINVAL, "world %d differs from the group's %d", world, lg->world);
    if (lg->members[(size_t)rank]) return set_err(nullptr, RD_EINVAL, "rank %d already joined", rank);
  } else if (!shm && !nccl_api().ok) {
    return set_err(nullptr, RD_ENCCL, "%s", nccl_api().why.c_str());
  }
  // rank's rows: the first H % G ranks get one extra row
  const int64_t H = global->height, base = H / world, extra = H % world;
  const int64_t row0 = rank * base + std::min<int64_t>(rank, extra);
  const int64_t rows = base + (rank < extra ? 1 : 0);
  int depth = global->tb_depth;
  if (depth == 0)  // the single-GPU rule on this rank's slab (the ranks' row counts differ by at most one)
    depth = auto_tb_for(global->dtype == RD_F64 ? 8 : 4, true, (int64_t)global->batch * (H / world) * global->width);
  if (world > 1 && rows < depth)
    return set_err(nullptr, RD_EINVAL, "slab of %lld rows is thinner than the halo (%d)", (long long)rows, depth);
  rd_grid g = *global;
  g.height = rows;
  g.tb_depth = depth;
  rd_sim* s = nullptr;
  // phi rows arrive below (owned rows only); create with phi = 0
  if (int rc = create_common(&g, params, nullptr, row0, H, depth, true, &s, nullptr, 0)) return rc;
  auto fail = [&](int rc) {
    std::string m = s->err;
    // a shared-memory group must not wait for a rank that gave up
    if (s->dist && s->dist->sg && s->dist->sg->seg) s->dist->sg->seg->failed.store(1);
    rd_destroy(s);
    return set_err(nullptr, rc, "%s", m.c_str());
  };
  DistState* d = new (std::nothrow) DistState();
  if (!d) return fail(RD_ENOMEM);
  s->dist = d;
  d->rank = rank, d->world = world, d->local = local, d->lg = lg;
  d->nb[0] = rank > 0 ? rank - 1 : -1;
  d->nb[1] = rank < world - 1 ? rank + 1 : -1;
  cudaGetDevice(&d->dev);
  {
    int fl = 0;
    cudaDeviceGetAttribute(&fl, cudaDevAttrCanFlushRemoteWrites, d->dev);
    d->flush = fl != 0;
  }
  if (cudaStreamCreateWithFlags(&d->xs, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&d->ev_start, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&d->ev_x, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&d->ev_grant[0], cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&d->ev_grant[1], cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&d->ev_land[0], cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&d->ev_land[1], cudaEventDisableTiming) != cudaSuccess) {
    cudaGetLastError();
    s->err = "dist streams/events";
    return fail(RD_ECUDA);
  }
  if (shm) {
    // map the segment rd_dist_shm_id made; the first rank in fixes the world
    const std::string name = shm_name(id);
    const int fd = shm_open(name.c_str(), O_RDWR, 0600);
    void* m = fd >= 0 ? mmap(nullptr, sizeof(ShmSeg), PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0) : MAP_FAILED;
    if (fd >= 0) close(fd);
    if (m == MAP_FAILED) {
      s->err = "unknown shared-memory dist id (rd_dist_shm_id; ranks must run on the box that made it)";
      return fail(RD_EINVAL);
    }
    d->sg = new ShmGroup();
    d->sg->seg = static_cast<ShmSeg*>(m);
    d->sg->name = name, d->sg->rank = rank, d->sg->world = world;
    uint32_t w0 = 0;
    if (!d->sg->seg->world.compare_exchange_strong(w0, (uint32_t)world) && w0 != (uint32_t)world) {
      s->err = "world differs from the shared-memory group's";
      return fail(RD_EINVAL);
    }
    // the name is no longer needed once every rank has mapped the segment
    if (d->sg->seg->joined.fetch_add(1) + 1 == (uint32_t)world) shm_unlink(name.c_str());
  } else if (!local) {
    ncclUniqueId uid;
    std::memcpy(uid.internal, id, NCCL_UNIQUE_ID_BYTES);
    ncclResult_t r = nccl_api().CommInitRank(&d->comm, world, uid, rank);
    if (r != ncclSuccess) {
      s->err = std::string("ncclCommInitRank: ") + nccl_api().GetErrorString(r);
      d->comm = nullptr;
      return fail(RD_ENCCL);
    }
    if (cudaMalloc(&d->d_red, 64 * sizeof(uint64_t)) != cudaSuccess) {
      cudaGetLastError();
      s->err = "dist reduction scratch";
      return fail(RD_ENOMEM);
    }
  }
  if (int rc = dist_rendezvous(s)) return fail(rc);
  // owned phi rows from the host, then their ghosts from the neighbours
  for (int64_t b = 0; b < s->B && phi_rows; ++b) {
    const char* src = (const char*)phi_rows + (size_t)b * rows * s->W * s->esz;
    if (cudaMemcpy2DAsync(plane_ptr(s, s->phi, b, 0), s->pitch * s->esz, src, s->W * s->esz, s->W * s->esz, rows,
                          cudaMemcpyHostToDevice, s->stream) != cudaSuccess) {
      cudaGetLastError();
      s->err = "phi upload";
      return fail(RD_ECUDA);
    }
    int bad = 0;
    if (int rc = check_finite_dev(s, plane_ptr(s, s->phi, b, 0), rows, &bad)) return fail(rc);
    if (bad) {
      s->err = "phi_rows contains non-finite values";
      return fail(RD_ENONFINITE);
    }
  }
  if (int rc = exchange_phi(s)) return fail(rc);
  if (cudaStreamSynchronize(s->stream) != cudaSuccess) return fail(RD_ECUDA);
  *out = s;
  return RD_OK;
}

void dist_geometry(const rd_sim* s, rd_geometry* out) {
  if (!s->dist) return;
  out->rank = s->dist->rank;
  out->world = s->dist->world;
  out->phi_rows_lo = 0;  // rd_create_dist takes the owned rows only
  out->phi_rows_hi = s->H;
  out->transport = s->dist->local ? RD_TRANSPORT_LOCAL : (s->dist->p2p ? RD_TRANSPORT_P2P : RD_TRANSPORT_NCCL);
  out->exchanges = s->dist->exchanges;
  out->flag_selftest = s->dist->selftest;
}

// Collective teardown: no rank frees its planes while a neighbour may still
// copy into them or hold them mapped.
void dist_destroy(rd_sim* s) {
  DistState* d = s->dist;
  if (!d) return;
  if (s->stream) cudaStreamSynchronize(s->stream);
  if (d->xs) cudaStreamSynchronize(d->xs);
  for (void* m : d->ipc) cudaIpcCloseMemHandle(m);
  d->ipc.clear();
  const bool joined = d->local ? (d->lg && !d->lg->members.empty() && d->lg->members[d->rank] == s)
                                : (d->sg ? d->sg->seg != nullptr : d->comm != nullptr);
  if (joined && d->world > 1 && !(d->sg && d->sg->seg->failed.load())) dist_barrier(s);
  if (d->comm) nccl_api().CommDestroy(d->comm);
  if (d->sg) {
    if (d->sg->seg) munmap(d->sg->seg, sizeof(ShmSeg));
    delete d->sg;
    d->sg = nullptr;
  }
  if (d->local && d->lg) {
    std::lock_guard<std::mutex> lk(d->lg->mu);
    if (!d->lg->members.empty() && d->lg->members[d->rank] == s && ++d->lg->left == d->lg->world) {
      std::lock_guard<std::mutex> lk2(g_local_mu);
      for (auto it = g_local.begin(); it != g_local.end(); ++it)
        if (it->second == d->lg) {
          g_local.erase(it);
          break;
        }
    }
  }
  if (d->d_red) cudaFree(d->d_red);
  if (d->ev_start) cudaEventDestroy(d->ev_start);
  if (d->ev_x) cudaEventDestroy(d->ev_x);
  for (int i = 0; i < 2; ++i) {
    if (d->ev_grant[i]) cudaEventDestroy(d->ev_grant[i]);
    if (d->ev_land[i]) cudaEventDestroy(d->ev_land[i]);
  }
  if (d->xs) cudaStreamDestroy(d->xs);
  delete d;
  s->dist = nullptr;
}

}  // namespace

extern "C" {

int rd_dist_unique_id(uint8_t id[128]) {
  if (!id) return set_err(nullptr, RD_EINVAL, "id is NULL");
  const auto& N = nccl_api();
  if (!N.ok) return set_err(nullptr, RD_ENCCL, "%s", N.why.c_str());
  ncclUniqueId uid;
  ncclResult_t r = N.GetUniqueId(&uid);
  if (r != ncclSuccess) return set_err(nullptr, RD_ENCCL, "ncclGetUniqueId: %s", N.GetErrorString(r));
  std::memcpy(id, uid.internal, NCCL_UNIQUE_ID_BYTES);
  return RD_OK;
}

int rd_dist_local_id(uint8_t id[128]) {
  if (!id) return set_err(nullptr, RD_EINVAL, "id is NULL");
  static std::atomic<uint64_t> counter{0};
  std::random_device rdev;
  const uint64_t tok = ((uint64_t)rdev() << 32 | rdev()) ^ (++counter * 0x9E3779B97F4A7C15ull);
  std::memset(id, 0, 128);
  std::memcpy(id, kLocalMagic, 8);
  std::memcpy(id + 8, &tok, 8);
  std::lock_guard<std::mutex> lk(g_local_mu);
  g_local[tok] = std::make_shared<LocalGroup>();
  return RD_OK;
}

int rd_dist_shm_id(uint8_t id[128]) {
  if (!id) return set_err(nullptr, RD_EINVAL, "id is NULL");
  static std::atomic<uint64_t> counter{0};
  std::random_device rdev;
  std::memset(id, 0, 128);
  std::memcpy(id, kShmMagic, 8);
  for (int attempt = 0; attempt < 8; ++attempt) {
    const uint64_t tok = ((uint64_t)rdev() << 32 | rdev()) ^ (++counter * 0x9E3779B97F4A7C15ull) ^ (uint64_t)getpid();
    std::memcpy(id + 8, &tok, 8);
    const std::string name = shm_name(id);
    const int fd = shm_open(name.c_str(), O_CREAT | O_EXCL | O_RDWR, 0600);
    if (fd < 0) continue;
    // a fresh segment is zero-filled: every counter of ShmSeg starts at 0
    const bool ok = ftruncate(fd, (off_t)sizeof(ShmSeg)) == 0;
    close(fd);
    if (ok) return RD_OK;
    shm_unlink(name.c_str());
  }
  return set_err(nullptr, RD_ENOMEM, "could not create a POSIX shared-memory segment (/dev/shm)");
}

int rd_create_dist(const rd_grid* global, const rd_params* params, const void* phi_rows, int32_t rank,
                   int32_t world, const uint8_t id[128], rd_sim** out) {
  return dist_create(global, params, phi_rows, rank, world, id, out);
}

}  // extern "C"
