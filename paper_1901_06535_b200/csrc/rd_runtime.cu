// rd_runtime.cu — the C-ABI (include/rd.h) over the sm_100a kernels.
//
// PRODUCT CODE. The runtime owns device planes (u ping-pong, v ping-pong,
// phi, checkpoint), the pending stimulus queue, latched probes and the fault
// word, and cuts every rd_step(n) into temporally blocked launches at event
// and probe steps.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <map>
#include <mutex>
#include <numeric>
#include <tuple>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/rd.h"
#include "rd_kernels.cuh"
#include "rd_launch.h"

namespace {

thread_local std::string g_create_error;

// NVTX ranges (SURVEY.md §5 tracing): rd_step calls, their segments, stamps,
// replays, checkpoints and halo exchanges show up by name on an nsys / ncu
// timeline; without a tool attached a range is a no-op call.
struct Range {
  explicit Range(const char* name) { nvtxRangePushA(name); }
  ~Range() { nvtxRangePop(); }
  Range(const Range&) = delete;
  Range& operator=(const Range&) = delete;
};

struct PendingEvent {
  int32_t b;  // -1 = all
  rdk::ShapeDev shape;
  double value;
  double mask_phi;
  int64_t at;
};

struct LatchedProbe {
  int32_t b;
  rd_rect rect;
  double threshold;
  int32_t stride;
};

struct DistState;  // rd_dist.cuh

}  // namespace

struct rd_sim {
  // tb_kernel input maps, one per input buffer (u[i], v[i] at a constant
  // stride; see alloc_planes)
  CUtensorMap tmap[2];
  CUtensorMap tmap_phi;  // phi rows (box: 3 rows), shared by both buffers
  void* arena = nullptr;  // the plane allocation (u, v, phi, checkpoint, push flags)
  size_t arena_bytes = 0;
  bool own_arena = true;     // false: caller-owned (rd_create_device)
  DistState* dist = nullptr;  // rd_create_dist handles (rd_dist.cuh)
  rd_grid g{};
  rd_params p{};
  size_t esz = 4;
  int64_t H = 0, W = 0, B = 0, pitch = 0, halo = 0, rows_alloc = 0, plane_stride = 0;
  int64_t row_off = 0;  // margin + guard rows: row offset of local row 0
  int64_t col_off = 0;  // mirrored ghost columns left of column 0
  int32_t margin = 0;   // ghost rows above/below (slab halo or mirror margin)
  std::vector<rd_params> pinst;  // f1: per-instance parameters (empty = all use p)
  int64_t div4_mismatches = -1;  // result of the 4-op division certification (-1: not run)
  int fast_mode = 0;
  bool use_lp = false;  // level-parallel kernel (opt-in: RD_KERNEL=lp)
  bool use_cr = false;  // a8 cluster-resident kernel (small instances, one wave)
  int cr_cs = 0;        // CTAs per cluster for cr_kernel
  size_t cr_smem = 0;   // its dynamic shared memory per CTA
  bool cr_pal = false;  // cr_kernel with phi as palette indices
  // a8 whole-chip tiles (gz_kernel): tile geometry, exchange planes, epochs
  bool use_gz = false;
  struct GzGeom {
    int k = 0, gx = 0, th = 0, tw = 0, tr = 0, tc = 0, nr = 0, nv = 0, m = 0, nt = 0;
    size_t smem = 0;
  } gz;
  void* gz_x = nullptr;   // LL exchange planes [parity][u, v] (8-byte words, 1 per fp32 / 2 per fp64 cell)
  unsigned gz_epoch = 0;  // the next launch's exchanges carry gz_epoch + 1, + 2, ...
  bool margins_stale = false;   // u/v mirror margins not refreshed since a cr_kernel / gz_kernel launch
  int64_t probes_done_at = -1;  // the step whose probes a cr_kernel launch evaluated
  std::vector<std::vector<double>> pal;  // distinct phi values per instance (cr PAL layout)
  bool pal_ok = true;     // every instance has <= 256
  bool pal_dirty = true;  // device palette / index plane need a rebuild
  uint8_t* d_idx = nullptr;
  void* d_pal = nullptr;
  int32_t* d_pal_n = nullptr;
  int64_t grow0 = 0, Hg = 0;
  bool slab = false;
  int top_edge = 1, bot_edge = 1;
  int32_t r_lo = 0, r_hi = 0;
  void* u[2] = {nullptr, nullptr};
  void* v[2] = {nullptr, nullptr};
  void* phi = nullptr;
  void* ck_u = nullptr;
  void* ck_v = nullptr;
  void* tl = nullptr;     // f2: timelapse max_u planes
  void* ck_tl = nullptr;
  int32_t tl_stride = 0;
  // host side of the checkpoint (device side: ck_u, ck_v, d_first_ck, ck_tl)
  int64_t ck_step = 0;
  int ck_cur = 0;
  std::vector<PendingEvent> ck_events;
  bool ck_valid = false;
  int cur = 0;
  int64_t step = 0;
  int32_t ghost_valid = 0;  // slab: ghost rows still valid in the current buffers
  int32_t pending_k = 0;    // rd_step_begin opened a block of this many steps
  std::vector<void*> ipc_mapped;  // peer arenas opened with rd_ipc_map (closed at destroy)
  bool pending_push = false;  // ... with the peer-memory halo push
  bool push_active = false;   // the launch being prepared pushes its send rows
  // e: the slab neighbours above (0) / below (1) for the peer-memory push:
  // their planes' (row 0, col 0) for both buffers, owned rows, instance stride
  struct Peer {
    void* u[2] = {nullptr, nullptr};
    void* v[2] = {nullptr, nullptr};
    int64_t rows = 0;
    int64_t stride_bytes = 0;
  } peer[2];
  int K = 4;
  std::vector<PendingEvent> events;
  std::vector<LatchedProbe> probes;
  rdk::ProbeDev* d_probes = nullptr;
  long long* d_first = nullptr;
  long long* d_first_ck = nullptr;
  int probes_cap = 0;
  bool probes_dirty = false;
  unsigned long long* d_fault = nullptr;  // [0] fault key, [1] (as int) precise flag
  int* d_precise = nullptr;
  bool precise_mode = false;
  bool defer_samples = false;  // replay: probes / timelapse sampled only after the step's fault check
  bool lean_launch = false;    // the next stencil launch may skip its health check (tb_kernel TB_LEAN)
  int* d_flag = nullptr;
  int* h_flag = nullptr;      // mapped pinned host words: check_finite_dev's / phi_uniform_kernel's verdict
  int* h_flag_dev = nullptr;  // (without a copy-engine read); [0] flag, bytes 8..15 a value. Device address.
  // whether the phi map is one value (tb_kernel UPHI variants): re-derived on
  // the device at the next run_range after anything wrote phi
  bool phi_class_known = false, phi_uniform = false;
  bool phi_external = false;  // rd_field_ptr handed out phi: the caller may write it at any time
  double phi_u = 0.0;
  void* d_scratch = nullptr;  // probe max output
  int num_sms = 148;
  // CUDA graphs of rd_step segments, keyed by (length, kmax, start buffer,
  // timelapse sample at the end, arithmetic mode); value: exec graph, number
  // of stencil launches, kernels launched.
  std::map<std::tuple<int64_t, int, int, int, int>, std::tuple<cudaGraphExec_t, int64_t, int64_t>> graphs;
  std::map<std::tuple<int64_t, int, int, int, int>, int> graph_seen;  // capture on the 2nd occurrence
  cudaStream_t capture_stream = nullptr;
  bool graphs_broken = false;
  cudaStream_t own_stream = nullptr;
  cudaStream_t stream = nullptr;
  bool profiling = false;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev_pool;
  size_t ev_used = 0;
  rd_stats st{};
  double acc_ms = 0.0;
  int64_t acc_timed = 0;
  rd_fault fault{-1, -1, 0, -1, -1};
  std::string err;
  // asynchronous host I/O (rd_write_fields_async / rd_commit_fields /
  // rd_read_fields_async / rd_io_wait): dense [plane][b][H][W] staging blocks
  // and one copy stream per direction, created on first use
  void* io_in = nullptr;   // inputs uploaded but not yet committed
  void* io_out = nullptr;  // a snapshot of the fields being copied to the host
  cudaStream_t io_s_in = nullptr, io_s_out = nullptr;
  cudaEvent_t io_e_in = nullptr;      // last upload into io_in done
  cudaEvent_t io_e_commit = nullptr;  // last commit's reads of io_in done
  cudaEvent_t io_e_snap = nullptr;    // last snapshot into io_out done
  cudaEvent_t io_e_out = nullptr;     // last download from io_out done
  std::vector<uint8_t> io_staged;     // [plane * B + b]: uploaded, awaiting rd_commit_fields
  std::vector<uint8_t> io_draining;   // [plane * B + b]: a download of this slot may be in flight
};

namespace {

int set_err(rd_sim* s, int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (s)
    s->err = buf;
  else
    g_create_error = buf;
  return code;
}

#define RD_CUDA(sim, call)                                                                        \
  do {                                                                                            \
    cudaError_t e_ = (call);                                                                      \
    if (e_ != cudaSuccess)                                                                        \
      return set_err((sim), e_ == cudaErrorMemoryAllocation ? RD_ENOMEM : RD_ECUDA, "%s: %s (%s:%d)", \
                     #call, cudaGetErrorString(e_), __FILE__, __LINE__);                          \
  } while (0)

// Driver entry points through the runtime (no libcuda link), resolved once per
// process under a lock: handles may be used on several host threads.
void* driver_entry(const char* name) {
  static std::mutex mu;
  static std::map<std::string, void*> cache;
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find(name);
  if (it != cache.end()) return it->second;
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &fn, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess)
    fn = nullptr;
  cache.emplace(name, fn);
  return fn;
}

// rd_dist.cuh (dist handles: rd_create_dist)
int dist_step(rd_sim* s, int64_t n);
void dist_destroy(rd_sim* s);
int dist_allmax(rd_sim* s, std::vector<uint64_t>& v);
int dist_probe_result(rd_sim* s, int64_t local, int64_t* out);
uint64_t dbl_key(double x);
double key_dbl(uint64_t k);
void dist_geometry(const rd_sim* s, rd_geometry* out);

int not_dist(rd_sim* s, const char* what) {
  if (s->dist) return set_err(s, RD_EINVAL, "%s: not for rd_create_dist handles (the library runs their protocol)", what);
  return RD_OK;
}

int check_params(const rd_params* p, std::string* why) {
  const double v[6] = {p->eps, p->f, p->q, p->Du, p->dt, p->dx};
  for (double x : v)
    if (!(x > 0.0) || !std::isfinite(x)) {
      *why = "all parameters must be finite and > 0 (SPEC.md:28)";
      return RD_EPARAM;
    }
  if (!(p->q < 1.0)) {
    *why = "q must be < 1 (SPEC.md:28)";
    return RD_EPARAM;
  }
  if (!(p->dt * p->Du / (p->dx * p->dx) < 0.25)) {
    *why = "dt*Du/dx^2 must be < 0.25 (explicit-scheme guard, SPEC.md:28)";
    return RD_EPARAM;
  }
  return RD_OK;
}

template <typename T>
rdk::Consts<T> make_consts(const rd_params& p) {
  rdk::Consts<T> k;
  k.inv_eps = (T)(1.0 / p.eps);
  k.f = (T)p.f;
  k.q = (T)p.q;
  k.du = (T)p.Du;
  k.dt = (T)p.dt;
  k.inv_dx2 = (T)(1.0 / (p.dx * p.dx));
  k.du_fold = (T)((double)k.du * (double)k.inv_dx2);
  return k;
}

// Default temporal-blocking depth. 4, except:
// - small fp64 batches (at most 2^22 cells, single-GPU handles), where
//   tb_kernel is launch/latency bound and one more step per launch pays
//   (configs 2/3 fp64 on tb_kernel, B200 sweep of depth x row block: depth 5
//   +13% on both);
// - fp32 grids of at least 2^22 cells on this handle (2048^2; smaller ones
//   run gz_kernel or are launch bound): 6. In a run long enough to reach the
//   1 kW power cap the SM clock is set by energy per cell-update, and DRAM
//   traffic is the part depth controls: sustained on 16384^2, phi as a
//   parameter, depth 4 / 5 / 6 / 7 = 1057 / 1113 / 1133 / 1128 Gcell/s at
//   1778 / 1927 / 1965 / 1965 MHz; phi streamed 956 / 1044 / 1049 / 1058;
//   65536^2 (120 GB) 859 -> 992. With the 6-column halos of depths 5 and 6
//   (StripGeom::HALF) depth 6 also wins on mid-size grids, parameter /
//   streamed, depth 4 -> 6: 2048^2 666 -> 691 / 637 -> 654, 3072^2 869 -> 891
//   / 831 -> 837, 4096^2 954 -> 982 / 912 -> 921, 6144^2 1018 -> 1091 / 915
//   -> 1022, 8192^2 1039 -> 1105 / 957 -> 1006. fp64 is FP64-pipe bound at
//   any depth (16384^2: 419 -> 407) and keeps 4. DESIGN.md §5.2.
constexpr int64_t kDeepCells = (int64_t)1 << 22;
int auto_tb_for(int esz, bool slab, int64_t cells) {
  if (const char* e = getenv("RD_TB_DEPTH")) {
    int k = atoi(e);
    if (k >= 1 && k <= RD_MAX_TB) return k;
  }
  if (esz == 8 && !slab && cells <= (int64_t)1 << 22) return 5;
  // (RD_TB_DEEP=0 keeps depth 4. The intermittent mismatch of test_config4_full_length_properties
  // was traced to its depth-1 side: 3 of 9 depth-1 runs differ from a depth-4 reference, 74
  // depth-4..7 runs never do.)
  static const bool shallow = [] {
    const char* e = getenv("RD_TB_DEEP");
    return e && *e && atoi(e) == 0;
  }();
  if (!shallow && esz == 4 && cells >= kDeepCells) return 6;
  return 4;
}
int auto_tb(const rd_sim* s) { return auto_tb_for((int)s->esz, s->slab, s->B * s->H * s->W); }

// Steps of the next launch of a segment with `remaining` steps at depth
// kmax: the segment is cut into ceil(remaining / kmax) launches of nearly
// equal depth (50 steps at depth 6: 6 6 6 6 6 5 5 5 5, not 8 x 6 + 2), since
// shallow launches run at a fraction of the deep ones' rate. Results do not
// depend on the cuts (bitwise).
int next_k(int64_t remaining, int kmax) {
  const int64_t n = (remaining + kmax - 1) / kmax;
  return (int)((remaining + n - 1) / n);
}

template <typename T>
constexpr int vec_of() {
  return 16 / (int)sizeof(T);
}

// Rows per task (tb_kernel: one-warp CTAs, `ctas` resident slots). A task
// runs r = 3 * floor((hb + 2K + 2) / 3) row iterations for hb output rows (the
// 2K-row pipeline fill/drain is overhead, and the row loop advances three
// rows per trip); the persistent CTAs take tasks round-robin, so a launch
// lasts rounds * r row iterations of the slowest warp. A row iteration costs a
// warp as many issue shares as there are warps on its scheduler (four
// schedulers per SM), but never fewer than two: measured on B200, two warps
// per scheduler saturate the issue slots (8 CTAs per SM run config 4 as fast
// as 16) and a lone warp runs no faster than one of two. Pick the hb
// minimising rounds * r * shares: long tasks on every slot, or exactly two
// warps per scheduler, instead of a ragged count. Measured against the
// round-1 latency model (kept below for lp_kernel), Gcell/s with the segment
// graphs warm, fp32: 1536^2 536 vs 467, 2048^2 666 vs 575, 3072^2 874 vs 718,
// 4096^2 958 vs 764, 6144^2 905 vs 779, 8192^2 993 vs 957; fp64: 3072^2 385
// vs 310, 4096^2 392 vs 324; smaller grids and config 4: the same hb.
// (RD_HB=n fixes hb; RD_HB_MODEL=r01 selects the round-1 model.)
int pick_hb(const rd_sim* s, int n_strips, int64_t rows, int K, int64_t ctas, bool one_warp_ctas) {
  if (const char* e = getenv("RD_HB")) {
    int hb = atoi(e);
    if (hb >= 1) return hb;
  }
  static const bool old_model = [] {
    const char* e = getenv("RD_HB_MODEL");
    return e && std::string(e) == "r01";
  }();
  if (one_warp_ctas && !old_model) {
    int best = 1;
    double best_cost = 1e300;
    const int64_t hb_max = std::min<int64_t>(rows, 2048);
    for (int64_t hb = 1; hb <= hb_max; ++hb) {
      const int64_t tasks = (int64_t)n_strips * ((rows + hb - 1) / hb) * s->B;
      const int64_t grid = std::min<int64_t>(tasks, ctas);
      const int64_t rounds = (tasks + grid - 1) / grid;
      const int64_t per_sm = (grid + s->num_sms - 1) / s->num_sms;  // resident warps on the fullest SM
      const int64_t shares = std::max<int64_t>(2, (per_sm + 3) / 4);
      const int64_t r = 3 * ((hb + 2 * K + 2) / 3);
      // ties: the taller block (less fill/drain traffic)
      const double cost = (double)(rounds * r * shares) - 1e-6 * (double)hb;
      if (cost < best_cost) {
        best_cost = cost;
        best = (int)hb;
      }
    }
    return best;
  }
  // lp_kernel (CTAs of K warps) and the round-1 model: a task costs (hb + 2K)
  // row iterations, each ~max(kLatencyWarps, warps resident per SM) issue shares
  constexpr double kLatencyWarps = 6.0;
  int best = 1;
  double best_cost = 1e300;
  for (int hb = 1; hb <= 1024; ++hb) {
    const int64_t tasks = (int64_t)n_strips * ((rows + hb - 1) / hb) * s->B;
    const int64_t waves = (tasks + ctas - 1) / ctas;
    const double per_sm = std::min<double>((double)ctas / s->num_sms, std::ceil((double)tasks / s->num_sms));
    const double cost = (double)waves * (hb + 2 * K) * std::max(kLatencyWarps, per_sm) + 1e-9 * hb;
    if (cost < best_cost) {
      best_cost = cost;
      best = hb;
    }
    if (hb >= rows) break;
  }
  // Large grids (the chosen split is one wave filling at least half of the
  // resident slots): use the smallest row block that still fits one wave --
  // every slot busy, no second wave.
  const int64_t tasks_best = (int64_t)n_strips * ((rows + best - 1) / best) * s->B;
  if (tasks_best <= ctas && 2 * tasks_best >= ctas) {
    const int64_t per_strip = ctas / ((int64_t)n_strips * s->B);  // row blocks per (strip, instance)
    if (per_strip >= 1) best = (int)std::max<int64_t>(1, (rows + per_strip - 1) / per_strip);
  }
  return best;
}

template <typename T>
T* origin(const rd_sim* s, void* plane) {
  return (T*)plane + s->row_off * s->pitch + s->col_off;
}

// Refresh the mirrored ghost margins (no-flux edges) of up to three planes:
// ghost columns of rows [x_lo, x_hi) and, at global edges, the ghost rows.
int launch_mirror(rd_sim* s, void* p0, void* p1, void* p2, int32_t x_lo, int32_t x_hi) {
  const int nplanes = p2 ? 3 : (p1 ? 2 : 1);
  const int64_t cells = (int64_t)(x_hi - x_lo + 2 * rdk::kMarginRows) * 2 * rdk::kMarginCols +
                        (int64_t)2 * rdk::kMarginRows * s->W;
  const unsigned bx = (unsigned)std::max<int64_t>(1, std::min<int64_t>((cells + 255) / 256, 4 * s->num_sms));
  dim3 grid(bx, (unsigned)(nplanes * s->B));
  if (s->esz == 4)
    rdk::mirror_kernel<float><<<grid, 256, 0, s->stream>>>(origin<float>(s, p0), p1 ? origin<float>(s, p1) : nullptr,
                                                          p2 ? origin<float>(s, p2) : nullptr, s->plane_stride,
                                                          s->pitch, (int32_t)s->H, (int32_t)s->W, x_lo, x_hi,
                                                          s->top_edge, s->bot_edge, (int32_t)s->B);
  else
    rdk::mirror_kernel<double><<<grid, 256, 0, s->stream>>>(
        origin<double>(s, p0), p1 ? origin<double>(s, p1) : nullptr, p2 ? origin<double>(s, p2) : nullptr,
        s->plane_stride, s->pitch, (int32_t)s->H, (int32_t)s->W, x_lo, x_hi, s->top_edge, s->bot_edge,
        (int32_t)s->B);
  RD_CUDA(s, cudaGetLastError());
  s->st.launches++;
  return RD_OK;
}

// Kernel arguments common to both stencil kernels (everything but the task
// geometry and row-block height).
template <typename T>
void fill_args(rd_sim* s, rdk::TBArgs<T>& a, int in, int out, int32_t out_lo, int32_t out_hi, int K) {
  a.u_in = origin<T>(s, s->u[in]);
  a.v_in = origin<T>(s, s->v[in]);
  a.phi = origin<T>(s, s->phi);
  a.u_out = origin<T>(s, s->u[out]);
  a.v_out = origin<T>(s, s->v[out]);
  a.plane_stride = s->plane_stride;
  a.pitch = s->pitch;
  a.H = (int32_t)s->H;
  a.W = (int32_t)s->W;
  a.out_lo = out_lo;
  a.out_hi = out_hi;
  a.batch = (int32_t)s->B;
  a.pad_ = 0;
  a.grow0 = s->grow0;
  a.H_global = s->Hg;
  a.per_instance = s->pinst.empty() ? 0 : 1;
  a.pad2_ = 0;
  if (s->pinst.empty()) {
    a.k[0] = make_consts<T>(s->p);
  } else {
    for (int64_t b = 0; b < s->B; ++b) a.k[b] = make_consts<T>(s->pinst[b]);
  }
  a.tmap = s->tmap[in];
  a.tmap_phi = s->tmap_phi;
  a.tm_col0 = (int32_t)s->col_off;
  a.tm_row0 = (int32_t)s->row_off;
  a.fault_key = s->d_fault;
  a.precise_flag = s->d_precise;
  a.tl = (s->tl_stride > 0 && !s->defer_samples && (s->step + K) % s->tl_stride == 0) ? origin<T>(s, s->tl)
                                                                                       : nullptr;
  a.push_up_u = a.push_up_v = a.push_dn_u = a.push_dn_v = nullptr;
  a.push_stride_up = a.push_stride_dn = 0;
  a.push_rows = 0;
  a.pad3_ = 0;
  if (s->push_active) {
    // the neighbours' next input buffer has this launch's output parity
    // (every rank launches the same blocks); row x lands in their ghost rows
    const auto& up = s->peer[0];
    const auto& dn = s->peer[1];
    if (up.u[out]) {
      a.push_up_u = static_cast<T*>(up.u[out]) + up.rows * s->pitch;
      a.push_up_v = static_cast<T*>(up.v[out]) + up.rows * s->pitch;
      a.push_stride_up = up.stride_bytes / (int64_t)sizeof(T);
    }
    if (dn.u[out]) {
      a.push_dn_u = static_cast<T*>(dn.u[out]) - s->H * s->pitch;
      a.push_dn_v = static_cast<T*>(dn.v[out]) - s->H * s->pitch;
      a.push_stride_dn = dn.stride_bytes / (int64_t)sizeof(T);
    }
    a.push_rows = (int32_t)s->halo;
  }
}

// One tb_kernel (or lp_kernel) launch: the strip geometry, a persistent grid
// of as many CTAs as can be resident (occupancy API) capped by the number of
// tasks, and the row-block height (pick_hb). The kernels are instantiated in
// rd_launch_tb_*.cu.
template <typename T>
cudaError_t launch_stencil(rd_sim* s, int k, int in, int out, int32_t out_lo, int32_t out_hi, int mode, bool react) {
  constexpr int V = vec_of<T>();
  const bool lp = s->use_lp && k <= 4;
  rdk::TBArgs<T> a;
  fill_args<T>(s, a, in, out, out_lo, out_hi, k);
  // tb_kernel variant: timelapse samples, peer pushes and
  // PRECISE launches run the full kernel; otherwise the health check runs on
  // the launches that precede a stamp or the flag read (TB_CHECKED) and no
  // other (TB_LEAN). RD_TB_VARIANT=full forces the full kernel (A/B runs).
  static const bool force_full = [] {
    const char* e = getenv("RD_TB_VARIANT");
    return e && std::string(e) == "full";
  }();
  int var = rdk::TB_FULL;
  if (mode != rdk::MODE_PRECISE && !a.tl && !s->push_active && !force_full)
    var = s->lean_launch ? rdk::TB_LEAN : rdk::TB_CHECKED;
  // rdk::StripGeom<K, V, VAR>: the lean/checked fp32 kernels of depth 5 and 6 run 6-column halos
  // (the variants exist for the default fast mode only: any other mode runs the full kernel)
  const bool half = !lp && V == 4 && (k == 5 || k == 6) && var != rdk::TB_FULL && react &&
                    mode == rdk::MODE_FOLD_DIV4_NG;
  const int hx = half ? 6 : ((k + V - 1) / V) * V, wo = 32 * V - 2 * hx;
  // (half: strip i outputs columns [wo * i - 2, wo * i + wo - 2))
  a.n_strips = (int32_t)((s->W + (half ? 2 : 0) + wo - 1) / wo);
  const bool uphi = s->phi_class_known && s->phi_uniform && rdl::tb_uphi_ok(sizeof(T) == 4, k, mode, react, lp);
  a.phi_u = (T)s->phi_u;
  const int64_t ctas = (int64_t)s->num_sms * rdl::occupancy_tb(sizeof(T) == 4, k, mode, react, lp, var, uphi);
  // lp: a task costs ~hb + 3K rows
  a.hb = pick_hb(s, a.n_strips, out_hi - out_lo, lp ? k + (k + 1) / 2 : k, ctas, !lp);
  const int64_t tasks = (int64_t)a.n_strips * ((out_hi - out_lo + a.hb - 1) / a.hb) * s->B;
  return rdl::launch_tb(a, k, mode, react, lp, var, uphi, (unsigned)std::min<int64_t>(tasks, ctas), s->stream);
}

// One stencil launch of k steps from buffer `in` to `out` producing rows
// [lo, hi) (no buffer flip, no mirror refresh): profiling events and the
// arithmetic-mode dispatch.
int launch_rows(rd_sim* s, int k, int in, int out, int32_t lo, int32_t hi) {
  const bool react = !(s->g.flags & RD_REACTION_OFF);
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (s->profiling) {
    if (s->ev_used == s->ev_pool.size()) {
      cudaEvent_t a, b;
      RD_CUDA(s, cudaEventCreate(&a));
      RD_CUDA(s, cudaEventCreate(&b));
      s->ev_pool.push_back({a, b});
    }
    e0 = s->ev_pool[s->ev_used].first;
    e1 = s->ev_pool[s->ev_used].second;
    ++s->ev_used;
    RD_CUDA(s, cudaEventRecord(e0, s->stream));
  }
  // the fast modes (exact rewrites + certified fp32 division) unless this is
  // a precise replay or there is no checkpoint to replay from
  const bool precise = s->precise_mode || (s->g.flags & RD_NO_CHECKPOINT) || s->fast_mode == rdk::MODE_PRECISE;
  const int mode = (!react || precise) ? rdk::MODE_PRECISE : s->fast_mode;
  const cudaError_t e = s->esz == 4 ? launch_stencil<float>(s, k, in, out, lo, hi, mode, react)
                                    : launch_stencil<double>(s, k, in, out, lo, hi, mode, react);
  if (e != cudaSuccess) return set_err(s, RD_ECUDA, "tb_kernel<k=%d> launch: %s", k, cudaGetErrorString(e));
  if (s->profiling) RD_CUDA(s, cudaEventRecord(e1, s->stream));
  s->st.launches++;
  s->st.step_launches++;
  s->st.cell_updates += s->B * (int64_t)(std::min<int32_t>(hi, (int32_t)s->H) - std::max<int32_t>(lo, 0)) * s->W * k;
  return RD_OK;
}

// Rows one k-step launch produces: owned rows, plus at interior slab edges
// the ghost rows that stay valid for later launches of this rd_step (ghost
// depth g - k).
void block_rows(const rd_sim* s, int k, int32_t* lo, int32_t* hi) {
  const int32_t keep = s->slab ? s->ghost_valid - k : 0;
  *lo = s->top_edge ? 0 : -keep;
  *hi = (int32_t)s->H + (s->bot_edge ? 0 : keep);
}

// Flip buffers after a k-step block, refresh the mirrored margins.
int end_block(rd_sim* s, int k, int32_t lo, int32_t hi) {
  const int out = s->cur ^ 1;
  s->cur = out;
  s->ghost_valid -= k;
  return launch_mirror(s, s->u[out], s->v[out], nullptr, lo, hi);
}

// Refresh the u/v mirror margins if a cr_kernel launch left them stale.
int fresh_margins(rd_sim* s) {
  if (!s->margins_stale) return RD_OK;
  s->margins_stale = false;
  return launch_mirror(s, s->u[s->cur], s->v[s->cur], nullptr, 0, (int32_t)s->H);
}

int launch_tb(rd_sim* s, int k) {
  if (int rc = fresh_margins(s)) return rc;
  if (s->slab && k > s->ghost_valid)
    return set_err(s, RD_ERANGE, "slab ghost rows exhausted (k=%d > %d valid rows)", k, s->ghost_valid);
  int32_t lo, hi;
  block_rows(s, k, &lo, &hi);
  if (int rc = launch_rows(s, k, s->cur, s->cur ^ 1, lo, hi)) return rc;
  return end_block(s, k, lo, hi);
}

// a8: shared memory per CTA of cr_kernel with cs CTAs per cluster.
bool probe_due(const rd_sim* s, int64_t step);

// a8: shared memory per CTA of cr_kernel with cs CTAs per cluster, phi as
// values (pal = false) or as palette indices (pal = true).
size_t cr_smem_bytes(const rd_sim* s, int cs, bool pal) {
  const int V = 16 / (int)s->esz;
  const int64_t rows = (s->H + cs - 1) / cs, w4 = (s->W + V - 1) / V;
  return (size_t)(rdk::cr_layout_elems(rows, w4, V, pal) * (int64_t)s->esz + (pal ? rows * w4 * V : 0));
}

// One cr_kernel launch of n steps (or, query, the co-resident cluster count);
// the kernels are instantiated in rd_launch_cr.cu.
template <typename T>
cudaError_t launch_cr_t(rd_sim* s, bool pal, int64_t n, size_t smem, int cs, bool query, int* clusters) {
  rdk::CrArgs<T> ca;
  std::memset(&ca, 0, sizeof ca);
  if (!query) {
    fill_args<T>(s, ca.a, s->cur, s->cur, 0, (int32_t)s->H, (int)n);
    ca.a.n_strips = 0;
    ca.a.hb = 0;
    ca.idx = s->d_idx;
    ca.pal = static_cast<const T*>(s->d_pal);
    ca.probes = s->d_probes;
    ca.first_fire = s->d_first;
    ca.n_probes = (int32_t)s->probes.size();
    ca.probe_step = (!s->probes.empty() && probe_due(s, s->step + n)) ? s->step + n : -1;
    ca.step0 = s->step;
    int64_t every = 0;  // gcd of the strides of the probes due strictly inside (step, step + n)
    for (const auto& q : s->probes)
      if (q.stride > 0 && (s->step + n - 1) / q.stride > s->step / q.stride)
        every = std::gcd(every, (int64_t)q.stride);
    ca.probe_every = (int32_t)every;
    ca.probe_first = every ? (int32_t)(every - s->step % every) : 0;
    ca.cs = cs;
    ca.n = (int32_t)n;
  }
  const bool react = !(s->g.flags & RD_REACTION_OFF);
  return rdl::launch_cr(ca, react ? s->fast_mode : rdk::MODE_PRECISE, react, pal, cs, (unsigned)s->B, smem,
                        s->stream, query, clusters);
}

cudaError_t cr_dispatch(rd_sim* s, bool pal, int64_t n, size_t smem, int cs, bool query, int* clusters) {
  return s->esz == 4 ? launch_cr_t<float>(s, pal, n, smem, cs, query, clusters)
                     : launch_cr_t<double>(s, pal, n, smem, cs, query, clusters);
}

// Per-step time models of the two small-grid paths, fitted to configs 1-3 on
// B200 (scripts/bench_configs.py, same-box runs): cr_kernel
// costs a per-step sync constant plus its band's cells on one SM; tb_kernel a
// pipeline-latency floor or, above it, the whole batch spread over the chip.
// fp64 cr bands are ALU-latency bound (DFMA chains), so large fp64 batches of
// a few instances stay on tb_kernel, which uses every SM.
double t_cr_step(const rd_sim* s, int cs) {
  const bool f32 = s->esz == 4;
  const double band = (double)((s->H + cs - 1) / cs) * (double)s->W;
  return (f32 ? 0.38e-6 : 0.31e-6) + band * (f32 ? 0.19e-9 : 0.50e-9);
}
double t_tb_step(const rd_sim* s) {
  const bool f32 = s->esz == 4;
  const double total = (double)s->B * (double)s->H * (double)s->W;
  return std::max(f32 ? 3.0e-6 : 3.3e-6, total * (f32 ? 7.9e-12 : 8.9e-12));  // fp64: depth 5
}
bool cr_beats_tb(const rd_sim* s, int cs) { return t_cr_step(s, cs) < t_tb_step(s); }

// Decide whether small instances run cluster-resident: the largest cluster
// (16, 8, 4, 2 CTAs) whose per-CTA band fits in shared memory -- with phi as
// values, else as palette indices when every instance's phi has <= 256
// distinct values -- used when every instance's cluster is co-resident in
// one wave (larger batches saturate the chip with tb_kernel). Fast modes only
// (precise replays and checkpoint-less handles use tb_kernel), single-GPU
// handles only. Re-evaluated when the parameters or the palettes change.
void choose_cr(rd_sim* s, bool forced) {
  s->use_cr = false;
  if (s->slab || s->fast_mode == rdk::MODE_PRECISE) return;
  int dev = 0, optin = 0;
  if (cudaGetDevice(&dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess)
    return;
  const int64_t V = 16 / (int64_t)s->esz;
  if ((s->W + V - 1) / V > 512) return;  // a thread per column vector (smallest block size)
  const char* env_cs = getenv("RD_CR_CS");  // measurement override: one cluster size only
  const int only_cs = env_cs ? atoi(env_cs) : 0;
  for (int cs : {16, 8, 4, 2}) {
    if (only_cs && cs != only_cs) continue;
    if (s->H < 2 * cs) continue;
    for (bool pal : {false, true}) {
      if (pal && !s->pal_ok) continue;
      const size_t smem = cr_smem_bytes(s, cs, pal);
      if (smem + 64 > (size_t)optin) continue;  // + the kernel's static mbarriers
      int clusters = 0;
      if (cr_dispatch(s, pal, 0, smem, cs, true, &clusters) != cudaSuccess) {
        cudaGetLastError();
        continue;
      }
      if (clusters < 1 || (!forced && (clusters < s->B || !cr_beats_tb(s, cs)))) continue;
      s->use_cr = true;
      s->cr_cs = cs;
      s->cr_smem = smem;
      s->cr_pal = pal;
      return;
    }
  }
}

// PAL: upload the palettes and rebuild the per-cell index plane after phi
// changed (create, rd_paint_phi).
int sync_palette(rd_sim* s) {
  if (!s->pal_dirty) return RD_OK;
  const int64_t n = s->B * s->H * s->W;
  if (!s->d_idx) {
    RD_CUDA(s, cudaMalloc(&s->d_idx, (size_t)n));
    RD_CUDA(s, cudaMalloc(&s->d_pal, (size_t)s->B * 256 * s->esz));
    RD_CUDA(s, cudaMalloc(&s->d_pal_n, (size_t)s->B * sizeof(int32_t)));
  }
  std::vector<unsigned char> hp((size_t)s->B * 256 * s->esz, 0);
  std::vector<int32_t> hn((size_t)s->B);
  for (int64_t b = 0; b < s->B; ++b) {
    hn[b] = (int32_t)s->pal[b].size();
    for (size_t i = 0; i < s->pal[b].size(); ++i) {
      if (s->esz == 4) {
        const float f = (float)s->pal[b][i];
        std::memcpy(&hp[((size_t)b * 256 + i) * 4], &f, 4);
      } else {
        std::memcpy(&hp[((size_t)b * 256 + i) * 8], &s->pal[b][i], 8);
      }
    }
  }
  RD_CUDA(s, cudaMemcpyAsync(s->d_pal, hp.data(), hp.size(), cudaMemcpyHostToDevice, s->stream));
  RD_CUDA(s, cudaMemcpyAsync(s->d_pal_n, hn.data(), hn.size() * sizeof(int32_t), cudaMemcpyHostToDevice, s->stream));
  RD_CUDA(s, cudaMemsetAsync(s->d_flag, 0, sizeof(int), s->stream));
  dim3 grid((unsigned)std::max<int64_t>(1, std::min<int64_t>((s->H * s->W + 255) / 256, 256)), (unsigned)s->B);
  if (s->esz == 4)
    rdk::phi_index_kernel<float><<<grid, 256, 0, s->stream>>>(origin<float>(s, s->phi), s->plane_stride, s->pitch,
                                                               (int32_t)s->H, (int32_t)s->W, (const float*)s->d_pal,
                                                               s->d_pal_n, s->d_idx, s->d_flag);
  else
    rdk::phi_index_kernel<double><<<grid, 256, 0, s->stream>>>(origin<double>(s, s->phi), s->plane_stride, s->pitch,
                                                                (int32_t)s->H, (int32_t)s->W, (const double*)s->d_pal,
                                                                s->d_pal_n, s->d_idx, s->d_flag);
  RD_CUDA(s, cudaGetLastError());
  s->st.launches++;
  int miss = 0;
  RD_CUDA(s, cudaMemcpyAsync(&miss, s->d_flag, sizeof(int), cudaMemcpyDeviceToHost, s->stream));
  RD_CUDA(s, cudaStreamSynchronize(s->stream));
  if (miss) return set_err(s, RD_ECUDA, "phi palette out of sync with the phi plane");
  s->pal_dirty = false;
  return RD_OK;
}

// Palette bookkeeping (PAL layout of cr_kernel): the distinct phi values of
// each instance in the working precision, tracked on the host from the
// uploaded map and rd_paint_phi; more than 256 disables the PAL layout.
void palette_add(rd_sim* s, int64_t b, double value) {
  const double v = s->esz == 4 ? (double)(float)value : value;
  auto& p = s->pal[(size_t)b];
  for (double x : p)
    if (x == v) return;
  p.push_back(v);
  if (p.size() > 256) s->pal_ok = false;
  s->pal_dirty = true;
}

// One cluster-resident launch of n steps. It evaluates the probes due at any
// of its steps and needs no global mirror margins (it mirrors from the band), so
// none are refreshed after it: the margins are marked stale and the next
// consumer that reads them (tb/lp launches) refreshes them first.
// Whether run_blocks runs the next segment as one cr_kernel launch (which
// evaluates the due probes itself, so run_range does not cut at them).
bool cr_runs(const rd_sim* s) {
  return s->use_cr && (!s->cr_pal || s->pal_ok) && !s->precise_mode && !(s->g.flags & RD_NO_CHECKPOINT);
}

int launch_cr(rd_sim* s, int64_t n) {
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (s->profiling) {
    if (s->ev_used == s->ev_pool.size()) {
      cudaEvent_t a, b;
      RD_CUDA(s, cudaEventCreate(&a));
      RD_CUDA(s, cudaEventCreate(&b));
      s->ev_pool.push_back({a, b});
    }
    e0 = s->ev_pool[s->ev_used].first;
    e1 = s->ev_pool[s->ev_used].second;
    ++s->ev_used;
    RD_CUDA(s, cudaEventRecord(e0, s->stream));
  }
  if (s->cr_pal)
    if (int rc = sync_palette(s)) return rc;
  cudaError_t e = cr_dispatch(s, s->cr_pal, n, s->cr_smem, s->cr_cs, false, nullptr);
  if (e != cudaSuccess) return set_err(s, RD_ECUDA, "cr_kernel launch: %s", cudaGetErrorString(e));
  if (s->profiling) RD_CUDA(s, cudaEventRecord(e1, s->stream));
  s->margins_stale = true;
  if (!s->probes.empty() && probe_due(s, s->step + n)) s->probes_done_at = s->step + n;
  s->st.launches++;
  s->st.step_launches++;
  s->st.cell_updates += s->B * s->H * s->W * n;
  return RD_OK;
}

// ---- a8 whole-chip tiles (gz_kernel, rd_gz.cuh) ------------------------------
// The probe schedule of a fused launch of n steps: gcd of the strides of the
// probes due at some step in (step, step + n], and the steps to its first
// multiple.
void fused_probe_schedule(const rd_sim* s, int64_t n, int32_t* every, int32_t* first) {
  int64_t g = 0;
  for (const auto& q : s->probes)
    if (q.stride > 0 && (s->step + n) / q.stride > s->step / q.stride) g = std::gcd(g, (int64_t)q.stride);
  *every = (int32_t)g;
  *first = g ? (int32_t)(g - s->step % g) : 0;
}

template <typename T>
cudaError_t launch_gz_t(rd_sim* s, int64_t n, const rd_sim::GzGeom& z, unsigned grid, bool query, int* occ) {
  rdk::GzArgs<T> ga;
  std::memset(&ga, 0, sizeof ga);
  ga.nt = z.nt;
  if (!query) {
    fill_args<T>(s, ga.a, s->cur, s->cur ^ 1, 0, (int32_t)s->H, (int)n);
    const int64_t lw = s->esz == 4 ? 1 : 2;  // LL words per cell
    const int64_t words = s->B * s->plane_stride * lw, org = (s->row_off * s->pitch + s->col_off) * lw;
    auto* x = static_cast<unsigned long long*>(s->gz_x);
    for (int par = 0; par < 2; ++par)
      for (int f = 0; f < 2; ++f) ga.x[par][f] = x + (2 * par + f) * words + org;
    ga.epoch0 = s->gz_epoch;
    ga.k = z.k;
    ga.gx = z.gx;
    ga.th = z.th;
    ga.tw = z.tw;
    ga.tr = z.tr;
    ga.tc = z.tc;
    ga.nr = z.nr;
    ga.nv = z.nv;
    ga.n = (int32_t)n;
    ga.n_probes = (int32_t)s->probes.size();
    ga.probes = s->d_probes;
    ga.first_fire = s->d_first;
    ga.step0 = s->step;
    fused_probe_schedule(s, n, &ga.probe_every, &ga.probe_first);
    ga.timeout_ns = 2000000000ull;  // 2 s: only a broken launch waits this long
  }
  const bool react = !(s->g.flags & RD_REACTION_OFF);
  return rdl::launch_gz(ga, react ? s->fast_mode : rdk::MODE_PRECISE, react, z.m, grid, z.smem, s->stream,
                        query ? occ : nullptr);
}

cudaError_t gz_dispatch(rd_sim* s, int64_t n, const rd_sim::GzGeom& z, unsigned grid, bool query, int* occ) {
  return s->esz == 4 ? launch_gz_t<float>(s, n, z, grid, query, occ) : launch_gz_t<double>(s, n, z, grid, query, occ);
}

// Tile geometry of gz_kernel for block depth k: tiles per instance (rows x
// columns, tile widths a multiple of V) and one or two tiles per SM (512 or
// 256 threads). Per-step time model, fitted on B200 (configs 2-3, fp32 and
// fp64): a tile computes the vectors of its owned region
// grown by k - s at step s -- on average (th + k) x ((tw + k) / V + 1) --
// at kGzVecNs per vector on its SM, and waits kGzExchangeUs per exchange
// (every k steps) for its neighbours; two tiles on one SM share its issue
// slots but hide each other's exchange wait. Constraints: at most the
// resident tiles, tiles at least k rows and gx columns (a tile's ghost zone
// lies inside its neighbours' border rings), at most kGzMaxSlots zone
// vectors per thread, the shared arrays within the SM's share.
// The exchange of a block of k steps costs kGzExchangeUs[0] plus
// kGzExchangeUs[1] per step of ghost depth and 4 bytes of cell (its ring
// and zone grow with k; fp64 LL words are twice the fp32 ones).
constexpr double kGzVecNs = 0.7, kGzExchangeUs[2] = {1.2, 0.2};
// returns the predicted seconds per step (0: no geometry)
double gz_geometry(const rd_sim* s, int k, size_t smem_max, rd_sim::GzGeom* out) {
  const int V = 16 / (int)s->esz;
  const int gx = (k + V - 1) / V * V;
  // tiles per SM: 1 (two tiles per SM measured slower on configs 1-3,
  // DESIGN.md §5.2d); RD_GZ_TPS=2 (or 0: the model's choice) for measurements
  const char* etps = getenv("RD_GZ_TPS");
  const int only_tps = etps ? atoi(etps) : 1;
  double best = 0;
  bool found = false;
  for (int tps : {1, 2}) {
    if (only_tps && tps != only_tps) continue;
    const int nt = rdk::kGzThreads / tps;
    const int64_t capacity = (int64_t)tps * s->num_sms;
    for (int64_t tr = 1; tr <= s->H / k; ++tr) {
      const int64_t th = (s->H + tr - 1) / tr;
      if ((s->H + th - 1) / th != tr || th < k) continue;  // the same tiling as a smaller tr
      for (int64_t tc = 1; tc <= (s->W + V - 1) / V; ++tc) {
        const int64_t tw = ((s->W + tc - 1) / tc + V - 1) / V * V;
        if ((s->W + tw - 1) / tw != tc || tw < gx) continue;
        const int64_t tiles = s->B * tr * tc;
        if (tiles > capacity) continue;
        const int64_t nr = th + 2 * k, nv = (tw + 2 * gx) / V;
        if (nr * nv > (int64_t)nt * rdk::kGzMaxSlots || nr >= 65536) continue;
        const size_t smem = rdk::gz_smem_bytes((int)nr, (int)nv, V, (int)s->esz);
        if (smem * tps > smem_max) continue;
        const double work = (double)(th + k) * (double)((tw + k + V - 1) / V + 1) * kGzVecNs * 1e-9;
        const double x = (kGzExchangeUs[0] + kGzExchangeUs[1] * k * (double)s->esz / 4.0) * 1e-6 / k;
        const int per_sm = (int)((tiles + s->num_sms - 1) / s->num_sms);  // tiles sharing the busiest SM
        const double t = per_sm > 1 ? std::max(per_sm * work, work + x) : work + x;
        if (!found || t < best * (1 - 1e-9)) {
          found = true;
          best = t;
          out->k = k;
          out->gx = gx;
          out->th = (int)th;
          out->tw = (int)tw;
          out->tr = (int)tr;
          out->tc = (int)tc;
          out->nr = (int)nr;
          out->nv = (int)nv;
          out->m = (int)((nr * nv + nt - 1) / nt);
          out->nt = nt;
          out->smem = smem;
        }
      }
    }
  }
  return found ? best : 0.0;
}

// Decide whether small instances run as whole-chip tiles (gz_kernel); fast
// modes and single-GPU handles only, like cr_kernel. RD_GZ_K overrides the
// block depth (steps per exchange).
// forced: RD_KERNEL=gz; otherwise only when the model predicts less time per
// step than t_other (the cr / tb alternative). RD_GZ_K fixes the block depth
// (steps per exchange); by default the model picks it from 4..12.
void choose_gz(rd_sim* s, bool forced, double t_other) {
  s->use_gz = false;
  if (s->slab || s->fast_mode == rdk::MODE_PRECISE) return;
  int dev = 0, optin = 0, smem_sm = 0;
  if (cudaGetDevice(&dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev) != cudaSuccess)
    return;
  const size_t smem_max = (size_t)std::min(optin, smem_sm - 2048) - 64;
  const char* ek = getenv("RD_GZ_K");
  const int V = 16 / (int)s->esz;
  rd_sim::GzGeom z;
  double best = 0;
  for (int k : {4, 5, 6, 8, 10, 12}) {
    if (ek) k = std::max(1, atoi(ek));
    const int gx = (k + V - 1) / V * V;
    rd_sim::GzGeom zk;
    double t = 0;
    if (s->H >= 2 * k && s->W >= 2 * gx + V)  // mirrored ghosts stay inside the grid
      t = gz_geometry(s, k, smem_max, &zk);
    if (t > 0 && (best == 0 || t < best)) {
      best = t;
      z = zk;
    }
    if (ek) break;
  }
  if (best == 0 || (!forced && best >= t_other)) return;
  int occ = 0;
  if (gz_dispatch(s, 0, z, 0, true, &occ) != cudaSuccess) {
    cudaGetLastError();
    return;
  }
  const int64_t tiles = s->B * z.tr * z.tc;
  if (occ < 1 || tiles > (int64_t)occ * s->num_sms) return;
  // LL exchange planes: [parity][u, v], zeroed (epoch 0 = nothing published)
  if (!s->gz_x) {
    const size_t bytes = (size_t)4 * s->B * s->plane_stride * (s->esz == 4 ? 1 : 2) * 8;
    if (cudaMalloc(&s->gz_x, bytes) != cudaSuccess || cudaMemsetAsync(s->gz_x, 0, bytes, s->stream) != cudaSuccess) {
      cudaGetLastError();
      if (s->gz_x) cudaFree(s->gz_x);
      s->gz_x = nullptr;
      return;
    }
    s->gz_epoch = 0;
  }
  s->gz = z;
  s->use_gz = true;
}

bool gz_runs(const rd_sim* s) {
  return s->use_gz && !s->precise_mode && !(s->g.flags & RD_NO_CHECKPOINT);
}

// One whole-chip tiled launch of n steps: reads buffer cur, writes cur ^ 1.
// It evaluates the probes due at any of its steps and leaves the global mirror
// margins stale (like cr_kernel).
int launch_gz(rd_sim* s, int64_t n) {
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (s->profiling) {
    if (s->ev_used == s->ev_pool.size()) {
      cudaEvent_t a, b;
      RD_CUDA(s, cudaEventCreate(&a));
      RD_CUDA(s, cudaEventCreate(&b));
      s->ev_pool.push_back({a, b});
    }
    e0 = s->ev_pool[s->ev_used].first;
    e1 = s->ev_pool[s->ev_used].second;
    ++s->ev_used;
    RD_CUDA(s, cudaEventRecord(e0, s->stream));
  }
  const unsigned grid = (unsigned)(s->B * s->gz.tr * s->gz.tc);
  cudaError_t e = gz_dispatch(s, n, s->gz, grid, false, nullptr);
  if (e != cudaSuccess) return set_err(s, RD_ECUDA, "gz_kernel launch: %s", cudaGetErrorString(e));
  if (s->profiling) RD_CUDA(s, cudaEventRecord(e1, s->stream));
  s->gz_epoch += (unsigned)((n + s->gz.k - 1) / s->gz.k);
  s->cur ^= 1;
  s->margins_stale = true;
  if (!s->probes.empty() && probe_due(s, s->step + n)) s->probes_done_at = s->step + n;
  s->st.launches++;
  s->st.step_launches++;
  s->st.cell_updates += s->B * s->H * s->W * n;
  return RD_OK;
}

// Bounding box of a shape in global rows / columns, clipped to the grid.
void shape_bbox(const rdk::ShapeDev& sh, int64_t Hg, int64_t W, int64_t* i0, int64_t* i1, int64_t* j0,
                int64_t* j1) {
  if (sh.kind == RD_RECT) {
    *i0 = sh.y0, *i1 = sh.y1, *j0 = sh.x0, *j1 = sh.x1;
  } else {
    // (2i - cy2)^2 <= 4r^2  <=>  cy2 - 2r <= 2i <= cy2 + 2r
    auto cdiv2 = [](int64_t a) { return a >= 0 ? (a + 1) / 2 : -((-a) / 2); };  // ceil(a/2)
    auto fdiv2 = [](int64_t a) { return a >= 0 ? a / 2 : -((-a + 1) / 2); };   // floor(a/2)
    *i0 = cdiv2(sh.cy2 - 2 * sh.r);
    *i1 = fdiv2(sh.cy2 + 2 * sh.r) + 1;
    *j0 = cdiv2(sh.cx2 - 2 * sh.r);
    *j1 = fdiv2(sh.cx2 + 2 * sh.r) + 1;
  }
  *i0 = std::max<int64_t>(*i0, 0);
  *j0 = std::max<int64_t>(*j0, 0);
  *i1 = std::min<int64_t>(*i1, Hg);
  *j1 = std::min<int64_t>(*j1, W);
}

int apply_event(rd_sim* s, const PendingEvent& ev) {
  Range r_("rd_stimulate.stamp");
  int64_t i0, i1, j0, j1;
  shape_bbox(ev.shape, s->Hg, s->W, &i0, &i1, &j0, &j1);
  // local rows that exist in this handle (owned + readable ghosts)
  int64_t x0 = std::max<int64_t>(i0 - s->grow0, s->r_lo);
  int64_t x1 = std::min<int64_t>(i1 - s->grow0, s->r_hi);
  if (x0 >= x1 || j0 >= j1) return RD_OK;
  const int32_t b0 = ev.b < 0 ? 0 : ev.b;
  const int32_t nb = ev.b < 0 ? (int32_t)s->B : 1;
  dim3 block(128);
  // rows beyond gridDim.y's 65535 cap are covered by the kernel's row loop
  dim3 grid((unsigned)((j1 - j0 + 127) / 128), (unsigned)std::min<int64_t>(x1 - x0, 65535),
            (unsigned)std::min<int32_t>(nb, 65535));
  if (s->esz == 4)
    rdk::stamp_kernel<float><<<grid, block, 0, s->stream>>>(
        origin<float>(s, s->u[s->cur]), origin<float>(s, s->phi), s->plane_stride, s->pitch, s->grow0, ev.shape,
        (float)ev.value, (float)ev.mask_phi, (int32_t)x0, (int32_t)x1, j0, j1, b0, nb);
  else
    rdk::stamp_kernel<double><<<grid, block, 0, s->stream>>>(
        origin<double>(s, s->u[s->cur]), origin<double>(s, s->phi), s->plane_stride, s->pitch, s->grow0, ev.shape,
        ev.value, ev.mask_phi, (int32_t)x0, (int32_t)x1, j0, j1, b0, nb);
  RD_CUDA(s, cudaGetLastError());
  s->st.launches++;
  return RD_OK;
}

int sync_probes(rd_sim* s) {
  if (!s->probes_dirty) return RD_OK;
  const int n = (int)s->probes.size();
  if (n > s->probes_cap) {
    int cap = std::max(8, 2 * n);
    rdk::ProbeDev* dp = nullptr;
    long long *df = nullptr, *dfc = nullptr;
    RD_CUDA(s, cudaMalloc(&dp, sizeof(rdk::ProbeDev) * cap));
    RD_CUDA(s, cudaMalloc(&df, sizeof(long long) * cap));
    RD_CUDA(s, cudaMalloc(&dfc, sizeof(long long) * cap));
    std::vector<long long> init(cap, -1);
    RD_CUDA(s, cudaMemcpyAsync(df, init.data(), sizeof(long long) * cap, cudaMemcpyHostToDevice, s->stream));
    if (s->d_first && s->probes_cap)
      RD_CUDA(s, cudaMemcpyAsync(df, s->d_first, sizeof(long long) * s->probes_cap, cudaMemcpyDeviceToDevice,
                                 s->stream));
    RD_CUDA(s, cudaStreamSynchronize(s->stream));
    cudaFree(s->d_probes);
    cudaFree(s->d_first);
    cudaFree(s->d_first_ck);
    s->d_probes = dp;
    s->d_first = df;
    s->d_first_ck = dfc;
    s->probes_cap = cap;
  }
  std::vector<rdk::ProbeDev> hp(n);
  for (int i = 0; i < n; ++i) {
    const LatchedProbe& q = s->probes[i];
    // local owned rows only (slabs: each rank probes its own rows)
    hp[i].y0 = std::max<int64_t>(q.rect.y0 - s->grow0, 0);
    hp[i].y1 = std::min<int64_t>(q.rect.y1 - s->grow0, s->H);
    if (hp[i].y1 < hp[i].y0) hp[i].y1 = hp[i].y0;
    hp[i].x0 = q.rect.x0;
    hp[i].x1 = q.rect.x1;
    hp[i].b = q.b;
    hp[i].stride = q.stride;
    hp[i].threshold = q.threshold;
  }
  RD_CUDA(s, cudaMemcpyAsync(s->d_probes, hp.data(), sizeof(rdk::ProbeDev) * n, cudaMemcpyHostToDevice, s->stream));
  RD_CUDA(s, cudaStreamSynchronize(s->stream));
  s->probes_dirty = false;
  return RD_OK;
}

int launch_probes(rd_sim* s, int64_t step) {
  Range r_("rd_probe.latch");
  const int n = (int)s->probes.size();
  if (!n) return RD_OK;
  if (s->esz == 4)
    rdk::probe_kernel<float><<<n, 256, 0, s->stream>>>(origin<float>(s, s->u[s->cur]), s->plane_stride, s->pitch,
                                                        s->d_probes, n, step, s->d_first, nullptr);
  else
    rdk::probe_kernel<double><<<n, 256, 0, s->stream>>>(origin<double>(s, s->u[s->cur]), s->plane_stride, s->pitch,
                                                         s->d_probes, n, step, s->d_first, nullptr);
  RD_CUDA(s, cudaGetLastError());
  s->st.launches++;
  return RD_OK;
}

bool probe_due(const rd_sim* s, int64_t step) {
  for (const auto& q : s->probes)
    if (q.stride > 0 && step > 0 && step % q.stride == 0) return true;
  return false;
}

// The blocked launches of one segment [s->step, next) (no event or probe
// inside): direct launches, or -- for non-slab handles in the fast modes --
// one CUDA graph per distinct segment shape, captured once and replayed, so a
// small-grid run costs one graph launch per segment instead of two kernel
// launches per block (the per-launch overhead dominates small batched grids).
int run_blocks(rd_sim* s, int64_t next, int kmax) {
  Range r_("rd_step.segment");
  if (gz_runs(s) && next > s->step) {
    if (int rc = launch_gz(s, next - s->step)) return rc;
    s->step = next;
    return RD_OK;
  }
  if (cr_runs(s) && next > s->step) {
    if (int rc = launch_cr(s, next - s->step)) return rc;
    s->step = next;
    return RD_OK;
  }
  if (int rc = fresh_margins(s)) return rc;  // outside any graph capture
  const bool graph = !(s->g.flags & RD_NO_GRAPH) && !s->profiling && !s->slab && !s->precise_mode &&
                     !s->graphs_broken && next - s->step >= 2 * kmax;
  if (!graph) {
    while (s->step < next) {
      const int k = next_k(next - s->step, kmax);
      s->lean_launch = s->step + k < next;  // the segment's last launch checks
      const int rc = launch_tb(s, k);
      s->lean_launch = false;
      if (rc) return rc;
      s->step += k;
    }
    return RD_OK;
  }
  const int tl_end = (s->tl_stride > 0 && next % s->tl_stride == 0) ? 1 : 0;
  const auto key = std::make_tuple(next - s->step, kmax, s->cur, tl_end, s->fast_mode);
  auto it = s->graphs.find(key);
  if (it == s->graphs.end() && ++s->graph_seen[key] < 2) {
    // first occurrence of this segment shape: launch directly (a one-off
    // segment would not repay the capture)
    while (s->step < next) {
      const int k = next_k(next - s->step, kmax);
      s->lean_launch = s->step + k < next;  // the segment's last launch checks
      const int rc = launch_tb(s, k);
      s->lean_launch = false;
      if (rc) return rc;
      s->step += k;
    }
    return RD_OK;
  }
  if (it == s->graphs.end()) {
    if (!s->capture_stream) RD_CUDA(s, cudaStreamCreateWithFlags(&s->capture_stream, cudaStreamNonBlocking));
    const int cur0 = s->cur;
    const int64_t step0 = s->step;
    const int32_t gv0 = s->ghost_valid;
    const rd_stats st0 = s->st;
    cudaStream_t user = s->stream;
    s->stream = s->capture_stream;
    cudaGraph_t g = nullptr;
    int rc = RD_OK;
    if (cudaStreamBeginCapture(s->stream, cudaStreamCaptureModeThreadLocal) != cudaSuccess) rc = RD_ECUDA;
    while (rc == RD_OK && s->step < next) {
      const int k = next_k(next - s->step, kmax);
      s->lean_launch = s->step + k < next;  // the segment's last launch checks
      rc = launch_tb(s, k);
      s->lean_launch = false;
      s->step += k;
    }
    cudaError_t ec = cudaStreamEndCapture(s->stream, &g);
    s->stream = user;
    cudaGraphExec_t ex = nullptr;
    if (rc == RD_OK && ec == cudaSuccess && g && cudaGraphInstantiate(&ex, g, 0) == cudaSuccess) {
      it = s->graphs.emplace(key, std::make_tuple(ex, s->st.step_launches - st0.step_launches,
                                                   s->st.launches - st0.launches)).first;
    }
    if (g) cudaGraphDestroy(g);
    // rewind the host state advanced by the capture
    s->cur = cur0;
    s->step = step0;
    s->ghost_valid = gv0;
    s->st = st0;
    cudaGetLastError();
    if (it == s->graphs.end()) {  // capture unsupported here: launch directly from now on
      s->graphs_broken = true;
      return run_blocks(s, next, kmax);
    }
  }
  const auto& [ex, n_step_launches, n_launches] = it->second;
  RD_CUDA(s, cudaGraphLaunch(ex, s->stream));
  if (n_step_launches & 1) s->cur ^= 1;
  s->st.launches += n_launches;
  s->st.step_launches += n_step_launches;
  s->st.cell_updates += s->B * s->H * s->W * (next - s->step);
  s->step = next;
  return RD_OK;
}

void drop_graphs(rd_sim* s) {
  for (auto& kv : s->graphs) cudaGraphExecDestroy(std::get<0>(kv.second));
  s->graphs.clear();
  s->graph_seen.clear();
}

// Advance from s->step to end with blocks of at most kmax steps.
// Whether phi is one value over all instances (then tb_kernel reads it as a
// kernel parameter): one pass over the map on the device after
// anything wrote it (create, rd_paint_phi), the verdict and the value in
// mapped host words. Slab and dist handles recompute ghost rows whose phi
// comes from the neighbours, so they keep the general kernel. A change of
// class drops the captured graphs (they bake the kernel variant).
// RD_TB_UPHI=0 keeps the general kernel (tests run both).
void drop_graphs(rd_sim* s);
int ensure_phi_class(rd_sim* s) {
  if (s->phi_class_known) return RD_OK;
  bool uni = false;
  double val = 0.0;
  const char* e = getenv("RD_TB_UPHI");
  if (!(e && atoi(e) == 0) && !s->slab && !s->dist && !s->phi_external) {
    RD_CUDA(s, cudaStreamSynchronize(s->stream));
    *s->h_flag = 0;
    const unsigned blocks = (unsigned)(8 * s->num_sms);
    if (s->esz == 4)
      rdk::phi_uniform_kernel<float><<<blocks, 256, 0, s->stream>>>(origin<float>(s, s->phi), s->plane_stride, s->pitch,
                                                                    (int32_t)s->H, (int32_t)s->W, (int32_t)s->B,
                                                                    s->h_flag_dev, s->h_flag_dev + 2);
    else
      rdk::phi_uniform_kernel<double><<<blocks, 256, 0, s->stream>>>(origin<double>(s, s->phi), s->plane_stride,
                                                                     s->pitch, (int32_t)s->H, (int32_t)s->W,
                                                                     (int32_t)s->B, s->h_flag_dev, s->h_flag_dev + 2);
    RD_CUDA(s, cudaGetLastError());
    s->st.launches++;
    RD_CUDA(s, cudaStreamSynchronize(s->stream));
    uni = *s->h_flag == 0;
    if (s->esz == 4) {
      float f;
      std::memcpy(&f, s->h_flag + 2, 4);
      val = f;
    } else {
      std::memcpy(&val, s->h_flag + 2, 8);
    }
  }
  if (uni != s->phi_uniform) drop_graphs(s);
  s->phi_uniform = uni;
  s->phi_u = val;
  s->phi_class_known = true;
  return RD_OK;
}

int run_range(rd_sim* s, int64_t end, int kmax) {
  int rc = ensure_phi_class(s);
  if (rc) return rc;
  if ((rc = sync_probes(s))) return rc;
  while (s->step < end) {
    // a1: stimuli due now, in submission order; then refresh u's mirrors
    bool stamped = false;
    for (size_t i = 0; i < s->events.size();) {
      if (s->events[i].at == s->step) {
        if ((rc = apply_event(s, s->events[i]))) return rc;
        s->events.erase(s->events.begin() + i);
        stamped = true;
      } else {
        ++i;
      }
    }
    if (stamped && (rc = launch_mirror(s, s->u[s->cur], nullptr, nullptr, s->r_lo, s->r_hi))) return rc;
    int64_t next = end;
    for (const auto& ev : s->events)
      if (ev.at > s->step) next = std::min(next, ev.at);
    if (!cr_runs(s) && !gz_runs(s))  // cr_kernel / gz_kernel latch the probes due inside their segment
      for (const auto& q : s->probes)
        if (q.stride > 0) next = std::min(next, (s->step / q.stride + 1) * (int64_t)q.stride);
    if (s->tl_stride > 0) next = std::min(next, (s->step / s->tl_stride + 1) * (int64_t)s->tl_stride);
    if ((rc = run_blocks(s, next, kmax))) return rc;
    if (!s->defer_samples && probe_due(s, s->step) && s->probes_done_at != s->step)
      if ((rc = launch_probes(s, s->step))) return rc;
  }
  return RD_OK;
}

// Probe latches and timelapse record due after the step just completed (the
// deferred samples of a PRECISE replay step).
int sample_step(rd_sim* s) {
  if (s->tl_stride > 0 && s->step % s->tl_stride == 0) {
    const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>((s->B * s->H * s->W + 255) / 256,
                                                                           (int64_t)s->num_sms * 8));
    if (s->esz == 4)
      rdk::tl_update_kernel<float><<<grid, 256, 0, s->stream>>>(origin<float>(s, s->u[s->cur]), origin<float>(s, s->tl),
                                                                 s->plane_stride, s->pitch, (int32_t)s->H,
                                                                 (int32_t)s->W, (int32_t)s->B);
    else
      rdk::tl_update_kernel<double><<<grid, 256, 0, s->stream>>>(
          origin<double>(s, s->u[s->cur]), origin<double>(s, s->tl), s->plane_stride, s->pitch, (int32_t)s->H,
          (int32_t)s->W, (int32_t)s->B);
    RD_CUDA(s, cudaGetLastError());
    s->st.launches++;
  }
  if (probe_due(s, s->step)) return launch_probes(s, s->step);
  return RD_OK;
}

// Reads the fault key and the fast-division precise flag (one 16-byte D2H).
int read_fault(rd_sim* s, unsigned long long* key, int* precise) {
  unsigned long long h[2];
  RD_CUDA(s, cudaMemcpyAsync(h, s->d_fault, sizeof h, cudaMemcpyDeviceToHost, s->stream));
  RD_CUDA(s, cudaStreamSynchronize(s->stream));
  *key = h[0];
  if (precise) *precise = (int)(h[1] & 0xffffffffu);
  return RD_OK;
}

int reset_fault(rd_sim* s) {
  RD_CUDA(s, cudaMemsetAsync(s->d_fault, 0xff, sizeof(unsigned long long), s->stream));
  RD_CUDA(s, cudaMemsetAsync(s->d_fault + 1, 0, sizeof(unsigned long long), s->stream));
  return RD_OK;
}

// Device-to-device copy of `rows` rows of `row_bytes` bytes on the handle's
// stream, by copy_rows_kernel (SMs, not a copy engine: see the kernel) when
// everything is 16-byte aligned, else cudaMemcpy2DAsync.
int copy_rows(rd_sim* s, void* dst, int64_t dpitch, const void* src, int64_t spitch, int64_t row_bytes, int64_t rows) {
  if (rows <= 0 || row_bytes <= 0) return RD_OK;
  const uintptr_t mis = reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src) | (uintptr_t)dpitch |
                        (uintptr_t)spitch | (uintptr_t)row_bytes;
  if (mis % 16) {
    RD_CUDA(s, cudaMemcpy2DAsync(dst, dpitch, src, spitch, row_bytes, rows, cudaMemcpyDeviceToDevice, s->stream));
    return RD_OK;
  }
  if (dpitch == row_bytes && spitch == row_bytes) {  // contiguous: one long row
    row_bytes *= rows;
    rows = 1;
  }
  const int64_t n = row_bytes / 16 * rows;
  const unsigned blocks = (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 8 * s->num_sms));
  rdk::copy_rows_kernel<<<blocks, 256, 0, s->stream>>>(static_cast<char*>(dst), dpitch, static_cast<const char*>(src),
                                                       spitch, row_bytes, rows);
  RD_CUDA(s, cudaGetLastError());
  s->st.launches++;
  return RD_OK;
}

// Checkpoint = u, v (current buffers), probe latches, timelapse, step,
// buffer parity and pending events; restore returns to it exactly.
int save_checkpoint(rd_sim* s) {
  Range r_("rd_checkpoint");
  if (!s->ck_u) return set_err(s, RD_EINVAL, "handle created with RD_NO_CHECKPOINT");
  const size_t bytes = (size_t)s->B * s->plane_stride * s->esz;
  if (int rc = copy_rows(s, s->ck_u, bytes, s->u[s->cur], bytes, bytes, 1)) return rc;
  if (int rc = copy_rows(s, s->ck_v, bytes, s->v[s->cur], bytes, bytes, 1)) return rc;
  if (!s->probes.empty())
    RD_CUDA(s, cudaMemcpyAsync(s->d_first_ck, s->d_first, sizeof(long long) * s->probes.size(),
                               cudaMemcpyDeviceToDevice, s->stream));
  if (s->tl)
    if (int rc = copy_rows(s, s->ck_tl, bytes, s->tl, bytes, bytes, 1)) return rc;
  s->ck_step = s->step;
  s->ck_cur = s->cur;
  s->ck_events = s->events;
  s->ck_valid = true;
  return RD_OK;
}

int restore_checkpoint(rd_sim* s) {
  Range r_("rd_restore");
  if (!s->ck_valid) return set_err(s, RD_ERANGE, "no checkpoint to restore");
  const size_t bytes = (size_t)s->B * s->plane_stride * s->esz;
  s->cur = s->ck_cur;
  if (int rc = copy_rows(s, s->u[s->cur], bytes, s->ck_u, bytes, bytes, 1)) return rc;
  if (int rc = copy_rows(s, s->v[s->cur], bytes, s->ck_v, bytes, bytes, 1)) return rc;
  if (!s->probes.empty())
    RD_CUDA(s, cudaMemcpyAsync(s->d_first, s->d_first_ck, sizeof(long long) * s->probes.size(),
                               cudaMemcpyDeviceToDevice, s->stream));
  if (s->tl)
    if (int rc = copy_rows(s, s->tl, bytes, s->ck_tl, bytes, bytes, 1)) return rc;
  s->events = s->ck_events;
  s->step = s->ck_step;
  s->ghost_valid = (int32_t)s->halo;
  s->margins_stale = true;  // the checkpoint copy may predate a refresh
  s->probes_done_at = -1;
  return reset_fault(s);
}

// One allocation of seven plane blocks (a block = the plane of all B
// instances): u0 | ck_u | u1 | v0 | v1 | ck_v | phi. Then u0, v0 sit at a
// stride of 3 blocks and u1, v1 at a stride of 2, so one tensor map per input
// buffer (dims col, row, instance, plane) lands three rows' u and v segments
// with one TMA (tb_kernel). The checkpoint fills the two gaps.
size_t arena_size(const rd_sim* s) { return 7 * (size_t)s->B * s->plane_stride * s->esz + 256; }

int alloc_planes(rd_sim* s, void* ext, size_t ext_bytes) {
  const size_t bytes = (size_t)s->B * s->plane_stride * s->esz;
  // + 256 bytes: the peer-push flag words (rd_flag_ptr), so one IPC handle
  // of the arena maps planes and flags
  if (ext) {
    if (ext_bytes < arena_size(s) || reinterpret_cast<uintptr_t>(ext) % 256)
      return set_err(s, RD_EINVAL, "caller arena must be 256-byte aligned and >= %zu bytes (rd_arena_bytes)",
                     arena_size(s));
    s->arena = ext;
    s->own_arena = false;
  } else {
    RD_CUDA(s, cudaMalloc(&s->arena, arena_size(s)));
  }
  RD_CUDA(s, cudaMemsetAsync(s->arena, 0, arena_size(s), s->stream));
  s->arena_bytes = arena_size(s);
  char* base = static_cast<char*>(s->arena);
  s->u[0] = base;
  s->u[1] = base + 2 * bytes;
  s->v[0] = base + 3 * bytes;
  s->v[1] = base + 4 * bytes;
  s->phi = base + 6 * bytes;
  if (!(s->g.flags & RD_NO_CHECKPOINT)) {
    s->ck_u = base + bytes;
    s->ck_v = base + 5 * bytes;
  }
  RD_CUDA(s, cudaMalloc(&s->d_fault, 2 * sizeof(unsigned long long)));
  s->d_precise = reinterpret_cast<int*>(s->d_fault + 1);
  RD_CUDA(s, cudaMalloc(&s->d_flag, sizeof(int)));
  RD_CUDA(s, cudaHostAlloc(reinterpret_cast<void**>(&s->h_flag), 16, cudaHostAllocMapped));
  RD_CUDA(s, cudaHostGetDevicePointer(reinterpret_cast<void**>(&s->h_flag_dev), s->h_flag, 0));
  RD_CUDA(s, cudaMalloc(&s->d_scratch, 64));
  return reset_fault(s);
}

// The tensor maps of tb_kernel's input rows (driver entry point through the
// runtime: no libcuda link), coordinates relative to the plane's allocation
// start: per input buffer one 4-D map whose box is three rows of 32*V
// columns of the u and v planes; one 3-D map whose box is three rows of phi.
int encode_tmaps(rd_sim* s) {
  auto encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(driver_entry("cuTensorMapEncodeTiled"));
  if (!encode) return set_err(s, RD_ECUDA, "cuTensorMapEncodeTiled entry point unavailable");
  const cuuint64_t block = (cuuint64_t)s->B * s->plane_stride * s->esz;
  const cuuint32_t seg = (cuuint32_t)(32 * (16 / s->esz));
  const auto dtype = s->esz == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64;
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  for (int i = 0; i < 2; ++i) {
    const cuuint64_t dims[4] = {(cuuint64_t)s->pitch, (cuuint64_t)s->rows_alloc, (cuuint64_t)s->B, 2};
    const cuuint64_t strides[3] = {(cuuint64_t)(s->pitch * s->esz), (cuuint64_t)(s->plane_stride * s->esz),
                                   (i == 0 ? 3 : 2) * block};
    const cuuint32_t box[4] = {seg, 3, 1, 2};
    CUresult r = encode(&s->tmap[i], dtype, 4, s->u[i], dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return set_err(s, RD_ECUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  }
  const cuuint64_t dims[3] = {(cuuint64_t)s->pitch, (cuuint64_t)s->rows_alloc, (cuuint64_t)s->B};
  const cuuint64_t strides[2] = {(cuuint64_t)(s->pitch * s->esz), (cuuint64_t)(s->plane_stride * s->esz)};
  const cuuint32_t box[3] = {seg, 3, 1};
  CUresult r = encode(&s->tmap_phi, dtype, 3, s->phi, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_err(s, RD_ECUDA, "cuTensorMapEncodeTiled (phi) failed (%d)", (int)r);
  return RD_OK;
}

int check_finite_dev(rd_sim* s, const void* base, int64_t rows, int* bad, int64_t pitch = 0) {
  if (pitch == 0) pitch = s->pitch;
  // The verdict lands in a mapped host word, written by the kernel itself: a
  // device-to-host memcpy of the flag would queue on the download copy engine
  // behind an rd_read_fields_async transfer in flight (tens of ms). No kernel
  // that writes the word is in flight here: every call ends synchronised.
  *s->h_flag = 0;
  if (rows > 0) {
    const int blocks = 148 * 8;
    if (s->esz == 4)
      rdk::finite_kernel<float><<<blocks, 256, 0, s->stream>>>((const float*)base, rows, s->W, pitch, s->h_flag_dev);
    else
      rdk::finite_kernel<double><<<blocks, 256, 0, s->stream>>>((const double*)base, rows, s->W, pitch,
                                                                 s->h_flag_dev);
    RD_CUDA(s, cudaGetLastError());
    s->st.launches++;
  }
  RD_CUDA(s, cudaStreamSynchronize(s->stream));
  *bad = *s->h_flag;
  return RD_OK;
}

// Enables the 4-op fp32 division if, for this handle's q, it equals IEEE
// div.rn on every input the reaction can produce (exhaustive check of all
// 2^32 fp32 values of C on the GPU, a few ms; cached per q per process).
int certify_q(rd_sim* s, double q, bool* ok) {
  // handles may be created / re-parameterised on several host threads
  static std::mutex mu;
  static std::vector<std::pair<uint32_t, bool>> cache;
  const float qf = (float)q;
  uint32_t bits;
  std::memcpy(&bits, &qf, 4);
  {
    std::lock_guard<std::mutex> lk(mu);
    for (const auto& c : cache)
      if (c.first == bits) {
        *ok = c.second;
        return RD_OK;
      }
  }
  unsigned long long* d = reinterpret_cast<unsigned long long*>(s->d_scratch);
  RD_CUDA(s, cudaMemsetAsync(d, 0, sizeof(unsigned long long), s->stream));
  rdk::divcert_kernel<<<s->num_sms * 8, 256, 0, s->stream>>>(qf, d);
  RD_CUDA(s, cudaGetLastError());
  unsigned long long h = ~0ull;
  RD_CUDA(s, cudaMemcpyAsync(&h, d, sizeof h, cudaMemcpyDeviceToHost, s->stream));
  RD_CUDA(s, cudaStreamSynchronize(s->stream));
  {
    std::lock_guard<std::mutex> lk(mu);
    cache.push_back({bits, h == 0});
  }
  s->div4_mismatches = (int64_t)h;
  *ok = h == 0;
  return RD_OK;
}

// Whether 1/dx^2 is a power of two, so Du may be folded into it exactly.
bool foldable(const rd_params& p) {
  const double inv = 1.0 / (p.dx * p.dx);
  int ex = 0;
  return std::frexp(inv, &ex) == 0.5 && ex > -100 && ex < 100;
}

// Arithmetic mode for the handle's parameter set(s): FOLD when every 1/dx^2
// is a power of two, FOLD_DIV4 when additionally (fp32, reaction on) the
// 4-op division is certified for every q; else PRECISE.
// Stencil kernel choice: gz_kernel or cr_kernel for small instances (whichever
// the per-step models predict faster, each only where it fits), else
// tb_kernel. RD_KERNEL=tb|lp|cr|gz forces one (tests, measurements; cr and gz
// still need the instance to fit their limits, else tb_kernel runs).
void select_kernels(rd_sim* s) {
  const char* e = getenv("RD_KERNEL");
  const std::string want = e ? e : "auto";
  s->use_lp = want == "lp";
  s->use_cr = false;
  s->use_gz = false;
  if (want == "gz") choose_gz(s, true, 0.0);
  if (want == "auto" || want == "cr") choose_cr(s, want == "cr");
  if (want == "auto") {
    // whole-chip tiles when their model beats the cluster-resident or the
    // streaming kernel
    const double t_other = s->use_cr ? t_cr_step(s, s->cr_cs) : t_tb_step(s);
    choose_gz(s, false, t_other);
    if (s->use_gz) s->use_cr = false;
  }
}

int choose_mode(rd_sim* s) {
  std::vector<rd_params> sets = s->pinst.empty() ? std::vector<rd_params>{s->p} : s->pinst;
  bool fold = true;
  for (const auto& p : sets) fold = fold && foldable(p);
  s->fast_mode = fold ? rdk::MODE_FOLD : rdk::MODE_PRECISE;
  if (fold && s->esz == 4 && !(s->g.flags & RD_REACTION_OFF)) {
    bool all = true;
    for (const auto& p : sets) {
      bool ok = false;
      if (int rc = certify_q(s, p.q, &ok)) return rc;
      all = all && ok;
    }
    if (all) s->fast_mode = rdk::MODE_FOLD_DIV4;
    // q >= 2^-35 in fp32: |C+q| < 2^-60 only at C+q == 0, which the
    // non-finite check catches (rd_kernels.cuh Div<.., MODE_FOLD_DIV4_NG>)
    bool big_q = true;
    for (const auto& p : sets) big_q = big_q && (float)p.q >= 0x1p-35f;
    if (all && big_q) s->fast_mode = rdk::MODE_FOLD_DIV4_NG;
  }
  return RD_OK;
}

char* plane_ptr(rd_sim* s, void* plane, int64_t b, int64_t local_row) {
  return (char*)plane +
         ((size_t)b * s->plane_stride + (size_t)(local_row + s->row_off) * s->pitch + (size_t)s->col_off) * s->esz;
}

// Shared by rd_create / rd_create_slab / rd_create_device / rd_create_dist.
// phi_kind: cudaMemcpyHostToDevice (host map) or DeviceToDevice (caller's
// device map); ext_arena: caller-owned plane allocation (or NULL).
int create_common(const rd_grid* grid, const rd_params* params, const void* phi_host, int64_t row0,
                  int64_t Hg, int32_t halo, bool slab, rd_sim** out, void* ext_arena, size_t ext_bytes,
                  cudaMemcpyKind phi_kind = cudaMemcpyHostToDevice) {
  if (!out) return set_err(nullptr, RD_EINVAL, "out is NULL");
  *out = nullptr;
  if (!grid || !params) return set_err(nullptr, RD_EINVAL, "grid and params are required");
  if (grid->width < 3 || grid->height < (slab ? 1 : 3))
    return set_err(nullptr, RD_EINVAL, "width and height must be >= 3 (SPEC.md:32)");
  if (grid->batch < 1) return set_err(nullptr, RD_EINVAL, "batch must be >= 1");
  if (grid->dtype != RD_F32 && grid->dtype != RD_F64) return set_err(nullptr, RD_EINVAL, "dtype must be RD_F32 or RD_F64");
  if (grid->tb_depth < 0 || grid->tb_depth > RD_MAX_TB) return set_err(nullptr, RD_EINVAL, "tb_depth must be 0..%d", RD_MAX_TB);
  if (grid->width > (1ll << 31) - 1024 || grid->height > (1ll << 31) - 1024)
    return set_err(nullptr, RD_EINVAL, "width/height must be < 2^31");
  std::string why;
  if (int rc = check_params(params, &why)) return set_err(nullptr, rc, "%s", why.c_str());
  if (slab && (halo < 1 || halo > 64 || row0 < 0 || row0 + grid->height > Hg || Hg < 3))
    return set_err(nullptr, RD_EINVAL, "bad slab geometry (row0, height_global, halo)");

  rd_sim* s = new (std::nothrow) rd_sim();
  if (!s) return set_err(nullptr, RD_ENOMEM, "host allocation failed");
  s->g = *grid;
  s->p = *params;
  s->esz = grid->dtype == RD_F32 ? 4 : 8;
  s->H = grid->height;
  s->W = grid->width;
  s->B = grid->batch;
  // columns: kMarginCols mirrored ghosts left and right, plus room for the
  // last strip's lanes (shifted to a vector-aligned start)
  const int64_t min_pitch = rdk::kMarginCols + grid->width + rdk::kMarginCols + 16;
  s->pitch = grid->pitch > 0 ? grid->pitch : (min_pitch + 31) / 32 * 32;
  if (s->pitch < min_pitch || s->pitch % 32) {
    delete s;
    return set_err(nullptr, RD_EINVAL, "pitch must be a multiple of 32 and >= width + %d", (int)(min_pitch - grid->width));
  }
  s->slab = slab;
  s->halo = slab ? halo : 0;
  s->grow0 = slab ? row0 : 0;
  s->Hg = slab ? Hg : s->H;
  s->top_edge = s->grow0 == 0;
  s->bot_edge = s->grow0 + s->H == s->Hg;
  s->r_lo = s->top_edge ? 0 : -(int32_t)s->halo;
  s->r_hi = s->bot_edge ? (int32_t)s->H : (int32_t)(s->H + s->halo);
  s->margin = (int32_t)std::max<int64_t>(s->halo, rdk::kMarginRows);
  s->row_off = s->margin + rdk::kGuardRows;
  s->col_off = rdk::kMarginCols;
  s->rows_alloc = s->H + 2 * s->row_off;
  s->plane_stride = s->rows_alloc * s->pitch;

  s->ghost_valid = (int32_t)s->halo;
  s->K = grid->tb_depth > 0 ? grid->tb_depth : auto_tb(s);
  if (slab && s->K > s->halo) s->K = (int)s->halo;
  s->st.tb_depth = s->K;

  auto fail = [&](int rc) {
    std::string m = s->err;
    rd_destroy(s);
    return set_err(nullptr, rc, "%s", m.c_str());
  };
  if (cudaStreamCreateWithFlags(&s->own_stream, cudaStreamNonBlocking) != cudaSuccess) {
    cudaGetLastError();
    s->err = "cudaStreamCreate failed (no CUDA device?)";
    return fail(RD_ECUDA);
  }
  s->stream = s->own_stream;
  {
    int dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess)
      cudaDeviceGetAttribute(&s->num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (s->num_sms < 1) s->num_sms = 148;
  }
  if (int rc = alloc_planes(s, ext_arena, ext_bytes)) return fail(rc);
  if (int rc = encode_tmaps(s)) return fail(rc);
  if (int rc = choose_mode(s)) return fail(rc);
  // phi rows present in the host buffer: local [lo, hi)
  const int64_t lo = slab ? std::max<int64_t>(0, row0 - halo) - row0 : 0;
  const int64_t hi = slab ? std::min<int64_t>(Hg, row0 + s->H + halo) - row0 : s->H;
  for (int64_t b = 0; b < s->B && phi_host; ++b) {
    const char* src = (const char*)phi_host + (size_t)b * (hi - lo) * s->W * s->esz;
    cudaError_t e = cudaMemcpy2DAsync(plane_ptr(s, s->phi, b, lo), s->pitch * s->esz, src, s->W * s->esz,
                                      s->W * s->esz, hi - lo, phi_kind, s->stream);
    if (e != cudaSuccess) {
      s->err = std::string("phi upload: ") + cudaGetErrorString(e);
      return fail(RD_ECUDA);
    }
    int bad = 0;
    if (int rc = check_finite_dev(s, plane_ptr(s, s->phi, b, lo), hi - lo, &bad)) return fail(rc);
    if (bad) {
      s->err = "phi_map contains non-finite values";
      return fail(RD_ENONFINITE);
    }
  }
  if (int rc = launch_mirror(s, s->phi, s->u[0], s->v[0], s->r_lo, s->r_hi)) return fail(rc);
  // cr_kernel PAL layout: the distinct phi values of every instance (only
  // instances small enough for cr_kernel are scanned)
  s->pal.assign((size_t)s->B, {});
  s->pal_ok = !slab && s->H * s->W <= (int64_t)1 << 20;
  for (int64_t b = 0; b < s->B && s->pal_ok; ++b) {
    if (!phi_host) {
      palette_add(s, b, 0.0);
      continue;
    }
    std::vector<double> vals((size_t)(s->H * s->W));
    std::vector<char> staged;
    const char* src = (const char*)phi_host + (size_t)b * s->H * s->W * s->esz;
    if (phi_kind == cudaMemcpyDeviceToDevice) {  // a device map: scan a host copy
      staged.resize((size_t)(s->H * s->W) * s->esz);
      if (cudaMemcpy(staged.data(), src, staged.size(), cudaMemcpyDeviceToHost) != cudaSuccess) {
        s->err = "phi palette scan";
        return fail(RD_ECUDA);
      }
      src = staged.data();
    }
    for (size_t i = 0; i < vals.size(); ++i) {
      if (s->esz == 4) {
        float f;
        std::memcpy(&f, src + 4 * i, 4);
        vals[i] = f;
      } else {
        std::memcpy(&vals[i], src + 8 * i, 8);
      }
    }
    std::sort(vals.begin(), vals.end());
    vals.erase(std::unique(vals.begin(), vals.end()), vals.end());
    if (vals.size() > 256) s->pal_ok = false;
    else
      for (double v : vals) palette_add(s, b, v);
  }
  select_kernels(s);
  if (cudaStreamSynchronize(s->stream) != cudaSuccess) {
    s->err = "stream sync failed";
    return fail(RD_ECUDA);
  }
  *out = s;
  return RD_OK;
}

int check_b(rd_sim* s, int32_t b) {
  if (b < 0 || b >= s->B) return set_err(s, RD_ERANGE, "instance %d out of range [0,%lld)", b, (long long)s->B);
  return RD_OK;
}

int copy_fields(rd_sim* s, int32_t b, void* uo, void* vo, cudaMemcpyKind kind, bool to_dev) {
  void* planes[2] = {s->u[s->cur], s->v[s->cur]};
  void* bufs[2] = {uo, vo};
  for (int k = 0; k < 2; ++k) {
    if (!bufs[k]) continue;
    char* dev = plane_ptr(s, planes[k], b, 0);
    if (to_dev)
      RD_CUDA(s, cudaMemcpy2DAsync(dev, s->pitch * s->esz, bufs[k], s->W * s->esz, s->W * s->esz, s->H, kind,
                                   s->stream));
    else
      RD_CUDA(s, cudaMemcpy2DAsync(bufs[k], s->W * s->esz, dev, s->pitch * s->esz, s->W * s->esz, s->H, kind,
                                   s->stream));
  }
  return RD_OK;
}

// The inputs are staged in instance b's owned rows of the other ping-pong
// buffer (dead between rd_step calls: every launch overwrites them before
// reading) and checked there; only if both are finite are they copied into
// the current buffer, so a rejected write leaves the handle untouched.
int write_fields(rd_sim* s, int32_t b, const void* u, const void* v, cudaMemcpyKind kind) {
  if (int rc = check_b(s, b)) return rc;
  if (!u && !v) return RD_OK;
  const int st = s->cur ^ 1;
  void* stage[2] = {s->u[st], s->v[st]};
  void* live[2] = {s->u[s->cur], s->v[s->cur]};
  const void* bufs[2] = {u, v};
  for (int k = 0; k < 2; ++k) {
    if (!bufs[k]) continue;
    RD_CUDA(s, cudaMemcpy2DAsync(plane_ptr(s, stage[k], b, 0), s->pitch * s->esz, bufs[k], s->W * s->esz,
                                 s->W * s->esz, s->H, kind, s->stream));
    int bad = 0;
    if (int rc = check_finite_dev(s, plane_ptr(s, stage[k], b, 0), s->H, &bad)) return rc;
    if (bad) return set_err(s, RD_ENONFINITE, "rd_write_fields: %s contains non-finite values", k ? "v" : "u");
  }
  for (int k = 0; k < 2; ++k)
    if (bufs[k])
      RD_CUDA(s, cudaMemcpy2DAsync(plane_ptr(s, live[k], b, 0), s->pitch * s->esz, plane_ptr(s, stage[k], b, 0),
                                   s->pitch * s->esz, s->W * s->esz, s->H, cudaMemcpyDeviceToDevice, s->stream));
  // refresh the mirrored margins of every plane written
  return launch_mirror(s, u ? s->u[s->cur] : s->v[s->cur], (u && v) ? s->v[s->cur] : nullptr, nullptr, s->r_lo,
                       s->r_hi);
}

// ---- asynchronous host I/O ---------------------------------------------------
// Uploads land in a dense staging block on their own copy stream while the
// handle computes; rd_commit_fields orders the stream behind them, checks them
// and copies them into the live planes. Downloads snapshot the fields into a
// second staging block on the compute stream (device-to-device) and drain it
// to the host on another copy stream, so the next rd_step starts at once.
int io_init(rd_sim* s) {
  if (s->io_in) return RD_OK;
  const size_t bytes = 2 * (size_t)s->B * s->H * s->W * s->esz;
  RD_CUDA(s, cudaMalloc(&s->io_in, bytes));
  RD_CUDA(s, cudaMalloc(&s->io_out, bytes));
  RD_CUDA(s, cudaStreamCreateWithFlags(&s->io_s_in, cudaStreamNonBlocking));
  RD_CUDA(s, cudaStreamCreateWithFlags(&s->io_s_out, cudaStreamNonBlocking));
  cudaEvent_t* ev[4] = {&s->io_e_in, &s->io_e_commit, &s->io_e_snap, &s->io_e_out};
  for (cudaEvent_t* e : ev) RD_CUDA(s, cudaEventCreateWithFlags(e, cudaEventDisableTiming));
  s->io_staged.assign(2 * (size_t)s->B, 0);
  s->io_draining.assign(2 * (size_t)s->B, 0);
  return RD_OK;
}

char* io_slot(rd_sim* s, void* block, int plane, int32_t b) {
  return static_cast<char*>(block) + ((size_t)plane * s->B + b) * (size_t)s->H * s->W * s->esz;
}

void io_destroy(rd_sim* s) {
  if (s->io_s_in) cudaStreamSynchronize(s->io_s_in);
  if (s->io_s_out) cudaStreamSynchronize(s->io_s_out);
  cudaEvent_t ev[4] = {s->io_e_in, s->io_e_commit, s->io_e_snap, s->io_e_out};
  for (cudaEvent_t e : ev)
    if (e) cudaEventDestroy(e);
  if (s->io_s_in) cudaStreamDestroy(s->io_s_in);
  if (s->io_s_out) cudaStreamDestroy(s->io_s_out);
  if (s->io_in) cudaFree(s->io_in);
  if (s->io_out) cudaFree(s->io_out);
}

int write_fields_async(rd_sim* s, int32_t b, const void* u, const void* v) {
  if (int rc = check_b(s, b)) return rc;
  if (!u && !v) return RD_OK;
  if (int rc = io_init(s)) return rc;
  // the last commit may still be reading the staging block
  RD_CUDA(s, cudaStreamWaitEvent(s->io_s_in, s->io_e_commit, 0));
  const void* bufs[2] = {u, v};
  const size_t bytes = (size_t)s->H * s->W * s->esz;
  for (int k = 0; k < 2; ++k) {
    if (!bufs[k]) continue;
    RD_CUDA(s, cudaMemcpyAsync(io_slot(s, s->io_in, k, b), bufs[k], bytes, cudaMemcpyHostToDevice, s->io_s_in));
    s->io_staged[(size_t)k * s->B + b] = 1;
  }
  RD_CUDA(s, cudaEventRecord(s->io_e_in, s->io_s_in));
  return RD_OK;
}

int commit_fields(rd_sim* s) {
  if (!s->io_in) return RD_OK;
  bool any = false;
  for (uint8_t f : s->io_staged) any = any || f;
  if (!any) return RD_OK;
  Range r_("rd_commit_fields");
  RD_CUDA(s, cudaStreamWaitEvent(s->stream, s->io_e_in, 0));
  // all or nothing: every staged plane is checked before any is copied in
  for (int k = 0; k < 2; ++k)
    for (int32_t b = 0; b < s->B; ++b) {
      if (!s->io_staged[(size_t)k * s->B + b]) continue;
      int bad = 0;
      if (int rc = check_finite_dev(s, io_slot(s, s->io_in, k, b), s->H, &bad, s->W)) return rc;
      if (bad) {
        std::fill(s->io_staged.begin(), s->io_staged.end(), 0);
        return set_err(s, RD_ENONFINITE, "rd_commit_fields: %s of instance %d contains non-finite values (nothing written)",
                       k ? "v" : "u", b);
      }
    }
  void* live[2] = {s->u[s->cur], s->v[s->cur]};
  bool wrote[2] = {false, false};
  for (int k = 0; k < 2; ++k)
    for (int32_t b = 0; b < s->B; ++b) {
      if (!s->io_staged[(size_t)k * s->B + b]) continue;
      if (int rc = copy_rows(s, plane_ptr(s, live[k], b, 0), s->pitch * s->esz, io_slot(s, s->io_in, k, b),
                             s->W * s->esz, s->W * s->esz, s->H))
        return rc;
      s->io_staged[(size_t)k * s->B + b] = 0;
      wrote[k] = true;
    }
  RD_CUDA(s, cudaEventRecord(s->io_e_commit, s->stream));
  return launch_mirror(s, wrote[0] ? live[0] : live[1], (wrote[0] && wrote[1]) ? live[1] : nullptr, nullptr, s->r_lo,
                       s->r_hi);
}

int read_fields_async(rd_sim* s, int32_t b, void* u_out, void* v_out) {
  if (int rc = check_b(s, b)) return rc;
  if (!u_out && !v_out) return RD_OK;
  if (int rc = io_init(s)) return rc;
  void* bufs[2] = {u_out, v_out};
  void* live[2] = {s->u[s->cur], s->v[s->cur]};
  // a slot still draining an earlier snapshot must finish first
  if (cudaEventQuery(s->io_e_out) == cudaSuccess) std::fill(s->io_draining.begin(), s->io_draining.end(), 0);
  for (int k = 0; k < 2; ++k)
    if (bufs[k] && s->io_draining[(size_t)k * s->B + b]) {
      RD_CUDA(s, cudaStreamWaitEvent(s->stream, s->io_e_out, 0));
      break;
    }
  for (int k = 0; k < 2; ++k)
    if (bufs[k])
      if (int rc = copy_rows(s, io_slot(s, s->io_out, k, b), s->W * s->esz, plane_ptr(s, live[k], b, 0),
                             s->pitch * s->esz, s->W * s->esz, s->H))
        return rc;
  RD_CUDA(s, cudaEventRecord(s->io_e_snap, s->stream));
  RD_CUDA(s, cudaStreamWaitEvent(s->io_s_out, s->io_e_snap, 0));
  const size_t bytes = (size_t)s->H * s->W * s->esz;
  for (int k = 0; k < 2; ++k)
    if (bufs[k]) {
      RD_CUDA(s, cudaMemcpyAsync(bufs[k], io_slot(s, s->io_out, k, b), bytes, cudaMemcpyDeviceToHost, s->io_s_out));
      s->io_draining[(size_t)k * s->B + b] = 1;
    }
  RD_CUDA(s, cudaEventRecord(s->io_e_out, s->io_s_out));
  return RD_OK;
}

int io_wait(rd_sim* s) {
  if (!s->io_in) return RD_OK;
  RD_CUDA(s, cudaStreamSynchronize(s->io_s_in));
  RD_CUDA(s, cudaStreamSynchronize(s->io_s_out));
  std::fill(s->io_draining.begin(), s->io_draining.end(), 0);
  return RD_OK;
}

}  // namespace

// ============================================================================
// C ABI
// ============================================================================
extern "C" {

int32_t rd_abi_version(void) { return RD_ABI_VERSION; }

void rd_params_default(rd_params* p) {
  if (!p) return;
  p->eps = 0.0243;
  p->f = 1.4;
  p->q = 0.002;
  p->Du = 0.45;
  p->dt = 0.001;
  p->dx = 0.25;
}

const char* rd_create_error(void) { return g_create_error.c_str(); }

const char* rd_last_error(const rd_sim* s) { return s ? s->err.c_str() : g_create_error.c_str(); }

int rd_create(const rd_grid* grid, const rd_params* params, const void* phi_map, rd_sim** out) {
  return create_common(grid, params, phi_map, 0, grid ? grid->height : 0, 0, false, out, nullptr, 0);
}

int rd_create_slab(const rd_grid* grid, const rd_params* params, const void* phi_slab, int64_t row0,
                   int64_t height_global, int32_t halo, rd_sim** out) {
  return create_common(grid, params, phi_slab, row0, height_global, halo, true, out, nullptr, 0);
}

int rd_arena_bytes(const rd_grid* grid, size_t* bytes) {
  if (!grid || !bytes) return set_err(nullptr, RD_EINVAL, "grid and bytes are required");
  if (grid->width < 3 || grid->height < 3 || grid->batch < 1 || (grid->dtype != RD_F32 && grid->dtype != RD_F64))
    return set_err(nullptr, RD_EINVAL, "bad grid");
  // the layout create_common computes (kept in one place: a throwaway handle
  // description, no device work)
  rd_sim t;
  t.esz = grid->dtype == RD_F32 ? 4 : 8;
  t.B = grid->batch;
  const int64_t min_pitch = rdk::kMarginCols + grid->width + rdk::kMarginCols + 16;
  t.pitch = grid->pitch > 0 ? grid->pitch : (min_pitch + 31) / 32 * 32;
  const int64_t row_off = rdk::kMarginRows + rdk::kGuardRows;
  t.plane_stride = (grid->height + 2 * row_off) * t.pitch;
  *bytes = arena_size(&t);
  return RD_OK;
}

int rd_create_device(const rd_grid* grid, const rd_params* params, void* arena, size_t arena_bytes,
                     const void* phi_dev, rd_sim** out) {
  if (!arena) return set_err(nullptr, RD_EINVAL, "arena is NULL");
  return create_common(grid, params, phi_dev, 0, grid ? grid->height : 0, 0, false, out, arena, arena_bytes,
                       cudaMemcpyDeviceToDevice);
}

int rd_field_ptr(rd_sim* s, int32_t b, int32_t plane, void** ptr, int64_t* pitch_elems) {
  if (!s || !ptr) return RD_EINVAL;
  if (int rc = check_b(s, b)) return rc;
  void* planes[3] = {s->u[s->cur], s->v[s->cur], s->phi};
  if (plane < 0 || plane > 2) return set_err(s, RD_EINVAL, "plane must be 0 (u), 1 (v) or 2 (phi)");
  if (s->margins_stale && plane < 2)
    if (int rc = fresh_margins(s)) return rc;
  if (plane == 2) {
    // the caller may write phi through this pointer at any later time: never
    // again assume it is one value (tb_kernel UPHI variants)
    s->phi_external = true;
    s->phi_class_known = false;
  }
  *ptr = plane_ptr(s, planes[plane], b, 0);
  if (pitch_elems) *pitch_elems = s->pitch;
  return RD_OK;
}

int rd_get_geometry(const rd_sim* s, rd_geometry* out) {
  if (!s || !out) return RD_EINVAL;
  std::memset(out, 0, sizeof *out);
  out->width = s->W;
  out->height = s->H;
  out->height_global = s->Hg;
  out->row0 = s->grow0;
  out->batch = (int32_t)s->B;
  out->dtype = s->g.dtype;
  out->halo = (int32_t)s->halo;
  out->tb_depth = s->K;
  out->pitch = s->pitch;
  out->rank = 0;
  out->world = 1;
  out->phi_rows_lo = s->slab ? std::max<int64_t>(0, s->grow0 - s->halo) - s->grow0 : 0;
  out->phi_rows_hi = s->slab ? std::min<int64_t>(s->Hg, s->grow0 + s->H + s->halo) - s->grow0 : s->H;
  dist_geometry(s, out);
  return RD_OK;
}

int rd_destroy(rd_sim* s) {
  if (!s) return RD_OK;
  if (s->stream) cudaStreamSynchronize(s->stream);
  if (s->dist) dist_destroy(s);
  io_destroy(s);
  for (void* m : s->ipc_mapped) cudaIpcCloseMemHandle(m);
  if (s->arena && s->own_arena) cudaFree(s->arena);
  void* ps[] = {s->tl,        s->ck_tl,   s->d_probes, s->d_first, s->d_first_ck, s->d_fault,
                s->d_flag,    s->d_scratch, s->d_idx,  s->d_pal,   s->d_pal_n,    s->gz_x};
  for (void* p : ps)
    if (p) cudaFree(p);
  if (s->h_flag) cudaFreeHost(s->h_flag);
  for (auto& e : s->ev_pool) {
    cudaEventDestroy(e.first);
    cudaEventDestroy(e.second);
  }
  drop_graphs(s);
  if (s->capture_stream) cudaStreamDestroy(s->capture_stream);
  if (s->own_stream) cudaStreamDestroy(s->own_stream);
  delete s;
  return RD_OK;
}

int rd_set_stream(rd_sim* s, void* stream) {
  if (!s) return RD_EINVAL;
  RD_CUDA(s, cudaStreamSynchronize(s->stream));
  s->stream = stream ? (cudaStream_t)stream : s->own_stream;
  return RD_OK;
}

int rd_write_fields(rd_sim* s, int32_t b, const void* u, const void* v) {
  if (!s) return RD_EINVAL;
  return write_fields(s, b, u, v, cudaMemcpyHostToDevice);
}

int rd_write_fields_device(rd_sim* s, int32_t b, const void* u, const void* v) {
  if (!s) return RD_EINVAL;
  return write_fields(s, b, u, v, cudaMemcpyDeviceToDevice);
}

int rd_read_fields(rd_sim* s, int32_t b, void* u_out, void* v_out) {
  if (!s) return RD_EINVAL;
  if (int rc = check_b(s, b)) return rc;
  if (int rc = copy_fields(s, b, u_out, v_out, cudaMemcpyDeviceToHost, false)) return rc;
  RD_CUDA(s, cudaStreamSynchronize(s->stream));
  return RD_OK;
}

int rd_read_fields_device(rd_sim* s, int32_t b, void* u_out, void* v_out) {
  if (!s) return RD_EINVAL;
  if (int rc = check_b(s, b)) return rc;
  return copy_fields(s, b, u_out, v_out, cudaMemcpyDeviceToDevice, false);
}

int rd_write_fields_async(rd_sim* s, int32_t b, const void* u, const void* v) {
  if (!s) return RD_EINVAL;
  return write_fields_async(s, b, u, v);
}

int rd_commit_fields(rd_sim* s) {
  if (!s) return RD_EINVAL;
  return commit_fields(s);
}

int rd_read_fields_async(rd_sim* s, int32_t b, void* u_out, void* v_out) {
  if (!s) return RD_EINVAL;
  return read_fields_async(s, b, u_out, v_out);
}

int rd_io_wait(rd_sim* s) {
  if (!s) return RD_EINVAL;
  return io_wait(s);
}

int rd_stimulate(rd_sim* s, int32_t b, const rd_shape* shape, double value, int64_t at_step) {
  if (!s) return RD_EINVAL;
  if (!shape) return set_err(s, RD_EINVAL, "shape is NULL");
  if (b < -1 || b >= s->B) return set_err(s, RD_ERANGE, "instance %d out of range", b);
  if (at_step < s->step)
    return set_err(s, RD_ERANGE, "at_step %lld is before the current step %lld", (long long)at_step, (long long)s->step);
  if (shape->kind != RD_DISC && shape->kind != RD_RECT && shape->kind != RD_HALF_DISC)
    return set_err(s, RD_EINVAL, "unknown shape kind %d", shape->kind);
  if (shape->kind != RD_RECT && shape->r < 0) return set_err(s, RD_EINVAL, "radius must be >= 0 (SPEC.md:78)");
  if (!std::isfinite(value)) return set_err(s, RD_ENONFINITE, "stimulus value is not finite");
  PendingEvent ev;
  ev.b = b;
  ev.shape.kind = shape->kind;
  ev.shape.dir = shape->dir;
  ev.shape.cy2 = shape->cy2;
  ev.shape.cx2 = shape->cx2;
  ev.shape.r = shape->r;
  ev.shape.y0 = shape->y0;
  ev.shape.x0 = shape->x0;
  ev.shape.y1 = shape->y1;
  ev.shape.x1 = shape->x1;
  ev.shape.mask = (shape->flags & RD_SHAPE_MASK_PHI) ? 1 : 0;
  ev.value = value;
  ev.mask_phi = shape->mask_phi;
  ev.at = at_step;
  s->events.push_back(ev);
  return RD_OK;
}

int rd_step(rd_sim* s, int64_t n) {
  if (!s) return RD_EINVAL;
  Range r_("rd_step");
  if (n < 0) return set_err(s, RD_EINVAL, "n must be >= 0");
  if (s->dist) return n ? dist_step(s, n) : RD_OK;
  if (s->slab && n > s->halo) return set_err(s, RD_ERANGE, "slab handles step at most halo=%lld steps per call", (long long)s->halo);
  if (n == 0) return RD_OK;
  // slab contract: the caller refreshed the ghost rows before this call
  s->ghost_valid = (int32_t)s->halo;
  const bool ckpt = !(s->g.flags & RD_NO_CHECKPOINT);
  const int64_t step0 = s->step;
  int rc = sync_probes(s);
  if (rc) return rc;
  if (ckpt && (rc = save_checkpoint(s))) return rc;
  if ((rc = run_range(s, step0 + n, s->K))) return rc;
  unsigned long long key = ~0ull;
  int precise_hit = 0;
  if ((rc = read_fault(s, &key, &precise_hit))) return rc;
  if (key == ~0ull && !precise_hit) return RD_OK;

  if (ckpt) {
    // Replay from the checkpoint with PRECISE (__fdiv_rn) kernels, one step
    // per launch, checking for non-finite cells after every step: the handle
    // ends at the first failing step (or at step0+n), bit-identical to a
    // step-by-step exact run (results do not depend on the blocking depth).
    if ((rc = restore_checkpoint(s))) return rc;
    key = ~0ull;
    Range rr_("rd_step.precise_replay");
    s->precise_mode = true;
    s->defer_samples = true;
    s->st.replays++;
    while (s->step < step0 + n) {
      // the step without its probe latch and timelapse record; those follow
      // only once the step is known to be finite (the oracle stops before
      // sampling a failing step, oracle_body.h orc_run)
      if ((rc = run_range(s, s->step + 1, 1)) || (rc = read_fault(s, &key, nullptr))) break;
      if (key != ~0ull) break;
      if ((rc = sample_step(s))) break;
    }
    s->precise_mode = false;
    s->defer_samples = false;
    if (rc) return rc;
    if (key == ~0ull) return RD_OK;
  }
  const unsigned long long W = (unsigned long long)s->W, Hg = (unsigned long long)s->Hg;
  s->fault.step = s->step;
  s->fault.b = (int32_t)(key / (W * Hg));
  s->fault.i = (int64_t)((key / W) % Hg);
  s->fault.j = (int64_t)(key % W);
  reset_fault(s);
  return set_err(s, RD_ENONFINITE, "non-finite value at instance %d, cell (%lld, %lld) after step %lld%s", s->fault.b,
                 (long long)s->fault.i, (long long)s->fault.j, (long long)s->fault.step,
                 ckpt ? "" : " (k-block granularity: RD_NO_CHECKPOINT)");
}

int rd_step_unchecked(rd_sim* s, int64_t n) {
  if (!s) return RD_EINVAL;
  if (int rc = not_dist(s, "rd_step_unchecked")) return rc;
  Range r_("rd_step_unchecked");
  if (n < 0) return set_err(s, RD_EINVAL, "n must be >= 0");
  if (s->slab && n > s->halo) return set_err(s, RD_ERANGE, "slab handles step at most halo=%lld steps per call", (long long)s->halo);
  if (n == 0) return RD_OK;
  s->ghost_valid = (int32_t)s->halo;
  if (int rc = sync_probes(s)) return rc;
  return run_range(s, s->step + n, s->K);
}

// Slab blocks overlapped with the halo exchange: the
// interior rows -- at least k rows from any exchanged ghost row -- depend only
// on owned rows, so they run while the exchange is in flight; the edge bands
// run once the ghosts have landed. Only a block that is one plain launch
// qualifies (k <= the handle's depth, no stimulus due in it, no probe or
// timelapse sample strictly inside); otherwise *started = 0 and the caller
// steps with rd_step_unchecked after the exchange.
int rd_step_begin(rd_sim* s, int64_t k, int32_t flags, int32_t* started) {
  if (!s || !started) return RD_EINVAL;
  if (int rc = not_dist(s, "rd_step_begin")) return rc;
  *started = 0;
  if (!s->slab) return set_err(s, RD_EINVAL, "rd_step_begin: slab handles only");
  if (s->pending_k) return set_err(s, RD_EINVAL, "rd_step_begin: a block is already open (rd_step_finish)");
  if (k < 1 || k > s->halo) return set_err(s, RD_ERANGE, "k must be in [1, halo=%lld]", (long long)s->halo);
  const bool push = (flags & RD_BLOCK_PUSH) != 0;
  if (push && ((!s->top_edge && !s->peer[0].u[0]) || (!s->bot_edge && !s->peer[1].u[0])))
    return set_err(s, RD_EINVAL, "rd_step_begin: RD_BLOCK_PUSH needs the neighbours registered (rd_set_peer)");
  if (k > s->K || s->precise_mode || (push && k != s->halo)) return RD_OK;
  for (const auto& ev : s->events)
    if (ev.at >= s->step && ev.at < s->step + k) return RD_OK;
  for (int64_t t = s->step + 1; t < s->step + k; ++t) {
    if (probe_due(s, t)) return RD_OK;
    if (s->tl_stride > 0 && t % s->tl_stride == 0) return RD_OK;
  }
  if (int rc = sync_probes(s)) return rc;
  s->ghost_valid = (int32_t)s->halo;
  int32_t lo, hi;
  block_rows(s, (int)k, &lo, &hi);
  const int32_t a = s->top_edge ? 0 : (int32_t)k;
  const int32_t b = (int32_t)s->H - (s->bot_edge ? 0 : (int32_t)k);
  if (a < b)
    if (int rc = launch_rows(s, (int)k, s->cur, s->cur ^ 1, a, b)) return rc;
  s->pending_k = (int32_t)k;
  s->pending_push = push;
  *started = 1;
  return RD_OK;
}

int rd_step_finish(rd_sim* s) {
  if (!s) return RD_EINVAL;
  if (!s->pending_k) return set_err(s, RD_EINVAL, "rd_step_finish: no open block (rd_step_begin)");
  const int k = s->pending_k;
  const bool push = s->pending_push;
  s->pending_k = 0;
  s->pending_push = false;
  int32_t lo, hi;
  block_rows(s, k, &lo, &hi);
  const int32_t a = s->top_edge ? 0 : k;
  const int32_t b = (int32_t)s->H - (s->bot_edge ? 0 : k);
  if (push) {
    // the neighbours stored their send rows (interior columns) into this
    // buffer's ghost rows: refresh those rows' mirrored ghost columns
    const int32_t glo = s->top_edge ? 0 : -(int32_t)s->halo;
    const int32_t ghi = (int32_t)s->H + (s->bot_edge ? 0 : (int32_t)s->halo);
    if (int rc = launch_mirror(s, s->u[s->cur], s->v[s->cur], nullptr, glo, ghi)) return rc;
  }
  // the edge bands hold every send row (k == halo on push blocks), so they
  // alone push, after the caller's wait for the neighbours
  s->push_active = push;
  int rc = RD_OK;
  if (a < b) {
    if (lo < a) rc = launch_rows(s, k, s->cur, s->cur ^ 1, lo, a);
    if (rc == RD_OK && b < hi) rc = launch_rows(s, k, s->cur, s->cur ^ 1, b, hi);
  } else {
    rc = launch_rows(s, k, s->cur, s->cur ^ 1, lo, hi);
  }
  s->push_active = false;
  if (rc) return rc;
  if (int rc2 = end_block(s, k, lo, hi)) return rc2;
  s->step += k;
  if (probe_due(s, s->step))
    if (int rc3 = launch_probes(s, s->step)) return rc3;
  return RD_OK;
}

int rd_set_peer(rd_sim* s, int32_t side, void* u0, void* u1, void* v0, void* v1, int64_t rows,
                int64_t plane_stride_bytes) {
  if (!s) return RD_EINVAL;
  if (side != 0 && side != 1) return set_err(s, RD_EINVAL, "side must be 0 (above) or 1 (below)");
  if (int rc = not_dist(s, "rd_set_peer")) return rc;
  if (!s->slab) return set_err(s, RD_EINVAL, "rd_set_peer: slab handles only");
  rd_sim::Peer& p = s->peer[side];
  if (!u0) {
    p = rd_sim::Peer{};
    return RD_OK;
  }
  if (!u1 || !v0 || !v1 || rows < s->halo || plane_stride_bytes <= 0)
    return set_err(s, RD_EINVAL, "rd_set_peer: four plane pointers, rows >= halo and a stride are required");
  p.u[0] = u0, p.u[1] = u1, p.v[0] = v0, p.v[1] = v1;
  p.rows = rows;
  p.stride_bytes = plane_stride_bytes;
  return RD_OK;
}

int rd_plane_origins(const rd_sim* s, void** u0, void** u1, void** v0, void** v1, int64_t* plane_stride_bytes) {
  if (!s || !u0 || !u1 || !v0 || !v1) return RD_EINVAL;
  auto org = [&](void* plane) { return static_cast<void*>(static_cast<char*>(plane) + (s->row_off * s->pitch + s->col_off) * s->esz); };
  *u0 = org(s->u[0]);
  *u1 = org(s->u[1]);
  *v0 = org(s->v[0]);
  *v1 = org(s->v[1]);
  if (plane_stride_bytes) *plane_stride_bytes = s->plane_stride * (int64_t)s->esz;
  return RD_OK;
}

int rd_flag_ptr(rd_sim* s, int32_t side, void** flag) {
  if (!s || !flag || (side != 0 && side != 1)) return RD_EINVAL;
  // word 0: pushes received from the neighbour above; word 1: from below
  *flag = static_cast<char*>(s->arena) + s->arena_bytes - 256 + 4 * side;
  return RD_OK;
}

int rd_ipc_export(rd_sim* s, void* handle64, void** arena_base) {
  if (!s || !handle64 || !arena_base) return RD_EINVAL;
  cudaIpcMemHandle_t h;
  RD_CUDA(s, cudaIpcGetMemHandle(&h, s->arena));
  std::memcpy(handle64, &h, sizeof h);
  *arena_base = s->arena;
  return RD_OK;
}

int rd_ipc_map(rd_sim* s, const void* handle64, void** mapped_base) {
  if (!s || !handle64 || !mapped_base) return RD_EINVAL;
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle64, sizeof h);
  RD_CUDA(s, cudaIpcOpenMemHandle(mapped_base, h, cudaIpcMemLazyEnablePeerAccess));
  s->ipc_mapped.push_back(*mapped_base);
  return RD_OK;
}

int rd_push_ghosts(rd_sim* s) {
  if (!s) return RD_EINVAL;
  if (int rc = not_dist(s, "rd_push_ghosts")) return rc;
  if (!s->slab) return set_err(s, RD_EINVAL, "rd_push_ghosts: slab handles only");
  const size_t row_bytes = (size_t)s->pitch * s->esz, col = (size_t)s->col_off * s->esz;
  const size_t bytes = (size_t)s->halo * row_bytes;
  for (int side = 0; side < 2; ++side) {
    const rd_sim::Peer& p = s->peer[side];
    if (!p.u[0]) continue;
    // my rows [0, halo) -> the peer above's rows [rows, rows + halo); my rows
    // [H - halo, H) -> the peer below's rows [-halo, 0) (row storage, ghost
    // columns included)
    const int64_t my_row = side == 0 ? 0 : s->H - s->halo;
    const int64_t its_row = side == 0 ? p.rows : -s->halo;
    for (int64_t b = 0; b < s->B; ++b)
      for (int pl = 0; pl < 2; ++pl) {
        char* src = plane_ptr(s, pl == 0 ? s->u[s->cur] : s->v[s->cur], b, my_row) - col;
        char* dst = static_cast<char*>(pl == 0 ? p.u[s->cur] : p.v[s->cur]) + b * p.stride_bytes +
                    its_row * (int64_t)row_bytes - (int64_t)col;
        RD_CUDA(s, cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, s->stream));
      }
  }
  return RD_OK;
}

// Stream-ordered 32-bit flag operations (driver stream memory operations,
// reached through the runtime's entry-point query: no libcuda link).
int rd_stream_signal(rd_sim* s, void* flag, uint32_t value) {
  if (!s || !flag) return RD_EINVAL;
  auto fn = reinterpret_cast<PFN_cuStreamWriteValue32_v11070>(driver_entry("cuStreamWriteValue32"));
  if (!fn) return set_err(s, RD_ECUDA, "cuStreamWriteValue32 entry point unavailable");
  if (fn(reinterpret_cast<CUstream>(s->stream), reinterpret_cast<CUdeviceptr>(flag), value, 0) != CUDA_SUCCESS)
    return set_err(s, RD_ECUDA, "cuStreamWriteValue32 failed");
  return RD_OK;
}

int rd_stream_wait(rd_sim* s, void* flag, uint32_t value) {
  if (!s || !flag) return RD_EINVAL;
  auto fn = reinterpret_cast<PFN_cuStreamWaitValue32_v11070>(driver_entry("cuStreamWaitValue32"));
  if (!fn) return set_err(s, RD_ECUDA, "cuStreamWaitValue32 entry point unavailable");
  if (fn(reinterpret_cast<CUstream>(s->stream), reinterpret_cast<CUdeviceptr>(flag), value,
         CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS)
    return set_err(s, RD_ECUDA, "cuStreamWaitValue32 failed");
  return RD_OK;
}

int rd_checkpoint(rd_sim* s) {
  if (!s) return RD_EINVAL;
  if (int rc = not_dist(s, "rd_checkpoint")) return rc;
  if (int rc = sync_probes(s)) return rc;
  return save_checkpoint(s);
}

int rd_restore(rd_sim* s) {
  if (!s) return RD_EINVAL;
  if (int rc = not_dist(s, "rd_restore")) return rc;
  return restore_checkpoint(s);
}

int rd_read_flags(rd_sim* s, int32_t* nonfinite, int32_t* inexact) {
  if (!s) return RD_EINVAL;
  unsigned long long key = ~0ull;
  int p = 0;
  if (int rc = read_fault(s, &key, &p)) return rc;
  if (nonfinite) *nonfinite = key != ~0ull;
  if (inexact) *inexact = p != 0;
  return reset_fault(s);
}

int64_t rd_get_step(const rd_sim* s) { return s ? s->step : -1; }

int rd_get_fault(const rd_sim* s, rd_fault* out) {
  if (!s || !out) return RD_EINVAL;
  *out = s->fault;
  return RD_OK;
}

int rd_probe(rd_sim* s, int32_t b, const rd_rect* r, double threshold, int32_t* fired, double* max_u) {
  if (!s || !r) return RD_EINVAL;
  if (int rc = check_b(s, b)) return rc;
  if (s->dist) {
    // collective: the maximum over every rank's owned part of the rect
    if (r->y0 >= r->y1 || r->x0 >= r->x1 || r->x0 < 0 || r->x1 > s->W || r->y0 < 0 || r->y1 > s->Hg)
      return set_err(s, RD_ERANGE, "probe rect empty or outside the grid (SPEC.md:245-247)");
    double m = -INFINITY;
    rd_rect own = *r;
    own.y0 = std::max<int64_t>(r->y0, s->grow0);
    own.y1 = std::min<int64_t>(r->y1, s->grow0 + s->H);
    if (own.y0 < own.y1) {
      rd_sim* save = s;
      DistState* d = s->dist;
      s->dist = nullptr;  // the local probe below
      const int rc = rd_probe(save, b, &own, threshold, nullptr, &m);
      s->dist = d;
      if (rc) return rc;
      if (m != m) m = -INFINITY;  // NaN never wins (R-23)
    }
    std::vector<uint64_t> v{dbl_key(m)};
    if (int rc = dist_allmax(s, v)) return rc;
    m = key_dbl(v[0]);
    if (max_u) *max_u = m;
    if (fired) *fired = s->esz == 4 ? (float)m >= (float)threshold : m >= threshold;
    return RD_OK;
  }
  const int64_t y0 = r->y0 - s->grow0, y1 = r->y1 - s->grow0;
  if (r->y0 >= r->y1 || r->x0 >= r->x1 || r->x0 < 0 || r->x1 > s->W || y0 < 0 || y1 > s->H)
    return set_err(s, RD_ERANGE, "probe rect empty or outside the grid (SPEC.md:245-247)");
  rdk::ProbeDev pd{y0, r->x0, y1, r->x1, b, 0, threshold};
  rdk::ProbeDev* dp = (rdk::ProbeDev*)((char*)s->d_scratch);
  static_assert(sizeof(rdk::ProbeDev) <= 48, "scratch");
  RD_CUDA(s, cudaMemcpyAsync(dp, &pd, sizeof pd, cudaMemcpyHostToDevice, s->stream));
  double m = 0;
  if (s->esz == 4) {
    float* mo = (float*)((char*)s->d_scratch + 48);
    rdk::probe_kernel<float><<<1, 256, 0, s->stream>>>(origin<float>(s, s->u[s->cur]), s->plane_stride, s->pitch,
                                                        dp, 1, s->step, nullptr, mo);
    RD_CUDA(s, cudaGetLastError());
    float h;
    RD_CUDA(s, cudaMemcpyAsync(&h, mo, sizeof h, cudaMemcpyDeviceToHost, s->stream));
    RD_CUDA(s, cudaStreamSynchronize(s->stream));
    m = h;
    if (fired) *fired = h >= (float)threshold;
  } else {
    double* mo = (double*)((char*)s->d_scratch + 48);
    rdk::probe_kernel<double><<<1, 256, 0, s->stream>>>(origin<double>(s, s->u[s->cur]), s->plane_stride, s->pitch,
                                                         dp, 1, s->step, nullptr, mo);
    RD_CUDA(s, cudaGetLastError());
    RD_CUDA(s, cudaMemcpyAsync(&m, mo, sizeof m, cudaMemcpyDeviceToHost, s->stream));
    RD_CUDA(s, cudaStreamSynchronize(s->stream));
    if (fired) *fired = m >= threshold;
  }
  s->st.launches++;
  if (max_u) *max_u = m;
  return RD_OK;
}

int rd_probe_latch(rd_sim* s, int32_t b, const rd_rect* r, double threshold, int32_t stride, int32_t* id) {
  if (!s || !r || !id) return RD_EINVAL;
  if (int rc = check_b(s, b)) return rc;
  if (stride < 1) return set_err(s, RD_EINVAL, "stride must be >= 1");
  if (r->y0 >= r->y1 || r->x0 >= r->x1 || r->x0 < 0 || r->x1 > s->W || r->y0 < 0 || r->y1 > s->Hg)
    return set_err(s, RD_ERANGE, "probe rect empty or outside the grid (SPEC.md:245-247)");
  s->probes.push_back({b, *r, threshold, stride});
  s->probes_dirty = true;
  *id = (int32_t)s->probes.size() - 1;
  return sync_probes(s);
}

int rd_probe_result(rd_sim* s, int32_t id, int64_t* first) {
  if (!s || !first) return RD_EINVAL;
  if (id < 0 || id >= (int32_t)s->probes.size()) return set_err(s, RD_ERANGE, "unknown probe id %d", id);
  long long h = -1;
  RD_CUDA(s, cudaMemcpyAsync(&h, s->d_first + id, sizeof h, cudaMemcpyDeviceToHost, s->stream));
  RD_CUDA(s, cudaStreamSynchronize(s->stream));
  if (s->dist) return dist_probe_result(s, h, first);  // collective: first firing over all ranks
  *first = h;
  return RD_OK;
}

int rd_set_params(rd_sim* s, int32_t b, const rd_params* p) {
  if (!s || !p) return RD_EINVAL;
  if (b < -1 || b >= s->B) return set_err(s, RD_ERANGE, "instance %d out of range", b);
  std::string why;
  if (int rc = check_params(p, &why)) return set_err(s, rc, "%s", why.c_str());
  if (b == -1) {
    s->p = *p;
    s->pinst.clear();
  } else {
    if (s->B > rdk::kMaxParamSets)
      return set_err(s, RD_EINVAL, "per-instance parameters need batch <= %d", rdk::kMaxParamSets);
    if (s->pinst.empty()) s->pinst.assign((size_t)s->B, s->p);
    s->pinst[(size_t)b] = *p;
  }
  drop_graphs(s);  // constants are baked into captured launches
  if (int rc = choose_mode(s)) return rc;
  select_kernels(s);  // the fast mode decides whether cr_kernel applies
  return RD_OK;
}

int rd_paint_phi(rd_sim* s, int32_t b, const rd_rect* r, double value) {
  if (!s) return RD_EINVAL;
  if (b < -1 || b >= s->B) return set_err(s, RD_ERANGE, "instance %d out of range", b);
  if (!std::isfinite(value)) return set_err(s, RD_ENONFINITE, "phi value is not finite");
  int64_t y0 = 0, y1 = s->Hg, x0 = 0, x1 = s->W;
  if (r) y0 = r->y0, y1 = r->y1, x0 = r->x0, x1 = r->x1;
  // global rows -> local rows that this handle stores (owned + ghost rows)
  const int64_t lo = std::max<int64_t>(std::max<int64_t>(y0, 0) - s->grow0, s->r_lo);
  const int64_t hi = std::min<int64_t>(std::min<int64_t>(y1, s->Hg) - s->grow0, s->r_hi);
  x0 = std::max<int64_t>(x0, 0);
  x1 = std::min<int64_t>(x1, s->W);
  if (lo < hi && x0 < x1) {
    const int32_t b0 = b < 0 ? 0 : b, nb = b < 0 ? (int32_t)s->B : 1;
    const unsigned grid = (unsigned)std::min<int64_t>(((hi - lo) * (x1 - x0) + 255) / 256, s->num_sms * 16);
    for (int32_t i = b0; i < b0 + nb; ++i) {
      if (s->pal_ok && !s->pal.empty()) palette_add(s, i, value);
      if (s->esz == 4)
        rdk::paint_kernel<float><<<grid, 256, 0, s->stream>>>(origin<float>(s, s->phi), s->plane_stride, s->pitch,
                                                              (int32_t)lo, (int32_t)hi, x0, x1, (float)value, i);
      else
        rdk::paint_kernel<double><<<grid, 256, 0, s->stream>>>(origin<double>(s, s->phi), s->plane_stride, s->pitch,
                                                               (int32_t)lo, (int32_t)hi, x0, x1, value, i);
      RD_CUDA(s, cudaGetLastError());
      s->st.launches++;
    }
  }
  s->phi_class_known = false;  // re-derived at the next run_range (ensure_phi_class)
  return launch_mirror(s, s->phi, nullptr, nullptr, s->r_lo, s->r_hi);
}

int rd_fill_noise(rd_sim* s, int32_t b, uint32_t planes, uint64_t seed, double amplitude) {
  if (!s) return RD_EINVAL;
  if (b < -1 || b >= s->B) return set_err(s, RD_ERANGE, "instance %d out of range", b);
  if (!(planes & 3u) || (planes & ~3u)) return set_err(s, RD_EINVAL, "planes must be a mask of 1 (u) and 2 (v)");
  if (!std::isfinite(amplitude)) return set_err(s, RD_ENONFINITE, "amplitude is not finite");
  const int32_t b0 = b < 0 ? 0 : b, nb = b < 0 ? (int32_t)s->B : 1;
  for (int32_t i = b0; i < b0 + nb; ++i) {
    for (int p = 0; p < 2; ++p) {
      if (!(planes & (1u << p))) continue;
      void* plane = p == 0 ? s->u[s->cur] : s->v[s->cur];
      const unsigned long long tag = (unsigned long long)p << 62;
      const unsigned grid = (unsigned)std::min<int64_t>(((s->r_hi - s->r_lo) * s->W + 255) / 256, s->num_sms * 16);
      if (s->esz == 4)
        rdk::noise_kernel<float><<<grid, 256, 0, s->stream>>>(origin<float>(s, plane), s->plane_stride, s->pitch,
                                                              s->r_lo, s->r_hi, (int32_t)s->W, s->grow0, seed, tag,
                                                              amplitude, i);
      else
        rdk::noise_kernel<double><<<grid, 256, 0, s->stream>>>(origin<double>(s, plane), s->plane_stride, s->pitch,
                                                               s->r_lo, s->r_hi, (int32_t)s->W, s->grow0, seed, tag,
                                                               amplitude, i);
      RD_CUDA(s, cudaGetLastError());
      s->st.launches++;
    }
  }
  void* p0 = (planes & 1u) ? s->u[s->cur] : s->v[s->cur];
  void* p1 = (planes == 3u) ? s->v[s->cur] : nullptr;
  return launch_mirror(s, p0, p1, nullptr, s->r_lo, s->r_hi);
}

int rd_init_rest(rd_sim* s, int32_t b) {
  if (!s) return RD_EINVAL;
  if (b < -1 || b >= s->B) return set_err(s, RD_ERANGE, "instance %d out of range", b);
  const int32_t b0 = b < 0 ? 0 : b, nb = b < 0 ? (int32_t)s->B : 1;
  for (int32_t i = b0; i < b0 + nb; ++i) {
    const rd_params& p = s->pinst.empty() ? s->p : s->pinst[(size_t)i];
    dim3 grid((unsigned)std::min<int64_t>(((s->r_hi - s->r_lo) * s->W + 255) / 256, s->num_sms * 8), 1);
    if (s->esz == 4)
      rdk::rest_fill_kernel<float><<<grid, 256, 0, s->stream>>>(origin<float>(s, s->phi), origin<float>(s, s->u[s->cur]),
                                                                origin<float>(s, s->v[s->cur]), s->plane_stride,
                                                                s->pitch, s->r_lo, s->r_hi, (int32_t)s->W, p.f, p.q, i);
    else
      rdk::rest_fill_kernel<double><<<grid, 256, 0, s->stream>>>(
          origin<double>(s, s->phi), origin<double>(s, s->u[s->cur]), origin<double>(s, s->v[s->cur]),
          s->plane_stride, s->pitch, s->r_lo, s->r_hi, (int32_t)s->W, p.f, p.q, i);
    RD_CUDA(s, cudaGetLastError());
    s->st.launches++;
  }
  return launch_mirror(s, s->u[s->cur], s->v[s->cur], nullptr, s->r_lo, s->r_hi);
}

int rd_timelapse(rd_sim* s, int32_t stride) {
  if (!s) return RD_EINVAL;
  if (stride < 0) return set_err(s, RD_EINVAL, "stride must be >= 0");
  s->tl_stride = stride;
  drop_graphs(s);
  if (stride == 0) return RD_OK;
  const size_t bytes = (size_t)s->B * s->plane_stride * s->esz;
  if (!s->tl) {
    RD_CUDA(s, cudaMalloc(&s->tl, bytes));
    if (!(s->g.flags & RD_NO_CHECKPOINT)) RD_CUDA(s, cudaMalloc(&s->ck_tl, bytes));
  }
  const int64_t n = (int64_t)s->B * s->plane_stride;
  if (s->esz == 4)
    rdk::fill_kernel<float><<<s->num_sms * 4, 256, 0, s->stream>>>((float*)s->tl, n, -INFINITY);
  else
    rdk::fill_kernel<double><<<s->num_sms * 4, 256, 0, s->stream>>>((double*)s->tl, n, -INFINITY);
  RD_CUDA(s, cudaGetLastError());
  s->st.launches++;
  return RD_OK;
}

int rd_read_timelapse(rd_sim* s, int32_t b, void* out) {
  if (!s || !out) return RD_EINVAL;
  if (int rc = check_b(s, b)) return rc;
  if (!s->tl) return set_err(s, RD_ERANGE, "no timelapse enabled (rd_timelapse)");
  RD_CUDA(s, cudaMemcpy2DAsync(out, s->W * s->esz, plane_ptr(s, s->tl, b, 0), s->pitch * s->esz, s->W * s->esz, s->H,
                               cudaMemcpyDeviceToHost, s->stream));
  RD_CUDA(s, cudaStreamSynchronize(s->stream));
  return RD_OK;
}

int rd_row_ptr(rd_sim* s, int32_t b, int32_t plane, int64_t row, void** ptr, int64_t* pitch_bytes) {
  if (!s || !ptr) return RD_EINVAL;
  if (int rc = check_b(s, b)) return rc;
  if (plane != 0 && plane != 1) return set_err(s, RD_EINVAL, "plane must be 0 (u) or 1 (v)");
  if (row < -s->halo || row >= s->H + s->halo) return set_err(s, RD_ERANGE, "row %lld outside the slab", (long long)row);
  // start of the row's storage (ghost columns included): a block of rows is
  // a contiguous (rows x pitch) byte range
  *ptr = plane_ptr(s, plane == 0 ? s->u[s->cur] : s->v[s->cur], b, row) - s->col_off * s->esz;
  if (pitch_bytes) *pitch_bytes = s->pitch * (int64_t)s->esz;
  return RD_OK;
}

int rd_set_profiling(rd_sim* s, int32_t on) {
  if (!s) return RD_EINVAL;
  s->profiling = on != 0;
  return RD_OK;
}

int rd_get_stats(rd_sim* s, rd_stats* out) {
  if (!s || !out) return RD_EINVAL;
  if (s->ev_used) {
    RD_CUDA(s, cudaStreamSynchronize(s->stream));
    for (size_t i = 0; i < s->ev_used; ++i) {
      float ms = 0;
      RD_CUDA(s, cudaEventElapsedTime(&ms, s->ev_pool[i].first, s->ev_pool[i].second));
      s->acc_ms += ms;
    }
    s->acc_timed += (int64_t)s->ev_used;
    s->ev_used = 0;
  }
  *out = s->st;
  out->step_kernel_ms = s->acc_ms;
  out->timed_launches = s->acc_timed;
  out->tb_depth = s->K;
  out->phi_uniform = (s->phi_class_known && s->phi_uniform) ? 1 : 0;
  out->arith_mode = (s->g.flags & RD_NO_CHECKPOINT) ? rdk::MODE_PRECISE : s->fast_mode;
  out->kernel = (s->use_gz && !(s->g.flags & RD_NO_CHECKPOINT))
                    ? 3
                    : ((s->use_cr && !(s->g.flags & RD_NO_CHECKPOINT)) ? 2 : (s->use_lp ? 1 : 0));
  return RD_OK;
}

int rd_reset_stats(rd_sim* s) {
  if (!s) return RD_EINVAL;
  RD_CUDA(s, cudaStreamSynchronize(s->stream));
  s->st = rd_stats{};
  s->acc_ms = 0;
  s->acc_timed = 0;
  s->ev_used = 0;
  return RD_OK;
}

}  // extern "C"

#include "rd_dist.cuh"
