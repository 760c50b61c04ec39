/*
 * rd.h — C ABI of the B200-native Oregonator reaction-diffusion engine.
 *
 * The hot path is explicit forward-Euler
 * time stepping of the two-variable Oregonator model, §2 Eq. 1
 * (PAPER.md:89-94):
 *     du/dt = (1/eps) [u - u^2 - (f v + phi(x,y)) (u - q)/(u + q)] + Du Lap(u)
 *     dv/dt = u - v
 * integrated "using an explicit forward Euler integration, with timestep dt
 * and five-node discrete Laplace operator with grid spacing dx"
 * (PAPER.md:122-124), with "catalytic stimulation ... by setting the
 * excitatory concentration (u) of stimulated pixels to 1.0".
 * Default parameters: Table 1.
 *
 * All entry points are plain C: opaque handle, plain host/device pointers and
 * sizes, int status codes (RD_OK = 0 or a negative RD_E* code). The handle
 * owns all device memory it allocates. Handles are not thread-safe (one
 * writer per handle). Work is issued on the handle's CUDA stream; every call
 * that returns data to the host synchronises that stream. A failing call
 * leaves a message for rd_last_error().
 *
 * Numerics: every binary floating-point operation is rounded
 * separately in the handle's precision (no FMA contraction), in the order
 *   L  = (((N + S) + (E + W)) - 4*C) * INV_DX2
 *   r  = (C - Q) / (C + Q)                          (IEEE division)
 *   R  = (C - C*C) - ((F*v + phi) * r)
 *   u' = C + DT * ((R * INV_EPS) + (DU * L))        v' = v + DT * (C - v)
 * with out-of-grid neighbours := the edge cell (no-flux), and every constant
 * computed in fp64 from rd_params and rounded once to the precision.
 * Results are bitwise independent of temporal-blocking depth, batching,
 * rd_step splitting and slab decomposition.
 */
#ifndef RD_H
#define RD_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RD_ABI_VERSION 2

typedef struct rd_sim rd_sim; /* opaque handle */

/* ---- status codes ---- */
enum {
  RD_OK = 0,
  RD_EINVAL = -1,      /* null pointer, dims < 3, batch < 1, bad kind/dtype, radius < 0 */
  RD_EPARAM = -2,      /* parameter invariants violated: all > 0, q < 1, dt*Du/dx^2 < 0.25 */
  RD_ERANGE = -3,      /* probe rect empty/outside the grid, at_step < current step, instance out of range */
  RD_ENONFINITE = -4,  /* non-finite input, or produced during rd_step; see rd_last_error / rd_get_fault */
  RD_ECUDA = -5,       /* CUDA runtime error (message has the CUDA error string) */
  RD_ENCCL = -6,       /* NCCL missing (dlopen libnccl.so.2) or an NCCL call failed (rd_create_dist) */
  RD_ENOMEM = -7       /* device or host allocation failed */
};

/* ---- precisions ---- */
enum { RD_F32 = 1, RD_F64 = 2 };

/* ---- rd_grid.flags ---- */
enum {
  RD_REACTION_OFF = 1u,   /* integrate u' = u + dt*Du*L, v' = v (diffusion-only conservation pin) */
  RD_NO_CHECKPOINT = 2u,  /* skip the per-rd_step checkpoint: faults are then reported at k-block
                             granularity and the fields are left at the end of the failing block */
  RD_NO_GRAPH = 4u        /* never replay rd_step segments through CUDA graphs */
};

/* ---- stimulus shape kinds ---- */
enum { RD_DISC = 1, RD_RECT = 2, RD_HALF_DISC = 3 };
enum { RD_SHAPE_MASK_PHI = 1u }; /* rd_shape.flags: write only cells whose phi == mask_phi */

/* Model parameters of Eq. 1 and its discretisation; Table 1 defaults via
 * rd_params_default. phi is per cell (the phi map). */
typedef struct {
  double eps, f, q, Du, dt, dx;
} rd_params;

/* Grid description. An instance is a height x width row-major grid; `batch`
 * independent instances (e.g. the AND-gate truth-table rows, BASELINE.json
 * configs[1]) are stepped together. tb_depth = time steps per HBM round trip
 * (0 = automatic; results do not depend on it). pitch = elements between
 * rows in device memory (0 = automatic, a multiple of 32). */
typedef struct {
  int64_t width, height;
  int32_t batch;
  int32_t dtype;    /* RD_F32 | RD_F64 */
  int32_t tb_depth; /* 0 = auto, else 1..RD_MAX_TB */
  uint32_t flags;   /* RD_REACTION_OFF | RD_NO_CHECKPOINT | RD_NO_GRAPH */
  int64_t pitch;
} rd_grid;

#define RD_MAX_TB 8

/* Stimulus shape, integer geometry (R-14). Cell (i, j) = (row, col).
 *   RD_DISC       (2i - cy2)^2 + (2j - cx2)^2 <= 4 r^2   (centre in half cells)
 *   RD_RECT       y0 <= i < y1 and x0 <= j < x1
 *   RD_HALF_DISC  the disc and (2j-cx2)*dx + (2i-cy2)*dy >= 0,
 *                 (dx,dy) = (1,0),(0,1),(-1,0),(0,-1) for dir 0..3
 * Shapes are clipped to the grid. With RD_SHAPE_MASK_PHI only
 * cells whose phi equals mask_phi (rounded to the precision) are written. */
typedef struct {
  int32_t kind;
  int32_t dir;
  int64_t cy2, cx2, r;
  int64_t y0, x0, y1, x1;
  uint32_t flags;
  uint32_t reserved;
  double mask_phi;
} rd_shape;

/* Axis-aligned probe rectangle [y0, y1) x [x0, x1). */
typedef struct {
  int64_t y0, x0, y1, x1;
} rd_rect;

/* First non-finite cell reported by rd_step (step after which it appeared). */
typedef struct {
  int64_t step;
  int32_t b;
  int32_t pad;
  int64_t i, j;
} rd_fault;

/* Kernel-level statistics for the measurement harness (bench.py). */
typedef struct {
  int64_t launches;        /* kernels this library launched since creation / last reset */
  int64_t step_launches;   /* of which stencil (time-step) kernels */
  int64_t cell_updates;    /* cell-updates performed by the stencil kernels (owned cells x steps) */
  double step_kernel_ms;   /* summed CUDA-event durations of stencil launches (profiling on) */
  int64_t timed_launches;  /* stencil launches covered by step_kernel_ms */
  int32_t tb_depth;        /* temporal-blocking depth in use */
  int32_t phi_uniform;     /* 1: the phi map is one value over every instance (checked on the device after
                              each change of phi), so tb_kernel takes it as a kernel parameter instead of
                              streaming the plane (plain single-GPU handles; results are identical) */
  int64_t replays;         /* rd_step calls replayed from the checkpoint (fault or fast-division guard) */
  int32_t arith_mode;      /* 0 precise (canonical ops), 2 exact rewrites, 3 exact rewrites + certified 4-op fp32 division,
                              4 as 3 without the min|C+q| guard (fp32 q >= 2^-35) */
  int32_t kernel;          /* stencil kernel of the fast path: 0 tb_kernel (temporal-blocked streaming),
                              1 lp_kernel (level-parallel), 2 cr_kernel (cluster-resident, a8),
                              3 gz_kernel (whole-chip tiles, a8) */
} rd_stats;

/* Where a handle's rows sit (rd_get_geometry). For rd_create / rd_create_device
 * handles row0 = 0, height = height_global, rank = 0, world = 1. */
enum { RD_TRANSPORT_NONE = 0, RD_TRANSPORT_P2P = 1, RD_TRANSPORT_NCCL = 2, RD_TRANSPORT_LOCAL = 3 };
typedef struct {
  int64_t width, height;  /* columns; rows this handle owns */
  int64_t height_global;  /* rows of the whole grid */
  int64_t row0;           /* global row of owned row 0 */
  int64_t pitch;          /* elements between rows in device memory (rd_field_ptr) */
  int64_t phi_rows_lo, phi_rows_hi; /* local rows [lo, hi) a create call's phi buffer covers */
  int64_t exchanges;      /* halo exchanges performed (dist handles) */
  int32_t batch, dtype, halo, tb_depth;
  int32_t rank, world;    /* dist handles: this rank of world; else 0 of 1 */
  int32_t transport;      /* RD_TRANSPORT_*: how a dist handle's halos travel */
  int32_t flag_selftest;  /* multi-process dist handles, world > 1: the create-time test of the stream-ordered
                             flag words across processes: 1 passed (P2P transport), -1 failed (NCCL send/recv
                             instead); 0 = not run (world 1, in-process group, mapping failed earlier) */
} rd_geometry;

/* ---- lifecycle ---- */

/* Table 1 defaults: eps=0.0243, f=1.4, q=0.002, Du=0.45, dt=0.001, dx=0.25. */
void rd_params_default(rd_params* p);

/* Create a handle. phi_map: HOST buffer [batch][height][width] of the grid's
 * dtype (copied; must be finite), or NULL for phi = 0 everywhere (then paint
 * it with rd_paint_phi). u = v = 0 initially (R-10).
 * Errors: RD_EINVAL, RD_EPARAM, RD_ENONFINITE (phi), RD_ENOMEM, RD_ECUDA. */
int rd_create(const rd_grid* grid, const rd_params* params, const void* phi_map, struct rd_sim** out);

/* Release all device memory and the stream (if owned). NULL is a no-op.
 * Collective for rd_create_dist handles (every rank destroys its handle; no
 * rank frees its planes while a neighbour may still reach them). A caller
 * arena (rd_create_device) is not freed. */
int rd_destroy(struct rd_sim* sim);

/* ---- PyTorch (caller-owned) device memory: SURVEY.md §8(b) rd_create_device ----
 * The planes live in ONE caller allocation (e.g. a torch uint8 CUDA tensor of
 * rd_arena_bytes bytes, 256-byte aligned) that the handle lays out itself:
 * u ping-pong, v ping-pong, phi and the checkpoint, each [batch][rows][pitch]
 * with mirrored ghost margins -- the no-flux boundary and tb_kernel's single
 * 4-D tensor map per row need that layout, so dense H x W
 * tensors cannot be adopted as they are. rd_field_ptr gives each plane's
 * (row 0, column 0) and pitch, for zero-copy strided views.
 *   rd_arena_bytes    bytes the grid needs (no device work).
 *   rd_create_device  as rd_create, with the caller's arena (kept alive by the
 *                     caller until rd_destroy) and phi_dev a DEVICE map
 *                     [batch][height][width] of dtype (or NULL = 0).
 *   rd_field_ptr      instance b's current u (plane 0), v (1) or phi (2):
 *                     device pointer of cell (0, 0), row pitch in elements.
 *                     Valid until the next rd_step (u, v ping-pong). Once phi's
 *                     pointer has been handed out the handle assumes nothing
 *                     about phi's values (rd_stats.phi_uniform stays 0).
 * Errors: RD_EINVAL (NULL / misaligned / too small arena, bad plane),
 * RD_ERANGE (b), plus those of rd_create. */
int rd_arena_bytes(const rd_grid* grid, size_t* bytes);
int rd_create_device(const rd_grid* grid, const rd_params* params, void* arena, size_t arena_bytes,
                     const void* phi_dev, struct rd_sim** out);
int rd_field_ptr(struct rd_sim* sim, int32_t b, int32_t plane, void** ptr, int64_t* pitch_elems);
int rd_get_geometry(const struct rd_sim* sim, rd_geometry* out);

/* ---- multi-GPU row slabs run by the library ----
 * BASELINE.json north_star: "a row-slab domain decomposition across the 8
 * GPUs of one box, with halo exchange by NCCL send/recv or CUDA P2P over
 * NVLink overlapped with interior compute" (the paper itself runs on one
 * tablet). One handle per rank: one process per GPU, or
 * one host thread per rank of one process.
 *   rd_dist_unique_id  a rendezvous id for ranks in several processes (an
 *                      NCCL unique id; make it on one rank and broadcast the
 *                      128 bytes, e.g. with torch.distributed). RD_ENCCL if
 *                      libnccl.so.2 cannot be loaded.
 *   rd_dist_shm_id     a rendezvous id for ranks that are processes of THIS
 *                      box, without NCCL: the rendezvous and the per-rd_step
 *                      flag reduction go through a POSIX shared-memory
 *                      segment the call creates (unlinked once every rank has
 *                      joined); halos travel by the same copy-engine push.
 *                      Ranks may share a device (that is how the
 *                      cross-process protocol is tested on one GPU). There is
 *                      no send/recv fallback: rd_create_dist fails (RD_ECUDA)
 *                      if a peer mapping or its flag words do not work. A
 *                      rank that waits longer than RD_DIST_TIMEOUT_S (300)
 *                      for the others fails with RD_ENCCL, as do they.
 *   rd_dist_local_id   a rendezvous id for ranks that are host threads of
 *                      THIS process (no NCCL; ranks may share a device, e.g.
 *                      to test on one GPU; distinct devices need peer access).
 *   rd_create_dist     rank `rank` of `world` (collective: every rank calls it
 *                      with the same global grid, params and id; returns when
 *                      all have joined). The rank owns global rows [row0,
 *                      row0 + rows): rows = H/G, the first H % G ranks one
 *                      more (rd_get_geometry). phi_rows: HOST
 *                      [batch][rows][width] of the OWNED rows (NULL = 0; the
 *                      ghost rows come from the neighbours). halo = the
 *                      temporal-blocking depth (grid->tb_depth, 0 = 4); every
 *                      slab needs rows >= halo.
 * On a dist handle, rd_step(n) runs the whole super-step inside the library:
 * a checkpoint; blocks of <= halo steps, each with its halo exchange (u and v
 * send rows straight into the neighbours' ghost rows by copy-engine
 * cudaMemcpyAsync over CUDA IPC / peer mappings, ordered by stream-ordered
 * counters, overlapped with the interior rows; RD_DIST_TRANSPORT=nccl, a
 * failed peer mapping, or a failed create-time test of those counters between
 * the processes selects grouped ncclSend/ncclRecv instead); one fault /
 * guard flag OR over the ranks (ncclAllReduce); on a fault every rank replays
 * step by step and stops at the first failing step, reporting the global first
 * cell. Results are bitwise those of one rd_create handle of the whole grid.
 * Collective calls (every rank, same arguments): rd_create_dist, rd_step,
 * rd_stimulate, rd_probe_latch, rd_timelapse, rd_set_params, rd_probe (global
 * max), rd_probe_result (global first firing), rd_destroy. Stimuli, probes,
 * timelapse and parameters decide the launch sequence, so rd_step checks a
 * digest of them on all ranks (RD_EINVAL if they differ). Local calls:
 * rd_write_fields / rd_read_fields (owned rows [rows][width]), rd_paint_phi,
 * rd_fill_noise, rd_init_rest (global coordinates). The low-level slab calls
 * (rd_step_begin/finish, rd_step_unchecked, rd_checkpoint/restore,
 * rd_push_ghosts, rd_set_peer) are refused (RD_EINVAL).
 * Errors: RD_EINVAL (arguments, unknown local id, slab thinner than the
 * halo), RD_ENCCL, RD_ECUDA, RD_ENOMEM, RD_ENONFINITE (phi). */
int rd_dist_unique_id(uint8_t id[128]);
int rd_dist_local_id(uint8_t id[128]);
int rd_dist_shm_id(uint8_t id[128]);
int rd_create_dist(const rd_grid* global, const rd_params* params, const void* phi_rows, int32_t rank,
                   int32_t world, const uint8_t id[128], struct rd_sim** out);

/* Use an external CUDA stream (cudaStream_t, e.g. torch's current stream)
 * for all subsequent work; NULL reverts to the handle's own (non-blocking)
 * stream. To share the legacy default stream pass cudaStreamLegacy (0x1). */
int rd_set_stream(struct rd_sim* sim, void* cuda_stream);

/* ---- state I/O (HOST buffers, [height][width] of dtype, row-major) ---- */

/* Overwrite instance b's u and/or v (either may be NULL). Values must be finite. */
int rd_write_fields(struct rd_sim* sim, int32_t b, const void* u, const void* v);

/* Copy instance b's current u and/or v to host (either may be NULL). Syncs. */
int rd_read_fields(struct rd_sim* sim, int32_t b, void* u_out, void* v_out);

/* Same with DEVICE buffers (pitch = width, dtype elements); async on the stream. */
int rd_read_fields_device(struct rd_sim* sim, int32_t b, void* u_out, void* v_out);
int rd_write_fields_device(struct rd_sim* sim, int32_t b, const void* u, const void* v);

/* Asynchronous host I/O: the same copies as rd_write_fields / rd_read_fields,
 * overlapped with rd_step on the copy engines, so that a caller who runs one
 * job after another on a handle (new fields in, n steps, fields out: the
 * paper's interactive use, as a batch loop) pays the host
 * copies only once per pipeline, not once per job. Host buffers should be
 * pinned (pageable memory works but copies synchronously) and are
 * [height][width] of dtype, as above. The first call allocates two dense
 * staging blocks of 2 * batch * height * width elements on the device.
 *   rd_write_fields_async  start uploading instance b's u and/or v into the
 *       staging block on the handle's upload stream and return. The handle's
 *       state is NOT changed; rd_step keeps working on the current fields. The
 *       host buffers must stay valid until rd_commit_fields or rd_io_wait
 *       returns.
 *   rd_commit_fields       wait for the uploads staged so far, check them
 *       (RD_ENONFINITE: nothing is written and the staged set is dropped) and
 *       copy them into the current fields, device to device, on the handle's
 *       stream. Syncs that stream. No staged upload: a no-op.
 *   rd_read_fields_async   snapshot instance b's current u and/or v into the
 *       second staging block (device to device, stream-ordered after the
 *       preceding rd_step) and start copying the snapshot to the host on the
 *       download stream; returns at once, and a following rd_step or
 *       rd_commit_fields does not disturb the snapshot. The host buffers hold
 *       the fields after rd_io_wait returns.
 *   rd_io_wait             block until every upload and download started so
 *       far has finished.
 * Errors: RD_ERANGE (b), RD_ENOMEM (staging blocks), RD_ECUDA, RD_ENONFINITE
 * (rd_commit_fields). rd_destroy waits for copies in flight. */
int rd_write_fields_async(struct rd_sim* sim, int32_t b, const void* u, const void* v);
int rd_commit_fields(struct rd_sim* sim);
int rd_read_fields_async(struct rd_sim* sim, int32_t b, void* u_out, void* v_out);
int rd_io_wait(struct rd_sim* sim);

/* ---- stimulation (a1) ---- */

/* Schedule u := value on the shape's cells of instance b (-1 = all) before
 * step at_step+1 is integrated, i.e. after at_step steps have completed
 * (SPEC.md:438). Events at the same step apply in submission order.
 * Errors: RD_EINVAL (shape), RD_ERANGE (at_step < current step, b out of range). */
int rd_stimulate(struct rd_sim* sim, int32_t b, const rd_shape* shape, double value, int64_t at_step);

/* ---- time stepping (a2-a8) ---- */

/* Advance all instances by n >= 0 steps. Applies due
 * stimuli, latches probes after every multiple of their stride, and checks
 * for non-finite cells. Returns RD_ENONFINITE if any cell became non-finite:
 * then (unless RD_NO_CHECKPOINT) the handle holds the state right after the
 * first failing step, rd_get_step() is that step and rd_get_fault() names the
 * first non-finite cell in (b, i, j) row-major order. rd_step(a); rd_step(b)
 * is bitwise identical to rd_step(a+b). */
int rd_step(struct rd_sim* sim, int64_t n);

/* Deferred health checking (slab super-steps): a checkpoint,
 * any number of unchecked blocks, one flag read, and -- if a flag is set --
 * restore + an exact step-by-step rd_step replay by the caller.
 *   rd_checkpoint      save u, v, probe latches, timelapse, step and pending
 *                      stimuli (async on the stream; RD_EINVAL with
 *                      RD_NO_CHECKPOINT).
 *   rd_step_unchecked  advance n steps with the fast kernels: no checkpoint,
 *                      no flag read, no host synchronisation.
 *   rd_read_flags      sync; *nonfinite = a non-finite cell was produced,
 *                      *inexact = the fast division's guard tripped (results
 *                      since the checkpoint must be replayed); clears both.
 *   rd_restore         return to the last checkpoint. */
int rd_checkpoint(struct rd_sim* sim);

/* Halo exchange overlapped with interior compute (slab
 * handles, same fast kernels as rd_step_unchecked):
 *   rd_step_begin   opens a block of k (1 <= k <= halo) steps: if the block is
 *                   one plain launch (k <= the handle's depth, no stimulus due
 *                   in [step, step+k), no probe or timelapse sample strictly
 *                   inside) it launches the interior rows -- those at least k
 *                   rows from any exchanged ghost row, which read owned rows
 *                   only -- and sets *started = 1; otherwise *started = 0,
 *                   nothing is launched, and the caller steps the block with
 *                   rd_step_unchecked once the exchange has landed.
 *   rd_step_finish  after the exchange of the block's input rows has landed
 *                   (on the handle's stream): launches the edge bands, flips
 *                   the buffers, refreshes the mirrors, advances the step and
 *                   runs probes due at the block's end.
 * The exchange reads rows [0, halo) and [rows-halo, rows) and writes the
 * ghost rows of the input buffer; the interior launch reads neither range's
 * ghosts and writes only the output buffer, so both may run concurrently.
 * flags: RD_BLOCK_PUSH -- peer-memory exchange: the
 * block's edge bands also store their send rows (owned rows [0, halo) and
 * [rows-halo, rows)) straight into the neighbours' ghost rows of their next
 * input buffer (rd_set_peer), so no separate exchange follows the block;
 * rd_step_finish first refreshes the mirrored columns of the ghost rows the
 * neighbours stored into. Push blocks need k == halo (else *started = 0).
 * The caller orders the ranks: between rd_step_begin and rd_step_finish the
 * handle's stream must wait until both neighbours have finished the previous
 * block (rd_stream_wait on a flag they rd_stream_signal after theirs).
 * Errors: RD_EINVAL (not a slab handle, block already open / not open,
 * RD_BLOCK_PUSH without registered neighbours), RD_ERANGE (k), RD_ECUDA. */
#define RD_BLOCK_PUSH 1
int rd_step_begin(struct rd_sim* sim, int64_t k, int32_t flags, int32_t* started);
int rd_step_finish(struct rd_sim* sim);

/* Peer-memory halo exchange, slab handles.
 *   rd_plane_origins  this handle's (row 0, col 0) device pointers of u and v
 *                     for both buffers, and its instance stride in bytes (to
 *                     hand to the neighbours; on another GPU they map them
 *                     with CUDA IPC).
 *   rd_set_peer       register the neighbour above (side 0) or below (side 1)
 *                     by those pointers (valid in this process), its owned
 *                     rows (>= halo) and instance stride; the same width (and
 *                     so the same row pitch) is assumed. u0 == NULL clears.
 *   rd_push_ghosts    copy this handle's send rows of the current buffer
 *                     (row storage, mirrored columns included) into the
 *                     registered neighbours' ghost rows of their current
 *                     buffer (the first exchange of a super-step).
 *   rd_stream_signal  stream-ordered write of `value` to the 32-bit device
 *                     word `flag` (e.g. a neighbour's, mapped here).
 *   rd_stream_wait    the handle's stream waits until *flag >= value.
 * Errors: RD_EINVAL (arguments, not a slab handle), RD_ECUDA. */
int rd_plane_origins(const struct rd_sim* sim, void** u0, void** u1, void** v0, void** v1,
                     int64_t* plane_stride_bytes);
int rd_set_peer(struct rd_sim* sim, int32_t side, void* u0, void* u1, void* v0, void* v1, int64_t rows,
                int64_t plane_stride_bytes);
int rd_push_ghosts(struct rd_sim* sim);
/* The handle's 32-bit flag word counting pushes received from the neighbour
 * above (side 0) / below (side 1); it lives in the plane allocation, so a
 * neighbour reaches it through the same IPC mapping. */
int rd_flag_ptr(struct rd_sim* sim, int32_t side, void** flag);
/* CUDA IPC of the plane allocation: export writes the 64-byte
 * cudaIpcMemHandle and this process's base address; map opens a neighbour's
 * handle here (peer access enabled lazily) and returns the mapped base -- a
 * neighbour pointer p maps to mapped + (p - its base). Mappings close at
 * rd_destroy. */
int rd_ipc_export(struct rd_sim* sim, void* handle64, void** arena_base);
int rd_ipc_map(struct rd_sim* sim, const void* handle64, void** mapped_base);
int rd_stream_signal(struct rd_sim* sim, void* flag, uint32_t value);
int rd_stream_wait(struct rd_sim* sim, void* flag, uint32_t value);
int rd_step_unchecked(struct rd_sim* sim, int64_t n);
int rd_read_flags(struct rd_sim* sim, int32_t* nonfinite, int32_t* inexact);
int rd_restore(struct rd_sim* sim);

int64_t rd_get_step(const struct rd_sim* sim);
int rd_get_fault(const struct rd_sim* sim, rd_fault* out);

/* ---- probes (a6) ---- */

/* Immediate probe: max of u over rect of instance b; fired = max >= threshold
 * (SPEC.md:243-247). Syncs. */
int rd_probe(struct rd_sim* sim, int32_t b, const rd_rect* rect, double threshold, int32_t* fired,
             double* max_u);

/* Latched probe: evaluated after every step that is a positive multiple of
 * stride, remembers the first such step with
 * max u >= threshold. Returns its id in *id. */
int rd_probe_latch(struct rd_sim* sim, int32_t b, const rd_rect* rect, double threshold, int32_t stride,
                   int32_t* id);

/* First firing step of latched probe id, or -1 if it has not fired. Syncs. */
int rd_probe_result(struct rd_sim* sim, int32_t id, int64_t* first_fire_step);

/* ---- per-instance parameters (batched sweeps) ---- */

/* Set the Eq. 1 parameters (Table 1) of
 * instance b, or of every instance (b = -1, which also drops per-instance
 * sets). Lets one batched launch sweep eps, f, q, Du, dt, dx across
 * instances (e.g. a calibration bisection); phi is already per instance.
 * Validation as rd_create (RD_EPARAM); per-instance sets need batch <= 32
 * (RD_EINVAL). Takes effect from the next rd_step. */
int rd_set_params(struct rd_sim* sim, int32_t b, const rd_params* params);

/* ---- seeded initial state on the device (config 4/5 inputs) ---- */

/* phi := value on the rectangle (global rows/columns, clipped; NULL = the
 * whole grid) of instance b (-1 = all): the per-pixel excitability map of
 * PAPER.md:108-110 built on the device (e.g. a background plus obstacle
 * rectangles, BASELINE.json configs[4]) instead of uploaded. */
int rd_paint_phi(struct rd_sim* sim, int32_t b, const rd_rect* rect, double value);

/* Fill u (planes bit 1) and/or v (bit 2) of instance b (-1 = all) with the
 * counter-based noise of DESIGN.md §4 in GLOBAL coordinates (so slabs of any
 * decomposition get the same values, ghost rows included): value at global
 * cell (i, j) of plane p = ((R(seed, p<<62 | i*W + j) >> 40) * 2^-24) *
 * amplitude, R(s, n) = SM(SM(s) + n), SM = SplitMix64; fp64 then rounded once
 * (BASELINE.json configs[3]: "u,v initialised i.i.d. uniform[0,0.1] from
 * seed"). Input generation only; equals rdinputs.noise_plane bitwise. */
int rd_fill_noise(struct rd_sim* sim, int32_t b, uint32_t planes, uint64_t seed, double amplitude);

/* ---- quiescent initial state ---- */

/* Set u = v = u*(phi) in every cell of instance b (-1 = all): the homogeneous
 * rest state of Eq. 1 for the cell's own phi, i.e. the root of
 * (u - u^2) - (f u + phi)(u - q)/(u + q) = 0 (PAPER.md:91 with v = u), found by
 * fp64 bisection on (0, 1) and rounded once to the dtype (SPEC.md:85-93,
 * :107: "quiescent medium = homogeneous (u*, v*) from steady_state"). */
int rd_init_rest(struct rd_sim* sim, int32_t b);

/* ---- timelapse ---- */

/* Record a timelapse of u ("records a timelapse of the
 * reaction at a rate set by the user ... only the concentration of u is
 * recorded over time"): after every step that is a positive multiple of
 * stride, max_u := pointwise max(max_u, u) (a NaN u never
 * replaces the recorded value). Fused into the stencil kernel's epilogue on
 * sampled steps. stride > 0 enables and resets max_u to -inf; 0 disables.
 * Errors: RD_EINVAL (stride < 0), RD_ENOMEM. */
int rd_timelapse(struct rd_sim* sim, int32_t stride);

/* Copy instance b's max_u to a HOST buffer [height][width] of dtype. Syncs.
 * RD_ERANGE if no timelapse is enabled. */
int rd_read_timelapse(struct rd_sim* sim, int32_t b, void* max_u_out);

/* ---- row slabs for multi-GPU domain decomposition ---- */

/* Create a handle owning rows [row0, row0 + grid->height) of a grid with
 * height_global rows, with `halo` ghost rows above and below (halo >= the
 * temporal-blocking depth). phi_slab: HOST [batch][rows][width] for the rows
 * [max(0,row0-halo), min(height_global, row0+height+halo)). Ghost rows at
 * interior slab edges must be refreshed by the caller after every rd_step
 * (n <= halo per call); global top/bottom edges use the no-flux clamp. */
int rd_create_slab(const rd_grid* grid, const rd_params* params, const void* phi_slab, int64_t row0,
                   int64_t height_global, int32_t halo, struct rd_sim** out);

/* Device pointer to the storage of local row `row` (-halo <= row < height +
 * halo) of instance b's CURRENT u (plane 0) or v (plane 1), and the row pitch
 * in bytes. A row's storage (pitch bytes) holds its cells plus its mirrored
 * ghost columns, so rows [r0, r1) are one contiguous (r1-r0)*pitch byte range
 * (what a halo exchange sends). Valid until the next rd_step (ping-pong). */
int rd_row_ptr(struct rd_sim* sim, int32_t b, int32_t plane, int64_t row, void** ptr, int64_t* pitch_bytes);

/* ---- measurement ---- */

/* Enable per-launch CUDA-event timing of stencil kernels (bench.py only). */
int rd_set_profiling(struct rd_sim* sim, int32_t on);
int rd_get_stats(struct rd_sim* sim, rd_stats* out);
int rd_reset_stats(struct rd_sim* sim);

/* Per-handle message of the last failing call ("" if none). */
const char* rd_last_error(const struct rd_sim* sim);

/* Message of the last failing rd_create* (no handle yet). */
const char* rd_create_error(void);

int32_t rd_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* RD_H */
