/*
 * rd_oracle.h — plain CPU oracle for the RDCSim Oregonator hot path.
 *
 * TEST INFRASTRUCTURE, NOT PRODUCT CODE. Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, constant or helper with the CUDA path
 * (paper_1901_06535_b200/csrc, include/rd.h).
 *
 * What it computes (§2, lines 87-125):
 *   Eq. 1   du/dt = (1/eps)[u - u^2 - (f v + phi)(u-q)/(u+q)] + Du Lap(u)
 *                            dv/dt = u - v
 *   Table 1 default parameters
 *   PAPER.md:122-124         explicit forward Euler, dt; five-node Laplacian, dx
 *   PAPER.md:124-125         stimulation: u := 1.0 on stimulated pixels
 * with the readings listed in DESIGN.md §3 (no-flux ghost = edge cell,
 * canonical expression tree, constants rounded once, events before the step
 * they are stamped with, probes latched every `stride` steps).
 *
 * Pins (tests/test_oracle_pins.py): SPEC worked examples (Laplacian impulse,
 * reaction terms, disc count), the closed-form homogeneous fixed point (cubic),
 * the Euler linearisation eigenvalues, a discrete-cosine eigenmode of the
 * Neumann Laplacian, diffusion-only conservation and maximum principle, D4
 * symmetry, first-order convergence, the paper's AND/diode outcomes.
 * Parity unpinned: the long-time dynamics of chaotic refractory-wake cells
 * beyond bitwise agreement (no closed form exists).
 */
#ifndef RD_ORACLE_H
#define RD_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_OK = 0, ORC_EINVAL = -1, ORC_ENONFINITE = -4, ORC_ENOMEM = -7 };
enum { ORC_REACTION_OFF = 1u };
enum { ORC_DISC = 1, ORC_RECT = 2, ORC_HALF_DISC = 3 };
enum { ORC_SHAPE_MASK_PHI = 1u };

typedef struct {
  double eps, f, q, Du, dt, dx;
} orc_params;

/* Stimulus shape (integer geometry in half-cell units, R-14):
 *   DISC      (2i-cy2)^2 + (2j-cx2)^2 <= 4 r^2
 *   RECT      y0 <= i < y1 and x0 <= j < x1
 *   HALF_DISC DISC and (2j-cx2)*dx + (2i-cy2)*dy >= 0, dir 0:+x 1:+y 2:-x 3:-y
 * flags & ORC_SHAPE_MASK_PHI: write only cells whose phi == mask_phi.      */
typedef struct {
  int32_t kind;
  int32_t dir;
  int64_t cy2, cx2, r;
  int64_t y0, x0, y1, x1;
  uint32_t flags;
  uint32_t pad_;
  double mask_phi;
} orc_shape;

typedef struct {
  int64_t y0, x0, y1, x1;
} orc_rect;

typedef struct {
  orc_shape shape;
  double value;
  int64_t at_step;
} orc_event;

typedef struct {
  orc_rect rect;
  double threshold;
  int64_t stride;
} orc_probe;

typedef struct {
  int64_t step, i, j;
} orc_fault;

void orc_params_default(orc_params* p);
double orc_rest_state(double phi, const orc_params* p);
int orc_shape_contains(const orc_shape* s, int64_t i, int64_t j);
int orc_num_threads(void);
void orc_set_num_threads(int n);

/* Per precision: SFX = f64 (reference) and f32 (the fp32 mode). */
#define ORC_DECL(T, SFX)                                                                        \
  double orc_reaction_##SFX(double u, double v, double phi, const orc_params* p, double* dv);   \
  void orc_laplacian_##SFX(int64_t H, int64_t W, const T* u, T* out, const orc_params* p);      \
  void orc_step_##SFX(int64_t H, int64_t W, const T* u, const T* v, const T* phi, T* uo, T* vo, \
                      const orc_params* p, uint32_t flags);                                      \
  int64_t orc_stamp_##SFX(int64_t H, int64_t W, T* u, const T* phi, const orc_shape* s,         \
                          double value);                                                         \
  double orc_probe_max_##SFX(int64_t H, int64_t W, const T* u, const orc_rect* r);              \
  int orc_run_##SFX(int64_t H, int64_t W, T* u, T* v, const T* phi, const orc_params* p,        \
                    uint32_t flags, int64_t step0, int64_t n_steps, const orc_event* events,     \
                    int64_t n_events, const orc_probe* probes, int64_t n_probes,                 \
                    int64_t* first_fire, orc_fault* fault, int64_t tl_stride, T* tl_max);        \
  void orc_timelapse_record_##SFX(int64_t H, int64_t W, const T* u, T* max_u);                   \
  void orc_rest_fill_##SFX(int64_t H, int64_t W, const T* phi, T* u, T* v, const orc_params* p);
ORC_DECL(double, f64)
ORC_DECL(float, f32)
#undef ORC_DECL

#ifdef __cplusplus
}
#endif
#endif
