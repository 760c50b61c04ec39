/* The multi-GPU calls of the C ABI from plain C (no Python), SURVEY.md §8(b):
 *   1. world = 1 over a real NCCL communicator (rd_dist_unique_id +
 *      rd_create_dist), fp64;
 *   2. a two-rank in-process group (rd_dist_local_id, one pthread per rank,
 *      both ranks on device 0), fp32 and fp64: each rank owns half the rows,
 *      its halo rows travel to the other by cudaMemcpyAsync inside librd;
 *   3. a two-rank group of PROCESSES (rd_dist_shm_id; the ranks are forked
 *      before this process touches CUDA), fp32 and fp64: no NCCL, no Python;
 *      each rank's arena is mapped into the other by CUDA IPC inside librd
 *      and the halo rows are pushed into it (transport P2P, the create-time
 *      flag self-test passing) -- the one-process-per-GPU protocol with both
 *      processes on device 0;
 * each compared with the oracle's C library on the whole grid, bitwise.
 * Test program only: it links the oracle (tests/ may), the product does not.
 *   gcc -O2 -Iinclude -Ioracle tests/c/dist_c_demo.c -Lpaper_1901_06535_b200 -lrd -Loracle -lorc -lpthread */
#include <math.h>
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <sys/mman.h>
#include <sys/wait.h>
#include <unistd.h>

#include "rd.h"
#include "rd_oracle.h"

enum { H = 97, W = 140, STEPS = 29 };

/* seeded-free deterministic init and a two-level phi map, in global rows */
static double u_init(int64_t i, int64_t j) { return 0.1 * (double)((i * 131 + j * 71) % 97) / 97.0; }
static double v_init(int64_t i, int64_t j) { return 0.05 * (double)((i * 29 + j * 113) % 89) / 89.0; }
static double phi_at(int64_t i, int64_t j) { return (i >= 30 && i < 70 && j >= 50 && j < 90) ? 0.0975 : 0.054; }

static void fill(void* dst, int esz, int64_t row0, int64_t rows, double (*f)(int64_t, int64_t)) {
  for (int64_t r = 0; r < rows; ++r)
    for (int64_t j = 0; j < W; ++j) {
      const double x = f(row0 + r, j);
      if (esz == 8)
        ((double*)dst)[r * W + j] = x;
      else
        ((float*)dst)[r * W + j] = (float)x;
    }
}

typedef struct {
  int rank, world, dtype;
  const uint8_t* id;
  unsigned char* u_global; /* rank writes its owned rows here */
  unsigned char* v_global;
  int rc;
  int expect_p2p; /* ranks in different processes: copy-engine pushes over CUDA IPC, self-test passed */
} job;

static void* run_rank(void* arg) {
  job* jb = (job*)arg;
  const int esz = jb->dtype == RD_F64 ? 8 : 4;
  const int64_t base = H / jb->world, extra = H % jb->world;
  const int64_t row0 = jb->rank * base + (jb->rank < extra ? jb->rank : extra);
  const int64_t rows = base + (jb->rank < extra ? 1 : 0);
  rd_grid g;
  memset(&g, 0, sizeof g);
  g.width = W, g.height = H, g.batch = 1, g.dtype = jb->dtype, g.tb_depth = 4;
  rd_params p;
  rd_params_default(&p);
  void* phi = malloc((size_t)rows * W * esz);
  void* u = malloc((size_t)rows * W * esz);
  void* v = malloc((size_t)rows * W * esz);
  fill(phi, esz, row0, rows, phi_at);
  fill(u, esz, row0, rows, u_init);
  fill(v, esz, row0, rows, v_init);
  rd_sim* s = NULL;
  jb->rc = rd_create_dist(&g, &p, phi, jb->rank, jb->world, jb->id, &s);
  if (jb->rc != RD_OK) {
    fprintf(stderr, "rank %d rd_create_dist: %s\n", jb->rank, rd_create_error());
    return NULL;
  }
  rd_geometry geo;
  rd_get_geometry(s, &geo);
  if (geo.row0 != row0 || geo.height != rows || geo.world != jb->world) {
    fprintf(stderr, "rank %d geometry\n", jb->rank);
    jb->rc = -100;
  }
  if (jb->expect_p2p && (geo.transport != RD_TRANSPORT_P2P || geo.flag_selftest != 1)) {
    fprintf(stderr, "rank %d transport %d selftest %d\n", jb->rank, geo.transport, geo.flag_selftest);
    jb->rc = -101;
  }
  rd_shape disc; /* centred on the slab edge of two ranks */
  memset(&disc, 0, sizeof disc);
  disc.kind = RD_DISC, disc.cy2 = 2 * (H / 2), disc.cx2 = 70, disc.r = 6;
  jb->rc |= rd_write_fields(s, 0, u, v);
  jb->rc |= rd_stimulate(s, -1, &disc, 1.0, 0);
  jb->rc |= rd_stimulate(s, -1, &disc, 1.0, 13);
  jb->rc |= rd_step(s, 11);
  jb->rc |= rd_step(s, STEPS - 11);
  if (jb->rc != RD_OK) fprintf(stderr, "rank %d: %s\n", jb->rank, rd_last_error(s));
  jb->rc |= rd_read_fields(s, 0, jb->u_global + (size_t)row0 * W * esz, jb->v_global + (size_t)row0 * W * esz);
  jb->rc |= rd_destroy(s); /* collective */
  free(phi), free(u), free(v);
  return NULL;
}

static int compare(int dtype, const unsigned char* U, const unsigned char* V, const char* what) {
  const int esz = dtype == RD_F64 ? 8 : 4;
  const size_t n = (size_t)H * W;
  unsigned char* ru = malloc(n * esz);
  unsigned char* rv = malloc(n * esz);
  unsigned char* phi = malloc(n * esz);
  fill(ru, esz, 0, H, u_init);
  fill(rv, esz, 0, H, v_init);
  fill(phi, esz, 0, H, phi_at);
  orc_params op;
  orc_params_default(&op);
  orc_event ev[2];
  memset(ev, 0, sizeof ev);
  for (int k = 0; k < 2; ++k) {
    ev[k].shape.kind = ORC_DISC, ev[k].shape.cy2 = 2 * (H / 2), ev[k].shape.cx2 = 70, ev[k].shape.r = 6;
    ev[k].value = 1.0, ev[k].at_step = k ? 13 : 0;
  }
  orc_fault f;
  const int st = esz == 8 ? orc_run_f64(H, W, (double*)ru, (double*)rv, (double*)phi, &op, 0, 0, STEPS, ev, 2, NULL,
                                        0, NULL, &f, 0, NULL)
                          : orc_run_f32(H, W, (float*)ru, (float*)rv, (float*)phi, &op, 0, 0, STEPS, ev, 2, NULL, 0,
                                        NULL, &f, 0, NULL);
  const int bad = st != 0 || memcmp(U, ru, n * esz) || memcmp(V, rv, n * esz);
  if (bad) fprintf(stderr, "%s: fields differ from the oracle\n", what);
  free(ru), free(rv), free(phi);
  return bad;
}

static int run_group(int world, int dtype, const uint8_t* id, const char* what) {
  const int esz = dtype == RD_F64 ? 8 : 4;
  unsigned char* U = calloc((size_t)H * W, esz);
  unsigned char* V = calloc((size_t)H * W, esz);
  job jobs[4];
  pthread_t th[4];
  for (int r = 0; r < world; ++r) {
    jobs[r] = (job){r, world, dtype, id, U, V, 0, 0};
    pthread_create(&th[r], NULL, run_rank, &jobs[r]);
  }
  int rc = 0;
  for (int r = 0; r < world; ++r) {
    pthread_join(th[r], NULL);
    rc |= jobs[r].rc;
  }
  if (rc) {
    fprintf(stderr, "%s: rank error\n", what);
    return 1;
  }
  const int bad = compare(dtype, U, V, what);
  free(U), free(V);
  return bad;
}

/* The ranks as forked processes (before the parent initialises CUDA): the
 * results come back through an anonymous shared mapping. */
static int run_forked(int world, int dtype, const char* what) {
  uint8_t id[128];
  if (rd_dist_shm_id(id) != RD_OK) {
    fprintf(stderr, "rd_dist_shm_id: %s\n", rd_create_error());
    return 1;
  }
  const int esz = dtype == RD_F64 ? 8 : 4;
  const size_t n = (size_t)H * W * esz;
  unsigned char* sh = mmap(NULL, 2 * n, PROT_READ | PROT_WRITE, MAP_SHARED | MAP_ANONYMOUS, -1, 0);
  if (sh == MAP_FAILED) return 1;
  pid_t pids[4];
  for (int r = 0; r < world; ++r) {
    pids[r] = fork();
    if (pids[r] == 0) {
      job jb = {r, world, dtype, id, sh, sh + n, 0, 1};
      run_rank(&jb);
      _exit(jb.rc ? 1 : 0);
    }
  }
  int rc = 0;
  for (int r = 0; r < world; ++r) {
    int st = 0;
    if (pids[r] < 0 || waitpid(pids[r], &st, 0) < 0 || !WIFEXITED(st) || WEXITSTATUS(st)) rc = 1;
  }
  if (rc) fprintf(stderr, "%s: rank error\n", what);
  const int bad = rc || compare(dtype, sh, sh + n, what);
  munmap(sh, 2 * n);
  return bad;
}

int main(void) {
  uint8_t id[128];
  /* first, while this process has no CUDA context to inherit */
  if (run_forked(2, RD_F32, "2 rank processes, fp32")) return 1;
  if (run_forked(2, RD_F64, "2 rank processes, fp64")) return 1;
  if (rd_dist_unique_id(id) != RD_OK) {
    fprintf(stderr, "rd_dist_unique_id: %s\n", rd_create_error());
    return 1;
  }
  if (run_group(1, RD_F64, id, "world 1 (NCCL), fp64")) return 1;
  for (int dt = 0; dt < 2; ++dt) {
    if (rd_dist_local_id(id) != RD_OK) return 1;
    if (run_group(2, dt ? RD_F64 : RD_F32, id, dt ? "2 local ranks, fp64" : "2 local ranks, fp32")) return 1;
  }
  /* error behaviour: an unknown in-process id, a rank outside the world */
  rd_grid g;
  memset(&g, 0, sizeof g);
  g.width = W, g.height = H, g.batch = 1, g.dtype = RD_F32;
  rd_params p;
  rd_params_default(&p);
  rd_sim* s = NULL;
  memcpy(id + 8, "notatokn", 8);
  if (rd_create_dist(&g, &p, NULL, 0, 2, id, &s) != RD_EINVAL || s) return 1;
  if (rd_create_dist(&g, &p, NULL, 2, 2, id, &s) != RD_EINVAL || s) return 1;
  printf(
      "C dist ABI ok: 2 rank processes (shared-memory group, IPC push) fp32 + fp64, world 1 over NCCL, 2 in-process "
      "ranks fp32 + fp64, bitwise equal to the oracle\n");
  return 0;
}
