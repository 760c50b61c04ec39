/* The C ABI used from plain C (no Python): create a two-instance batch,
 * schedule stimuli, step in two calls, read fields, probe -- and compare with
 * the oracle's C library bitwise, in fp64 and fp32; then the asynchronous
 * host I/O calls (stage, snapshot, commit, step). Also checks error codes.
 * Test program only: it links the oracle (tests/ may), the product does not.
 *   gcc -O2 -Iinclude -Ioracle tests/c/abi_c_demo.c -Lpaper_1901_06535_b200 -lrd -Loracle -lorc */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "rd.h"
#include "rd_oracle.h"

enum { H = 150, W = 220, B = 2, STEPS = 120 };

static int run(int dtype) {
  const size_t esz = dtype == RD_F64 ? 8 : 4, n = (size_t)H * W;
  unsigned char* phi = calloc(B * n, esz);
  unsigned char* u = calloc(B * n, esz);
  unsigned char* v = calloc(B * n, esz);
  unsigned char* ru = calloc(n, esz);
  unsigned char* rv = calloc(n, esz);
  for (int b = 0; b < B; ++b)
    for (size_t c = 0; c < n; ++c) {
      const size_t i = c / W, j = c % W;
      const double p = (i >= 40 && i < 80 && j >= 60 + 40 * b && j < 140) ? 0.0975 : 0.054;
      if (esz == 8)
        ((double*)phi)[b * n + c] = p;
      else
        ((float*)phi)[b * n + c] = (float)p;
    }
  rd_grid g;
  memset(&g, 0, sizeof g);
  g.width = W, g.height = H, g.batch = B, g.dtype = dtype;
  rd_params p;
  rd_params_default(&p);
  rd_sim* s = NULL;
  if (rd_create(&g, &p, phi, &s) != RD_OK) {
    fprintf(stderr, "rd_create: %s\n", rd_create_error());
    return 1;
  }
  rd_shape disc;
  memset(&disc, 0, sizeof disc);
  disc.kind = RD_DISC, disc.cy2 = H, disc.cx2 = 60, disc.r = 5;
  rd_shape rect;
  memset(&rect, 0, sizeof rect);
  rect.kind = RD_RECT, rect.y0 = 10, rect.x0 = 150, rect.y1 = 20, rect.x1 = 200;
  int rc = rd_stimulate(s, -1, &disc, 1.0, 0);
  rc |= rd_stimulate(s, 1, &rect, 1.0, 10);
  rc |= rd_step(s, 50);
  rc |= rd_step(s, STEPS - 50);
  if (rc != RD_OK || rd_get_step(s) != STEPS) {
    fprintf(stderr, "step: %s\n", rd_last_error(s));
    return 1;
  }
  /* error behaviour: a stimulus in the past, an instance out of range */
  if (rd_stimulate(s, 0, &disc, 1.0, 5) != RD_ERANGE || rd_read_fields(s, B, ru, rv) != RD_ERANGE ||
      strlen(rd_last_error(s)) == 0) {
    fprintf(stderr, "error codes\n");
    return 1;
  }
  int bad = 0;
  for (int b = 0; b < B; ++b) {
    if (rd_read_fields(s, b, u + b * n * esz, v + b * n * esz) != RD_OK) return 1;
    /* the oracle on the same inputs (u = v = 0 initially, R-10) */
    memset(ru, 0, n * esz);
    memset(rv, 0, n * esz);
    orc_params op;
    orc_params_default(&op);
    orc_event ev[2];
    memset(ev, 0, sizeof ev);
    ev[0].shape.kind = ORC_DISC, ev[0].shape.cy2 = H, ev[0].shape.cx2 = 60, ev[0].shape.r = 5;
    ev[0].value = 1.0, ev[0].at_step = 0;
    ev[1].shape.kind = ORC_RECT, ev[1].shape.y0 = 10, ev[1].shape.x0 = 150, ev[1].shape.y1 = 20,
    ev[1].shape.x1 = 200;
    ev[1].value = 1.0, ev[1].at_step = 10;
    orc_fault f;
    const int st = esz == 8 ? orc_run_f64(H, W, (double*)ru, (double*)rv, (double*)(phi + b * n * esz), &op, 0, 0,
                                          STEPS, ev, b == 1 ? 2 : 1, NULL, 0, NULL, &f, 0, NULL)
                            : orc_run_f32(H, W, (float*)ru, (float*)rv, (float*)(phi + b * n * esz), &op, 0, 0,
                                          STEPS, ev, b == 1 ? 2 : 1, NULL, 0, NULL, &f, 0, NULL);
    if (st != 0) return 1;
    const int du = memcmp(u + b * n * esz, ru, n * esz), dv = memcmp(v + b * n * esz, rv, n * esz);
    if (du || dv) {
      fprintf(stderr, "instance %d (%s): fields differ\n", b, esz == 8 ? "f64" : "f32");
      bad = 1;
    }
    /* the probe: max u over a rect equals the oracle's */
    rd_rect r = {60, 40, 90, 120};
    orc_rect orr = {60, 40, 90, 120};
    int32_t fired = 0;
    double mx = 0;
    if (rd_probe(s, b, &r, 0.1, &fired, &mx) != RD_OK) return 1;
    const double omx = esz == 8 ? orc_probe_max_f64(H, W, (double*)ru, &orr) : orc_probe_max_f32(H, W, (float*)ru, &orr);
    if (mx != omx || fired != (omx >= 0.1)) {
      fprintf(stderr, "probe %d: %g vs %g\n", b, mx, omx);
      bad = 1;
    }
  }
  /* asynchronous host I/O: stage the oracle's last fields (instance B-1's,
   * still in ru / rv) as new inputs of instance 0, snapshot instance 0 before
   * the commit, commit, step, and compare with the oracle continuing from
   * those inputs on instance 0's phi */
  {
    unsigned char* su = calloc(n, esz);
    unsigned char* sv = calloc(n, esz);
    enum { MORE = 7 };
    int rc2 = rd_write_fields_async(s, 0, ru, rv);
    rc2 |= rd_read_fields_async(s, 0, su, sv);
    rc2 |= rd_commit_fields(s);
    rc2 |= rd_step(s, MORE);
    rc2 |= rd_io_wait(s);
    if (rc2 != RD_OK || rd_write_fields_async(s, B, ru, rv) != RD_ERANGE) {
      fprintf(stderr, "async I/O: %s\n", rd_last_error(s));
      return 1;
    }
    if (memcmp(su, u, n * esz) || memcmp(sv, v, n * esz)) {
      fprintf(stderr, "async snapshot differs from the fields before the commit\n");
      bad = 1;
    }
    if (rd_read_fields(s, 0, su, sv) != RD_OK) return 1;
    orc_params op;
    orc_params_default(&op);
    orc_fault f;
    const int st = esz == 8 ? orc_run_f64(H, W, (double*)ru, (double*)rv, (double*)phi, &op, 0, 0, MORE, NULL, 0, NULL, 0,
                                          NULL, &f, 0, NULL)
                            : orc_run_f32(H, W, (float*)ru, (float*)rv, (float*)phi, &op, 0, 0, MORE, NULL, 0, NULL, 0,
                                          NULL, &f, 0, NULL);
    if (st != 0 || memcmp(su, ru, n * esz) || memcmp(sv, rv, n * esz)) {
      fprintf(stderr, "async commit + steps differ from the oracle (%s)\n", esz == 8 ? "f64" : "f32");
      bad = 1;
    }
    free(su), free(sv);
  }
  rd_destroy(s);
  free(phi), free(u), free(v), free(ru), free(rv);
  return bad;
}

int main(void) {
  rd_sim* s = NULL;
  rd_grid g;
  memset(&g, 0, sizeof g);
  g.width = 2, g.height = 8, g.batch = 1, g.dtype = RD_F32;
  if (rd_create(&g, NULL, NULL, &s) != RD_EINVAL || s != NULL) {
    fprintf(stderr, "width 2 must be RD_EINVAL\n");
    return 1;
  }
  if (run(RD_F64) || run(RD_F32)) return 1;
  printf("C ABI ok: fp64 + fp32, 2-instance batch, bitwise equal to the oracle\n");
  return 0;
}
