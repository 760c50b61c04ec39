// rd_gz.cuh — gz_kernel: small batched instances spread over the whole chip.
//
// PRODUCT CODE. Independent of oracle/ (no shared code, headers or constants).
//
// a2-a5 + a8 (+ a6 probes fused): the time loop of PAPER.md:122-124 (Eq. 1,
// forward Euler, five-node Laplacian, no-flux edges) for instances too small
// to stream through tb_kernel efficiently (configs 1-3, P:153-154 and the
// gate/diode geometries of §4). cr_kernel keeps one instance inside one
// thread-block cluster, i.e. at most 16 SMs per instance; gz_kernel cuts every
// instance into tiles, one CTA per tile over all SMs (cooperative launch, so
// every tile is resident), and exchanges tile borders through L2 only once
// every k steps (temporal blocking across the tile boundary):
//   * a tile holds its owned cells plus a ghost zone k rows / gx >= k columns
//     deep; every 16-byte vector of the zone belongs to one thread for the
//     whole launch (u, v in its registers; u also in a shared-memory
//     ping-pong buffer for the neighbouring threads, phi in shared memory);
//   * step s of a block (1..k) computes only the owned region grown by k - s
//     cells (rows exactly, columns by whole vectors) -- the cells whose k-step
//     dependency cone lies inside the loaded zone. A vector's layer L (its
//     distance from the owned region) fixes its active steps (s <= k - L), so
//     the zone's vectors are dealt to the threads sorted by layer, row-major
//     within a layer: the lanes of a warp start and stop computing together,
//     and the west / east neighbour of a vector usually sits in the adjacent
//     lane (a shuffle instead of a shared load);
//   * after k steps a tile stores its owned border ring (k rows / gx columns
//     deep) into an exchange plane as 8-byte words that carry 4 bytes of data
//     and the exchange's epoch (the LL format: no fence, no separate flag --
//     a reader that sees the epoch sees the data of the same single-copy-atomic
//     word), two parities; neighbours poll exactly the words of their ghost
//     zone until the epoch matches;
//   * global edges are mirrored (ghost = the even reflection of the cells,
//     which evolves bit for bit like the cells it mirrors),
//     so reflected ghost cells are read like any other ghost cell.
// Results are bitwise those of tb_kernel / cr_kernel / the oracle: the same
// row_update on the same operands, only the order in which cells are
// computed differs.
#pragma once
#include "rd_kernels.cuh"

namespace rdk {

#ifdef RD_GZ_PROF
// measurement build only: per-CTA cycle counts of the phases of a block
// (compute, publish, first fetch pass, remaining wait, barrier), summed over
// launches; read with rd_gz_prof_dump (rd_runtime.cu)
__device__ unsigned long long g_gz_prof[2048 * 8];
#endif

constexpr int kGzThreads = 512;  // threads of a one-tile-per-SM CTA; 256 when two tiles share an SM
constexpr int kGzMaxSlots = 6;  // zone vectors per thread

template <typename T>
struct GzArgs {
  TBArgs<T> a;  // fields ((row 0, col 0) of instance 0), geometry, constants, flags, timelapse
  // exchange planes of 8-byte LL words (row-major like the fields: word
  // (x, j) of instance b at b * plane_stride + x * pitch + j times the words
  // per cell, 1 for fp32, 2 for fp64); [parity][u, v]
  unsigned long long* x[2][2];
  unsigned epoch0;  // exchange j of this launch carries epoch0 + j + 1
  int32_t k;        // steps per exchange block (ghost rows)
  int32_t gx;       // ghost columns (multiple of V, >= k)
  int32_t th, tw;   // tile rows / columns (tw a multiple of V); the last tiles are smaller
  int32_t tr, tc;   // tiles per instance (rows x columns)
  int32_t nr, nv;   // tile array: rows (th + 2k) and vectors per row ((tw + 2 gx) / V)
  int32_t n;        // steps in this launch
  int32_t nt;       // threads per tile (kernel instantiation): 512 or 256
  int32_t n_probes;
  const ProbeDev* probes;  // a6 fused: latched probes
  long long* first_fire;
  int64_t step0;        // global step at the launch's start
  int32_t probe_every;  // gcd of the strides of the probes due at some step in (step0, step0 + n] (0: none)
  int32_t probe_first;  // steps from step0 to the first multiple of probe_every
  unsigned long long timeout_ns;  // a ghost wait longer than this abandons the launch (PRECISE replay)
};

// even reflection about the faces of [0, n) for |overshoot| <= n
__device__ __forceinline__ int gz_refl(int g, int n) { return g < 0 ? -1 - g : (g >= n ? 2 * n - 1 - g : g); }

__device__ __forceinline__ unsigned long long gz_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ void ll_st2(unsigned long long* p, unsigned long long a, unsigned long long b) {
  asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b) : "memory");
}
__device__ __forceinline__ unsigned long long ll_ld(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// LL words of one value: fp32 -> 1 word (epoch | bits), fp64 -> 2 (lo, hi halves)
template <typename T>
struct LL;
template <>
struct LL<float> {
  static constexpr int W = 1;
  static __device__ __forceinline__ void pack(float x, unsigned ep, unsigned long long* w) {
    w[0] = ((unsigned long long)ep << 32) | __float_as_uint(x);
  }
  static __device__ __forceinline__ float unpack(const unsigned long long* w) { return __uint_as_float((unsigned)w[0]); }
};
template <>
struct LL<double> {
  static constexpr int W = 2;
  static __device__ __forceinline__ void pack(double x, unsigned ep, unsigned long long* w) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(x);
    w[0] = ((unsigned long long)ep << 32) | (b & 0xffffffffull);
    w[1] = ((unsigned long long)ep << 32) | (b >> 32);
  }
  static __device__ __forceinline__ double unpack(const unsigned long long* w) {
    return __longlong_as_double((long long)((w[1] << 32) | (w[0] & 0xffffffffull)));
  }
};

// Publish V values (one 16-byte vector) as LL words at word index wi.
template <typename T, int V>
__device__ __forceinline__ void ll_put(unsigned long long* plane, int64_t wi, const T* x, unsigned ep) {
  constexpr int NW = V * LL<T>::W;  // 4 words (fp32: 4 cells; fp64: 2 cells x 2 halves)
  unsigned long long w[NW];
#pragma unroll
  for (int e = 0; e < V; ++e) LL<T>::pack(x[e], ep, w + e * LL<T>::W);
#pragma unroll
  for (int i = 0; i < NW; i += 2) ll_st2(plane + wi + i, w[i], w[i + 1]);
}

// The u and v words of up to V cells (lane e at word index wi[e], lanes
// outside `need` skipped) once all carry epoch ep: every word is loaded
// before any is checked, so a ready ghost vector costs one L2 round trip;
// not-ready words are re-polled. Writes the values to us[e] / vs[e]; false on
// timeout.
template <typename T, int V>
__device__ __forceinline__ bool ll_fetch(const unsigned long long* xu, const unsigned long long* xv,
                                         const int64_t (&wi)[V], unsigned need, unsigned ep, T* us, T* vs,
                                         unsigned long long deadline) {
  constexpr int LW = LL<T>::W;
  unsigned long long wu[V * LW], wv[V * LW];
  for (;;) {
#pragma unroll
    for (int e = 0; e < V; ++e)
#pragma unroll
      for (int h = 0; h < LW; ++h) {
        wu[e * LW + h] = ((need >> e) & 1u) ? ll_ld(xu + wi[e] + h) : ((unsigned long long)ep << 32);
        wv[e * LW + h] = ((need >> e) & 1u) ? ll_ld(xv + wi[e] + h) : ((unsigned long long)ep << 32);
      }
    bool ok = true;
#pragma unroll
    for (int i = 0; i < V * LW; ++i) ok = ok && (unsigned)(wu[i] >> 32) == ep && (unsigned)(wv[i] >> 32) == ep;
#ifdef RD_GZ_TIMING_NO_WAIT  // measurement build only: results are wrong
    ok = true;
#endif
    if (ok) break;
    if (gz_now() > deadline) return false;
  }
#pragma unroll
  for (int e = 0; e < V; ++e)
    if ((need >> e) & 1u) {
      us[e] = LL<T>::unpack(wu + e * LW);
      vs[e] = LL<T>::unpack(wv + e * LW);
    }
  return true;
}

// a6: after global step gstep, every probe of instance b due then fires iff
// some cell of its rect is >= its threshold (probe_kernel's max test, NaN
// ignored): each thread tests the owned cells of its vectors (registers); the
// latch keeps the smallest firing step.
template <typename T, int V, int M>
__device__ __forceinline__ void gz_probes(const GzArgs<T>& ga, int b, int row0, int col0, const int (&o)[M],
                                          const unsigned (&lf)[M], int PW, const T (&u)[M][V], int64_t gstep) {
  for (int p = 0; p < ga.n_probes; ++p) {
    const ProbeDev pr = ga.probes[p];
    if (pr.b != b || pr.stride <= 0 || gstep % pr.stride != 0) continue;  // uniform over the CTA
    bool hit = false;
#pragma unroll
    for (int m = 0; m < M; ++m) {
      if ((lf[m] & 0xffu) != 0) continue;  // owned vectors only (layer 0; unused slots are 0xff)
      const int x = o[m] / PW, j = o[m] % PW - V;
      const int gr = row0 + x;
      if (gr < pr.y0 || gr >= pr.y1) continue;
#pragma unroll
      for (int e = 0; e < V; ++e) {
        const int gc = col0 + j + e;
        hit = hit || (gc >= pr.x0 && gc < pr.x1 && u[m][e] >= (T)pr.threshold);
      }
    }
    if (__any_sync(0xffffffffu, hit) && (threadIdx.x & 31) == 0)
      atomicMin(reinterpret_cast<unsigned long long*>(ga.first_fire + p), (unsigned long long)gstep);
  }
}

// shared memory of a tile array of nr rows x nv vectors: u ping-pong, phi and
// the exchange's v staging plane (rows padded by a vector on each side), and
// the layer-sorted vector list
__host__ __device__ constexpr size_t gz_smem_bytes(int nr, int nv, int V, int esz) {
  return (size_t)4 * nr * (nv + 2) * V * esz + (size_t)nr * nv * 4;
}

// NT threads per tile: 512 (one tile per SM) or 256 (two tiles per SM, so
// one tile computes while the other waits for its neighbours' words)
template <typename T, bool REACT, int MODE, int M, bool PROBE, int NT>
__global__ void __launch_bounds__(NT, kGzThreads / NT) gz_kernel(const __grid_constant__ GzArgs<T> ga) {
  constexpr int V = 16 / (int)sizeof(T);
  constexpr int LW = LL<T>::W;
  const TBArgs<T>& a = ga.a;
  const int ntile = ga.tr * ga.tc;
  const int b = blockIdx.x / ntile, tile = blockIdx.x % ntile;
  const int ti = tile / ga.tc, tj = tile % ga.tc;
  const int H = a.H, W = a.W, k = ga.k, GX = ga.gx;
  const int r0 = ti * ga.th, r1 = min(r0 + ga.th, H);
  const int c0 = tj * ga.tw, c1 = min(c0 + ga.tw, W);
  const int row0 = r0 - k, col0 = c0 - GX;  // global (row, column) of array cell (0, 0)
  // tile array coordinates: x = global row - row0, j = global column - col0
  const int xo0 = k, xo1 = k + (r1 - r0);    // owned rows
  const int jo0 = GX, jo1 = GX + (c1 - c0);  // owned columns
  const int xz1 = xo1 + k, jz1 = jo1 + GX;   // the zone: rows [0, xz1), columns [0, jz1)
  const int vz1 = (jz1 + V - 1) / V;
  const int PW = (ga.nv + 2) * V;  // shared row pitch: a pad vector on each side
  const int plane = ga.nr * PW;
  extern __shared__ __align__(16) unsigned char gz_smem[];
  T* U0 = reinterpret_cast<T*>(gz_smem);
  T* U1 = U0 + plane;
  T* Ps = U1 + plane;
  T* Vx = Ps + plane;  // staging of the ghost zone's v at an exchange
  uint32_t* list = reinterpret_cast<uint32_t*>(Vx + plane);
  __shared__ int abort_flag;
  __shared__ int warp_tot[NT / 32];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int64_t inst = (int64_t)b * a.plane_stride, pitch = a.pitch;

  // the u buffers start zeroed: cells never computed are read as finite
  // stale values, never as leftovers of an earlier kernel
  for (int i = t; i < 2 * plane * (int)sizeof(T) / 16; i += NT) reinterpret_cast<int4*>(gz_smem)[i] = make_int4(0, 0, 0, 0);
  if (t == 0) abort_flag = 0;

  // the zone's vectors of layer <= k, sorted by layer, row-major within a
  // layer (a CTA-wide stable compaction per layer)
  auto layer = [&](int x, int vc) {
    const int dx = max(max(xo0 - x, x - (xo1 - 1)), 0);
    const int j0 = vc * V;
    const int dc = j0 + V <= jo0 ? jo0 - (j0 + V - 1) : (j0 >= jo1 ? j0 - jo1 + 1 : 0);
    return max(dx, dc);
  };
  const int nzone = xz1 * vz1;
  int count = 0;
  for (int L = 0; L <= k; ++L) {
    for (int i0 = 0; i0 < nzone; i0 += NT) {
      const int i = i0 + t;
      const int x = i / vz1, vc = i - (i / vz1) * vz1;
      const bool f = i < nzone && layer(x, vc) == L;
      const unsigned bal = __ballot_sync(0xffffffffu, f);
      if (lane == 0) warp_tot[warp] = __popc(bal);
      __syncthreads();
      int pre = 0, tot = 0;
      for (int w = 0; w < NT / 32; ++w) {
        const int c = warp_tot[w];
        pre += w < warp ? c : 0;
        tot += c;
      }
      if (f) list[count + pre + __popc(bal & ((1u << lane) - 1u))] = ((uint32_t)x << 16) | (uint32_t)vc;
      count += tot;
      __syncthreads();
    }
  }

  // this thread's vectors: list entries t, t + NT, ...; per slot the shared
  // offset o and lf = layer | 0x100 west neighbour in lane - 1 | 0x200 east
  // neighbour in lane + 1 | 0x400 straddles W (unused slot: layer 0xff)
  T u[M][V], v[M][V];
  int o[M];
  unsigned lf[M];
  const T* fu = a.u_in + inst;
  const T* fv = a.v_in + inst;
  const T* fp = a.phi + inst;
#pragma unroll
  for (int m = 0; m < M; ++m) {
    const int i = t + NT * m;
    o[m] = 0;
    lf[m] = 0xffu;
#pragma unroll
    for (int e = 0; e < V; ++e) u[m][e] = v[m][e] = T(0);
    if (i >= count) continue;
    const uint32_t id = list[i];
    const int x = (int)(id >> 16), vc = (int)(id & 0xffffu);
    o[m] = x * PW + V + vc * V;
    unsigned f = (unsigned)layer(x, vc);
    if (lane > 0 && list[i - 1] == id - 1u) f |= 0x100u;
    if (lane < 31 && i + 1 < count && list[i + 1] == id + 1u) f |= 0x200u;
    if (f == 0 || (f & 0xffu) == 0) {
      if (vc * V + V > jo1 && jo1 % V != 0) f |= 0x400u;
    }
    lf[m] = f;
    // the zone from the fields, mirrored at the global edges
    const int gr = gz_refl(row0 + x, H), gc = col0 + vc * V;
    if (gc >= 0 && gc + V <= W) {
      const int64_t g = (int64_t)gr * pitch + gc;
      *reinterpret_cast<int4*>(u[m]) = *reinterpret_cast<const int4*>(fu + g);
      *reinterpret_cast<int4*>(v[m]) = *reinterpret_cast<const int4*>(fv + g);
      *reinterpret_cast<int4*>(Ps + o[m]) = *reinterpret_cast<const int4*>(fp + g);
    } else {
#pragma unroll
      for (int e = 0; e < V; ++e) {
        const int64_t g = (int64_t)gr * pitch + gz_refl(gc + e, W);
        u[m][e] = fu[g];
        v[m][e] = fv[g];
        Ps[o[m] + e] = fp[g];
      }
    }
    *reinterpret_cast<int4*>(U0 + o[m]) = *reinterpret_cast<const int4*>(u[m]);
  }
  __syncthreads();

  const Consts<T> kc = a.k[a.per_instance ? b : 0];
  float minb = INFINITY;
  int p = 0;  // U[p] holds the latest step
  int to_probe = ga.probe_first;
#ifdef RD_GZ_PROF
  __shared__ unsigned long long pf_blockmax, pf_passmax, pf_loadmax;
  unsigned long long pf_c = 0, pf_pub = 0, pf_bar = 0, pf_n = 0, pf_f = 0, pf_p = 0, pf_l = 0;
#endif
  for (int s0 = 0, blk = 0; s0 < ga.n; s0 += k, ++blk) {
    const int kb = min(k, ga.n - s0);
#ifdef RD_GZ_PROF
    const unsigned long long pf0 = clock64();
    if (t == 0) pf_blockmax = pf_passmax = pf_loadmax = 0;
#endif
    for (int s = 1; s <= kb; ++s) {
      const unsigned lmax = (unsigned)(k - s);  // active: layer <= k - s
      const T* src = p ? U1 : U0;
      T* dst = p ? U0 : U1;
#pragma unroll
      for (int m = 0; m < M; ++m) {
        const T from_w = __shfl_up_sync(0xffffffffu, u[m][V - 1], 1);
        const T from_e = __shfl_down_sync(0xffffffffu, u[m][0], 1);
        if ((lf[m] & 0xffu) > lmax) continue;
        const T* c = src + o[m];
        T N_[V], S_[V], E[V], Wn[V], ph[V], uo[V], vo[V];
        *reinterpret_cast<int4*>(N_) = *reinterpret_cast<const int4*>(c - PW);
        *reinterpret_cast<int4*>(S_) = *reinterpret_cast<const int4*>(c + PW);
        *reinterpret_cast<int4*>(ph) = *reinterpret_cast<const int4*>(Ps + o[m]);
        const T wl = (lf[m] & 0x100u) ? from_w : c[-1];
        const T er = (lf[m] & 0x200u) ? from_e : c[V];
#pragma unroll
        for (int q = 0; q < V; ++q) {
          Wn[q] = q == 0 ? wl : u[m][q - 1];
          E[q] = q == V - 1 ? er : u[m][q + 1];
        }
        row_update<T, V, REACT, MODE>(u[m], N_, S_, E, Wn, v[m], ph, kc, uo, vo, minb);
#pragma unroll
        for (int q = 0; q < V; ++q) {
          u[m][q] = uo[q];
          v[m][q] = vo[q];
        }
        *reinterpret_cast<int4*>(dst + o[m]) = *reinterpret_cast<const int4*>(uo);
      }
      __syncthreads();
      p ^= 1;
      if (PROBE && --to_probe == 0) {
        to_probe = ga.probe_every;
        gz_probes<T, V, M>(ga, b, row0, col0, o, lf, PW, u, ga.step0 + s0 + s);
      }
    }
    if (s0 + kb >= ga.n) break;
#ifdef RD_GZ_TIMING_NO_EXCHANGE  // measurement build only: results are wrong
    continue;
#endif
    // ---- exchange (parity blk & 1): publish the owned border ring as LL
    // words, then poll the ghost zone's words and reload them
#ifdef RD_GZ_PROF
    const unsigned long long pf1 = clock64();
    pf_c += pf1 - pf0;
    ++pf_n;
#endif
    const unsigned ep = ga.epoch0 + (unsigned)blk + 1u;
    unsigned long long* xu = ga.x[blk & 1][0] + inst * LW;
    unsigned long long* xv = ga.x[blk & 1][1] + inst * LW;
#pragma unroll
    for (int m = 0; m < M; ++m) {
      if ((lf[m] & 0xffu) != 0) continue;
      const int x = o[m] / PW, j0 = o[m] % PW - V;
      if (!(x < xo0 + k || x >= xo1 - k || j0 < jo0 + GX || j0 + V > jo1 - GX)) continue;  // inside the ring
      const int64_t wi = ((int64_t)(row0 + x) * pitch + (col0 + j0)) * LW;  // lanes >= W: margin words
      ll_put<T, V>(xu, wi, u[m], ep);
      ll_put<T, V>(xv, wi, v[m], ep);
    }
#ifdef RD_GZ_PROF
    const unsigned long long pf2 = clock64();
    pf_pub += pf2 - pf1;
#endif
    {
      // the ghost zone cell by cell over the whole CTA (all of a thread's
      // words requested before any is checked: one L2 round trip when the
      // neighbours are done; words not yet published are re-polled): u into
      // the current buffer, v into the staging plane; then every thread
      // takes its ghost slots from shared memory
      T* cur = p ? U1 : U0;
      const unsigned long long deadline = gz_now() + ga.timeout_ns;
#ifdef RD_GZ_PROF
      unsigned long long pf_passes = 0;
      const unsigned long long pf_f0 = clock64();
#endif
      const int gw = jz1 - (jo1 - jo0);        // ghost cells of an owned row
      const int n_top = xo0 * jz1;             // cells of the ghost rows above
      const int n_mid = (xo1 - xo0) * gw;      // ghost cells beside the owned rows
      const int n_all = n_top + n_mid + k * jz1;  // + the ghost rows below
      constexpr int G = 4;  // cells per thread in flight
      bool ok = true;
      for (int c0 = 0; ok && c0 < n_all; c0 += NT * G) {
        unsigned long long wu[G][LW], wv[G][LW];
        int off[G];
        int64_t wi[G];
#pragma unroll
        for (int g = 0; g < G; ++g) {
          const int c = c0 + t + NT * g;
          int x, j;
          if (c < n_top) {
            x = c / jz1, j = c - x * jz1;
          } else if (c < n_top + n_mid) {
            const int r = (c - n_top) / gw, q = c - n_top - r * gw;
            x = xo0 + r, j = q < jo0 ? q : jo1 + (q - jo0);
          } else {
            const int r = (c - n_top - n_mid) / jz1;
            x = xo1 + r, j = c - n_top - n_mid - r * jz1;
          }
          off[g] = c < n_all ? x * PW + V + j : -1;
          wi[g] = ((int64_t)gz_refl(row0 + x, H) * pitch + gz_refl(col0 + j, W)) * LW;
        }
        unsigned pending = 0;
#pragma unroll
        for (int g = 0; g < G; ++g) pending |= (unsigned)(off[g] >= 0) << g;
        while (pending) {
#ifdef RD_GZ_PROF
          ++pf_passes;
#endif
#pragma unroll
          for (int g = 0; g < G; ++g)
#pragma unroll
            for (int h = 0; h < LW; ++h)
              if ((pending >> g) & 1u) {
                wu[g][h] = ll_ld(xu + wi[g] + h);
                wv[g][h] = ll_ld(xv + wi[g] + h);
              }
#pragma unroll
          for (int g = 0; g < G; ++g) {
            if (!((pending >> g) & 1u)) continue;
            bool r = true;
#pragma unroll
            for (int h = 0; h < LW; ++h) r = r && (unsigned)(wu[g][h] >> 32) == ep && (unsigned)(wv[g][h] >> 32) == ep;
#ifdef RD_GZ_TIMING_NO_WAIT  // measurement build only: results are wrong
            r = true;
#endif
            if (r) {
              cur[off[g]] = LL<T>::unpack(wu[g]);
              Vx[off[g]] = LL<T>::unpack(wv[g]);
              pending &= ~(1u << g);
            }
          }
          if (pending && gz_now() > deadline) {
            ok = false;
            break;
          }
        }
      }
      if (!ok) atomicExch(&abort_flag, 1);
#ifdef RD_GZ_PROF
      atomicMax(&pf_passmax, pf_passes);
      atomicMax(&pf_loadmax, clock64() - pf_f0);
#endif
      __syncthreads();
#pragma unroll
      for (int m = 0; m < M; ++m) {
        const unsigned L = lf[m] & 0xffu;
        if (L == 0xffu || (L == 0 && !(lf[m] & 0x400u))) continue;  // unused, or owned and current
        const int j0 = o[m] % PW - V;
#pragma unroll
        for (int e = 0; e < V; ++e) {
          if (L == 0 && j0 + e < jo1) continue;  // owned lane of a vector straddling W
          u[m][e] = cur[o[m] + e];
          v[m][e] = Vx[o[m] + e];
        }
      }
    }
#ifdef RD_GZ_PROF
    const unsigned long long pf3 = clock64();
    atomicMax(&pf_blockmax, pf3 - pf2);  // the slowest thread's fetch (first pass + waits)
#endif
    __syncthreads();
#ifdef RD_GZ_PROF
    pf_bar += clock64() - pf3;
    pf_f += pf_blockmax;
    pf_p += pf_passmax;
    pf_l += pf_loadmax;
#endif
    if (abort_flag) break;
  }

  // write back the owned cells to the output buffer; health check; timelapse
  // (probes due at any step, the last included, were tested in the loop)
  bool bad = false;
  T* ou = a.u_out + inst;
  T* ov = a.v_out + inst;
#pragma unroll
  for (int m = 0; m < M; ++m) {
    if ((lf[m] & 0xffu) != 0) continue;
    const int x = o[m] / PW, j0 = o[m] % PW - V;
    const int64_t g = (int64_t)(row0 + x) * pitch + (col0 + j0);
#pragma unroll
    for (int e = 0; e < V; ++e) {
      if (col0 + j0 + e >= W) continue;
      ou[g + e] = u[m][e];
      ov[g + e] = v[m][e];
      if (MODE != MODE_PRECISE) bad = bad || !Ops<T>::finite(u[m][e]) || !Ops<T>::finite(v[m][e]);
      if (a.tl) {
        T* tp = a.tl + inst + g + e;
        if (u[m][e] > *tp) *tp = u[m][e];
      }
    }
  }
  if (MODE != MODE_PRECISE && ((REACT && minb < kFastDivMinB) || bad || abort_flag)) *a.precise_flag = 1;
#ifdef RD_GZ_PROF
  if (t == 0 && blockIdx.x < 2048) {
    unsigned long long* q = g_gz_prof + blockIdx.x * 8;
    atomicAdd(q + 0, pf_c);
    atomicAdd(q + 1, pf_pub);
    atomicAdd(q + 2, pf_f);
    atomicAdd(q + 3, pf_bar);
    atomicAdd(q + 4, pf_n);
    atomicAdd(q + 5, pf_p);
    atomicAdd(q + 6, pf_l);
  }
#endif
}

}  // namespace rdk
