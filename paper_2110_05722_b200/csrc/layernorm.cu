// LayerNorm forward / backward.
//   forward   F/kernels.py:235-270  (single traversal; mean and mean-of-squares
//             are independent reductions; sigma = sqrt(var + eps) is cached)
//   backward  F/gradients.py:103-144 (two independent row reductions over one
//             traversal; dw/db column sums are deterministic two-stage)
//
// Fast path: one warp per row, the row cached in registers (cols % 8 == 0,
// cols <= 1024).  Row sums are taken on values shifted by the row's first
// element (no E[x^2]-E[x]^2 cancellation in fp32) and combined across lanes in
// fp64, matching the reference's float64 statistics to fp32 precision.
// Backward uses the stable equivalent of the reference's alpha/beta form:
//   dx = (g - mean(g) - xhat * mean(g*xhat)) / sigma,  g = w*dy,
// where sum(g) and sum(g*xhat) are the two independent reductions.
#include "common.cuh"

namespace ls2 {

constexpr int kLnWarps = 4;
constexpr int kLnBwdWarps = 8;
constexpr int kLnMaxBlocks = kNumSMs;

template <typename T, typename C>
__device__ __forceinline__ void ld_group(const T* p, C (&v)[8]) {
  Pack8<T> q = ld8(p);
#pragma unroll
  for (int e = 0; e < 8; ++e) v[e] = cvt<C>(q.v[e]);
}
template <typename T, typename C>
__device__ __forceinline__ void st_group(T* p, const C (&v)[8]) {
  Pack8<T> q;
#pragma unroll
  for (int e = 0; e < 8; ++e) q.v[e] = cvt<T>(v[e]);
  st8(p, q);
}

// fp32 LayerNorm row pieces in packed f32x2 pair math (per-lane rounding identical
// to the scalar expressions they replace; the statistics accumulate even/odd
// elements in two partial sums)
template <typename T, int ITERS>
__device__ __forceinline__ void row_stats_f2(const Pack8<T> (&v)[ITERS], int lane, int64_t cgs,
                                             float pivot, float& s1, float& s2) {
  float2 a = f2s(0.f), q = f2s(0.f);
  const float2 np = f2s(-pivot);
#pragma unroll
  for (int it = 0; it < ITERS; ++it) {
    if (lane + 32 * it < cgs) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 d = f2add(pair_f2(v[it], e), np);
        a = f2add(a, d);
        q = f2fma(d, d, q);
      }
    }
  }
  s1 = a.x + a.y;
  s2 = q.x + q.y;
}

// o = ((v - pivot) - msh) * rs * w + b for 8 elements
template <typename T, typename TW>
__device__ __forceinline__ void ln_norm8_f2(const Pack8<T>& v, const Pack8<TW>& w,
                                            const Pack8<TW>& b, float pivot, float msh, float rs,
                                            float* o) {
  const float2 np = f2s(-pivot), nm = f2s(-msh), r2 = f2s(rs);
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const float2 t = f2mul(f2add(f2add(pair_f2(v, e), np), nm), r2);
    const float2 y = f2fma(t, pair_f2(w, e), pair_f2(b, e));
    o[2 * e] = y.x;
    o[2 * e + 1] = y.y;
  }
}

template <typename Tin, typename Tout, typename Tstat, int ITERS>
__global__ void __launch_bounds__(kLnWarps * 32, 7) ln_fwd_warp(
    const Tin* __restrict__ x, const Tin* __restrict__ w, const Tin* __restrict__ b,
    Tout* __restrict__ y, Tstat* __restrict__ mu, Tstat* __restrict__ sigma,
    int* __restrict__ degenerate, int64_t rows, int64_t cols, double eps) {
  using C = typename CompOf<Tin>::type;
  const int lane = threadIdx.x & 31;
  const int64_t cgs = cols / 8;
  // affine parameters staged in shared memory (registers decide occupancy here)
  extern __shared__ __align__(16) unsigned char ln_par[];
  Pack8<Tin>* sw = reinterpret_cast<Pack8<Tin>*>(ln_par);
  Pack8<Tin>* sb = sw + cgs;
  for (int64_t g = threadIdx.x; g < cgs; g += blockDim.x) {
    sw[g] = ld8(w + g * 8);
    sb[g] = ld8(b + g * 8);
  }
  __syncthreads();
  const double inv_m = 1.0 / (double)cols;
  for (int64_t r = (int64_t)blockIdx.x * kLnWarps + (threadIdx.x >> 5); r < rows;
       r += (int64_t)gridDim.x * kLnWarps) {
    const Tin* xr = x + r * cols;
    Pack8<Tin> v[ITERS];   // row kept packed; (x - pivot) is recomputed on use
#pragma unroll
    for (int it = 0; it < ITERS; ++it) {
      const int64_t g = lane + 32 * it;
      if (g < cgs) v[it] = ld8(xr + g * 8);
    }
    const C pivot = __shfl_sync(0xffffffffu, cvt<C>(v[0].v[0]), 0);
    C s1 = 0, s2 = 0;
    if constexpr (std::is_same<C, float>::value) {
      row_stats_f2(v, lane, cgs, pivot, s1, s2);
    } else {
#pragma unroll
      for (int it = 0; it < ITERS; ++it) {
        if (lane + 32 * it < cgs) {
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const C d = cvt<C>(v[it].v[e]) - pivot;
            s1 += d;
            s2 += d * d;
          }
        }
      }
    }
    const double S1 = warp_sum((double)s1);
    const double S2 = warp_sum((double)s2);
    const double mean_sh = S1 * inv_m;
    double var = S2 * inv_m - mean_sh * mean_sh;
    if (var < 0.0) var = 0.0;
    if (eps == 0.0 && var <= 0.0 && degenerate && lane == 0) *degenerate = 1;
    const double sg = sqrt(var + eps);
    const C rs = (C)(1.0 / sg);
    const C msh = (C)mean_sh;
    if (lane == 0) {
      mu[r] = (Tstat)((double)pivot + mean_sh);
      sigma[r] = (Tstat)sg;
    }
    Tout* yr = y + r * cols;
#pragma unroll
    for (int it = 0; it < ITERS; ++it) {
      const int64_t g = lane + 32 * it;
      if (g < cgs) {
        C o[8];
        const Pack8<Tin> wq = sw[g], bq = sb[g];
        if constexpr (std::is_same<C, float>::value) {
          ln_norm8_f2(v[it], wq, bq, pivot, msh, rs, o);
        } else {
#pragma unroll
          for (int e = 0; e < 8; ++e)
            o[e] = ((cvt<C>(v[it].v[e]) - pivot) - msh) * rs * cvt<C>(wq.v[e]) + cvt<C>(bq.v[e]);
        }
        st_group(yr + g * 8, o);
      }
    }
  }
}

// Fused bias+dropout+residual -> LayerNorm (F/kernels.py:367-382 then :235-270):
//   yres = keep*(x+bias)*dscale + res  (stored: it is the next residual stream),
//   u    = LN(yres)  with (mu, sigma) cached.
// The LayerNorm consumes the stored (rounded) yres, so results equal the
// unfused pair exactly; one launch and one pass instead of two.
template <typename Tin, typename Tout, typename Tstat, int ITERS, bool DROP, bool GEN = true>
__global__ void __launch_bounds__(kLnWarps * 32, 7) ln_fwd_bdr_warp(
    const Tin* __restrict__ x, const Tin* __restrict__ bias, const Tin* __restrict__ res,
    Tout* __restrict__ yres, uint8_t* __restrict__ bits, const Tin* __restrict__ w,
    const Tin* __restrict__ b, Tout* __restrict__ u, Tstat* __restrict__ mu,
    Tstat* __restrict__ sigma, int64_t rows, int64_t cols, double eps, uint64_t seed,
    const uint64_t* seed_ptr, uint64_t thresh, typename CompOf<Tin>::type dscale) {
  using C = typename CompOf<Tin>::type;
  const int lane = threadIdx.x & 31;
  const int64_t cgs = cols / 8;
  if (seed_ptr) seed = *seed_ptr;
  extern __shared__ __align__(16) unsigned char ln_par[];
  Pack8<Tin>* sw = reinterpret_cast<Pack8<Tin>*>(ln_par);
  Pack8<Tin>* sb = sw + cgs;
  Pack8<Tin>* sc = sb + cgs;
  for (int64_t g = threadIdx.x; g < cgs; g += blockDim.x) {
    sw[g] = ld8(w + g * 8);
    sb[g] = ld8(b + g * 8);
    sc[g] = ld8(bias + g * 8);
  }
  __syncthreads();
  const double inv_m = 1.0 / (double)cols;
  for (int64_t r = (int64_t)blockIdx.x * kLnWarps + (threadIdx.x >> 5); r < rows;
       r += (int64_t)gridDim.x * kLnWarps) {
    Pack8<Tout> v[ITERS];   // the stored yres, packed; LN statistics read it back
    // every load of the row first (x, residual and the bank's keep bits of all
    // ITERS groups), so one memory round trip covers the row: issued inside the
    // compute loop, the next group's loads queued behind this group's store
    Pack8<Tin> pxs[ITERS], prs[ITERS];
    uint32_t kbs[ITERS];
#pragma unroll
    for (int it = 0; it < ITERS; ++it) {
      const int64_t g = lane + 32 * it;
      kbs[it] = 0xFF;
      if (g < cgs) {
        pxs[it] = ld8(x + r * cols + g * 8);
        prs[it] = ld8(res + r * cols + g * 8);
        if (DROP && !GEN) kbs[it] = bits[r * cgs + g];      // precomputed by the mask bank
      }
    }
#pragma unroll
    for (int it = 0; it < ITERS; ++it) {
      const int64_t g = lane + 32 * it;
      if (g < cgs) {
        const Pack8<Tin>& px = pxs[it];
        const Pack8<Tin>& pr = prs[it];
        uint32_t kb = kbs[it];
        if (DROP && GEN) {
          kb = keep_byte(seed, (uint64_t)(r * cgs + g) * 8, thresh);
          bits[r * cgs + g] = (uint8_t)kb;
        }
        Pack8<Tout> q;
        const Pack8<Tin> cq = sc[g];
        if constexpr (std::is_same<C, float>::value) {
          const float2 ds2 = f2s(dscale);
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            float2 a = f2add(pair_f2(px, e), pair_f2(cq, e));
            if (DROP) {
              const float2 k2 = make_float2(__uint_as_float(((kb >> (2 * e)) & 1u) * 0x3f800000u),
                                            __uint_as_float(((kb >> (2 * e + 1)) & 1u) * 0x3f800000u));
              a = f2mul(f2mul(a, k2), ds2);
            }
            const float2 y = f2add(a, pair_f2(pr, e));
            q.v[2 * e] = cvt<Tout>(y.x);
            q.v[2 * e + 1] = cvt<Tout>(y.y);
          }
        } else {
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            C a = add_rn(cvt<C>(px.v[e]), cvt<C>(cq.v[e]));
            if (DROP) a = mul_rn(mul_rn(a, bitval<C>(kb, e)), dscale);
            q.v[e] = cvt<Tout>(add_rn(a, cvt<C>(pr.v[e])));
          }
        }
        v[it] = q;
        st8(yres + r * cols + g * 8, q);
      }
    }
    const C pivot = __shfl_sync(0xffffffffu, cvt<C>(v[0].v[0]), 0);
    C s1 = 0, s2 = 0;
    if constexpr (std::is_same<C, float>::value) {
      row_stats_f2(v, lane, cgs, pivot, s1, s2);
    } else {
#pragma unroll
      for (int it = 0; it < ITERS; ++it) {
        if (lane + 32 * it < cgs) {
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const C d = cvt<C>(v[it].v[e]) - pivot;
            s1 += d;
            s2 += d * d;
          }
        }
      }
    }
    const double S1 = warp_sum((double)s1);
    const double S2 = warp_sum((double)s2);
    const double mean_sh = S1 * inv_m;
    double var = S2 * inv_m - mean_sh * mean_sh;
    if (var < 0.0) var = 0.0;
    const double sg = sqrt(var + eps);
    const C rs = (C)(1.0 / sg);
    const C msh = (C)mean_sh;
    if (lane == 0) {
      mu[r] = (Tstat)((double)pivot + mean_sh);
      sigma[r] = (Tstat)sg;
    }
#pragma unroll
    for (int it = 0; it < ITERS; ++it) {
      const int64_t g = lane + 32 * it;
      if (g < cgs) {
        C o[8];
        const Pack8<Tin> wq = sw[g], bq = sb[g];
        if constexpr (std::is_same<C, float>::value) {
          ln_norm8_f2(v[it], wq, bq, pivot, msh, rs, o);
        } else {
#pragma unroll
          for (int e = 0; e < 8; ++e)
            o[e] = ((cvt<C>(v[it].v[e]) - pivot) - msh) * rs * cvt<C>(wq.v[e]) + cvt<C>(bq.v[e]);
        }
        st_group(u + r * cols + g * 8, o);
      }
    }
  }
}

// generic: CTA per row, any cols
template <typename Tin, typename Tout, typename Tstat>
__global__ void ln_fwd_block(const Tin* __restrict__ x, const Tin* __restrict__ w,
                             const Tin* __restrict__ b, Tout* __restrict__ y,
                             Tstat* __restrict__ mu, Tstat* __restrict__ sigma,
                             int* __restrict__ degenerate, int64_t rows, int64_t cols,
                             double eps) {
  using C = typename CompOf<Tin>::type;
  __shared__ double red[2][32];
  for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
    const Tin* xr = x + r * cols;
    const C pivot = cvt<C>(xr[0]);
    double s1 = 0, s2 = 0;
    for (int64_t c = threadIdx.x; c < cols; c += blockDim.x) {
      const double d = (double)(cvt<C>(xr[c]) - pivot);
      s1 += d;
      s2 += d * d;
    }
    s1 = warp_sum(s1);
    s2 = warp_sum(s2);
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) { red[0][wid] = s1; red[1][wid] = s2; }
    __syncthreads();
    double S1 = 0, S2 = 0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) { S1 += red[0][i]; S2 += red[1][i]; }
    __syncthreads();
    const double mean_sh = S1 / (double)cols;
    double var = S2 / (double)cols - mean_sh * mean_sh;
    if (var < 0.0) var = 0.0;
    if (eps == 0.0 && var <= 0.0 && degenerate && threadIdx.x == 0) *degenerate = 1;
    const double sg = sqrt(var + eps);
    if (threadIdx.x == 0) {
      mu[r] = (Tstat)((double)pivot + mean_sh);
      sigma[r] = (Tstat)sg;
    }
    const C rs = (C)(1.0 / sg), msh = (C)mean_sh;
    for (int64_t c = threadIdx.x; c < cols; c += blockDim.x)
      y[r * cols + c] = cvt<Tout>(((cvt<C>(xr[c]) - pivot) - msh) * rs * cvt<C>(w[c]) + cvt<C>(b[c]));
  }
}

// ---------------------------------------------------------------------------
// backward
// ---------------------------------------------------------------------------
// Warp per row, row in registers, next row prefetched while the current one is
// reduced (memory-level parallelism for these short, latency-bound passes).
// BDR: the LN input gradient (+ residual) dyo is also pushed through the
// preceding bias+dropout+residual backward (F/gradients.py:147-159):
//   dproj = keep * dyo * dscale,  dbias = column sums of dproj
// so one pass yields dyo (residual stream gradient), dproj, and the column
// partials of (dw, db[, dbias]) as partial[block][NP][cols].
template <typename Tin, typename Tout, typename Tstat, int ITERS, bool RES, bool BDR, bool DROP>
__global__ void __launch_bounds__(kLnBwdWarps * 32) ln_bwd_warp(
    const Tin* __restrict__ dy, const Tin* __restrict__ x, const Tin* __restrict__ w,
    const Tstat* __restrict__ mu, const Tstat* __restrict__ sigma, const Tin* __restrict__ dres,
    Tout* __restrict__ dx, const uint8_t* __restrict__ bits, Tout* __restrict__ dproj,
    typename CompOf<Tin>::type dscale, double* __restrict__ partial, int64_t rows, int64_t cols) {
  using C = typename CompOf<Tin>::type;
  constexpr int NP = BDR ? 3 : 2;
  __shared__ C red[kLnBwdWarps][NP][256];  // per-warp column partials, one chunk at a time
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t cgs = cols / 8;
  C wv[ITERS][8], acc[NP][ITERS][8];
#pragma unroll
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int e = 0; e < 8; ++e)
#pragma unroll
      for (int k = 0; k < NP; ++k) acc[k][it][e] = 0;
    const int64_t g = lane + 32 * it;
    if (g < cgs) ld_group(w + g * 8, wv[it]);
  }
  const C inv_m = (C)(1.0 / (double)cols);
  const int64_t stride = (int64_t)gridDim.x * kLnBwdWarps;
  int64_t r = (int64_t)blockIdx.x * kLnBwdWarps + wid;
  Pack8<Tin> nd[ITERS], nx[ITERS], nr[ITERS];   // prefetched row
  auto fetch = [&](int64_t rr) {
#pragma unroll
    for (int it = 0; it < ITERS; ++it) {
      const int64_t g = lane + 32 * it;
      if (rr < rows && g < cgs) {
        nd[it] = ld8(dy + rr * cols + g * 8);
        nx[it] = ld8(x + rr * cols + g * 8);
        if (RES) nr[it] = ld8(dres + rr * cols + g * 8);
      }
    }
  };
  fetch(r);
  for (; r < rows; r += stride) {
    // current row stays packed in its storage type; values are re-derived on use
    Pack8<Tin> cd[ITERS], cx[ITERS], cr[ITERS];
#pragma unroll
    for (int it = 0; it < ITERS; ++it) {
      cd[it] = nd[it];
      cx[it] = nx[it];
      if (RES) cr[it] = nr[it];
    }
    const C m_r = (C)mu[r];
    const C rs = (C)(1.0 / (double)sigma[r]);
    fetch(r + stride);
    C r1 = 0, r3 = 0;
#pragma unroll
    for (int it = 0; it < ITERS; ++it) {
      if (lane + 32 * it < cgs) {
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const C dv = cvt<C>(cd[it].v[e]);
          const C xh = (cvt<C>(cx[it].v[e]) - m_r) * rs;
          const C gg = wv[it][e] * dv;
          r1 += gg;
          r3 += gg * xh;
          acc[0][it][e] += dv * xh;
          acc[1][it][e] += dv;
        }
      }
    }
    r1 = warp_sum(r1) * inv_m;
    r3 = warp_sum(r3) * inv_m;
#pragma unroll
    for (int it = 0; it < ITERS; ++it) {
      const int64_t g = lane + 32 * it;
      if (g < cgs) {
        Pack8<Tout> o;
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const C xh = (cvt<C>(cx[it].v[e]) - m_r) * rs;
          const C gg = wv[it][e] * cvt<C>(cd[it].v[e]);
          C v = (gg - r1 - xh * r3) * rs;
          if (RES) v += cvt<C>(cr[it].v[e]);
          o.v[e] = cvt<Tout>(v);
        }
        st8(dx + r * cols + g * 8, o);
        if (BDR) {
          const uint32_t kb = DROP ? bits[r * cgs + g] : 0xFF;
          Pack8<Tout> pj;
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            C v = cvt<C>(o.v[e]);
            if (DROP) v = mul_rn(mul_rn(v, bitval<C>(kb, e)), dscale);
            acc[NP - 1][it][e] += v;
            pj.v[e] = cvt<Tout>(v);
          }
          st8(dproj + r * cols + g * 8, pj);
        }
      }
    }
  }
  // CTA reduction of the warps' column partials (fixed order) in chunks of 256 cols
#pragma unroll
  for (int it = 0; it < ITERS; ++it) {
    const int64_t g = lane + 32 * it;
    if (g < cgs) {
#pragma unroll
      for (int e = 0; e < 8; ++e)
#pragma unroll
        for (int k = 0; k < NP; ++k) red[wid][k][lane * 8 + e] = acc[k][it][e];
    }
    __syncthreads();
    const int64_t base = (int64_t)it * 256;
    for (int c = threadIdx.x; c < NP * 256; c += blockDim.x) {
      const int k = c / 256, cc = c % 256;
      if (base + cc >= cols) continue;
      double s = 0;
#pragma unroll
      for (int q = 0; q < kLnBwdWarps; ++q) s += (double)red[q][k][cc];
      partial[((int64_t)blockIdx.x * NP + k) * cols + base + cc] = s;
    }
    __syncthreads();
  }
}

// One-wave variant (fp32 compute): a CTA of RW warps takes RW rows per round,
// one row per warp held in registers, so every row of a 4096-token batch is in
// flight at once (maximum memory-level parallelism, no per-warp row loop).  The
// warps' per-element contributions (dy*xhat, dy[, dproj]) are staged in shared
// memory as stg[RW][NP][cols] and column-reduced in warp order by all threads
// (fixed order -> deterministic); each thread carries up to kLnPairs column
// sums across rounds and leaves partial[block][NP][cols] for the finish.
constexpr int kLnStageMaxWarps = 28;   // 896 threads -> up to 72 registers per thread
constexpr int kLnStageWideWarps = 15;  // rows of 513..1024 columns: 480 threads, 128 registers

inline int ln_stage_rw(int64_t rows, int64_t cols) {
  // stg[rw][3][cols] + acc[3][cols] floats within 200 KB
  int64_t rw = (200 * 1024) / (3 * cols * 4) - 1;
  rw = rw < 1 ? 1 : (rw > kLnStageMaxWarps ? kLnStageMaxWarps : rw);
  if (cols > 512 && rw > kLnStageWideWarps) rw = kLnStageWideWarps;  // ITERS == 4 kernels
  const int64_t need = ceil_div(rows, (int64_t)kLnMaxBlocks);
  if (need < rw) rw = need < 1 ? 1 : need;
  return (int)rw;
}

template <typename Tin, typename Tout, typename Tstat, int ITERS, bool RES, bool BDR, bool DROP,
          bool PIPE>
__global__ void __launch_bounds__((ITERS >= 4 ? kLnStageWideWarps : kLnStageMaxWarps) * 32, 1)
ln_bwd_stage(
    const Tin* __restrict__ dy, const Tin* __restrict__ x, const Tin* __restrict__ w,
    const Tstat* __restrict__ mu, const Tstat* __restrict__ sigma, const Tin* __restrict__ dres,
    Tout* __restrict__ dx, const uint8_t* __restrict__ bits, Tout* __restrict__ dproj,
    float dscale, double* __restrict__ partial, int64_t rows, int64_t cols) {
  constexpr int NP = BDR ? 3 : 2;
  extern __shared__ __align__(16) float stg[];   // [rw][NP][cols], then acc[NP][cols]
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int rw = blockDim.x >> 5;
  const int64_t cgs = cols / 8;
  const int npairs = NP * (int)cols;
  float* accs = stg + (int64_t)rw * npairs;
  for (int p = threadIdx.x; p < npairs; p += blockDim.x) accs[p] = 0.f;
  Pack8<Tin> wv[ITERS];
#pragma unroll
  for (int it = 0; it < ITERS; ++it) {
    const int64_t g = lane + 32 * it;
    if (g < cgs) wv[it] = ld8(w + g * 8);
  }
  const float inv_m = (float)(1.0 / (double)cols);
  // PIPE (the CTA has several row batches): batch k's loads are issued before
  // batch k-1's staged column contributions are folded into accs, so the fold
  // overlaps the loads.  The fold order is the same either way: PIPE does not
  // change results.
  const int64_t base0 = (int64_t)blockIdx.x * rw;
  for (int64_t base = base0; base < rows; base += (int64_t)gridDim.x * rw) {
    const int64_t r = base + wid;
    float* my = stg + (int64_t)wid * npairs;
    Pack8<Tin> cd[ITERS], cx[ITERS], cr[ITERS];
    uint32_t kbs[ITERS];   // keep bits loaded with the row (not after the reductions)
    float m_r = 0.f, rs = 0.f;
    if (r < rows) {
#pragma unroll
      for (int it = 0; it < ITERS; ++it) {
        const int64_t g = lane + 32 * it;
        kbs[it] = 0xFF;
        if (g < cgs) {
          cd[it] = ld8_stream(dy + r * cols + g * 8);
          cx[it] = ld8_stream(x + r * cols + g * 8);
          if (RES) cr[it] = ld8_stream(dres + r * cols + g * 8);
          if (BDR && DROP) kbs[it] = bits[r * cgs + g];
        }
      }
      m_r = (float)mu[r];
      rs = (float)(1.0 / (double)sigma[r]);
    }
    if (PIPE && base != base0) {     // fold the previous batch (staged, synced)
      for (int p = threadIdx.x; p < npairs; p += blockDim.x) {
        float s = 0.f;
        for (int q = 0; q < rw; ++q) s += stg[(int64_t)q * npairs + p];
        accs[p] += s;
      }
      __syncthreads();               // folded before the stage is overwritten
    }
    if (r < rows) {
      // packed pair math: xh = x*rs - m*rs, gg = w*dy, sums of gg and gg*xh
      const float2 rs2 = f2s(rs), nmrs2 = f2s(-m_r * rs);
      float2 r1v = f2s(0.f), r3v = f2s(0.f);
#pragma unroll
      for (int it = 0; it < ITERS; ++it) {
        const int64_t g = lane + 32 * it;
        if (g < cgs) {
          float2 c0[4], c1[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float2 dv = pair_f2(cd[it], e);
            const float2 xh = f2fma(pair_f2(cx[it], e), rs2, nmrs2);
            const float2 gg = f2mul(pair_f2(wv[it], e), dv);
            r1v = f2add(r1v, gg);
            r3v = f2fma(gg, xh, r3v);
            c0[e] = f2mul(dv, xh);
            c1[e] = dv;
          }
          float4* d0 = reinterpret_cast<float4*>(my + g * 8);
          d0[0] = make_float4(c0[0].x, c0[0].y, c0[1].x, c0[1].y);
          d0[1] = make_float4(c0[2].x, c0[2].y, c0[3].x, c0[3].y);
          float4* d1 = reinterpret_cast<float4*>(my + cols + g * 8);
          d1[0] = make_float4(c1[0].x, c1[0].y, c1[1].x, c1[1].y);
          d1[1] = make_float4(c1[2].x, c1[2].y, c1[3].x, c1[3].y);
        }
      }
      const float r1 = warp_sum(r1v.x + r1v.y) * inv_m;
      const float r3 = warp_sum(r3v.x + r3v.y) * inv_m;
      const float2 nr1 = f2s(-r1), nr3 = f2s(-r3);
#pragma unroll
      for (int it = 0; it < ITERS; ++it) {
        const int64_t g = lane + 32 * it;
        if (g < cgs) {
          Pack8<Tout> o;
          float2 ov[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float2 dv = pair_f2(cd[it], e);
            const float2 xh = f2fma(pair_f2(cx[it], e), rs2, nmrs2);
            const float2 gg = f2mul(pair_f2(wv[it], e), dv);
            // (gg - r1 - xh*r3) * rs (+ dres)
            float2 v = f2mul(f2fma(xh, nr3, f2add(gg, nr1)), rs2);
            if (RES) v = f2add(v, pair_f2(cr[it], e));
            o.v[2 * e] = cvt<Tout>(v.x);
            o.v[2 * e + 1] = cvt<Tout>(v.y);
            ov[e] = v;
          }
          st8(dx + r * cols + g * 8, o);
          if (BDR) {
            const uint32_t kb = kbs[it];
            Pack8<Tout> pj;
            float c2[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) {
              float v = cvt<float>(o.v[e]);
              if (DROP) v = mul_rn(mul_rn(v, bitval<float>(kb, e)), dscale);
              c2[e] = v;
              pj.v[e] = cvt<Tout>(v);
            }
            (void)ov;
            st8(dproj + r * cols + g * 8, pj);
            float4* d2 = reinterpret_cast<float4*>(my + 2 * cols + g * 8);
            d2[0] = make_float4(c2[0], c2[1], c2[2], c2[3]);
            d2[1] = make_float4(c2[4], c2[5], c2[6], c2[7]);
          }
        }
      }
    } else {
      for (int c = lane; c < npairs; c += 32) my[c] = 0.f;
    }
    __syncthreads();                 // the batch is staged
    if (!PIPE) {
      for (int p = threadIdx.x; p < npairs; p += blockDim.x) {
        float s = 0.f;
        for (int q = 0; q < rw; ++q) s += stg[(int64_t)q * npairs + p];
        accs[p] += s;
      }
      __syncthreads();
    }
  }
  // the last batch's fold; thread p owns accs[p] in every fold, so no barrier
  if (PIPE && base0 < rows) {
    for (int p = threadIdx.x; p < npairs; p += blockDim.x) {
      float s = 0.f;
      for (int q = 0; q < rw; ++q) s += stg[(int64_t)q * npairs + p];
      accs[p] += s;
    }
  }
  for (int p = threadIdx.x; p < npairs; p += blockDim.x)
    partial[(int64_t)blockIdx.x * npairs + p] = (double)accs[p];
}

// Several row batches per CTA (d >= 768: T-big, BERT): each warp keeps its column
// partials in registers over all of its rows and the CTA folds them ONCE at the
// end (warp order, fp32), instead of staging every batch in shared memory and
// folding it behind a barrier.  Per-row math is ln_bwd_stage's, so dx / dproj
// are identical; the partials differ only in fp32 summation order.
// 8 warps at ITERS = 4 (243 registers), 16 at ITERS <= 2
template <int ITERS>
constexpr int ln_reg_warps() { return ITERS >= 4 ? 8 : 16; }
template <typename Tin, typename Tout, typename Tstat, int ITERS, bool RES, bool BDR, bool DROP>
__global__ void __launch_bounds__(ln_reg_warps<ITERS>() * 32, 1) ln_bwd_reg(
    const Tin* __restrict__ dy, const Tin* __restrict__ x, const Tin* __restrict__ w,
    const Tstat* __restrict__ mu, const Tstat* __restrict__ sigma, const Tin* __restrict__ dres,
    Tout* __restrict__ dx, const uint8_t* __restrict__ bits, Tout* __restrict__ dproj,
    float dscale, double* __restrict__ partial, int64_t rows, int64_t cols) {
  constexpr int NP = BDR ? 3 : 2;
  extern __shared__ __align__(16) float red[];   // [warps][NP][cols], the final fold
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int64_t cgs = cols / 8;
  const int npairs = NP * (int)cols;
  float acc[NP][ITERS][8];
#pragma unroll
  for (int k = 0; k < NP; ++k)
#pragma unroll
    for (int it = 0; it < ITERS; ++it)
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[k][it][e] = 0.f;
  Pack8<Tin> wv[ITERS];
#pragma unroll
  for (int it = 0; it < ITERS; ++it) {
    const int64_t g = lane + 32 * it;
    if (g < cgs) wv[it] = ld8(w + g * 8);
  }
  const float inv_m = (float)(1.0 / (double)cols);
  for (int64_t r = (int64_t)blockIdx.x * nw + wid; r < rows; r += (int64_t)gridDim.x * nw) {
    Pack8<Tin> cd[ITERS], cx[ITERS], cr[ITERS];
    uint32_t kbs[ITERS];
#pragma unroll
    for (int it = 0; it < ITERS; ++it) {
      const int64_t g = lane + 32 * it;
      kbs[it] = 0xFF;
      if (g < cgs) {
        cd[it] = ld8_stream(dy + r * cols + g * 8);
        cx[it] = ld8_stream(x + r * cols + g * 8);
        if (RES) cr[it] = ld8_stream(dres + r * cols + g * 8);
        if (BDR && DROP) kbs[it] = bits[r * cgs + g];
      }
    }
    const float m_r = (float)mu[r];
    const float rs = (float)(1.0 / (double)sigma[r]);
    const float2 rs2 = f2s(rs), nmrs2 = f2s(-m_r * rs);
    float2 r1v = f2s(0.f), r3v = f2s(0.f);
#pragma unroll
    for (int it = 0; it < ITERS; ++it) {
      if (lane + 32 * it < cgs) {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 dv = pair_f2(cd[it], e);
          const float2 xh = f2fma(pair_f2(cx[it], e), rs2, nmrs2);
          const float2 gg = f2mul(pair_f2(wv[it], e), dv);
          r1v = f2add(r1v, gg);
          r3v = f2fma(gg, xh, r3v);
          const float2 c0 = f2mul(dv, xh);
          acc[0][it][2 * e] += c0.x;
          acc[0][it][2 * e + 1] += c0.y;
          acc[1][it][2 * e] += dv.x;
          acc[1][it][2 * e + 1] += dv.y;
        }
      }
    }
    const float r1 = warp_sum(r1v.x + r1v.y) * inv_m;
    const float r3 = warp_sum(r3v.x + r3v.y) * inv_m;
    const float2 nr1 = f2s(-r1), nr3 = f2s(-r3);
#pragma unroll
    for (int it = 0; it < ITERS; ++it) {
      const int64_t g = lane + 32 * it;
      if (g < cgs) {
        Pack8<Tout> o;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 dv = pair_f2(cd[it], e);
          const float2 xh = f2fma(pair_f2(cx[it], e), rs2, nmrs2);
          const float2 gg = f2mul(pair_f2(wv[it], e), dv);
          float2 v = f2mul(f2fma(xh, nr3, f2add(gg, nr1)), rs2);
          if (RES) v = f2add(v, pair_f2(cr[it], e));
          o.v[2 * e] = cvt<Tout>(v.x);
          o.v[2 * e + 1] = cvt<Tout>(v.y);
        }
        st8(dx + r * cols + g * 8, o);
        if (BDR) {
          const uint32_t kb = kbs[it];
          Pack8<Tout> pj;
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            float v = cvt<float>(o.v[e]);
            if (DROP) v = mul_rn(mul_rn(v, bitval<float>(kb, e)), dscale);
            acc[NP - 1][it][e] += v;
            pj.v[e] = cvt<Tout>(v);
          }
          st8(dproj + r * cols + g * 8, pj);
        }
      }
    }
  }
  float* my = red + (int64_t)wid * npairs;
#pragma unroll
  for (int it = 0; it < ITERS; ++it) {
    const int64_t g = lane + 32 * it;
    if (g < cgs) {
#pragma unroll
      for (int k = 0; k < NP; ++k) {
        float4* d = reinterpret_cast<float4*>(my + k * cols + g * 8);
        d[0] = make_float4(acc[k][it][0], acc[k][it][1], acc[k][it][2], acc[k][it][3]);
        d[1] = make_float4(acc[k][it][4], acc[k][it][5], acc[k][it][6], acc[k][it][7]);
      }
    }
  }
  __syncthreads();
  for (int p = threadIdx.x; p < npairs; p += blockDim.x) {
    float t = 0.f;
    for (int q = 0; q < nw; ++q) t += red[(int64_t)q * npairs + p];
    partial[(int64_t)blockIdx.x * npairs + p] = (double)t;
  }
}

// generic backward: CTA per row for dx; param partials by a column-parallel kernel
template <typename Tin, typename Tout, typename Tstat>
__global__ void ln_bwd_block(const Tin* __restrict__ dy, const Tin* __restrict__ x,
                             const Tin* __restrict__ w, const Tstat* __restrict__ mu,
                             const Tstat* __restrict__ sigma, const Tin* __restrict__ dres,
                             Tout* __restrict__ dx, int64_t rows, int64_t cols) {
  using C = typename CompOf<Tin>::type;
  __shared__ double red[2][32];
  for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
    const C m_r = (C)mu[r];
    const C rs = (C)(1.0 / (double)sigma[r]);
    double s1 = 0, s3 = 0;
    for (int64_t c = threadIdx.x; c < cols; c += blockDim.x) {
      const C g = cvt<C>(w[c]) * cvt<C>(dy[r * cols + c]);
      const C xh = (cvt<C>(x[r * cols + c]) - m_r) * rs;
      s1 += (double)g;
      s3 += (double)(g * xh);
    }
    s1 = warp_sum(s1);
    s3 = warp_sum(s3);
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) { red[0][wid] = s1; red[1][wid] = s3; }
    __syncthreads();
    double S1 = 0, S3 = 0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) { S1 += red[0][i]; S3 += red[1][i]; }
    __syncthreads();
    const C r1 = (C)(S1 / (double)cols), r3 = (C)(S3 / (double)cols);
    for (int64_t c = threadIdx.x; c < cols; c += blockDim.x) {
      const C g = cvt<C>(w[c]) * cvt<C>(dy[r * cols + c]);
      const C xh = (cvt<C>(x[r * cols + c]) - m_r) * rs;
      C o = (g - r1 - xh * r3) * rs;
      if (dres) o += cvt<C>(dres[r * cols + c]);
      dx[r * cols + c] = cvt<Tout>(o);
    }
  }
}

template <typename Tin, typename Tstat>
__global__ void ln_param_partial(const Tin* __restrict__ dy, const Tin* __restrict__ x,
                                 const Tstat* __restrict__ mu, const Tstat* __restrict__ sigma,
                                 double* __restrict__ partial, int64_t rows, int64_t cols) {
  const int64_t per = (rows + gridDim.x - 1) / gridDim.x;
  const int64_t r0 = blockIdx.x * per, r1 = min(rows, r0 + per);
  for (int64_t c = threadIdx.x; c < cols; c += blockDim.x) {
    double sw = 0, sb = 0;
    for (int64_t r = r0; r < r1; ++r) {
      const double d = cvt<double>(dy[r * cols + c]);
      const double xh = (cvt<double>(x[r * cols + c]) - (double)mu[r]) / (double)sigma[r];
      sw += d * xh;
      sb += d;
    }
    partial[((int64_t)blockIdx.x * 2 + 0) * cols + c] = sw;
    partial[((int64_t)blockIdx.x * 2 + 1) * cols + c] = sb;
  }
}

// CTA = 32 warps x 32 columns, warp w reduces partial blocks w, w+32, ...;
// fixed-order combination of the warp sums (deterministic).
template <typename Tp, int NP>
__global__ void __launch_bounds__(1024) ln_param_finish(const double* __restrict__ partial,
                                                        int nblk, int64_t cols,
                                                        Tp* __restrict__ o0, Tp* __restrict__ o1,
                                                        Tp* __restrict__ o2, int beta_mask) {
  __shared__ double red[NP][32][33];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t c = (int64_t)blockIdx.x * 32 + lane;
  double s[NP];
#pragma unroll
  for (int k = 0; k < NP; ++k) s[k] = 0;
  if (c < cols) {
    for (int g = w; g < nblk; g += 32)
#pragma unroll
      for (int k = 0; k < NP; ++k) s[k] += partial[((int64_t)g * NP + k) * cols + c];
  }
#pragma unroll
  for (int k = 0; k < NP; ++k) red[k][w][lane] = s[k];
  __syncthreads();
  if (w == 0 && c < cols) {
    Tp* outs[3] = {o0, o1, o2};
#pragma unroll
    for (int k = 0; k < NP; ++k) {
      double t = 0;
#pragma unroll
      for (int q = 0; q < 32; ++q) t += red[k][q][lane];
      if (beta_mask & (1 << k)) t += cvt<double>(outs[k][c]);
      outs[k][c] = cvt<Tp>(t);
    }
  }
}

inline int ln_generic_blocks(int64_t rows) {
  const int64_t g = ceil_div(rows, (int64_t)16);
  return (int)(g < 1 ? 1 : (g > kLnMaxBlocks ? kLnMaxBlocks : g));
}

inline bool ln_vec_ok(int64_t cols, std::initializer_list<const void*> ptrs) {
  if (cols % 8 != 0 || cols > 1024 || cols < 8) return false;
  for (const void* p : ptrs)
    if (p && !aligned16(p)) return false;
  return true;
}

inline int ln_iters(int64_t cols) { return cols <= 256 ? 1 : cols <= 512 ? 2 : 4; }

// partial-row count of the vectorised backward (both the fp32 one-wave kernel
// and the f64 warp kernel use this grid, so the deferred-partial layout depends
// on (rows, cols) only)
inline int ln_bwd_blocks(int64_t rows, int64_t cols) {
  const int64_t g = ceil_div(rows, (int64_t)ln_stage_rw(rows, cols));
  return (int)(g < 1 ? 1 : (g > kLnMaxBlocks ? kLnMaxBlocks : g));
}

// launch the fp32 one-wave kernel (C == float) or the f64 warp kernel
template <typename Tin, typename Tout, typename Tstat, int I, bool R, bool B, bool D>
int ln_bwd_launch(const void* dy, const void* x, const void* w, const void* mu, const void* sigma,
                  const void* dres, void* dx, const uint8_t* bits, void* dproj, double dscale,
                  void* ws, int64_t rows, int64_t cols, cudaStream_t st) {
  using C = typename CompOf<Tin>::type;
  const int nblk = ln_bwd_blocks(rows, cols);
  if constexpr (std::is_same<C, double>::value) {
    ln_bwd_warp<Tin, Tout, Tstat, I, R, B, D><<<nblk, kLnBwdWarps * 32, 0, st>>>(
        (const Tin*)dy, (const Tin*)x, (const Tin*)w, (const Tstat*)mu, (const Tstat*)sigma,
        (const Tin*)dres, (Tout*)dx, bits, (Tout*)dproj, (C)dscale, (double*)ws, rows, cols);
  } else {
    constexpr int NP = B ? 3 : 2;
    const int rw = ln_stage_rw(rows, cols);
    const size_t smem = (size_t)(rw + 1) * NP * cols * sizeof(float);
    auto go = [&](auto pipe) {
      constexpr bool P = decltype(pipe)::value;
      static bool attr = false;
      if (!attr) {
        cudaFuncSetAttribute(ln_bwd_stage<Tin, Tout, Tstat, I, R, B, D, P>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        attr = true;
      }
      ln_bwd_stage<Tin, Tout, Tstat, I, R, B, D, P><<<nblk, rw * 32, smem, st>>>(
          (const Tin*)dy, (const Tin*)x, (const Tin*)w, (const Tstat*)mu, (const Tstat*)sigma,
          (const Tin*)dres, (Tout*)dx, bits, (Tout*)dproj, (float)dscale, (double*)ws, rows,
          cols);
    };
    // d >= 512 (ITERS >= 2): register partials, one fold per CTA (ln_bwd_reg).  T-big
    // 31.9 -> 20.2 us, BERT-128 25.0 -> 17.5 us, T-base 7.22 -> 7.15 us per launch.
    // LS2_LN_BWD_REG=0: the staged kernel (each fold overlapping the next batch's
    // loads when a CTA has several batches)
    static const bool reg_ok = [] {
      const char* e = getenv("LS2_LN_BWD_REG");
      return !(e && e[0] == '0');
    }();
    if (reg_ok && I >= 2) {
      constexpr int kW = ln_reg_warps<I>();
      const size_t rsm = (size_t)kW * NP * cols * sizeof(float);
      static bool rattr = false;
      if (!rattr) {
        cudaFuncSetAttribute(ln_bwd_reg<Tin, Tout, Tstat, I, R, B, D>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        rattr = true;
      }
      ln_bwd_reg<Tin, Tout, Tstat, I, R, B, D><<<nblk, kW * 32, rsm, st>>>(
          (const Tin*)dy, (const Tin*)x, (const Tin*)w, (const Tstat*)mu, (const Tstat*)sigma,
          (const Tin*)dres, (Tout*)dx, bits, (Tout*)dproj, (float)dscale, (double*)ws, rows,
          cols);
    } else if (rows > (int64_t)nblk * rw) {
      go(std::true_type{});
    } else {
      go(std::false_type{});
    }
  }
  return check_launch(B ? "layernorm_bwd_bdr" : "layernorm_bwd");
}

#define LS2_DISPATCH_STAT(TS, ...)                                                    \
  [&]() -> int {                                                                     \
    if (TS == LS2_F32) { using Tstat = float; return __VA_ARGS__(); }                \
    if (TS == LS2_F64) { using Tstat = double; return __VA_ARGS__(); }               \
    return fail(LS2_ERR_DTYPE, "layernorm: stats must be f32 or f64");               \
  }()

}  // namespace ls2

using namespace ls2;

extern "C" {

int ls2_layernorm_fwd(const void* x, const void* w, const void* b, void* y, void* mu, void* sigma,
                      int* degenerate, int64_t rows, int64_t cols, double eps, int tin, int tout,
                      int tstat, void* stream) {
  if (rows <= 0) return LS2_OK;
  if (cols < 2) return fail(LS2_ERR_SHAPE, "layernorm needs m >= 2");
  cudaStream_t st = as_stream(stream);
  const bool vec = ln_vec_ok(cols, {x, w, b, y});
  return LS2_DISPATCH_IO(tin, tout, "layernorm_fwd", [&] {
    return LS2_DISPATCH_STAT(tstat, [&] {
      if (vec) {
        const int64_t want = ceil_div(rows, kLnWarps);
        const int it_ = ln_iters(cols);
        const void* fn = it_ == 1 ? (const void*)ln_fwd_warp<Tin, Tout, Tstat, 1>
                       : it_ == 2 ? (const void*)ln_fwd_warp<Tin, Tout, Tstat, 2>
                                  : (const void*)ln_fwd_warp<Tin, Tout, Tstat, 4>;
        const size_t psm = 2 * (size_t)cols * sizeof(Tin);
        const int grid = resident_grid(fn, kLnWarps * 32, psm, want);
        switch (it_) {
          case 1: ln_fwd_warp<Tin, Tout, Tstat, 1><<<grid, kLnWarps * 32, psm, st>>>((const Tin*)x, (const Tin*)w, (const Tin*)b, (Tout*)y, (Tstat*)mu, (Tstat*)sigma, degenerate, rows, cols, eps); break;
          case 2: ln_fwd_warp<Tin, Tout, Tstat, 2><<<grid, kLnWarps * 32, psm, st>>>((const Tin*)x, (const Tin*)w, (const Tin*)b, (Tout*)y, (Tstat*)mu, (Tstat*)sigma, degenerate, rows, cols, eps); break;
          default: ln_fwd_warp<Tin, Tout, Tstat, 4><<<grid, kLnWarps * 32, psm, st>>>((const Tin*)x, (const Tin*)w, (const Tin*)b, (Tout*)y, (Tstat*)mu, (Tstat*)sigma, degenerate, rows, cols, eps); break;
        }
      } else {
        const int grid = (int)std::min<int64_t>(rows, kNumSMs * 16);
        ln_fwd_block<Tin, Tout, Tstat><<<grid, 256, 0, st>>>((const Tin*)x, (const Tin*)w, (const Tin*)b, (Tout*)y, (Tstat*)mu, (Tstat*)sigma, degenerate, rows, cols, eps);
      }
      return check_launch("layernorm_fwd");
    });
  });
}

int ls2_layernorm_bwd_nblk(int64_t rows, int64_t cols) {
  return (cols % 8 == 0 && cols <= 1024 && cols >= 8) ? ln_bwd_blocks(rows, cols) : 0;
}

int64_t ls2_layernorm_bwd_ws_bytes(int64_t rows, int64_t cols) {
  (void)rows;
  return (int64_t)kLnMaxBlocks * 3 * cols * (int64_t)sizeof(double);
}

int ls2_bdr_layernorm_fwd(const void* x, const void* bias, const void* res, void* yres,
                          uint8_t* keep_bits, const void* w, const void* b, void* u, void* mu,
                          void* sigma, int64_t rows, int64_t cols, double eps, int use_drop,
                          uint64_t seed, const uint64_t* seed_ptr, uint64_t thresh, double dscale,
                          int tin, int tout, int tstat, void* stream) {
  if (rows <= 0) return LS2_OK;
  if (!ln_vec_ok(cols, {x, bias, res, yres, w, b, u}))
    return fail(LS2_ERR_SHAPE, "bdr_layernorm_fwd: needs cols % 8 == 0, <= 1024, aligned");
  cudaStream_t st = as_stream(stream);
  return LS2_DISPATCH_IO(tin, tout, "bdr_layernorm_fwd", [&] {
    return LS2_DISPATCH_STAT(tstat, [&] {
      using C = typename CompOf<Tin>::type;
      auto go = [&](auto iters, auto drop, auto genc) {
        constexpr int I = decltype(iters)::value;
        constexpr bool D = decltype(drop)::value, G = decltype(genc)::value;
        const size_t psm = 3 * (size_t)cols * sizeof(Tin);
        const int grid = resident_grid((const void*)ln_fwd_bdr_warp<Tin, Tout, Tstat, I, D, G>,
                                       kLnWarps * 32, psm, ceil_div(rows, kLnWarps));
        ln_fwd_bdr_warp<Tin, Tout, Tstat, I, D, G><<<grid, kLnWarps * 32, psm, st>>>(
            (const Tin*)x, (const Tin*)bias, (const Tin*)res, (Tout*)yres, keep_bits,
            (const Tin*)w, (const Tin*)b, (Tout*)u, (Tstat*)mu, (Tstat*)sigma, rows, cols, eps,
            seed, seed_ptr, thresh, (C)dscale);
        return check_launch("bdr_layernorm_fwd");
      };
      using I1 = std::integral_constant<int, 1>;
      using I2 = std::integral_constant<int, 2>;
      using I4 = std::integral_constant<int, 4>;
      using T_ = std::true_type;
      using F_ = std::false_type;
      const int it = ln_iters(cols);
      if (use_drop == 2)      // read the keep bits (mask bank)
        return it == 1 ? go(I1{}, T_{}, F_{}) : it == 2 ? go(I2{}, T_{}, F_{}) : go(I4{}, T_{}, F_{});
      if (use_drop)
        return it == 1 ? go(I1{}, T_{}, T_{}) : it == 2 ? go(I2{}, T_{}, T_{}) : go(I4{}, T_{}, T_{});
      return it == 1 ? go(I1{}, F_{}, T_{}) : it == 2 ? go(I2{}, F_{}, T_{}) : go(I4{}, F_{}, T_{});
    });
  });
}

int ls2_layernorm_bwd_bdr(const void* dy, const void* x, const void* w, const void* mu,
                          const void* sigma, const void* dres, void* dx, const uint8_t* keep_bits,
                          void* dproj, int use_drop, double dscale, void* dw, void* db,
                          void* dbias, int tparam, int beta_mask, void* ws, int64_t rows,
                          int64_t cols, int tin, int tout, int tstat, void* stream) {
  if (rows <= 0) return LS2_OK;
  if (!ln_vec_ok(cols, {dy, x, w, dres, dx, dproj}))
    return fail(LS2_ERR_SHAPE, "layernorm_bwd_bdr: needs cols % 8 == 0, <= 1024, aligned");
  cudaStream_t st = as_stream(stream);
  const int nblk = ln_bwd_blocks(rows, cols);
  int rc = LS2_DISPATCH_IO(tin, tout, "layernorm_bwd_bdr", [&] {
    return LS2_DISPATCH_STAT(tstat, [&] {
      auto go = [&](auto iters, auto res, auto drop) {
        constexpr int I = decltype(iters)::value;
        constexpr bool R = decltype(res)::value, D = decltype(drop)::value;
        return ln_bwd_launch<Tin, Tout, Tstat, I, R, true, D>(dy, x, w, mu, sigma, dres, dx,
                                                              keep_bits, dproj, dscale, ws, rows,
                                                              cols, st);
      };
      using I1 = std::integral_constant<int, 1>;
      using I2 = std::integral_constant<int, 2>;
      using I4 = std::integral_constant<int, 4>;
      using T_ = std::true_type;
      using F_ = std::false_type;
      const int it = ln_iters(cols);
      auto by_iters = [&](auto res, auto drop) {
        return it == 1 ? go(I1{}, res, drop) : it == 2 ? go(I2{}, res, drop) : go(I4{}, res, drop);
      };
      if (dres) return use_drop ? by_iters(T_{}, T_{}) : by_iters(T_{}, F_{});
      return use_drop ? by_iters(F_{}, T_{}) : by_iters(F_{}, F_{});
    });
  });
  if (rc || !dw) return rc;   // dw == NULL: partials stay in ws (deferred finish)
  return LS2_DISPATCH_ONE(tparam, "layernorm_bwd_bdr_finish", [&] {
    ln_param_finish<Tx, 3><<<(unsigned)ceil_div(cols, 32), 1024, 0, st>>>(
        (const double*)ws, nblk, cols, (Tx*)dw, (Tx*)db, (Tx*)dbias, beta_mask);
    return check_launch("layernorm_bwd_bdr_finish");
  });
}

int ls2_layernorm_bwd(const void* dy, const void* x, const void* w, const void* mu,
                      const void* sigma, const void* dres, void* dx, void* dw, void* db,
                      int tparam, int beta_param, void* ws, int64_t rows, int64_t cols, int tin,
                      int tout, int tstat, void* stream) {
  if (cols < 2) return fail(LS2_ERR_SHAPE, "layernorm needs m >= 2");
  cudaStream_t st = as_stream(stream);
  if (rows <= 0) return LS2_OK;
  const bool vec = ln_vec_ok(cols, {dy, x, w, dres, dx});
  const int nblk = vec ? ln_bwd_blocks(rows, cols) : ln_generic_blocks(rows);
  int rc = LS2_DISPATCH_IO(tin, tout, "layernorm_bwd", [&] {
    return LS2_DISPATCH_STAT(tstat, [&] {
      if (vec) {
        auto go = [&](auto iters, auto res) {
          constexpr int I = decltype(iters)::value;
          constexpr bool R = decltype(res)::value;
          return ln_bwd_launch<Tin, Tout, Tstat, I, R, false, false>(
              dy, x, w, mu, sigma, dres, dx, nullptr, nullptr, 1.0, ws, rows, cols, st);
        };
        using I1 = std::integral_constant<int, 1>;
        using I2 = std::integral_constant<int, 2>;
        using I4 = std::integral_constant<int, 4>;
        using T_ = std::true_type;
        using F_ = std::false_type;
        const int it = ln_iters(cols);
        if (dres) return it == 1 ? go(I1{}, T_{}) : it == 2 ? go(I2{}, T_{}) : go(I4{}, T_{});
        return it == 1 ? go(I1{}, F_{}) : it == 2 ? go(I2{}, F_{}) : go(I4{}, F_{});
      }
      const int grid = (int)std::min<int64_t>(rows, kNumSMs * 16);
      ln_bwd_block<Tin, Tout, Tstat><<<grid, 256, 0, st>>>(
          (const Tin*)dy, (const Tin*)x, (const Tin*)w, (const Tstat*)mu, (const Tstat*)sigma,
          (const Tin*)dres, (Tout*)dx, rows, cols);
      int r = check_launch("layernorm_bwd");
      if (r) return r;
      ln_param_partial<Tin, Tstat><<<nblk, 256, 0, st>>>((const Tin*)dy, (const Tin*)x,
                                                         (const Tstat*)mu, (const Tstat*)sigma,
                                                         (double*)ws, rows, cols);
      return check_launch("layernorm_param_partial");
    });
  });
  if (rc) return rc;
  if (!dw || !db) return LS2_OK;
  return LS2_DISPATCH_ONE(tparam, "layernorm_param_finish", [&] {
    ln_param_finish<Tx, 2><<<(unsigned)ceil_div(cols, 32), 1024, 0, st>>>(
        (const double*)ws, nblk, cols, (Tx*)dw, (Tx*)db, nullptr, beta_param ? 3 : 0);
    return check_launch("layernorm_param_finish");
  });
}

}  // extern "C"
