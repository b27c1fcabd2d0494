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

template <typename Tin, typename Tout, typename Tstat, int ITERS>
__global__ void __launch_bounds__(kLnWarps * 32) ln_fwd_warp(
    const Tin* __restrict__ x, const Tin* __restrict__ w, const Tin* __restrict__ b,
    Tout* __restrict__ y, Tstat* __restrict__ mu, Tstat* __restrict__ sigma,
    int* __restrict__ degenerate, int64_t rows, int64_t cols, double eps) {
  using C = typename CompOf<Tin>::type;
  const int lane = threadIdx.x & 31;
  const int64_t cgs = cols / 8;
  C wv[ITERS][8], bv[ITERS][8];
#pragma unroll
  for (int it = 0; it < ITERS; ++it) {
    const int64_t g = lane + 32 * it;
    if (g < cgs) {
      ld_group(w + g * 8, wv[it]);
      ld_group(b + g * 8, bv[it]);
    }
  }
  const double inv_m = 1.0 / (double)cols;
  for (int64_t r = (int64_t)blockIdx.x * kLnWarps + (threadIdx.x >> 5); r < rows;
       r += (int64_t)gridDim.x * kLnWarps) {
    const Tin* xr = x + r * cols;
    C v[ITERS][8];
#pragma unroll
    for (int it = 0; it < ITERS; ++it) {
      const int64_t g = lane + 32 * it;
      if (g < cgs) ld_group(xr + g * 8, v[it]);
    }
    const C pivot = __shfl_sync(0xffffffffu, v[0][0], 0);
    C s1 = 0, s2 = 0;
#pragma unroll
    for (int it = 0; it < ITERS; ++it) {
      if (lane + 32 * it < cgs) {
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          v[it][e] -= pivot;
          s1 += v[it][e];
          s2 += v[it][e] * v[it][e];
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
#pragma unroll
        for (int e = 0; e < 8; ++e) o[e] = (v[it][e] - msh) * rs * wv[it][e] + bv[it][e];
        st_group(yr + g * 8, o);
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
template <typename Tin, typename Tout, typename Tstat, int ITERS, bool RES>
__global__ void __launch_bounds__(kLnBwdWarps * 32) ln_bwd_warp(
    const Tin* __restrict__ dy, const Tin* __restrict__ x, const Tin* __restrict__ w,
    const Tstat* __restrict__ mu, const Tstat* __restrict__ sigma, const Tin* __restrict__ dres,
    Tout* __restrict__ dx, double* __restrict__ partial, int64_t rows, int64_t cols) {
  using C = typename CompOf<Tin>::type;
  __shared__ double red[kLnBwdWarps][2][256];  // per-warp column partials, one chunk at a time
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t cgs = cols / 8;
  C wv[ITERS][8], adw[ITERS][8], adb[ITERS][8];
#pragma unroll
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int e = 0; e < 8; ++e) { adw[it][e] = 0; adb[it][e] = 0; }
    const int64_t g = lane + 32 * it;
    if (g < cgs) ld_group(w + g * 8, wv[it]);
  }
  const C inv_m = (C)(1.0 / (double)cols);
  for (int64_t r = (int64_t)blockIdx.x * kLnBwdWarps + wid; r < rows;
       r += (int64_t)gridDim.x * kLnBwdWarps) {
    const C m_r = (C)mu[r];
    const C rs = (C)(1.0 / (double)sigma[r]);
    C xh[ITERS][8], gg[ITERS][8];
    C r1 = 0, r3 = 0;
#pragma unroll
    for (int it = 0; it < ITERS; ++it) {
      const int64_t g = lane + 32 * it;
      if (g < cgs) {
        C d[8];
        ld_group(dy + r * cols + g * 8, d);
        ld_group(x + r * cols + g * 8, xh[it]);
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          xh[it][e] = (xh[it][e] - m_r) * rs;
          gg[it][e] = wv[it][e] * d[e];
          r1 += gg[it][e];
          r3 += gg[it][e] * xh[it][e];
          adw[it][e] += d[e] * xh[it][e];
          adb[it][e] += d[e];
        }
      }
    }
    r1 = warp_sum(r1) * inv_m;
    r3 = warp_sum(r3) * inv_m;
#pragma unroll
    for (int it = 0; it < ITERS; ++it) {
      const int64_t g = lane + 32 * it;
      if (g < cgs) {
        C o[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) o[e] = (gg[it][e] - r1 - xh[it][e] * r3) * rs;
        if (RES) {
          C rr[8];
          ld_group(dres + r * cols + g * 8, rr);
#pragma unroll
          for (int e = 0; e < 8; ++e) o[e] += rr[e];
        }
        st_group(dx + r * cols + g * 8, o);
      }
    }
  }
  // CTA reduction of the warps' column partials (fixed order) in chunks of 256 cols
#pragma unroll
  for (int it = 0; it < ITERS; ++it) {
    const int64_t g = lane + 32 * it;
    if (g < cgs) {
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        red[wid][0][lane * 8 + e] = (double)adw[it][e];
        red[wid][1][lane * 8 + e] = (double)adb[it][e];
      }
    }
    __syncthreads();
    const int64_t base = (int64_t)it * 256;
    for (int c = threadIdx.x; c < 256 && base + c < cols; c += blockDim.x) {
      double sw = 0, sb = 0;
#pragma unroll
      for (int k = 0; k < kLnBwdWarps; ++k) { sw += red[k][0][c]; sb += red[k][1][c]; }
      partial[((int64_t)blockIdx.x * 2 + 0) * cols + base + c] = sw;
      partial[((int64_t)blockIdx.x * 2 + 1) * cols + base + c] = sb;
    }
    __syncthreads();
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
template <typename Tp>
__global__ void __launch_bounds__(1024) ln_param_finish(const double* __restrict__ partial,
                                                        int nblk, int64_t cols,
                                                        Tp* __restrict__ dw, Tp* __restrict__ db,
                                                        int beta) {
  __shared__ double red[2][32][33];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t c = (int64_t)blockIdx.x * 32 + lane;
  double sw0 = 0, sw1 = 0, sb0 = 0, sb1 = 0;
  if (c < cols) {
    int g = w;
    for (; g + 32 < nblk; g += 64) {
      sw0 += partial[((int64_t)g * 2 + 0) * cols + c];
      sb0 += partial[((int64_t)g * 2 + 1) * cols + c];
      sw1 += partial[((int64_t)(g + 32) * 2 + 0) * cols + c];
      sb1 += partial[((int64_t)(g + 32) * 2 + 1) * cols + c];
    }
    for (; g < nblk; g += 32) {
      sw0 += partial[((int64_t)g * 2 + 0) * cols + c];
      sb0 += partial[((int64_t)g * 2 + 1) * cols + c];
    }
  }
  red[0][w][lane] = sw0 + sw1;
  red[1][w][lane] = sb0 + sb1;
  __syncthreads();
  if (w == 0 && c < cols) {
    double sw = 0, sb = 0;
#pragma unroll
    for (int k = 0; k < 32; ++k) { sw += red[0][k][lane]; sb += red[1][k][lane]; }
    if (beta) { sw += cvt<double>(dw[c]); sb += cvt<double>(db[c]); }
    dw[c] = cvt<Tp>(sw);
    db[c] = cvt<Tp>(sb);
  }
}

inline bool ln_vec_ok(int64_t cols, std::initializer_list<const void*> ptrs) {
  if (cols % 8 != 0 || cols > 1024 || cols < 8) return false;
  for (const void* p : ptrs)
    if (p && !aligned16(p)) return false;
  return true;
}

inline int ln_iters(int64_t cols) { return cols <= 256 ? 1 : cols <= 512 ? 2 : 4; }

inline int ln_bwd_blocks(int64_t rows) {
  int64_t g = ceil_div(rows, kLnBwdWarps * 2);
  return (int)(g < 1 ? 1 : (g > kLnMaxBlocks ? kLnMaxBlocks : g));
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
        const int grid = (int)std::min<int64_t>(ceil_div(rows, kLnWarps), kNumSMs * 16);
        switch (ln_iters(cols)) {
          case 1: ln_fwd_warp<Tin, Tout, Tstat, 1><<<grid, kLnWarps * 32, 0, st>>>((const Tin*)x, (const Tin*)w, (const Tin*)b, (Tout*)y, (Tstat*)mu, (Tstat*)sigma, degenerate, rows, cols, eps); break;
          case 2: ln_fwd_warp<Tin, Tout, Tstat, 2><<<grid, kLnWarps * 32, 0, st>>>((const Tin*)x, (const Tin*)w, (const Tin*)b, (Tout*)y, (Tstat*)mu, (Tstat*)sigma, degenerate, rows, cols, eps); break;
          default: ln_fwd_warp<Tin, Tout, Tstat, 4><<<grid, kLnWarps * 32, 0, st>>>((const Tin*)x, (const Tin*)w, (const Tin*)b, (Tout*)y, (Tstat*)mu, (Tstat*)sigma, degenerate, rows, cols, eps); break;
        }
      } else {
        const int grid = (int)std::min<int64_t>(rows, kNumSMs * 16);
        ln_fwd_block<Tin, Tout, Tstat><<<grid, 256, 0, st>>>((const Tin*)x, (const Tin*)w, (const Tin*)b, (Tout*)y, (Tstat*)mu, (Tstat*)sigma, degenerate, rows, cols, eps);
      }
      return check_launch("layernorm_fwd");
    });
  });
}

int64_t ls2_layernorm_bwd_ws_bytes(int64_t rows, int64_t cols) {
  (void)rows;
  return (int64_t)kLnMaxBlocks * 2 * cols * (int64_t)sizeof(double);
}

int ls2_layernorm_bwd(const void* dy, const void* x, const void* w, const void* mu,
                      const void* sigma, const void* dres, void* dx, void* dw, void* db,
                      int tparam, int beta_param, void* ws, int64_t rows, int64_t cols, int tin,
                      int tout, int tstat, void* stream) {
  if (cols < 2) return fail(LS2_ERR_SHAPE, "layernorm needs m >= 2");
  cudaStream_t st = as_stream(stream);
  if (rows <= 0) return LS2_OK;
  const bool vec = ln_vec_ok(cols, {dy, x, w, dres, dx});
  const int nblk = ln_bwd_blocks(rows);
  int rc = LS2_DISPATCH_IO(tin, tout, "layernorm_bwd", [&] {
    return LS2_DISPATCH_STAT(tstat, [&] {
      if (vec) {
        auto go = [&](auto iters, auto res) {
          constexpr int I = decltype(iters)::value;
          constexpr bool R = decltype(res)::value;
          ln_bwd_warp<Tin, Tout, Tstat, I, R><<<nblk, kLnBwdWarps * 32, 0, st>>>(
              (const Tin*)dy, (const Tin*)x, (const Tin*)w, (const Tstat*)mu, (const Tstat*)sigma,
              (const Tin*)dres, (Tout*)dx, (double*)ws, rows, cols);
          return check_launch("layernorm_bwd");
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
    ln_param_finish<Tx><<<(unsigned)ceil_div(cols, 32), 1024, 0, st>>>((const double*)ws, nblk, cols, (Tx*)dw,
                                                         (Tx*)db, beta_param);
    return check_launch("layernorm_param_finish");
  });
}

}  // extern "C"
