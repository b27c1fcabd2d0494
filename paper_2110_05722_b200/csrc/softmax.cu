// Attention softmax (masked, scaled), its backward, and log-softmax.
//   softmax_forward        F/kernels.py:277-307 (3-step: max, partition, normalize;
//                          masked positions excluded and emitting exact 0)
//   AttentionMask          F/kernels.py:113-144 (masks computed from indices here)
//   softmax_backward       F/gradients.py:77-100 (+ the 1/sqrt(hd) of F/model.py:490)
//   log_softmax_forward    F/kernels.py:310-331
//
// The reference picks a row-reduction "strategy" per shape (F/kernels.py:80-106);
// the B200 analogue is the shape template chosen here: G lanes per row (a
// sub-warp group, G = 1..32), each lane holding ITERS chunks of VEC contiguous
// elements in registers; rows longer than 32*16*VEC use one CTA per row.
#include <cfloat>
#include <type_traits>

#include "common.cuh"

namespace ls2 {

struct MaskSpec {
  int kind;
  int64_t lq, heads;
  const int64_t* lens;
  const uint8_t* dense;
};

__device__ __forceinline__ bool kept(const MaskSpec& m, int64_t row, int64_t col, int64_t cols) {
  switch (m.kind) {
    case LS2_MASK_CAUSAL: return col <= row % m.lq;
    case LS2_MASK_PADDING: return col < m.lens[row / (m.heads * m.lq)];
    case LS2_MASK_DENSE: return m.dense[row * cols + col] != 0;
    default: return true;
  }
}

// the row's kept columns are a prefix [0, limit) for every mask kind but dense:
// evaluated once per row instead of per element (the padding length is a load)
__device__ __forceinline__ int64_t kept_limit(const MaskSpec& m, int64_t row, int64_t cols) {
  switch (m.kind) {
    case LS2_MASK_CAUSAL: return row % m.lq + 1;
    case LS2_MASK_PADDING: return m.lens[row / (m.heads * m.lq)];
    default: return cols;
  }
}

__device__ __forceinline__ float fexp(float x) { return __expf(x); }
__device__ __forceinline__ double fexp(double x) { return exp(x); }
__device__ __forceinline__ float flog(float x) { return __logf(x); }
__device__ __forceinline__ double flog(double x) { return log(x); }
template <typename C> __device__ __forceinline__ C neg_inf() { return -INFINITY; }

// MODE 0: softmax, MODE 1: log-softmax.  ACC64: f64 partition sum (the explicit
// row_serial strategy, which must agree with the tree kernel to 1 ULP); the
// default (shape-rule) path sums in fp32
template <typename Tin, typename Tout, int VEC, int ITERS, int MODE, bool ACC64 = false>
__global__ void __launch_bounds__(256) softmax_rows(const Tin* __restrict__ x, Tout* __restrict__ y,
                                                    int64_t rows, int64_t cols, int G, MaskSpec m,
                                                    double in_scale, int* all_masked) {
  using C = typename CompOf<Tin>::type;
  const int lane = threadIdx.x & 31;
  const int sub = lane % G;
  const int rows_per_warp = 32 / G;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const C sc = (C)in_scale;
  for (int64_t r0 = warp * rows_per_warp; r0 < rows; r0 += nwarps * rows_per_warp) {
    const int64_t r = r0 + lane / G;
    const bool live = r < rows;
    const bool dense = m.kind == LS2_MASK_DENSE;
    const int64_t lim = live && !dense ? kept_limit(m, r, cols) : cols;
    C v[ITERS][VEC];
    C mx = neg_inf<C>();
#pragma unroll
    for (int it = 0; it < ITERS; ++it) {
      const int64_t c0 = (int64_t)(sub + G * it) * VEC;
      if (VEC == 8 && live && c0 < cols) {
        Pack8<Tin> q = ld8(x + r * cols + c0);
#pragma unroll
        for (int e = 0; e < VEC; ++e) v[it][e] = cvt<C>(q.v[e]);
      } else {
#pragma unroll
        for (int e = 0; e < VEC; ++e)
          v[it][e] = (live && c0 + e < cols) ? cvt<C>(x[r * cols + c0 + e]) : (C)0;
      }
#pragma unroll
      for (int e = 0; e < VEC; ++e) {
        const int64_t c = c0 + e;
        const bool ok = live && c < cols && c < lim && (!dense || kept(m, r, c, cols));
        v[it][e] = ok ? v[it][e] * sc : neg_inf<C>();
        mx = max(mx, v[it][e]);
      }
    }
    mx = warp_max(mx, G);
    // the partition sum accumulates in f64 (the reference's float64 reduction), so
    // this template and the tree kernel round it identically (1-ULP agreement)
    using Z = typename std::conditional<ACC64, double, C>::type;
    Z zd = 0;
#pragma unroll
    for (int it = 0; it < ITERS; ++it)
#pragma unroll
      for (int e = 0; e < VEC; ++e) {
        const C ex = (v[it][e] == neg_inf<C>()) ? (C)0 : fexp(v[it][e] - mx);
        if (MODE == 0) v[it][e] = ex;
        zd += (Z)ex;
      }
    zd = warp_sum(zd, G);
    if (!live) continue;
    if (MODE == 0 && mx == neg_inf<C>() && all_masked && sub == 0) *all_masked = 1;
    const C z = (C)zd;
    const C rz = (MODE == 0) ? (z > (C)0 ? (C)1 / z : (C)0) : flog(z);
#pragma unroll
    for (int it = 0; it < ITERS; ++it) {
      const int64_t c0 = (int64_t)(sub + G * it) * VEC;
      C o[VEC];
#pragma unroll
      for (int e = 0; e < VEC; ++e) o[e] = (MODE == 0) ? v[it][e] * rz : (v[it][e] - mx) - rz;
      if (VEC == 8 && c0 < cols) {
        Pack8<Tout> q;
#pragma unroll
        for (int e = 0; e < VEC; ++e) q.v[e] = cvt<Tout>(o[e]);
        st8(y + r * cols + c0, q);
      } else {
#pragma unroll
        for (int e = 0; e < VEC; ++e)
          if (c0 + e < cols) y[r * cols + c0 + e] = cvt<Tout>(o[e]);
      }
    }
  }
}

template <typename Tin, typename Tout, int VEC, int ITERS>
__global__ void __launch_bounds__(256) softmax_bwd_rows(const Tin* __restrict__ dy,
                                                        const Tin* __restrict__ q,
                                                        Tout* __restrict__ dx, int64_t rows,
                                                        int64_t cols, int G, double out_scale) {
  using C = typename CompOf<Tin>::type;
  const int lane = threadIdx.x & 31;
  const int sub = lane % G;
  const int rows_per_warp = 32 / G;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r0 = warp * rows_per_warp; r0 < rows; r0 += nwarps * rows_per_warp) {
    const int64_t r = r0 + lane / G;
    const bool live = r < rows;
    C dv[ITERS][VEC], qv[ITERS][VEC];
    C s = 0;
#pragma unroll
    for (int it = 0; it < ITERS; ++it) {
      const int64_t c0 = (int64_t)(sub + G * it) * VEC;
      if (VEC == 8 && live && c0 < cols) {
        Pack8<Tin> a = ld8(dy + r * cols + c0), b = ld8(q + r * cols + c0);
#pragma unroll
        for (int e = 0; e < VEC; ++e) { dv[it][e] = cvt<C>(a.v[e]); qv[it][e] = cvt<C>(b.v[e]); }
      } else {
#pragma unroll
        for (int e = 0; e < VEC; ++e) {
          const bool ok = live && c0 + e < cols;
          dv[it][e] = ok ? cvt<C>(dy[r * cols + c0 + e]) : (C)0;
          qv[it][e] = ok ? cvt<C>(q[r * cols + c0 + e]) : (C)0;
        }
      }
#pragma unroll
      for (int e = 0; e < VEC; ++e) s += dv[it][e] * qv[it][e];
    }
    s = warp_sum(s, G);
    if (!live) continue;
    const C os = (C)out_scale;
#pragma unroll
    for (int it = 0; it < ITERS; ++it) {
      const int64_t c0 = (int64_t)(sub + G * it) * VEC;
      C o[VEC];
#pragma unroll
      for (int e = 0; e < VEC; ++e) o[e] = qv[it][e] * (dv[it][e] - s) * os;
      if (VEC == 8 && c0 < cols) {
        Pack8<Tout> p;
#pragma unroll
        for (int e = 0; e < VEC; ++e) p.v[e] = cvt<Tout>(o[e]);
        st8(dx + r * cols + c0, p);
      } else {
#pragma unroll
        for (int e = 0; e < VEC; ++e)
          if (c0 + e < cols) dx[r * cols + c0 + e] = cvt<Tout>(o[e]);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// long rows: one CTA per row (online max/sum pass, then an output pass)
// ---------------------------------------------------------------------------
// Fixed-shape CTA reductions (lane shuffles, then warp slots in order):
// deterministic for a given blockDim.
template <typename T>
__device__ __forceinline__ T block_max(T v, T* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) red[wid] = v;
  __syncthreads();
  T m = red[0];
  for (int i = 1; i < (int)(blockDim.x >> 5); ++i) m = max(m, red[i]);
  __syncthreads();
  return m;
}

template <typename T>
__device__ __forceinline__ T block_sum(T v, T* red) {
  v = warp_sum(v);
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) red[wid] = v;
  __syncthreads();
  T s = 0;
  for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s += red[i];
  __syncthreads();
  return s;
}

// row_parallel_tree (F/kernels.py:63-74, selected at :80-106): one CTA per row,
// three passes over the row (max; f64 partition sum of exp(v - max); output).
// The statistics are the warp template's exactly (same max, same exp, an f64 sum
// rounded once), so the two strategies agree to within 1 ULP.
template <typename Tin, typename Tout, int MODE>
__global__ void softmax_block(const Tin* __restrict__ x, Tout* __restrict__ y, int64_t rows,
                              int64_t cols, MaskSpec msk, double in_scale, int* all_masked) {
  using C = typename CompOf<Tin>::type;
  __shared__ C redm[32];
  __shared__ double reds[32];
  const C sc = (C)in_scale;
  for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
    const Tin* xr = x + r * cols;
    C m = neg_inf<C>();
    for (int64_t c = threadIdx.x; c < cols; c += blockDim.x)
      if (kept(msk, r, c, cols)) m = max(m, cvt<C>(xr[c]) * sc);
    m = block_max(m, redm);
    double zd = 0;
    if (m != neg_inf<C>())
      for (int64_t c = threadIdx.x; c < cols; c += blockDim.x)
        if (kept(msk, r, c, cols)) zd += (double)fexp(cvt<C>(xr[c]) * sc - m);
    zd = block_sum(zd, reds);
    if (MODE == 0 && m == neg_inf<C>() && all_masked && threadIdx.x == 0) *all_masked = 1;
    const C z = (C)zd;
    const C rz = (MODE == 0) ? (z > (C)0 ? (C)1 / z : (C)0) : flog(z);
    for (int64_t c = threadIdx.x; c < cols; c += blockDim.x) {
      const C v = cvt<C>(xr[c]) * sc;
      C o;
      if (MODE == 0) o = kept(msk, r, c, cols) ? fexp(v - m) * rz : (C)0;
      else o = (v - m) - rz;
      y[r * cols + c] = cvt<Tout>(o);
    }
  }
}

template <typename Tin, typename Tout>
__global__ void softmax_bwd_block(const Tin* __restrict__ dy, const Tin* __restrict__ q,
                                  Tout* __restrict__ dx, int64_t rows, int64_t cols,
                                  double out_scale) {
  using C = typename CompOf<Tin>::type;
  __shared__ C red[32];
  for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
    C s = 0;
    for (int64_t c = threadIdx.x; c < cols; c += blockDim.x)
      s += cvt<C>(dy[r * cols + c]) * cvt<C>(q[r * cols + c]);
    s = warp_sum(s);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    s = 0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s += red[i];
    __syncthreads();
    for (int64_t c = threadIdx.x; c < cols; c += blockDim.x) {
      const C qv = cvt<C>(q[r * cols + c]);
      dx[r * cols + c] = cvt<Tout>(qv * (cvt<C>(dy[r * cols + c]) - s) * (C)out_scale);
    }
  }
}

struct RowShape {
  int vec, G, iters;
  bool block;
};

inline RowShape row_shape(int64_t cols, bool vec8) {
  RowShape s;
  s.vec = vec8 ? 8 : 1;
  const int64_t chunks = ceil_div(cols, s.vec);
  int G = 1;
  while (G < 32 && G < chunks) G <<= 1;
  int64_t it = ceil_div(chunks, G);
  int iters = 1;
  while (iters < it) iters <<= 1;
  s.G = G;
  s.iters = iters;
  s.block = iters > (vec8 ? 4 : 8);
  return s;
}

inline int rows_grid(int64_t rows, int G) {
  const int64_t warps = ceil_div(rows, 32 / G);
  int64_t blocks = ceil_div(warps, 8);
  if (blocks > kNumSMs * 32) blocks = kNumSMs * 32;
  return (int)(blocks < 1 ? 1 : blocks);
}

template <int MODE, typename Tin, typename Tout>
int launch_rows(const void* x, void* y, int64_t rows, int64_t cols, const MaskSpec& m,
                double in_scale, int* all_masked, cudaStream_t st, int strategy = 0) {
  const bool v8 = cols % 8 == 0 && aligned16(x) && aligned16(y);
  RowShape s = row_shape(cols, v8);
  if (s.block || strategy == LS2_SOFTMAX_TREE) {
    const int grid = (int)std::min<int64_t>(rows, kNumSMs * 16);
    softmax_block<Tin, Tout, MODE><<<grid, 512, 0, st>>>((const Tin*)x, (Tout*)y, rows, cols, m,
                                                          in_scale, all_masked);
    return check_launch("softmax_block");
  }
  const int grid = rows_grid(rows, s.G);
#define LS2_SM_CASE(V, I)                                                                 \
  if (s.vec == V && s.iters == I) {                                                       \
    if (strategy == LS2_SOFTMAX_SERIAL)                                                   \
      softmax_rows<Tin, Tout, V, I, MODE, true><<<grid, 256, 0, st>>>(                    \
          (const Tin*)x, (Tout*)y, rows, cols, s.G, m, in_scale, all_masked);             \
    else                                                                                  \
      softmax_rows<Tin, Tout, V, I, MODE><<<grid, 256, 0, st>>>((const Tin*)x, (Tout*)y, rows, \
                                                               cols, s.G, m, in_scale, all_masked); \
    return check_launch("softmax_rows");                                                  \
  }
  LS2_SM_CASE(8, 1) LS2_SM_CASE(8, 2) LS2_SM_CASE(8, 4)
  LS2_SM_CASE(1, 1) LS2_SM_CASE(1, 2) LS2_SM_CASE(1, 4) LS2_SM_CASE(1, 8)
#undef LS2_SM_CASE
  return fail(LS2_ERR_SHAPE, "softmax: no shape template");
}

template <typename Tin, typename Tout>
int launch_bwd_rows(const void* dy, const void* q, void* dx, int64_t rows, int64_t cols,
                    double out_scale, cudaStream_t st) {
  const bool v8 = cols % 8 == 0 && aligned16(dy) && aligned16(q) && aligned16(dx);
  RowShape s = row_shape(cols, v8);
  if (s.block) {
    const int grid = (int)std::min<int64_t>(rows, kNumSMs * 16);
    softmax_bwd_block<Tin, Tout><<<grid, 512, 0, st>>>((const Tin*)dy, (const Tin*)q, (Tout*)dx,
                                                        rows, cols, out_scale);
    return check_launch("softmax_bwd_block");
  }
  const int grid = rows_grid(rows, s.G);
#define LS2_SMB_CASE(V, I)                                                                \
  if (s.vec == V && s.iters == I) {                                                       \
    softmax_bwd_rows<Tin, Tout, V, I><<<grid, 256, 0, st>>>((const Tin*)dy, (const Tin*)q,  \
                                                           (Tout*)dx, rows, cols, s.G, out_scale); \
    return check_launch("softmax_bwd_rows");                                              \
  }
  LS2_SMB_CASE(8, 1) LS2_SMB_CASE(8, 2) LS2_SMB_CASE(8, 4)
  LS2_SMB_CASE(1, 1) LS2_SMB_CASE(1, 2) LS2_SMB_CASE(1, 4) LS2_SMB_CASE(1, 8)
#undef LS2_SMB_CASE
  return fail(LS2_ERR_SHAPE, "softmax_bwd: no shape template");
}

}  // namespace ls2

using namespace ls2;

extern "C" {

int ls2_softmax_fwd(const void* x, void* y, int64_t rows, int64_t cols, int mask_kind, int64_t lq,
                    int64_t heads, const int64_t* valid_lens, const uint8_t* dense_keep,
                    double in_scale, int* all_masked, int tin, int tout, void* stream) {
  return ls2_softmax_fwd_strategy(x, y, rows, cols, mask_kind, lq, heads, valid_lens, dense_keep,
                                  in_scale, all_masked, LS2_SOFTMAX_AUTO, tin, tout, stream);
}

int ls2_softmax_fwd_strategy(const void* x, void* y, int64_t rows, int64_t cols, int mask_kind,
                             int64_t lq, int64_t heads, const int64_t* valid_lens,
                             const uint8_t* dense_keep, double in_scale, int* all_masked,
                             int strategy, int tin, int tout, void* stream) {
  if (rows <= 0 || cols <= 0) return LS2_OK;
  if (strategy < LS2_SOFTMAX_AUTO || strategy > LS2_SOFTMAX_TREE)
    return fail(LS2_ERR_SHAPE, "softmax: unknown strategy");
  if ((mask_kind == LS2_MASK_CAUSAL || mask_kind == LS2_MASK_PADDING) && lq <= 0)
    return fail(LS2_ERR_SHAPE, "softmax: mask needs lq >= 1");
  MaskSpec m{mask_kind, lq < 1 ? 1 : lq, heads < 1 ? 1 : heads, valid_lens, dense_keep};
  return LS2_DISPATCH_IO(tin, tout, "softmax_fwd", [&] {
    return launch_rows<0, Tin, Tout>(x, y, rows, cols, m, in_scale, all_masked,
                                     as_stream(stream), strategy);
  });
}

int ls2_log_softmax_fwd(const void* h, void* y, int64_t rows, int64_t cols, int tin, int tout,
                        void* stream) {
  return ls2_log_softmax_fwd_strategy(h, y, rows, cols, LS2_SOFTMAX_AUTO, tin, tout, stream);
}

int ls2_log_softmax_fwd_strategy(const void* h, void* y, int64_t rows, int64_t cols, int strategy,
                                 int tin, int tout, void* stream) {
  if (rows <= 0 || cols <= 0) return LS2_OK;
  if (strategy < LS2_SOFTMAX_AUTO || strategy > LS2_SOFTMAX_TREE)
    return fail(LS2_ERR_SHAPE, "log_softmax: unknown strategy");
  MaskSpec m{LS2_MASK_NONE, 1, 1, nullptr, nullptr};
  return LS2_DISPATCH_IO(tin, tout, "log_softmax_fwd", [&] {
    return launch_rows<1, Tin, Tout>(h, y, rows, cols, m, 1.0, nullptr, as_stream(stream),
                                     strategy);
  });
}

int ls2_softmax_bwd(const void* dy, const void* q, void* dx, int64_t rows, int64_t cols,
                    double out_scale, int tin, int tout, void* stream) {
  if (rows <= 0 || cols <= 0) return LS2_OK;
  return LS2_DISPATCH_IO(tin, tout, "softmax_bwd", [&] {
    return launch_bwd_rows<Tin, Tout>(dy, q, dx, rows, cols, out_scale, as_stream(stream));
  });
}

}  // extern "C"
