// Fused element-wise tails with 1-bit dropout masks, and deterministic
// column sums for their bias gradients.
//   bias_dropout_residual      F/kernels.py:367-382, F/gradients.py:147-159
//   bias_relu_dropout          F/kernels.py:385-403, F/gradients.py:162-172
//   bias column sums           F/model.py:501,726,766 and F/model.py:258
//
// Layout: x[rows, cols] row-major.  A thread owns 8 consecutive elements of a
// row ("column group" cg, 16-byte loads for 16-bit types) and one byte of each
// bit mask; the CTA tiles (rows_per_pass x column groups) and walks rows with a
// fixed stride, so the per-thread column-group never changes and bias loads,
// bias-gradient partials and mask bytes need no div/mod in the loop.
#include "common.cuh"

namespace ls2 {

constexpr int kTPB = 256;
constexpr int kMaxColsumBlocks = kNumSMs;  // one partial row per SM: short finish

struct Tiling {
  int64_t cgs;      // column groups per row (cols / 8)
  int threads;      // CTA size
  int rpp;          // rows per pass per CTA
  int64_t passes;   // total row passes
};

inline Tiling tiling(int64_t rows, int64_t cols) {
  Tiling t;
  t.cgs = cols / 8;
  if (t.cgs <= kTPB) {
    t.threads = kTPB;
    t.rpp = (int)(kTPB / t.cgs);
  } else {
    t.threads = (int)(ceil_div(t.cgs, 32) * 32);
    t.rpp = 1;
  }
  t.passes = ceil_div(rows, t.rpp);
  return t;
}

// tiling for kernels that also reduce columns: 1024-thread CTAs (256 for f64, whose
// smem partials are twice as wide) so <= 148 CTAs still keep every SM busy
inline Tiling tiling_cs(int64_t rows, int64_t cols, bool f64) {
  const int tpb = f64 ? 256 : 1024;
  Tiling t;
  t.cgs = cols / 8;
  if (t.cgs <= tpb) {
    t.rpp = (int)(tpb / t.cgs);
    t.threads = (int)(ceil_div((int64_t)t.rpp * t.cgs, 32) * 32);
  } else {
    t.threads = (int)(ceil_div(t.cgs, 32) * 32);
    t.rpp = 1;
  }
  t.passes = ceil_div(rows, t.rpp);
  return t;
}

// fixed (shape-only) grid for the column-sum kernels => deterministic results
inline int colsum_blocks(int64_t passes) {
  int64_t g = ceil_div(passes, 2);
  return (int)(g < 1 ? 1 : (g > kMaxColsumBlocks ? kMaxColsumBlocks : g));
}

// fast path: cols % 8 == 0, cols/8 <= 1024, all pointers 16-byte aligned
inline bool vec_ok(int64_t cols, std::initializer_list<const void*> ptrs) {
  if (cols % 8 != 0 || cols / 8 > 1024) return false;
  if (cols > 6144) return false;  // bwd colsum smem (rpp*cols doubles) stays <= 48 KB
  for (const void* p : ptrs)
    if (p && !aligned16(p)) return false;
  return true;
}

template <typename T>
__device__ __forceinline__ void load_row_group(const T* p, float (&v)[8]) {
  Pack8<T> q = ld8(p);
#pragma unroll
  for (int e = 0; e < 8; ++e) v[e] = cvt<float>(q.v[e]);
}
template <typename T>
__device__ __forceinline__ void load_row_group(const T* p, double (&v)[8]) {
  Pack8<T> q = ld8(p);
#pragma unroll
  for (int e = 0; e < 8; ++e) v[e] = cvt<double>(q.v[e]);
}
template <typename T, typename C>
__device__ __forceinline__ void store_row_group(T* p, const C (&v)[8]) {
  Pack8<T> q;
#pragma unroll
  for (int e = 0; e < 8; ++e) q.v[e] = cvt<T>(v[e]);
  st8(p, q);
}

// ---------------------------------------------------------------------------
// column-sum stage 2: out[c] (+)= sum_g partial[g, c] in fixed order
// ---------------------------------------------------------------------------
// CTA = 32 warps x 32 columns; warp w sums partial rows w, w+32, ... (coalesced
// 256-byte row segments), then the 32 warp sums are added in fixed order ->
// deterministic, and with <= 148 partial rows only ~5 dependent L2 round trips.
template <typename Tout>
__global__ void __launch_bounds__(1024) colsum_finish_kernel(const double* __restrict__ partial,
                                                             int nblk, int64_t cols,
                                                             Tout* __restrict__ out, int beta) {
  __shared__ double red[32][33];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t c = (int64_t)blockIdx.x * 32 + lane;
  double s0 = 0, s1 = 0;
  if (c < cols) {
    int g = w;
    for (; g + 32 < nblk; g += 64) {
      s0 += partial[(int64_t)g * cols + c];
      s1 += partial[(int64_t)(g + 32) * cols + c];
    }
    for (; g < nblk; g += 32) s0 += partial[(int64_t)g * cols + c];
  }
  red[w][lane] = s0 + s1;
  __syncthreads();
  if (w == 0 && c < cols) {
    double s = 0;
#pragma unroll
    for (int k = 0; k < 32; ++k) s += red[k][lane];
    if (beta) s += cvt<double>(out[c]);
    out[c] = cvt<Tout>(s);
  }
}

int colsum_finish(const double* partial, int nblk, int64_t cols, void* out, int tout, int beta,
                  cudaStream_t st) {
  return LS2_DISPATCH_ONE(tout, "colsum_finish", [&] {
    colsum_finish_kernel<Tx><<<(unsigned)ceil_div(cols, 32), 1024, 0, st>>>(partial, nblk, cols,
                                                                          (Tx*)out, beta);
    return check_launch("colsum_finish");
  });
}

// CTA-level reduction of the per-thread 8-column partials (rpp row lanes per
// column group) into partial[blockIdx, cols], fixed order.  smem holds the
// partials in the compute type (f32, or f64 for the f64 path).
template <typename C>
__device__ __forceinline__ void cta_colsum_store(const C (&acc)[8], int64_t cgs, int rpp,
                                                 int64_t cols, double* __restrict__ partial,
                                                 C* smem) {
  const int tid = threadIdx.x;
  const int lane_row = (int)(tid / cgs);
  const int64_t cg = tid % cgs;
  if (lane_row < rpp) {
#pragma unroll
    for (int e = 0; e < 8; ++e) smem[(int64_t)lane_row * cols + cg * 8 + e] = acc[e];
  }
  __syncthreads();
  for (int64_t c = tid; c < cols; c += blockDim.x) {
    double s = 0.0;
    for (int r = 0; r < rpp; ++r) s += (double)smem[(int64_t)r * cols + c];
    partial[(int64_t)blockIdx.x * cols + c] = s;
  }
}

// rows a thread of the vectorised elementwise kernels has in flight per pass
constexpr int kRowsInFlight = 4;

template <typename C>
__device__ __forceinline__ C* colsum_smem() {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  return reinterpret_cast<C*>(smem_raw);
}

// ---------------------------------------------------------------------------
// bias + dropout + residual
// ---------------------------------------------------------------------------
template <typename Tin, typename Tout, bool DROP, bool GEN>
__global__ void __launch_bounds__(1024) bdr_fwd_vec(const Tin* __restrict__ x, const Tin* __restrict__ bias,
                                  const Tin* __restrict__ res, Tout* __restrict__ y,
                                  uint8_t* __restrict__ bits, int64_t rows, int64_t cols,
                                  int64_t cgs, int rpp, uint64_t seed, const uint64_t* seed_ptr, uint64_t thresh,
                                  typename CompOf<Tin>::type scale) {
  using C = typename CompOf<Tin>::type;
  const int lane_row = (int)(threadIdx.x / cgs);
  if (lane_row >= rpp) return;
  const int64_t cg = threadIdx.x % cgs;
  C b[8];
  load_row_group(bias + cg * 8, b);
  for (int64_t r = (int64_t)blockIdx.x * rpp + lane_row; r < rows; r += (int64_t)gridDim.x * rpp) {
    const int64_t g = r * cgs + cg;
    C xv[8], rv[8];
    load_row_group(x + g * 8, xv);
    load_row_group(res + g * 8, rv);
    uint32_t kb = 0xFF;
    if (DROP) {
      if (GEN) {
        kb = keep_byte(seed_ptr ? *seed_ptr : seed, (uint64_t)g * 8, thresh);
        bits[g] = (uint8_t)kb;
      } else {
        kb = bits[g];
      }
    }
    C o[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      C a = add_rn(xv[e], b[e]);
      if (DROP) a = mul_rn(mul_rn(a, bitval<C>(kb, e)), scale);
      o[e] = add_rn(a, rv[e]);
    }
    store_row_group(y + g * 8, o);
  }
}

// generic path: any cols / alignment; one thread per 8-element flat group
template <typename Tin, typename Tout, bool DROP, bool GEN>
__global__ void bdr_fwd_flat(const Tin* __restrict__ x, const Tin* __restrict__ bias,
                             const Tin* __restrict__ res, Tout* __restrict__ y,
                             uint8_t* __restrict__ bits, int64_t n, int64_t cols, uint64_t seed, const uint64_t* seed_ptr,
                             uint64_t thresh, typename CompOf<Tin>::type scale) {
  using C = typename CompOf<Tin>::type;
  const int64_t groups = (n + 7) / 8;
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < groups;
       g += (int64_t)gridDim.x * blockDim.x) {
    uint32_t kb = 0xFF;
    if (DROP) {
      if (GEN) {
        kb = keep_byte(seed_ptr ? *seed_ptr : seed, (uint64_t)g * 8, thresh);
        const int64_t valid = n - g * 8;
        if (valid < 8) kb &= (1u << valid) - 1u;
        bits[g] = (uint8_t)kb;
      } else {
        kb = bits[g];
      }
    }
    for (int e = 0; e < 8; ++e) {
      const int64_t i = g * 8 + e;
      if (i >= n) break;
      C a = add_rn(cvt<C>(x[i]), cvt<C>(bias[i % cols]));
      if (DROP) a = mul_rn(mul_rn(a, bitval<C>(kb, e)), scale);
      y[i] = cvt<Tout>(add_rn(a, cvt<C>(res[i])));
    }
  }
}

template <typename Tin, typename Tout, bool DROP>
__global__ void __launch_bounds__(1024) bdr_bwd_vec(const Tin* __restrict__ dy, const uint8_t* __restrict__ bits,
                                  Tout* __restrict__ dx, double* __restrict__ partial,
                                  int64_t rows, int64_t cols, int64_t cgs, int rpp,
                                  typename CompOf<Tin>::type scale) {
  using C = typename CompOf<Tin>::type;
  const int lane_row = (int)(threadIdx.x / cgs);
  const int64_t cg = threadIdx.x % cgs;
  C acc[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) acc[e] = 0;
  if (lane_row < rpp) {
    for (int64_t r = (int64_t)blockIdx.x * rpp + lane_row; r < rows; r += (int64_t)gridDim.x * rpp) {
      const int64_t g = r * cgs + cg;
      C d[8];
      load_row_group(dy + g * 8, d);
      const uint32_t kb = DROP ? bits[g] : 0xFF;
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        if (DROP) d[e] = mul_rn(mul_rn(d[e], bitval<C>(kb, e)), scale);
        acc[e] += d[e];
      }
      store_row_group(dx + g * 8, d);
    }
  }
  cta_colsum_store(acc, cgs, rpp, cols, partial, colsum_smem<C>());
}

template <typename Tin, typename Tout, bool DROP>
__global__ void bdr_bwd_flat(const Tin* __restrict__ dy, const uint8_t* __restrict__ bits,
                             Tout* __restrict__ dx, int64_t n, typename CompOf<Tin>::type scale) {
  using C = typename CompOf<Tin>::type;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    C d = cvt<C>(dy[i]);
    if (DROP) d = mul_rn(mul_rn(d, bitval<C>(bits[i >> 3], (int)(i & 7))), scale);
    dx[i] = cvt<Tout>(d);
  }
}

// ---------------------------------------------------------------------------
// bias + relu + dropout
// ---------------------------------------------------------------------------
template <typename Tin, typename Tout, bool DROP, bool GEN>
__global__ void __launch_bounds__(1024) brd_fwd_vec(const Tin* __restrict__ x, const Tin* __restrict__ bias,
                                  Tout* __restrict__ y, uint8_t* __restrict__ kbits,
                                  uint8_t* __restrict__ rbits, int64_t rows, int64_t cols,
                                  int64_t cgs, int rpp, uint64_t seed, const uint64_t* seed_ptr, uint64_t thresh,
                                  typename CompOf<Tin>::type scale) {
  using C = typename CompOf<Tin>::type;
  const int lane_row = (int)(threadIdx.x / cgs);
  if (lane_row >= rpp) return;
  const int64_t cg = threadIdx.x % cgs;
  C b[8];
  load_row_group(bias + cg * 8, b);
  // (one row per pass: unrolling 4 rows in flight measured slower here, 7.97 -> 8.34 us)
  for (int64_t r = (int64_t)blockIdx.x * rpp + lane_row; r < rows; r += (int64_t)gridDim.x * rpp) {
    const int64_t g = r * cgs + cg;
    C xv[8];
    load_row_group(x + g * 8, xv);
    uint32_t kb = 0xFF;
    if (DROP) {
      if (GEN) {
        kb = keep_byte(seed_ptr ? *seed_ptr : seed, (uint64_t)g * 8, thresh);
        kbits[g] = (uint8_t)kb;
      } else {
        kb = kbits[g];
      }
    }
    uint32_t rb = 0;
    C o[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      C a = add_rn(xv[e], b[e]);
      const bool pos = a > (C)0;
      rb |= (uint32_t)pos << e;
      a = mul_rn(a, (C)(pos ? 1 : 0));
      if (DROP) a = mul_rn(mul_rn(a, bitval<C>(kb, e)), scale);
      o[e] = a;
    }
    if (rbits) rbits[g] = (uint8_t)rb;
    store_row_group(y + g * 8, o);
  }
}

template <typename Tin, typename Tout, bool DROP, bool GEN>
__global__ void brd_fwd_flat(const Tin* __restrict__ x, const Tin* __restrict__ bias,
                             Tout* __restrict__ y, uint8_t* __restrict__ kbits,
                             uint8_t* __restrict__ rbits, int64_t n, int64_t cols, uint64_t seed, const uint64_t* seed_ptr,
                             uint64_t thresh, typename CompOf<Tin>::type scale) {
  using C = typename CompOf<Tin>::type;
  const int64_t groups = (n + 7) / 8;
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < groups;
       g += (int64_t)gridDim.x * blockDim.x) {
    uint32_t kb = 0xFF;
    if (DROP) {
      if (GEN) {
        kb = keep_byte(seed_ptr ? *seed_ptr : seed, (uint64_t)g * 8, thresh);
        const int64_t valid = n - g * 8;
        if (valid < 8) kb &= (1u << valid) - 1u;
        kbits[g] = (uint8_t)kb;
      } else {
        kb = kbits[g];
      }
    }
    uint32_t rb = 0;
    for (int e = 0; e < 8; ++e) {
      const int64_t i = g * 8 + e;
      if (i >= n) break;
      C a = add_rn(cvt<C>(x[i]), cvt<C>(bias[i % cols]));
      const bool pos = a > (C)0;
      rb |= (uint32_t)pos << e;
      a = mul_rn(a, (C)(pos ? 1 : 0));
      if (DROP) a = mul_rn(mul_rn(a, bitval<C>(kb, e)), scale);
      y[i] = cvt<Tout>(a);
    }
    if (rbits) rbits[g] = (uint8_t)rb;
  }
}

template <typename Tin, typename Tout, bool DROP>
__global__ void __launch_bounds__(1024) brd_bwd_vec(const Tin* __restrict__ dy, const uint8_t* __restrict__ kbits,
                                  const uint8_t* __restrict__ rbits, Tout* __restrict__ dx,
                                  double* __restrict__ partial, int64_t rows, int64_t cols,
                                  int64_t cgs, int rpp, typename CompOf<Tin>::type scale) {
  using C = typename CompOf<Tin>::type;
  const int lane_row = (int)(threadIdx.x / cgs);
  const int64_t cg = threadIdx.x % cgs;
  C acc[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) acc[e] = 0;
  if (lane_row < rpp) {
    // kRowsInFlight rows per pass: all their loads issue before any use, so a
    // thread keeps several 16-byte reads in flight (same row order as a plain
    // grid-stride loop: the column sums are unchanged bit for bit)
    const int64_t stride = (int64_t)gridDim.x * rpp;
    for (int64_t r0 = (int64_t)blockIdx.x * rpp + lane_row; r0 < rows; r0 += kRowsInFlight * stride) {
      Pack8<Tin> pd[kRowsInFlight];
      uint32_t rb[kRowsInFlight], kb[kRowsInFlight];
#pragma unroll
      for (int u = 0; u < kRowsInFlight; ++u) {
        const int64_t r = r0 + u * stride;
        if (r < rows) {
          const int64_t g = r * cgs + cg;
          pd[u] = ld8_stream(dy + g * 8);
          rb[u] = rbits[g];
          kb[u] = DROP ? kbits[g] : 0xFF;
        }
      }
#pragma unroll
      for (int u = 0; u < kRowsInFlight; ++u) {
        const int64_t r = r0 + u * stride;
        if (r < rows) {
          const int64_t g = r * cgs + cg;
          C d[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            // (d * relu) * keep == d * (relu & keep) for 0/1 factors, signed zeros
            // and NaN included: one multiply by the combined bit
            d[e] = mul_rn(cvt<C>(pd[u].v[e]), bitval<C>(DROP ? rb[u] & kb[u] : rb[u], e));
            if (DROP) d[e] = mul_rn(d[e], scale);
            acc[e] += d[e];
          }
          store_row_group(dx + g * 8, d);
        }
      }
    }
  }
  cta_colsum_store(acc, cgs, rpp, cols, partial, colsum_smem<C>());
}

template <typename Tin, typename Tout, bool DROP>
__global__ void brd_bwd_flat(const Tin* __restrict__ dy, const uint8_t* __restrict__ kbits,
                             const uint8_t* __restrict__ rbits, Tout* __restrict__ dx, int64_t n,
                             typename CompOf<Tin>::type scale) {
  using C = typename CompOf<Tin>::type;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    C d = mul_rn(cvt<C>(dy[i]), bitval<C>(rbits[i >> 3], (int)(i & 7)));
    if (DROP) d = mul_rn(mul_rn(d, bitval<C>(kbits[i >> 3], (int)(i & 7))), scale);
    dx[i] = cvt<Tout>(d);
  }
}

// ---------------------------------------------------------------------------
// generic column sums (stage 1): thread per column, CTA per row chunk
// ---------------------------------------------------------------------------
template <typename T>
__global__ void colsum_stage1(const T* __restrict__ x, int64_t rows, int64_t cols,
                              double* __restrict__ partial) {
  const int64_t per = (rows + gridDim.x - 1) / gridDim.x;
  const int64_t r0 = blockIdx.x * per;
  const int64_t r1 = min(rows, r0 + per);
  for (int64_t c = threadIdx.x; c < cols; c += blockDim.x) {
    double s = 0.0;
    for (int64_t r = r0; r < r1; ++r) s += cvt<double>(x[r * cols + c]);
    partial[(int64_t)blockIdx.x * cols + c] = s;
  }
}

// generic-path bias gradient: column sums of dx recomputed from dy in the
// compute precision (so 16-bit dx storage does not round the sum's terms)
template <typename Tin>
__global__ void masked_colsum_stage1(const Tin* __restrict__ dy, const uint8_t* __restrict__ kbits,
                                     const uint8_t* __restrict__ rbits, int use_drop,
                                     typename CompOf<Tin>::type scale, int64_t rows, int64_t cols,
                                     double* __restrict__ partial) {
  using C = typename CompOf<Tin>::type;
  const int64_t per = (rows + gridDim.x - 1) / gridDim.x;
  const int64_t r0 = blockIdx.x * per;
  const int64_t r1 = min(rows, r0 + per);
  for (int64_t c = threadIdx.x; c < cols; c += blockDim.x) {
    double s = 0.0;
    for (int64_t r = r0; r < r1; ++r) {
      const int64_t i = r * cols + c;
      C d = cvt<C>(dy[i]);
      if (rbits) d = mul_rn(d, bitval<C>(rbits[i >> 3], (int)(i & 7)));
      if (use_drop) d = mul_rn(mul_rn(d, bitval<C>(kbits[i >> 3], (int)(i & 7))), scale);
      s += (double)d;
    }
    partial[(int64_t)blockIdx.x * cols + c] = s;
  }
}

template <typename Tin>
int masked_colsum(const Tin* dy, const uint8_t* kbits, const uint8_t* rbits, int use_drop,
                  double scale, int64_t rows, int64_t cols, void* out, int tout, int beta, void* ws,
                  cudaStream_t st);

template <typename T>
__global__ void bias_add_kernel(T* __restrict__ x, const T* __restrict__ bias, int64_t n,
                                int64_t cols) {
  using C = typename CompOf<T>::type;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    x[i] = cvt<T>(add_rn(cvt<C>(x[i]), cvt<C>(bias[i % cols])));
}

// vectorized stage 1: same (row lanes x column groups) tiling as the fused tails
template <typename Tin>
__global__ void __launch_bounds__(1024) colsum_vec(const Tin* __restrict__ x,
                                                   double* __restrict__ partial, int64_t rows,
                                                   int64_t cols, int64_t cgs, int rpp) {
  using C = typename CompOf<Tin>::type;
  const int lane_row = (int)(threadIdx.x / cgs);
  const int64_t cg = threadIdx.x % cgs;
  C acc[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) acc[e] = 0;
  if (lane_row < rpp) {
    for (int64_t r = (int64_t)blockIdx.x * rpp + lane_row; r < rows; r += (int64_t)gridDim.x * rpp) {
      C v[8];
      load_row_group(x + (r * cgs + cg) * 8, v);
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[e] += v[e];
    }
  }
  cta_colsum_store(acc, cgs, rpp, cols, partial, colsum_smem<C>());
}

inline int colsum_generic(const void* x, int tin, int64_t rows, int64_t cols, void* out, int tout,
                          int beta, void* ws, cudaStream_t st) {
  if (vec_ok(cols, {x})) {
    Tiling t = tiling_cs(rows, cols, tin == LS2_F64);
    const int grid = colsum_blocks(t.passes);
    const size_t sm = (size_t)t.rpp * cols * (tin == LS2_F64 ? 8 : 4);
    int rc = LS2_DISPATCH_ONE(tin, "colsum", [&] {
      colsum_vec<Tx><<<grid, t.threads, sm, st>>>((const Tx*)x, (double*)ws, rows, cols, t.cgs,
                                                  t.rpp);
      return check_launch("colsum_vec");
    });
    if (rc || !out) return rc;
    return colsum_finish((const double*)ws, grid, cols, out, tout, beta, st);
  }
  const int nblk = colsum_blocks(ceil_div(rows, 16));
  int rc = LS2_DISPATCH_ONE(tin, "colsum", [&] {
    colsum_stage1<Tx><<<nblk, kTPB, 0, st>>>((const Tx*)x, rows, cols, (double*)ws);
    return check_launch("colsum_stage1");
  });
  if (rc) return rc;
  return colsum_finish((const double*)ws, nblk, cols, out, tout, beta, st);
}

template <typename T>
inline typename CompOf<T>::type cscale(double s) {
  return (typename CompOf<T>::type)s;
}

template <typename Tin>
int masked_colsum(const Tin* dy, const uint8_t* kbits, const uint8_t* rbits, int use_drop,
                  double scale, int64_t rows, int64_t cols, void* out, int tout, int beta, void* ws,
                  cudaStream_t st) {
  const int nblk = colsum_blocks(ceil_div(rows, 16));
  masked_colsum_stage1<Tin><<<nblk, kTPB, 0, st>>>(dy, kbits, rbits, use_drop, cscale<Tin>(scale),
                                                   rows, cols, (double*)ws);
  int rc = check_launch("masked_colsum_stage1");
  if (rc) return rc;
  return colsum_finish((const double*)ws, nblk, cols, out, tout, beta, st);
}

}  // namespace ls2

using namespace ls2;

extern "C" {

int ls2_colsum_nblk(int64_t rows, int64_t cols, int dtype) {
  if (cols % 8 != 0 || cols / 8 > 1024 || cols > 6144 || rows <= 0) return 0;
  return colsum_blocks(tiling_cs(rows, cols, dtype == LS2_F64).passes);
}

int64_t ls2_colsum_ws_bytes(int64_t rows, int64_t cols) {
  (void)rows;
  return (int64_t)kMaxColsumBlocks * cols * (int64_t)sizeof(double);
}

int ls2_colsum(const void* x, int tin, void* out, int tout, int beta, void* ws, int64_t rows,
               int64_t cols, void* stream) {
  if (cols <= 0) return LS2_OK;
  if (rows <= 0) {
    if (beta) return LS2_OK;
    return cudaMemsetAsync(out, 0, cols * (tout == LS2_F64 ? 8 : tout == LS2_F32 ? 4 : 2),
                           as_stream(stream)) == cudaSuccess ? LS2_OK : fail(LS2_ERR_CUDA, "memset");
  }
  return colsum_generic(x, tin, rows, cols, out, tout, beta, ws, as_stream(stream));
}

int ls2_bias_add(void* x, const void* bias, int64_t rows, int64_t cols, int dtype, void* stream) {
  const int64_t n = rows * cols;
  if (n <= 0) return LS2_OK;
  return LS2_DISPATCH_ONE(dtype, "bias_add", [&] {
    bias_add_kernel<Tx><<<grid_for(n), kTPB, 0, as_stream(stream)>>>((Tx*)x, (const Tx*)bias, n, cols);
    return check_launch("bias_add");
  });
}

int ls2_bias_dropout_residual_fwd(const void* x, const void* bias, const void* res, void* y,
                                  uint8_t* keep_bits, int64_t rows, int64_t cols, int use_drop,
                                  int gen, uint64_t seed, const uint64_t* seed_ptr, uint64_t thresh, double scale, int tin,
                                  int tout, void* stream) {
  const int64_t n = rows * cols;
  if (n <= 0) return LS2_OK;
  cudaStream_t st = as_stream(stream);
  const bool vec = vec_ok(cols, {x, bias, res, y});
  return LS2_DISPATCH_IO(tin, tout, "bias_dropout_residual_fwd", [&] {
    auto sc = cscale<Tin>(scale);
    auto launch = [&](auto drop, auto genc) {
      constexpr bool D = decltype(drop)::value, G = decltype(genc)::value;
      if (vec) {
        Tiling t = tiling(rows, cols);
        int grid = resident_grid((const void*)bdr_fwd_vec<Tin, Tout, D, G>, t.threads, 0, t.passes);
        bdr_fwd_vec<Tin, Tout, D, G><<<grid, t.threads, 0, st>>>(
            (const Tin*)x, (const Tin*)bias, (const Tin*)res, (Tout*)y, keep_bits, rows, cols,
            t.cgs, t.rpp, seed, seed_ptr, thresh, sc);
      } else {
        bdr_fwd_flat<Tin, Tout, D, G><<<grid_for(ceil_div(n, 8)), kTPB, 0, st>>>(
            (const Tin*)x, (const Tin*)bias, (const Tin*)res, (Tout*)y, keep_bits, n, cols, seed,
            seed_ptr, thresh, sc);
      }
      return check_launch("bias_dropout_residual_fwd");
    };
    using T_ = std::true_type;
    using F_ = std::false_type;
    if (!use_drop) return launch(F_{}, F_{});
    return gen ? launch(T_{}, T_{}) : launch(T_{}, F_{});
  });
}

int ls2_bias_dropout_residual_bwd(const void* dy, const uint8_t* keep_bits, void* dx, void* dbias,
                                  int tbias, int beta_bias, void* ws, int64_t rows, int64_t cols,
                                  int use_drop, double scale, int tin, int tout, void* stream) {
  const int64_t n = rows * cols;
  if (n <= 0) return LS2_OK;
  cudaStream_t st = as_stream(stream);
  const bool vec = vec_ok(cols, {dy, dx});
  int rc = LS2_DISPATCH_IO(tin, tout, "bias_dropout_residual_bwd", [&] {
    auto sc = cscale<Tin>(scale);
    if (vec) {
      Tiling t = tiling_cs(rows, cols, tin == LS2_F64);
      int grid = colsum_blocks(t.passes);
      size_t sm = (size_t)t.rpp * cols * sizeof(typename CompOf<Tin>::type);
      if (use_drop)
        bdr_bwd_vec<Tin, Tout, true><<<grid, t.threads, sm, st>>>(
            (const Tin*)dy, keep_bits, (Tout*)dx, (double*)ws, rows, cols, t.cgs, t.rpp, sc);
      else
        bdr_bwd_vec<Tin, Tout, false><<<grid, t.threads, sm, st>>>(
            (const Tin*)dy, keep_bits, (Tout*)dx, (double*)ws, rows, cols, t.cgs, t.rpp, sc);
      int r = check_launch("bias_dropout_residual_bwd");
      if (r || !dbias) return r;  // dbias == NULL: partials stay in ws (deferred finish)
      return colsum_finish((const double*)ws, grid, cols, dbias, tbias, beta_bias, st);
    }
    if (use_drop)
      bdr_bwd_flat<Tin, Tout, true><<<grid_for(n), kTPB, 0, st>>>((const Tin*)dy, keep_bits,
                                                                   (Tout*)dx, n, sc);
    else
      bdr_bwd_flat<Tin, Tout, false><<<grid_for(n), kTPB, 0, st>>>((const Tin*)dy, keep_bits,
                                                                    (Tout*)dx, n, sc);
    int r = check_launch("bias_dropout_residual_bwd");
    if (r || !dbias) return r;
    return masked_colsum<Tin>((const Tin*)dy, keep_bits, nullptr, use_drop, scale, rows, cols,
                              dbias, tbias, beta_bias, ws, st);
  });
  return rc;
}

int ls2_bias_relu_dropout_fwd(const void* x, const void* bias, void* y, uint8_t* keep_bits,
                              uint8_t* relu_bits, int64_t rows, int64_t cols, int use_drop,
                              int gen, uint64_t seed, const uint64_t* seed_ptr, uint64_t thresh, double scale, int tin,
                              int tout, void* stream) {
  const int64_t n = rows * cols;
  if (n <= 0) return LS2_OK;
  cudaStream_t st = as_stream(stream);
  const bool vec = vec_ok(cols, {x, bias, y});
  return LS2_DISPATCH_IO(tin, tout, "bias_relu_dropout_fwd", [&] {
    auto sc = cscale<Tin>(scale);
    auto launch = [&](auto drop, auto genc) {
      constexpr bool D = decltype(drop)::value, G = decltype(genc)::value;
      if (vec) {
        Tiling t = tiling(rows, cols);
        int grid = resident_grid((const void*)brd_fwd_vec<Tin, Tout, D, G>, t.threads, 0, t.passes);
        brd_fwd_vec<Tin, Tout, D, G><<<grid, t.threads, 0, st>>>(
            (const Tin*)x, (const Tin*)bias, (Tout*)y, keep_bits, relu_bits, rows, cols, t.cgs,
            t.rpp, seed, seed_ptr, thresh, sc);
      } else {
        brd_fwd_flat<Tin, Tout, D, G><<<grid_for(ceil_div(n, 8)), kTPB, 0, st>>>(
            (const Tin*)x, (const Tin*)bias, (Tout*)y, keep_bits, relu_bits, n, cols, seed,
            seed_ptr, thresh, sc);
      }
      return check_launch("bias_relu_dropout_fwd");
    };
    using T_ = std::true_type;
    using F_ = std::false_type;
    if (!use_drop) return launch(F_{}, F_{});
    return gen ? launch(T_{}, T_{}) : launch(T_{}, F_{});
  });
}

int ls2_bias_relu_dropout_bwd(const void* dy, const uint8_t* keep_bits, const uint8_t* relu_bits,
                              void* dx, void* dbias, int tbias, int beta_bias, void* ws,
                              int64_t rows, int64_t cols, int use_drop, double scale, int tin,
                              int tout, void* stream) {
  const int64_t n = rows * cols;
  if (n <= 0) return LS2_OK;
  cudaStream_t st = as_stream(stream);
  const bool vec = vec_ok(cols, {dy, dx});
  return LS2_DISPATCH_IO(tin, tout, "bias_relu_dropout_bwd", [&] {
    auto sc = cscale<Tin>(scale);
    if (vec) {
      Tiling t = tiling_cs(rows, cols, tin == LS2_F64);
      int grid = colsum_blocks(t.passes);
      size_t sm = (size_t)t.rpp * cols * sizeof(typename CompOf<Tin>::type);
      if (use_drop)
        brd_bwd_vec<Tin, Tout, true><<<grid, t.threads, sm, st>>>(
            (const Tin*)dy, keep_bits, relu_bits, (Tout*)dx, (double*)ws, rows, cols, t.cgs,
            t.rpp, sc);
      else
        brd_bwd_vec<Tin, Tout, false><<<grid, t.threads, sm, st>>>(
            (const Tin*)dy, keep_bits, relu_bits, (Tout*)dx, (double*)ws, rows, cols, t.cgs,
            t.rpp, sc);
      int r = check_launch("bias_relu_dropout_bwd");
      if (r || !dbias) return r;  // dbias == NULL: partials stay in ws (deferred finish)
      return colsum_finish((const double*)ws, grid, cols, dbias, tbias, beta_bias, st);
    }
    if (use_drop)
      brd_bwd_flat<Tin, Tout, true><<<grid_for(n), kTPB, 0, st>>>(
          (const Tin*)dy, keep_bits, relu_bits, (Tout*)dx, n, sc);
    else
      brd_bwd_flat<Tin, Tout, false><<<grid_for(n), kTPB, 0, st>>>(
          (const Tin*)dy, keep_bits, relu_bits, (Tout*)dx, n, sc);
    int r = check_launch("bias_relu_dropout_bwd");
    if (r || !dbias) return r;
    return masked_colsum<Tin>((const Tin*)dy, keep_bits, relu_bits, use_drop, scale, rows, cols,
                              dbias, tbias, beta_bias, ws, st);
  });
}

}  // extern "C"
