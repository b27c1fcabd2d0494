// Label-smoothed cross-entropy criterion.
//   log_softmax + ls_cross_entropy_forward  F/kernels.py:310-360
//   ls_cross_entropy_backward                F/gradients.py:47-74
//   criterion glue (argmax/correct, exp)     F/model.py:908-932
//
// ls2_criterion_fused: one CTA per logits row.  The row is read from HBM once
// into registers (V <= 32768 for 16-bit logits), max/argmax, partition sum and
// the row sum of logits are reduced in one traversal, the smoothed loss is
//   loss_r = -(1-a) * logq[k] - (a/V) * sum_i logq[i],
//   sum_i logq[i] = sum_i h_i - V * (max + log Z),
// and dlogits = (softmax - a/V - (1-a)[i==k]) * grad_scale is written back
// over the same row (in place).  Longer rows take a two-pass variant whose
// second read hits L2.  Per-row (loss, correct) partials are reduced in a fixed
// order by a single-CTA kernel, so the loss is bit-reproducible.
#include <cfloat>

#include "common.cuh"

namespace ls2 {

constexpr int kCeThreads = 512;

struct MaxIdx {
  float v;
  int64_t i;
};

__device__ __forceinline__ void mi_merge(MaxIdx& a, const MaxIdx& b) {
  // numpy argmax: first index among equal maxima; NaN propagates as max
  if (b.v > a.v || (b.v == a.v && b.i < a.i) || (isnan(b.v) && !isnan(a.v))) a = b;
}

__device__ MaxIdx block_argmax(MaxIdx m) {
  __shared__ float sv[32];
  __shared__ int64_t si[32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    MaxIdx b{__shfl_xor_sync(0xffffffffu, m.v, o), __shfl_xor_sync(0xffffffffu, m.i, o)};
    mi_merge(m, b);
  }
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) { sv[wid] = m.v; si[wid] = m.i; }
  __syncthreads();
  MaxIdx r{sv[0], si[0]};
  for (int k = 1; k < (int)(blockDim.x >> 5); ++k) mi_merge(r, MaxIdx{sv[k], si[k]});
  __syncthreads();
  return r;
}

__device__ float block_max(float v) {
  __shared__ float s[32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) s[wid] = v;
  __syncthreads();
  float r = s[0];
  for (int k = 1; k < (int)(blockDim.x >> 5); ++k) r = fmaxf(r, s[k]);
  __syncthreads();
  return r;
}

__device__ int block_min(int v) {
  __shared__ int s[32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) s[wid] = v;
  __syncthreads();
  int r = s[0];
  for (int k = 1; k < (int)(blockDim.x >> 5); ++k) r = min(r, s[k]);
  __syncthreads();
  return r;
}

template <typename T>
__device__ T block_sum(T v) {
  __shared__ T s[32];
  v = warp_sum(v);
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) s[wid] = v;
  __syncthreads();
  T r = 0;
  for (int k = 0; k < (int)(blockDim.x >> 5); ++k) r += s[k];
  __syncthreads();
  return r;
}

// exp(h - max) in (0, 1] is cached in the logits' storage type; for fp16 it is
// scaled by 2^15 so values down to ~1e-9 stay normal (fp16 subnormals would
// cost the gradient precision of the smallest probabilities)
template <typename T> struct ExCache { static constexpr float kScale = 1.f, kInv = 1.f; };
template <> struct ExCache<__half> { static constexpr float kScale = 32768.f, kInv = 1.f / 32768.f; };

// ITERS > 0: register-cached single pass (8*ITERS elements per thread);
// ITERS == 0: two passes over the row.
template <typename T, int ITERS>
__global__ void __launch_bounds__(kCeThreads, ITERS >= 4 ? 1 : 2) criterion_kernel(
    const T* __restrict__ logits, const int64_t* __restrict__ targets, T* dlogits, T* logq_out,
    double* __restrict__ row_stats, int* __restrict__ bad_target, int64_t rows, int64_t V,
    double alpha, int64_t pad_id, int has_pad, double grad_scale) {
  const int64_t r = blockIdx.x;
  if (r >= rows) return;
  const T* h = logits + r * V;
  const int64_t tgt = targets[r];
  const bool valid = !(has_pad && tgt == pad_id);
  const bool tgt_ok = tgt >= 0 && tgt < V;
  if (valid && !tgt_ok && threadIdx.x == 0 && bad_target) *bad_target = 1;

  // the row stays in registers in its storage type (16-bit: 4 regs per 8 values)
  Pack8<T> cache[ITERS > 0 ? ITERS : 1];
  MaxIdx mi{-INFINITY, INT64_MAX};
  float sh = 0.f;
  if (ITERS > 0) {
    // pass 1: max and sum of logits (fp32 max only; the argmax index is found
    // afterwards as the first position holding the row max: numpy's tie rule)
    float m = -INFINITY;
#pragma unroll
    for (int it = 0; it < (ITERS > 0 ? ITERS : 1); ++it) {
      const int c0 = (it * kCeThreads + (int)threadIdx.x) * 8;
      if (c0 < V) cache[it] = ld8_stream(h + c0);
    }
#pragma unroll
    for (int it = 0; it < (ITERS > 0 ? ITERS : 1); ++it) {
      const int c0 = (it * kCeThreads + (int)threadIdx.x) * 8;
      if (c0 < V) {
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const float v = cvt<float>(cache[it].v[e]);
          sh += v;
          m = fmaxf(m, v);
        }
      }
    }
    const float mx = block_max(m);
    // pass 2: first index of the max, and e = exp(h - max) (kept in the cache in
    // place of h unless log-probabilities are requested)
    int first = INT32_MAX;
    float z = 0.f;
    const float l2e = 1.4426950408889634f, mxl = mx * l2e;
#pragma unroll
    for (int it = 0; it < (ITERS > 0 ? ITERS : 1); ++it) {
      const int c0 = (it * kCeThreads + (int)threadIdx.x) * 8;
      if (c0 < V) {
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const float v = cvt<float>(cache[it].v[e]);
          if (v == mx && c0 + e < first) first = c0 + e;
          const float ex = exp2f(fmaf(v, l2e, -mxl));
          z += ex;
          if (!logq_out) cache[it].v[e] = cvt<T>(ex * ExCache<T>::kScale);
        }
      }
    }
    first = block_min(first);
    z = block_sum(z);
    const double shd = block_sum((double)sh);
    const double lse = (double)mx + log((double)z);
    if (threadIdx.x == 0) {
      double loss = 0.0;
      if (valid && tgt_ok) {
        const double ht = (double)cvt<float>(h[tgt]);
        loss = -(1.0 - alpha) * (ht - lse) - (alpha / (double)V) * (shd - (double)V * lse);
      }
      row_stats[2 * r] = loss;
      row_stats[2 * r + 1] = (valid && tgt_ok && first == tgt) ? 1.0 : 0.0;
    }
    const float rz = 1.f / z;
    const float lz = (float)log((double)z);
    const float a_v = (float)(alpha / (double)V);
    const float one_m_a = (float)(1.0 - alpha);
    const float gs = (float)grad_scale;
    __syncthreads();  // all reads of h[tgt] are done before the in-place overwrite
#pragma unroll
    for (int it = 0; it < (ITERS > 0 ? ITERS : 1); ++it) {
      const int c0 = (it * kCeThreads + (int)threadIdx.x) * 8;
      if (c0 < V) {
        if (logq_out) {
          Pack8<T> q;
#pragma unroll
          for (int e = 0; e < 8; ++e) q.v[e] = cvt<T>((cvt<float>(cache[it].v[e]) - mx) - lz);
          st8(logq_out + r * V + c0, q);
        }
        if (dlogits) {
          Pack8<T> q;
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const float ex = logq_out ? exp2f(fmaf(cvt<float>(cache[it].v[e]), l2e, -mxl))
                                      : cvt<float>(cache[it].v[e]) * ExCache<T>::kInv;
            float g = ex * rz - a_v;
            if (c0 + e == tgt) g -= one_m_a;
            q.v[e] = cvt<T>(valid ? g * gs : 0.f);
          }
          st8(dlogits + r * V + c0, q);
        }
      }
    }
    return;
  }
  // two-pass fallback for rows that do not fit in registers (second read hits L2)
  for (int64_t c = threadIdx.x; c < V; c += kCeThreads) {
    const float v = cvt<float>(h[c]);
    sh += v;
    mi_merge(mi, MaxIdx{v, c});
  }
  mi = block_argmax(mi);
  const float mx = mi.v;
  float z = 0.f;
  for (int64_t c = threadIdx.x; c < V; c += kCeThreads) z += __expf(cvt<float>(h[c]) - mx);
  z = block_sum(z);
  const double shd = block_sum((double)sh);
  const double lse = (double)mx + log((double)z);
  if (threadIdx.x == 0) {
    double loss = 0.0;
    if (valid && tgt_ok) {
      const double ht = (double)cvt<float>(h[tgt]);
      loss = -(1.0 - alpha) * (ht - lse) - (alpha / (double)V) * (shd - (double)V * lse);
    }
    row_stats[2 * r] = loss;
    row_stats[2 * r + 1] = (valid && tgt_ok && mi.i == tgt) ? 1.0 : 0.0;
  }
  const float rz = 1.f / z;
  const float lz = (float)log((double)z);
  const float a_v = (float)(alpha / (double)V);
  const float one_m_a = (float)(1.0 - alpha);
  const float gs = (float)grad_scale;
  __syncthreads();  // all reads of h[tgt] are done before the in-place overwrite
  for (int64_t c = threadIdx.x; c < V; c += kCeThreads) {
    const float sv = cvt<float>(h[c]) - mx;
    if (logq_out) logq_out[r * V + c] = cvt<T>(sv - lz);
    if (dlogits) {
      float g = __expf(sv) * rz - a_v;
      if (c == tgt) g -= one_m_a;
      dlogits[r * V + c] = cvt<T>(valid ? g * gs : 0.f);
    }
  }
}

// ---------------------------------------------------------------------------
// Persistent TMA-pipelined variant (16-bit logits, V % 8 == 0, 2 rows fit in smem).
// One 1024-thread CTA per SM walks rows blockIdx.x, +gridDim.x, ...; row k+1 is
// bulk-copied (cp.async.bulk, mbarrier completion) into the other smem buffer
// while row k is reduced, so the HBM read of the next row overlaps the ALU work
// and the (fire-and-forget) gradient stores of the current one.  Per row:
//   pass 1  sum(h) and max(h)                      (smem reads)
//   pass 2  e = exp(h - max), Z = sum(e), first argmax; e (scaled) overwrites h
//   pass 3  dlogits = (e/Z - a/V - (1-a)[i==k]) * grad_scale  -> HBM, in place
// The CTA accumulates its rows' (loss, correct, count) in row order and leaves
// one triple per CTA for the fixed-order final reduce (deterministic).
// ---------------------------------------------------------------------------
constexpr int kCeTmaThreads = 1024;
constexpr int kCeTmaWarps = kCeTmaThreads / 32;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes,
                                          uint64_t* bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// packed helpers: two 16-bit values <-> float2, fp32x2 FMA/ADD (sm_100 FFMA2/FADD2)
template <typename T> struct Pair;
template <> struct Pair<__half> {
  using P2 = __half2;
  static __device__ __forceinline__ float2 f(P2 v) { return __half22float2(v); }
  static __device__ __forceinline__ P2 pack(float2 v) { return __float22half2_rn(v); }
  static __device__ __forceinline__ P2 max(P2 a, P2 b) { return __hmax2(a, b); }
  static __device__ __forceinline__ float hi_lo_max(P2 v) { return fmaxf(__low2float(v), __high2float(v)); }
  static constexpr float kLog2Scale = 15.f;   // exps cached as e * 2^15 (see ExCache)
};
template <> struct Pair<__nv_bfloat16> {
  using P2 = __nv_bfloat162;
  static __device__ __forceinline__ float2 f(P2 v) { return __bfloat1622float2(v); }
  static __device__ __forceinline__ P2 pack(float2 v) { return __float22bfloat162_rn(v); }
  static __device__ __forceinline__ P2 max(P2 a, P2 b) { return __hmax2(a, b); }
  static __device__ __forceinline__ float hi_lo_max(P2 v) { return fmaxf(__low2float(v), __high2float(v)); }
  static constexpr float kLog2Scale = 0.f;
};

__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  float2 d;
  asm("{.reg .b64 ra, rb, rc, rd;\n mov.b64 ra, {%2, %3};\n mov.b64 rb, {%4, %5};\n"
      " mov.b64 rc, {%6, %7};\n fma.rn.f32x2 rd, ra, rb, rc;\n mov.b64 {%0, %1}, rd;}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return d;
}
__device__ __forceinline__ float2 fadd2(float2 a, float2 b) {
  float2 d;
  asm("{.reg .b64 ra, rb, rd;\n mov.b64 ra, {%2, %3};\n mov.b64 rb, {%4, %5};\n"
      " add.rn.f32x2 rd, ra, rb;\n mov.b64 {%0, %1}, rd;}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return d;
}
__device__ __forceinline__ float ex2_ftz(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// CH = 16-byte chunks per thread per row (compile-time, fully unrolled)
template <typename T, int CH>
__global__ void __launch_bounds__(kCeTmaThreads, 1) criterion_tma_kernel(
    const T* __restrict__ logits, const int64_t* __restrict__ targets, T* dlogits,
    double* __restrict__ cta_stats, int* __restrict__ bad_target, int64_t rows, int V,
    double alpha, int64_t pad_id, int has_pad, double grad_scale) {
  using PT = Pair<T>;
  using P2 = typename PT::P2;
  struct alignas(16) Chunk { P2 h[4]; };
  extern __shared__ __align__(128) uint8_t ce_smem[];
  __shared__ uint64_t bar[2];
  __shared__ float s_max[kCeTmaWarps], s_z[kCeTmaWarps];
  __shared__ double s_sh[kCeTmaWarps];
  __shared__ int s_first[kCeTmaWarps];
  __shared__ float s_ht;
  const uint32_t row_bytes = (uint32_t)V * sizeof(T);
  const uint32_t buf_stride = (row_bytes + 127u) & ~127u;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int nchunk = V / 8;
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if ((int64_t)blockIdx.x < rows)
      bulk_load(ce_smem, logits + (int64_t)blockIdx.x * V, row_bytes, &bar[0]);
  }
  __syncthreads();
  const float l2e = 1.4426950408889634f;
  const float a_v = (float)(alpha / (double)V);
  const float one_m_a = (float)(1.0 - alpha);
  double acc_loss = 0.0, acc_corr = 0.0, acc_cnt = 0.0;  // thread 0 only
  int k = 0;
  for (int64_t r = blockIdx.x; r < rows; r += gridDim.x, ++k) {
    const int b = k & 1;
    const int64_t rn = r + gridDim.x;
    const int64_t tgt = targets[r];
    mbar_wait(&bar[b], (uint32_t)((k >> 1) & 1));
    if (tid == 0 && rn < rows) {
      // the other buffer was last read (and written by the generic proxy) in
      // the previous iteration, which every thread has left (barrier below)
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      bulk_load(ce_smem + (b ^ 1) * buf_stride, logits + rn * V, row_bytes, &bar[b ^ 1]);
    }
    Chunk* row = reinterpret_cast<Chunk*>(ce_smem + b * buf_stride);
    const bool valid = !(has_pad && tgt == pad_id);
    const bool tgt_ok = tgt >= 0 && tgt < V;
    if (valid && !tgt_ok && tid == 0 && bad_target) *bad_target = 1;
    const int tchunk = (valid && tgt_ok) ? (int)(tgt >> 3) : -1;
    if (tchunk >= 0 && tid == tchunk % kCeTmaThreads)
      s_ht = cvt<float>(reinterpret_cast<const T*>(row)[tgt]);
    // pass 1: packed max, fp32x2 sum
    P2 m2 = PT::pack(make_float2(-INFINITY, -INFINITY));
    float2 s2 = make_float2(0.f, 0.f);
#pragma unroll
    for (int j = 0; j < CH; ++j) {
      const int c = tid + j * kCeTmaThreads;
      if (c < nchunk) {
        const Chunk q = row[c];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          m2 = PT::max(m2, q.h[e]);
          s2 = fadd2(s2, PT::f(q.h[e]));
        }
      }
    }
    const float mloc = PT::hi_lo_max(m2);
    float m = mloc;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (lane == 0) s_max[wid] = m;
    __syncthreads();
    float mx = s_max[lane];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    // pass 2: e = 2^(log2e*(h - max) + log2 scale), Z, e overwrites h.  The
    // first argmax is searched (on the raw values) only by threads whose own
    // maximum is the row maximum, in chunk order.
    const float off = PT::kLog2Scale - mx * l2e;
    const float2 l2e2 = make_float2(l2e, l2e), off2 = make_float2(off, off);
    const bool mine = (mloc == mx);
    float2 z2 = make_float2(0.f, 0.f);
    int first = INT32_MAX;
#pragma unroll
    for (int j = 0; j < CH; ++j) {
      const int c = tid + j * kCeTmaThreads;
      if (c < nchunk) {
        Chunk q = row[c];
        if (mine && first == INT32_MAX) {
          const T* hv = reinterpret_cast<const T*>(&q);
#pragma unroll
          for (int e = 0; e < 8; ++e)
            if (first == INT32_MAX && cvt<float>(hv[e]) == mx) first = c * 8 + e;
        }
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 a = ffma2(PT::f(q.h[e]), l2e2, off2);
          const float2 ex = make_float2(ex2_ftz(a.x), ex2_ftz(a.y));
          z2 = fadd2(z2, ex);
          q.h[e] = PT::pack(ex);
        }
        row[c] = q;
      }
    }
    float z = z2.x + z2.y;
    double shd = (double)s2.x + (double)s2.y;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      z += __shfl_xor_sync(0xffffffffu, z, o);
      shd += __shfl_xor_sync(0xffffffffu, shd, o);
      first = min(first, __shfl_xor_sync(0xffffffffu, first, o));
    }
    if (lane == 0) { s_z[wid] = z; s_sh[wid] = shd; s_first[wid] = first; }
    __syncthreads();
    float zt = s_z[lane];
    int ft = s_first[lane];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      zt += __shfl_xor_sync(0xffffffffu, zt, o);
      ft = min(ft, __shfl_xor_sync(0xffffffffu, ft, o));
    }
    if (tid == 0) {
      double sht = 0.0;
      for (int q = 0; q < kCeTmaWarps; ++q) sht += s_sh[q];
      // zt = 2^scale * Z
      const double lse = (double)mx + log((double)zt) - (double)PT::kLog2Scale * 0.6931471805599453;
      if (valid && tgt_ok) {
        acc_loss += -(1.0 - alpha) * ((double)s_ht - lse) -
                    (alpha / (double)V) * (sht - (double)V * lse);
        acc_corr += (ft == tgt) ? 1.0 : 0.0;
      }
      acc_cnt += valid ? 1.0 : 0.0;
    }
    // pass 3: gradient (e * gs / Z - gs * a/V) streamed to HBM over the consumed row
    if (dlogits) {
      const float gs = valid ? (float)grad_scale : 0.f;
      const float cz = gs / zt;                 // zt carries the cache scale
      const float2 cz2 = make_float2(cz, cz), of2 = make_float2(-a_v * gs, -a_v * gs);
      T* drow = dlogits + r * (int64_t)V;
#pragma unroll
      for (int j = 0; j < CH; ++j) {
        const int c = tid + j * kCeTmaThreads;
        if (c < nchunk) {
          Chunk q = row[c];
#pragma unroll
          for (int e = 0; e < 4; ++e) q.h[e] = PT::pack(ffma2(PT::f(q.h[e]), cz2, of2));
          *reinterpret_cast<uint4*>(drow + c * 8) = *reinterpret_cast<const uint4*>(&q);
        }
      }
      if (tchunk >= 0 && tid == tchunk % kCeTmaThreads) {
        // same thread, later store: the target element gets its -(1-a) term
        const float et = cvt<float>(reinterpret_cast<const T*>(row)[tgt]);
        drow[tgt] = cvt<T>(fmaf(et, cz, -a_v * gs) - one_m_a * gs);
      }
    }
    __syncthreads();  // buffer b fully consumed before it is refilled
  }
  if (tid == 0) {
    cta_stats[3 * blockIdx.x + 0] = acc_loss;
    cta_stats[3 * blockIdx.x + 1] = acc_corr;
    cta_stats[3 * blockIdx.x + 2] = acc_cnt;
  }
}

// fixed-order sum of per-CTA (loss, correct, count) triples: one warp, lane l
// sums triples l, l+32, ... then a fixed xor-tree (same order every run)
__global__ void criterion_reduce_cta(const double* __restrict__ cta_stats, int n,
                                     double* __restrict__ out3) {
  const int lane = threadIdx.x;
  double a = 0, b = 0, c = 0;
  for (int i = lane; i < n; i += 32) {
    a += cta_stats[3 * i];
    b += cta_stats[3 * i + 1];
    c += cta_stats[3 * i + 2];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
    c += __shfl_xor_sync(0xffffffffu, c, o);
  }
  if (lane == 0) {
    out3[0] = a;
    out3[1] = c;
    out3[2] = b;
  }
}

// fixed-order reduce of per-row (loss, correct) + valid count
__global__ void criterion_reduce(const double* __restrict__ row_stats,
                                 const int64_t* __restrict__ targets, int64_t rows,
                                 int64_t pad_id, int has_pad, double* __restrict__ out3) {
  __shared__ double s0[256], s1[256], s2[256];
  double a = 0, b = 0, c = 0;
  for (int64_t r = threadIdx.x; r < rows; r += blockDim.x) {
    a += row_stats[2 * r];
    b += row_stats[2 * r + 1];
    c += (has_pad && targets[r] == pad_id) ? 0.0 : 1.0;
  }
  s0[threadIdx.x] = a; s1[threadIdx.x] = b; s2[threadIdx.x] = c;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) {
      s0[threadIdx.x] += s0[threadIdx.x + o];
      s1[threadIdx.x] += s1[threadIdx.x + o];
      s2[threadIdx.x] += s2[threadIdx.x + o];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    out3[0] = s0[0];
    out3[1] = s2[0];
    out3[2] = s1[0];
  }
}

// reference-API loss from precomputed log-probs (warp per row, f64 sums)
template <typename T>
__global__ void ls_ce_fwd_kernel(const T* __restrict__ logq, const int64_t* __restrict__ targets,
                                 double* __restrict__ row_stats, int* bad_target, int64_t rows,
                                 int64_t V, double alpha, int64_t pad_id, int has_pad) {
  const int lane = threadIdx.x & 31;
  for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < rows;
       r += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t t = targets[r];
    const bool valid = !(has_pad && t == pad_id);
    double s = 0.0;
    for (int64_t c = lane; c < V; c += 32) s += cvt<double>(logq[r * V + c]);
    s = warp_sum(s);
    if (lane == 0) {
      double loss = 0.0;
      if (valid) {
        if (t < 0 || t >= V) {
          if (bad_target) *bad_target = 1;
        } else {
          loss = -(1.0 - alpha) * cvt<double>(logq[r * V + t]) - (alpha / (double)V) * s;
        }
      }
      row_stats[2 * r] = loss;
      row_stats[2 * r + 1] = 0.0;
    }
  }
}

// reference-API backward from probs: op order of F/gradients.py:69-73
template <typename Tin, typename Tout>
__global__ void ls_ce_bwd_kernel(const Tin* __restrict__ probs, const int64_t* __restrict__ targets,
                                 Tout* __restrict__ dh, int* bad_target, int64_t rows, int64_t V,
                                 double alpha, int64_t pad_id, int has_pad, double grad_scale) {
  using C = typename CompOf<Tin>::type;
  const C a_v = (C)(alpha / (double)V), one_m_a = (C)(1.0 - alpha), gs = (C)grad_scale;
  for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
    const int64_t t = targets[r];
    const bool valid = !(has_pad && t == pad_id);
    if (valid && (t < 0 || t >= V) && bad_target && threadIdx.x == 0) *bad_target = 1;
    for (int64_t c = threadIdx.x; c < V; c += blockDim.x) {
      C g = add_rn(cvt<C>(probs[r * V + c]), -a_v);
      if (c == t) g = add_rn(g, -one_m_a);
      if (grad_scale != 1.0) g = mul_rn(g, gs);
      dh[r * V + c] = cvt<Tout>(valid ? g : (C)0);
    }
  }
}

}  // namespace ls2

using namespace ls2;

extern "C" {

int ls2_criterion_fused(const void* logits, const int64_t* targets, void* dlogits, void* logq_out,
                        double* row_stats, double* out3, int* bad_target, int64_t rows, int64_t v,
                        double alpha, int64_t pad_id, int has_pad, double grad_scale,
                        int t_logits, void* stream) {
  if (rows <= 0) return cudaMemsetAsync(out3, 0, 3 * sizeof(double), as_stream(stream)) == cudaSuccess ? LS2_OK : fail(LS2_ERR_CUDA, "memset");
  if (v < 2) return fail(LS2_ERR_SHAPE, "criterion needs >= 2 classes");
  cudaStream_t st = as_stream(stream);
  const bool v8 = v % 8 == 0 && aligned16(logits) && (!dlogits || aligned16(dlogits)) &&
                  (!logq_out || aligned16(logq_out));
  // persistent TMA path: 16-bit rows, two row buffers in shared memory; the
  // per-CTA stats triples live in row_stats (needs 3 * grid <= 2 * rows)
  const int64_t buf = ((v * 2 + 127) / 128) * 128;
  if (v8 && !logq_out && rows >= 256 && 2 * buf <= 200 * 1024 && v < (1 << 24) &&
      (t_logits == LS2_F16 || t_logits == LS2_BF16)) {
    const int grid = (int)std::min<int64_t>(rows, kNumSMs);
    const int smem = (int)(2 * buf);
    const int need = (int)ceil_div(v / 8, (int64_t)kCeTmaThreads);
    auto go = [&](auto tag) -> int {
      using T = typename decltype(tag)::type;
      auto launch = [&](auto ch) -> int {
        constexpr int CH = decltype(ch)::value;
        static bool attr_set[64] = {};
        int dev = 0;
        cudaGetDevice(&dev);
        if (!attr_set[dev & 63]) {
          cudaFuncSetAttribute(criterion_tma_kernel<T, CH>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
          attr_set[dev & 63] = true;
        }
        criterion_tma_kernel<T, CH><<<grid, kCeTmaThreads, smem, st>>>(
            (const T*)logits, targets, (T*)dlogits, row_stats, bad_target, rows, (int)v, alpha,
            pad_id, has_pad, grad_scale);
        return check_launch("criterion_fused");
      };
      int rc = need <= 1 ? launch(std::integral_constant<int, 1>{})
             : need <= 2 ? launch(std::integral_constant<int, 2>{})
             : need <= 4 ? launch(std::integral_constant<int, 4>{})
                         : launch(std::integral_constant<int, 7>{});
      if (rc) return rc;
      criterion_reduce_cta<<<1, 32, 0, st>>>(row_stats, grid, out3);
      return check_launch("criterion_reduce");
    };
    if (t_logits == LS2_F16) return go(std::type_identity<__half>{});
    return go(std::type_identity<__nv_bfloat16>{});
  }
  int rc = [&]() -> int {
    auto go = [&](auto tag, auto iters) {
      using T = typename decltype(tag)::type;
      constexpr int I = decltype(iters)::value;
      criterion_kernel<T, I><<<(unsigned)rows, kCeThreads, 0, st>>>(
          (const T*)logits, targets, (T*)dlogits, (T*)logq_out, row_stats, bad_target, rows, v,
          alpha, pad_id, has_pad, grad_scale);
      return check_launch("criterion_fused");
    };
    const int64_t per = ceil_div(v, (int64_t)kCeThreads * 8);
    auto pick = [&](auto tag) {
      if (!v8 || per > 8) return go(tag, std::integral_constant<int, 0>{});
      if (per <= 1) return go(tag, std::integral_constant<int, 1>{});
      if (per <= 2) return go(tag, std::integral_constant<int, 2>{});
      if (per <= 4) return go(tag, std::integral_constant<int, 4>{});
      return go(tag, std::integral_constant<int, 8>{});
    };
    if (t_logits == LS2_F16) return pick(std::type_identity<__half>{});
    if (t_logits == LS2_BF16) return pick(std::type_identity<__nv_bfloat16>{});
    if (t_logits == LS2_F32) return pick(std::type_identity<float>{});
    return fail(LS2_ERR_DTYPE, "criterion_fused: logits must be f16/bf16/f32");
  }();
  if (rc) return rc;
  criterion_reduce<<<1, 256, 0, st>>>(row_stats, targets, rows, pad_id, has_pad, out3);
  return check_launch("criterion_reduce");
}

int ls2_ls_ce_fwd(const void* logq, const int64_t* targets, double* row_stats, double* out3,
                  int* bad_target, int64_t rows, int64_t v, double alpha, int64_t pad_id,
                  int has_pad, int tin, void* stream) {
  cudaStream_t st = as_stream(stream);
  if (rows <= 0) return cudaMemsetAsync(out3, 0, 3 * sizeof(double), st) == cudaSuccess ? LS2_OK : fail(LS2_ERR_CUDA, "memset");
  int rc = LS2_DISPATCH_ONE(tin, "ls_ce_fwd", [&] {
    ls_ce_fwd_kernel<Tx><<<grid_for(rows * 32), 256, 0, st>>>((const Tx*)logq, targets, row_stats,
                                                              bad_target, rows, v, alpha, pad_id,
                                                              has_pad);
    return check_launch("ls_ce_fwd");
  });
  if (rc) return rc;
  criterion_reduce<<<1, 256, 0, st>>>(row_stats, targets, rows, pad_id, has_pad, out3);
  return check_launch("criterion_reduce");
}

int ls2_ls_ce_bwd(const void* probs, const int64_t* targets, void* dh, int* bad_target,
                  int64_t rows, int64_t v, double alpha, int64_t pad_id, int has_pad,
                  double grad_scale, int tin, int tout, void* stream) {
  if (rows <= 0) return LS2_OK;
  cudaStream_t st = as_stream(stream);
  return LS2_DISPATCH_IO(tin, tout, "ls_ce_bwd", [&] {
    const int grid = (int)std::min<int64_t>(rows, kNumSMs * 16);
    ls_ce_bwd_kernel<Tin, Tout><<<grid, 256, 0, st>>>((const Tin*)probs, targets, (Tout*)dh,
                                                       bad_target, rows, v, alpha, pad_id, has_pad,
                                                       grad_scale);
    return check_launch("ls_ce_bwd");
  });
}

}  // extern "C"
