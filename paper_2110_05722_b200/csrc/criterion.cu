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
#include <cooperative_groups.h>

#include <cfloat>

#include "common.cuh"

namespace cg = cooperative_groups;

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
// ---------------------------------------------------------------------------
// Persistent row kernel (16-bit logits, V % 8 == 0).  A cluster of C CTAs owns
// a row (C = 1 while two rows fit in one SM's shared memory; C = 2..16 for
// V up to 512k, SURVEY §7 hard part 7): CTA q holds columns [q*S, q*S+len_q).
// Each CTA walks rows cid, cid+ncl, ...; its slice of row k+2 is bulk-copied
// (cp.async.bulk, mbarrier completion) into the buffer row k has just left,
// so two row loads are in flight while row k is reduced.  Every logit is read
// from HBM once and its gradient written once.  Per row, per thread:
//   load     its CH 16-byte chunks from shared memory into registers (the only
//            shared-memory pass; the buffer is released right after)
//   pass 1   packed max, fp32x2 sum of h
//   pass 2   e = 2^(log2e (h - m_q) + log2 scale) in registers, Z_q, first argmax
//   pass 3   dlogits = (e s_q / Z - a/V - (1-a)[i==k]) * grad_scale -> HBM, in place
// where m_q is the slice max.  With C > 1 the CTAs push (m_q, Z_q, sum h,
// first, h[target]) into every cluster CTA's shared memory (DSMEM) and after
// ONE cluster barrier per row merge them online-softmax style,
//   M = max m_q,  Z = sum_q Z_q 2^(log2e (m_q - M)),  s_q = 2^(log2e (m_q - M)),
// with the same fixed shuffle tree in every CTA: identical M and Z everywhere,
// deterministic results.  Rank 0 of each cluster accumulates the rows'
// (loss, correct, count) in row order for the fixed-order final reduce.
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


// G row groups per CTA (1024/G threads each, named barriers): with G = 2 the
// two halves of the SM work on different rows, so one half's exp pass (MUFU)
// overlaps the other's gradient stores instead of every warp hitting the same
// pipe at once.  G = 1 double-buffers (row k+2 loads while k is reduced); G = 2
// gives each group one buffer, refilled with the group's next row as soon as
// the current one is in registers.  Clusters (C > 1) use G = 1.
template <int G>
__device__ __forceinline__ void group_sync(int g) {
  if constexpr (G == 1) {
    __syncthreads();
  } else {
    asm volatile("bar.sync %0, %1;" ::"r"(1 + g), "r"(kCeTmaThreads / G) : "memory");
  }
}

template <typename T, int CH, int G>
__global__ void __launch_bounds__(kCeTmaThreads, 1) criterion_rows_kernel(
    const T* __restrict__ logits, const int64_t* __restrict__ targets, T* dlogits,
    double* __restrict__ cl_stats, int* __restrict__ bad_target, int64_t rows, int V, int S,
    double alpha, int64_t pad_id, int has_pad, double grad_scale, int ldr) {
  using PT = Pair<T>;
  using P2 = typename PT::P2;
  struct alignas(16) Chunk { P2 h[4]; };
  constexpr int kMaxC = 16;
  constexpr int NT = kCeTmaThreads / G;         // threads per row group
  constexpr int WG = NT / 32;                   // warps per row group
  constexpr int NB = G == 1 ? 2 : 1;            // row buffers per group
  extern __shared__ __align__(128) uint8_t ce_smem[];
  __shared__ uint64_t bar[2];
  __shared__ float s_max[G][WG], s_z[G][WG];
  __shared__ double s_sh[G][WG];
  __shared__ int s_first[G][WG];
  __shared__ float s_ht[G];
  __shared__ double s_acc[G][3];     // per group: (loss, correct, count) in row order
  // cluster exchange slots [group][row parity][source rank], pushed by the
  // source CTA's group; xbar[group][parity] counts the C pushes (DSMEM mbarrier
  // arrivals with cluster-scope release), so each row group syncs with the
  // same group of the other CTAs only, and the two groups stay out of phase
  __shared__ float x_max[G][2][kMaxC], x_z[G][2][kMaxC], x_ht[G][2][kMaxC];
  __shared__ double x_sh[G][2][kMaxC];
  __shared__ int x_first[G][2][kMaxC];
  __shared__ uint64_t xbar[G][2];
  cg::cluster_group cl = cg::this_cluster();
  const int C = (int)cl.num_blocks();
  const int q = C > 1 ? (int)cl.block_rank() : 0;
  const int64_t cid = blockIdx.x / C, ncl = gridDim.x / C;
  const int col0 = q * S;
  const int len = C == 1 ? S : min(S, V - col0);   // C == 1: S = row pitch (>= V)
  const uint32_t slice_bytes = (uint32_t)len * sizeof(T);
  const uint32_t buf_stride = ((uint32_t)S * sizeof(T) + 127u) & ~127u;
  const int tid = threadIdx.x, lane = tid & 31;
  const int g = tid / NT, gt = tid % NT, gw = gt >> 5;
  const int nchunk = len / 8;
  // group-local row k of group g: cid + (k*G + g) * ncl
  const int64_t rstride = (int64_t)G * ncl;
  const int64_t r0 = cid + (int64_t)g * ncl;
  if (gt == 0) {
    for (int i = 0; i < NB; ++i) mbar_init(&bar[g * NB + i], 1);
    if (C > 1) {
      mbar_init(&xbar[g][0], C);
      mbar_init(&xbar[g][1], C);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int i = 0; i < NB; ++i)
      if (r0 + i * rstride < rows)
        bulk_load(ce_smem + (g * NB + i) * buf_stride, logits + (r0 + i * rstride) * ldr + col0,
                  slice_bytes, &bar[g * NB + i]);
    s_acc[g][0] = s_acc[g][1] = s_acc[g][2] = 0.0;
  }
  if (C > 1) cl.sync();   // every CTA's barriers initialised before any remote arrive
  else __syncthreads();
  const float l2e = 1.4426950408889634f;
  const float a_v = (float)(alpha / (double)V);
  const float one_m_a = (float)(1.0 - alpha);
  int64_t tgt_next = r0 < rows ? targets[r0] : 0;
  int k = 0;
  for (int64_t r = r0; r < rows; r += rstride, ++k) {
    const int bi = g * NB + (k % NB);
    const int xb = k & 1;                                  // cluster slot parity
    const int64_t tgt = tgt_next;
    if (r + rstride < rows) tgt_next = targets[r + rstride];
    const bool valid = !(has_pad && tgt == pad_id);
    const bool tgt_ok = tgt >= 0 && tgt < V;
    if (valid && !tgt_ok && gt == 0 && q == 0 && bad_target) *bad_target = 1;
    const int64_t lt = tgt - col0;                         // target's local column
    const bool own_t = valid && tgt_ok && lt >= 0 && lt < len;
    mbar_wait(&bar[bi], (uint32_t)((k / NB) & 1));
    const Chunk* row = reinterpret_cast<const Chunk*>(ce_smem + bi * buf_stride);
    // all CH chunks of this thread in range: straight-line passes (warp-uniform
    // for every warp but the one straddling the slice end)
    const bool full = gt + (CH - 1) * NT < nchunk;
    Chunk hq[CH];
    if (full) {
#pragma unroll
      for (int j = 0; j < CH; ++j) hq[j] = row[gt + j * NT];
    } else {
#pragma unroll
      for (int j = 0; j < CH; ++j) {
        const int c = gt + j * NT;
        if (c < nchunk) hq[j] = row[c];
      }
    }
    // a row pitch past V (V % 8 != 0, C == 1): the last chunk's columns >= V
    // read as -inf (no max, no exp); they are left out of sum(h) below
    const int tailc = (ldr != V) ? V / 8 : -1, tailn = V & 7;
    if (tailc >= 0) {
#pragma unroll
      for (int j = 0; j < CH; ++j)
        if (gt + j * NT == tailc) {
          T* hv = reinterpret_cast<T*>(&hq[j]);
#pragma unroll
          for (int e = 0; e < 8; ++e)
            if (e >= tailn) hv[e] = cvt<T>(-INFINITY);
        }
    }
    if (gt == 0) s_ht[g] = own_t ? cvt<float>(reinterpret_cast<const T*>(row)[lt]) : 0.f;
    // pass 1 (registers): packed max, fp32x2 sum
    P2 m2 = PT::pack(make_float2(-INFINITY, -INFINITY));
    float2 s2 = make_float2(0.f, 0.f);
    auto pass1 = [&](auto fc) {
      constexpr bool F = decltype(fc)::value;
#pragma unroll
      for (int j = 0; j < CH; ++j) {
        if (F || gt + j * NT < nchunk) {
          if (gt + j * NT == tailc) {      // masked tail: max over all, sum of the valid
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              m2 = PT::max(m2, hq[j].h[e]);
              const float2 f = PT::f(hq[j].h[e]);
              s2.x += (2 * e < tailn) ? f.x : 0.f;
              s2.y += (2 * e + 1 < tailn) ? f.y : 0.f;
            }
          } else {
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              m2 = PT::max(m2, hq[j].h[e]);
              s2 = fadd2(s2, PT::f(hq[j].h[e]));
            }
          }
        }
      }
    };
    if (full) pass1(std::true_type{}); else pass1(std::false_type{});
    const float mloc = PT::hi_lo_max(m2);
    float m = mloc;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (lane == 0) s_max[g][gw] = m;
    group_sync<G>(g);              // the row buffer is consumed: refill it
    if (gt == 0 && r + NB * rstride < rows) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      bulk_load(ce_smem + bi * buf_stride, logits + (r + NB * rstride) * ldr + col0, slice_bytes,
                &bar[bi]);
    }
    float mq = lane < WG ? s_max[g][lane] : -INFINITY;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mq = fmaxf(mq, __shfl_xor_sync(0xffffffffu, mq, o));
    // pass 2 (registers): exps relative to the slice max, Z_q, first argmax
    const float off = PT::kLog2Scale - mq * l2e;
    const float2 l2e2 = make_float2(l2e, l2e), off2 = make_float2(off, off);
    int first = INT32_MAX;
    if (mloc == mq) {
#pragma unroll
      for (int j = 0; j < CH; ++j) {
        const int c = gt + j * NT;
        if (c < nchunk && first == INT32_MAX) {
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float2 hv = PT::f(hq[j].h[e]);
            if (first == INT32_MAX && hv.x == mq) first = col0 + c * 8 + 2 * e;
            if (first == INT32_MAX && hv.y == mq) first = col0 + c * 8 + 2 * e + 1;
          }
        }
      }
    }
    float2 z2 = make_float2(0.f, 0.f);
    auto pass2 = [&](auto fc) {
      constexpr bool F = decltype(fc)::value;
#pragma unroll
      for (int j = 0; j < CH; ++j) {
        if (F || gt + j * NT < nchunk) {
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float2 a = ffma2(PT::f(hq[j].h[e]), l2e2, off2);
            const float2 ex = make_float2(ex2_ftz(a.x), ex2_ftz(a.y));
            z2 = fadd2(z2, ex);
            hq[j].h[e] = PT::pack(ex);
          }
        }
      }
    };
    if (full) pass2(std::true_type{}); else pass2(std::false_type{});
    float z = z2.x + z2.y;
    double sh = (double)s2.x + (double)s2.y;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      z += __shfl_xor_sync(0xffffffffu, z, o);
      sh += __shfl_xor_sync(0xffffffffu, sh, o);
      first = min(first, __shfl_xor_sync(0xffffffffu, first, o));
    }
    if (lane == 0) { s_z[g][gw] = z; s_sh[g][gw] = sh; s_first[g][gw] = first; }
    group_sync<G>(g);
    float M, zt, scale;
    if (C == 1) {
      M = mq;
      zt = lane < WG ? s_z[g][lane] : 0.f;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) zt += __shfl_xor_sync(0xffffffffu, zt, o);
      scale = 1.f;
      if (gw == 0) {
        int ft = lane < WG ? s_first[g][lane] : INT32_MAX;
        double sht = lane < WG ? s_sh[g][lane] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          ft = min(ft, __shfl_xor_sync(0xffffffffu, ft, o));
          sht += __shfl_xor_sync(0xffffffffu, sht, o);
        }
        if (lane == 0) {
          const double lse = (double)M + log((double)zt) - (double)PT::kLog2Scale * 0.6931471805599453;
          if (valid && tgt_ok) {
            s_acc[g][0] += -(1.0 - alpha) * ((double)s_ht[g] - lse) -
                           (alpha / (double)V) * (sht - (double)V * lse);
            s_acc[g][1] += (ft == tgt) ? 1.0 : 0.0;
          }
          s_acc[g][2] += valid ? 1.0 : 0.0;
        }
      }
    } else {
      if (gw == 0) {
        float zz = lane < WG ? s_z[g][lane] : 0.f;
        double ss = lane < WG ? s_sh[g][lane] : 0.0;
        int ff = lane < WG ? s_first[g][lane] : INT32_MAX;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          zz += __shfl_xor_sync(0xffffffffu, zz, o);
          ss += __shfl_xor_sync(0xffffffffu, ss, o);
          ff = min(ff, __shfl_xor_sync(0xffffffffu, ff, o));
        }
        if (lane < C) {
          *cl.map_shared_rank(&x_max[g][xb][q], lane) = mq;
          *cl.map_shared_rank(&x_z[g][xb][q], lane) = zz;
          *cl.map_shared_rank(&x_sh[g][xb][q], lane) = ss;
          *cl.map_shared_rank(&x_first[g][xb][q], lane) = ff;
          *cl.map_shared_rank(&x_ht[g][xb][q], lane) = s_ht[g];
          // release the pushes to CTA `lane`: arrive on its barrier for this group/parity
          uint32_t rb;
          asm volatile("mapa.shared::cluster.u32 %0, %1, %2;"
                       : "=r"(rb) : "r"(smem_u32(&xbar[g][xb])), "r"((uint32_t)lane));
          asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(rb)
                       : "memory");
        }
      }
      {   // the one exchange per row: all C pushes of this group have landed here
        const uint32_t lb = smem_u32(&xbar[g][xb]);
        const uint32_t par = (uint32_t)((k >> 1) & 1);
        asm volatile(
            "{\n .reg .pred p;\n XW_%=:\n"
            " mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
            " @!p bra XW_%=;\n}" ::"r"(lb), "r"(par) : "memory");
      }
      const float mp = lane < C ? x_max[g][xb][lane] : -INFINITY;
      M = mp;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
      zt = lane < C ? x_z[g][xb][lane] * exp2f((mp - M) * l2e) : 0.f;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) zt += __shfl_xor_sync(0xffffffffu, zt, o);
      scale = exp2f((mq - M) * l2e);
      if (q == 0 && gw == 0) {
        int ft = (lane < C && mp == M) ? x_first[g][xb][lane] : INT32_MAX;
        double sht = lane < C ? x_sh[g][xb][lane] : 0.0;
        float ht = lane < C ? x_ht[g][xb][lane] : 0.f;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          ft = min(ft, __shfl_xor_sync(0xffffffffu, ft, o));
          sht += __shfl_xor_sync(0xffffffffu, sht, o);
          ht += __shfl_xor_sync(0xffffffffu, ht, o);
        }
        if (lane == 0) {
          const double lse = (double)M + log((double)zt) - (double)PT::kLog2Scale * 0.6931471805599453;
          if (valid && tgt_ok) {
            s_acc[g][0] += -(1.0 - alpha) * ((double)ht - lse) -
                           (alpha / (double)V) * (sht - (double)V * lse);
            s_acc[g][1] += (ft == tgt) ? 1.0 : 0.0;
          }
          s_acc[g][2] += valid ? 1.0 : 0.0;
        }
      }
    }
    // pass 3 (registers -> HBM): gradient, in place
    if (dlogits) {
      const float gs = valid ? (float)grad_scale : 0.f;
      const float cz = gs * scale / zt;                   // zt carries the cache scale
      const float2 cz2 = make_float2(cz, cz), of2 = make_float2(-a_v * gs, -a_v * gs);
      T* drow = dlogits + r * (int64_t)ldr + col0;
      auto pass3 = [&](auto fc) {
        constexpr bool F = decltype(fc)::value;
#pragma unroll
        for (int j = 0; j < CH; ++j) {
          const int c = gt + j * NT;
          if (F || c < nchunk) {
            Chunk o;
#pragma unroll
            for (int e = 0; e < 4; ++e) o.h[e] = PT::pack(ffma2(PT::f(hq[j].h[e]), cz2, of2));
            *reinterpret_cast<uint4*>(drow + c * 8) = *reinterpret_cast<const uint4*>(&o);
          }
        }
      };
      if (full) pass3(std::true_type{}); else pass3(std::false_type{});
      if (own_t && gt == (int)((lt >> 3) % NT)) {
        // same thread, later store: the target element gets its -(1-a) term
        // (its exp re-read from the register chunk with compile-time indices)
        const int jt = (int)((lt >> 3) / NT), et = (int)(lt & 7);
        float ev = 0.f;
#pragma unroll
        for (int j = 0; j < CH; ++j)
#pragma unroll
          for (int e = 0; e < 4; ++e)
            if (j == jt) {
              const float2 f = PT::f(hq[j].h[e]);
              if (2 * e == et) ev = f.x;
              if (2 * e + 1 == et) ev = f.y;
            }
        drow[lt] = cvt<T>(fmaf(ev, cz, -a_v * gs) - one_m_a * gs);
      }
    }
  }
  __syncthreads();
  if (tid == 0 && q == 0) {
    double l = 0.0, c1 = 0.0, n = 0.0;
    for (int i = 0; i < G; ++i) { l += s_acc[i][0]; c1 += s_acc[i][1]; n += s_acc[i][2]; }
    cl_stats[3 * cid + 0] = l;
    cl_stats[3 * cid + 1] = c1;
    cl_stats[3 * cid + 2] = n;
  }
  if (C > 1) cl.sync();  // no CTA exits while remote stores into it may be in flight
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

// Row ownership for the persistent kernel: C = 1 (S = V) while two rows fit in
// 200 KB of shared memory, else the smallest cluster whose slices of S <= 32768
// 16-bit elements (64 KB, double-buffered) cover the row.  0: no fit.
static int ce_cluster_size(int64_t v, int* slice) {
  if (2 * (((v * 2 + 127) / 128) * 128) <= 200 * 1024) {
    *slice = (int)v;
    return 1;
  }
  for (int c = 2; c <= 16; c *= 2) {
    const int64_t s = ceil_div(ceil_div(v, (int64_t)c), (int64_t)8) * 8;
    if (s <= 32768 && (c - 1) * s < v) {
      *slice = (int)s;
      return c;
    }
  }
  return 0;
}

template <typename T, int CH, int G>
static int launch_ce_rows_ch(const T* logits, const int64_t* targets, T* dlogits, double* row_stats,
                             double* out3, int* bad_target, int64_t rows, int64_t v, int C, int S,
                             double alpha, int64_t pad_id, int has_pad, double grad_scale,
                             int64_t ldr, cudaStream_t st) {
  auto kern = criterion_rows_kernel<T, CH, G>;
  const int smem = 2 * (int)(((int64_t)S * 2 + 127) / 128 * 128);   // G*NB == 2 buffers
  static std::mutex mu;
  static std::map<std::tuple<int, int, int>, int> max_clusters;   // (dev, C, smem)
  int dev = 0;
  cudaGetDevice(&dev);
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.blockDim = dim3(kCeTmaThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cfg.attrs = attr;
  cfg.numAttrs = C > 1 ? 1 : 0;
  int ncl;
  {
    std::lock_guard<std::mutex> lk(mu);
    auto key = std::make_tuple(dev, C, smem);
    auto it = max_clusters.find(key);
    if (it == max_clusters.end()) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      int n = kNumSMs;
      if (C > 1) {
        if (C > 8) cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        cfg.gridDim = dim3(C * kNumSMs);
        if (cudaOccupancyMaxActiveClusters(&n, (void*)kern, &cfg) != cudaSuccess || n <= 0) {
          cudaGetLastError();
          n = 0;
        }
      }
      it = max_clusters.emplace(key, n).first;
    }
    ncl = it->second;
  }
  // per-cluster stats triples live in row_stats (3 * clusters <= 2 * rows)
  ncl = (int)std::min<int64_t>(ncl, (2 * rows) / 3);
  if (ncl <= 0) return -1;
  cfg.gridDim = dim3(C * ncl);
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, logits, targets, dlogits, row_stats, bad_target,
                                     rows, (int)v, S, alpha, pad_id, has_pad, grad_scale, (int)ldr);
  if (e != cudaSuccess) return fail(LS2_ERR_CUDA, std::string("criterion_rows: ") + cudaGetErrorString(e));
  if (int rc = check_launch("criterion_rows")) return rc;
  criterion_reduce_cta<<<1, 32, 0, st>>>(row_stats, ncl, out3);
  return check_launch("criterion_reduce");
}

template <typename T>
static int launch_ce_rows(const T* logits, const int64_t* targets, T* dlogits, double* row_stats,
                          double* out3, int* bad_target, int64_t rows, int64_t v, int C, int S,
                          double alpha, int64_t pad_id, int has_pad, double grad_scale,
                          int64_t ldr, cudaStream_t st) {
#define LS2_CE_GO(CH_, G_)                                                                        \
  return launch_ce_rows_ch<T, CH_, G_>(logits, targets, dlogits, row_stats, out3, bad_target,     \
                                       rows, v, C, S, alpha, pad_id, has_pad, grad_scale, ldr, st)
  // two row groups per CTA while a row fits 8 chunks per thread of a 512-thread group
  static const bool groups2 = [] {
    const char* e = getenv("LS2_CE_GROUPS");
    return !(e && e[0] == '1');
  }();
  const int need2 = (int)ceil_div((int64_t)S / 8, (int64_t)(kCeTmaThreads / 2));
  if (groups2 && need2 <= 8) {
    if (need2 <= 1) LS2_CE_GO(1, 2);
    if (need2 <= 2) LS2_CE_GO(2, 2);
    if (need2 <= 4) LS2_CE_GO(4, 2);
    LS2_CE_GO(8, 2);
  }
  const int need = (int)ceil_div((int64_t)S / 8, (int64_t)kCeTmaThreads);
  if (need <= 1) LS2_CE_GO(1, 1);
  if (need <= 2) LS2_CE_GO(2, 1);
  if (need <= 4) LS2_CE_GO(4, 1);
  LS2_CE_GO(7, 1);
#undef LS2_CE_GO
}

}  // namespace ls2

using namespace ls2;

extern "C" {

int ls2_criterion_fused_ld(const void* logits, int64_t ld, const int64_t* targets, void* dlogits,
                           double* row_stats, double* out3, int* bad_target, int64_t rows,
                           int64_t v, double alpha, int64_t pad_id, int has_pad,
                           double grad_scale, int t_logits, void* stream) {
  if (ld == v) return ls2_criterion_fused(logits, targets, dlogits, nullptr, row_stats, out3,
                                          bad_target, rows, v, alpha, pad_id, has_pad, grad_scale,
                                          t_logits, stream);
  if (rows <= 0) return cudaMemsetAsync(out3, 0, 3 * sizeof(double), as_stream(stream)) == cudaSuccess ? LS2_OK : fail(LS2_ERR_CUDA, "memset");
  if (v < 2 || ld < v || ld % 8 != 0 || ld - v >= 8 || !aligned16(logits) ||
      (dlogits && !aligned16(dlogits)) || (t_logits != LS2_F16 && t_logits != LS2_BF16))
    return fail(LS2_ERR_SHAPE, "criterion_fused_ld: needs 16-bit logits, ld = V rounded up to 8");
  int slice = 0;
  if (ce_cluster_size(ld, &slice) != 1 || rows < 2)
    return fail(LS2_ERR_SHAPE, "criterion_fused_ld: row too long for the padded-pitch path");
  cudaStream_t st = as_stream(stream);
  int rc = t_logits == LS2_F16
               ? launch_ce_rows<__half>((const __half*)logits, targets, (__half*)dlogits, row_stats,
                                        out3, bad_target, rows, v, 1, (int)ld, alpha, pad_id,
                                        has_pad, grad_scale, ld, st)
               : launch_ce_rows<__nv_bfloat16>((const __nv_bfloat16*)logits, targets,
                                               (__nv_bfloat16*)dlogits, row_stats, out3,
                                               bad_target, rows, v, 1, (int)ld, alpha, pad_id,
                                               has_pad, grad_scale, ld, st);
  return rc < 0 ? fail(LS2_ERR_SHAPE, "criterion_fused_ld: no launch configuration") : rc;
}

int ls2_criterion_fused(const void* logits, const int64_t* targets, void* dlogits, void* logq_out,
                        double* row_stats, double* out3, int* bad_target, int64_t rows, int64_t v,
                        double alpha, int64_t pad_id, int has_pad, double grad_scale,
                        int t_logits, void* stream) {
  if (rows <= 0) return cudaMemsetAsync(out3, 0, 3 * sizeof(double), as_stream(stream)) == cudaSuccess ? LS2_OK : fail(LS2_ERR_CUDA, "memset");
  if (v < 2) return fail(LS2_ERR_SHAPE, "criterion needs >= 2 classes");
  cudaStream_t st = as_stream(stream);
  const bool v8 = v % 8 == 0 && aligned16(logits) && (!dlogits || aligned16(dlogits)) &&
                  (!logq_out || aligned16(logq_out));
  // persistent row kernel (16-bit rows in shared memory, clusters for long rows)
  int cslice = 0;
  const int ccl = ce_cluster_size(v, &cslice);
  if (v8 && !logq_out && ccl > 0 && rows >= 2 && v < (1 << 24) &&
      (t_logits == LS2_F16 || t_logits == LS2_BF16)) {
    int rc = t_logits == LS2_F16
                 ? launch_ce_rows<__half>((const __half*)logits, targets, (__half*)dlogits,
                                          row_stats, out3, bad_target, rows, v, ccl, cslice,
                                          alpha, pad_id, has_pad, grad_scale, v, st)
                 : launch_ce_rows<__nv_bfloat16>(
                       (const __nv_bfloat16*)logits, targets, (__nv_bfloat16*)dlogits, row_stats,
                       out3, bad_target, rows, v, ccl, cslice, alpha, pad_id, has_pad, grad_scale,
                       v, st);
    if (rc >= 0) return rc;        // -1: no cluster fits; take the generic path
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
