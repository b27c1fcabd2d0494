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
