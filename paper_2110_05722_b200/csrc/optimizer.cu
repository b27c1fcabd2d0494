// Single-pass mixed-precision trainer over the contiguous fp16 workspace.
//   zero_grads / _unscaled_grads / adam_step / sgd_step   F/trainer.py:125-177
//   engine scale + narrow                                  F/engine.py:149-157
//
// Bit-exact contract: every f32 operation is issued in numpy's order with
// explicit round-to-nearest intrinsics (no FMA contraction), and the narrow to
// binary16 is RNE, so params/moments match the reference trainer bit for bit.
// The whole-workspace non-finite check (skip-all semantics) is a device counter
// filled by the pass before the update; the update kernel reads it and returns
// early, so a skipped step needs no host round trip.
#include "common.cuh"

namespace ls2 {

__device__ __forceinline__ bool skip_step(const int* nonfinite, const double* loss) {
  if (nonfinite && *nonfinite != 0) return true;
  if (loss && !isfinite(*loss)) return true;
  return false;
}

__device__ __forceinline__ float h2f(uint16_t h) { return __half2float(__ushort_as_half(h)); }
__device__ __forceinline__ uint16_t f2h(float f) { return __half_as_ushort(__float2half_rn(f)); }

struct AdamK {
  float lr, b1, omb1, b2, omb2, eps, wd, ls, bc1, bc2;
  bool unscale;
};

__device__ __forceinline__ void adam_elem(float& p, float g, float& m, float& v, const AdamK& k) {
  if (k.unscale) g = __fdiv_rn(g, k.ls);
  m = __fadd_rn(__fmul_rn(k.b1, m), __fmul_rn(k.omb1, g));
  v = __fadd_rn(__fmul_rn(k.b2, v), __fmul_rn(k.omb2, __fmul_rn(g, g)));
  const float mh = __fdiv_rn(m, k.bc1);
  const float vh = __fdiv_rn(v, k.bc2);
  const float q = __fdiv_rn(mh, __fadd_rn(__fsqrt_rn(vh), k.eps));
  p = __fsub_rn(p, __fmul_rn(k.lr, __fadd_rn(q, __fmul_rn(k.wd, p))));
}

__device__ __forceinline__ AdamK adam_constants(const float* __restrict__ hyper,
                                                 const float* __restrict__ bc, int64_t bc_len,
                                                 int64_t t_host, const int64_t* applied) {
  const int64_t t = t_host > 0 ? t_host : (*applied + 1);
  float bc1, bc2;
  if (t < bc_len) {
    bc1 = bc[2 * t];
    bc2 = bc[2 * t + 1];
  } else {   // past the table: f32(1 - beta**t) in f64, the betas stored after it
    const double* betas = reinterpret_cast<const double*>(bc + 2 * bc_len);
    bc1 = __double2float_rn(1.0 - pow(betas[0], (double)t));
    bc2 = __double2float_rn(1.0 - pow(betas[1], (double)t));
  }
  return AdamK{hyper[0], hyper[1], hyper[2], hyper[3], hyper[4], hyper[5], hyper[6], hyper[7],
               bc1, bc2, hyper[7] != 1.0f};
}

// Adam over elements [0, n) of the given spans; CTA `bid` of `nblk` grid-strides.
__device__ __forceinline__ void adam_range(uint16_t* __restrict__ p16,
                                           const uint16_t* __restrict__ g16,
                                           float* __restrict__ m, float* __restrict__ v,
                                           int64_t n, const AdamK& k, bool vec, int64_t bid,
                                           int64_t nblk) {
  const int64_t stride = nblk * blockDim.x;
  const int64_t first = bid * (int64_t)blockDim.x + threadIdx.x;
  int64_t tail = 0;
  if (vec) {
    const int64_t groups = n / 8;
    for (int64_t gi = first; gi < groups; gi += stride) {
      const uint4 pp = __ldcs(reinterpret_cast<const uint4*>(p16) + gi);
      const uint4 gg = __ldcs(reinterpret_cast<const uint4*>(g16) + gi);
      float4 m0 = __ldcs(reinterpret_cast<const float4*>(m) + 2 * gi);
      float4 m1 = __ldcs(reinterpret_cast<const float4*>(m) + 2 * gi + 1);
      float4 v0 = __ldcs(reinterpret_cast<const float4*>(v) + 2 * gi);
      float4 v1 = __ldcs(reinterpret_cast<const float4*>(v) + 2 * gi + 1);
      const uint16_t* ph = reinterpret_cast<const uint16_t*>(&pp);
      const uint16_t* gh = reinterpret_cast<const uint16_t*>(&gg);
      float* mm[2] = {&m0.x, &m1.x};
      float* vv[2] = {&v0.x, &v1.x};
      uint4 po;
      uint16_t* oh = reinterpret_cast<uint16_t*>(&po);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        float p = h2f(ph[e]);
        adam_elem(p, h2f(gh[e]), mm[e >> 2][e & 3], vv[e >> 2][e & 3], k);
        oh[e] = f2h(p);
      }
      __stcs(reinterpret_cast<uint4*>(p16) + gi, po);
      __stcs(reinterpret_cast<float4*>(m) + 2 * gi, m0);
      __stcs(reinterpret_cast<float4*>(m) + 2 * gi + 1, m1);
      __stcs(reinterpret_cast<float4*>(v) + 2 * gi, v0);
      __stcs(reinterpret_cast<float4*>(v) + 2 * gi + 1, v1);
    }
    tail = groups * 8;
  }
  for (int64_t i = tail + first; i < n; i += stride) {
    float p = h2f(p16[i]);
    adam_elem(p, h2f(g16[i]), m[i], v[i], k);
    p16[i] = f2h(p);
  }
}

__global__ void adam_kernel(uint16_t* __restrict__ p16, const uint16_t* __restrict__ g16,
                            float* __restrict__ m, float* __restrict__ v, int64_t n,
                            const float* __restrict__ hyper, const float* __restrict__ bc,
                            int64_t bc_len, int64_t t_host, const int64_t* __restrict__ applied,
                            const int* nonfinite, const double* loss, bool vec) {
  if (skip_step(nonfinite, loss)) return;
  const AdamK k = adam_constants(hyper, bc, bc_len, t_host, applied);
  adam_range(p16, g16, m, v, n, k, vec, blockIdx.x, gridDim.x);
}

// The sharded optimizer's update: the rank's element spans {offset, length}
// (int64 pairs, device) of the flat workspace, one grid row (blockIdx.y) per span.
__global__ void adam_spans_kernel(uint16_t* __restrict__ p16, const uint16_t* __restrict__ g16,
                                  float* __restrict__ m, float* __restrict__ v,
                                  const int64_t* __restrict__ spans,
                                  const float* __restrict__ hyper, const float* __restrict__ bc,
                                  int64_t bc_len, int64_t t_host,
                                  const int64_t* __restrict__ applied, const int* nonfinite,
                                  const double* loss, bool vec_ok) {
  if (skip_step(nonfinite, loss)) return;
  const AdamK k = adam_constants(hyper, bc, bc_len, t_host, applied);
  const int64_t off = spans[2 * blockIdx.y], n = spans[2 * blockIdx.y + 1];
  const bool vec = vec_ok && (off & 7) == 0;
  adam_range(p16 + off, g16 + off, m + off, v + off, n, k, vec, blockIdx.x, gridDim.x);
}

__global__ void sgd_kernel(uint16_t* __restrict__ p16, const uint16_t* __restrict__ g16,
                           float* __restrict__ vel, int64_t n, const float* __restrict__ hyper,
                           const int* nonfinite, const double* loss) {
  if (skip_step(nonfinite, loss)) return;
  const float lr = hyper[0], mom = hyper[1], wd = hyper[2], ls = hyper[3];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    float g = h2f(g16[i]);
    if (ls != 1.0f) g = __fdiv_rn(g, ls);
    float p = h2f(p16[i]);
    if (wd != 0.0f) g = __fadd_rn(g, __fmul_rn(wd, p));
    const float vn = __fadd_rn(__fmul_rn(mom, vel[i]), g);
    vel[i] = vn;
    p = __fsub_rn(p, __fmul_rn(lr, vn));
    p16[i] = f2h(p);
  }
}

__global__ void step_commit_kernel(int64_t* applied, const int* nonfinite, const double* loss,
                                   int* applied_flag) {
  const bool ok = !skip_step(nonfinite, loss);
  if (ok) *applied += 1;
  if (applied_flag) *applied_flag = ok ? 1 : 0;
}

// step_commit plus the step's 5-number report {loss sum, tokens, correct,
// applied, non-finite count} in one launch (the D2H source of train_step)
__global__ void step_report_kernel(int64_t* applied, const int* nonfinite, const double* totals,
                                   double* report) {
  const bool ok = !skip_step(nonfinite, totals);
  if (ok && applied) *applied += 1;   // applied == NULL: report only (before the update)
  report[0] = totals[0];
  report[1] = totals[1];
  report[2] = totals[2];
  report[3] = ok ? 1.0 : 0.0;
  report[4] = (double)*nonfinite;
}

__device__ __forceinline__ int warp_count(int c) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  return c;
}

__device__ __forceinline__ bool h_nonfinite(uint16_t h) { return (h & 0x7C00u) == 0x7C00u; }

// g16 = RNE(acc * f32(loss_scale / count) * post); counts non-finite outputs
__global__ void scale_narrow_kernel(const float* __restrict__ acc, uint16_t* __restrict__ g16,
                                    int64_t n, double loss_scale, const double* out3,
                                    int64_t count_host, float post, int* nonfinite, bool vec) {
  double cnt = count_host >= 0 ? (double)count_host : out3[1];
  if (cnt < 1.0) cnt = 1.0;
  const float s = __fmul_rn((float)(loss_scale / cnt), post);
  int bad = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  if (vec) {
    const int64_t groups = n / 8;
    for (int64_t gi = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; gi < groups; gi += stride) {
      const float4 a0 = __ldcs(reinterpret_cast<const float4*>(acc) + 2 * gi);
      const float4 a1 = __ldcs(reinterpret_cast<const float4*>(acc) + 2 * gi + 1);
      const float av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
      uint4 o;
      uint16_t* oh = reinterpret_cast<uint16_t*>(&o);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        oh[e] = f2h(__fmul_rn(av[e], s));
        bad += h_nonfinite(oh[e]);
      }
      reinterpret_cast<uint4*>(g16)[gi] = o;
    }
    for (int64_t i = groups * 8 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
      g16[i] = f2h(__fmul_rn(acc[i], s));
      bad += h_nonfinite(g16[i]);
    }
  } else {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
      g16[i] = f2h(__fmul_rn(acc[i], s));
      bad += h_nonfinite(g16[i]);
    }
  }
  if (nonfinite) {
    bad = warp_count(bad);
    if ((threadIdx.x & 31) == 0 && bad) atomicAdd(nonfinite, bad);
  }
}

// Deferred column-sum finishes fused with the narrow pass.  Every bias / LayerNorm
// parameter gradient of the step was left as per-block partial column sums
// (partial[g][k][c], g < nblk) by its producing kernel; one launch reduces them
// all in fixed order, scales like scale_narrow and writes the fp16 gradients.
// desc row: {dst (element offset in the workspace), cols, part (double offset),
//            nblk, stride (doubles per block), k}
// One CTA (8 warps) per 64 columns of one deferred tensor: lane l owns columns
// c0 + 2l, +1 (16-byte loads), warp w sums partial rows w, w+8, ... with four
// loads in flight, and the 8 warp sums are folded in warp order (deterministic).
constexpr int kFinishCols = 64;
template <bool ACC32>
__global__ void __launch_bounds__(256) finish_narrow_kernel(
    const int64_t* __restrict__ desc, const int32_t* __restrict__ chunks,
    const double* __restrict__ part_base, uint16_t* __restrict__ g16,
    float* __restrict__ acc32, double loss_scale,
    const double* out3, int64_t count_host, float post, int* nonfinite) {
  __shared__ double red[8][kFinishCols + 1];
  const int di = chunks[2 * blockIdx.x], c0 = chunks[2 * blockIdx.x + 1];
  const int64_t* d = desc + 6 * di;
  const int64_t dst = d[0], cols = d[1], part = d[2], stride = d[4], k = d[5];
  const int nblk = (int)d[3];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t c = c0 + 2 * lane;
  const double* p = part_base + part + k * cols + c;
  double sx = 0, sy = 0;
  if (c + 1 < cols && (cols & 1) == 0) {
    double2 a0 = make_double2(0, 0), a1 = a0, a2 = a0, a3 = a0;
    int g = w;
    for (; g + 24 < nblk; g += 32) {
      const double2 v0 = *reinterpret_cast<const double2*>(p + (int64_t)g * stride);
      const double2 v1 = *reinterpret_cast<const double2*>(p + (int64_t)(g + 8) * stride);
      const double2 v2 = *reinterpret_cast<const double2*>(p + (int64_t)(g + 16) * stride);
      const double2 v3 = *reinterpret_cast<const double2*>(p + (int64_t)(g + 24) * stride);
      a0.x += v0.x; a0.y += v0.y; a1.x += v1.x; a1.y += v1.y;
      a2.x += v2.x; a2.y += v2.y; a3.x += v3.x; a3.y += v3.y;
    }
    for (; g < nblk; g += 8) {
      const double2 v = *reinterpret_cast<const double2*>(p + (int64_t)g * stride);
      a0.x += v.x; a0.y += v.y;
    }
    sx = (a0.x + a1.x) + (a2.x + a3.x);
    sy = (a0.y + a1.y) + (a2.y + a3.y);
  } else {
    for (int g = w; g < nblk; g += 8) {
      if (c < cols) sx += p[(int64_t)g * stride];
      if (c + 1 < cols) sy += p[(int64_t)g * stride + 1];
    }
  }
  red[w][2 * lane] = sx;
  red[w][2 * lane + 1] = sy;
  __syncthreads();
  if (w < 2) {
    const int cc = lane + 32 * w;
    const int64_t col = c0 + cc;
    int bad = 0;
    if (ACC32) {   // unscaled f32 column sums into the accumulator (reduced, then narrowed)
      if (col < cols) {
        double t = 0;
#pragma unroll
        for (int q = 0; q < 8; ++q) t += red[q][cc];
        acc32[dst + col] = (float)t;
      }
      return;
    }
    if (col < cols) {
      double t = 0;
#pragma unroll
      for (int q = 0; q < 8; ++q) t += red[q][cc];
      double cnt = count_host >= 0 ? (double)count_host : out3[1];
      if (cnt < 1.0) cnt = 1.0;
      const float sc = __fmul_rn((float)(loss_scale / cnt), post);
      const uint16_t h = f2h(__fmul_rn((float)t, sc));
      g16[dst + col] = h;
      bad = h_nonfinite(h);
    }
    if (nonfinite) {
      bad = warp_count(bad);
      if (lane == 0 && bad) atomicAdd(nonfinite, bad);
    }
  }
}

__global__ void count_nonfinite_kernel(const uint16_t* __restrict__ g16, int64_t n, int* nonfinite) {
  int bad = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    bad += h_nonfinite(g16[i]);
  bad = warp_count(bad);
  if ((threadIdx.x & 31) == 0 && bad) atomicAdd(nonfinite, bad);
}

inline int stream_grid(int64_t work) {
  int64_t g = ceil_div(work, 256);
  const int64_t cap = (int64_t)kNumSMs * 8;  // persistent-ish: 8 CTAs of 256 per SM
  return (int)(g < 1 ? 1 : (g > cap ? cap : g));
}

}  // namespace ls2

using namespace ls2;

extern "C" {

int ls2_adam(uint16_t* p16, const uint16_t* g16, float* m, float* v, int64_t n, const float* hyper,
             const float* bc_table, int64_t bc_len, int64_t t_host, const int64_t* applied,
             const int* nonfinite, const double* loss, void* stream) {
  if (n <= 0) return LS2_OK;
  if (t_host <= 0 && !applied) return fail(LS2_ERR_SHAPE, "adam: need t_host or applied counter");
  const bool vec = aligned16(p16) && aligned16(g16) && aligned16(m) && aligned16(v);
  adam_kernel<<<stream_grid(vec ? ceil_div(n, 8) : n), 256, 0, as_stream(stream)>>>(
      p16, g16, m, v, n, hyper, bc_table, bc_len, t_host, applied, nonfinite, loss, vec);
  return check_launch("adam");
}

int ls2_adam_spans(uint16_t* p16, const uint16_t* g16, float* m, float* v, const int64_t* spans,
                   int64_t n_spans, int64_t max_len, const float* hyper, const float* bc_table,
                   int64_t bc_len, int64_t t_host, const int64_t* applied, const int* nonfinite,
                   const double* loss, void* stream) {
  if (n_spans <= 0 || max_len <= 0) return LS2_OK;
  if (n_spans > 65535) return fail(LS2_ERR_SHAPE, "adam_spans: too many spans");
  if (t_host <= 0 && !applied) return fail(LS2_ERR_SHAPE, "adam: need t_host or applied counter");
  const bool vec = aligned16(p16) && aligned16(g16) && aligned16(m) && aligned16(v);
  int64_t gx = ceil_div(ceil_div(max_len, 8), 256);
  const int64_t cap = ceil_div((int64_t)kNumSMs * 8, n_spans);
  gx = gx < 1 ? 1 : (gx > cap ? cap : gx);
  adam_spans_kernel<<<dim3((unsigned)gx, (unsigned)n_spans), 256, 0, as_stream(stream)>>>(
      p16, g16, m, v, spans, hyper, bc_table, bc_len, t_host, applied, nonfinite, loss, vec);
  return check_launch("adam_spans");
}

int ls2_sgd(uint16_t* p16, const uint16_t* g16, float* vel, int64_t n, const float* hyper,
            const int* nonfinite, const double* loss, void* stream) {
  if (n <= 0) return LS2_OK;
  sgd_kernel<<<stream_grid(n), 256, 0, as_stream(stream)>>>(p16, g16, vel, n, hyper, nonfinite,
                                                            loss);
  return check_launch("sgd");
}

int ls2_step_commit(int64_t* applied, const int* nonfinite, const double* loss, int* applied_flag,
                    void* stream) {
  step_commit_kernel<<<1, 1, 0, as_stream(stream)>>>(applied, nonfinite, loss, applied_flag);
  return check_launch("step_commit");
}

int ls2_step_report(int64_t* applied, const int* nonfinite, const double* totals, double* report,
                    void* stream) {
  step_report_kernel<<<1, 1, 0, as_stream(stream)>>>(applied, nonfinite, totals, report);
  return check_launch("step_report");
}

int ls2_scale_narrow(const float* acc32, uint16_t* g16, int64_t n, double loss_scale,
                     const double* out3, int64_t count_host, float post, int* nonfinite,
                     void* stream) {
  if (n <= 0) return LS2_OK;
  if (count_host < 0 && !out3) return fail(LS2_ERR_SHAPE, "scale_narrow: no token count");
  const bool vec = aligned16(acc32) && aligned16(g16);
  scale_narrow_kernel<<<stream_grid(vec ? ceil_div(n, 8) : n), 256, 0, as_stream(stream)>>>(
      acc32, g16, n, loss_scale, out3, count_host, post, nonfinite, vec);
  return check_launch("scale_narrow");
}

int ls2_finish_narrow(const int64_t* desc, const int32_t* chunks, int64_t n_chunks,
                      const double* partial_base, uint16_t* g16, double loss_scale,
                      const double* out3, int64_t count_host, float post, int* nonfinite,
                      void* stream) {
  if (n_chunks <= 0) return LS2_OK;
  if (count_host < 0 && !out3) return fail(LS2_ERR_SHAPE, "finish_narrow: no token count");
  finish_narrow_kernel<false><<<(unsigned)n_chunks, 256, 0, as_stream(stream)>>>(
      desc, chunks, partial_base, g16, nullptr, loss_scale, out3, count_host, post, nonfinite);
  return check_launch("finish_narrow");
}

int ls2_finish_acc32(const int64_t* desc, const int32_t* chunks, int64_t n_chunks,
                     const double* partial_base, float* acc32, void* stream) {
  if (n_chunks <= 0) return LS2_OK;
  finish_narrow_kernel<true><<<(unsigned)n_chunks, 256, 0, as_stream(stream)>>>(
      desc, chunks, partial_base, nullptr, acc32, 1.0, nullptr, 1, 1.0f, nullptr);
  return check_launch("finish_acc32");
}

int ls2_count_nonfinite_f16(const uint16_t* g16, int64_t n, int* nonfinite, void* stream) {
  if (n <= 0) return LS2_OK;
  count_nonfinite_kernel<<<stream_grid(n), 256, 0, as_stream(stream)>>>(g16, n, nonfinite);
  return check_launch("count_nonfinite");
}

}  // extern "C"
