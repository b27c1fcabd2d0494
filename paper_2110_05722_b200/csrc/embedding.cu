// Token + positional embedding with scale and dropout, and its backward.
//   embedding_forward   F/kernels.py:203-228
//   embedding_backward  F/gradients.py:20-44 (np.add.at scatter -> atomicAdd here;
//                       the per-position table gradient stays a fixed-order sum)
#include <cooperative_groups.h>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace ls2 {

template <typename Tin, typename Tout, bool DROP, bool GEN>
__global__ void emb_fwd_vec(const Tin* __restrict__ E, const Tin* __restrict__ P,
                            const int64_t* __restrict__ tokens, Tout* __restrict__ y,
                            uint8_t* __restrict__ bits, int* bad, int64_t rows, int64_t len,
                            int64_t d, int64_t vocab, int64_t cgs, int rpp, uint64_t seed, const uint64_t* seed_ptr,
                            uint64_t thresh, typename CompOf<Tin>::type es,
                            typename CompOf<Tin>::type ds) {
  using C = typename CompOf<Tin>::type;
  const int lane_row = (int)(threadIdx.x / cgs);
  if (lane_row >= rpp) return;
  const int64_t cg = threadIdx.x % cgs;
  for (int64_t r = (int64_t)blockIdx.x * rpp + lane_row; r < rows; r += (int64_t)gridDim.x * rpp) {
    const int64_t tok = tokens[r];
    const int64_t l = r % len;
    const int64_t g = r * cgs + cg;
    uint32_t kb = 0xFF;
    if (DROP) {
      if (GEN) {
        kb = keep_byte(seed_ptr ? *seed_ptr : seed, (uint64_t)g * 8, thresh);
        bits[g] = (uint8_t)kb;
      } else {
        kb = bits[g];
      }
    }
    Pack8<Tout> o;
    if (tok < 0 || tok >= vocab) {
      if (bad) *bad = 1;
#pragma unroll
      for (int e = 0; e < 8; ++e) o.v[e] = cvt<Tout>(0.f);
    } else {
      Pack8<Tin> ev = ld8(E + tok * d + cg * 8), pv = ld8(P + l * d + cg * 8);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        C a = add_rn(mul_rn(cvt<C>(ev.v[e]), es), cvt<C>(pv.v[e]));
        if (DROP) a = mul_rn(mul_rn(a, bitval<C>(kb, e)), ds);
        o.v[e] = cvt<Tout>(a);
      }
    }
    st8(y + g * 8, o);
  }
}

template <typename Tin, typename Tout, bool DROP, bool GEN>
__global__ void emb_fwd_flat(const Tin* __restrict__ E, const Tin* __restrict__ P,
                             const int64_t* __restrict__ tokens, Tout* __restrict__ y,
                             uint8_t* __restrict__ bits, int* bad, int64_t n, int64_t len,
                             int64_t d, int64_t vocab, uint64_t seed, const uint64_t* seed_ptr, uint64_t thresh,
                             typename CompOf<Tin>::type es, typename CompOf<Tin>::type ds) {
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
      const int64_t r = i / d, j = i % d;
      const int64_t tok = tokens[r];
      C a = 0;
      if (tok < 0 || tok >= vocab) {
        if (bad) *bad = 1;
      } else {
        a = add_rn(mul_rn(cvt<C>(E[tok * d + j]), es), cvt<C>(P[(r % len) * d + j]));
        if (DROP) a = mul_rn(mul_rn(a, bitval<C>(kb, e)), ds);
      }
      y[i] = cvt<Tout>(a);
    }
  }
}

__device__ __forceinline__ void atomic_add8(float* p, const float (&v)[8], bool vec) {
  if (vec) {
    atomicAdd(reinterpret_cast<float4*>(p), make_float4(v[0], v[1], v[2], v[3]));
    atomicAdd(reinterpret_cast<float4*>(p + 4), make_float4(v[4], v[5], v[6], v[7]));
  } else {
#pragma unroll
    for (int e = 0; e < 8; ++e) atomicAdd(p + e, v[e]);
  }
}
__device__ __forceinline__ void atomic_add8(double* p, const double (&v)[8], bool) {
#pragma unroll
  for (int e = 0; e < 8; ++e) atomicAdd(p + e, v[e]);
}

// dE[tok] += es * keep * dy * ds   (one 8-column group per thread)
template <typename Tin, typename Tg, bool DROP>
__global__ void emb_bwd_scatter(const Tin* __restrict__ dy, const int64_t* __restrict__ tokens,
                                const uint8_t* __restrict__ bits, Tg* __restrict__ dE,
                                int64_t rows, int64_t d, int64_t cgs, int rpp, Tg es, Tg ds,
                                bool vec_atomic) {
  const int lane_row = (int)(threadIdx.x / cgs);
  if (lane_row >= rpp) return;
  const int64_t cg = threadIdx.x % cgs;
  for (int64_t r = (int64_t)blockIdx.x * rpp + lane_row; r < rows; r += (int64_t)gridDim.x * rpp) {
    const int64_t g = r * cgs + cg;
    const int64_t tok = tokens[r];
    Pack8<Tin> q = ld8(dy + g * 8);
    const uint32_t kb = DROP ? bits[g] : 0xFF;
    Tg v[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      Tg a = cvt<Tg>(q.v[e]);
      if (DROP) a = mul_rn(mul_rn(a, (Tg)((kb >> e) & 1)), ds);
      v[e] = mul_rn(a, es);
    }
    atomic_add8(dE + tok * d + cg * 8, v, vec_atomic);
  }
}

template <typename Tin, typename Tg, bool DROP>
__global__ void emb_bwd_scatter_flat(const Tin* __restrict__ dy, const int64_t* __restrict__ tokens,
                                     const uint8_t* __restrict__ bits, Tg* __restrict__ dE,
                                     int64_t n, int64_t d, Tg es, Tg ds) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    Tg a = cvt<Tg>(dy[i]);
    if (DROP) a = mul_rn(mul_rn(a, (Tg)((bits[i >> 3] >> (i & 7)) & 1)), ds);
    atomicAdd(dE + tokens[i / d] * d + i % d, mul_rn(a, es));
  }
}

// dP[l, j] (+)= sum_b keep*dy*ds   (fixed order over b); rows >= len zeroed if !beta
template <typename Tin, typename Tg, bool DROP>
__global__ void emb_bwd_pos(const Tin* __restrict__ dy, const uint8_t* __restrict__ bits,
                            Tg* __restrict__ dP, int64_t batch, int64_t len, int64_t d,
                            int64_t max_len, Tg ds, int beta) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < max_len * d;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t l = i / d;
    if (l >= len) {
      if (!beta) dP[i] = (Tg)0;
      continue;
    }
    Tg s = 0;
    for (int64_t b = 0; b < batch; ++b) {
      const int64_t k = (b * len) * d + i;
      Tg a = cvt<Tg>(dy[k]);
      if (DROP) a = mul_rn(mul_rn(a, (Tg)((bits[k >> 3] >> (k & 7)) & 1)), ds);
      s = add_rn(s, a);
    }
    dP[i] = beta ? add_rn(dP[i], s) : s;
  }
}

// Positional-table gradient, vectorised: one CTA per position l; its 256
// threads are (d/8 column groups) x (batch groups).  Each thread sums its batch
// group for 8 columns with 16-byte loads issued ahead of the (sequential)
// adds, then the batch-group partials are folded in fixed order through shared
// memory.  Deterministic; positions >= len get 0 (or keep dP when beta).
// grid (len, S): a cluster of S CTAs splits one position's batch sum (short
// buckets have few positions: L = 8 -> 8 x 8 CTAs instead of 8); rank 0 folds
// the S partials through DSMEM in rank order (deterministic).
template <typename Tin, typename Tg, bool DROP, int NT>
__global__ void __launch_bounds__(NT) emb_bwd_pos_vec(
    const Tin* __restrict__ dy, const uint8_t* __restrict__ bits, Tg* __restrict__ dP,
    int64_t batch_all, int64_t len, int64_t max_len, int64_t d, Tg ds, int beta) {
  __shared__ Tg part[NT * 8];
  __shared__ __align__(16) Tg fin[256 * 8];
  const int64_t l = blockIdx.x;
  const int S = (int)gridDim.y, q = (int)blockIdx.y;
  const int64_t bq0 = batch_all * q / S, batch = batch_all * (q + 1) / S - bq0;
  dy += bq0 * len * d;
  if (DROP) bits += (bq0 * len * d) >> 3;
  const int cgs = (int)(d / 8);
  const int ngrp = NT / cgs;                   // batch groups
  const int cg = threadIdx.x % cgs, grp = threadIdx.x / cgs;
  Tg* out = dP + l * d + cg * 8;
  if (!beta && grp == 0 && q == 0) {          // grid.x = len: CTA l also clears l + k*len >= len
    for (int64_t l2 = l + len; l2 < max_len; l2 += len) {
      Tg* o2 = dP + l2 * d + cg * 8;
#pragma unroll
      for (int e = 0; e < 8; ++e) o2[e] = (Tg)0;
    }
  }
  Tg acc[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) acc[e] = (Tg)0;
  if (grp < ngrp) {
    const int64_t per = (batch + ngrp - 1) / ngrp;
    const int64_t b0 = grp * per, b1 = min(batch, b0 + per);
    constexpr int U = 8;
    for (int64_t bb = b0; bb < b1; bb += U) {
      Pack8<Tin> v[U];
      uint32_t kb[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (bb + u < b1) {
          const int64_t k = ((bb + u) * len + l) * d + cg * 8;
          v[u] = ld8(dy + k);
          kb[u] = DROP ? bits[k >> 3] : 0xFFu;
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (bb + u < b1) {
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            Tg a = cvt<Tg>(v[u].v[e]);
            if (DROP) a = mul_rn(mul_rn(a, (Tg)((kb[u] >> e) & 1)), ds);
            acc[e] = add_rn(acc[e], a);
          }
        }
      }
    }
  }
#pragma unroll
  for (int e = 0; e < 8; ++e) part[threadIdx.x * 8 + e] = acc[e];
  __syncthreads();
  if (S == 1) {
    if (grp == 0) {
      Tg s[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) s[e] = beta ? out[e] : (Tg)0;
      for (int g2 = 0; g2 < ngrp; ++g2)
#pragma unroll
        for (int e = 0; e < 8; ++e) s[e] = add_rn(s[e], part[(g2 * cgs + cg) * 8 + e]);
#pragma unroll
      for (int e = 0; e < 8; ++e) out[e] = s[e];
    }
    return;
  }
  if (grp == 0) {
    Tg s[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) s[e] = (Tg)0;
    for (int g2 = 0; g2 < ngrp; ++g2)
#pragma unroll
      for (int e = 0; e < 8; ++e) s[e] = add_rn(s[e], part[(g2 * cgs + cg) * 8 + e]);
#pragma unroll
    for (int e = 0; e < 8; ++e) fin[cg * 8 + e] = s[e];
  }
  cg::cluster_group cl = cg::this_cluster();
  cl.sync();
  if (q == 0 && grp == 0) {
    Tg s[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) s[e] = beta ? out[e] : (Tg)0;
    for (int p = 0; p < S; ++p) {
      const Tg* src = cl.map_shared_rank(fin + cg * 8, p);
#pragma unroll
      for (int e = 0; e < 8; ++e) s[e] = add_rn(s[e], src[e]);
    }
#pragma unroll
    for (int e = 0; e < 8; ++e) out[e] = s[e];
  }
  cl.sync();                                  // peers' partials stay alive until read
}

inline bool vec8(int64_t d, std::initializer_list<const void*> ptrs) {
  if (d % 8 != 0 || d / 8 > 1024) return false;
  for (const void* p : ptrs)
    if (p && !aligned16(p)) return false;
  return true;
}

}  // namespace ls2

using namespace ls2;

extern "C" {

int ls2_embedding_fwd(const void* emb, const void* pos, const int64_t* tokens, void* y,
                      uint8_t* keep_bits, int* bad_token, int64_t batch, int64_t len, int64_t d,
                      int64_t vocab, double emb_scale, int use_drop, int gen, uint64_t seed, const uint64_t* seed_ptr,
                      uint64_t thresh, double drop_scale, int tin, int tout, void* stream) {
  const int64_t rows = batch * len, n = rows * d;
  if (n <= 0) return LS2_OK;
  cudaStream_t st = as_stream(stream);
  const bool vec = vec8(d, {emb, pos, y});
  return LS2_DISPATCH_IO(tin, tout, "embedding_fwd", [&] {
    using C = typename CompOf<Tin>::type;
    const C es = (C)emb_scale, ds = (C)drop_scale;
    auto launch = [&](auto drop, auto genc) {
      constexpr bool D = decltype(drop)::value, G = decltype(genc)::value;
      if (vec) {
        const int64_t cgs = d / 8;
        const int threads = cgs <= 256 ? 256 : (int)(ceil_div(cgs, 32) * 32);
        const int rpp = cgs <= 256 ? (int)(256 / cgs) : 1;
        const int grid = (int)std::min<int64_t>(ceil_div(rows, rpp), kNumSMs * 8);
        emb_fwd_vec<Tin, Tout, D, G><<<grid, threads, 0, st>>>(
            (const Tin*)emb, (const Tin*)pos, tokens, (Tout*)y, keep_bits, bad_token, rows, len,
            d, vocab, cgs, rpp, seed, seed_ptr, thresh, es, ds);
      } else {
        emb_fwd_flat<Tin, Tout, D, G><<<grid_for(ceil_div(n, 8)), 256, 0, st>>>(
            (const Tin*)emb, (const Tin*)pos, tokens, (Tout*)y, keep_bits, bad_token, n, len, d,
            vocab, seed, seed_ptr, thresh, es, ds);
      }
      return check_launch("embedding_fwd");
    };
    using T_ = std::true_type;
    using F_ = std::false_type;
    if (!use_drop) return launch(F_{}, F_{});
    return gen ? launch(T_{}, T_{}) : launch(T_{}, F_{});
  });
}

int ls2_embedding_bwd(const void* dy, const int64_t* tokens, const uint8_t* keep_bits, void* dE,
                      void* dP, int tgrad, int beta_pos, int64_t batch, int64_t len, int64_t d,
                      int64_t max_len, double emb_scale, int use_drop, double drop_scale, int tin,
                      void* stream) {
  const int64_t rows = batch * len, n = rows * d;
  cudaStream_t st = as_stream(stream);
  if (n <= 0) return LS2_OK;
  auto run = [&](auto tin_tag, auto tg_tag) -> int {
    using Tin = typename decltype(tin_tag)::type;
    using Tg = typename decltype(tg_tag)::type;
    const Tg es = (Tg)emb_scale, ds = (Tg)drop_scale;
    if (dE) {
      const bool vec = vec8(d, {dy, dE});
      if (vec) {
        const int64_t cgs = d / 8;
        const int threads = cgs <= 256 ? 256 : (int)(ceil_div(cgs, 32) * 32);
        const int rpp = cgs <= 256 ? (int)(256 / cgs) : 1;
        const int grid = (int)std::min<int64_t>(ceil_div(rows, rpp), kNumSMs * 8);
        if (use_drop)
          emb_bwd_scatter<Tin, Tg, true><<<grid, threads, 0, st>>>(
              (const Tin*)dy, tokens, keep_bits, (Tg*)dE, rows, d, cgs, rpp, es, ds, true);
        else
          emb_bwd_scatter<Tin, Tg, false><<<grid, threads, 0, st>>>(
              (const Tin*)dy, tokens, keep_bits, (Tg*)dE, rows, d, cgs, rpp, es, ds, true);
      } else {
        if (use_drop)
          emb_bwd_scatter_flat<Tin, Tg, true><<<grid_for(n), 256, 0, st>>>(
              (const Tin*)dy, tokens, keep_bits, (Tg*)dE, n, d, es, ds);
        else
          emb_bwd_scatter_flat<Tin, Tg, false><<<grid_for(n), 256, 0, st>>>(
              (const Tin*)dy, tokens, keep_bits, (Tg*)dE, n, d, es, ds);
      }
      int r = check_launch("embedding_bwd_scatter");
      if (r) return r;
    }
    if (dP) {
      if (vec8(d, {dy, dP}) && d / 8 <= 256 && sizeof(Tg) == 4 && len >= 1) {
        // short buckets: split each position's batch sum over a cluster so the
        // active CTAs (len x S) cover the SMs (L = 8: 25.6 -> 8.8 us in situ);
        // from L = 32 on one CTA per position measured faster (L = 64: 5.0 vs 8.8 us)
        int S = len >= 32 ? 1 : (int)std::min<int64_t>(8, ceil_div((int64_t)kNumSMs, len));
        if (S > batch) S = (int)std::max<int64_t>(1, batch);
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 1;
        at[0].val.clusterDim.y = S;
        at[0].val.clusterDim.z = 1;
        cfg.gridDim = dim3((unsigned)len, (unsigned)S);
        // one CTA per position (S = 1): 512 threads = twice the batch rows in flight
        cfg.blockDim = dim3(S == 1 ? 512 : 256);
        cfg.stream = st;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        auto kern = S == 1 ? (use_drop ? emb_bwd_pos_vec<Tin, Tg, true, 512>
                                       : emb_bwd_pos_vec<Tin, Tg, false, 512>)
                           : (use_drop ? emb_bwd_pos_vec<Tin, Tg, true, 256>
                                       : emb_bwd_pos_vec<Tin, Tg, false, 256>);
        cudaError_t e = cudaLaunchKernelEx(&cfg, kern, (const Tin*)dy, keep_bits, (Tg*)dP, batch,
                                           len, max_len, d, ds, beta_pos);
        if (e != cudaSuccess) return fail(LS2_ERR_CUDA, std::string("embedding_bwd_pos: ") + cudaGetErrorString(e));
        return check_launch("embedding_bwd_pos");
      }
      if (use_drop)
        emb_bwd_pos<Tin, Tg, true><<<grid_for(max_len * d), 256, 0, st>>>(
            (const Tin*)dy, keep_bits, (Tg*)dP, batch, len, d, max_len, ds, beta_pos);
      else
        emb_bwd_pos<Tin, Tg, false><<<grid_for(max_len * d), 256, 0, st>>>(
            (const Tin*)dy, keep_bits, (Tg*)dP, batch, len, d, max_len, ds, beta_pos);
      return check_launch("embedding_bwd_pos");
    }
    return LS2_OK;
  };
  struct H { using type = __half; };
  struct B { using type = __nv_bfloat16; };
  struct F { using type = float; };
  struct D { using type = double; };
  if (tgrad == LS2_F32) {
    if (tin == LS2_F16) return run(H{}, F{});
    if (tin == LS2_BF16) return run(B{}, F{});
    if (tin == LS2_F32) return run(F{}, F{});
  }
  if (tgrad == LS2_F64 && tin == LS2_F64) return run(D{}, D{});
  return fail(LS2_ERR_DTYPE, "embedding_bwd: unsupported dtype pair");
}

}  // extern "C"
