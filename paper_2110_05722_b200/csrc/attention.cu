// Fused short-sequence attention (fp16, head dim 64, L <= 128), forward and backward.
//
// Replaces, per attention block, the reference's chain (F/model.py:362-376 and
// :482-495): scores = Q K^T * 1/sqrt(hd); softmax_forward(mask) (F/kernels.py:277-307);
// ctx = P V; merge heads — and backward: dP = dctx V^T; softmax_backward
// (F/gradients.py:77-100) * 1/sqrt(hd); dQ = dS K; dK = dS^T Q; dV = P^T dctx.
//
// One CTA per (batch, head).  Q/K/V/dO are read straight out of the fused
// projection buffers (row stride = ld, head h at column h*64) with cp.async into
// padded shared memory; the four contractions run on tensor cores
// (mma.sync m16n8k16, fp32 accumulate); the softmax is computed in registers on
// the accumulator fragments; P (needed by backward, as the reference stashes it)
// is written once in fp16; the context / gradients are written straight into the
// merged [B, L, H*64] layouts.  Nothing but P ever round-trips through HBM.
#include "common.cuh"

namespace ls2 {

constexpr int kHd = 64;
constexpr int kPad = 8;                  // halves of padding per smem row (bank spread)
constexpr int kRow = kHd + kPad;         // 72 halves = 144 B

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
  const int n = valid ? 16 : 0;   // zero-fill rows past the sequence end
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(smem)), "l"(gmem),
               "r"(n));
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::);
}

__device__ __forceinline__ void ldsm_x4(uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3,
                                        const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(smem_u32(p)));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3,
                                          const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(smem_u32(p)));
}

__device__ __forceinline__ void mma16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0,
                                         uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};\n"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ uint32_t pack_h2(float lo, float hi) {
  __half2 h = __floats2half2_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&h);
}
__device__ __forceinline__ float2 unpack_h2(uint32_t v) {
  __half2 h = *reinterpret_cast<__half2*>(&v);
  return __half22float2(h);
}

// A fragment (16x16) of a row-major smem matrix at (r0, c0)
__device__ __forceinline__ void frag_a(uint32_t (&a)[4], const __half* s, int ld, int r0, int c0,
                                       int lane) {
  const int r = r0 + (lane & 7) + 8 * ((lane >> 3) & 1);
  const int c = c0 + 8 * (lane >> 4);
  ldsm_x4(a[0], a[1], a[2], a[3], s + r * ld + c);
}
// A fragment (16x16) of X^T where X is row-major in smem: A[m][kk] = X[kk][m]
__device__ __forceinline__ void frag_a_t(uint32_t (&a)[4], const __half* s, int ld, int m0,
                                         int kk0, int lane) {
  const int r = kk0 + (lane & 7) + 8 * (lane >> 4);
  const int c = m0 + 8 * ((lane >> 3) & 1);
  ldsm_x4_t(a[0], a[1], a[2], a[3], s + r * ld + c);
}
// B fragments for two n-tiles (n0, n0+8), k16 at k0, from smem stored [n][k] (B col-major)
__device__ __forceinline__ void frag_b_nk(uint32_t (&b)[4], const __half* s, int ld, int n0,
                                          int k0, int lane) {
  const int r = n0 + (lane & 7) + 8 * (lane >> 4);
  const int c = k0 + 8 * ((lane >> 3) & 1);
  ldsm_x4(b[0], b[1], b[2], b[3], s + r * ld + c);
}
// B fragments for two n-tiles, from smem stored [k][n] (B row-major) via .trans
__device__ __forceinline__ void frag_b_kn(uint32_t (&b)[4], const __half* s, int ld, int k0,
                                          int n0, int lane) {
  const int r = k0 + (lane & 7) + 8 * ((lane >> 3) & 1);
  const int c = n0 + 8 * (lane >> 4);
  ldsm_x4_t(b[0], b[1], b[2], b[3], s + r * ld + c);
}

// load rows [0, rows_pad) x 64 halves of a (b,h) slice into smem (zero past `rows`)
__device__ __forceinline__ void load_tile(__half* s, const __half* g, int64_t ld, int rows,
                                          int rows_pad) {
  for (int i = threadIdx.x; i < rows_pad * 8; i += blockDim.x) {
    const int r = i >> 3, ch = i & 7;
    const bool ok = r < rows;
    cp_async16(s + r * kRow + ch * 8, g + (ok ? (int64_t)r * ld : 0) + ch * 8, ok);
  }
}

struct AttnArgs {
  const __half *q, *k, *v;
  int64_t ldq, ldk, ldv;
  __half* probs;          // [B, H, Lq, Lk]
  __half* o;              // ctx, merged [B, Lq, ldo]
  int64_t ldo;
  int H, Lq, Lk;
  int mask;               // LS2_MASK_*
  const int64_t* lens;
  float scale;
};

template <int QT, int KT>
__global__ void __launch_bounds__(32 * QT) attn_fwd_kernel(AttnArgs a) {
  constexpr int LQ = 16 * QT, LK = 16 * KT, PLD = LK + kPad;
  extern __shared__ __align__(16) __half sm[];
  __half* Qs = sm;                         // [LQ][72]  (reused for O staging)
  __half* Ks = Qs + LQ * kRow;             // [LK][72]
  __half* Vs = Ks + LK * kRow;             // [LK][72]
  __half* Ps = Vs + LK * kRow;             // [LQ][LK+8]
  const int bh = blockIdx.x, b = bh / a.H, h = bh % a.H;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  // Q, K first (one cp.async group), V second: S = QK^T and the softmax run
  // while V is still in flight
  load_tile(Qs, a.q + (int64_t)b * a.Lq * a.ldq + h * kHd, a.ldq, a.Lq, LQ);
  load_tile(Ks, a.k + (int64_t)b * a.Lk * a.ldk + h * kHd, a.ldk, a.Lk, LK);
  asm volatile("cp.async.commit_group;\n" ::);
  load_tile(Vs, a.v + (int64_t)b * a.Lk * a.ldv + h * kHd, a.ldv, a.Lk, LK);
  asm volatile("cp.async.commit_group;\n" ::);
  asm volatile("cp.async.wait_group 1;\n" ::);
  __syncthreads();

  // S = Q K^T for rows [16w, 16w+16)
  float s[2 * KT][4];
#pragma unroll
  for (int j = 0; j < 2 * KT; ++j) s[j][0] = s[j][1] = s[j][2] = s[j][3] = 0.f;
#pragma unroll
  for (int kk = 0; kk < kHd; kk += 16) {
    uint32_t af[4];
    frag_a(af, Qs, kRow, 16 * w, kk, lane);
#pragma unroll
    for (int nt = 0; nt < KT; ++nt) {
      uint32_t bf[4];
      frag_b_nk(bf, Ks, kRow, 16 * nt, kk, lane);
      mma16816(s[2 * nt], af, bf[0], bf[1]);
      mma16816(s[2 * nt + 1], af, bf[2], bf[3]);
    }
  }
  // masked softmax on the fragments: thread owns rows g, g+8; cols 8j + 2t, +1
  const int g = lane >> 2, t = lane & 3;
  const int r0 = 16 * w + g, r1 = r0 + 8;
  const int64_t len = a.mask == LS2_MASK_PADDING ? a.lens[b] : a.Lk;
  float m0 = -INFINITY, m1 = -INFINITY;
#pragma unroll
  for (int j = 0; j < 2 * KT; ++j) {
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int c = 8 * j + 2 * t + e;
      bool k0 = c < len, k1 = c < len;
      if (a.mask == LS2_MASK_CAUSAL) { k0 = k0 && c <= r0; k1 = k1 && c <= r1; }
      s[j][e] = k0 ? s[j][e] * a.scale : -INFINITY;
      s[j][2 + e] = k1 ? s[j][2 + e] * a.scale : -INFINITY;
      m0 = fmaxf(m0, s[j][e]);
      m1 = fmaxf(m1, s[j][2 + e]);
    }
  }
  m0 = fmaxf(m0, __shfl_xor_sync(0xffffffffu, m0, 1));
  m0 = fmaxf(m0, __shfl_xor_sync(0xffffffffu, m0, 2));
  m1 = fmaxf(m1, __shfl_xor_sync(0xffffffffu, m1, 1));
  m1 = fmaxf(m1, __shfl_xor_sync(0xffffffffu, m1, 2));
  float z0 = 0.f, z1 = 0.f;
#pragma unroll
  for (int j = 0; j < 2 * KT; ++j) {
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      s[j][e] = s[j][e] == -INFINITY ? 0.f : __expf(s[j][e] - m0);
      s[j][2 + e] = s[j][2 + e] == -INFINITY ? 0.f : __expf(s[j][2 + e] - m1);
      z0 += s[j][e];
      z1 += s[j][2 + e];
    }
  }
  z0 += __shfl_xor_sync(0xffffffffu, z0, 1);
  z0 += __shfl_xor_sync(0xffffffffu, z0, 2);
  z1 += __shfl_xor_sync(0xffffffffu, z1, 1);
  z1 += __shfl_xor_sync(0xffffffffu, z1, 2);
  const float i0 = z0 > 0.f ? 1.f / z0 : 0.f, i1 = z1 > 0.f ? 1.f / z1 : 0.f;
  uint32_t p[2 * KT][2];   // fp16 P in C-fragment order
#pragma unroll
  for (int j = 0; j < 2 * KT; ++j) {
    p[j][0] = pack_h2(s[j][0] * i0, s[j][1] * i0);
    p[j][1] = pack_h2(s[j][2] * i1, s[j][3] * i1);
    *reinterpret_cast<uint32_t*>(Ps + r0 * PLD + 8 * j + 2 * t) = p[j][0];
    *reinterpret_cast<uint32_t*>(Ps + r1 * PLD + 8 * j + 2 * t) = p[j][1];
  }
  asm volatile("cp.async.wait_group 0;\n" ::);
  __syncthreads();
  // O = P V (P fragments reused as A operands: C layout of two n-tiles == A layout)
  float o[8][4];
#pragma unroll
  for (int j = 0; j < 8; ++j) o[j][0] = o[j][1] = o[j][2] = o[j][3] = 0.f;
#pragma unroll
  for (int kt = 0; kt < KT; ++kt) {
    const uint32_t af[4] = {p[2 * kt][0], p[2 * kt][1], p[2 * kt + 1][0], p[2 * kt + 1][1]};
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) {
      uint32_t bf[4];
      frag_b_kn(bf, Vs, kRow, 16 * kt, 16 * nt, lane);
      mma16816(o[2 * nt], af, bf[0], bf[1]);
      mma16816(o[2 * nt + 1], af, bf[2], bf[3]);
    }
  }
  // stage O into Qs (this warp's own rows only), then coalesced stores
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    *reinterpret_cast<uint32_t*>(Qs + r0 * kRow + 8 * j + 2 * t) = pack_h2(o[j][0], o[j][1]);
    *reinterpret_cast<uint32_t*>(Qs + r1 * kRow + 8 * j + 2 * t) = pack_h2(o[j][2], o[j][3]);
  }
  __syncthreads();
  __half* og = a.o + (int64_t)b * a.Lq * a.ldo + h * kHd;
  for (int i = threadIdx.x; i < a.Lq * 8; i += blockDim.x) {
    const int r = i >> 3, ch = i & 7;
    *reinterpret_cast<uint4*>(og + (int64_t)r * a.ldo + ch * 8) =
        *reinterpret_cast<const uint4*>(Qs + r * kRow + ch * 8);
  }
  __half* pg = a.probs + (int64_t)bh * a.Lq * a.Lk;
  if ((a.Lk & 7) == 0) {
    const int cpr = a.Lk >> 3;
    for (int i = threadIdx.x; i < a.Lq * cpr; i += blockDim.x) {
      const int r = i / cpr, ch = i % cpr;
      *reinterpret_cast<uint4*>(pg + (int64_t)r * a.Lk + ch * 8) =
          *reinterpret_cast<const uint4*>(Ps + r * PLD + ch * 8);
    }
  } else {
    for (int i = threadIdx.x; i < a.Lq * a.Lk; i += blockDim.x)
      pg[i] = Ps[(i / a.Lk) * PLD + i % a.Lk];
  }
}

struct AttnBwdArgs {
  const __half *q, *k, *v, *probs, *dout;
  int64_t ldq, ldk, ldv, lddo;
  __half *dq, *dk, *dv;
  int64_t lddq, lddk, lddv;
  int H, Lq, Lk;
  float scale;
  // optional bias-gradient partials (the projection biases' column sums of the
  // stored dQ / dK / dV): row b, columns h*64.. of each, f64, one row per batch
  double *csq, *csk, *csv;
  int64_t ldcsq, ldcsk, ldcsv;
};

// column sums of one warp's 16-row tile of a result (the fp16-rounded values
// the kernel stores; rows >= valid excluded).  Each thread holds rows g, g+8 of
// columns 8j + 2t, +1 (j < 8); the sum over the 8 row groups g is a fixed-order
// reduce-scatter (halve the columns per xor-16/8/4 round: 8 + 4 + 2 shuffles
// instead of 48), after which lane (g, t) owns columns 8g + 2t, +1 -> cs[0..63].
__device__ __forceinline__ void tile_colsum(const float (&acc)[8][4], int r0, int valid,
                                            float* cs, int lane) {
  const int g = lane >> 2, t = lane & 3;
  float v[16];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const float2 v0 = r0 < valid ? unpack_h2(pack_h2(acc[j][0], acc[j][1])) : make_float2(0.f, 0.f);
    const float2 v1 = r0 + 8 < valid ? unpack_h2(pack_h2(acc[j][2], acc[j][3])) : make_float2(0.f, 0.f);
    v[2 * j] = v0.x + v1.x;
    v[2 * j + 1] = v0.y + v1.y;
  }
  const bool h2 = (g & 4) != 0, h1 = (g & 2) != 0, h0 = (g & 1) != 0;
#pragma unroll
  for (int q = 0; q < 8; ++q) {            // xor 16: keep half [8*h2, 8*h2 + 8)
    const float send = h2 ? v[q] : v[8 + q];
    const float keep = h2 ? v[8 + q] : v[q];
    v[q] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {            // xor 8
    const float send = h1 ? v[q] : v[4 + q];
    const float keep = h1 ? v[4 + q] : v[q];
    v[q] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
  }
#pragma unroll
  for (int q = 0; q < 2; ++q) {            // xor 4
    const float send = h0 ? v[q] : v[2 + q];
    const float keep = h0 ? v[2 + q] : v[q];
    v[q] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
  }
  cs[8 * g + 2 * t] = v[0];
  cs[8 * g + 2 * t + 1] = v[1];
}

// fold the per-warp tile sums in warp order and write the f64 partial rows
template <int QT, int KT>
__device__ __forceinline__ void attn_bwd_colsum_store(const AttnBwdArgs& a, int bh, const float* cs) {
  constexpr int NW = QT > KT ? QT : KT;
  const int b = bh / a.H, h = bh % a.H;
  for (int i = threadIdx.x; i < 3 * 64; i += blockDim.x) {
    const int which = i >> 6, c = i & 63;
    double* dst = which == 0 ? a.csq : which == 1 ? a.csk : a.csv;
    if (!dst) continue;
    const int64_t ld = which == 0 ? a.ldcsq : which == 1 ? a.ldcsk : a.ldcsv;
    const int nw = which == 0 ? QT : KT;
    float sacc = 0.f;
    for (int w = 0; w < nw; ++w) sacc += cs[(which * NW + w) * 64 + c];
    dst[(int64_t)b * ld + h * kHd + c] = (double)sacc;
  }
}

__device__ __forceinline__ void store_rows(__half* gbase, int64_t ld, const __half* s, int rows) {
  for (int i = threadIdx.x; i < rows * 8; i += blockDim.x) {
    const int r = i >> 3, ch = i & 7;
    *reinterpret_cast<uint4*>(gbase + (int64_t)r * ld + ch * 8) =
        *reinterpret_cast<const uint4*>(s + r * kRow + ch * 8);
  }
}

// 2 * max(QT, KT) warps in two concurrent roles per phase:
//   phase A  query warps: dP = dO V^T, dS = P (dP - rowsum(dP P)) * scale -> smem
//            key warps:   dV = P^T dO  (needs only P and dO: runs beside dS)
//   phase B  query warps: dQ = dS K
//            key warps:   dK = dS^T Q
// so the dependent chain per CTA is two 32-MMA steps, not two 64-MMA steps.
// issue the cp.async loads of one (batch, head) item: Q, K, V, dO tiles and P
// (split: V, dO, P form one cp.async group and Q, K a second one, so phase A,
// which needs only the first, can start while Q and K are still in flight)
__device__ __forceinline__ void attn_bwd_issue(const AttnBwdArgs& a, int bh, __half* Qs, __half* Ks,
                                               __half* Vs, __half* Os, __half* Ps, int LQ, int LK,
                                               int PLD, bool split = false) {
  const int b = bh / a.H, h = bh % a.H;
  load_tile(Vs, a.v + (int64_t)b * a.Lk * a.ldv + h * kHd, a.ldv, a.Lk, LK);
  load_tile(Os, a.dout + (int64_t)b * a.Lq * a.lddo + h * kHd, a.lddo, a.Lq, LQ);
  const __half* pg = a.probs + (int64_t)bh * a.Lq * a.Lk;
  if ((a.Lk & 7) == 0) {
    const int cpr = LK >> 3;
    for (int i = threadIdx.x; i < LQ * cpr; i += blockDim.x) {
      const int r = i / cpr, ch = i % cpr;
      const bool ok = r < a.Lq && ch * 8 < a.Lk;
      cp_async16(Ps + r * PLD + ch * 8, pg + (ok ? (int64_t)r * a.Lk + ch * 8 : 0), ok);
    }
  } else {
    for (int i = threadIdx.x; i < LQ * LK; i += blockDim.x) {
      const int r = i / LK, c = i % LK;
      Ps[r * PLD + c] = (r < a.Lq && c < a.Lk) ? pg[(int64_t)r * a.Lk + c] : __float2half(0.f);
    }
  }
  if (split) asm volatile("cp.async.commit_group;\n" ::);
  load_tile(Qs, a.q + (int64_t)b * a.Lq * a.ldq + h * kHd, a.ldq, a.Lq, LQ);
  load_tile(Ks, a.k + (int64_t)b * a.Lk * a.ldk + h * kHd, a.ldk, a.Lk, LK);
  asm volatile("cp.async.commit_group;\n" ::);
}

// 2 * max(QT, KT) warps in two concurrent roles per phase:
//   phase A  query warps: dP = dO V^T, dS = P (dP - rowsum(dP P)) * scale -> smem
//            key warps:   dV = P^T dO  (needs only P and dO: runs beside dS)
//   phase B  query warps: dQ = dS K
//            key warps:   dK = dS^T Q
// so the dependent chain per item is two 32-MMA steps, not two 64-MMA steps.
template <int QT, int KT, bool WAIT_QK = false>
__device__ __forceinline__ void attn_bwd_compute(const AttnBwdArgs& a, int bh, const __half* Qs,
                                                 const __half* Ks, const __half* Vs,
                                                 const __half* Os, const __half* Ps, __half* Ss,
                                                 float* cs) {
  constexpr int PLD = 16 * KT + kPad;
  constexpr int NW = QT > KT ? QT : KT;
  const int b = bh / a.H, h = bh % a.H;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const bool qw = w < NW;             // query-tile role (else key-tile role)
  const int tw = qw ? w : w - NW;     // tile index of this warp

  // ---- phase A ----
  if (qw && tw < QT) {
    float dp[2 * KT][4];
#pragma unroll
    for (int j = 0; j < 2 * KT; ++j) dp[j][0] = dp[j][1] = dp[j][2] = dp[j][3] = 0.f;
#pragma unroll
    for (int kk = 0; kk < kHd; kk += 16) {
      uint32_t af[4];
      frag_a(af, Os, kRow, 16 * tw, kk, lane);
#pragma unroll
      for (int nt = 0; nt < KT; ++nt) {
        uint32_t bf[4];
        frag_b_nk(bf, Vs, kRow, 16 * nt, kk, lane);
        mma16816(dp[2 * nt], af, bf[0], bf[1]);
        mma16816(dp[2 * nt + 1], af, bf[2], bf[3]);
      }
    }
    const int r0 = 16 * tw + g, r1 = r0 + 8;
    float s0 = 0.f, s1 = 0.f;
#pragma unroll
    for (int j = 0; j < 2 * KT; ++j) {
      const float2 x0 = unpack_h2(*reinterpret_cast<const uint32_t*>(Ps + r0 * PLD + 8 * j + 2 * t));
      const float2 x1 = unpack_h2(*reinterpret_cast<const uint32_t*>(Ps + r1 * PLD + 8 * j + 2 * t));
      s0 += dp[j][0] * x0.x + dp[j][1] * x0.y;
      s1 += dp[j][2] * x1.x + dp[j][3] * x1.y;
    }
    s0 += __shfl_xor_sync(0xffffffffu, s0, 1);
    s0 += __shfl_xor_sync(0xffffffffu, s0, 2);
    s1 += __shfl_xor_sync(0xffffffffu, s1, 1);
    s1 += __shfl_xor_sync(0xffffffffu, s1, 2);
#pragma unroll
    for (int j = 0; j < 2 * KT; ++j) {
      const float2 x0 = unpack_h2(*reinterpret_cast<const uint32_t*>(Ps + r0 * PLD + 8 * j + 2 * t));
      const float2 x1 = unpack_h2(*reinterpret_cast<const uint32_t*>(Ps + r1 * PLD + 8 * j + 2 * t));
      *reinterpret_cast<uint32_t*>(Ss + r0 * PLD + 8 * j + 2 * t) =
          pack_h2(x0.x * (dp[j][0] - s0) * a.scale, x0.y * (dp[j][1] - s0) * a.scale);
      *reinterpret_cast<uint32_t*>(Ss + r1 * PLD + 8 * j + 2 * t) =
          pack_h2(x1.x * (dp[j][2] - s1) * a.scale, x1.y * (dp[j][3] - s1) * a.scale);
    }
  } else if (!qw && tw < KT) {
    float dv[8][4];
#pragma unroll
    for (int j = 0; j < 8; ++j) dv[j][0] = dv[j][1] = dv[j][2] = dv[j][3] = 0.f;
#pragma unroll
    for (int qt = 0; qt < QT; ++qt) {
      uint32_t ap[4];
      frag_a_t(ap, Ps, PLD, 16 * tw, 16 * qt, lane);
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) {
        uint32_t bo[4];
        frag_b_kn(bo, Os, kRow, 16 * qt, 16 * nt, lane);
        mma16816(dv[2 * nt], ap, bo[0], bo[1]);
        mma16816(dv[2 * nt + 1], ap, bo[2], bo[3]);
      }
    }
    const int r0 = 16 * tw + g, r1 = r0 + 8;
    __half* d0 = a.dv + ((int64_t)b * a.Lk + r0) * a.lddv + h * kHd + 2 * t;
    __half* d1 = d0 + 8 * a.lddv;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (r0 < a.Lk) *reinterpret_cast<uint32_t*>(d0 + 8 * j) = pack_h2(dv[j][0], dv[j][1]);
      if (r1 < a.Lk) *reinterpret_cast<uint32_t*>(d1 + 8 * j) = pack_h2(dv[j][2], dv[j][3]);
    }
    if (a.csv) tile_colsum(dv, r0, a.Lk, cs + (2 * NW + tw) * 64, lane);
  }
  if (WAIT_QK) asm volatile("cp.async.wait_group 0;\n" ::);   // Q, K (second group)
  __syncthreads();
  // ---- phase B ----
  if (qw && tw < QT) {
    float dq[8][4];
#pragma unroll
    for (int j = 0; j < 8; ++j) dq[j][0] = dq[j][1] = dq[j][2] = dq[j][3] = 0.f;
#pragma unroll
    for (int kt = 0; kt < KT; ++kt) {
      uint32_t af[4];
      frag_a(af, Ss, PLD, 16 * tw, 16 * kt, lane);
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) {
        uint32_t bf[4];
        frag_b_kn(bf, Ks, kRow, 16 * kt, 16 * nt, lane);
        mma16816(dq[2 * nt], af, bf[0], bf[1]);
        mma16816(dq[2 * nt + 1], af, bf[2], bf[3]);
      }
    }
    const int r0 = 16 * tw + g, r1 = r0 + 8;
    __half* d0 = a.dq + ((int64_t)b * a.Lq + r0) * a.lddq + h * kHd + 2 * t;
    __half* d1 = d0 + 8 * a.lddq;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (r0 < a.Lq) *reinterpret_cast<uint32_t*>(d0 + 8 * j) = pack_h2(dq[j][0], dq[j][1]);
      if (r1 < a.Lq) *reinterpret_cast<uint32_t*>(d1 + 8 * j) = pack_h2(dq[j][2], dq[j][3]);
    }
    if (a.csq) tile_colsum(dq, r0, a.Lq, cs + tw * 64, lane);
  } else if (!qw && tw < KT) {
    float dk[8][4];
#pragma unroll
    for (int j = 0; j < 8; ++j) dk[j][0] = dk[j][1] = dk[j][2] = dk[j][3] = 0.f;
#pragma unroll
    for (int qt = 0; qt < QT; ++qt) {
      uint32_t as[4];
      frag_a_t(as, Ss, PLD, 16 * tw, 16 * qt, lane);
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) {
        uint32_t bq[4];
        frag_b_kn(bq, Qs, kRow, 16 * qt, 16 * nt, lane);
        mma16816(dk[2 * nt], as, bq[0], bq[1]);
        mma16816(dk[2 * nt + 1], as, bq[2], bq[3]);
      }
    }
    const int r0 = 16 * tw + g, r1 = r0 + 8;
    __half* d0 = a.dk + ((int64_t)b * a.Lk + r0) * a.lddk + h * kHd + 2 * t;
    __half* d1 = d0 + 8 * a.lddk;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (r0 < a.Lk) *reinterpret_cast<uint32_t*>(d0 + 8 * j) = pack_h2(dk[j][0], dk[j][1]);
      if (r1 < a.Lk) *reinterpret_cast<uint32_t*>(d1 + 8 * j) = pack_h2(dk[j][2], dk[j][3]);
    }
    if (a.csk) tile_colsum(dk, r0, a.Lk, cs + (NW + tw) * 64, lane);
  }
}

// one CTA per item (tiles up to 128 x 128)
template <int QT, int KT>
__global__ void __launch_bounds__(64 * (QT > KT ? QT : KT), (QT > KT ? QT : KT) <= 4 ? 4 : 1)
attn_bwd_kernel(AttnBwdArgs a) {
  constexpr int LQ = 16 * QT, LK = 16 * KT, PLD = LK + kPad;
  extern __shared__ __align__(16) __half sm[];
  __half* Qs = sm;                    // [LQ][72]
  __half* Ks = Qs + LQ * kRow;        // [LK][72]
  __half* Vs = Ks + LK * kRow;        // [LK][72]
  __half* Os = Vs + LK * kRow;        // dO [LQ][72]
  __half* Ps = Os + LQ * kRow;        // [LQ][LK+8]
  __half* Ss = Ps + LQ * PLD;         // dS [LQ][LK+8]
  float* cs = reinterpret_cast<float*>(Ss + LQ * PLD);   // [3][NW][64] bias-grad tile sums
  attn_bwd_issue(a, blockIdx.x, Qs, Ks, Vs, Os, Ps, LQ, LK, PLD, true);
  asm volatile("cp.async.wait_group 1;\n" ::);        // V, dO, P
  __syncthreads();
  attn_bwd_compute<QT, KT, true>(a, blockIdx.x, Qs, Ks, Vs, Os, Ps, Ss, cs);
  if (a.csq || a.csk || a.csv) {
    __syncthreads();
    attn_bwd_colsum_store<QT, KT>(a, blockIdx.x, cs);
  }
}

// Persistent, double-buffered (tiles up to 64 x 64, two CTAs per SM): a CTA
// walks items blockIdx.x, +gridDim.x, ... and the next item's five tiles load
// (cp.async) while the current one is computed and stored, so an SM's loads,
// tensor-core work and stores overlap instead of running as three phases.
template <int QT, int KT>
__global__ void __launch_bounds__(64 * (QT > KT ? QT : KT), 2)
attn_bwd_persist(AttnBwdArgs a, int nitems) {
  constexpr int LQ = 16 * QT, LK = 16 * KT, PLD = LK + kPad;
  constexpr int STAGE = 2 * LQ * kRow + 2 * LK * kRow + LQ * PLD;   // halves
  constexpr int NW = QT > KT ? QT : KT;
  extern __shared__ __align__(16) __half sm[];
  __half* Ss = sm + 2 * STAGE;
  float* cs0 = reinterpret_cast<float*>(Ss + LQ * PLD);   // [2 parity][3][NW][64]
  const bool colsum = a.csq || a.csk || a.csv;
  auto stage = [&](int s, __half*& Qs, __half*& Ks, __half*& Vs, __half*& Os, __half*& Ps) {
    Qs = sm + s * STAGE;
    Ks = Qs + LQ * kRow;
    Vs = Ks + LK * kRow;
    Os = Vs + LK * kRow;
    Ps = Os + LQ * kRow;
  };
  __half *Qs, *Ks, *Vs, *Os, *Ps;
  if ((int)blockIdx.x < nitems) {
    stage(0, Qs, Ks, Vs, Os, Ps);
    attn_bwd_issue(a, blockIdx.x, Qs, Ks, Vs, Os, Ps, LQ, LK, PLD);
  }
  int k = 0;
  for (int item = blockIdx.x; item < nitems; item += gridDim.x, ++k) {
    const int nxt = item + gridDim.x;
    if (nxt < nitems) {
      stage((k + 1) & 1, Qs, Ks, Vs, Os, Ps);
      attn_bwd_issue(a, nxt, Qs, Ks, Vs, Os, Ps, LQ, LK, PLD);
      asm volatile("cp.async.wait_group 1;\n" ::);
    } else {
      asm volatile("cp.async.wait_group 0;\n" ::);
    }
    __syncthreads();
    stage(k & 1, Qs, Ks, Vs, Os, Ps);
    float* cs = cs0 + (k & 1) * 3 * NW * 64;
    attn_bwd_compute<QT, KT>(a, item, Qs, Ks, Vs, Os, Ps, Ss, cs);
    __syncthreads();   // stage k&1 and dS are free for the item after next
    // the tile sums are parity-buffered, so this fold overlaps the next item
    if (colsum) attn_bwd_colsum_store<QT, KT>(a, item, cs);
  }
}

inline size_t fwd_smem(int qt, int kt) {
  return (size_t)(16 * qt * kRow + 2 * 16 * kt * kRow + 16 * qt * (16 * kt + kPad)) * 2;
}
inline size_t bwd_smem(int qt, int kt) {
  const int nw = qt > kt ? qt : kt;
  return (size_t)(2 * 16 * qt * kRow + 2 * 16 * kt * kRow + 2 * 16 * qt * (16 * kt + kPad)) * 2 +
         (size_t)3 * nw * 64 * 4;
}

template <int QT, int KT>
int launch_fwd(const AttnArgs& a, int nbh, cudaStream_t st) {
  const size_t sm = fwd_smem(QT, KT);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(attn_fwd_kernel<QT, KT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    attr = true;
  }
  attn_fwd_kernel<QT, KT><<<nbh, 32 * QT, sm, st>>>(a);
  return check_launch("attention_fwd");
}

template <int QT, int KT>
int launch_bwd(const AttnBwdArgs& a, int nbh, cudaStream_t st) {
  if constexpr (QT <= 4 && KT <= 4) {
    static const bool persist = [] {
      const char* e = getenv("LS2_ATTN_PERSIST");
      return !(e && e[0] == '0');
    }();
    // persistent only while the items roughly fill the resident CTA slots: with
    // many small items (short sequences, e.g. L = 8 -> 4096 (batch, head) pairs)
    // one CTA per item keeps them all in flight instead of serialising ~14 per CTA
    if (persist && nbh <= 4 * kNumSMs) {
      constexpr int LQ = 16 * QT, LK = 16 * KT, PLD = LK + kPad;
      constexpr int NW = QT > KT ? QT : KT;
      const size_t sm = (size_t)(2 * (2 * LQ * kRow + 2 * LK * kRow + LQ * PLD) + LQ * PLD) * 2 +
                        (size_t)2 * 3 * NW * 64 * 4;
      static bool attr = false;
      if (!attr) {
        cudaFuncSetAttribute(attn_bwd_persist<QT, KT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)sm);
        attr = true;
      }
      const int grid = nbh < 2 * kNumSMs ? nbh : 2 * kNumSMs;
      attn_bwd_persist<QT, KT><<<grid, 64 * (QT > KT ? QT : KT), sm, st>>>(a, nbh);
      return check_launch("attention_bwd");
    }
  }
  const size_t sm = bwd_smem(QT, KT);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(attn_bwd_kernel<QT, KT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    attr = true;
  }
  attn_bwd_kernel<QT, KT><<<nbh, 64 * (QT > KT ? QT : KT), sm, st>>>(a);
  return check_launch("attention_bwd");
}

#define LS2_ATTN_TILES(X, ...)                                                             \
  X(1, 1, __VA_ARGS__) X(1, 2, __VA_ARGS__) X(1, 4, __VA_ARGS__) X(1, 8, __VA_ARGS__)      \
  X(2, 1, __VA_ARGS__) X(2, 2, __VA_ARGS__) X(2, 4, __VA_ARGS__) X(2, 8, __VA_ARGS__)      \
  X(4, 1, __VA_ARGS__) X(4, 2, __VA_ARGS__) X(4, 4, __VA_ARGS__) X(4, 8, __VA_ARGS__)      \
  X(8, 1, __VA_ARGS__) X(8, 2, __VA_ARGS__) X(8, 4, __VA_ARGS__) X(8, 8, __VA_ARGS__)      \
  X(3, 3, __VA_ARGS__)

// 16-row tile counts per (lq, lk): powers of two, plus 48 x 48 for the square
// 33..48 buckets of length-bucketed batches (L = 36 would otherwise pad to 64
// and spend 1.8x the work)
inline int tiles_of(int L) { return L <= 16 ? 1 : L <= 32 ? 2 : L <= 64 ? 4 : 8; }
inline void tile_pair(int lq, int lk, int& qt, int& kt) {
  qt = tiles_of(lq);
  kt = tiles_of(lk);
  if (qt == 4 && kt == 4 && lq <= 48 && lk <= 48) qt = kt = 3;
}

}  // namespace ls2

using namespace ls2;

extern "C" {

int ls2_attention_supported(int64_t lq, int64_t lk, int64_t hd, int dtype) {
  return dtype == LS2_F16 && hd == kHd && lq >= 1 && lk >= 1 && lq <= 128 && lk <= 128;
}

int ls2_attention_fwd(const void* q, int64_t ldq, const void* k, int64_t ldk, const void* v,
                      int64_t ldv, void* probs, void* o, int64_t ldo, int64_t batch,
                      int64_t heads, int64_t lq, int64_t lk, int64_t hd, int mask_kind,
                      const int64_t* lens, double scale, void* stream) {
  if (!ls2_attention_supported(lq, lk, hd, LS2_F16))
    return fail(LS2_ERR_SHAPE, "attention_fwd: needs fp16, hd == 64, L <= 128");
  if (mask_kind == LS2_MASK_PADDING && !lens) return fail(LS2_ERR_SHAPE, "attention: no lens");
  if (mask_kind == LS2_MASK_DENSE) return fail(LS2_ERR_SHAPE, "attention: dense masks unsupported");
  AttnArgs a{(const __half*)q, (const __half*)k, (const __half*)v, ldq, ldk, ldv,
             (__half*)probs, (__half*)o, ldo, (int)heads, (int)lq, (int)lk, mask_kind, lens,
             (float)scale};
  int qt, kt;
  tile_pair((int)lq, (int)lk, qt, kt);
  const int nbh = (int)(batch * heads);
  cudaStream_t st = as_stream(stream);
#define LS2_FWD_CASE(QT_, KT_, ...) if (qt == QT_ && kt == KT_) return launch_fwd<QT_, KT_>(a, nbh, st);
  LS2_ATTN_TILES(LS2_FWD_CASE, 0)
#undef LS2_FWD_CASE
  return fail(LS2_ERR_SHAPE, "attention_fwd: no tile config");
}

int ls2_attention_bwd(const void* q, int64_t ldq, const void* k, int64_t ldk, const void* v,
                      int64_t ldv, const void* probs, const void* dout, int64_t lddo, void* dq,
                      int64_t lddq, void* dk, int64_t lddk, void* dv, int64_t lddv,
                      int64_t batch, int64_t heads, int64_t lq, int64_t lk, int64_t hd,
                      double scale, void* stream) {
  return ls2_attention_bwd_bias(q, ldq, k, ldk, v, ldv, probs, dout, lddo, dq, lddq, dk, lddk, dv,
                                lddv, batch, heads, lq, lk, hd, scale, nullptr, 0, nullptr, 0,
                                nullptr, 0, stream);
}

int ls2_attention_bwd_bias(const void* q, int64_t ldq, const void* k, int64_t ldk, const void* v,
                           int64_t ldv, const void* probs, const void* dout, int64_t lddo,
                           void* dq, int64_t lddq, void* dk, int64_t lddk, void* dv, int64_t lddv,
                           int64_t batch, int64_t heads, int64_t lq, int64_t lk, int64_t hd,
                           double scale, double* csq, int64_t ldcsq, double* csk, int64_t ldcsk,
                           double* csv, int64_t ldcsv, void* stream) {
  if (!ls2_attention_supported(lq, lk, hd, LS2_F16))
    return fail(LS2_ERR_SHAPE, "attention_bwd: needs fp16, hd == 64, L <= 128");
  AttnBwdArgs a{(const __half*)q, (const __half*)k, (const __half*)v, (const __half*)probs,
                (const __half*)dout, ldq, ldk, ldv, lddo, (__half*)dq, (__half*)dk, (__half*)dv,
                lddq, lddk, lddv, (int)heads, (int)lq, (int)lk, (float)scale,
                csq, csk, csv, ldcsq, ldcsk, ldcsv};
  int qt, kt;
  tile_pair((int)lq, (int)lk, qt, kt);
  const int nbh = (int)(batch * heads);
  cudaStream_t st = as_stream(stream);
#define LS2_BWD_CASE(QT_, KT_, ...) if (qt == QT_ && kt == KT_) return launch_bwd<QT_, KT_>(a, nbh, st);
  LS2_ATTN_TILES(LS2_BWD_CASE, 0)
#undef LS2_BWD_CASE
  return fail(LS2_ERR_SHAPE, "attention_bwd: no tile config");
}

}  // extern "C"
