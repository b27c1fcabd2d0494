// Fused short-sequence attention on the 5th-generation tensor cores
// (tcgen05 + TMEM + TMA), fp16, head dim 64, Lq, Lk <= 64.
//
// Replaces, per attention block, the reference's chain (F/model.py:362-376 and
// :482-495): scores = Q K^T * 1/sqrt(hd); softmax_forward(mask)
// (F/kernels.py:277-307); ctx = P V; merge heads — and the backward
// dP = dctx V^T; softmax_backward (F/gradients.py:77-100) * 1/sqrt(hd);
// dQ = dS K; dK = dS^T Q; dV = P^T dctx.
//
// Work unit ("tile"): one head of G = floor(64 / max(Lq, Lk)) consecutive
// sequences.  Their rows are packed into one 64-row operand tile (a 3-D TMA box
// (64 columns, L rows, G sequences) over the [B, L, ld] projection buffer, with
// the 128-byte swizzle UMMA reads directly); cross-sequence products are masked,
// so short buckets (L = 8 -> 8 sequences per tile) keep the tensor-core tiles
// full instead of launching one tiny item per (batch, head).
//
// One CTA (4 warps) owns TWO tiles ("slots").  Every product is a UMMA
// M64 x N64 x K16 chain issued by one thread into tensor memory; slot s's
// accumulators sit at TMEM lane offset 16*s, so with the M = 64 data-path layout
// (tile row 16w + i -> TMEM lane 32w + i) lane i of warp w reads row 16w + (i&15)
// of slot i >> 4 with one tcgen05.ld — all 128 threads have a row to work on.
//
// Forward:  S = Q K^T (TMEM) -> per-row masked softmax in registers -> P (fp16,
//           swizzled smem) -> O = P V (TMEM) -> fp16 -> TMA store;
//           per-row (max, 1/sum) go to `stats` instead of the probabilities.
// Backward: S = Q K^T and dP = dO V^T (TMEM) -> P recomputed bit-identically from
//           S and the stats -> dS = P (dP - rowsum(dP P)) * scale -> P, dS (smem)
//           -> dV = P^T dO, dQ = dS K, dK = dS^T Q (TMEM) -> fp16 -> TMA store;
//           optional per-sequence column sums of the stored dQ / dK / dV (the
//           projection biases' gradient partials, f64 rows per batch).
// Per (batch, head) HBM traffic: fwd reads Q, K, V and writes O (+8 B per row of
// stats); bwd reads Q, K, V, dO (+ stats) and writes dQ, dK, dV — the [L x L]
// probabilities never touch HBM.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>

#include "common.cuh"

namespace ls2 {
namespace tc {
PFN_cuTensorMapEncodeTiled_v12000 encode_fn();
}
namespace atc {

constexpr int kTile = 64 * 128;      // one 64-row x 64-column fp16 operand tile (8 KB)
constexpr int kThreads = 256;

struct Args {
  int H, Lq, Lk, G, B, ntiles, mask;
  const int64_t* lens;
  float scale;                       // scale * log2(e): the softmax runs in the log2 domain
  float dscale;                      // scale itself (dS = P (dP - rowsum) * scale)
  float2* stats;                     // [B][H][Lq] (row max in the log2 domain, 1 / row sum)
  uint32_t id_s, id64_km, id64_mm, id_cs;   // instruction descriptors (M, N, A / B majors)
  uint32_t id128_pv, id128_mm;              // M = 128, N = 64: A K-major / A MN-major, B MN-major
  double *csq, *csk, *csv;
  int64_t ldcsq, ldcsk, ldcsv;
  unsigned long long* trace;         // optional phase timestamps [grid][16] (ls2_attention_tc_trace)
};

__device__ __forceinline__ void stamp(const Args& a, int k) {
  if (a.trace && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    a.trace[blockIdx.x * 16 + k] = t;
  }
}

__device__ __forceinline__ uint32_t sptr(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sptr(b)), "r"(n));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sptr(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n W_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra W_%=;\n}" ::"r"(sptr(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int c0, int c1,
                                            int c2, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(sptr(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(sptr(bar))
      : "memory");
}
__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, int c0, int c1, int c2,
                                             const void* src) {
  asm volatile(
      "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(
          reinterpret_cast<uint64_t>(map)),
      "r"(c0), "r"(c1), "r"(c2), "r"(sptr(src))
      : "memory");
}
__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tc_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// UMMA shared-memory descriptor, 128-byte swizzle (1 KB atoms of 8 rows x 128 B)
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
// a 64 x 64 tile stored [row][64 contiguous] used as a K-major operand (rows = M/N,
// contiguous = K): the K16 step moves 32 B inside the swizzle atom
__device__ __forceinline__ uint64_t kdesc(uint32_t base, int kk) {
  return sdesc(base + kk * 32, 16, 1024);
}
// the same tile used as an MN-major operand (rows = K, contiguous = M/N): the
// K16 step moves 16 rows = 2 KB
__device__ __forceinline__ uint64_t mdesc(uint32_t base, int kk) {
  return sdesc(base + kk * 2048, kTile, 1024);
}

__device__ __forceinline__ void commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   sptr(bar))
               : "memory");
}

// 32 fp32 columns of this thread's TMEM lane
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&f)[32]) {
  uint32_t v[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),
        "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]),
        "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
        "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]),
        "=r"(v[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    asm volatile("" : "+r"(v[j]));   // no use may move above the wait
    f[j] = __uint_as_float(v[j]);
  }
}

__device__ __forceinline__ uint32_t pack_h2(float lo, float hi) {
  __half2 h = __floats2half2_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&h);
}
__device__ __forceinline__ float2 unpack_h2(uint32_t v) {
  __half2 h = *reinterpret_cast<__half2*>(&v);
  return __half22float2(h);
}
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// byte offset of 16-byte chunk ch of row r in a 128-byte-swizzled tile
__device__ __forceinline__ int swz(int r, int ch) { return r * 128 + ((ch ^ (r & 7)) << 4); }

// zero rows [r0, 64) of a tile (rows no TMA box covers: the UMMAs read them)
__device__ __forceinline__ void zero_tail(uint8_t* tile, int r0) {
  for (int i = r0 * 8 + threadIdx.x; i < 64 * 8; i += kThreads)
    *reinterpret_cast<uint4*>(tile + i * 16) = make_uint4(0, 0, 0, 0);
}

// Tile layout.  The two slots' operand tiles sit back to back ([X0 | X1], 128
// rows), so every product is ONE M = 128 UMMA chain for both slots:
//   S = [Q0; Q1] [K0; K1]^T and dP = [dO0; dO1] [V0; V1]^T  (N = 128; the useful
//       blocks are the diagonal ones, slot s at columns 64s ..)
//   O = Pbd [V0; V1], dV = Pbd^T [dO0; dO1], dQ = dSbd [K0; K1], dK = dSbd^T [Q0; Q1]
//       (K = 128), where Xbd = [[X0, 0], [0, X1]] is a block-diagonal buffer: two
//       16 KB column chunks (chunk c = keys of slot c), the off-diagonal halves
//       zeroed once.  One buffer serves both operand majors (K-major chunks for
//       O / dQ, MN-major blocks LBO = 16 KB apart for dV / dK).
// Tensor memory (M = 128): tile row m <-> lane m.  Warp w reads lane quadrant
// q = w & 3 (rows 32q .. 32q+31, slot = q >> 1) and column half h2 = w >> 2;
// warps w and w ^ 4 share rows and meet at named barrier 1 + q.
constexpr int kPair = 2 * kTile;     // [X0 | X1]: 128 rows, 16 KB

// MN-major step kk of a 128-row (K) operand whose two 64-wide M blocks are
// 16 KB apart ([X0 | X1] pair regions side by side)
__device__ __forceinline__ uint64_t mdesc_bd(uint32_t base, int kk) {
  return sdesc(base + kk * 2048, kPair, 1024);
}

enum { KM = 0, MN = 1 };

template <int AM, int BM, int NK>
__device__ __forceinline__ void mma128(uint32_t d, uint32_t a, uint32_t b, uint32_t idesc) {
#pragma unroll
  for (int kk = 0; kk < NK; ++kk) {
    const uint64_t da = AM == KM ? kdesc(a, kk) : mdesc_bd(a, kk);
    const uint64_t db = BM == KM ? kdesc(b, kk) : mdesc(b, kk);
    const uint32_t acc = kk ? 1u : 0u;
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
        " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d),
        "l"(da), "l"(db), "r"(idesc), "r"(acc)
        : "memory");
  }
}

// per-slot M = 64 product (K = 64): D[tmem + lane offset 16 s] = A_s B_s
template <int AM, int BM>
__device__ __forceinline__ void mma64(uint32_t d, uint32_t a, uint32_t b, uint32_t idesc) {
#pragma unroll
  for (int kk = 0; kk < 4; ++kk) {
    const uint64_t da = AM == KM ? kdesc(a, kk) : mdesc(a, kk);
    const uint64_t db = BM == KM ? kdesc(b, kk) : mdesc(b, kk);
    const uint32_t acc = kk ? 1u : 0u;
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
        " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d),
        "l"(da), "l"(db), "r"(idesc), "r"(acc)
        : "memory");
  }
}

// Reading an M = 64 result (slot s at TMEM lane offset 16 s; tile row 16 q + i at
// lane 32 q + i): lane i of a quadrant-q warp holds row 16 q + (i & 15) of slot
// i >> 4, i.e. row m64 of a [X0 | X1] staging region
__device__ __forceinline__ int m64_row() {
  const int lane = threadIdx.x & 31, q = (threadIdx.x >> 5) & 3;
  return 64 * (lane >> 4) + 16 * q + (lane & 15);
}

struct RowInfo {
  int m, slot, rin, g, pos, b, h, j, q, half, idx;
  bool ok;
  int lo, hi;
  int64_t len;
};
// indices of this thread's row; the padding length is only loaded here (its
// latency overlaps the operand loads) and applied by row_mask after the first wait
__device__ __forceinline__ RowInfo row_info(const Args& a, int tile0, bool has1) {
  RowInfo r;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  r.q = warp & 3;
  r.half = warp >> 2;
  r.idx = r.q * 32 + lane;
  r.m = 32 * r.q + lane;
  r.slot = r.m >> 6;
  r.rin = r.m & 63;
  const int t = tile0 + r.slot;
  r.h = t % a.H;
  r.j = t / a.H;
  r.g = r.rin / a.Lq;
  r.pos = r.rin - r.g * a.Lq;
  r.b = r.j * a.G + r.g;
  r.ok = (r.slot == 0 || has1) && r.g < a.G && r.b < a.B;
  r.len = (r.ok && a.mask == LS2_MASK_PADDING) ? __ldg(a.lens + r.b) : (int64_t)a.Lk;
  return r;
}
// unmasked keys of the row, relative to this thread's 32 columns: [lo, hi)
__device__ __forceinline__ void row_mask(const Args& a, RowInfo& r) {
  int n = r.len < a.Lk ? (int)r.len : a.Lk;
  if (a.mask == LS2_MASK_CAUSAL) n = r.pos + 1 < n ? r.pos + 1 : n;
  r.lo = r.g * a.Lk - 32 * r.half;
  r.hi = r.ok ? r.lo + n : r.lo;
}

// exchange a per-row partial with the partner warp (same rows, other column half)
__device__ __forceinline__ float partner(float* buf, const RowInfo& r, float v) {
  buf[r.half * 128 + r.idx] = v;
  asm volatile("bar.sync %0, 64;" ::"r"(1 + r.q) : "memory");
  return buf[(r.half ^ 1) * 128 + r.idx];
}

// 16-byte chunk stores of this thread's 32 columns of row m into a 128-row region
// (a [X0 | X1] pair, or chunk c of a block-diagonal buffer)
__device__ __forceinline__ void st_cols(uint8_t* region, int m, int half, const uint32_t (&w)[16]) {
#pragma unroll
  for (int c = 0; c < 4; ++c)
    *reinterpret_cast<uint4*>(region + swz(m, 4 * half + c)) =
        make_uint4(w[4 * c], w[4 * c + 1], w[4 * c + 2], w[4 * c + 3]);
}
__device__ __forceinline__ void st_cols_f(uint8_t* region, int m, int half, const float (&f)[32]) {
  uint32_t w[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) w[j] = pack_h2(f[2 * j], f[2 * j + 1]);
  st_cols(region, m, half, w);
}

// rows the TMA boxes leave untouched must read as zero (the block-diagonal
// products multiply them by zero, and 0 * garbage may be NaN): each slot's tail
// rows past G*L, and every tile of a missing second slot
__device__ __forceinline__ void zero_unloaded(uint8_t* pair, int rows, bool has1) {
  if (rows < 64) zero_tail(pair, rows);
  zero_tail(pair + kTile, has1 ? rows : 0);
}

__global__ void __launch_bounds__(kThreads, 3) attn_tc_fwd_kernel(
    const __grid_constant__ CUtensorMap mq, const __grid_constant__ CUtensorMap mk,
    const __grid_constant__ CUtensorMap mv, const __grid_constant__ CUtensorMap mo,
    const __grid_constant__ Args a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                           ~uintptr_t(1023));
  uint8_t* Qs = sm;                  // [Q0 | Q1], doubles as the O staging
  uint8_t* Ks = sm + kPair;
  uint8_t* Vs = sm + 2 * kPair;
  uint8_t* Pt = sm + 3 * kPair;      // [P0 | P1]
  __shared__ __align__(8) uint64_t bar_qk, bar_v, bar_s, bar_o;
  __shared__ uint32_t tmem_base;
  __shared__ float xm[256], xz[256];
  const int warp = threadIdx.x >> 5;
  const int tile0 = 2 * blockIdx.x;
  const bool has1 = tile0 + 1 < a.ntiles;
  const int nb = has1 ? 2 : 1;
  const int qrows = a.G * a.Lq, krows = a.G * a.Lk;
  stamp(a, 0);

  if (threadIdx.x == 0) {            // barriers, then the operand loads right away
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mq)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mk)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mv)) : "memory");
    mbar_init(&bar_qk, 1);
    mbar_init(&bar_v, 1);
    mbar_init(&bar_s, 1);
    mbar_init(&bar_o, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    mbar_expect_tx(&bar_qk, (uint32_t)(nb * (qrows + krows) * 128));
    for (int s = 0; s < nb; ++s) {
      const int t = tile0 + s, h = t % a.H, b0 = (t / a.H) * a.G;
      tma_load_3d(Qs + s * kTile, &mq, h * 64, 0, b0, &bar_qk);
      tma_load_3d(Ks + s * kTile, &mk, h * 64, 0, b0, &bar_qk);
    }
    mbar_expect_tx(&bar_v, (uint32_t)(nb * krows * 128));
    for (int s = 0; s < nb; ++s) {
      const int t = tile0 + s, h = t % a.H, b0 = (t / a.H) * a.G;
      tma_load_3d(Vs + s * kTile, &mv, h * 64, 0, b0, &bar_v);
    }
  }
  if (warp == 1) {   // S (cols 0-127), then O (0-63, per-slot M = 64 layout); warp 1, so
                     // the allocation runs beside warp 0's barrier setup and TMA issue
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(
        sptr(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  zero_unloaded(Qs, qrows, has1);
  zero_unloaded(Ks, krows, has1);
  zero_unloaded(Vs, krows, has1);
  fence_async_smem();
  tc_before();
  __syncthreads();
  tc_after();
  const uint32_t tmem = tmem_base;
  stamp(a, 1);
  // after the fences above (which would wait for them): the padding length load
  // overlaps the operand loads
  RowInfo r = row_info(a, tile0, has1);

  if (threadIdx.x == 0) {
    mbar_wait(&bar_qk, 0);
    stamp(a, 2);
    tc_after();
    mma128<KM, KM, 4>(tmem, sptr(Qs), sptr(Ks), a.id_s);
    commit(&bar_s);
  }
  __syncwarp();

  const uint32_t tlane = tmem + ((uint32_t)(32 * r.q) << 16);
  mbar_wait(&bar_s, 0);
  stamp(a, 3);
  tc_after();
  row_mask(a, r);
  float x[32];
  tmem_ld32(tlane + 64 * r.slot + 32 * r.half, x);
  // masked softmax over the row (log2 domain: t = s * scale * log2 e)
  float m = -INFINITY;
#pragma unroll
  for (int c = 0; c < 32; ++c) {
    x[c] = (c >= r.lo && c < r.hi) ? __fmul_rn(x[c], a.scale) : -INFINITY;
    m = fmaxf(m, x[c]);
  }
  m = fmaxf(m, partner(xm, r, m));
  float z = 0.f;
#pragma unroll
  for (int c = 0; c < 32; ++c) {
    x[c] = x[c] == -INFINITY ? 0.f : ex2(__fsub_rn(x[c], m));
    z += x[c];
  }
  z += partner(xz, r, z);
  const float iz = z > 0.f ? 1.f / z : 0.f;
  {
    uint32_t w[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) w[j] = pack_h2(__fmul_rn(x[2 * j], iz), __fmul_rn(x[2 * j + 1], iz));
    st_cols(Pt, r.m, r.half, w);
  }
  if (r.ok && r.half == 0) a.stats[((int64_t)r.b * a.H + r.h) * a.Lq + r.pos] = make_float2(m, iz);
  fence_async_smem();
  tc_before();
  __syncthreads();
  stamp(a, 4);

  if (threadIdx.x == 0) {
    tc_after();
    mbar_wait(&bar_v, 0);
    for (int s2 = 0; s2 < nb; ++s2)       // O_s = P_s V_s into the (read) S columns
      mma64<KM, MN>(tmem + ((uint32_t)(16 * s2) << 16), sptr(Pt + s2 * kTile), sptr(Vs + s2 * kTile),
                    a.id64_km);
    commit(&bar_o);
  }
  __syncwarp();
  mbar_wait(&bar_o, 0);
  stamp(a, 5);
  tc_after();
  tmem_ld32(tlane + 32 * r.half, x);
  st_cols_f(Qs, m64_row(), r.half, x);   // Q is dead once S completed
  fence_async_smem();
  tc_before();
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int s2 = 0; s2 < nb; ++s2) {
      const int t = tile0 + s2, h = t % a.H, b0 = (t / a.H) * a.G;
      tma_store_3d(&mo, h * 64, 0, b0, Qs + s2 * kTile);
    }
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    stamp(a, 6);
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
  }
  __syncwarp();
  if (warp == 1) {
    tc_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tmem));
  }
  stamp(a, 7);
}

__global__ void __launch_bounds__(kThreads, 2) attn_tc_bwd_kernel(
    const __grid_constant__ CUtensorMap mq, const __grid_constant__ CUtensorMap mk,
    const __grid_constant__ CUtensorMap mv, const __grid_constant__ CUtensorMap mdo,
    const __grid_constant__ CUtensorMap mdq, const __grid_constant__ CUtensorMap mdk,
    const __grid_constant__ CUtensorMap mdv, const __grid_constant__ Args a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                           ~uintptr_t(1023));
  uint8_t* Qs = sm;                  // [Q0 | Q1]; Q, K, V double as dQ, dK, dV staging
  uint8_t* Ks = sm + kPair;
  uint8_t* Vs = sm + 2 * kPair;
  uint8_t* Os = sm + 3 * kPair;      // dO
  uint8_t* Pt = sm + 4 * kPair;      // [P0 | P1]
  uint8_t* St = sm + 5 * kPair;      // [dS0 | dS1]
  uint8_t* Ib = sm + 6 * kPair;      // slot indicator [16 x 128] (4 KB), the column-sum B operand
  __shared__ __align__(8) uint64_t bar_ld, bar_ov, bar_1, bar_1b, bar_dv, bar_2, bar_cs;
  __shared__ uint32_t tmem_base;
  __shared__ float xr[256];
  const int warp = threadIdx.x >> 5;
  const int tile0 = 2 * blockIdx.x;
  const bool has1 = tile0 + 1 < a.ntiles;
  const int nb = has1 ? 2 : 1;
  const int qrows = a.G * a.Lq, krows = a.G * a.Lk;
  stamp(a, 0);

  if (threadIdx.x == 0) {            // barriers, then the operand loads right away
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mq)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mk)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mdo)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mv)) : "memory");
    mbar_init(&bar_ld, 1);
    mbar_init(&bar_ov, 1);
    mbar_init(&bar_1, 1);
    mbar_init(&bar_1b, 1);
    mbar_init(&bar_dv, 1);
    mbar_init(&bar_2, 1);
    mbar_init(&bar_cs, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    // Q, K first (S = Q K^T starts on them), then dO, V (dP = dO V^T)
    mbar_expect_tx(&bar_ld, (uint32_t)(nb * (qrows + krows) * 128));
    for (int s = 0; s < nb; ++s) {
      const int t = tile0 + s, h = t % a.H, b0 = (t / a.H) * a.G;
      tma_load_3d(Qs + s * kTile, &mq, h * 64, 0, b0, &bar_ld);
      tma_load_3d(Ks + s * kTile, &mk, h * 64, 0, b0, &bar_ld);
    }
    mbar_expect_tx(&bar_ov, (uint32_t)(nb * (qrows + krows) * 128));
    for (int s = 0; s < nb; ++s) {
      const int t = tile0 + s, h = t % a.H, b0 = (t / a.H) * a.G;
      tma_load_3d(Os + s * kTile, &mdo, h * 64, 0, b0, &bar_ov);
      tma_load_3d(Vs + s * kTile, &mv, h * 64, 0, b0, &bar_ov);
    }
    stamp(a, 8);
  }
  if (warp == 1) {   // S (0-127), dP (128-255); then dV, dQ, dK (0-191, M = 64 layout)
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(
        sptr(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  stamp(a, 9);
  zero_unloaded(Qs, qrows, has1);
  zero_unloaded(Os, qrows, has1);
  zero_unloaded(Ks, krows, has1);
  zero_unloaded(Vs, krows, has1);
  {   // indicator: K chunk c (rows of slot c) has ones in row c, zeros elsewhere
    const int i = threadIdx.x;                         // 256 x 16 B = the 4 KB
    const int c = i >> 7, row = (i >> 3) & 15;
    const uint32_t one = row == c ? 0x3C003C00u : 0u;  // fp16 1.0 pairs
    *reinterpret_cast<uint4*>(Ib + i * 16) = make_uint4(one, one, one, one);
  }
  stamp(a, 10);
  fence_async_smem();
  tc_before();
  __syncthreads();
  tc_after();
  const uint32_t tmem = tmem_base;
  stamp(a, 1);
  // after the fences above (which would wait for them): the padding length and
  // softmax statistics loads overlap the operand loads
  RowInfo r = row_info(a, tile0, has1);
  float2 st = make_float2(0.f, 0.f);
  if (r.ok) st = __ldg(a.stats + ((int64_t)r.b * a.H + r.h) * a.Lq + r.pos);

  if (threadIdx.x == 0) {
    mbar_wait(&bar_ld, 0);
    stamp(a, 2);
    tc_after();
    mma128<KM, KM, 4>(tmem, sptr(Qs), sptr(Ks), a.id_s);          // S
    commit(&bar_1);
    mbar_wait(&bar_ov, 0);
    tc_after();
    mma128<KM, KM, 4>(tmem + 128, sptr(Os), sptr(Vs), a.id_s);    // dP
    commit(&bar_1b);
  }
  __syncwarp();

  const uint32_t tlane = tmem + ((uint32_t)(32 * r.q) << 16);
  mbar_wait(&bar_1, 0);
  stamp(a, 3);
  tc_after();
  row_mask(a, r);
  float x[32];
  tmem_ld32(tlane + 64 * r.slot + 32 * r.half, x);
  uint32_t pw[16];                   // P of this half row, fp16 pairs (as the forward stored it)
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    float p2[2];
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int c = 2 * j + e;
      p2[e] = (c >= r.lo && c < r.hi) ? __fmul_rn(ex2(__fsub_rn(__fmul_rn(x[c], a.scale), st.x)), st.y)
                                      : 0.f;
    }
    pw[j] = pack_h2(p2[0], p2[1]);
  }
  st_cols(Pt, r.m, r.half, pw);
  // P complete, S read: dV = P^T dO (M = 64 per slot, TMEM columns 0-63, which
  // S no longer needs) runs while the threads form dS
  fence_async_smem();
  tc_before();
  __syncthreads();
  if (threadIdx.x == 0) {
    tc_after();
    for (int s2 = 0; s2 < nb; ++s2)
      mma64<MN, MN>(tmem + ((uint32_t)(16 * s2) << 16), sptr(Pt + s2 * kTile), sptr(Os + s2 * kTile),
                    a.id64_mm);
    commit(&bar_dv);
  }
  __syncwarp();
  mbar_wait(&bar_1b, 0);
  tc_after();
  tmem_ld32(tlane + 128 + 64 * r.slot + 32 * r.half, x);    // dP
  float rs = 0.f;
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    const float2 p = unpack_h2(pw[j]);
    rs += x[2 * j] * p.x + x[2 * j + 1] * p.y;
  }
  rs += partner(xr, r, rs);
  {
    const float ds = a.dscale;
    uint32_t dw[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const float2 p = unpack_h2(pw[j]);
      dw[j] = pack_h2(p.x * (x[2 * j] - rs) * ds, p.y * (x[2 * j + 1] - rs) * ds);
    }
    st_cols(St, r.m, r.half, dw);
  }
  // dV (done while dS was formed) -> fp16 staging in V's tile (dP has been read)
  const int mr = m64_row();
  mbar_wait(&bar_dv, 0);
  tc_after();
  tmem_ld32(tlane + 32 * r.half, x);
  st_cols_f(Vs, mr, r.half, x);      // dV
  fence_async_smem();
  tc_before();
  __syncthreads();                   // dS and the dV staging complete, dP read
  stamp(a, 4);
  if (threadIdx.x == 0) {
    tc_after();
    for (int s2 = 0; s2 < nb; ++s2) {   // per-slot M = 64 products, slot s at lane offset 16 s
      const uint32_t d = tmem + ((uint32_t)(16 * s2) << 16);
      mma64<KM, MN>(d + 64, sptr(St + s2 * kTile), sptr(Ks + s2 * kTile), a.id64_km);  // dQ = dS K
      mma64<MN, MN>(d + 128, sptr(St + s2 * kTile), sptr(Qs + s2 * kTile), a.id64_mm); // dK = dS^T Q
    }
    commit(&bar_2);
    for (int s = 0; s < nb; ++s) {       // dV leaves while dQ, dK run
      const int t = tile0 + s, h = t % a.H, b0 = (t / a.H) * a.G;
      tma_store_3d(&mdv, h * 64, 0, b0, Vs + s * kTile);
    }
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  }
  __syncwarp();
  mbar_wait(&bar_2, 0);
  stamp(a, 5);
  tc_after();
  tmem_ld32(tlane + 64 + 32 * r.half, x);
  st_cols_f(Qs, mr, r.half, x);      // dQ (row = query)
  tmem_ld32(tlane + 128 + 32 * r.half, x);
  st_cols_f(Ks, mr, r.half, x);      // dK (row = key)
  fence_async_smem();
  tc_before();
  __syncthreads();
  stamp(a, 6);
  if (threadIdx.x == 0) {
    for (int s = 0; s < nb; ++s) {
      const int t = tile0 + s, h = t % a.H, b0 = (t / a.H) * a.G;
      tma_store_3d(&mdq, h * 64, 0, b0, Qs + s * kTile);
      tma_store_3d(&mdk, h * 64, 0, b0, Ks + s * kTile);
    }
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  }
  if (a.csq || a.csk || a.csv) {
    // bias-gradient partials on the tensor cores: column sums of the staged fp16
    // dQ / dK / dV over each slot's rows = [dQ^T; dK^T] Ind and [dV^T; -] Ind, with
    // Ind the [128 rows x 16] slot indicator (UMMA M128 N16, fp32 accumulate in
    // TMEM columns 0-15 and 32-47, free since dV was read).  Row m of the result
    // holds column m & 63 of dQ (m < 64) or dK, for slot 0 (col 0) and 1 (col 1).
    // The tile's sums go to row b0 = first batch of its group, the group's other
    // rows get zeros, so summing all B rows gives the bias gradient.
    if (threadIdx.x == 0) {
      tc_after();
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const uint64_t db = sdesc(sptr(Ib) + (kk >> 2) * 2048 + (kk & 3) * 32, 16, 1024);
        const uint32_t acc = kk ? 1u : 0u;
        asm volatile(
            "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
            " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(tmem),
            "l"(mdesc_bd(sptr(Qs), kk)), "l"(db), "r"(a.id_cs), "r"(acc)
            : "memory");
        asm volatile(
            "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
            " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(tmem + 32),
            "l"(mdesc_bd(sptr(Vs), kk)), "l"(db), "r"(a.id_cs), "r"(acc)
            : "memory");
      }
      commit(&bar_cs);
    }
    __syncwarp();
    if (r.half == 0) {
      mbar_wait(&bar_cs, 0);
      tc_after();
      uint32_t u[4];
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0, %1}, [%2];"
                   : "=r"(u[0]), "=r"(u[1]) : "r"(tlane));
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0, %1}, [%2];"
                   : "=r"(u[2]), "=r"(u[3]) : "r"(tlane + 32));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int j = 0; j < 4; ++j) asm volatile("" : "+r"(u[j]));
      const int c = r.m & 63;
      for (int sl = 0; sl < nb; ++sl) {
        const int t = tile0 + sl, b0 = (t / a.H) * a.G, col = (t % a.H) * 64 + c;
        double* cqk = r.m < 64 ? a.csq : a.csk;
        const int64_t ldqk = r.m < 64 ? a.ldcsq : a.ldcsk;
        if (cqk) cqk[(int64_t)b0 * ldqk + col] = (double)__uint_as_float(u[sl]);
        if (r.m < 64 && a.csv) a.csv[(int64_t)b0 * a.ldcsv + col] = (double)__uint_as_float(u[2 + sl]);
      }
    } else if (a.G > 1) {
      // zeros in the other rows of each group: thread (m, 64 columns of the
      // three matrices) per (slot, row g)
      const int c = r.m & 63;
      for (int sl = 0; sl < nb; ++sl) {
        const int t = tile0 + sl, b0 = (t / a.H) * a.G, col = (t % a.H) * 64 + c;
        for (int g = 1; g < a.G && b0 + g < a.B; ++g) {
          double* cqk = r.m < 64 ? a.csq : a.csk;
          const int64_t ldqk = r.m < 64 ? a.ldcsq : a.ldcsk;
          if (cqk) cqk[(int64_t)(b0 + g) * ldqk + col] = 0.0;
          if (r.m < 64 && a.csv) a.csv[(int64_t)(b0 + g) * a.ldcsv + col] = 0.0;
        }
      }
    }
  }
  stamp(a, 7);
  if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
  tc_before();
  __syncthreads();                   // every TMEM read done
  if (warp == 1) {
    tc_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
  }
}

// ---------------------------------------------------------------------------
// 64 < L <= 128 (T-big, BERT-128): one (batch, head) per CTA as ONE 128-row
// tile.  S = Q K^T and dP = dO V^T are the same M = 128 x N = 128 chains as
// above; P, dS live in a [128 queries x 128 keys] buffer of two 64-key chunks
// (16 KB apart), so O = P V, dQ = dS K are K = 128 chains over the chunks
// (K-major) and dV = P^T dO, dK = dS^T Q read the same buffer MN-major.  Each
// thread owns one row (TMEM lane) and one 64-column half of S / dP.  The
// backward computes dV first and then reuses P's buffer for dS (96 KB of
// shared memory: two CTAs per SM).  Bias partials: column sums of the fp32
// dQ / dK / dV (warp reduce-scatter, then the four row quadrants in order).
// ---------------------------------------------------------------------------
constexpr size_t kFwd128Smem = 5 * kPair + 1024;    // Q, K, V, P (2 chunks)
constexpr size_t kBwd128Smem = 6 * kPair + 1024;    // Q, K, V, dO, P|dS (2 chunks)

// rows [L, 128) of a 128-row region: zero (no TMA box writes them)
__device__ __forceinline__ void zero_rows128(uint8_t* pair, int L) {
  if (L < 64) {
    zero_tail(pair, L);
    zero_tail(pair + kTile, 0);
  } else {
    zero_tail(pair + kTile, L - 64);
  }
}

// K = 128 chain: A is the two-chunk P / dS buffer (K-major: kdesc per chunk, or
// MN-major with its 64-wide M blocks 16 KB apart), B an MN-major 128-row tile
template <int AM>
__device__ __forceinline__ void mma_k128(uint32_t d, uint32_t a, uint32_t b, uint32_t idesc) {
#pragma unroll
  for (int kk = 0; kk < 8; ++kk) {
    const uint64_t da = AM == KM ? kdesc(a + (kk >> 2) * kPair, kk & 3) : mdesc_bd(a, kk);
    const uint64_t db = mdesc(b, kk);
    const uint32_t acc = kk ? 1u : 0u;
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
        " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d),
        "l"(da), "l"(db), "r"(idesc), "r"(acc)
        : "memory");
  }
}

struct Row128 {
  int m, q, half, idx, b, h;
  bool ok;
  int lo, hi;     // unmasked keys relative to this thread's 64 columns
};

__device__ __forceinline__ float partner128(float* buf, const Row128& r, float v) {
  buf[r.half * 128 + r.idx] = v;
  asm volatile("bar.sync %0, 64;" ::"r"(1 + r.q) : "memory");
  return buf[(r.half ^ 1) * 128 + r.idx];
}

__device__ __forceinline__ float partner_pair(float* buf, int q, int half, int lane, float v) {
  buf[half * 128 + q * 32 + lane] = v;
  asm volatile("bar.sync %0, 64;" ::"r"(1 + q) : "memory");
  const float o = buf[(half ^ 1) * 128 + q * 32 + lane];
  asm volatile("bar.sync %0, 64;" ::"r"(1 + q) : "memory");   // buf reusable afterwards
  return o;
}

__device__ __forceinline__ Row128 row128(const Args& a) {
  Row128 r;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  r.q = warp & 3;
  r.half = warp >> 2;
  r.idx = r.q * 32 + lane;
  r.m = r.idx;
  r.b = blockIdx.x / a.H;
  r.h = blockIdx.x % a.H;
  r.ok = r.m < a.Lq;
  int64_t len = a.Lk;
  if (a.mask == LS2_MASK_PADDING) len = __ldg(a.lens + r.b);
  int n = len < a.Lk ? (int)len : a.Lk;
  if (a.mask == LS2_MASK_CAUSAL) n = r.m + 1 < n ? r.m + 1 : n;
  r.lo = -64 * r.half;
  r.hi = r.ok ? n - 64 * r.half : r.lo;
  return r;
}

__device__ __forceinline__ void tmem_ld64(uint32_t taddr, float (&x)[64]) {
  float a[32], b[32];
  tmem_ld32(taddr, a);
  tmem_ld32(taddr + 32, b);
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    x[i] = a[i];
    x[32 + i] = b[i];
  }
}

// column sums over the CTA's 128 rows of a [128 x 64] fp32 TMEM result whose
// thread holds 32 columns (half) of one row: warp reduce-scatter (lane l ends
// with column l of its half), then the four row quadrants in order -> f64 row
// `b` of the partial buffer
__device__ __forceinline__ void colsum128(float (&x)[32], int q, int half, float* red,
                                          double* out) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const bool up = (lane & o) != 0;
#pragma unroll
    for (int i = 0; i < o; ++i) {
      const float send = up ? x[i] : x[i + o];
      const float keep = up ? x[i + o] : x[i];
      x[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
    }
  }
  red[q * 64 + 32 * half + lane] = x[0];
  __syncthreads();
  if (threadIdx.x < 64 && out) {
    const int c = threadIdx.x;
    out[c] = (double)(((red[c] + red[64 + c]) + red[128 + c]) + red[192 + c]);
  }
  __syncthreads();
}

__global__ void __launch_bounds__(kThreads, 2) attn_tc128_fwd_kernel(
    const __grid_constant__ CUtensorMap mq, const __grid_constant__ CUtensorMap mk,
    const __grid_constant__ CUtensorMap mv, const __grid_constant__ CUtensorMap mo,
    const __grid_constant__ Args a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                           ~uintptr_t(1023));
  uint8_t* Qs = sm;                  // 128 rows; doubles as the O staging
  uint8_t* Ks = sm + kPair;
  uint8_t* Vs = sm + 2 * kPair;
  uint8_t* Pb = sm + 3 * kPair;      // [128 queries x 128 keys]: chunk c = keys 64c ..
  __shared__ __align__(8) uint64_t bar_qk, bar_v, bar_s, bar_o;
  __shared__ uint32_t tmem_base;
  __shared__ float xm[256], xz[256];
  const int warp = threadIdx.x >> 5;
  const int b = blockIdx.x / a.H, h = blockIdx.x % a.H;
  if (threadIdx.x == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mq)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mk)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mv)) : "memory");
    mbar_init(&bar_qk, 1);
    mbar_init(&bar_v, 1);
    mbar_init(&bar_s, 1);
    mbar_init(&bar_o, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    mbar_expect_tx(&bar_qk, (uint32_t)((a.Lq + a.Lk) * 128));
    tma_load_3d(Qs, &mq, h * 64, 0, b, &bar_qk);
    tma_load_3d(Ks, &mk, h * 64, 0, b, &bar_qk);
    mbar_expect_tx(&bar_v, (uint32_t)(a.Lk * 128));
    tma_load_3d(Vs, &mv, h * 64, 0, b, &bar_v);
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(
        sptr(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  zero_rows128(Qs, a.Lq);
  zero_rows128(Ks, a.Lk);
  zero_rows128(Vs, a.Lk);
  fence_async_smem();
  tc_before();
  __syncthreads();
  tc_after();
  const uint32_t tmem = tmem_base;
  Row128 r = row128(a);
  if (threadIdx.x == 0) {
    mbar_wait(&bar_qk, 0);
    tc_after();
    mma128<KM, KM, 4>(tmem, sptr(Qs), sptr(Ks), a.id_s);      // S (cols 0-127)
    commit(&bar_s);
  }
  __syncwarp();
  const uint32_t tlane = tmem + ((uint32_t)(32 * r.q) << 16);
  mbar_wait(&bar_s, 0);
  tc_after();
  float x[64];
  tmem_ld64(tlane + 64 * r.half, x);
  float m = -INFINITY;
#pragma unroll
  for (int c = 0; c < 64; ++c) {
    x[c] = (c >= r.lo && c < r.hi) ? __fmul_rn(x[c], a.scale) : -INFINITY;
    m = fmaxf(m, x[c]);
  }
  m = fmaxf(m, partner128(xm, r, m));
  float z = 0.f;
#pragma unroll
  for (int c = 0; c < 64; ++c) {
    x[c] = x[c] == -INFINITY ? 0.f : ex2(__fsub_rn(x[c], m));
    z += x[c];
  }
  z += partner128(xz, r, z);
  const float iz = z > 0.f ? 1.f / z : 0.f;
#pragma unroll
  for (int sub = 0; sub < 2; ++sub) {
    uint32_t w[16];
#pragma unroll
    for (int j = 0; j < 16; ++j)
      w[j] = pack_h2(__fmul_rn(x[32 * sub + 2 * j], iz), __fmul_rn(x[32 * sub + 2 * j + 1], iz));
    st_cols(Pb + r.half * kPair, r.m, sub, w);
  }
  if (r.ok && r.half == 0) a.stats[((int64_t)r.b * a.H + r.h) * a.Lq + r.m] = make_float2(m, iz);
  fence_async_smem();
  tc_before();
  __syncthreads();                   // P complete, S read
  if (threadIdx.x == 0) {
    tc_after();
    mbar_wait(&bar_v, 0);
    mma_k128<KM>(tmem, sptr(Pb), sptr(Vs), a.id128_pv);      // O = P V (cols 0-63)
    commit(&bar_o);
  }
  __syncwarp();
  mbar_wait(&bar_o, 0);
  tc_after();
  {
    float o[32];
    tmem_ld32(tlane + 32 * r.half, o);
    st_cols_f(Qs, r.m, r.half, o);
  }
  fence_async_smem();
  tc_before();
  __syncthreads();
  if (threadIdx.x == 0) {
    tma_store_3d(&mo, h * 64, 0, b, Qs);
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
  }
  __syncwarp();
  if (warp == 1) {
    tc_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tmem));
  }
}

__global__ void __launch_bounds__(kThreads, 2) attn_tc128_bwd_kernel(
    const __grid_constant__ CUtensorMap mq, const __grid_constant__ CUtensorMap mk,
    const __grid_constant__ CUtensorMap mv, const __grid_constant__ CUtensorMap mdo,
    const __grid_constant__ CUtensorMap mdq, const __grid_constant__ CUtensorMap mdk,
    const __grid_constant__ CUtensorMap mdv, const __grid_constant__ Args a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                           ~uintptr_t(1023));
  uint8_t* Qs = sm;                  // Q, K, V double as dQ, dK, dV staging
  uint8_t* Ks = sm + kPair;
  uint8_t* Vs = sm + 2 * kPair;
  uint8_t* Os = sm + 3 * kPair;      // dO
  uint8_t* Pb = sm + 4 * kPair;      // P, then dS: [128 queries x 128 keys], two chunks
  __shared__ __align__(8) uint64_t bar_ld, bar_1, bar_2, bar_3;
  __shared__ uint32_t tmem_base;
  __shared__ float xr[256];
  const int warp = threadIdx.x >> 5;
  const int b = blockIdx.x / a.H, h = blockIdx.x % a.H;
  if (threadIdx.x == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mq)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mk)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mdo)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mv)) : "memory");
    mbar_init(&bar_ld, 1);
    mbar_init(&bar_1, 1);
    mbar_init(&bar_2, 1);
    mbar_init(&bar_3, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    mbar_expect_tx(&bar_ld, (uint32_t)(2 * (a.Lq + a.Lk) * 128));
    tma_load_3d(Qs, &mq, h * 64, 0, b, &bar_ld);
    tma_load_3d(Ks, &mk, h * 64, 0, b, &bar_ld);
    tma_load_3d(Os, &mdo, h * 64, 0, b, &bar_ld);
    tma_load_3d(Vs, &mv, h * 64, 0, b, &bar_ld);
  }
  if (warp == 1) {   // S (0-127), dP (128-255); then dV (0-63), dQ (64-127), dK (128-191)
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(
        sptr(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  zero_rows128(Qs, a.Lq);
  zero_rows128(Os, a.Lq);
  zero_rows128(Ks, a.Lk);
  zero_rows128(Vs, a.Lk);
  fence_async_smem();
  tc_before();
  __syncthreads();
  tc_after();
  const uint32_t tmem = tmem_base;
  Row128 r = row128(a);
  float2 st = make_float2(0.f, 0.f);
  if (r.ok) st = __ldg(a.stats + ((int64_t)r.b * a.H + r.h) * a.Lq + r.m);
  if (threadIdx.x == 0) {
    mbar_wait(&bar_ld, 0);
    tc_after();
    mma128<KM, KM, 4>(tmem, sptr(Qs), sptr(Ks), a.id_s);          // S
    mma128<KM, KM, 4>(tmem + 128, sptr(Os), sptr(Vs), a.id_s);    // dP
    commit(&bar_1);
  }
  __syncwarp();
  const uint32_t tlane = tmem + ((uint32_t)(32 * r.q) << 16);
  mbar_wait(&bar_1, 0);
  tc_after();
  uint32_t pw[32];                   // P of this half row, fp16 pairs
  {
    float x[64];
    tmem_ld64(tlane + 64 * r.half, x);
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      float p2[2];
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int c = 2 * j + e;
        p2[e] = (c >= r.lo && c < r.hi)
                    ? __fmul_rn(ex2(__fsub_rn(__fmul_rn(x[c], a.scale), st.x)), st.y)
                    : 0.f;
      }
      pw[j] = pack_h2(p2[0], p2[1]);
    }
  }
#pragma unroll
  for (int sub = 0; sub < 2; ++sub) {
    uint32_t w[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) w[j] = pw[16 * sub + j];
    st_cols(Pb + r.half * kPair, r.m, sub, w);
  }
  uint32_t dw[32];
  {
    float x[64];
    tmem_ld64(tlane + 128 + 64 * r.half, x);                  // dP
    float rs = 0.f;
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const float2 p = unpack_h2(pw[j]);
      rs += x[2 * j] * p.x + x[2 * j + 1] * p.y;
    }
    rs += partner128(xr, r, rs);
    const float ds = a.dscale;
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const float2 p = unpack_h2(pw[j]);
      dw[j] = pack_h2(p.x * (x[2 * j] - rs) * ds, p.y * (x[2 * j + 1] - rs) * ds);
    }
  }
  fence_async_smem();
  tc_before();
  __syncthreads();                   // P complete, S and dP read
  if (threadIdx.x == 0) {
    tc_after();
    mma_k128<MN>(tmem, sptr(Pb), sptr(Os), a.id128_mm);       // dV = P^T dO (cols 0-63)
    commit(&bar_2);
  }
  __syncwarp();
  mbar_wait(&bar_2, 0);              // P no longer read: its buffer takes dS
  tc_after();
#pragma unroll
  for (int sub = 0; sub < 2; ++sub) {
    uint32_t w[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) w[j] = dw[16 * sub + j];
    st_cols(Pb + r.half * kPair, r.m, sub, w);
  }
  fence_async_smem();
  tc_before();
  __syncthreads();
  if (threadIdx.x == 0) {
    tc_after();
    mma_k128<KM>(tmem + 64, sptr(Pb), sptr(Ks), a.id128_pv);  // dQ = dS K
    mma_k128<MN>(tmem + 128, sptr(Pb), sptr(Qs), a.id128_mm); // dK = dS^T Q
    commit(&bar_3);
  }
  __syncwarp();
  __shared__ float red[256];
  {   // dV (row = key) -> V's tile (V dead since dP), bias partial, store
    float x[32];
    tmem_ld32(tlane + 32 * r.half, x);
    st_cols_f(Vs, r.m, r.half, x);
    colsum128(x, r.q, r.half, red, a.csv ? a.csv + (int64_t)b * a.ldcsv + h * 64 : nullptr);
  }
  fence_async_smem();
  __syncthreads();
  if (threadIdx.x == 0) {
    tma_store_3d(&mdv, h * 64, 0, b, Vs);
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  }
  mbar_wait(&bar_3, 0);              // dQ, dK done: Q, K dead
  tc_after();
  {
    float x[32];
    tmem_ld32(tlane + 64 + 32 * r.half, x);
    st_cols_f(Qs, r.m, r.half, x);
    colsum128(x, r.q, r.half, red, a.csq ? a.csq + (int64_t)b * a.ldcsq + h * 64 : nullptr);
  }
  {
    float x[32];
    tmem_ld32(tlane + 128 + 32 * r.half, x);
    st_cols_f(Ks, r.m, r.half, x);
    colsum128(x, r.q, r.half, red, a.csk ? a.csk + (int64_t)b * a.ldcsk + h * 64 : nullptr);
  }
  fence_async_smem();
  tc_before();
  __syncthreads();
  if (threadIdx.x == 0) {
    tma_store_3d(&mdq, h * 64, 0, b, Qs);
    tma_store_3d(&mdk, h * 64, 0, b, Ks);
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
  }
  __syncwarp();
  if (warp == 1) {
    tc_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
  }
}

// ---------------------------------------------------------------------------
// 128 < L <= 512 (BERT-512): flash-style kernels on the same tcgen05 blocks.
// Work units are 128-row blocks of one (batch, head); K / V (or Q / dO) stream
// through two-slot TMA rings in 128-row chunks (rows past L are TMA zero fill),
// and the [B, H, L, L] scores never touch HBM.
//  * forward (per query block): S_c = Q K_c^T for every key chunk into TMEM
//    (4 x 128 = 512 columns), row statistics over all chunks (max, 1/sum),
//    then P_c -> shared memory (two-slot ring) and O += P_c V_c (TMEM columns
//    0-63, S_0's columns, free once P_0 is formed);
//  * backward dQ (per query block): D = rowsum(dO * O), then per key chunk
//    S_c, dP_c -> P_c, dS_c = P_c (dP_c - D) scale -> dQ += dS_c K_c;
//  * backward dK / dV (per key block): per query chunk S, dP -> P, dS ->
//    dV += P^T dO_i, dK += dS^T Q_i.
// The statistics [B][H][L][4] hold (max in the log2 domain, 1/sum, D, -).
// Bias partials: one f64 row per (batch, 128-row block).  Deterministic.
// ---------------------------------------------------------------------------
constexpr int kFlashMaxChunks = 4;
constexpr size_t kFlashFwdSmem = 13 * kPair + 1024;       // Q, K[4], V[4], P[2] (2 chunks each)
constexpr size_t kFlashDqSmem = 13 * kPair + 1024;        // Q, dO, O, K[4], V[4], dS (2 chunks)
constexpr size_t kFlashDkvSmem = 10 * kPair + 1024;       // K, V, Q[2], dO[2], P (2), dS (2)

template <int AM>
__device__ __forceinline__ void mma_k128_acc(uint32_t d, uint32_t a, uint32_t b, uint32_t idesc,
                                             bool accum) {
#pragma unroll
  for (int kk = 0; kk < 8; ++kk) {
    const uint64_t da = AM == KM ? kdesc(a + (kk >> 2) * kPair, kk & 3) : mdesc_bd(a, kk);
    const uint64_t db = mdesc(b, kk);
    const uint32_t acc = (kk || accum) ? 1u : 0u;
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
        " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d),
        "l"(da), "l"(db), "r"(idesc), "r"(acc)
        : "memory");
  }
}

// keys [0, n) of query row `qpos` of batch b are kept
__device__ __forceinline__ int flash_keep_n(const Args& a, int b, int qpos) {
  int n = a.Lk;
  if (a.mask == LS2_MASK_PADDING) {
    const int64_t len = __ldg(a.lens + b);
    n = len < n ? (int)len : n;
  }
  if (a.mask == LS2_MASK_CAUSAL) n = qpos + 1 < n ? qpos + 1 : n;
  return n;
}

__device__ __forceinline__ void st_row64(uint8_t* chunk_region, int m, const uint32_t (&w)[32]) {
  uint32_t lo[16], hi[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) { lo[j] = w[j]; hi[j] = w[16 + j]; }
  st_cols(chunk_region, m, 0, lo);
  st_cols(chunk_region, m, 1, hi);
}

__global__ void __launch_bounds__(kThreads, 1) attn_flash_fwd_kernel(
    const __grid_constant__ CUtensorMap mq, const __grid_constant__ CUtensorMap mk,
    const __grid_constant__ CUtensorMap mv, const __grid_constant__ CUtensorMap mo,
    const __grid_constant__ Args a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                           ~uintptr_t(1023));
  uint8_t* Qs = sm;                        // doubles as the O staging
  uint8_t* Kr = sm + kPair;                // one slot per key chunk (<= 4)
  uint8_t* Vr = sm + 5 * kPair;            // one slot per key chunk
  uint8_t* Pr = sm + 9 * kPair;            // 2 slots x 2 chunks
  __shared__ __align__(8) uint64_t bar_q, kfull[kFlashMaxChunks], vfull[kFlashMaxChunks],
      pfree[2], bar_s, bar_o;
  __shared__ uint32_t tmem_base;
  __shared__ float xm[256], xz[256];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nqb = (a.Lq + 127) / 128;
  const int qb = blockIdx.x % nqb, bh = blockIdx.x / nqb;
  const int b = bh / a.H, h = bh % a.H;
  const int nk = (a.Lk + 127) / 128;
  if (threadIdx.x == 0) {
    mbar_init(&bar_q, 1); mbar_init(&bar_s, 1); mbar_init(&bar_o, 1);
    for (int i = 0; i < kFlashMaxChunks; ++i) { mbar_init(&kfull[i], 1); mbar_init(&vfull[i], 1); }
    for (int i = 0; i < 2; ++i) mbar_init(&pfree[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    mbar_expect_tx(&bar_q, (uint32_t)kPair);
    tma_load_3d(Qs, &mq, h * 64, qb * 128, b, &bar_q);
    for (int c = 0; c < nk; ++c) {
      mbar_expect_tx(&kfull[c], (uint32_t)kPair);
      tma_load_3d(Kr + c * kPair, &mk, h * 64, c * 128, b, &kfull[c]);
      mbar_expect_tx(&vfull[c], (uint32_t)kPair);
      tma_load_3d(Vr + c * kPair, &mv, h * 64, c * 128, b, &vfull[c]);
    }
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        sptr(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_before();
  __syncthreads();
  tc_after();
  const uint32_t tmem = tmem_base;
  const int q = warp & 3, half = warp >> 2, m = 32 * q + lane;
  const int qpos = qb * 128 + m;
  const bool ok = qpos < a.Lq;
  const int nkeep = flash_keep_n(a, b, qpos);
  if (threadIdx.x == 0) {          // S_c for every key chunk
    mbar_wait(&bar_q, 0);
    for (int c = 0; c < nk; ++c) {
      mbar_wait(&kfull[c], 0);
      tc_after();
      mma128<KM, KM, 4>(tmem + 128 * c, sptr(Qs), sptr(Kr + c * kPair), a.id_s);
    }
    commit(&bar_s);
  }
  __syncwarp();
  const uint32_t tlane = tmem + ((uint32_t)(32 * q) << 16);
  mbar_wait(&bar_s, 0);
  tc_after();
  // pass 1: the row maximum over every chunk (log2 domain; no exponentials)
  float mx = -INFINITY;
  for (int c = 0; c < nk; ++c) {
    float x[64];
    tmem_ld64(tlane + 128 * c + 64 * half, x);
    const int k0 = 128 * c + 64 * half;
#pragma unroll
    for (int j = 0; j < 64; ++j)
      if (ok && k0 + j < nkeep) mx = fmaxf(mx, __fmul_rn(x[j], a.scale));
  }
  mx = fmaxf(mx, partner_pair(xm, q, half, lane, mx));
  // pass 2 (below): P = exp2(s - max) unnormalised (<= 1) into the ring, its row
  // sum on the side; O is divided by the sum when it leaves TMEM, so every score
  // takes ONE exponential
  float z = 0.f;
  // P_c -> ring, O += P_c V_c
  for (int c = 0; c < nk; ++c) {
    const int ps = c & 1;
    if (c >= 2) mbar_wait(&pfree[ps], (uint32_t)(((c - 2) >> 1) & 1));
    float x[64];
    tmem_ld64(tlane + 128 * c + 64 * half, x);
    const int k0 = 128 * c + 64 * half;
    uint32_t w[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      float p2[2];
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int kk = k0 + 2 * j + e;
        p2[e] = (ok && kk < nkeep) ? ex2(__fsub_rn(__fmul_rn(x[2 * j + e], a.scale), mx)) : 0.f;
      }
      w[j] = pack_h2(p2[0], p2[1]);
      // the sum of the STORED (fp16-rounded) probabilities normalises O = P V
      const float2 pr = unpack_h2(w[j]);
      z += pr.x + pr.y;
    }
    st_row64(Pr + ps * 2 * kPair + half * kPair, m, w);
    fence_async_smem();
    tc_before();
    __syncthreads();                 // P_c complete; S_c read (and S_0 before O lands)
    if (threadIdx.x == 0) {
      tc_after();
      mbar_wait(&vfull[c], 0);
      mma_k128_acc<KM>(tmem, sptr(Pr + ps * 2 * kPair), sptr(Vr + c * kPair), a.id128_pv,
                       c > 0);
      commit(&pfree[ps]);
    }
    __syncwarp();
  }
  if (threadIdx.x == 0) commit(&bar_o);
  __syncwarp();
  z += partner_pair(xz, q, half, lane, z);
  const float iz = z > 0.f ? 1.f / z : 0.f;
  if (ok && half == 0) {
    float4* st4 = reinterpret_cast<float4*>(a.stats) + ((int64_t)b * a.H + h) * a.Lq + qpos;
    *st4 = make_float4(mx, iz, 0.f, 0.f);
  }
  mbar_wait(&bar_o, 0);
  tc_after();
  {
    float o[32];
    tmem_ld32(tlane + 32 * half, o);
#pragma unroll
    for (int j = 0; j < 32; ++j) o[j] = __fmul_rn(o[j], iz);
    st_cols_f(Qs, m, half, o);
  }
  fence_async_smem();
  tc_before();
  __syncthreads();
  if (threadIdx.x == 0) {
    tma_store_3d(&mo, h * 64, qb * 128, b, Qs);
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
  }
  __syncwarp();
  if (warp == 1) {
    tc_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

// the 32 fp16 columns [32 h, 32 h + 32) of row m of a 64-column swizzled tile
__device__ __forceinline__ void ld_cols(const uint8_t* region, int m, int half, float (&f)[32]) {
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const uint4 u = *reinterpret_cast<const uint4*>(region + swz(m, 4 * half + c));
    const uint32_t w4[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float2 p = unpack_h2(w4[j]);
      f[8 * c + 2 * j] = p.x;
      f[8 * c + 2 * j + 1] = p.y;
    }
  }
}

__global__ void __launch_bounds__(kThreads, 1) attn_flash_dq_kernel(
    const __grid_constant__ CUtensorMap mq, const __grid_constant__ CUtensorMap mk,
    const __grid_constant__ CUtensorMap mv, const __grid_constant__ CUtensorMap mdo,
    const __grid_constant__ CUtensorMap mo, const __grid_constant__ CUtensorMap mdq,
    const __grid_constant__ Args a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                           ~uintptr_t(1023));
  uint8_t* Qs = sm;                        // doubles as the dQ staging
  uint8_t* Ds = sm + kPair;                // dO
  uint8_t* Os = sm + 2 * kPair;            // O (for D)
  uint8_t* Kr = sm + 3 * kPair;            // one slot per key chunk (<= 4)
  uint8_t* Vr = sm + 7 * kPair;            // one slot per key chunk
  uint8_t* Sr = sm + 11 * kPair;           // dS (2 chunks)
  __shared__ __align__(8) uint64_t bar_ld, kvfull[kFlashMaxChunks], dsfree, bar_sd, bar_q;
  __shared__ uint32_t tmem_base;
  __shared__ float xr[256];
  __shared__ float red[256];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nqb = (a.Lq + 127) / 128;
  const int qb = blockIdx.x % nqb, bh = blockIdx.x / nqb;
  const int b = bh / a.H, h = bh % a.H;
  const int nk = (a.Lk + 127) / 128;
  if (threadIdx.x == 0) {
    mbar_init(&bar_ld, 1); mbar_init(&bar_sd, 1); mbar_init(&bar_q, 1); mbar_init(&dsfree, 1);
    for (int i = 0; i < kFlashMaxChunks; ++i) mbar_init(&kvfull[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    mbar_expect_tx(&bar_ld, (uint32_t)(3 * kPair));
    tma_load_3d(Qs, &mq, h * 64, qb * 128, b, &bar_ld);
    tma_load_3d(Ds, &mdo, h * 64, qb * 128, b, &bar_ld);
    tma_load_3d(Os, &mo, h * 64, qb * 128, b, &bar_ld);
    for (int c = 0; c < nk; ++c) {
      mbar_expect_tx(&kvfull[c], (uint32_t)(2 * kPair));
      tma_load_3d(Kr + c * kPair, &mk, h * 64, c * 128, b, &kvfull[c]);
      tma_load_3d(Vr + c * kPair, &mv, h * 64, c * 128, b, &kvfull[c]);
    }
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        sptr(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_before();
  __syncthreads();
  tc_after();
  const uint32_t tmem = tmem_base;
  const int q = warp & 3, half = warp >> 2, m = 32 * q + lane;
  const int qpos = qb * 128 + m;
  const bool ok = qpos < a.Lq;
  const int nkeep = flash_keep_n(a, b, qpos);
  float4* st4 = reinterpret_cast<float4*>(a.stats) + ((int64_t)b * a.H + h) * a.Lq + qpos;
  float4 stv = ok ? *st4 : make_float4(0.f, 0.f, 0.f, 0.f);
  mbar_wait(&bar_ld, 0);
  float D;
  {   // D = rowsum(dO * O) over the head's 64 columns
    float fo[32], fd[32];
    ld_cols(Os, m, half, fo);
    ld_cols(Ds, m, half, fd);
    float t = 0.f;
#pragma unroll
    for (int j = 0; j < 32; ++j) t = fmaf(fd[j], fo[j], t);
    D = t + partner_pair(xr, q, half, lane, t);
  }
  if (ok && half == 0) { stv.z = D; *st4 = stv; }
  const uint32_t tlane = tmem + ((uint32_t)(32 * q) << 16);
  for (int c = 0; c < nk; ++c) {
    if (threadIdx.x == 0) {
      mbar_wait(&kvfull[c], 0);
      tc_after();
      mma128<KM, KM, 4>(tmem, sptr(Qs), sptr(Kr + c * kPair), a.id_s);           // S
      mma128<KM, KM, 4>(tmem + 128, sptr(Ds), sptr(Vr + c * kPair), a.id_s);     // dP
      commit(&bar_sd);
    }
    __syncwarp();
    mbar_wait(&bar_sd, (uint32_t)(c & 1));
    tc_after();
    if (c >= 1) mbar_wait(&dsfree, (uint32_t)((c - 1) & 1));   // dS buffer read
    uint32_t w[32];
    {
      float x[64], dp[64];
      tmem_ld64(tlane + 64 * half, x);
      tmem_ld64(tlane + 128 + 64 * half, dp);
      const int k0 = 128 * c + 64 * half;
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        float v2[2];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int i = 2 * j + e;
          const float p = (ok && k0 + i < nkeep)
                              ? __fmul_rn(ex2(__fsub_rn(__fmul_rn(x[i], a.scale), stv.x)), stv.y)
                              : 0.f;
          v2[e] = p * (dp[i] - D) * a.dscale;
        }
        w[j] = pack_h2(v2[0], v2[1]);
      }
    }
    st_row64(Sr + half * kPair, m, w);
    fence_async_smem();
    tc_before();
    __syncthreads();                 // dS_c complete; S, dP read
    if (threadIdx.x == 0) {
      tc_after();
      mma_k128_acc<KM>(tmem + 256, sptr(Sr), sptr(Kr + c * kPair), a.id128_pv,
                       c > 0);                                                   // dQ += dS K
      commit(&dsfree);
    }
    __syncwarp();
  }
  if (threadIdx.x == 0) commit(&bar_q);
  __syncwarp();
  mbar_wait(&bar_q, 0);
  tc_after();
  {
    float x[32];
    tmem_ld32(tlane + 256 + 32 * half, x);
    st_cols_f(Qs, m, half, x);
    if (!ok) {
#pragma unroll
      for (int j = 0; j < 32; ++j) x[j] = 0.f;
    }
    colsum128(x, q, half, red,
              a.csq ? a.csq + ((int64_t)b * nqb + qb) * a.ldcsq + h * 64 : nullptr);
  }
  fence_async_smem();
  tc_before();
  __syncthreads();
  if (threadIdx.x == 0) {
    tma_store_3d(&mdq, h * 64, qb * 128, b, Qs);
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
  }
  __syncwarp();
  if (warp == 1) {
    tc_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

__global__ void __launch_bounds__(kThreads, 1) attn_flash_dkv_kernel(
    const __grid_constant__ CUtensorMap mq, const __grid_constant__ CUtensorMap mk,
    const __grid_constant__ CUtensorMap mv, const __grid_constant__ CUtensorMap mdo,
    const __grid_constant__ CUtensorMap mdk, const __grid_constant__ CUtensorMap mdv,
    const __grid_constant__ Args a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                           ~uintptr_t(1023));
  uint8_t* Ks = sm;                        // doubles as the dK staging
  uint8_t* Vs = sm + kPair;                // doubles as the dV staging
  uint8_t* Qr = sm + 2 * kPair;            // 2 slots
  uint8_t* Dr = sm + 4 * kPair;            // dO, 2 slots
  uint8_t* Pb = sm + 6 * kPair;            // P (2 chunks)
  uint8_t* Sb = sm + 8 * kPair;            // dS (2 chunks)
  __shared__ __align__(8) uint64_t bar_kv, qfull[2], bar_sd, bar_mm;
  __shared__ uint32_t tmem_base;
  __shared__ float xr[256];
  __shared__ float red[256];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nkb = (a.Lk + 127) / 128;
  const int kb = blockIdx.x % nkb, bh = blockIdx.x / nkb;
  const int b = bh / a.H, h = bh % a.H;
  const int nq = (a.Lq + 127) / 128;
  if (threadIdx.x == 0) {
    mbar_init(&bar_kv, 1); mbar_init(&bar_sd, 1); mbar_init(&bar_mm, 1);
    for (int i = 0; i < 2; ++i) mbar_init(&qfull[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    mbar_expect_tx(&bar_kv, (uint32_t)(2 * kPair));
    tma_load_3d(Ks, &mk, h * 64, kb * 128, b, &bar_kv);
    tma_load_3d(Vs, &mv, h * 64, kb * 128, b, &bar_kv);
    for (int c = 0; c < nq && c < 2; ++c) {
      mbar_expect_tx(&qfull[c], (uint32_t)(2 * kPair));
      tma_load_3d(Qr + c * kPair, &mq, h * 64, c * 128, b, &qfull[c]);
      tma_load_3d(Dr + c * kPair, &mdo, h * 64, c * 128, b, &qfull[c]);
    }
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        sptr(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_before();
  __syncthreads();
  tc_after();
  const uint32_t tmem = tmem_base;
  const int q = warp & 3, half = warp >> 2, m = 32 * q + lane;
  const uint32_t tlane = tmem + ((uint32_t)(32 * q) << 16);
  const float4* st4 = reinterpret_cast<const float4*>(a.stats) + ((int64_t)b * a.H + h) * a.Lq;
  for (int c = 0; c < nq; ++c) {
    const int s = c & 1;
    const int qpos = c * 128 + m;                      // this thread's query row (S: M = query)
    const bool ok = qpos < a.Lq;
    const int nkeep = flash_keep_n(a, b, qpos);
    const float4 stv = ok ? st4[qpos] : make_float4(0.f, 0.f, 0.f, 0.f);
    if (threadIdx.x == 0) {
      if (c == 0) mbar_wait(&bar_kv, 0);
      mbar_wait(&qfull[s], (uint32_t)((c >> 1) & 1));
      tc_after();
      mma128<KM, KM, 4>(tmem, sptr(Qr + s * kPair), sptr(Ks), a.id_s);           // S
      mma128<KM, KM, 4>(tmem + 128, sptr(Dr + s * kPair), sptr(Vs), a.id_s);     // dP
      commit(&bar_sd);
    }
    __syncwarp();
    mbar_wait(&bar_sd, (uint32_t)(c & 1));
    tc_after();
    if (c >= 1) mbar_wait(&bar_mm, (uint32_t)((c - 1) & 1));   // P / dS buffers read
    uint32_t pw[32], dw[32];
    {
      float x[64], dp[64];
      tmem_ld64(tlane + 64 * half, x);
      tmem_ld64(tlane + 128 + 64 * half, dp);
      const int k0 = kb * 128 + 64 * half;
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        float p2[2], d2[2];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int i = 2 * j + e;
          const float p = (ok && k0 + i < nkeep)
                              ? __fmul_rn(ex2(__fsub_rn(__fmul_rn(x[i], a.scale), stv.x)), stv.y)
                              : 0.f;
          p2[e] = p;
          d2[e] = p * (dp[i] - stv.z) * a.dscale;
        }
        pw[j] = pack_h2(p2[0], p2[1]);
        dw[j] = pack_h2(d2[0], d2[1]);
      }
    }
    st_row64(Pb + half * kPair, m, pw);
    st_row64(Sb + half * kPair, m, dw);
    fence_async_smem();
    tc_before();
    __syncthreads();                 // P, dS complete; S, dP read
    if (threadIdx.x == 0) {
      tc_after();
      mma_k128_acc<MN>(tmem + 256, sptr(Pb), sptr(Dr + s * kPair), a.id128_mm, c > 0);  // dV
      mma_k128_acc<MN>(tmem + 320, sptr(Sb), sptr(Qr + s * kPair), a.id128_mm, c > 0);  // dK
      commit(&bar_mm);
      if (c + 2 < nq) {
        mbar_wait(&bar_mm, (uint32_t)(c & 1));
        mbar_expect_tx(&qfull[s], (uint32_t)(2 * kPair));
        tma_load_3d(Qr + s * kPair, &mq, h * 64, (c + 2) * 128, b, &qfull[s]);
        tma_load_3d(Dr + s * kPair, &mdo, h * 64, (c + 2) * 128, b, &qfull[s]);
      }
    }
    __syncwarp();
  }
  mbar_wait(&bar_mm, (uint32_t)((nq - 1) & 1));
  tc_after();
  const int64_t prow = (int64_t)b * nkb + kb;
  {
    float x[32];
    tmem_ld32(tlane + 256 + 32 * half, x);              // dV (row = key)
    st_cols_f(Vs, m, half, x);
    colsum128(x, q, half, red, a.csv ? a.csv + prow * a.ldcsv + h * 64 : nullptr);
  }
  {
    float x[32];
    tmem_ld32(tlane + 320 + 32 * half, x);              // dK
    st_cols_f(Ks, m, half, x);
    colsum128(x, q, half, red, a.csk ? a.csk + prow * a.ldcsk + h * 64 : nullptr);
  }
  fence_async_smem();
  tc_before();
  __syncthreads();
  if (threadIdx.x == 0) {
    tma_store_3d(&mdv, h * 64, kb * 128, b, Vs);
    tma_store_3d(&mdk, h * 64, kb * 128, b, Ks);
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
  }
  __syncwarp();
  if (warp == 1) {
    tc_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

// [B][L][ld] fp16 operand, columns [0, cols) from `base`: boxes of 64 columns x L
// rows x G sequences, 128-byte swizzle, zero fill past L / B
bool make_map3(CUtensorMap* m, const void* base, int64_t cols, int64_t L, int64_t B, int64_t ld,
               int G) {
  auto fn = tc::encode_fn();
  if (!fn) return false;
  cuuint64_t dims[3] = {(cuuint64_t)cols, (cuuint64_t)L, (cuuint64_t)B};
  cuuint64_t strides[2] = {(cuuint64_t)(ld * 2), (cuuint64_t)(L * ld * 2)};
  cuuint32_t box[3] = {64, (cuuint32_t)L, (cuuint32_t)G};
  cuuint32_t es[3] = {1, 1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, const_cast<void*>(base), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// the same operand with 128-row boxes (flash kernels: one 128-row block per load)
bool make_map3_rows(CUtensorMap* m, const void* base, int64_t cols, int64_t L, int64_t B,
                    int64_t ld, int box_rows) {
  auto fn = tc::encode_fn();
  if (!fn) return false;
  cuuint64_t dims[3] = {(cuuint64_t)cols, (cuuint64_t)L, (cuuint64_t)B};
  cuuint64_t strides[2] = {(cuuint64_t)(ld * 2), (cuuint64_t)(L * ld * 2)};
  cuuint32_t box[3] = {64, (cuuint32_t)box_rows, 1};
  cuuint32_t es[3] = {1, 1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, const_cast<void*>(base), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// UMMA instruction descriptor: fp16 A/B, fp32 D, M = 64, N = 64
// UMMA instruction descriptor: fp16 A/B, fp32 D
constexpr uint32_t idesc(bool a_mn, bool b_mn, uint32_t n, uint32_t m = 128) {
  return (1u << 4) | ((a_mn ? 1u : 0u) << 15) | ((b_mn ? 1u : 0u) << 16) | ((n >> 3) << 17) |
         ((m >> 4) << 24);
}

constexpr size_t kFwdSmem = 4 * kPair + 1024;
constexpr size_t kBwdSmem = 6 * kPair + 4096 + 1024;

unsigned long long* g_trace = nullptr;

bool aligned16(const void* p, int64_t ld) {
  return (reinterpret_cast<uintptr_t>(p) & 15) == 0 && (ld & 7) == 0;
}

int fill_args(Args& a, int64_t batch, int64_t heads, int64_t lq, int64_t lk, int mask_kind,
              const int64_t* lens, double scale, float2* stats) {
  a.H = (int)heads;
  a.Lq = (int)lq;
  a.Lk = (int)lk;
  const int64_t lmax = lq > lk ? lq : lk;
  a.G = lmax > 64 ? 1 : (int)(64 / lmax);      // L > 64: one 128-row tile per (b, h)
  a.B = (int)batch;
  a.ntiles = (int)(heads * ((batch + a.G - 1) / a.G));
  a.mask = mask_kind;
  a.lens = lens;
  a.scale = (float)(scale * 1.4426950408889634);
  a.dscale = (float)scale;
  a.stats = stats;
  a.id_s = idesc(false, false, 128);
  a.id64_km = idesc(false, true, 64, 64);
  a.id64_mm = idesc(true, true, 64, 64);
  a.id_cs = idesc(true, false, 16);
  a.id128_pv = idesc(false, true, 64, 128);
  a.id128_mm = idesc(true, true, 64, 128);
  a.csq = a.csk = a.csv = nullptr;
  a.ldcsq = a.ldcsk = a.ldcsv = 0;
  a.trace = g_trace;
  return LS2_OK;
}

}  // namespace atc
}  // namespace ls2

using namespace ls2;

extern "C" {

/* debugging aid: per-CTA phase timestamps (globaltimer ns, [grid][8]) of the next
 * attention_tc launches go to `buf` (NULL turns it off) */
int ls2_attention_tc_trace(void* buf) {
  atc::g_trace = (unsigned long long*)buf;
  return LS2_OK;
}

int ls2_attention_tc_supported(int64_t lq, int64_t lk, int64_t hd, int dtype) {
  static const bool off = [] {
    const char* e = std::getenv("LS2_ATTN_TC");
    return e && e[0] == '0';
  }();
  if (off || dtype != LS2_F16 || hd != 64 || lq < 1 || lk < 1) return 0;
  if (lq <= 128 && lk <= 128) return 1;
  return lq == lk && lq <= 128 * atc::kFlashMaxChunks;     // flash kernels: self-attention
}

int ls2_attention_tc_fwd(const void* q, int64_t ldq, const void* k, int64_t ldk, const void* v,
                         int64_t ldv, void* stats, void* o, int64_t ldo, int64_t batch,
                         int64_t heads, int64_t lq, int64_t lk, int64_t hd, int mask_kind,
                         const int64_t* lens, double scale, void* stream) {
  if (!ls2_attention_tc_supported(lq, lk, hd, LS2_F16))
    return fail(LS2_ERR_SHAPE, "attention_tc_fwd: needs fp16, hd == 64, L <= 128 (or Lq == Lk <= 512)");
  if (mask_kind == LS2_MASK_PADDING && !lens) return fail(LS2_ERR_SHAPE, "attention_tc: no lens");
  if (mask_kind == LS2_MASK_DENSE) return fail(LS2_ERR_SHAPE, "attention_tc: dense masks unsupported");
  if (mask_kind == LS2_MASK_CAUSAL && lq != lk) return fail(LS2_ERR_SHAPE, "attention_tc: causal needs lq == lk");
  if (!atc::aligned16(q, ldq) || !atc::aligned16(k, ldk) || !atc::aligned16(v, ldv) ||
      !atc::aligned16(o, ldo))
    return fail(LS2_ERR_SHAPE, "attention_tc: operands need 16-byte alignment");
  if (batch <= 0 || heads <= 0) return LS2_OK;
  atc::Args a;
  atc::fill_args(a, batch, heads, lq, lk, mask_kind, lens, scale, (float2*)stats);
  CUtensorMap mq, mk, mv, mo;
  const int64_t cols = heads * 64;
  if (lq > 128 || lk > 128) {      // flash: stats are [B][H][Lq][4] floats
    if (!atc::make_map3_rows(&mq, q, cols, lq, batch, ldq, 128) ||
        !atc::make_map3_rows(&mk, k, cols, lk, batch, ldk, 128) ||
        !atc::make_map3_rows(&mv, v, cols, lk, batch, ldv, 128) ||
        !atc::make_map3_rows(&mo, o, cols, lq, batch, ldo, 128))
      return fail(LS2_ERR_CUDA, "attention_flash_fwd: cuTensorMapEncodeTiled failed");
    static bool fattr = false;
    if (!fattr) {
      cudaFuncSetAttribute(atc::attn_flash_fwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)atc::kFlashFwdSmem);
      fattr = true;
    }
    const int64_t nqb = (lq + 127) / 128;
    atc::attn_flash_fwd_kernel<<<(unsigned)(batch * heads * nqb), atc::kThreads,
                                 atc::kFlashFwdSmem, as_stream(stream)>>>(mq, mk, mv, mo, a);
    return check_launch("attention_flash_fwd");
  }
  if (!atc::make_map3(&mq, q, cols, lq, batch, ldq, a.G) ||
      !atc::make_map3(&mk, k, cols, lk, batch, ldk, a.G) ||
      !atc::make_map3(&mv, v, cols, lk, batch, ldv, a.G) ||
      !atc::make_map3(&mo, o, cols, lq, batch, ldo, a.G))
    return fail(LS2_ERR_CUDA, "attention_tc_fwd: cuTensorMapEncodeTiled failed");
  if (lq > 64 || lk > 64) {
    static bool attr128 = false;
    if (!attr128) {
      cudaFuncSetAttribute(atc::attn_tc128_fwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)atc::kFwd128Smem);
      attr128 = true;
    }
    atc::attn_tc128_fwd_kernel<<<(unsigned)(batch * heads), atc::kThreads, atc::kFwd128Smem,
                                 as_stream(stream)>>>(mq, mk, mv, mo, a);
    return check_launch("attention_tc128_fwd");
  }
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(atc::attn_tc_fwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)atc::kFwdSmem);
    attr = true;
  }
  const int grid = (a.ntiles + 1) / 2;
  atc::attn_tc_fwd_kernel<<<grid, atc::kThreads, atc::kFwdSmem, as_stream(stream)>>>(mq, mk, mv, mo,
                                                                                     a);
  return check_launch("attention_tc_fwd");
}

int ls2_attention_tc_bwd(const void* q, int64_t ldq, const void* k, int64_t ldk, const void* v,
                         int64_t ldv, const void* stats, const void* dout, int64_t lddo, void* dq,
                         int64_t lddq, void* dk, int64_t lddk, void* dv, int64_t lddv,
                         int64_t batch, int64_t heads, int64_t lq, int64_t lk, int64_t hd,
                         int mask_kind, const int64_t* lens, double scale, double* csq,
                         int64_t ldcsq, double* csk, int64_t ldcsk, double* csv, int64_t ldcsv,
                         void* stream) {
  if (!ls2_attention_tc_supported(lq, lk, hd, LS2_F16))
    return fail(LS2_ERR_SHAPE, "attention_tc_bwd: needs fp16, hd == 64, L <= 128");
  if (mask_kind == LS2_MASK_PADDING && !lens) return fail(LS2_ERR_SHAPE, "attention_tc: no lens");
  if (mask_kind == LS2_MASK_DENSE) return fail(LS2_ERR_SHAPE, "attention_tc: dense masks unsupported");
  if (mask_kind == LS2_MASK_CAUSAL && lq != lk) return fail(LS2_ERR_SHAPE, "attention_tc: causal needs lq == lk");
  if (!atc::aligned16(q, ldq) || !atc::aligned16(k, ldk) || !atc::aligned16(v, ldv) ||
      !atc::aligned16(dout, lddo) || !atc::aligned16(dq, lddq) || !atc::aligned16(dk, lddk) ||
      !atc::aligned16(dv, lddv))
    return fail(LS2_ERR_SHAPE, "attention_tc: operands need 16-byte alignment");
  if (batch <= 0 || heads <= 0) return LS2_OK;
  atc::Args a;
  atc::fill_args(a, batch, heads, lq, lk, mask_kind, lens, scale,
                 const_cast<float2*>((const float2*)stats));
  a.csq = csq; a.csk = csk; a.csv = csv;
  a.ldcsq = ldcsq; a.ldcsk = ldcsk; a.ldcsv = ldcsv;
  CUtensorMap mq, mk, mv, mdo, mdq, mdk, mdv;
  const int64_t cols = heads * 64;
  if (!atc::make_map3(&mq, q, cols, lq, batch, ldq, a.G) ||
      !atc::make_map3(&mk, k, cols, lk, batch, ldk, a.G) ||
      !atc::make_map3(&mv, v, cols, lk, batch, ldv, a.G) ||
      !atc::make_map3(&mdo, dout, cols, lq, batch, lddo, a.G) ||
      !atc::make_map3(&mdq, dq, cols, lq, batch, lddq, a.G) ||
      !atc::make_map3(&mdk, dk, cols, lk, batch, lddk, a.G) ||
      !atc::make_map3(&mdv, dv, cols, lk, batch, lddv, a.G))
    return fail(LS2_ERR_CUDA, "attention_tc_bwd: cuTensorMapEncodeTiled failed");
  if (lq > 64 || lk > 64) {
    static bool attr128 = false;
    if (!attr128) {
      cudaFuncSetAttribute(atc::attn_tc128_bwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)atc::kBwd128Smem);
      attr128 = true;
    }
    atc::attn_tc128_bwd_kernel<<<(unsigned)(batch * heads), atc::kThreads, atc::kBwd128Smem,
                                 as_stream(stream)>>>(mq, mk, mv, mdo, mdq, mdk, mdv, a);
    return check_launch("attention_tc128_bwd");
  }
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(atc::attn_tc_bwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)atc::kBwdSmem);
    attr = true;
  }
  const int grid = (a.ntiles + 1) / 2;
  atc::attn_tc_bwd_kernel<<<grid, atc::kThreads, atc::kBwdSmem, as_stream(stream)>>>(
      mq, mk, mv, mdo, mdq, mdk, mdv, a);
  return check_launch("attention_tc_bwd");
}

// the backward with the forward's output O (ctx): the flash kernels (Lq == Lk > 128)
// need D = rowsum(dO * O); shorter rows ignore it and take ls2_attention_tc_bwd
int ls2_attention_tc_bwd_o(const void* q, int64_t ldq, const void* k, int64_t ldk, const void* v,
                           int64_t ldv, const void* o, int64_t ldo, void* stats, const void* dout,
                           int64_t lddo, void* dq, int64_t lddq, void* dk, int64_t lddk, void* dv,
                           int64_t lddv, int64_t batch, int64_t heads, int64_t lq, int64_t lk,
                           int64_t hd, int mask_kind, const int64_t* lens, double scale,
                           double* csq, int64_t ldcsq, double* csk, int64_t ldcsk, double* csv,
                           int64_t ldcsv, void* stream) {
  if (lq <= 128 && lk <= 128)
    return ls2_attention_tc_bwd(q, ldq, k, ldk, v, ldv, stats, dout, lddo, dq, lddq, dk, lddk, dv,
                                lddv, batch, heads, lq, lk, hd, mask_kind, lens, scale, csq, ldcsq,
                                csk, ldcsk, csv, ldcsv, stream);
  if (!ls2_attention_tc_supported(lq, lk, hd, LS2_F16))
    return fail(LS2_ERR_SHAPE, "attention_flash_bwd: needs fp16, hd == 64, Lq == Lk <= 512");
  if (!o) return fail(LS2_ERR_SHAPE, "attention_flash_bwd: needs the forward output O");
  if (mask_kind == LS2_MASK_PADDING && !lens) return fail(LS2_ERR_SHAPE, "attention_tc: no lens");
  if (mask_kind == LS2_MASK_DENSE) return fail(LS2_ERR_SHAPE, "attention_tc: dense masks unsupported");
  if (!atc::aligned16(q, ldq) || !atc::aligned16(k, ldk) || !atc::aligned16(v, ldv) ||
      !atc::aligned16(o, ldo) || !atc::aligned16(dout, lddo) || !atc::aligned16(dq, lddq) ||
      !atc::aligned16(dk, lddk) || !atc::aligned16(dv, lddv))
    return fail(LS2_ERR_SHAPE, "attention_tc: operands need 16-byte alignment");
  if (batch <= 0 || heads <= 0) return LS2_OK;
  atc::Args a;
  atc::fill_args(a, batch, heads, lq, lk, mask_kind, lens, scale, (float2*)stats);
  a.csq = csq; a.csk = csk; a.csv = csv;
  a.ldcsq = ldcsq; a.ldcsk = ldcsk; a.ldcsv = ldcsv;
  CUtensorMap mq, mk, mv, mo, mdo, mdq, mdk, mdv;
  const int64_t cols = heads * 64;
  if (!atc::make_map3_rows(&mq, q, cols, lq, batch, ldq, 128) ||
      !atc::make_map3_rows(&mk, k, cols, lk, batch, ldk, 128) ||
      !atc::make_map3_rows(&mv, v, cols, lk, batch, ldv, 128) ||
      !atc::make_map3_rows(&mo, o, cols, lq, batch, ldo, 128) ||
      !atc::make_map3_rows(&mdo, dout, cols, lq, batch, lddo, 128) ||
      !atc::make_map3_rows(&mdq, dq, cols, lq, batch, lddq, 128) ||
      !atc::make_map3_rows(&mdk, dk, cols, lk, batch, lddk, 128) ||
      !atc::make_map3_rows(&mdv, dv, cols, lk, batch, lddv, 128))
    return fail(LS2_ERR_CUDA, "attention_flash_bwd: cuTensorMapEncodeTiled failed");
  static bool fattr = false;
  if (!fattr) {
    cudaFuncSetAttribute(atc::attn_flash_dq_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)atc::kFlashDqSmem);
    cudaFuncSetAttribute(atc::attn_flash_dkv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)atc::kFlashDkvSmem);
    fattr = true;
  }
  const int64_t nqb = (lq + 127) / 128, nkb = (lk + 127) / 128;
  atc::attn_flash_dq_kernel<<<(unsigned)(batch * heads * nqb), atc::kThreads, atc::kFlashDqSmem,
                              as_stream(stream)>>>(mq, mk, mv, mdo, mo, mdq, a);
  if (int rc = check_launch("attention_flash_dq")) return rc;
  atc::attn_flash_dkv_kernel<<<(unsigned)(batch * heads * nkb), atc::kThreads, atc::kFlashDkvSmem,
                               as_stream(stream)>>>(mq, mk, mv, mdo, mdk, mdv, a);
  return check_launch("attention_flash_dkv");
}

}  // extern "C"
