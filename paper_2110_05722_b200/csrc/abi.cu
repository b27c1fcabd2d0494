// Status plumbing and the counter-RNG / mask kernels.
//   F/numerics.py:133-163 (splitmix64 counter RNG, derive_seed)
//   F/kernels.py:155-166  (make_dropout_mask)
#include <mutex>

#include "common.cuh"

namespace ls2 {

static thread_local std::string t_err;
std::atomic<int64_t> g_launches{0};

void set_error(const std::string& msg) { t_err = msg; }
int fail(int code, const std::string& msg) {
  t_err = msg;
  return code;
}

// U[0,1) doubles, bit-identical to rand_uniform_array(seed, start, n)
__global__ void rand_uniform_kernel(double* out, uint64_t seed, int64_t start, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t z = mix64(seed + (uint64_t)(start + i) * kPhi);
    out[i] = (double)(z >> 11) * (1.0 / 9007199254740992.0);
  }
}

__global__ void dropout_bits_kernel(uint8_t* bits, int64_t n, uint64_t seed, const uint64_t* seed_ptr, uint64_t thresh) {
  int64_t groups = (n + 7) / 8;
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < groups;
       g += (int64_t)gridDim.x * blockDim.x) {
    uint32_t b = keep_byte(seed_ptr ? *seed_ptr : seed, (uint64_t)g * 8, thresh);
    int64_t valid = n - g * 8;
    if (valid < 8) b &= (1u << valid) - 1u;
    bits[g] = (uint8_t)b;
  }
}

// 32 keep bits with the integer work split across the FMA-heavy pipe (64-bit
// products, the last shift done as mul.hi by 2) and the ALU pipe (shifts, xors,
// the compare): each pipe takes one warp instruction every other cycle, so
// balancing them is what sets the draw rate (ncu: fmaheavy and alu both busy).  The compare is a carry chain: z3hi + ~Thi carries
// out iff z3hi > Thi, and addc shifts that carry into the word MSB-first; ties
// (z3hi == Thi, probability 2^-32 per draw) are caught by a running max of the
// sums and the word is then redrawn with the exact 64-bit form.
__device__ __forceinline__ uint32_t mulhi_u32(uint32_t a, uint32_t b) {
  uint32_t r;
  asm("mul.hi.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}

__device__ __noinline__ uint32_t keep_word_exact(uint64_t seed, uint64_t first, uint64_t thresh) {
  return keep_bits_n<32>(seed, first, thresh);
}

__device__ __forceinline__ uint32_t keep_word_fast(uint64_t seed, uint64_t first, uint64_t thresh) {
  constexpr uint32_t kAlo = (uint32_t)kMixA, kAhi = (uint32_t)(kMixA >> 32);
  constexpr uint32_t kBlo = (uint32_t)kMixB, kBhi = (uint32_t)(kMixB >> 32);
  const uint64_t T = thresh << 11;
  const uint32_t nThi = ~(uint32_t)(T >> 32);
  uint64_t x = seed + (first + 31) * kPhi;        // MSB-first: element first+31 .. first
  uint32_t b = 0, tie = 0;
#pragma unroll
  for (int e = 31; e >= 0; --e) {
    const uint32_t xlo = (uint32_t)x, xhi = (uint32_t)(x >> 32);
    // y1 = x ^ (x >> 30)   (ALU: funnel shift + xors)
    const uint32_t y1lo = xlo ^ __funnelshift_r(xlo, xhi, 30);
    const uint32_t y1hi = xhi ^ (xhi >> 30);
    // z1 = y1 * A
    const uint64_t p = (uint64_t)y1lo * kAlo;
    const uint32_t z1lo = (uint32_t)p;
    const uint32_t z1hi = (uint32_t)(p >> 32) + y1lo * kAhi + y1hi * kAlo;
    // y2 = z1 ^ (z1 >> 27)  (ALU)
    const uint32_t y2lo = z1lo ^ __funnelshift_r(z1lo, z1hi, 27);
    const uint32_t y2hi = z1hi ^ (z1hi >> 27);
    // high word of z2 = y2 * B, then z3 = z2 ^ (z2 >> 31)
    const uint32_t z2hi = __umulhi(y2lo, kBlo) + y2lo * kBhi + y2hi * kBlo;
    const uint32_t z3hi = z2hi ^ mulhi_u32(z2hi, 2u);
    uint32_t sum;
    asm("add.cc.u32 %0, %2, %3;\n\taddc.u32 %1, %1, %1;"
        : "=r"(sum), "+r"(b) : "r"(z3hi), "r"(nThi));
    tie = max(tie, sum);                            // sum == ~0 <=> z3hi == Thi
    x -= kPhi;
  }
  if (__builtin_expect(tie == 0xFFFFFFFFu, 0)) return keep_word_exact(seed, first, thresh);
  return b;
}

// Every dropout site of a step in one launch (the mask bank).  desc rows
// {seed slot, elements, first 32-bit word} (int64), sorted by first word;
// site s fills words [first_s, first_s + ceil(n_s/32)) of `words` with the
// keep bits of elements [0, n_s) drawn with seed seeds[slot_s] (bits past n_s
// are 0).  One thread per 32-element word, grid-stride, coalesced 4-byte stores.
__global__ void __launch_bounds__(256) dropout_bits_multi_kernel(
    const int64_t* __restrict__ desc, int nsites, int64_t total_words, uint32_t* __restrict__ words,
    const uint64_t* __restrict__ seeds, uint64_t thresh, const int64_t* __restrict__ stamp,
    const int64_t* __restrict__ want) {
  if (stamp && want && *stamp == *want) return;    // bits already drawn for this step
  __shared__ int64_t s_first[65];
  __shared__ int64_t s_n[64];
  __shared__ uint64_t s_seed[64];
  for (int i = threadIdx.x; i < nsites; i += blockDim.x) {
    s_first[i] = desc[4 * i + 2];
    s_n[i] = desc[4 * i + 1];
    s_seed[i] = seeds[desc[4 * i]];
  }
  if (threadIdx.x == 0) s_first[nsites] = total_words;
  __syncthreads();
  int site = 0;
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < total_words;
       w += (int64_t)gridDim.x * blockDim.x) {
    while (w >= s_first[site + 1]) ++site;           // w only grows: sites in order
    const int64_t e0 = (w - s_first[site]) * 32;
    uint32_t b = keep_word_fast(s_seed[site], (uint64_t)e0, thresh);
    const int64_t valid = s_n[site] - e0;
    if (valid < 32) b &= valid <= 0 ? 0u : ((1u << valid) - 1u);
    words[w] = b;
  }
}

template <typename T>
__global__ void bits_to_dense_kernel(const uint8_t* bits, T* dense, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    dense[i] = cvt<T>((float)((bits[i >> 3] >> (i & 7)) & 1));
}

template <typename T>
__global__ void dense_to_bits_kernel(const T* dense, uint8_t* bits, int64_t n) {
  int64_t groups = (n + 7) / 8;
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < groups;
       g += (int64_t)gridDim.x * blockDim.x) {
    uint32_t b = 0;
    for (int e = 0; e < 8 && g * 8 + e < n; ++e)
      b |= (uint32_t)(cvt<float>(dense[g * 8 + e]) != 0.0f) << e;
    bits[g] = (uint8_t)b;
  }
}

}  // namespace ls2

using namespace ls2;

// Up to kMaxSpans copies of 8-byte words in ONE launch (the step's batch and seed
// tables, read straight from pinned host memory through UVA): one kernel node in a
// captured step instead of one copy-engine node per buffer.  Thread w copies word
// w of the concatenation, so every word crosses the bus in one round trip.
constexpr int kMaxSpans = 8;
struct CopySpans {
  uint64_t* dst[kMaxSpans];
  const uint64_t* src[kMaxSpans];
  int64_t start[kMaxSpans + 1];   // word offsets of each span in the concatenation
  int n;
};

__global__ void copy_spans_kernel(CopySpans s) {
  const int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (w >= s.start[s.n]) return;
  int i = 0;
  while (i + 1 < s.n && w >= s.start[i + 1]) ++i;
  const int64_t k = w - s.start[i];
  s.dst[i][k] = s.src[i][k];
}

extern "C" {

const char* ls2_last_error(void) { return t_err.c_str(); }
int ls2_version(void) { return 1; }
int ls2_num_kernels_launched(int64_t* out) {
  *out = g_launches.load();
  return LS2_OK;
}

int ls2_rand_uniform(double* out, uint64_t seed, int64_t start, int64_t n, void* stream) {
  if (n <= 0) return LS2_OK;
  rand_uniform_kernel<<<grid_for(n), 256, 0, as_stream(stream)>>>(out, seed, start, n);
  return check_launch("rand_uniform");
}

int ls2_dropout_bits(uint8_t* bits, int64_t n, uint64_t seed, const uint64_t* seed_ptr, uint64_t thresh, void* stream) {
  if (n <= 0) return LS2_OK;
  dropout_bits_kernel<<<grid_for(ceil_div(n, 8)), 256, 0, as_stream(stream)>>>(bits, n, seed, seed_ptr,
                                                                                thresh);
  return check_launch("dropout_bits");
}

int ls2_dropout_bits_multi_ex(const int64_t* desc, int nsites, int64_t total_words, uint8_t* base,
                              const uint64_t* seeds, uint64_t thresh, const int64_t* stamp,
                              const int64_t* want, int ctas_per_sm, void* stream) {
  if (total_words <= 0 || nsites <= 0) return LS2_OK;
  if (nsites > 64) return fail(LS2_ERR_SHAPE, "dropout_bits_multi: at most 64 sites");
  if ((reinterpret_cast<uintptr_t>(base) & 3) != 0)
    return fail(LS2_ERR_SHAPE, "dropout_bits_multi: base must be 4-byte aligned");
  static int occ = 0;
  if (!occ) {
    int per = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, dropout_bits_multi_kernel, 256, 0);
    occ = per > 0 ? per : 8;
  }
  const int per = ctas_per_sm > 0 ? std::min(ctas_per_sm, occ) : occ;
  const int g = (int)std::min<int64_t>((int64_t)kNumSMs * per, ceil_div(total_words, (int64_t)256));
  dropout_bits_multi_kernel<<<g, 256, 0, as_stream(stream)>>>(
      desc, nsites, total_words, reinterpret_cast<uint32_t*>(base), seeds, thresh, stamp, want);
  return check_launch("dropout_bits_multi");
}

int ls2_dropout_bits_multi(const int64_t* desc, int nsites, int64_t total_words, uint8_t* base,
                           const uint64_t* seeds, uint64_t thresh, const int64_t* stamp,
                           const int64_t* want, void* stream) {
  return ls2_dropout_bits_multi_ex(desc, nsites, total_words, base, seeds, thresh, stamp, want, 0,
                                   stream);
}

int ls2_copy_spans(void* const* dst, const void* const* src, const int64_t* nbytes, int n,
                   void* stream) {
  if (n < 0 || n > kMaxSpans) return fail(LS2_ERR_SHAPE, "copy_spans: 0..8 spans");
  CopySpans s{};
  s.n = n;
  int64_t words = 0;
  for (int i = 0; i < n; ++i) {
    if ((nbytes[i] & 7) || (reinterpret_cast<uintptr_t>(dst[i]) & 7) ||
        (reinterpret_cast<uintptr_t>(src[i]) & 7))
      return fail(LS2_ERR_SHAPE, "copy_spans: 8-byte sizes and alignment");
    s.dst[i] = static_cast<uint64_t*>(dst[i]);
    s.src[i] = static_cast<const uint64_t*>(src[i]);
    s.start[i] = words;
    words += nbytes[i] / 8;
  }
  s.start[n] = words;
  if (words == 0) return LS2_OK;
  copy_spans_kernel<<<(unsigned)ceil_div(words, 256), 256, 0, as_stream(stream)>>>(s);
  return check_launch("copy_spans");
}

int ls2_bits_to_dense(const uint8_t* bits, void* dense, int dtype, int64_t n, void* stream) {
  if (n <= 0) return LS2_OK;
  return LS2_DISPATCH_ONE(dtype, "bits_to_dense", [&] {
    bits_to_dense_kernel<Tx><<<grid_for(n), 256, 0, as_stream(stream)>>>(bits, (Tx*)dense, n);
    return check_launch("bits_to_dense");
  });
}

int ls2_dense_to_bits(const void* dense, int dtype, uint8_t* bits, int64_t n, void* stream) {
  if (n <= 0) return LS2_OK;
  return LS2_DISPATCH_ONE(dtype, "dense_to_bits", [&] {
    dense_to_bits_kernel<Tx><<<grid_for(ceil_div(n, 8)), 256, 0, as_stream(stream)>>>(
        (const Tx*)dense, bits, n);
    return check_launch("dense_to_bits");
  });
}

}  // extern "C"
