// Shared device/host helpers for the sm_100a hot-path kernels.
#pragma once

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <map>
#include <mutex>
#include <tuple>
#include <string>
#include <type_traits>

#include "../../include/ls2.h"

namespace ls2 {

// ---------------------------------------------------------------------------
// status / error text (host)
// ---------------------------------------------------------------------------
void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
extern std::atomic<int64_t> g_launches;

inline int check_launch(const char* what) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(LS2_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  return LS2_OK;
}

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

constexpr int kNumSMs = 148;  // B200; grid sizes below are fixed for determinism

// ---------------------------------------------------------------------------
// element types
// ---------------------------------------------------------------------------
template <typename T> struct CompOf { using type = float; };
template <> struct CompOf<double> { using type = double; };

template <typename C, typename T> __device__ __forceinline__ C to_c(T v);
template <> __device__ __forceinline__ float to_c<float, __half>(__half v) { return __half2float(v); }
template <> __device__ __forceinline__ float to_c<float, __nv_bfloat16>(__nv_bfloat16 v) { return __bfloat162float(v); }
template <> __device__ __forceinline__ float to_c<float, float>(float v) { return v; }
template <> __device__ __forceinline__ double to_c<double, double>(double v) { return v; }
template <> __device__ __forceinline__ double to_c<double, float>(float v) { return (double)v; }

template <typename T, typename C> __device__ __forceinline__ T from_c(C v);
template <> __device__ __forceinline__ __half from_c<__half, float>(float v) { return __float2half_rn(v); }
template <> __device__ __forceinline__ __nv_bfloat16 from_c<__nv_bfloat16, float>(float v) { return __float2bfloat16_rn(v); }
template <> __device__ __forceinline__ float from_c<float, float>(float v) { return v; }
template <> __device__ __forceinline__ double from_c<double, double>(double v) { return v; }
template <> __device__ __forceinline__ float from_c<float, double>(double v) { return (float)v; }

// general conversion (single rounding from double where possible)
template <typename To, typename From>
__device__ __forceinline__ To cvt(From v) {
  if constexpr (std::is_same<To, From>::value) {
    return v;
  } else if constexpr (std::is_same<To, __half>::value) {
    if constexpr (std::is_same<From, double>::value) return __double2half(v);
    else return __float2half_rn((float)v);
  } else if constexpr (std::is_same<To, __nv_bfloat16>::value) {
    if constexpr (std::is_same<From, double>::value) return __double2bfloat16(v);
    else return __float2bfloat16_rn((float)v);
  } else if constexpr (std::is_same<From, __half>::value) {
    return (To)__half2float(v);
  } else if constexpr (std::is_same<From, __nv_bfloat16>::value) {
    return (To)__bfloat162float(v);
  } else {
    return (To)v;
  }
}

// IEEE-exact arithmetic in the compute type (no FMA contraction) so the fused
// element-wise ops reproduce numpy's float32 op order bit for bit.
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }

// 8 consecutive elements; loaded/stored with 16-byte transactions.
template <typename T>
struct alignas(16) Pack8 {
  T v[8];
};

// elements 2e, 2e+1 of a pack widened to fp32 (one packed conversion for 16-bit types)
template <typename T> __device__ __forceinline__ float2 pair_f2(const Pack8<T>& p, int e);
template <> __device__ __forceinline__ float2 pair_f2<__half>(const Pack8<__half>& p, int e) {
  return __half22float2(*reinterpret_cast<const __half2*>(&p.v[2 * e]));
}
template <> __device__ __forceinline__ float2 pair_f2<__nv_bfloat16>(const Pack8<__nv_bfloat16>& p, int e) {
  return __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&p.v[2 * e]));
}
template <> __device__ __forceinline__ float2 pair_f2<float>(const Pack8<float>& p, int e) {
  return make_float2(p.v[2 * e], p.v[2 * e + 1]);
}

// packed fp32 pair arithmetic (sm_100 FFMA2 / FADD2 / FMUL2), each lane rounded
// exactly like its scalar counterpart
__device__ __forceinline__ float2 f2fma(float2 a, float2 b, float2 c) {
  float2 d;
  asm("{.reg .b64 ra, rb, rc, rd;\n mov.b64 ra, {%2, %3};\n mov.b64 rb, {%4, %5};\n"
      " mov.b64 rc, {%6, %7};\n fma.rn.f32x2 rd, ra, rb, rc;\n mov.b64 {%0, %1}, rd;}"
      : "=f"(d.x), "=f"(d.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return d;
}
__device__ __forceinline__ float2 f2add(float2 a, float2 b) {
  float2 d;
  asm("{.reg .b64 ra, rb, rd;\n mov.b64 ra, {%2, %3};\n mov.b64 rb, {%4, %5};\n"
      " add.rn.f32x2 rd, ra, rb;\n mov.b64 {%0, %1}, rd;}"
      : "=f"(d.x), "=f"(d.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return d;
}
__device__ __forceinline__ float2 f2mul(float2 a, float2 b) {
  float2 d;
  asm("{.reg .b64 ra, rb, rd;\n mov.b64 ra, {%2, %3};\n mov.b64 rb, {%4, %5};\n"
      " mul.rn.f32x2 rd, ra, rb;\n mov.b64 {%0, %1}, rd;}"
      : "=f"(d.x), "=f"(d.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return d;
}
__device__ __forceinline__ float2 f2s(float v) { return make_float2(v, v); }

template <typename T>
__device__ __forceinline__ Pack8<T> ld8(const T* p) {
  Pack8<T> r;
  constexpr int kWords = sizeof(Pack8<T>) / 16;
  const uint4* s = reinterpret_cast<const uint4*>(p);
  uint4* d = reinterpret_cast<uint4*>(&r);
#pragma unroll
  for (int i = 0; i < kWords; ++i) d[i] = __ldg(s + i);
  return r;
}

template <typename T>
__device__ __forceinline__ Pack8<T> ld8_stream(const T* p) {  // evict-first streaming read
  Pack8<T> r;
  constexpr int kWords = sizeof(Pack8<T>) / 16;
  const uint4* s = reinterpret_cast<const uint4*>(p);
  uint4* d = reinterpret_cast<uint4*>(&r);
#pragma unroll
  for (int i = 0; i < kWords; ++i) d[i] = __ldcs(s + i);
  return r;
}

template <typename T>
__device__ __forceinline__ void st8(T* p, const Pack8<T>& v) {
  constexpr int kWords = sizeof(Pack8<T>) / 16;
  uint4* d = reinterpret_cast<uint4*>(p);
  const uint4* s = reinterpret_cast<const uint4*>(&v);
#pragma unroll
  for (int i = 0; i < kWords; ++i) d[i] = s[i];
}

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

// ---------------------------------------------------------------------------
// splitmix64 counter RNG (F/numerics.py:133-155)
// ---------------------------------------------------------------------------
constexpr uint64_t kPhi = 0x9E3779B97F4A7C15ull;
constexpr uint64_t kMixA = 0xBF58476D1CE4E5B9ull;
constexpr uint64_t kMixB = 0x94D049BB133111EBull;

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * kMixA;
  z = (z ^ (z >> 27)) * kMixB;
  return z ^ (z >> 31);
}

// keep test  (mix64(x) >> 11) >= thresh  <=>  mix64(x) >= T,  T = thresh << 11,
// evaluated on 32-bit halves: only the HIGH word of the last multiply is formed
// unless it ties with T's high word (probability 2^-32), when the low word
// decides.  Bit-identical to the 64-bit form (tests pin it against the
// reference RNG), ~20 integer instructions per draw instead of ~26.
__device__ __forceinline__ bool keep_draw(uint32_t xlo, uint32_t xhi, uint32_t Thi, uint32_t Tlo) {
  constexpr uint32_t kAlo = (uint32_t)kMixA, kAhi = (uint32_t)(kMixA >> 32);
  constexpr uint32_t kBlo = (uint32_t)kMixB, kBhi = (uint32_t)(kMixB >> 32);
  const uint32_t y1lo = xlo ^ __funnelshift_r(xlo, xhi, 30);
  const uint32_t y1hi = xhi ^ (xhi >> 30);
  const uint64_t p = (uint64_t)y1lo * kAlo;
  const uint32_t z1lo = (uint32_t)p;
  const uint32_t z1hi = (uint32_t)(p >> 32) + y1lo * kAhi + y1hi * kAlo;
  const uint32_t y2lo = z1lo ^ __funnelshift_r(z1lo, z1hi, 27);
  const uint32_t y2hi = z1hi ^ (z1hi >> 27);
  const uint32_t z2hi = __umulhi(y2lo, kBlo) + y2lo * kBhi + y2hi * kBlo;
  const uint32_t z3hi = z2hi ^ (z2hi >> 31);
  if (__builtin_expect(z3hi != Thi, 1)) return z3hi > Thi;
  const uint32_t z2lo = y2lo * kBlo;
  const uint32_t z3lo = z2lo ^ __funnelshift_r(z2lo, z2hi, 31);
  return z3lo >= Tlo;
}

// keep bits for flat elements [first, first + N): bit e set iff
// mix(seed + (first+e)*phi)>>11 >= thresh (F/numerics.py:145-155, F/kernels.py:155-166).
// The counter is advanced by +phi (strength-reduced from the multiply).
template <int N>
__device__ __forceinline__ uint32_t keep_bits_n(uint64_t seed, uint64_t first, uint64_t thresh) {
  uint64_t x = seed + first * kPhi;
  const uint64_t T = thresh << 11;        // thresh <= 2^53
  const uint32_t Thi = (uint32_t)(T >> 32), Tlo = (uint32_t)T;
  uint32_t b = 0;
#pragma unroll
  for (int e = 0; e < N; ++e) {
    b |= (uint32_t)keep_draw((uint32_t)x, (uint32_t)(x >> 32), Thi, Tlo) << e;
    x += kPhi;
  }
  return b;
}

// bit e of w as 0 or 1 in type C: a select, not an integer->float conversion
// (I2FP on the conversion pipe was a throttle in the mask-applying kernels);
// the value, and so every product with it, is unchanged
template <typename C>
__device__ __forceinline__ C bitval(uint32_t w, int e) {
  return ((w >> e) & 1u) ? (C)1 : (C)0;
}

__device__ __forceinline__ uint32_t keep_byte(uint64_t seed, uint64_t first, uint64_t thresh) {
  return keep_bits_n<8>(seed, first, thresh);
}

// ---------------------------------------------------------------------------
// reductions
// ---------------------------------------------------------------------------
template <typename T>
__device__ __forceinline__ T warp_sum(T v, int width = 32) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
    if (o < width) v += __shfl_xor_sync(0xffffffffu, v, o, width);
  return v;
}

template <typename T>
__device__ __forceinline__ T warp_max(T v, int width = 32) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
    if (o < width) v = max(v, __shfl_xor_sync(0xffffffffu, v, o, width));
  return v;
}

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// grid = min(work blocks, every resident slot on the chip): one full wave of a
// grid-stride kernel instead of 1.x waves with an idle tail
inline int resident_grid(const void* fn, int threads, size_t smem, int64_t want) {
  static std::mutex mu;
  static std::map<std::tuple<const void*, int, size_t>, int> cache;
  int per_sm = 0;
  {
    std::lock_guard<std::mutex> g(mu);
    auto key = std::make_tuple(fn, threads, smem);
    auto it = cache.find(key);
    if (it == cache.end()) {
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads, smem) != cudaSuccess) {
        cudaGetLastError();
        per_sm = 1;
      }
      if (per_sm < 1) per_sm = 1;
      cache[key] = per_sm;
    } else {
      per_sm = it->second;
    }
  }
  const int64_t cap = (int64_t)kNumSMs * per_sm;
  return (int)(want < 1 ? 1 : (want > cap ? cap : want));
}

inline int grid_for(int64_t work, int tpb = 256) {
  int64_t g = ceil_div(work, tpb);
  if (g > kNumSMs * 16) g = kNumSMs * 16;
  return (int)(g < 1 ? 1 : g);
}

}  // namespace ls2

// dtype dispatch over the (input, output) pairs the kernels are built for.
#define LS2_DISPATCH_IO(TIN, TOUT, NAME, ...)                                                  \
  [&]() -> int {                                                                             \
    if (TIN == LS2_F16 && TOUT == LS2_F16) { using Tin = __half; using Tout = __half; return __VA_ARGS__(); } \
    if (TIN == LS2_F16 && TOUT == LS2_F32) { using Tin = __half; using Tout = float; return __VA_ARGS__(); } \
    if (TIN == LS2_BF16 && TOUT == LS2_BF16) { using Tin = __nv_bfloat16; using Tout = __nv_bfloat16; return __VA_ARGS__(); } \
    if (TIN == LS2_BF16 && TOUT == LS2_F32) { using Tin = __nv_bfloat16; using Tout = float; return __VA_ARGS__(); } \
    if (TIN == LS2_F32 && TOUT == LS2_F32) { using Tin = float; using Tout = float; return __VA_ARGS__(); } \
    if (TIN == LS2_F32 && TOUT == LS2_F16) { using Tin = float; using Tout = __half; return __VA_ARGS__(); } \
    if (TIN == LS2_F32 && TOUT == LS2_BF16) { using Tin = float; using Tout = __nv_bfloat16; return __VA_ARGS__(); } \
    if (TIN == LS2_F64 && TOUT == LS2_F64) { using Tin = double; using Tout = double; return __VA_ARGS__(); } \
    return ::ls2::fail(LS2_ERR_DTYPE, std::string(NAME) + ": unsupported dtype pair");         \
  }()

#define LS2_DISPATCH_ONE(T, NAME, ...)                                                          \
  [&]() -> int {                                                                             \
    if (T == LS2_F16) { using Tx = __half; return __VA_ARGS__(); }                             \
    if (T == LS2_BF16) { using Tx = __nv_bfloat16; return __VA_ARGS__(); }                     \
    if (T == LS2_F32) { using Tx = float; return __VA_ARGS__(); }                              \
    if (T == LS2_F64) { using Tx = double; return __VA_ARGS__(); }                             \
    return ::ls2::fail(LS2_ERR_DTYPE, std::string(NAME) + ": unsupported dtype");              \
  }()
