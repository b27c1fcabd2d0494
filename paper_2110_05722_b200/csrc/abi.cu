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
