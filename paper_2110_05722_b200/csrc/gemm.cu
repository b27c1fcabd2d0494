// GEMMs on cuBLAS (tensor cores), row-major semantics.
//   replaces the blocked matmul of F/kernels.py:413-447 (the reference's
//   "plain blocked matmul" stand-in for cuBLAS)
//
// Stacked operands with two batch levels (i < n1, j < n2) are served either as
// one strided batch (when the two levels collapse to a single stride) or as a
// pointer-array batch whose pointers a tiny kernel writes into caller scratch.
// The pointer-array form lets the attention contractions read Q/K/V directly
// out of the fused [B, L, 3d] projection and write the context straight into
// the merged [B, L, d] layout, so no head split/merge copies exist.
#include <cublas_v2.h>

#include "common.cuh"

namespace ls2 {

struct Blas {
  cublasHandle_t h = nullptr;
  void* ws = nullptr;
  size_t ws_bytes = 0;
};

inline size_t esize(int t) { return t == LS2_F64 ? 8 : t == LS2_F32 ? 4 : 2; }
inline cudaDataType_t cuda_type(int t) {
  switch (t) {
    case LS2_F16: return CUDA_R_16F;
    case LS2_BF16: return CUDA_R_16BF;
    case LS2_F32: return CUDA_R_32F;
    default: return CUDA_R_64F;
  }
}

__global__ void fill_ptrs_kernel(const char* A, const char* B, char* C, int64_t n2, int64_t total,
                                 int64_t sA1, int64_t sA2, int64_t sB1, int64_t sB2, int64_t sC1,
                                 int64_t sC2, const void** out) {
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < total;
       b += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = b / n2, j = b % n2;
    out[b] = A + i * sA1 + j * sA2;
    out[total + b] = B + i * sB1 + j * sB2;
    out[2 * total + b] = C + i * sC1 + j * sC2;
  }
}

inline int blas_fail(cublasStatus_t s, const char* what) {
  return fail(LS2_ERR_CUBLAS, std::string(what) + ": cublas status " + std::to_string((int)s));
}

}  // namespace ls2

using namespace ls2;

extern "C" {

void* ls2_blas_create(void) {
  Blas* b = new Blas();
  if (cublasCreate(&b->h) != CUBLAS_STATUS_SUCCESS) {
    delete b;
    set_error("cublasCreate failed");
    return nullptr;
  }
  b->ws_bytes = 64ull << 20;
  if (cudaMalloc(&b->ws, b->ws_bytes) != cudaSuccess) {
    cublasDestroy(b->h);
    delete b;
    set_error("cudaMalloc(cublas workspace) failed");
    return nullptr;
  }
  cublasSetWorkspace(b->h, b->ws, b->ws_bytes);
  // fp32 compute, no TF32, no reduced-precision split-K reductions
  cublasSetMathMode(b->h, (cublasMath_t)(CUBLAS_DEFAULT_MATH |
                                         CUBLAS_MATH_DISALLOW_REDUCED_PRECISION_REDUCTION));
  return b;
}

void ls2_blas_destroy(void* p) {
  Blas* b = reinterpret_cast<Blas*>(p);
  if (!b) return;
  if (b->h) cublasDestroy(b->h);
  if (b->ws) cudaFree(b->ws);
  delete b;
}

int64_t ls2_gemm_scratch_bytes(int64_t n1, int64_t n2) { return 3 * n1 * n2 * (int64_t)sizeof(void*); }

int ls2_gemm(void* hp, int trans_a, int trans_b, int64_t m, int64_t n, int64_t k, double alpha,
             const void* A, int64_t lda, int64_t sA1, int64_t sA2, const void* B, int64_t ldb,
             int64_t sB1, int64_t sB2, double beta, void* C, int64_t ldc, int64_t sC1,
             int64_t sC2, int64_t n1, int64_t n2, int tab, int tc, void* ptr_scratch,
             void* stream) {
  Blas* b = reinterpret_cast<Blas*>(hp);
  if (!b) return fail(LS2_ERR_CUBLAS, "gemm: null blas handle");
  if (m <= 0 || n <= 0 || n1 <= 0 || n2 <= 0) return LS2_OK;
  const bool f64 = tab == LS2_F64;
  if (f64 != (tc == LS2_F64)) return fail(LS2_ERR_DTYPE, "gemm: f64 must not be mixed");
  if (!f64 && !(tc == tab || tc == LS2_F32)) return fail(LS2_ERR_DTYPE, "gemm: bad output dtype");
  cublasSetStream(b->h, as_stream(stream));
  const cublasComputeType_t ct = f64 ? CUBLAS_COMPUTE_64F : CUBLAS_COMPUTE_32F;
  const float af = (float)alpha, bf = (float)beta;
  const void* pa = f64 ? (const void*)&alpha : (const void*)&af;
  const void* pb = f64 ? (const void*)&beta : (const void*)&bf;
  const cublasOperation_t opA = trans_a ? CUBLAS_OP_T : CUBLAS_OP_N;
  const cublasOperation_t opB = trans_b ? CUBLAS_OP_T : CUBLAS_OP_N;
  const cudaDataType_t tAB = cuda_type(tab), tC = cuda_type(tc);
  const int64_t total = n1 * n2;
  cublasStatus_t s;
  if (total == 1) {
    s = cublasGemmEx(b->h, opB, opA, (int)n, (int)m, (int)k, pa, B, tAB, (int)ldb, A, tAB,
                     (int)lda, pb, C, tC, (int)ldc, ct, CUBLAS_GEMM_DEFAULT);
    return s == CUBLAS_STATUS_SUCCESS ? LS2_OK : blas_fail(s, "cublasGemmEx");
  }
  // collapse two batch levels into one stride when possible
  int64_t stA, stB, stC;
  bool strided = false;
  if (n2 == 1) {
    stA = sA1; stB = sB1; stC = sC1; strided = true;
  } else if (n1 == 1) {
    stA = sA2; stB = sB2; stC = sC2; strided = true;
  } else if (sA1 == n2 * sA2 && sB1 == n2 * sB2 && sC1 == n2 * sC2) {
    stA = sA2; stB = sB2; stC = sC2; strided = true;
  }
  if (strided) {
    s = cublasGemmStridedBatchedEx(b->h, opB, opA, (int)n, (int)m, (int)k, pa, B, tAB, (int)ldb,
                                   stB, A, tAB, (int)lda, stA, pb, C, tC, (int)ldc, stC,
                                   (int)total, ct, CUBLAS_GEMM_DEFAULT);
    return s == CUBLAS_STATUS_SUCCESS ? LS2_OK : blas_fail(s, "cublasGemmStridedBatchedEx");
  }
  if (!ptr_scratch) return fail(LS2_ERR_SHAPE, "gemm: pointer-array batch needs scratch");
  const size_t ea = esize(tab), ec = esize(tc);
  const void** ptrs = reinterpret_cast<const void**>(ptr_scratch);
  fill_ptrs_kernel<<<grid_for(total), 256, 0, as_stream(stream)>>>(
      (const char*)A, (const char*)B, (char*)C, n2, total, sA1 * ea, sA2 * ea, sB1 * ea, sB2 * ea,
      sC1 * ec, sC2 * ec, ptrs);
  int rc = check_launch("gemm_fill_ptrs");
  if (rc) return rc;
  s = cublasGemmBatchedEx(b->h, opB, opA, (int)n, (int)m, (int)k, pa, (const void* const*)(ptrs + total),
                          tAB, (int)ldb, (const void* const*)ptrs, tAB, (int)lda, pb,
                          (void* const*)(ptrs + 2 * total), tC, (int)ldc, (int)total, ct,
                          CUBLAS_GEMM_DEFAULT);
  return s == CUBLAS_STATUS_SUCCESS ? LS2_OK : blas_fail(s, "cublasGemmBatchedEx");
}

}  // extern "C"
