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
#include <cublasLt.h>
#include <cublas_v2.h>

#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>
#include <tuple>
#include <vector>
#include <cstring>
#include <string>

#include <algorithm>

#include "common.cuh"

namespace ls2 {

// cuBLASLt plan for one (shape, layout, dtype, epilogue, alignment) key
struct LtPlan {
  cublasLtMatmulDesc_t op = nullptr;
  cublasLtMatrixLayout_t a = nullptr, b = nullptr, c = nullptr;
  cublasLtMatmulAlgo_t algo;
  bool ok = false;
  char tag[96] = {0};
};

using LtKey = std::tuple<int, int, int64_t, int64_t, int64_t, int64_t, int64_t, int64_t, int, int,
                         int, int, int>;

struct Blas {
  cublasHandle_t h = nullptr;
  cublasLtHandle_t lt = nullptr;
  void* ws = nullptr;
  size_t ws_bytes = 0;
  std::map<LtKey, LtPlan> plans;
  std::mutex mu;
};

inline int align_of(const void* p) {
  uintptr_t v = reinterpret_cast<uintptr_t>(p);
  int a = 256;
  while (a > 1 && (v % a)) a >>= 1;
  return a;
}

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

// pointer lists of ls2_gemm_list travel by value in the kernel's parameters (so
// a captured graph replays them without any host memory)
constexpr int kMaxList = 64;
struct PtrList {
  const void* p[3 * kMaxList];
};

__global__ void fill_list_kernel(PtrList l, int n, const void** out) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) out[i] = l.p[i];
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
  if (cublasLtCreate(&b->lt) != CUBLAS_STATUS_SUCCESS) b->lt = nullptr;
  // fp32 compute, no TF32, no reduced-precision split-K reductions
  cublasSetMathMode(b->h, (cublasMath_t)(CUBLAS_DEFAULT_MATH |
                                         CUBLAS_MATH_DISALLOW_REDUCED_PRECISION_REDUCTION));
  return b;
}

void ls2_blas_destroy(void* p) {
  Blas* b = reinterpret_cast<Blas*>(p);
  if (!b) return;
  for (auto& kv : b->plans) {
    LtPlan& p = kv.second;
    if (p.op) cublasLtMatmulDescDestroy(p.op);
    if (p.a) cublasLtMatrixLayoutDestroy(p.a);
    if (p.b) cublasLtMatrixLayoutDestroy(p.b);
    if (p.c) cublasLtMatrixLayoutDestroy(p.c);
  }
  if (b->lt) cublasLtDestroy(b->lt);
  if (b->h) cublasDestroy(b->h);
  if (b->ws) cudaFree(b->ws);
  delete b;
}

}  // extern "C"

namespace ls2 {

// Time the heuristic's candidates on the real operands once per key (outside
// graph capture) and keep the fastest.  With beta != 0 the candidates write a
// scratch D so C is left untouched.  Off unless LS2_GEMM_TUNE=1 (the
// heuristic's first choice is taken otherwise).  Reduction schemes are restricted to fp32
// workspace reductions (no fp16 split-K partial sums, no in-place atomics).
// off by default: candidates timed in isolation (hot L2, one kernel at a time)
// picked algorithms that were slower inside the real step (3.67 vs 3.60 ms at
// T-base on the same box).  LS2_GEMM_TUNE=1 tunes every GEMM, =w only the
// weight-gradient ones (fp32 output).
static int tuning_mode() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("LS2_GEMM_TUNE");
    on = !e ? 0 : e[0] == '1' ? 1 : e[0] == 'w' ? 2 : e[0] == 'd' ? 3 : 0;
  }
  return on;
}
static bool tuning_enabled(int tc = -1) {
  const int m = tuning_mode();
  return m == 1 || (m == 2 && tc == LS2_F32) || (m == 3 && tc != LS2_F32);
}

// Candidates are timed as a CUDA graph of kTuneReps back-to-back launches on a
// private stream, so the number is device time (the step replays graphs too),
// not the few microseconds of host overhead per cublasLtMatmul call.
constexpr int kTuneReps = 8;

// LS2_GEMM_PICK="<tag substring>=<heuristic index>;..." pins the algorithm of the
// plans whose tag contains the substring (in-step A/B experiments, see
// tools/gemm_pick_sweep.sh); LS2_GEMM_LIST=1 prints every plan's candidates.
static std::vector<std::pair<std::string, int>> gemm_picks() {
  std::vector<std::pair<std::string, int>> out;
  const char* e = getenv("LS2_GEMM_PICK");
  if (!e) return out;
  std::string s(e);
  size_t pos = 0;
  while (pos < s.size()) {
    size_t end = s.find(';', pos);
    if (end == std::string::npos) end = s.size();
    const std::string item = s.substr(pos, end - pos);
    const size_t eq = item.rfind('=');
    if (eq != std::string::npos) out.emplace_back(item.substr(0, eq), std::atoi(item.c_str() + eq + 1));
    pos = end + 1;
  }
  return out;
}

static void lt_describe(const cublasLtMatmulAlgo_t& a, int& tile, int& stages, int& splitk) {
  size_t w = 0;
  tile = stages = splitk = 0;
  cublasLtMatmulAlgoConfigGetAttribute(&a, CUBLASLT_ALGO_CONFIG_TILE_ID, &tile, sizeof(tile), &w);
  cublasLtMatmulAlgoConfigGetAttribute(&a, CUBLASLT_ALGO_CONFIG_STAGES_ID, &stages, sizeof(stages), &w);
  cublasLtMatmulAlgoConfigGetAttribute(&a, CUBLASLT_ALGO_CONFIG_SPLITK_NUM, &splitk, sizeof(splitk), &w);
}

static void lt_tune(Blas* bl, LtPlan* plan, const cublasLtMatmulHeuristicResult_t* res, int found,
                    const void* A, const void* B, double beta, void* C, int64_t m, int64_t ldc,
                    int tc, cudaStream_t st) {
  plan->algo = res[0].algo;
  static const bool list = getenv("LS2_GEMM_LIST") != nullptr;
  if (list) {
    for (int i = 0; i < found; ++i) {
      int tile, stages, splitk;
      lt_describe(res[i].algo, tile, stages, splitk);
      fprintf(stderr, "[ls2 gemm list] %s #%d tile=%d stages=%d splitk=%d ws=%zu\n", plan->tag, i,
              tile, stages, splitk, res[i].workspaceSize);
    }
  }
  static const std::vector<std::pair<std::string, int>> picks = gemm_picks();
  for (const auto& pk : picks) {
    if (strstr(plan->tag, pk.first.c_str()) && pk.second >= 0 && pk.second < found &&
        res[pk.second].workspaceSize <= bl->ws_bytes) {
      plan->algo = res[pk.second].algo;
      return;
    }
  }
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(st, &cap);
  if (found <= 1 || !tuning_enabled(tc) || cap != cudaStreamCaptureStatusNone) return;
  cudaStreamSynchronize(st);
  cudaStream_t ts;
  if (cudaStreamCreateWithFlags(&ts, cudaStreamNonBlocking) != cudaSuccess) { cudaGetLastError(); return; }
  void* D = C;
  void* tmp = nullptr;
  if (beta != 0.0) {
    const size_t bytes = (size_t)m * (size_t)ldc * esize(tc);
    if (cudaMalloc(&tmp, bytes) != cudaSuccess) { cudaGetLastError(); cudaStreamDestroy(ts); return; }
    D = tmp;
  }
  const float af = 1.f, bf = (float)beta;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f, first_ms = -1.f;
  for (int i = 0; i < found; ++i) {
    if (res[i].workspaceSize > bl->ws_bytes) continue;
    auto run = [&]() {
      return cublasLtMatmul(bl->lt, plan->op, &af, B, plan->a, A, plan->b, &bf, C, plan->c, D,
                            plan->c, &res[i].algo, bl->ws, bl->ws_bytes, ts);
    };
    if (run() != CUBLAS_STATUS_SUCCESS || cudaStreamSynchronize(ts) != cudaSuccess) {
      cudaGetLastError();
      continue;
    }
    cudaGraph_t g = nullptr;
    cudaGraphExec_t ge = nullptr;
    bool ok = cudaStreamBeginCapture(ts, cudaStreamCaptureModeThreadLocal) == cudaSuccess;
    for (int r = 0; ok && r < kTuneReps; ++r) ok = run() == CUBLAS_STATUS_SUCCESS;
    if (cudaStreamEndCapture(ts, &g) != cudaSuccess) ok = false;
    if (ok && cudaGraphInstantiate(&ge, g, 0) != cudaSuccess) ok = false;
    if (ok) {
      cudaGraphLaunch(ge, ts);  // warm
      // median of 5 timed replays: one noisy sample must not pick the algorithm
      float t[5];
      for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(e0, ts);
        cudaGraphLaunch(ge, ts);
        cudaEventRecord(e1, ts);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&t[rep], e0, e1);
      }
      std::sort(t, t + 5);
      const float ms = t[2] / kTuneReps;
      if (i == 0) first_ms = ms;
      // leave the heuristic's first choice only for a clear (> 2%) gain
      if (i == 0 ? ms < best : ms < best * 0.98f) {
        best = ms;
        plan->algo = res[i].algo;
      }
    }
    if (ge) cudaGraphExecDestroy(ge);
    if (g) cudaGraphDestroy(g);
    cudaGetLastError();
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  static const bool log = getenv("LS2_GEMM_LOG") != nullptr;
  if (log) {
    int tile = 0, splitk = 0;
    size_t w = 0;
    cublasLtMatmulAlgoConfigGetAttribute(&plan->algo, CUBLASLT_ALGO_CONFIG_TILE_ID, &tile, sizeof(tile), &w);
    cublasLtMatmulAlgoConfigGetAttribute(&plan->algo, CUBLASLT_ALGO_CONFIG_SPLITK_NUM, &splitk, sizeof(splitk), &w);
    fprintf(stderr, "[ls2 gemm] %s beta=%g candidates=%d best=%.2f us (heuristic #0 %.2f us) tile=%d splitk=%d\n",
            plan->tag, beta, found, best * 1e3f, first_ms * 1e3f, tile, splitk);
  }
  cudaStreamSynchronize(ts);
  if (tmp) cudaFree(tmp);
  cudaStreamDestroy(ts);
  cudaGetLastError();
}

/* C = alpha*op(A)@op(B) + beta*C (+ bias[n] broadcast over rows) on cuBLASLt, row-major.
 * Returns LS2_ERR_CUBLAS when no Lt algorithm supports the combination (caller falls back). */
// which operand-major combinations go to the hand-written tcgen05 GEMM
// (LS2_TC_GEMM: 'f' forward X W^T, 'd' data gradient dY W, 'w' weight gradient
// dY^T X, 'a' all of them, '0' none)
static bool tc_route(int trans_a, int trans_b) {
  static int mask = [] {
    const char* e = std::getenv("LS2_TC_GEMM");
    const std::string s = e ? e : "";
    int m = 0;
    if (s.find('f') != std::string::npos) m |= 1;
    if (s.find('d') != std::string::npos) m |= 2;
    if (s.find('w') != std::string::npos) m |= 4;
    if (s.find('a') != std::string::npos) m |= 7;
    return m;
  }();
  if (!trans_a && trans_b) return mask & 1;
  if (!trans_a && !trans_b) return mask & 2;
  if (trans_a && !trans_b) return mask & 4;
  return false;
}

// bmode: 0 none, 1 bias add (bias[n]), 2 bias gradient of op(A) (sum over K -> [m]),
// 3 bias gradient of op(B) (sum over K -> [n]); the gradient vector has type tc
static int lt_matmul(Blas* bl, int trans_a, int trans_b, int64_t m, int64_t n, int64_t k,
                     double alpha, const void* A, int64_t lda, const void* B, int64_t ldb,
                     double beta, void* C, int64_t ldc, const void* bias, int tab, int tc,
                     cudaStream_t st, int bmode = -1) {
  if (bmode < 0) bmode = bias ? 1 : 0;
  if (m <= 0 || n <= 0) return LS2_OK;
  // LS2_TC_MIN_MACS: route only products of at least this many MACs;
  // LS2_TC_2SM=1: use the persistent two-SM kernel for the routed ones
  static const double tc_min_macs = [] {
    const char* e = std::getenv("LS2_TC_MIN_MACS");
    return e ? std::atof(e) : 0.0;
  }();
  static const bool tc_2sm = [] {
    const char* e = std::getenv("LS2_TC_2SM");
    return e && e[0] == '1';
  }();
  if (bmode <= 1 && tc_route(trans_a, trans_b) && (double)m * n * k >= tc_min_macs &&
      ls2_gemm_tc_supported(trans_a, trans_b, m, n, k, A, lda, B, ldb, beta, C, ldc, tab, tc) &&
      (!bias || aligned16(bias)) && (!tc_2sm || n % 128 == 0))
    return ls2_gemm_tc(trans_a, trans_b, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc, bias, tab,
                       tc, tc_2sm ? -3 : 0, st);
  if (!bl || !bl->lt) return fail(LS2_ERR_CUBLAS, "gemm_lt: no cublasLt handle");
  if (tab == LS2_F64 || tc == LS2_F64) return fail(LS2_ERR_CUBLAS, "gemm_lt: f64 not routed to Lt");
  const int al = std::min(std::min(align_of(A), align_of(B)), std::min(align_of(C),
                          bias ? align_of(bias) : 256));
  LtKey key{trans_a, trans_b, m, n, k, lda, ldb, ldc, tab, tc, bmode, beta != 0.0, al};
  LtPlan* plan;
  {
    std::lock_guard<std::mutex> g(bl->mu);
    plan = &bl->plans[key];
    if (!plan->op) {
      const cublasOperation_t opA = trans_b ? CUBLAS_OP_T : CUBLAS_OP_N;  // Lt A := row-major B
      const cublasOperation_t opB = trans_a ? CUBLAS_OP_T : CUBLAS_OP_N;  // Lt B := row-major A
      cublasLtMatmulDescCreate(&plan->op, CUBLAS_COMPUTE_32F, CUDA_R_32F);
      cublasLtMatmulDescSetAttribute(plan->op, CUBLASLT_MATMUL_DESC_TRANSA, &opA, sizeof(opA));
      cublasLtMatmulDescSetAttribute(plan->op, CUBLASLT_MATMUL_DESC_TRANSB, &opB, sizeof(opB));
      if (bias) {
        // row-major A/B are Lt's B/A (the product is computed transposed)
        cublasLtEpilogue_t ep = bmode == 2 ? CUBLASLT_EPILOGUE_BGRADB
                              : bmode == 3 ? CUBLASLT_EPILOGUE_BGRADA : CUBLASLT_EPILOGUE_BIAS;
        cublasLtMatmulDescSetAttribute(plan->op, CUBLASLT_MATMUL_DESC_EPILOGUE, &ep, sizeof(ep));
        cudaDataType_t bt = cuda_type(tc);
        cublasLtMatmulDescSetAttribute(plan->op, CUBLASLT_MATMUL_DESC_BIAS_DATA_TYPE, &bt, sizeof(bt));
        cublasLtMatmulDescSetAttribute(plan->op, CUBLASLT_MATMUL_DESC_BIAS_POINTER, &bias, sizeof(bias));
      }
      snprintf(plan->tag, sizeof(plan->tag), "ta=%d tb=%d m=%lld n=%lld k=%lld tab=%d tc=%d bias=%d",
               trans_a, trans_b, (long long)m, (long long)n, (long long)k, tab, tc, bmode);
      const cudaDataType_t tAB = cuda_type(tab), tC = cuda_type(tc);
      cublasLtMatrixLayoutCreate(&plan->a, tAB, trans_b ? k : n, trans_b ? n : k, ldb);
      cublasLtMatrixLayoutCreate(&plan->b, tAB, trans_a ? m : k, trans_a ? k : m, lda);
      cublasLtMatrixLayoutCreate(&plan->c, tC, n, m, ldc);
      cublasLtMatmulPreference_t pref;
      cublasLtMatmulPreferenceCreate(&pref);
      size_t wsb = bl->ws_bytes;
      cublasLtMatmulPreferenceSetAttribute(pref, CUBLASLT_MATMUL_PREF_MAX_WORKSPACE_BYTES, &wsb, sizeof(wsb));
      uint32_t a32 = (uint32_t)al;
      cublasLtMatmulPreferenceSetAttribute(pref, CUBLASLT_MATMUL_PREF_MIN_ALIGNMENT_A_BYTES, &a32, sizeof(a32));
      cublasLtMatmulPreferenceSetAttribute(pref, CUBLASLT_MATMUL_PREF_MIN_ALIGNMENT_B_BYTES, &a32, sizeof(a32));
      cublasLtMatmulPreferenceSetAttribute(pref, CUBLASLT_MATMUL_PREF_MIN_ALIGNMENT_C_BYTES, &a32, sizeof(a32));
      cublasLtMatmulPreferenceSetAttribute(pref, CUBLASLT_MATMUL_PREF_MIN_ALIGNMENT_D_BYTES, &a32, sizeof(a32));
      uint32_t red = CUBLASLT_REDUCTION_SCHEME_NONE | CUBLASLT_REDUCTION_SCHEME_COMPUTE_TYPE;
      cublasLtMatmulPreferenceSetAttribute(pref, CUBLASLT_MATMUL_PREF_REDUCTION_SCHEME_MASK, &red, sizeof(red));
      cublasLtMatmulHeuristicResult_t res[32];
      int found = 0;
      cublasStatus_t s = cublasLtMatmulAlgoGetHeuristic(bl->lt, plan->op, plan->a, plan->b, plan->c,
                                                        plan->c, pref, 32, res, &found);
      cublasLtMatmulPreferenceDestroy(pref);
      plan->ok = (s == CUBLAS_STATUS_SUCCESS && found > 0);
      if (plan->ok) lt_tune(bl, plan, res, found, A, B, beta, C, m, ldc, tc, st);
    }
  }
  if (!plan->ok) return fail(LS2_ERR_CUBLAS, "gemm_lt: no algorithm for this combination");
  if (bias)
    cublasLtMatmulDescSetAttribute(plan->op, CUBLASLT_MATMUL_DESC_BIAS_POINTER, &bias, sizeof(bias));
  const float af = (float)alpha, bf = (float)beta;
  cublasStatus_t s = cublasLtMatmul(bl->lt, plan->op, &af, B, plan->a, A, plan->b, &bf, C, plan->c,
                                    C, plan->c, &plan->algo, bl->ws, bl->ws_bytes, st);
  return s == CUBLAS_STATUS_SUCCESS ? LS2_OK : blas_fail(s, "cublasLtMatmul");
}

}  // namespace ls2

extern "C" {

int ls2_gemm_lt(void* hp, int trans_a, int trans_b, int64_t m, int64_t n, int64_t k, double alpha,
                const void* A, int64_t lda, const void* B, int64_t ldb, double beta, void* C,
                int64_t ldc, const void* bias, int tab, int tc, void* stream) {
  return lt_matmul(reinterpret_cast<Blas*>(hp), trans_a, trans_b, m, n, k, alpha, A, lda, B, ldb,
                   beta, C, ldc, bias, tab, tc, as_stream(stream));
}

int ls2_gemm_lt_bgrad(void* hp, int trans_a, int trans_b, int64_t m, int64_t n, int64_t k,
                      double alpha, const void* A, int64_t lda, const void* B, int64_t ldb,
                      double beta, void* C, int64_t ldc, void* bgrad, int which, int tab, int tc,
                      void* stream) {
  if (!bgrad) return fail(LS2_ERR_SHAPE, "gemm_lt_bgrad: null gradient vector");
  return lt_matmul(reinterpret_cast<Blas*>(hp), trans_a, trans_b, m, n, k, alpha, A, lda, B, ldb,
                   beta, C, ldc, bgrad, tab, tc, as_stream(stream), which ? 3 : 2);
}

int64_t ls2_gemm_scratch_bytes(int64_t n1, int64_t n2) { return 3 * n1 * n2 * (int64_t)sizeof(void*); }

int ls2_gemm(void* hp, int trans_a, int trans_b, int64_t m, int64_t n, int64_t k, double alpha,
             const void* A, int64_t lda, int64_t sA1, int64_t sA2, const void* B, int64_t ldb,
             int64_t sB1, int64_t sB2, double beta, void* C, int64_t ldc, int64_t sC1,
             int64_t sC2, int64_t n1, int64_t n2, int tab, int tc, void* ptr_scratch,
             int ptrs_ready, void* stream) {
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
  if (total == 1 && !f64 && b->lt) {
    // single GEMMs go through the tuned cuBLASLt plans; GemmEx only if Lt has no algorithm
    if (lt_matmul(b, trans_a, trans_b, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc, nullptr,
                  tab, tc, as_stream(stream)) == LS2_OK)
      return LS2_OK;
  }
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
  if (!ptrs_ready) {  // callers cache the arrays per (addresses, strides): filled once
    fill_ptrs_kernel<<<grid_for(total), 256, 0, as_stream(stream)>>>(
        (const char*)A, (const char*)B, (char*)C, n2, total, sA1 * ea, sA2 * ea, sB1 * ea,
        sB2 * ea, sC1 * ec, sC2 * ec, ptrs);
    int rc = check_launch("gemm_fill_ptrs");
    if (rc) return rc;
  }
  s = cublasGemmBatchedEx(b->h, opB, opA, (int)n, (int)m, (int)k, pa, (const void* const*)(ptrs + total),
                          tAB, (int)ldb, (const void* const*)ptrs, tAB, (int)lda, pb,
                          (void* const*)(ptrs + 2 * total), tC, (int)ldc, (int)total, ct,
                          CUBLAS_GEMM_DEFAULT);
  return s == CUBLAS_STATUS_SUCCESS ? LS2_OK : blas_fail(s, "cublasGemmBatchedEx");
}

int ls2_gemm_list(void* hp, int trans_a, int trans_b, int64_t m, int64_t n, int64_t k,
                  double alpha, const void* const* a_list, int64_t lda, const void* const* b_list,
                  int64_t ldb, double beta, void* const* c_list, int64_t ldc, int count, int tab,
                  int tc, void* ptr_scratch, int ptrs_ready, void* stream) {
  Blas* b = reinterpret_cast<Blas*>(hp);
  if (!b) return fail(LS2_ERR_CUBLAS, "gemm_list: null blas handle");
  if (count <= 0 || m <= 0 || n <= 0) return LS2_OK;
  if (count > kMaxList) return fail(LS2_ERR_SHAPE, "gemm_list: at most 64 products per call");
  if (!a_list || !b_list || !c_list) return fail(LS2_ERR_SHAPE, "gemm_list: null pointer list");
  if (tab == LS2_F64 || tc == LS2_F64) return fail(LS2_ERR_DTYPE, "gemm_list: f64 not batched");
  if (!(tc == tab || tc == LS2_F32)) return fail(LS2_ERR_DTYPE, "gemm_list: bad output dtype");
  if (count == 1)
    return lt_matmul(b, trans_a, trans_b, m, n, k, alpha, a_list[0], lda, b_list[0], ldb, beta,
                     c_list[0], ldc, nullptr, tab, tc, as_stream(stream));
  if (!ptr_scratch) return fail(LS2_ERR_SHAPE, "gemm_list: needs pointer scratch");
  const void** ptrs = reinterpret_cast<const void**>(ptr_scratch);
  if (!ptrs_ready) {   // callers cache the table per address list: filled once
    PtrList l;
    for (int i = 0; i < count; ++i) {
      l.p[i] = a_list[i];
      l.p[count + i] = b_list[i];
      l.p[2 * count + i] = c_list[i];
    }
    fill_list_kernel<<<1, 256, 0, as_stream(stream)>>>(l, 3 * count, ptrs);
    int rc = check_launch("gemm_fill_list");
    if (rc) return rc;
  }
  cublasSetStream(b->h, as_stream(stream));
  const float af = (float)alpha, bf = (float)beta;
  const cublasOperation_t opA = trans_a ? CUBLAS_OP_T : CUBLAS_OP_N;
  const cublasOperation_t opB = trans_b ? CUBLAS_OP_T : CUBLAS_OP_N;
  const cudaDataType_t tAB = cuda_type(tab), tC = cuda_type(tc);
  cublasStatus_t s = cublasGemmBatchedEx(
      b->h, opB, opA, (int)n, (int)m, (int)k, &af, (const void* const*)(ptrs + count), tAB,
      (int)ldb, (const void* const*)ptrs, tAB, (int)lda, &bf, (void* const*)(ptrs + 2 * count),
      tC, (int)ldc, count, CUBLAS_COMPUTE_32F, CUBLAS_GEMM_DEFAULT);
  return s == CUBLAS_STATUS_SUCCESS ? LS2_OK : blas_fail(s, "cublasGemmBatchedEx(list)");
}

}  // extern "C"
