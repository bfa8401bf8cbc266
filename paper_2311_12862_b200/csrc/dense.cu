// K=1 stride-1 layers on one coordinate set: the kernel map is the identity,
// so the "sparse conv" is a plain dense GEMM y[n][co] = x[n][ci] W[ci][co]
// (dgrad: dx = dy W^T). Plain GEMMs go to cuBLAS (measured 2x faster than the
// gathered-GEMM kernel's dense mode on these memory-bound shapes,
// tools/k1_bench.py); the epilogues cuBLAS cannot fuse (a residual add into a
// T output) stay on k_gconv_tc.
#include <cublas_v2.h>

#include "sk_internal.hpp"

namespace sk {

namespace {
// One cuBLAS handle per CUDA stream, created on first use, bound to that
// stream once and never destroyed. Re-binding a handle to another stream
// resets its workspace (cuBLAS then re-allocates it: a device-wide stall each
// time the runners' streams alternate), and a handle is not safe for
// concurrent host threads, hence the per-handle mutex around the (short) call.
struct StreamHandle {
    std::mutex mu;
    cublasHandle_t h = nullptr;
};
StreamHandle* handle_for(cudaStream_t st) {
    static std::mutex mu;
    static std::map<cudaStream_t, StreamHandle*>* table = new std::map<cudaStream_t, StreamHandle*>();
    std::lock_guard<std::mutex> g(mu);
    StreamHandle*& e = (*table)[st];
    if (!e) {
        auto* n = new StreamHandle();
        if (cublasCreate(&n->h) != CUBLAS_STATUS_SUCCESS ||
            cublasSetStream(n->h, st) != CUBLAS_STATUS_SUCCESS) {
            delete n;
            return nullptr;
        }
        e = n;
    }
    return e;
}
}  // namespace

// Column-major view: a row-major [r][c] matrix is a col-major c x r matrix.
// forward: y^T (co x n) = W_cm (co x ci) * x^T (ci x n)
// dgrad:   dx^T (ci x n) = (W_cm)^T (ci x co) * dy^T (co x n)
bool dense_identity_gemm(sk_dtype dt, long long rows, int c_in, int c_out, const void* x,
                         const void* w, void* y, float* y_accum, bool dgrad, cudaStream_t st) {
    if (dt != SK_F16 && dt != SK_BF16) return false;
    if (rows <= 0 || rows > INT32_MAX) return false;
    StreamHandle* sh = handle_for(st);
    if (!sh) return false;
    std::lock_guard<std::mutex> g(sh->mu);
    cublasHandle_t h = sh->h;
    const cudaDataType_t ab = dt == SK_F16 ? CUDA_R_16F : CUDA_R_16BF;
    const int m = dgrad ? c_in : c_out;   // rows of the col-major result
    const int k = dgrad ? c_out : c_in;
    const float one = 1.f, zero = 0.f;
    const cublasStatus_t s = cublasGemmEx(
        h, dgrad ? CUBLAS_OP_T : CUBLAS_OP_N, CUBLAS_OP_N, m, (int)rows, k, &one, w, ab, c_out,
        x, ab, k, y_accum ? &one : &zero, y_accum ? (void*)y_accum : y,
        y_accum ? CUDA_R_32F : ab, m, CUBLAS_COMPUTE_32F, CUBLAS_GEMM_DEFAULT);
    return s == CUBLAS_STATUS_SUCCESS;
}

}  // namespace sk
