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
// Process-wide pool of cuBLAS handles, created once and never destroyed: a
// handle serves one host thread at a time, and creating one per (short-lived)
// worker thread cost a cudaMalloc of its workspace, which stalls the device.
struct HandlePool {
    std::mutex mu;
    std::vector<cublasHandle_t> free;
};
HandlePool& pool() {
    static HandlePool* p = new HandlePool();
    return *p;
}
cublasHandle_t acquire() {
    {
        std::lock_guard<std::mutex> g(pool().mu);
        if (!pool().free.empty()) {
            cublasHandle_t h = pool().free.back();
            pool().free.pop_back();
            return h;
        }
    }
    cublasHandle_t h = nullptr;
    if (cublasCreate(&h) != CUBLAS_STATUS_SUCCESS) return nullptr;
    return h;
}
void release(cublasHandle_t h) {
    std::lock_guard<std::mutex> g(pool().mu);
    pool().free.push_back(h);
}
}  // namespace

// Column-major view: a row-major [r][c] matrix is a col-major c x r matrix.
// forward: y^T (co x n) = W_cm (co x ci) * x^T (ci x n)
// dgrad:   dx^T (ci x n) = (W_cm)^T (ci x co) * dy^T (co x n)
bool dense_identity_gemm(sk_dtype dt, long long rows, int c_in, int c_out, const void* x,
                         const void* w, void* y, float* y_accum, bool dgrad, cudaStream_t st) {
    if (dt != SK_F16 && dt != SK_BF16) return false;
    if (rows <= 0 || rows > INT32_MAX) return false;
    cublasHandle_t h = acquire();
    if (!h) return false;
    struct Back {
        cublasHandle_t h;
        ~Back() { release(h); }
    } back{h};
    if (cublasSetStream(h, st) != CUBLAS_STATUS_SUCCESS) return false;
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
