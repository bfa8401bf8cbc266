// Host-side cost of the runtime calls a forward makes per layer (B200 box):
// cuTensorMapEncodeTiled, <<<>>> vs cudaLaunchKernelEx(+PDL), event record +
// stream wait, cudaFuncSetAttribute. Measured: 0.04 / 3.9 / 2.2 / 0.23 / 0.06 us.
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/host_costs tools/host_costs.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <chrono>
#include <cstdio>
__global__ void k_empty(int* p) { if (p && threadIdx.x == 1234567) *p = 1; }
int main() {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    auto enc = (CUresult(*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                            const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                            CUtensorMapL2promotion, CUtensorMapFloatOOBfill))fn;
    void* buf; cudaMalloc(&buf, 64 << 20);
    CUtensorMap m;
    cuuint64_t dims[2] = {96, 125000}; cuuint64_t strides[1] = {192}; cuuint32_t box[2] = {32, 128}; cuuint32_t es[2] = {1, 1};
    for (int i = 0; i < 100; ++i) enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    auto t0 = std::chrono::steady_clock::now();
    const int N = 20000;
    for (int i = 0; i < N; ++i) enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    auto t1 = std::chrono::steady_clock::now();
    printf("cuTensorMapEncodeTiled: %.3f us/call\n", std::chrono::duration<double, std::micro>(t1 - t0).count() / N);
    cudaStream_t st; cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    for (int i = 0; i < 100; ++i) k_empty<<<148, 256, 0, st>>>(nullptr);
    cudaStreamSynchronize(st);
    t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < 2000; ++i) k_empty<<<148, 256, 0, st>>>(nullptr);
    t1 = std::chrono::steady_clock::now();
    printf("<<<>>> launch: %.3f us/call\n", std::chrono::duration<double, std::micro>(t1 - t0).count() / 2000);
    cudaStreamSynchronize(st);
    cudaLaunchConfig_t cfg = {}; cfg.gridDim = 148; cfg.blockDim = 256; cfg.stream = st;
    cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization; at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < 2000; ++i) cudaLaunchKernelEx(&cfg, k_empty, (int*)nullptr);
    t1 = std::chrono::steady_clock::now();
    printf("cudaLaunchKernelEx+PDL: %.3f us/call\n", std::chrono::duration<double, std::micro>(t1 - t0).count() / 2000);
    cudaStreamSynchronize(st);
    cudaEvent_t e; cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < 2000; ++i) { cudaEventRecord(e, st); cudaStreamWaitEvent(st, e, 0); }
    t1 = std::chrono::steady_clock::now();
    printf("eventRecord+streamWaitEvent: %.3f us/pair\n", std::chrono::duration<double, std::micro>(t1 - t0).count() / 2000);
    void* p;
    t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < 2000; ++i) cudaFuncSetAttribute((const void*)k_empty, cudaFuncAttributeMaxDynamicSharedMemorySize, 1024);
    t1 = std::chrono::steady_clock::now();
    printf("cudaFuncSetAttribute: %.3f us/call\n", std::chrono::duration<double, std::micro>(t1 - t0).count() / 2000);
    return 0;
}
