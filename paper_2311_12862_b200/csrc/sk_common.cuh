// sk200 internal: error plumbing, device buffers, coordinate packing/hash,
// and the raw PTX wrappers (mbarrier, cp.async, tcgen05, TMEM) used by the
// sm_100a kernels. Written directly against the PTX ISA; no CUTLASS/CuTe.
#pragma once

#include <cuda_fp16.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <initializer_list>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

#include "sk200.h"

namespace sk {

// ---- errors (mirror sparsekit ValidationError / ContractError) -------------
struct Error : std::runtime_error {
    sk_status code;
    Error(sk_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] inline void fail(sk_status c, const std::string& m) { throw Error(c, m); }
inline void validate(bool ok, const std::string& m) {
    if (!ok) fail(SK_ERR_VALIDATION, m);
}
inline void contract(bool ok, const std::string& m) {
    if (!ok) fail(SK_ERR_CONTRACT, m);
}
#define SK_CUDA(x)                                                                          \
    do {                                                                                    \
        cudaError_t e_ = (x);                                                               \
        if (e_ != cudaSuccess)                                                              \
            ::sk::fail(SK_ERR_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_) +      \
                                        " (" __FILE__ ":" + std::to_string(__LINE__) + ")"); \
    } while (0)
// every library kernel launch is followed by SK_LAUNCH_CHECK(), which also
// counts it (sk_kernel_launches: the bench's gpu_launches evidence)
std::atomic<unsigned long long>& launch_counter();
// programmatic dependent launch for this host thread's launches (launch_pdl);
// a runner sets it from sk_net_set_pdl around its calls (capi.cu)
bool& pdl_enabled();
struct PdlScope {
    bool prev;
    explicit PdlScope(bool on) : prev(pdl_enabled()) { pdl_enabled() = on; }
    ~PdlScope() { pdl_enabled() = prev; }
};
#define SK_LAUNCH_CHECK()                      \
    do {                                       \
        ::sk::launch_counter().fetch_add(1);   \
        SK_CUDA(cudaGetLastError());           \
    } while (0)

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
// small fills as a library kernel launched with launch_pdl when PDL is on: a
// memset node is a full drain point on both sides (no programmatic overlap
// with the kernels around it) in a map pipeline of short kernels (capi.cu)
void fill_async(void* p, int byte, size_t bytes, cudaStream_t st);

#if defined(__CUDACC__)
// Launch with programmatic stream serialization (see pdl_wait): the kernel's
// launch latency and pre-wait prologue overlap the predecessor's tail.
template <typename... KArgs, typename... Args>
void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    SK_CUDA(cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...));
    launch_counter().fetch_add(1);
}
#endif

// ---- device buffer (stream-ordered allocator + host-side block cache) -------
// Freed blocks stay in a host-side cache per (stream, size class) and go back
// to the next allocation of that class on the same stream (stream order makes
// the reuse safe). A run of similar scans then makes no cudaMallocAsync /
// cudaFreeAsync calls: each costs 1-2 us of host time, and the ~200 per
// MinkUNet scan fell right after a sync, with the GPU idle (capi.cu).
void* cache_alloc(size_t n, cudaStream_t s);
void cache_free(void* p, size_t n, cudaStream_t s);
void cache_trim();
// Cross-stream readiness of a lazily built, cached object (map, prepared map,
// transposed map, pair lists, down-sampled set, block index): `on` is the
// stream it was built on. A caller on another stream waits for everything
// enqueued on `on` so far (an event recorded now: it may over-wait, never
// under-wait). Same stream: nothing to do, so the single-stream hot path pays
// nothing (capi.cu).
struct BuiltOn {
    cudaStream_t s = nullptr;
    bool set = false;  // unset: built synchronously / not lazily, nothing to wait for
    void mark(cudaStream_t st) {
        s = st;
        set = true;
    }
};
void stream_after(const BuiltOn& on, cudaStream_t st);
// Small device->host reads (counts, error flags) through host-mapped pinned
// memory written by a one-thread kernel, then a stream sync: no copy engine,
// so they never queue behind a large D2H on another stream (capi.cu).
// Segments are concatenated into dst (<= 4 segments, <= 64 bytes in all).
struct RbSeg {
    const void* src;
    size_t bytes;
};
void read_back(cudaStream_t st, std::initializer_list<RbSeg> segs, void* dst);

// Raise a kernel's dynamic shared memory limit to >= smem, once per (kernel,
// high-water mark). Serialised and keyed by the kernel's address: runners on
// several host threads launch the same kernels concurrently (capi.cu).
void ensure_smem(const void* kern, size_t smem);

struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    cudaStream_t stream = nullptr;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept { *this = std::move(o); }
    DevBuf& operator=(DevBuf&& o) noexcept {
        if (this != &o) {
            reset();
            p = o.p; bytes = o.bytes; stream = o.stream;
            o.p = nullptr; o.bytes = 0;
        }
        return *this;
    }
    ~DevBuf() { reset(); }
    void alloc(size_t n, cudaStream_t s) {
        reset();
        stream = s;
        bytes = n;
        if (n) p = cache_alloc(n, s);
    }
    void reset() {
        if (p) cache_free(p, bytes, stream);
        p = nullptr;
        bytes = 0;
    }
    template <class T> T* as() const { return static_cast<T*>(p); }
};

// ---- coordinate packing ------------------------------------------------------
// 63-bit key: batch 12 bits | x,y,z 17 bits each (biased by 2^16). The top
// bit is always 0, so kEmpty (all ones) never collides with a real key.
constexpr uint64_t kEmpty = ~0ull;
constexpr int32_t kBias = 1 << 16;
constexpr int32_t kBatchMax = 1 << 12;

__host__ __device__ inline bool packable(int32_t b, int32_t x, int32_t y, int32_t z) {
    return b >= 0 && b < kBatchMax && x >= -kBias && x < kBias && y >= -kBias && y < kBias &&
           z >= -kBias && z < kBias;
}
__host__ __device__ inline uint64_t pack_key(int32_t b, int32_t x, int32_t y, int32_t z) {
    return (uint64_t(uint32_t(b)) << 51) | (uint64_t(uint32_t(x + kBias)) << 34) |
           (uint64_t(uint32_t(y + kBias)) << 17) | uint64_t(uint32_t(z + kBias));
}
// Fibonacci (multiplicative) hashing: the TOP log2(cap) bits of k * 2^64/phi
// -- one 64-bit multiply per probe; every key bit reaches the slot bits.
// mask = cap - 1 (cap a power of two).
__host__ __device__ inline uint64_t hash_slot(uint64_t k, uint64_t mask) {
#if defined(__CUDA_ARCH__)
    const int bits = __popcll(mask);
#else
    const int bits = __builtin_popcountll(mask);
#endif
    return (k * 0x9E3779B97F4A7C15ull) >> (64 - bits);
}
__host__ __device__ inline int64_t floor_div(int64_t a, int64_t b) {
    int64_t q = a / b;
    if ((a % b != 0) && ((a < 0) != (b < 0))) --q;
    return q;
}

// ---- PTX wrappers (sm_100a) ----------------------------------------------------
#if defined(__CUDACC__)
constexpr uint32_t kSuspendHintNs = 1000000;  // 1 ms: effectively 'until the phase completes'
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}
// try_wait with a suspend-time hint: the waiting warp stays suspended until
// the phase completes (or the hint expires) instead of re-polling, so waiting
// warps do not compete for issue slots and MIO bandwidth
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    uint32_t addr = smem_u32(bar);
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(addr),
        "r"(parity), "r"(kSuspendHintNs)
        : "memory");
}
// Waits of warps that are not on the tensor-core critical path: probe, then
// back off with nanosleep between probes, so a dozen waiting warps do not
// flood the MIO pipe (shared by every LDS/STS/LDGSTS of the SM) with polls.
template <int NS = 64>
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
    uint32_t addr = smem_u32(bar);
    uint32_t done = 0;
    for (;;) {
        asm volatile(
            "{\n.reg .pred P1;\n"
            "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n"
            "selp.b32 %0, 1, 0, P1;\n}\n"
            : "=r"(done)
            : "r"(addr), "r"(parity)
            : "memory");
        if (done) return;
        __nanosleep(NS);
    }
}
// 16-byte cp.async, zero-filled when src_bytes == 0 (sentinel rows, channel tails)
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, uint32_t src_bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src),
                 "r"(src_bytes)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
    asm volatile("cp.async.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// TMEM allocation (one warp), power-of-two columns >= 32
__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem, uint32_t ncols) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(dst_smem)),
                 "r"(ncols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols)
                 : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
// D[tmem] (+)= A[smem] * B[smem]^T, kind::f16 (fp16/bf16 in, fp32 accumulate)
__device__ __forceinline__ void tc_mma_f16(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                           uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
        "}\n" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}
// arrive on an mbarrier when all prior tcgen05 ops of this thread complete
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::
                     "r"(smem_u32(bar))
                 : "memory");
}
// 32 lanes x 32 consecutive fp32 columns -> 32 registers per thread
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
          "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
          "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
          "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
          "=r"(r[31])
        : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld_wait() {
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ bool elect_one() {
    uint32_t pred = 0;
    asm volatile(
        "{\n"
        ".reg .pred P;\n"
        "elect.sync _|P, 0xffffffff;\n"
        "selp.b32 %0, 1, 0, P;\n"
        "}\n"
        : "=r"(pred));
    return pred != 0;
}
// Programmatic dependent launch (launch_pdl): a kernel launched with the
// attribute may start while its stream predecessor is still running; it must
// pass pdl_wait() (griddepcontrol.wait: the predecessor grid has completed and
// its memory is visible) before touching any global memory the predecessor
// reads or writes. pdl_trigger() lets the NEXT kernel begin launching.
// Both are no-ops for kernels launched without the attribute.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void red_add_v4(float* addr, float a, float b, float c, float d) {
    asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(addr), "f"(a), "f"(b),
                 "f"(c), "f"(d)
                 : "memory");
}
// warp-aggregated shared-memory histogram increment: the whole warp calls it
// (d < 0: no-op lane); one atomic per distinct digit in the warp, so skewed
// digit distributions do not serialise on one bank
__device__ __forceinline__ void hist_add(uint32_t* h, int d) {
    const unsigned peers = __match_any_sync(0xffffffffu, d);
    if (d >= 0 && (int)(threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(&h[d], (uint32_t)__popc(peers));
}
#endif

}  // namespace sk
