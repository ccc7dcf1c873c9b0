// Peer-memory plumbing for the fused multi-GPU halo (slabs.IpcHalo).
//
// Every rank exports, through CUDA IPC, its field store and a small inbox of
// step counters.  Neighbours map them (over NVLink on an NVSwitch node; on
// the same device when several test ranks share one GPU).  Per step:
//   tlbm_peer_wait   -- one thread spins (acquire, system scope) until every
//                       inbox counter reached the step; bounded by a timeout
//                       so a lost neighbour raises instead of hanging the GPU
//   tlbm_step        -- boundary layers with halo_* set: the fused kernel
//                       stores its outgoing z planes straight into the
//                       neighbour's ghost tiles (peer stores, no pack / copy)
//   tlbm_peer_signal -- system-scope fence, then the step counter is stored
//                       into each neighbour's inbox
#include <cuda.h>

#include <cstring>

#include "common.cuh"

namespace tlbm {
namespace {

__device__ __forceinline__ unsigned long long load_acquire_sys(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void store_release_sys(unsigned long long *p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ unsigned long long global_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__global__ void wait_kernel(const unsigned long long *inbox, int n, unsigned long long value,
                            unsigned long long timeout_ns, unsigned int *error) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    const unsigned long long t0 = global_ns();
    for (int i = 0; i < n; ++i) {
        while (load_acquire_sys(inbox + i) < value) {
            if (global_ns() - t0 > timeout_ns) {
                atomicOr(error, 1u);
                return;
            }
            __nanosleep(200);
        }
    }
}

__global__ void signal_kernel(unsigned long long *a, unsigned long long *b,
                              unsigned long long value) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    __threadfence_system();
    if (a) store_release_sys(a, value);
    if (b) store_release_sys(b, value);
}

}  // namespace
}  // namespace tlbm

using namespace tlbm;

static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle is 64 bytes");

extern "C" int tlbm_ipc_export(void *d_ptr, void *h_handle, uint64_t *h_offset) {
    cudaIpcMemHandle_t handle;
    int rc = cuda_check(cudaIpcGetMemHandle(&handle, d_ptr), "cudaIpcGetMemHandle");
    if (rc) return rc;
    // the handle names the whole allocation; report d_ptr's offset inside it
    void *fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    rc = cuda_check(cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q),
                    "cudaGetDriverEntryPoint(cuMemGetAddressRange)");
    if (rc) return rc;
    if (!fn || q != cudaDriverEntryPointSuccess) {
        set_error("cuMemGetAddressRange unavailable");
        return TLBM_ERR_CUDA;
    }
    using range_fn = CUresult (*)(CUdeviceptr *, size_t *, CUdeviceptr);
    CUdeviceptr base = 0;
    size_t size = 0;
    if (reinterpret_cast<range_fn>(fn)(&base, &size, (CUdeviceptr)d_ptr) != CUDA_SUCCESS) {
        set_error("cuMemGetAddressRange failed");
        return TLBM_ERR_CUDA;
    }
    memcpy(h_handle, &handle, sizeof(handle));
    *h_offset = (uint64_t)((CUdeviceptr)d_ptr - base);
    return TLBM_OK;
}

extern "C" int tlbm_ipc_import(const void *h_handle, uint64_t offset, void **d_ptr) {
    cudaIpcMemHandle_t handle;
    memcpy(&handle, h_handle, sizeof(handle));
    void *base = nullptr;
    int rc = cuda_check(cudaIpcOpenMemHandle(&base, handle, cudaIpcMemLazyEnablePeerAccess),
                        "cudaIpcOpenMemHandle");
    if (rc) return rc;
    *d_ptr = static_cast<char *>(base) + offset;
    return TLBM_OK;
}

extern "C" int tlbm_ipc_close(void *d_base) {
    return cuda_check(cudaIpcCloseMemHandle(d_base), "cudaIpcCloseMemHandle");
}

extern "C" int tlbm_peer_wait(const uint64_t *d_inbox, int n, uint64_t value,
                              uint64_t timeout_ns, uint32_t *d_error, void *stream) {
    if (n <= 0) return TLBM_OK;
    wait_kernel<<<1, 32, 0, as_stream(stream)>>>(
        reinterpret_cast<const unsigned long long *>(d_inbox), n, value, timeout_ns, d_error);
    return launch_check("wait_kernel");
}

extern "C" int tlbm_peer_signal(uint64_t *d_peer_a, uint64_t *d_peer_b, uint64_t value,
                                void *stream) {
    if (!d_peer_a && !d_peer_b) return TLBM_OK;
    signal_kernel<<<1, 32, 0, as_stream(stream)>>>(reinterpret_cast<unsigned long long *>(d_peer_a),
                                                   reinterpret_cast<unsigned long long *>(d_peer_b),
                                                   value);
    return launch_check("signal_kernel");
}
