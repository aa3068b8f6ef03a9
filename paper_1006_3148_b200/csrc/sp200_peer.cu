// Peer-memory plumbing for the fused z-slab halo delivery:
// CUDA IPC handles for the grids of neighbouring ranks (one process per GPU,
// NVLink / NVSwitch peer mappings) and stream-ordered pass counters between
// ranks.  Replaces the reference's halo transport (sp/transport.py:58-60,
// 194-237; sp/halo.py:239-271) for z-slabs: the fused pass stores the planes
// a neighbour needs straight into its grid (sp_temporal_mirror), then bumps
// the neighbour's counter; the neighbour's stream waits on its own counter
// before the pass that reads those planes.  No kernel spins on another
// rank's progress unless stream memory operations are unavailable.
#include <string.h>

#include "sp200_device.cuh"
#include "sp200_internal.h"

namespace sp200 {

// fallbacks when cuStreamWriteValue32 / cuStreamWaitValue32 are unavailable
__global__ void k_signal(uint32_t *flag, uint32_t value) {
    __threadfence_system();
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(flag), "r"(value) : "memory");
}

__global__ void k_wait(const uint32_t *flag, uint32_t value) {
    uint32_t x;
    do {
        asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(x) : "l"(flag) : "memory");
    } while ((int32_t)(x - value) < 0);
}

typedef CUresult (*StreamValueFn)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
typedef CUresult (*AddrRangeFn)(CUdeviceptr *, size_t *, CUdeviceptr);

static void *driver_fn(const char *name) {
    void *ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint(name, &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
        return ptr;
    return nullptr;
}

}  // namespace sp200

using namespace sp200;

extern "C" {

int sp_ipc_handle(const void *ptr, void *handle, int64_t *offset) {
    if (!ptr || !handle || !offset) return set_error(SP_EINVAL, "null argument");
    static AddrRangeFn range = reinterpret_cast<AddrRangeFn>(driver_fn("cuMemGetAddressRange"));
    if (!range) return set_error(SP_ECUDA, "cuMemGetAddressRange unavailable");
    CUdeviceptr base = 0;
    size_t size = 0;
    if (range(&base, &size, reinterpret_cast<CUdeviceptr>(ptr)) != CUDA_SUCCESS)
        return set_error(SP_EINVAL, "sp_ipc_handle: not a device allocation");
    cudaIpcMemHandle_t h;
    cudaError_t e = cudaIpcGetMemHandle(&h, reinterpret_cast<void *>(base));
    if (e != cudaSuccess) return set_error(SP_ECUDA, "cudaIpcGetMemHandle: %s", cudaGetErrorString(e));
    memcpy(handle, &h, sizeof(h));
    *offset = (int64_t)(reinterpret_cast<CUdeviceptr>(ptr) - base);
    return SP_OK;
}

int sp_ipc_open(const void *handle, void **ptr) {
    if (!handle || !ptr) return set_error(SP_EINVAL, "null argument");
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, sizeof(h));
    cudaError_t e = cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) return set_error(SP_ECUDA, "cudaIpcOpenMemHandle: %s", cudaGetErrorString(e));
    return SP_OK;
}

int sp_ipc_close(void *ptr) {
    cudaError_t e = cudaIpcCloseMemHandle(ptr);
    if (e != cudaSuccess) return set_error(SP_ECUDA, "cudaIpcCloseMemHandle: %s", cudaGetErrorString(e));
    return SP_OK;
}

int sp_signal(uint32_t *flag, uint32_t value, void *stream) {
    if (!flag) return set_error(SP_EINVAL, "null flag");
    static StreamValueFn wr = reinterpret_cast<StreamValueFn>(driver_fn("cuStreamWriteValue32"));
    // default flags: a memory fence orders the stream's earlier writes
    // (including peer stores of the pass) before the counter
    if (wr && !tuning().signal_kernels &&
        wr(reinterpret_cast<CUstream>(stream), reinterpret_cast<CUdeviceptr>(flag), value, 0) ==
            CUDA_SUCCESS)
        return SP_OK;
    k_signal<<<1, 1, 0, as_stream(stream)>>>(flag, value);
    count_launch();
    return check_launch("k_signal");
}

int sp_wait(const uint32_t *flag, uint32_t value, void *stream) {
    if (!flag) return set_error(SP_EINVAL, "null flag");
    static StreamValueFn wt = reinterpret_cast<StreamValueFn>(driver_fn("cuStreamWaitValue32"));
    if (wt && !tuning().signal_kernels &&
        wt(reinterpret_cast<CUstream>(stream), reinterpret_cast<CUdeviceptr>(flag), value,
           CU_STREAM_WAIT_VALUE_GEQ) == CUDA_SUCCESS)
        return SP_OK;
    k_wait<<<1, 1, 0, as_stream(stream)>>>(flag, value);
    count_launch();
    return check_launch("k_wait");
}

}  // extern "C"
