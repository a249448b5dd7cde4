// peer.cu -- device memory shared between the ranks of a sharded state
// (SURVEY.md 8(e)): CUDA IPC mappings of the partner shards, so the
// multi-source gate kernel (apply.cu) reads partner amplitudes directly over
// NVLink / NVSwitch inside the gate pass -- the exchange overlaps the math
// instead of a staging copy (NCCL send/recv) followed by a local pass.
//
// Buffers come from cudaMalloc here (IPC handles name whole allocations, so
// an exported buffer must be an allocation base, which the caching
// allocators of frameworks do not guarantee).
#include <cstring>

#include "common.cuh"

using namespace diaq;

extern "C" int diaq_alloc(int64_t bytes, void **ptr) {
    if (!ptr || bytes <= 0) return set_error(DIAQ_ERR_VALUE, "diaq_alloc: bad arguments");
    *ptr = nullptr;
    const cudaError_t e = cudaMalloc(ptr, (size_t)bytes);
    if (e != cudaSuccess) {
        cudaGetLastError();
        *ptr = nullptr;
        return set_error(DIAQ_ERR_RESOURCE, "diaq_alloc: %lld bytes: %s", (long long)bytes, cudaGetErrorString(e));
    }
    return DIAQ_OK;
}

extern "C" int diaq_free(void *ptr) {
    if (!ptr) return DIAQ_OK;
    const cudaError_t e = cudaFree(ptr);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return set_error(DIAQ_ERR_CUDA, "diaq_free: %s", cudaGetErrorString(e));
    }
    return DIAQ_OK;
}

extern "C" int diaq_ipc_handle(const void *ptr, void *handle_out) {
    if (!ptr || !handle_out) return set_error(DIAQ_ERR_VALUE, "diaq_ipc_handle: null argument");
    cudaIpcMemHandle_t h;
    const cudaError_t e = cudaIpcGetMemHandle(&h, const_cast<void *>(ptr));
    if (e != cudaSuccess) {
        cudaGetLastError();
        return set_error(DIAQ_ERR_CUDA, "cudaIpcGetMemHandle: %s", cudaGetErrorString(e));
    }
    memcpy(handle_out, &h, sizeof(h));
    return DIAQ_OK;
}

extern "C" int diaq_ipc_open(const void *handle, void **ptr_out) {
    if (!handle || !ptr_out) return set_error(DIAQ_ERR_VALUE, "diaq_ipc_open: null argument");
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, sizeof(h));
    *ptr_out = nullptr;
    const cudaError_t e = cudaIpcOpenMemHandle(ptr_out, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) {
        cudaGetLastError();
        *ptr_out = nullptr;
        return set_error(DIAQ_ERR_CUDA, "cudaIpcOpenMemHandle: %s", cudaGetErrorString(e));
    }
    return DIAQ_OK;
}

extern "C" int diaq_ipc_close(void *ptr) {
    if (!ptr) return DIAQ_OK;
    const cudaError_t e = cudaIpcCloseMemHandle(ptr);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return set_error(DIAQ_ERR_CUDA, "cudaIpcCloseMemHandle: %s", cudaGetErrorString(e));
    }
    return DIAQ_OK;
}
