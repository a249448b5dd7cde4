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

// ---- cross-rank ordering without host synchronisation ----------------------
//
// A cross-shard gate reads the partners' current buffers and writes this
// rank's other buffer, which partners read during the previous cross-shard
// gate.  Each rank records an interprocess event on its stream before the
// gate (everything it enqueued so far: its writes of the current buffer, its
// reads of partner buffers in the previous gate); after a host barrier that
// only orders the *enqueueing* (no device drain), every rank makes its
// stream wait on the partners' events.  Kernels never spin on each other:
// the ordering is the driver's stream-wait on a completed record.

extern "C" int diaq_ipc_event_create(void **ev) {
    if (!ev) return set_error(DIAQ_ERR_VALUE, "diaq_ipc_event_create: null argument");
    cudaEvent_t e;
    const cudaError_t r = cudaEventCreateWithFlags(&e, cudaEventInterprocess | cudaEventDisableTiming);
    if (r != cudaSuccess) {
        cudaGetLastError();
        *ev = nullptr;
        return set_error(DIAQ_ERR_CUDA, "cudaEventCreateWithFlags(interprocess): %s", cudaGetErrorString(r));
    }
    *ev = (void *)e;
    return DIAQ_OK;
}

extern "C" int diaq_ipc_event_handle(void *ev, void *handle_out) {
    if (!ev || !handle_out) return set_error(DIAQ_ERR_VALUE, "diaq_ipc_event_handle: null argument");
    cudaIpcEventHandle_t h;
    const cudaError_t r = cudaIpcGetEventHandle(&h, (cudaEvent_t)ev);
    if (r != cudaSuccess) {
        cudaGetLastError();
        return set_error(DIAQ_ERR_CUDA, "cudaIpcGetEventHandle: %s", cudaGetErrorString(r));
    }
    memcpy(handle_out, &h, sizeof(h));
    return DIAQ_OK;
}

extern "C" int diaq_ipc_event_open(const void *handle, void **ev_out) {
    if (!handle || !ev_out) return set_error(DIAQ_ERR_VALUE, "diaq_ipc_event_open: null argument");
    cudaIpcEventHandle_t h;
    memcpy(&h, handle, sizeof(h));
    cudaEvent_t e;
    const cudaError_t r = cudaIpcOpenEventHandle(&e, h);
    if (r != cudaSuccess) {
        cudaGetLastError();
        *ev_out = nullptr;
        return set_error(DIAQ_ERR_CUDA, "cudaIpcOpenEventHandle: %s", cudaGetErrorString(r));
    }
    *ev_out = (void *)e;
    return DIAQ_OK;
}

extern "C" int diaq_event_record(void *ev, void *stream) {
    if (!ev) return set_error(DIAQ_ERR_VALUE, "diaq_event_record: null event");
    const cudaError_t r = cudaEventRecord((cudaEvent_t)ev, (cudaStream_t)stream);
    if (r != cudaSuccess) {
        cudaGetLastError();
        return set_error(DIAQ_ERR_CUDA, "cudaEventRecord: %s", cudaGetErrorString(r));
    }
    return DIAQ_OK;
}

extern "C" int diaq_stream_wait_event(void *stream, void *ev) {
    if (!ev) return set_error(DIAQ_ERR_VALUE, "diaq_stream_wait_event: null event");
    const cudaError_t r = cudaStreamWaitEvent((cudaStream_t)stream, (cudaEvent_t)ev, 0);
    if (r != cudaSuccess) {
        cudaGetLastError();
        return set_error(DIAQ_ERR_CUDA, "cudaStreamWaitEvent: %s", cudaGetErrorString(r));
    }
    return DIAQ_OK;
}

extern "C" int diaq_event_destroy(void *ev) {
    if (!ev) return DIAQ_OK;
    const cudaError_t r = cudaEventDestroy((cudaEvent_t)ev);
    if (r != cudaSuccess) {
        cudaGetLastError();
        return set_error(DIAQ_ERR_CUDA, "cudaEventDestroy: %s", cudaGetErrorString(r));
    }
    return DIAQ_OK;
}
