// abi.cu -- library-level C-ABI entry points: errors, layout, counters.
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <string>

#include <mutex>
#include <unordered_set>
#include <vector>

#include "common.cuh"

namespace diaq {

static thread_local std::string g_last_error;
static Tuning g_tuning;
Tuning &tuning() { return g_tuning; }
static std::atomic<uint64_t> g_launches{0};

int set_error(int code, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_last_error = buf;
    return code;
}

void count_launch(int n) { g_launches.fetch_add((uint64_t)n, std::memory_order_relaxed); }

int sm_count() {
    static int cached[64] = {0};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) {
        cudaGetLastError();
        return kSms;
    }
    if (!cached[dev]) {
        int sms = kSms;
        if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) {
            cudaGetLastError();
            sms = kSms;
        }
        cached[dev] = sms;
    }
    return cached[dev];
}

int occupancy(const void *kernel, int threads, size_t smem) {
    struct Key {
        int dev;
        const void *f;
        int threads;
        size_t smem;
        int per_sm;
    };
    static std::mutex mu;
    static std::vector<Key> memo;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) cudaGetLastError();
    {
        std::lock_guard<std::mutex> lk(mu);
        for (const Key &k : memo)
            if (k.dev == dev && k.f == kernel && k.threads == threads && k.smem == smem) return k.per_sm;
    }
    int per_sm = 1;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem) != cudaSuccess || per_sm < 1) {
        cudaGetLastError();
        per_sm = 1;
    }
    std::lock_guard<std::mutex> lk(mu);
    memo.push_back({dev, kernel, threads, smem, per_sm});
    return per_sm;
}

int check_launch(const char *what) {
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return set_error(DIAQ_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
    return DIAQ_OK;
}

}  // namespace diaq

using namespace diaq;

extern "C" int diaq_version(void) { return 1; }

extern "C" int diaq_tune(const char *key, int64_t value) {
    if (!key) return set_error(DIAQ_ERR_VALUE, "diaq_tune: null key");
    const std::string k(key);
    Tuning &t = g_tuning;
    if (k == "spmv_raster") t.spmv_raster = (int)value;
    else if (k == "spmv_chunk") t.spmv_chunk = (int)(value < 1 ? 1 : value);
    else if (k == "spmv_xpol") t.spmv_xpol = (int)value;
    else if (k == "spmv_ctas_per_sm") t.spmv_ctas_per_sm = (int)value;
    else if (k == "spmv_banded") t.spmv_banded = (int)value;
    else if (k == "spmv_strips") t.spmv_strips = (int)value;
    else if (k == "spmv_tma") t.spmv_tma = (int)value;
    else if (k == "spmv_tma_stages") t.spmv_tma_stages = (int)value;
    else if (k == "spmv_async") t.spmv_async = (int)value;
    else if (k == "gate_ctas_per_sm") t.gate_ctas_per_sm = (int)(value < 1 ? 1 : value);
    else if (k == "fused_dense2") t.fused_dense2 = (int)value;
    else if (k == "fused_gperm_rows") t.fused_gperm_rows = (int)value;
    else if (k == "fused_gperm") t.fused_gperm = (int)value;
    else if (k == "fused_seq") t.fused_seq = (int)value;
    else if (k == "fused_nbuf") t.fused_nbuf = (int)value;
    else if (k == "fused_jit") t.fused_jit = (int)value;
    else if (k == "fused_tbits") t.fused_tbits = (int)(value <= 7 ? 7 : 8);
    else if (k == "fused_gstore") t.fused_gstore = (int)value;
    else if (k == "fused_dstore") t.fused_dstore = (int)value;
    else if (k == "fused_ppipe") t.fused_ppipe = (int)(value < 0 ? 0 : value > 3 ? 3 : value);
    else if (k == "fused_plain_pair") t.fused_plain_pair = (int)value;
    else if (k == "fused_pair_store") t.fused_pair_store = (int)value;
    else if (k == "fused_bank_spread") t.fused_bank_spread = (int)value;
    else if (k == "fused_perm") t.fused_perm = (int)value;
    else if (k == "fused_estore") t.fused_estore = (int)value;
    else if (k == "fused_reorder") t.fused_reorder = (int)value;
    else if (k == "fused_dyn") t.fused_dyn = (int)value;
    else if (k == "fused_lookahead") t.fused_lookahead = (int)value;
    else if (k == "fused_unit") t.fused_unit = (int)value;
    else if (k == "fused_slots") t.fused_slots = (int)value;
    else if (k == "fused_slot_gates") t.fused_slot_gates = (int)(value < 1 ? 1 : value);
    else if (k == "fused_maxph") t.fused_maxph = (int)(value < 1 ? 1 : value);
    else if (k == "kron_flat") t.kron_flat = (int)value;
    else if (k == "kron_ctas_per_sm") t.kron_ctas_per_sm = (int)(value < 1 ? 1 : value);
    else return set_error(DIAQ_ERR_VALUE, "diaq_tune: unknown key %s", key);
    ++t.epoch;
    return DIAQ_OK;
}

extern "C" const char *diaq_last_error(void) { return g_last_error.c_str(); }

extern "C" int diaq_device_count(int *count) {
    int c = 0;
    const cudaError_t e = cudaGetDeviceCount(&c);
    if (count) *count = (e == cudaSuccess) ? c : 0;
    if (e != cudaSuccess) {
        cudaGetLastError();
        return set_error(DIAQ_ERR_CUDA, "cudaGetDeviceCount: %s", cudaGetErrorString(e));
    }
    return DIAQ_OK;
}

extern "C" uint64_t diaq_launch_count(void) { return g_launches.load(); }

extern "C" void diaq_reset_launch_count(void) { g_launches.store(0); }

// Row-aligned layout: diagonal i starts at an element index s_i with
// (s_i + min(d_i, 0)) % 8 == 0, so the element of row r is 128-byte aligned
// whenever r % 8 == 0 (arena base is >= 512-byte aligned).
extern "C" int diaq_layout(int64_t n, int64_t nd, const int64_t *offs, int64_t *starts, int64_t *total) {
    if (n < 1) return set_error(DIAQ_ERR_SHAPE, "n_dim must be >= 1, got %lld", (long long)n);
    if (nd < 0 || (nd > 0 && (!offs || !starts)) || !total) return set_error(DIAQ_ERR_VALUE, "diaq_layout: bad arguments");
    int64_t cur = 0;
    for (int64_t i = 0; i < nd; ++i) {
        const int64_t d = offs[i];
        const int64_t a = d < 0 ? -d : d;
        if (a > n - 1)
            return set_error(DIAQ_ERR_VALUE, "diagonal %lld out of range for n_dim=%lld", (long long)d, (long long)n);
        if (i > 0 && offs[i - 1] >= d) return set_error(DIAQ_ERR_VALUE, "offsets must be strictly ascending");
        const int64_t want = (d < 0 ? -d : 0) & 7;  // s % 8 == (-min(d,0)) % 8
        int64_t s = cur + ((want - (cur & 7)) & 7);
        starts[i] = s;
        cur = s + (n - a);
    }
    *total = (cur + 7) & ~7ll;
    return DIAQ_OK;
}

// ---- per-gate timing events (reference run() per_gate timings, sim.py:193-199) ----
extern "C" int diaq_timer_create(int n, void **events) {
    if (n < 0 || (n > 0 && !events)) return set_error(DIAQ_ERR_VALUE, "diaq_timer_create: bad arguments");
    for (int i = 0; i < n; ++i) {
        cudaEvent_t e;
        if (cudaEventCreate(&e) != cudaSuccess) {
            for (int j = 0; j < i; ++j) cudaEventDestroy((cudaEvent_t)events[j]);
            return set_error(DIAQ_ERR_CUDA, "cudaEventCreate: %s", cudaGetErrorString(cudaGetLastError()));
        }
        events[i] = (void *)e;
    }
    return DIAQ_OK;
}

// waits for events[n-1]; ms_out[i] = time between events[i] and events[i+1]
// events recorded since the last diaq_timer_elapsed that read them
static std::mutex g_marked_mu;
static std::unordered_set<void *> g_marked;

namespace diaq {
cudaError_t timer_record(void *event, cudaStream_t s) {
    const cudaError_t e = cudaEventRecord((cudaEvent_t)event, s);
    if (e == cudaSuccess) {
        std::lock_guard<std::mutex> lk(g_marked_mu);
        g_marked.insert(event);
    }
    return e;
}
}  // namespace diaq

extern "C" int diaq_timer_elapsed(int n, void **events, float *ms_out) {
    if (n < 1 || !events || !ms_out) return set_error(DIAQ_ERR_VALUE, "diaq_timer_elapsed: bad arguments");
    if (cudaEventSynchronize((cudaEvent_t)events[n - 1]) != cudaSuccess)
        return set_error(DIAQ_ERR_CUDA, "cudaEventSynchronize: %s", cudaGetErrorString(cudaGetLastError()));
    // events a fused pass did not record (all its gates but the last) read as
    // zero-length intervals; the others are measured from the last recorded
    // one.  Only events marked by this run are read (an unrecorded event costs
    // a failing driver call, and one left from an earlier run would be stale).
    std::lock_guard<std::mutex> lk(g_marked_mu);
    void *last = events[0];
    g_marked.erase(events[0]);
    for (int i = 0; i + 1 < n; ++i) {
        float ms = 0.0f;
        auto it = g_marked.find(events[i + 1]);
        if (it != g_marked.end() &&
            cudaEventElapsedTime(&ms, (cudaEvent_t)last, (cudaEvent_t)events[i + 1]) == cudaSuccess) {
            ms_out[i] = ms;
            last = events[i + 1];
        } else {
            cudaGetLastError();
            ms_out[i] = 0.0f;
        }
        if (it != g_marked.end()) g_marked.erase(it);
    }
    return DIAQ_OK;
}

extern "C" int diaq_timer_destroy(int n, void **events) {
    {
        std::lock_guard<std::mutex> lk(g_marked_mu);
        for (int i = 0; i < n; ++i) g_marked.erase(events[i]);
    }
    for (int i = 0; i < n; ++i)
        if (events[i]) cudaEventDestroy((cudaEvent_t)events[i]);
    return DIAQ_OK;
}

extern "C" int diaq_timer_record(void *event, void *stream) {
    if (timer_record(event, (cudaStream_t)stream) != cudaSuccess)
        return set_error(DIAQ_ERR_CUDA, "cudaEventRecord: %s", cudaGetErrorString(cudaGetLastError()));
    return DIAQ_OK;
}
