// sample.cu -- the reference's inverse-CDF sampler on the device.
//
// Reference: sim.py:142-161.  p = |a|^2, q = round(p, 12), cdf = np.cumsum(q)
// (a SEQUENTIAL float64 sum), hits = min(searchsorted(cdf, u, 'right'), N-1)
// for the splitmix64 uniforms u.  Counts must match the reference exactly, so
// every step reproduces numpy's float64 operations bit for bit:
//
//  * |a| as numpy computes it for complex128 on this build: with m = max(|re|,
//    |im|), r = min/m, |a| = m * sqrt(fma(r, r, 1)) (checked against numpy on
//    4e5 samples); p = |a|*|a|; q = rint(p * 1e12) / 1e12 (numpy's round).
//  * the cumsum c_i = fl(c_{i-1} + q_i) is sequential, but it is exactly
//    computable in parallel per binade: while c stays in [2^e, 2^(e+1)) its
//    values are integer multiples of U = 2^(e-52), and fl(c + q) = c +
//    RNE(q / U) * U as long as no tie occurs and the result stays in the
//    binade.  So within a segment c_i = U * (K0 + inclusive_scan(k)) with
//    k_i = RNE(q_i / U) -- an exact int64 scan.  A segment ends at the first
//    element that leaves the binade or hits an exact tie; that one step is
//    done in float64 on the host (same IEEE rounding) and a new segment
//    starts.  c grows from >= 1e-12 to ~1, so there are at most ~45 segments.
//  * searchsorted is a per-shot binary search over the materialised cdf.
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <vector>

#include "common.cuh"

namespace diaq {

__device__ __forceinline__ double np_cabs(double2 a) {
    double x = fabs(a.x), y = fabs(a.y);
    if (x < y) {
        const double t = x;
        x = y;
        y = t;
    }
    if (x == 0.0) return 0.0;
    const double r = __ddiv_rn(y, x);
    return __dmul_rn(x, __dsqrt_rn(__fma_rn(r, r, 1.0)));
}

__global__ void __launch_bounds__(kThreads) sample_q_kernel(const double2 *x, int64_t n, double *q, double *psum_part,
                                                            unsigned long long *first_nz) {
    double s = 0.0;
    unsigned long long first = ~0ull;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        const double a = np_cabs(x[i]);
        const double p = __dmul_rn(a, a);
        const double qi = __ddiv_rn(rint(__dmul_rn(p, 1e12)), 1e12);
        q[i] = qi;
        s += p;
        if (qi > 0.0 && (unsigned long long)i < first) first = (unsigned long long)i;
    }
    __shared__ double red[kThreads / 32];
    __shared__ unsigned long long redf[kThreads / 32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        s += __shfl_down_sync(0xffffffffu, s, o);
        const unsigned long long f = __shfl_down_sync(0xffffffffu, first, o);
        first = f < first ? f : first;
    }
    if ((threadIdx.x & 31) == 0) {
        red[threadIdx.x >> 5] = s;
        redf[threadIdx.x >> 5] = first;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        unsigned long long f = ~0ull;
        for (int w = 0; w < kThreads / 32; ++w) {
            t += red[w];
            f = redf[w] < f ? redf[w] : f;
        }
        psum_part[blockIdx.x] = t;
        if (f != ~0ull) atomicMin(first_nz, f);
    }
}

// k_i = RNE(q_i * 2^(52-e)) and the exit condition of the segment
__global__ void __launch_bounds__(kThreads) sample_k_kernel(const double *q, int64_t i0, int64_t cnt, double scale,
                                                            long long *k, unsigned char *tie) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < cnt; j += stride) {
        const double v = __dmul_rn(q[i0 + j], scale);  // exact: scaling by a power of two
        const double f = floor(v);
        const double fr = v - f;                        // exact
        tie[j] = fr == 0.5;
        // clamp: anything >= 2^53 ends the segment at this element, and the
        // clamp keeps the prefix up to the first exit exact (no int64 overflow)
        const double r = rint(v);                       // round half to even
        k[j] = r >= 9007199254740992.0 ? (1ll << 53) : (long long)r;
    }
}

__global__ void __launch_bounds__(kThreads) sample_exit_kernel(const long long *S, const unsigned char *tie, int64_t cnt,
                                                               long long kbase, unsigned long long *exit_at) {
    const long long lim = 1ll << 53;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < cnt; j += stride)
        if (tie[j] || kbase + S[j] >= lim) atomicMin(exit_at, (unsigned long long)j);
}

__global__ void __launch_bounds__(kThreads) sample_c_kernel(const long long *S, int64_t i0, int64_t cnt, long long kbase,
                                                            double U, double *c) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < cnt; j += stride)
        c[i0 + j] = __dmul_rn((double)(kbase + S[j]), U);  // exact: integer < 2^53 times a power of two
}

__global__ void sample_search_kernel(const double *c, int64_t n, const double *u, int64_t shots, long long *hits) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= shots) return;
    const double uk = u[k];
    int64_t lo = 0, hi = n;  // first index with c > u
    while (lo < hi) {
        const int64_t mid = lo + (hi - lo) / 2;
        if (c[mid] <= uk) lo = mid + 1;
        else hi = mid;
    }
    hits[k] = lo < n - 1 ? lo : n - 1;
}

// Small states (n <= 2^24): the whole binade walk in ONE CTA, no host round
// trip.  The CTA scans chunks of kWalkE * kWalkThreads elements: k_i =
// RNE(q_i / U) in the current binade, an exclusive block scan of the
// per-thread sums, the first element that leaves the binade or ties, c
// written up to it, the exiting element as one float64 add, then the next
// binade -- the same arithmetic as the host-driven path below.  Each thread
// owns kWalkE consecutive elements of a chunk; chunks move through shared
// memory (coalesced cp.async loads, double-buffered so the next chunk lands
// while this one is scanned; c staged back the same way for coalesced
// stores), and a chunk that stays in its binade costs one block scan and one
// __syncthreads_or -- the exit bookkeeping runs only at the ~45 binade ends.
constexpr int kWalkThreads = 512;
constexpr int kWalkE = 12;
constexpr int kWalkChunk = kWalkE * kWalkThreads;
constexpr size_t kWalkSmem = 2 * sizeof(double) * kWalkChunk;

__device__ __forceinline__ long long walk_k(double v) {
    const double r = rint(v);  // round half to even
    return r >= 9007199254740992.0 ? (1ll << 53) : (long long)r;
}

// chunk [p, p + kWalkChunk) of q into buf (zeros past n), one commit group
__device__ __forceinline__ void walk_fetch(double *buf, const double *q, int64_t p, int64_t n) {
    for (int k = threadIdx.x; k < kWalkChunk; k += kWalkThreads) {
        if (p + k < n) {
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(buf + k)), "l"(q + p + k)
                         : "memory");
        } else {
            buf[k] = 0.0;
        }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
}

__global__ void __launch_bounds__(kWalkThreads, 1) sample_walk_kernel(const double *__restrict__ q, int64_t n,
                                                                      const unsigned long long *first_nz,
                                                                      double *__restrict__ c) {
    using BlockScan = cub::BlockScan<long long, kWalkThreads, cub::BLOCK_SCAN_WARP_SCANS>;
    __shared__ typename BlockScan::TempStorage scan_tmp;
    __shared__ long long s_exit;
    __shared__ double s_cur;
    extern __shared__ double wbuf[];  // two chunk buffers
    const int tid = threadIdx.x;
    const unsigned long long f = *first_nz;
    const int64_t first = f == ~0ull ? n : (int64_t)f;
    for (int64_t j = tid; j < first && j < n; j += blockDim.x) c[j] = 0.0;
    if (first >= n) return;
    const long long lim = 1ll << 53;
    double cur = q[first];
    if (tid == 0) c[first] = cur;
    int64_t pos = first + 1;
    int cb = 0;  // buffer of the current chunk
    walk_fetch(wbuf, q, pos, n);
    while (pos < n) {
        // binade of cur (a normal double: q >= 1e-12 when nonzero): cur in [2^eb, 2^(eb+1))
        const int eb = (int)((__double_as_longlong(cur) >> 52) & 0x7ff) - 1023;
        const double U = __longlong_as_double((long long)(eb - 52 + 1023) << 52);
        const double scale = __longlong_as_double((long long)(52 - eb + 1023) << 52);
        long long kbase = (long long)__dmul_rn(cur, scale);  // exact integer in [2^52, 2^53)
        while (pos < n) {
            double *buf = wbuf + cb * kWalkChunk;
            double *nbuf = wbuf + (cb ^ 1) * kWalkChunk;
            __syncthreads();  // nbuf (the previous chunk) fully drained to c
            walk_fetch(nbuf, q, pos + kWalkChunk, n);  // the next chunk flies under this one
            asm volatile("cp.async.wait_group 1;" ::: "memory");
            __syncthreads();
            double *mine = buf + tid * kWalkE;
            const int64_t b = pos + (int64_t)tid * kWalkE;
            long long kv[kWalkE], tsum = 0;
            unsigned ties = 0;
#pragma unroll
            for (int j = 0; j < kWalkE; ++j) {  // q = 0 past n
                const double v = __dmul_rn(mine[j], scale);  // exact: scaling by a power of two
                kv[j] = walk_k(v);
                ties |= (unsigned)((v - floor(v)) == 0.5) << j;
                tsum += kv[j];
            }
            long long excl, total;
            BlockScan(scan_tmp).ExclusiveSum(tsum, excl, total);
            long long run = kbase + excl;
            int my = -1;
            const int64_t rem = n - b;
            const int lim_j = rem < kWalkE ? (int)rem : kWalkE;  // valid elements of this thread
#pragma unroll
            for (int j = 0; j < kWalkE; ++j) {
                run += kv[j];
                if (my < 0 && j < lim_j && (((ties >> j) & 1u) || run >= lim)) my = j;
            }
            const bool exits = __syncthreads_or(my >= 0);
            int64_t xat = pos + kWalkChunk;  // first element not written from the integer scan
            if (exits) {
                if (tid == 0) s_exit = LLONG_MAX;
                __syncthreads();
                if (my >= 0) atomicMin(&s_exit, (long long)(b + my));
                __syncthreads();
                xat = s_exit;
            }
            run = kbase + excl;
#pragma unroll
            for (int j = 0; j < kWalkE; ++j) {  // own slots only: no hazard with other threads' reads
                run += kv[j];
                mine[j] = __dmul_rn((double)run, U);
            }
            __syncthreads();
            int64_t wend = xat < n ? xat : n;
            if (wend > pos + kWalkChunk) wend = pos + kWalkChunk;
            for (int k = tid; pos + k < wend; k += kWalkThreads) c[pos + k] = buf[k];
            if (!exits) {
                kbase += total;
                pos += kWalkChunk;
                cb ^= 1;
                continue;
            }
            __syncthreads();  // c before the exit is written
            if (tid == 0) {   // the exiting element: one float64 add (IEEE, round to nearest even)
                const double sum = __dadd_rn(c[xat - 1], q[xat]);
                c[xat] = sum;
                s_cur = sum;
            }
            asm volatile("cp.async.wait_group 0;" ::: "memory");  // drop the prefetched chunk
            __syncthreads();
            cur = s_cur;
            pos = xat + 1;
            if (pos < n) walk_fetch(wbuf + cb * kWalkChunk, q, pos, n);
            break;
        }
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
}

static int grid_of(int64_t n) {
    const int sms = sm_count();
    return (int)std::max<int64_t>(1, std::min<int64_t>((n + kThreads - 1) / kThreads, (int64_t)sms * 8));
}

}  // namespace diaq

using namespace diaq;

#define DIAQ_CK(call)                                                                                \
    do {                                                                                             \
        cudaError_t e_ = (call);                                                                     \
        if (e_ != cudaSuccess) {                                                                     \
            rc = set_error(DIAQ_ERR_CUDA, "diaq_sample_hits: %s (%s)", #call, cudaGetErrorString(e_)); \
            goto done;                                                                               \
        }                                                                                            \
    } while (0)

extern "C" int diaq_sample_hits(int64_t n, const void *x, const double *u_host, int64_t shots, int64_t *hits_host,
                                double *norm2_out, void *stream) {
    if (!x || n < 1 || shots < 0 || (shots > 0 && (!u_host || !hits_host)))
        return set_error(DIAQ_ERR_VALUE, "diaq_sample_hits: bad arguments");
    cudaStream_t s = (cudaStream_t)stream;
    int rc = DIAQ_OK;
    // scan chunks grow geometrically: the running sum's binades (each a
    // segment of exact integer scan) double in length along the index, so a
    // chunk about twice the last segment wastes little work past an exit and
    // keeps the host round trips to ~ one per binade
    const int64_t C = std::min<int64_t>(n, (int64_t)1 << 26);
    int64_t want = std::min<int64_t>(C, (int64_t)1 << 16);
    double *q = nullptr, *c = nullptr, *part = nullptr, *ud = nullptr;
    long long *k = nullptr, *S = nullptr, *hd = nullptr;
    unsigned char *tie = nullptr;
    unsigned long long *flag = nullptr;
    void *tmp = nullptr;
    size_t tmp_bytes = 0;
    const int gq = grid_of(n);
    std::vector<double> hpart((size_t)gq);
    unsigned long long first = ~0ull;
    DIAQ_CK(cudaMallocAsync((void **)&q, sizeof(double) * (size_t)n, s));
    DIAQ_CK(cudaMallocAsync((void **)&c, sizeof(double) * (size_t)n, s));
    DIAQ_CK(cudaMallocAsync((void **)&part, sizeof(double) * (size_t)gq, s));
    DIAQ_CK(cudaMallocAsync((void **)&k, sizeof(long long) * (size_t)C, s));
    DIAQ_CK(cudaMallocAsync((void **)&S, sizeof(long long) * (size_t)C, s));
    DIAQ_CK(cudaMallocAsync((void **)&tie, (size_t)C, s));
    DIAQ_CK(cudaMallocAsync((void **)&flag, sizeof(unsigned long long), s));
    cub::DeviceScan::InclusiveSum(nullptr, tmp_bytes, k, S, (int)C, s);
    DIAQ_CK(cudaMallocAsync(&tmp, std::max<size_t>(tmp_bytes, 16), s));
    DIAQ_CK(cudaMemsetAsync(flag, 0xff, sizeof(unsigned long long), s));
    sample_q_kernel<<<gq, kThreads, 0, s>>>((const double2 *)x, n, q, part, flag);
    count_launch();
    DIAQ_CK(cudaGetLastError());
    DIAQ_CK(cudaMemcpyAsync(hpart.data(), part, sizeof(double) * (size_t)gq, cudaMemcpyDeviceToHost, s));
    DIAQ_CK(cudaMemcpyAsync(&first, flag, sizeof(first), cudaMemcpyDeviceToHost, s));
    DIAQ_CK(cudaStreamSynchronize(s));
    if (norm2_out) {
        double t = 0.0;
        for (double v : hpart) t += v;
        *norm2_out = t;
    }
    if (shots == 0) goto done;
    if (n <= ((int64_t)1 << 24)) {  // one-CTA device walk (no round trips)
        cudaFuncSetAttribute(sample_walk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kWalkSmem);
        sample_walk_kernel<<<1, kWalkThreads, kWalkSmem, s>>>(q, n, flag, c);
        count_launch();
        DIAQ_CK(cudaGetLastError());
        goto search;
    }
    // elements before the first nonzero q have cdf 0
    if (first == ~0ull) {
        DIAQ_CK(cudaMemsetAsync(c, 0, sizeof(double) * (size_t)n, s));
    } else {
        const int64_t s0 = (int64_t)first;
        if (s0 > 0) DIAQ_CK(cudaMemsetAsync(c, 0, sizeof(double) * (size_t)s0, s));
        double cur = 0.0;
        DIAQ_CK(cudaMemcpyAsync(&cur, q + s0, sizeof(double), cudaMemcpyDeviceToHost, s));
        DIAQ_CK(cudaStreamSynchronize(s));
        DIAQ_CK(cudaMemcpyAsync(c + s0, &cur, sizeof(double), cudaMemcpyHostToDevice, s));
        int64_t i = s0 + 1;
        while (i < n) {
            int e = 0;
            std::frexp(cur, &e);            // cur in [2^(e-1), 2^e)
            const int eb = e - 1;            // binade exponent
            const double U = std::ldexp(1.0, eb - 52);
            const double scale = std::ldexp(1.0, 52 - eb);
            long long kbase = (long long)std::ldexp(cur, 52 - eb);  // exact integer in [2^52, 2^53)
            // walk chunks until the segment ends
            while (i < n) {
                const int64_t cnt = std::min<int64_t>(want, n - i);
                const int g = grid_of(cnt);
                sample_k_kernel<<<g, kThreads, 0, s>>>(q, i, cnt, scale, k, tie);
                cub::DeviceScan::InclusiveSum(tmp, tmp_bytes, k, S, (int)cnt, s);
                DIAQ_CK(cudaMemsetAsync(flag, 0xff, sizeof(unsigned long long), s));
                sample_exit_kernel<<<g, kThreads, 0, s>>>(S, tie, cnt, kbase, flag);
                count_launch(3);
                DIAQ_CK(cudaGetLastError());
                unsigned long long ex = ~0ull;
                long long last = 0;
                DIAQ_CK(cudaMemcpyAsync(&ex, flag, sizeof(ex), cudaMemcpyDeviceToHost, s));
                DIAQ_CK(cudaMemcpyAsync(&last, S + cnt - 1, sizeof(last), cudaMemcpyDeviceToHost, s));
                DIAQ_CK(cudaStreamSynchronize(s));
                const int64_t upto = ex == ~0ull ? cnt : (int64_t)ex;
                if (upto > 0) {
                    sample_c_kernel<<<grid_of(upto), kThreads, 0, s>>>(S, i, upto, kbase, U, c);
                    count_launch();
                    DIAQ_CK(cudaGetLastError());
                }
                if (ex == ~0ull) {
                    kbase += last;
                    i += cnt;
                    want = std::min<int64_t>(C, want * 2);
                    continue;
                }
                want = std::min<int64_t>(C, std::max<int64_t>((int64_t)1 << 16, 2 * (upto + 1)));
                // the exiting element: one float64 step on the host, then a new segment
                long long sprev = 0;
                double qx = 0.0;
                if (upto > 0) DIAQ_CK(cudaMemcpyAsync(&sprev, S + upto - 1, sizeof(sprev), cudaMemcpyDeviceToHost, s));
                DIAQ_CK(cudaMemcpyAsync(&qx, q + i + upto, sizeof(qx), cudaMemcpyDeviceToHost, s));
                DIAQ_CK(cudaStreamSynchronize(s));
                const double cprev = (double)(kbase + sprev) * U;
                volatile double sum = cprev + qx;  // IEEE add, round to nearest even
                cur = sum;
                // pageable source: staged before the call returns, so &cur may be reused
                DIAQ_CK(cudaMemcpyAsync(c + i + upto, &cur, sizeof(double), cudaMemcpyHostToDevice, s));
                i += upto + 1;
                break;
            }
        }
    }
search:
    DIAQ_CK(cudaMallocAsync((void **)&ud, sizeof(double) * (size_t)shots, s));
    DIAQ_CK(cudaMallocAsync((void **)&hd, sizeof(long long) * (size_t)shots, s));
    DIAQ_CK(cudaMemcpyAsync(ud, u_host, sizeof(double) * (size_t)shots, cudaMemcpyHostToDevice, s));
    sample_search_kernel<<<(unsigned)((shots + kThreads - 1) / kThreads), kThreads, 0, s>>>(c, n, ud, shots, hd);
    count_launch();
    DIAQ_CK(cudaGetLastError());
    DIAQ_CK(cudaMemcpyAsync(hits_host, hd, sizeof(long long) * (size_t)shots, cudaMemcpyDeviceToHost, s));
    DIAQ_CK(cudaStreamSynchronize(s));
done:
    for (void *p : {(void *)q, (void *)c, (void *)part, (void *)k, (void *)S, (void *)tie, (void *)flag, tmp,
                    (void *)ud, (void *)hd})
        if (p) cudaFreeAsync(p, s);
    return rc;
}
