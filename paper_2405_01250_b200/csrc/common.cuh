// common.cuh -- shared device helpers for the DiaQ sm_100a kernels.
//
// Arithmetic helpers spell every rounding step with __dmul_rn/__dadd_rn/
// __fma_rn so nvcc cannot contract differently from the reference:
//   * spmv / spgemm terms: tr = re*xr - im*xi, ti = re*xi + im*xr with every
//     product rounded (numpy float64 ufuncs, reference matrix.py:214-215,
//     276-277);
//   * gate apply: numpy complex128 multiply (reference sim.py:76-78),
//     either the AVX-512 FMA form or the plain form (DIAQ_CMUL_*).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/diaq_b200.h"

namespace diaq {

constexpr int kThreads = 256;
constexpr int kSms = 148;          // B200 SM count (grid sizing default)
constexpr int kParamDiags = 64;    // diagonals passed by value in kernel params

// ---- loads / stores with cache policy ---------------------------------------

__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}

__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}

// streamed, read-once data (matrix diagonals): no L1 allocation, L2 evict-first
__device__ __forceinline__ double2 ld_stream(const double2 *p, uint64_t pol) {
    double2 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;"
                 : "=d"(v.x), "=d"(v.y)
                 : "l"(p), "l"(pol));
    return v;
}

// reused read-only data (state vector windows): normal L1/L2 allocation
__device__ __forceinline__ double2 ld_reuse(const double2 *p) {
    double2 v;
    asm volatile("ld.global.nc.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
    return v;
}

__device__ __forceinline__ double2 ld_reuse_hint(const double2 *p, uint64_t pol) {
    double2 v;
    asm volatile("ld.global.nc.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;"
                 : "=d"(v.x), "=d"(v.y)
                 : "l"(p), "l"(pol));
    return v;
}

// plain coherent load (buffers that may alias the output)
__device__ __forceinline__ double2 ld_plain(const double2 *p) {
    double2 v;
    asm volatile("ld.global.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p) : "memory");
    return v;
}

// write-once output: streaming store
__device__ __forceinline__ void st_stream(double2 *p, double2 v) {
    asm volatile("st.global.cs.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(v.x), "d"(v.y) : "memory");
}

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

// global -> shared 16-byte copy through L2 only (LDGSTS); no register is
// held while it is in flight
__device__ __forceinline__ void cp_async16(void *dst, const void *src, uint64_t pol) {
    asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src),
                 "l"(pol)
                 : "memory");
}

// 256-bit streaming store of two adjacent elements (p must be 32-byte aligned)
__device__ __forceinline__ void st_stream2(double2 *p, double2 a, double2 b) {
    asm volatile("st.global.cs.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(a.x), "d"(a.y), "d"(b.x), "d"(b.y)
                 : "memory");
}

__device__ __forceinline__ void st_plain(double2 *p, double2 v) {
    asm volatile("st.global.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(v.x), "d"(v.y) : "memory");
}

// ---- exact-rounding complex arithmetic ------------------------------------

// spmv/spgemm term: (re*xr - im*xi, re*xi + im*xr), each product rounded
__device__ __forceinline__ double2 cmul_plain(double2 v, double2 x) {
    return make_double2(__dsub_rn(__dmul_rn(v.x, x.x), __dmul_rn(v.y, x.y)),
                        __dadd_rn(__dmul_rn(v.x, x.y), __dmul_rn(v.y, x.x)));
}

// numpy complex128 multiply on AVX-512: re = fma(vr,xr,-(vi*xi)), im = fma(vr,xi,vi*xr)
__device__ __forceinline__ double2 cmul_fma(double2 v, double2 x) {
    return make_double2(__fma_rn(v.x, x.x, -__dmul_rn(v.y, x.y)),
                        __fma_rn(v.x, x.y, __dmul_rn(v.y, x.x)));
}

template <int MODE>
__device__ __forceinline__ double2 cmul(double2 v, double2 x) {
    if constexpr (MODE == DIAQ_CMUL_FMA) return cmul_fma(v, x);
    else return cmul_plain(v, x);
}

// products with a coefficient whose other part is an exact zero (see
// fused.cu dense1_full): equal to both cmul forms up to the sign of a zero
__device__ __forceinline__ double2 cmul_re(double vr, double2 x) {
    return make_double2(__dmul_rn(vr, x.x), __dmul_rn(vr, x.y));
}

__device__ __forceinline__ double2 cmul_im(double vi, double2 x) {
    return make_double2(-__dmul_rn(vi, x.y), __dmul_rn(vi, x.x));
}

__device__ __forceinline__ double2 cadd(double2 a, double2 b) {
    return make_double2(__dadd_rn(a.x, b.x), __dadd_rn(a.y, b.y));
}

// insert a zero bit at each of the (ascending) positions sh[0..K-1]
template <int K>
__device__ __forceinline__ uint64_t insert_zero_bits(uint64_t g, const int *sh) {
#pragma unroll
    for (int i = 0; i < K; ++i) {
        const uint64_t low = g & ((1ull << sh[i]) - 1ull);
        g = ((g >> sh[i]) << (sh[i] + 1)) | low;
    }
    return g;
}

}  // namespace diaq

// ---- host-side error plumbing (defined in abi.cu) ------------------------
namespace diaq {
// launch-geometry knobs (diaq_tune); results never depend on them
struct Tuning {
    int spmv_raster = 1;       // 0: strips fastest per tile, 1: column chunks
    int spmv_chunk = 8;        // strips per work item in raster 1
    int spmv_xpol = 0;         // 0: x evict_normal, 1: x evict_last
    int spmv_ctas_per_sm = 0;  // 0: occupancy maximum
    int spmv_banded = 1;       // stage banded x windows in shared memory
    int spmv_strips = 1;       // strip raster for far offsets (0: plain row order)
    int spmv_tma = 0;          // banded path through the TMA bulk-copy pipeline (opt-in: measured slower)
    int spmv_tma_stages = 4;   // tiles in flight per CTA
    int spmv_async = 1;        // banded path through cp.async (LDGSTS) staging (default: fastest)
    int gate_ctas_per_sm = 32;
    int fused_dense2 = 1;      // dense two-qubit gates in registers (sequence phases)
    int fused_gperm_rows = 0;  // 1: global tails only while they keep 128-byte rows whole (measured slower: an extra pass costs more than partial-row writes)
    int fused_gperm = 1;       // trailing permutation runs leaving the tile folded into the pass's store
    int fused_seq = 1;         // sequence phases (compile-time register bit per dense step)
    int fused_nbuf = 0;        // fused pass tile buffers: 0 auto (2 unless it costs occupancy), 1, 2
    int fused_perm = 1;        // fold permutation gates (X/CX/SWAP) into the fused passes' smem addressing
    int kron_flat = 1;         // kron_identity as one arena-linear store stream
    int kron_ctas_per_sm = 32;  // CTAs per SM launched (4 resident; later ones refill)
};
Tuning &tuning();
// SM count of the current device and resident CTAs per SM of a kernel,
// asked of the runtime once per (device, kernel, block, smem) -- each query
// costs microseconds, which is the whole budget of a small launch
int sm_count();
int occupancy(const void *kernel, int threads, size_t smem);
int set_error(int code, const char *fmt, ...);
void count_launch(int n = 1);
int check_launch(const char *what);
}  // namespace diaq
