// dev_common.cuh -- device-only helpers shared by the AOT kernels and the
// runtime-specialised (NVRTC) fused passes: no host code, no includes under
// NVRTC (the JIT prelude supplies the fixed-width types and DIAQ_CMUL_*).
//
// Arithmetic helpers spell every rounding step with __dmul_rn/__dadd_rn/
// __fma_rn so nvcc cannot contract differently from the reference:
//   * spmv / spgemm terms: tr = re*xr - im*xi, ti = re*xi + im*xr with every
//     product rounded (numpy float64 ufuncs, reference matrix.py:214-215,
//     276-277);
//   * gate apply: numpy complex128 multiply (reference sim.py:76-78),
//     either the AVX-512 FMA form or the plain form (DIAQ_CMUL_*).
#pragma once
#ifndef __CUDACC_RTC__
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/diaq_b200.h"
#endif

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

// same, without an L2 policy operand
__device__ __forceinline__ void cp_async16_nohint(void *dst, const void *src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}

// 256-bit streaming store of two adjacent elements (p must be 32-byte aligned)
__device__ __forceinline__ void st_stream2(double2 *p, double2 a, double2 b) {
    asm volatile("st.global.cs.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(a.x), "d"(a.y), "d"(b.x), "d"(b.y)
                 : "memory");
}

__device__ __forceinline__ void st_hint(double2 *p, double2 v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(p), "d"(v.x), "d"(v.y), "l"(pol) : "memory");
}

__device__ __forceinline__ void st_plain(double2 *p, double2 v) {
    asm volatile("st.global.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(v.x), "d"(v.y) : "memory");
}

// ---- thread-block clusters (distributed shared memory) ---------------------

// all threads of all CTAs of the cluster; release/acquire on shared::cluster
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory");
}

// 16-byte load from CTA `rank`'s shared memory at this CTA's offset `local`
__device__ __forceinline__ double2 ld_dsmem(uint32_t local, uint32_t rank) {
    uint32_t ra;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(local), "r"(rank));
    double2 v;
    asm volatile("ld.shared::cluster.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(ra) : "memory");
    return v;
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
    if constexpr (MODE == DIAQ_CMUL_PLAIN) return cmul_plain(v, x);
    else return cmul_fma(v, x);
}

// ---- contracted forms (DIAQ_CMUL_CONTRACT; 1e-12 tolerance, not bitwise) ----
// a x + b y as one chain of fused multiply-adds: 1 DMUL + 3 DFMA per part
__device__ __forceinline__ double2 cmac2_c(double2 a, double2 x, double2 b, double2 y) {
    return make_double2(__fma_rn(a.x, x.x, __fma_rn(-a.y, x.y, __fma_rn(b.x, y.x, -__dmul_rn(b.y, y.y)))),
                        __fma_rn(a.x, x.y, __fma_rn(a.y, x.x, __fma_rn(b.x, y.y, __dmul_rn(b.y, y.x)))));
}

// real a, b: a x + b y (RY, H): 1 DMUL + 1 DFMA per part
__device__ __forceinline__ double2 cmac2_rr(double a, double2 x, double b, double2 y) {
    return make_double2(__fma_rn(a, x.x, __dmul_rn(b, y.x)), __fma_rn(a, x.y, __dmul_rn(b, y.y)));
}

// real a, imaginary b = i bi: a x + i bi y (RX rows)
__device__ __forceinline__ double2 cmac2_ri(double a, double2 x, double bi, double2 y) {
    return make_double2(__fma_rn(a, x.x, -__dmul_rn(bi, y.y)), __fma_rn(a, x.y, __dmul_rn(bi, y.x)));
}

// unit-diagonal rows (contracted rotations with the common diagonal entry
// factored out of the pass, fused.cu unit forms): x + b y, 1 DFMA per part
__device__ __forceinline__ double2 cmac1_r(double2 x, double b, double2 y) {
    return make_double2(__fma_rn(b, y.x, x.x), __fma_rn(b, y.y, x.y));
}

// x + i bi y
__device__ __forceinline__ double2 cmac1_i(double2 x, double bi, double2 y) {
    return make_double2(__fma_rn(-bi, y.y, x.x), __fma_rn(bi, y.x, x.y));
}

// acc + a x (continuing a contracted chain)
__device__ __forceinline__ double2 cfma_c(double2 a, double2 x, double2 acc) {
    return make_double2(__fma_rn(a.x, x.x, __fma_rn(-a.y, x.y, acc.x)), __fma_rn(a.x, x.y, __fma_rn(a.y, x.x, acc.y)));
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
