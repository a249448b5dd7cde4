// spmv.cu -- DiaQ sparse matrix-vector product y = A x on sm_100a.
//
// Reference: matrix.py:253-278.  For every row r the reference adds, in
// ascending diagonal order d, the term D_d[r+min(d,0)] * x[r+d] with
// tr = re*xr - im*xi, ti = re*xi + im*xr (each product rounded) into
// zero-initialised accumulators.  This kernel is output-stationary: one
// thread owns one row, walks the diagonals in the same ascending order with
// the same rounding, and writes y exactly once -- results are bitwise equal
// to the reference, independent of the launch geometry.
//
// Memory plan (HBM-bound, 16*sum(N-|d|) + 32*N algorithmic bytes):
//   * diagonals are streamed once: LDG.128 with L1::no_allocate and an
//     L2 evict_first policy so they do not push x out of L2;
//   * x is read through L1/L2 (reused by every diagonal of a row window);
//   * y is written once with a streaming store;
//   * tile order is strip-rastered: with far offsets +-S (config 4:
//     S = 2^21 rows = 32 MiB of x), plain row order would evict x between
//     its uses by rows r-S, r, r+S (reuse distance ~ S*(16*nd+32) B = 369 MB
//     > 126 MB L2).  Tiles are visited as (b, j) with the strip index j
//     fastest, t = j*(S/T) + b, so the tiles that share an x window run
//     back to back and x comes from HBM about once.
#include <algorithm>
#include <cstring>
#include <cstdlib>
#include <vector>

#include "common.cuh"

namespace diaq {

struct SpmvDiag {
    const double2 *row0;  // element of row r is row0[r]
    int64_t lo, hi;       // valid rows [lo, hi)
    int64_t off;          // d
    int band, resid;      // banded path: x band and offset inside it (d = center[band] + resid)
};

constexpr int kMaxBands = 4;
constexpr int kMaxHalo = 32;

constexpr int kMaxParts = 64;

template <int MAXD>
struct SpmvParams {
    int64_t n;
    int part_bits;                    // sharded x (kernels instantiated with kParts): slice q of
    const double2 *parts[kMaxParts];  // 2^part_bits elements at parts[q] (own or peer-mapped)
    int64_t r0, rend;  // rows [r0, rend) of y are produced
    int64_t ntiles, stride_tiles, nstrips, nitems;
    int64_t nchunks;   // raster 1: chunks of `chunk` strips per column
    int raster, chunk;
    const double2 *x;
    double2 *y;
    int nd;
    int nbands, halo;               // banded path: x windows staged in shared memory
    int64_t center[kMaxBands];
    SpmvDiag dg[MAXD];
};

template <int XPOL>
__device__ __forceinline__ double2 ld_x(const double2 *p, uint64_t pol_last) {
    if constexpr (XPOL == 1) return ld_reuse_hint(p, pol_last);
    else return ld_reuse(p);
}

// one row: ascending-d accumulation with reference rounding
template <int ND, int XPOL>
__device__ __forceinline__ double2 spmv_row(const SpmvDiag *dg, int nd, int64_t r, const double2 *x,
                                            uint64_t pol, uint64_t pol_last) {
    double2 v[ND > 0 ? ND : 1], xv[ND > 0 ? ND : 1];
#pragma unroll
    for (int i = 0; i < ND; ++i) {
        const bool ok = (r >= dg[i].lo) & (r < dg[i].hi);
        if (ok) {
            v[i] = ld_stream(dg[i].row0 + r, pol);
            xv[i] = ld_x<XPOL>(x + r + dg[i].off, pol_last);
        } else {
            v[i] = make_double2(0.0, 0.0);
            xv[i] = make_double2(0.0, 0.0);
        }
    }
    double2 acc = make_double2(0.0, 0.0);
#pragma unroll
    for (int i = 0; i < ND; ++i) {
        const bool ok = (r >= dg[i].lo) & (r < dg[i].hi);
        if (ok) acc = cadd(acc, cmul_plain(v[i], xv[i]));
    }
    (void)nd;
    return acc;
}

// runtime diagonal count (ND == 0): same order, loads not hoisted
template <int XPOL>
__device__ __forceinline__ double2 spmv_row_dyn(const SpmvDiag *dg, int nd, int64_t r,
                                                const double2 *x, uint64_t pol, uint64_t pol_last) {
    double2 acc = make_double2(0.0, 0.0);
#pragma unroll 4
    for (int i = 0; i < nd; ++i) {
        if (r >= dg[i].lo && r < dg[i].hi) {
            const double2 v = ld_stream(dg[i].row0 + r, pol);
            const double2 xv = ld_x<XPOL>(x + r + dg[i].off, pol_last);
            acc = cadd(acc, cmul_plain(v, xv));
        }
    }
    return acc;
}

// Work item -> tiles.  raster 0: item = (b, j) with the strip j fastest, one
// tile per item.  raster 1: item = (b, chunk of strips) -- one CTA walks
// `chunk` strips of column b, so the x tile of strip j is reused by the same
// CTA for strips j-1, j, j+1 (L1/L2 hits) and HBM sees x about once.
template <int MAXD, int ND, int XPOL>
__global__ void __launch_bounds__(kThreads) spmv_kernel(const __grid_constant__ SpmvParams<MAXD> p) {
    const uint64_t pol = policy_evict_first();
    const uint64_t pol_last = XPOL ? policy_evict_last() : 0ull;
    for (int64_t it = blockIdx.x; it < p.nitems; it += gridDim.x) {
        int64_t b, j0, j1;
        if (p.raster == 0) {
            j0 = it % p.nstrips;
            b = it / p.nstrips;
            j1 = j0 + 1;
        } else {
            const int64_t jc = it % p.nchunks;
            b = it / p.nchunks;
            j0 = jc * p.chunk;
            j1 = j0 + p.chunk < p.nstrips ? j0 + p.chunk : p.nstrips;
        }
        if (b >= p.stride_tiles) continue;
        for (int64_t j = j0; j < j1; ++j) {
            const int64_t t = j * p.stride_tiles + b;
            if (t >= p.ntiles) break;
            const int64_t r = p.r0 + t * kThreads + threadIdx.x;
            if (r >= p.rend) continue;
            double2 acc;
            if constexpr (ND > 0) acc = spmv_row<ND, XPOL>(p.dg, p.nd, r, p.x, pol, pol_last);
            else acc = spmv_row_dyn<XPOL>(p.dg, p.nd, r, p.x, pol, pol_last);
            st_stream(p.y + r, acc);
        }
    }
}

// Banded variant: the offsets form <= 4 bands (e.g. config 4: {-S, 0, +S}
// each +-8).  Per 256-row tile every band's x window [r0 + c - h, r0 + 256 +
// c + h) is staged once in shared memory by coalesced loads, and every row
// reads its x values from there -- one L2 request per x line per band
// instead of one per diagonal (the near offsets +-8 otherwise re-read x
// lines through L1 misses and cost ~27% extra x traffic from HBM).  Same
// per-row ascending-d arithmetic: bitwise identical results.
template <int ND>
__global__ void __launch_bounds__(kThreads) spmv_banded_kernel(const __grid_constant__ SpmvParams<kParamDiags> p) {
    __shared__ double2 xs[kMaxBands][kThreads + 2 * kMaxHalo];
    const uint64_t pol = policy_evict_first();
    const int h = p.halo;
    const int w = kThreads + 2 * h;
    for (int64_t it = blockIdx.x; it < p.nitems; it += gridDim.x) {
        const int64_t j = it % p.nstrips;
        const int64_t b = it / p.nstrips;
        const int64_t t = j * p.stride_tiles + b;
        if (b >= p.stride_tiles || t >= p.ntiles) continue;  // uniform over the CTA
        const int64_t r0t = p.r0 + t * kThreads;
        for (int bd = 0; bd < p.nbands; ++bd) {
            const int64_t base = r0t + p.center[bd] - h;
            for (int i = threadIdx.x; i < w; i += kThreads) {
                const int64_t idx = base + i;
                xs[bd][i] = (idx >= 0 && idx < p.n) ? ld_reuse(p.x + idx) : make_double2(0.0, 0.0);
            }
        }
        __syncthreads();
        const int64_t r = r0t + threadIdx.x;
        if (r < p.rend) {
            double2 v[ND], xv[ND];
#pragma unroll
            for (int i = 0; i < ND; ++i) {
                const bool ok = (r >= p.dg[i].lo) & (r < p.dg[i].hi);
                v[i] = ok ? ld_stream(p.dg[i].row0 + r, pol) : make_double2(0.0, 0.0);
                xv[i] = xs[p.dg[i].band][threadIdx.x + h + p.dg[i].resid];
            }
            double2 acc = make_double2(0.0, 0.0);
#pragma unroll
            for (int i = 0; i < ND; ++i) {
                const bool ok = (r >= p.dg[i].lo) & (r < p.dg[i].hi);
                if (ok) acc = cadd(acc, cmul_plain(v[i], xv[i]));
            }
            st_stream(p.y + r, acc);
        }
        __syncthreads();
    }
}


// ---- cp.async variant (banded matrices) --------------------------------------
// Every diagonal value of the tile is copied global -> shared with
// cp.async (LDGSTS: no register is held while the load is in flight), so all
// ND loads of a row are outstanding at once at full occupancy (128-thread
// CTAs, 16 per SM), instead of the ~3 that fit in registers.
constexpr int kAsyncThreads = 128;


// parameters sized by the diagonal count (a launch copies the whole block:
// the 64-diagonal table was ~4 KB per call of a 3-diagonal product)
template <int ND, bool kParts>
__global__ void __launch_bounds__(kAsyncThreads) spmv_async_kernel(const __grid_constant__ SpmvParams<ND> p) {
    __shared__ __align__(16) double2 sd[ND > 0 ? ND : 1][kAsyncThreads];
    __shared__ __align__(16) double2 xs[kMaxBands][kAsyncThreads + 2 * kMaxHalo];
    const uint64_t pol = policy_evict_first();
    uint64_t polx;
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(polx));
    const int h = p.halo;
    const int w = kAsyncThreads + 2 * h;
    for (int64_t it = blockIdx.x; it < p.nitems; it += gridDim.x) {
        const int64_t j = it % p.nstrips;
        const int64_t b = it / p.nstrips;
        const int64_t t = j * p.stride_tiles + b;
        if (b >= p.stride_tiles || t >= p.ntiles) continue;  // uniform over the CTA
        const int64_t r0t = p.r0 + t * kAsyncThreads;
        const int64_t r = r0t + threadIdx.x;
#pragma unroll
        for (int i = 0; i < ND; ++i)
            if (r < p.rend && r >= p.dg[i].lo && r < p.dg[i].hi) cp_async16(&sd[i][threadIdx.x], p.dg[i].row0 + r, pol);
        for (int bd = 0; bd < p.nbands; ++bd) {
            const int64_t base = r0t + p.center[bd] - h;
            for (int i = threadIdx.x; i < w; i += kAsyncThreads) {
                const int64_t idx = base + i;
                if (idx >= 0 && idx < p.n) {
                    if constexpr (kParts)  // x slice of the owning rank: a peer load across the boundary
                        cp_async16(&xs[bd][i], p.parts[idx >> p.part_bits] + (idx & ((1ll << p.part_bits) - 1)), polx);
                    else
                        cp_async16(&xs[bd][i], p.x + idx, polx);
                }
            }
        }
        asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
        __syncthreads();
        if (r < p.rend) {
            double2 acc = make_double2(0.0, 0.0);
#pragma unroll
            for (int i = 0; i < ND; ++i) {
                if ((r >= p.dg[i].lo) & (r < p.dg[i].hi))
                    acc = cadd(acc, cmul_plain(sd[i][threadIdx.x], xs[p.dg[i].band][threadIdx.x + h + p.dg[i].resid]));
            }
            st_stream(p.y + r, acc);
        }
        __syncthreads();
    }
}

// ---- TMA bulk-copy pipeline (banded matrices) --------------------------------
// A single elected thread streams each tile's inputs into shared memory with
// cp.async.bulk (one contiguous copy per diagonal segment and per x band
// window, completion counted on an mbarrier), double-buffered so the copies
// of tile k+1 overlap the arithmetic of tile k.  The loads need no registers,
// so memory-level parallelism no longer trades against occupancy.

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}

constexpr int kTmaMaxStages = 4;

// stage layout in dynamic shared memory: ND diagonal segments of 256
// elements, then nbands x windows of 256 + 2h elements
struct TmaLayout {
    int ndiag, nbands, w;       // w = 256 + 2h
    uint32_t stage_elems;       // double2 elements per stage
};

// issue the copies of the tile at rows [r0, r0 + 256) into stage buffer `sb`
template <int ND>
__device__ __forceinline__ void tma_issue(const SpmvParams<kParamDiags> &p, double2 *sb, int w, int64_t r0,
                                          uint64_t *bar, uint64_t pol_first, uint64_t pol_x) {
    uint32_t total = 0;
    const int h = p.halo;
    for (int i = 0; i < ND; ++i) {
        const int64_t a = r0 > p.dg[i].lo ? r0 : p.dg[i].lo;
        const int64_t b = r0 + kThreads < p.dg[i].hi ? r0 + kThreads : p.dg[i].hi;
        if (a < b) total += (uint32_t)(b - a) * 16u;
    }
    for (int bd = 0; bd < p.nbands; ++bd) {
        const int64_t lo = r0 + p.center[bd] - h, hi = r0 + kThreads + p.center[bd] + h;
        const int64_t a = lo > 0 ? lo : 0, b = hi < p.n ? hi : p.n;
        if (a < b) total += (uint32_t)(b - a) * 16u;
    }
    mbar_expect_tx(bar, total);
    for (int i = 0; i < ND; ++i) {
        const int64_t a = r0 > p.dg[i].lo ? r0 : p.dg[i].lo;
        const int64_t b = r0 + kThreads < p.dg[i].hi ? r0 + kThreads : p.dg[i].hi;
        if (a < b) bulk_g2s(sb + i * kThreads + (a - r0), p.dg[i].row0 + a, (uint32_t)(b - a) * 16u, bar, pol_first);
    }
    double2 *xb = sb + ND * kThreads;
    for (int bd = 0; bd < p.nbands; ++bd) {
        const int64_t lo = r0 + p.center[bd] - h, hi = r0 + kThreads + p.center[bd] + h;
        const int64_t a = lo > 0 ? lo : 0, b = hi < p.n ? hi : p.n;
        if (a < b) bulk_g2s(xb + bd * w + (a - lo), p.x + a, (uint32_t)(b - a) * 16u, bar, pol_x);
    }
}

template <int ND>
__global__ void __launch_bounds__(kThreads) spmv_tma_kernel(const __grid_constant__ SpmvParams<kParamDiags> p,
                                                            int nstages) {
    extern __shared__ __align__(128) double2 smem_stage[];
    __shared__ __align__(8) uint64_t bars[kTmaMaxStages];
    const int h = p.halo;
    const int w = kThreads + 2 * h;
    const uint32_t stage_elems = (uint32_t)(ND * kThreads + p.nbands * w);
    uint64_t pol_first = 0, pol_x = 0;
    if (threadIdx.x == 0) {
        pol_first = policy_evict_first();
        asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol_x));
        for (int s = 0; s < nstages; ++s) mbar_init(&bars[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    auto tile_of = [&](int64_t it, int64_t &r0) -> bool {
        const int64_t j = it % p.nstrips, b = it / p.nstrips;
        const int64_t t = j * p.stride_tiles + b;
        if (b >= p.stride_tiles || t >= p.ntiles) return false;
        r0 = p.r0 + t * kThreads;
        return true;
    };
    auto next_valid = [&](int64_t it, int64_t &r0) -> int64_t {
        while (it < p.nitems && !tile_of(it, r0)) it += gridDim.x;
        return it;
    };
    // ring of in-flight tiles: the producer (thread 0) keeps nstages-1 ahead
    int64_t q_it[kTmaMaxStages], q_r0[kTmaMaxStages];
    int64_t scratch = 0;
    int64_t fetch_it = next_valid(blockIdx.x, scratch);
    int issued = 0;
    for (; issued < nstages && fetch_it < p.nitems; ++issued) {
        q_it[issued] = fetch_it;
        tile_of(fetch_it, q_r0[issued]);
        if (threadIdx.x == 0) tma_issue<ND>(p, smem_stage + issued * stage_elems, w, q_r0[issued], &bars[issued],
                                            pol_first, pol_x);
        fetch_it = next_valid(fetch_it + gridDim.x, scratch);
    }
    uint32_t parity = 0;
    for (int k = 0; k < issued || fetch_it < p.nitems; ++k) {
        const int slot = k % nstages;
        if (k >= issued) break;
        mbar_wait(&bars[slot], parity);
        const double2 *sb = smem_stage + slot * stage_elems;
        const double2 *xb = sb + ND * kThreads;
        const int64_t r0 = q_r0[slot];
        const int64_t r = r0 + threadIdx.x;
        if (r < p.rend) {
            double2 acc = make_double2(0.0, 0.0);
#pragma unroll
            for (int i = 0; i < ND; ++i) {
                if ((r >= p.dg[i].lo) & (r < p.dg[i].hi)) {
                    const double2 v = sb[i * kThreads + threadIdx.x];
                    const double2 xv = xb[p.dg[i].band * w + threadIdx.x + h + p.dg[i].resid];
                    acc = cadd(acc, cmul_plain(v, xv));
                }
            }
            st_stream(p.y + r, acc);
        }
        __syncthreads();  // slot fully consumed before it is refilled
        if (fetch_it < p.nitems) {
            int64_t r0n = 0;
            tile_of(fetch_it, r0n);
            q_r0[slot] = r0n;
            q_it[slot] = fetch_it;
            if (threadIdx.x == 0) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                tma_issue<ND>(p, smem_stage + slot * stage_elems, w, r0n, &bars[slot], pol_first, pol_x);
            }
            ++issued;
            int64_t dummy = 0;
            fetch_it = next_valid(fetch_it + gridDim.x, dummy);
        }
        if (slot == nstages - 1) parity ^= 1u;
    }
    (void)q_it;
}

// large diagonal counts: tables in global memory, raster 0
__global__ void __launch_bounds__(kThreads)
spmv_kernel_global(int64_t r0, int64_t rend, int nd, const SpmvDiag *__restrict__ dg, const double2 *x,
                   double2 *y, int64_t ntiles, int64_t stride_tiles, int64_t nstrips, int64_t nitems) {
    const uint64_t pol = policy_evict_first();
    for (int64_t it = blockIdx.x; it < nitems; it += gridDim.x) {
        const int64_t j = it % nstrips;
        const int64_t b = it / nstrips;
        const int64_t t = j * stride_tiles + b;
        if (b >= stride_tiles || t >= ntiles) continue;
        const int64_t r = r0 + t * kThreads + threadIdx.x;
        if (r >= rend) continue;
        double2 acc = spmv_row_dyn<0>(dg, nd, r, x, pol, 0ull);
        st_stream(y + r, acc);
    }
}

// strip raster: pick S = the smallest "far" offset (reuse distance beyond a
// quarter of L2), rounded to whole tiles; linear order when none is far.
void spmv_raster(int64_t n, int64_t nd, const int64_t *offs, int64_t *ntiles, int64_t *stride,
                 int64_t *nstrips) {
    const int64_t nt = (n + kThreads - 1) / kThreads;
    const int64_t l2_budget = 126ll * 1024 * 1024 / 4;
    const int64_t bytes_per_row = 16 * nd + 32;
    const int64_t far_rows = std::max<int64_t>(4 * kThreads, l2_budget / bytes_per_row);
    int64_t s = 0;
    for (int64_t i = 0; i < nd; ++i) {
        const int64_t a = offs[i] < 0 ? -offs[i] : offs[i];
        if (a > far_rows && (s == 0 || a < s)) s = a;
    }
    *ntiles = nt;
    if (s == 0 || !tuning().spmv_strips) {
        *stride = nt;
        *nstrips = 1;
        return;
    }
    int64_t st = (s + kThreads / 2) / kThreads;
    if (st < 1) st = 1;
    *stride = st;
    *nstrips = (nt + st - 1) / st;
}

static int grid_for(const void *func, int64_t items, int ctas_per_sm = 0) {
    const int sms = sm_count();
    int per_sm = occupancy(func, kThreads, 0);
    if (ctas_per_sm > 0 && ctas_per_sm < per_sm) per_sm = ctas_per_sm;
    const int64_t g = std::min<int64_t>(items, (int64_t)sms * per_sm);
    return (int)std::max<int64_t>(g, 1);
}

template <int ND, int XPOL>
static int launch_param_x(const SpmvParams<kParamDiags> &p, cudaStream_t s) {
    const void *f = (const void *)spmv_kernel<kParamDiags, ND, XPOL>;
    const int grid = grid_for(f, p.nitems, tuning().spmv_ctas_per_sm);
    spmv_kernel<kParamDiags, ND, XPOL><<<grid, kThreads, 0, s>>>(p);
    count_launch();
    return check_launch("spmv_kernel");
}

template <int ND>
static void shrink_params(const SpmvParams<kParamDiags> &p, SpmvParams<ND> &q) {
    q.n = p.n;
    q.part_bits = p.part_bits;
    memcpy(q.parts, p.parts, sizeof(q.parts));
    q.r0 = p.r0;
    q.rend = p.rend;
    q.ntiles = p.ntiles;
    q.stride_tiles = p.stride_tiles;
    q.nstrips = p.nstrips;
    q.nitems = p.nitems;
    q.nchunks = p.nchunks;
    q.raster = p.raster;
    q.chunk = p.chunk;
    q.x = p.x;
    q.y = p.y;
    q.nd = p.nd;
    q.nbands = p.nbands;
    q.halo = p.halo;
    for (int b = 0; b < kMaxBands; ++b) q.center[b] = p.center[b];
    for (int i = 0; i < ND; ++i) q.dg[i] = p.dg[i];
}

// Per-thread cache of the last whole-matrix spmv launch (diaq_spmv on a
// <= 12-diagonal matrix): the planned parameters and grid, keyed by the
// matrix (arena, size, offsets, starts), the device and the tuning epoch.
// A repeated spmv of the same matrix -- the launch-bound small configs --
// then costs a key compare, two pointer stores and the launch.
struct SpmvLaunchCache {
    bool valid = false;
    int dev = -1;
    uint64_t epoch = 0;
    const void *vals = nullptr;
    int64_t n = 0, nd = 0;
    int64_t offs[12] = {0}, starts[12] = {0};
    int grid = 0;
    int (*fire)(SpmvLaunchCache &, const void *, void *, cudaStream_t) = nullptr;
    alignas(16) unsigned char q[sizeof(SpmvParams<12>)];
    bool pending = false;  // remember_async may fill it during this planning call
};
static thread_local SpmvLaunchCache g_spmv_cache;

template <int ND>
static int fire_async(SpmvLaunchCache &c, const void *x, void *y, cudaStream_t s) {
    SpmvParams<ND> &q = *reinterpret_cast<SpmvParams<ND> *>(c.q);
    q.x = (const double2 *)x;
    q.y = (double2 *)y;
    spmv_async_kernel<ND, false><<<c.grid, kAsyncThreads, 0, s>>>(q);
    count_launch();
    return check_launch("spmv_async_kernel");
}

template <int ND>
static void remember_async(const SpmvParams<ND> &q, int grid) {
    SpmvLaunchCache &c = g_spmv_cache;
    if (!c.pending) return;
    static_assert(sizeof(SpmvParams<ND>) <= sizeof(c.q), "cache slot");
    memcpy(c.q, &q, sizeof(q));
    c.grid = grid;
    c.fire = fire_async<ND>;
    c.valid = true;
}

template <int ND, bool kParts>
static int launch_async(const SpmvParams<kParamDiags> &p, cudaStream_t s) {
    const void *f = (const void *)spmv_async_kernel<ND, kParts>;
    SpmvParams<ND> q;
    shrink_params(p, q);
    const int64_t nrows = q.rend - q.r0;
    const int64_t nt = (nrows + kAsyncThreads - 1) / kAsyncThreads;
    const int64_t scale = kThreads / kAsyncThreads;  // strip stride in 128-row tiles
    q.ntiles = nt;
    q.stride_tiles = q.nstrips > 1 ? q.stride_tiles * scale : nt;
    q.nstrips = (nt + q.stride_tiles - 1) / q.stride_tiles;
    q.raster = 0;
    q.nitems = q.stride_tiles * q.nstrips;
    const int sms = sm_count();
    int per_sm = occupancy(f, kAsyncThreads, 0);
    if (tuning().spmv_ctas_per_sm > 0) per_sm = std::min(per_sm, tuning().spmv_ctas_per_sm);
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(q.nitems, (int64_t)sms * std::max(1, per_sm)));
    if constexpr (!kParts) remember_async<ND>(q, grid);
    spmv_async_kernel<ND, kParts><<<grid, kAsyncThreads, 0, s>>>(q);
    count_launch();
    return check_launch("spmv_async_kernel");
}

template <int ND>
static int launch_param(const SpmvParams<kParamDiags> &p, cudaStream_t s) {
    if constexpr (ND > 0) {
        if (p.nbands > 0 && tuning().spmv_async) return launch_async<ND, false>(p, s);
        if (p.nbands > 0 && tuning().spmv_tma) {
            const void *f = (const void *)spmv_tma_kernel<ND>;
            SpmvParams<kParamDiags> q = p;
            q.raster = 0;
            q.nitems = q.stride_tiles * q.nstrips;
            const int nstages = std::max(2, std::min(kTmaMaxStages, tuning().spmv_tma_stages));
            const size_t stage_bytes = 16 * (size_t)(ND * kThreads + q.nbands * (kThreads + 2 * q.halo));
            const size_t smem = stage_bytes * (size_t)nstages;
            cudaFuncSetAttribute(spmv_tma_kernel<ND>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            int per_sm = 1;
            const int sms = sm_count();
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, f, kThreads, smem);
            cudaGetLastError();
            if (tuning().spmv_ctas_per_sm > 0) per_sm = std::min(per_sm, tuning().spmv_ctas_per_sm);
            const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(q.nitems, (int64_t)sms * std::max(1, per_sm)));
            spmv_tma_kernel<ND><<<grid, kThreads, smem, s>>>(q, nstages);
            count_launch();
            return check_launch("spmv_tma_kernel");
        }
        if (p.nbands > 0) {
            const void *f = (const void *)spmv_banded_kernel<ND>;
            SpmvParams<kParamDiags> q = p;
            q.raster = 0;
            q.nitems = q.stride_tiles * q.nstrips;
            const int grid = grid_for(f, q.nitems, tuning().spmv_ctas_per_sm);
            spmv_banded_kernel<ND><<<grid, kThreads, 0, s>>>(q);
            count_launch();
            return check_launch("spmv_banded_kernel");
        }
    }
    return tuning().spmv_xpol ? launch_param_x<ND, 1>(p, s) : launch_param_x<ND, 0>(p, s);
}

// group ascending offsets into <= kMaxBands bands of half-width <= kMaxHalo
static void plan_bands(SpmvParams<kParamDiags> &p) {
    p.nbands = 0;
    p.halo = 0;
    if (!tuning().spmv_banded || p.nd > 12) return;
    int nb = 0;
    int64_t first[kMaxBands + 1], last[kMaxBands + 1];
    for (int i = 0; i < p.nd; ++i) {
        const int64_t d = p.dg[i].off;
        if (nb > 0 && d - first[nb - 1] <= 2 * kMaxHalo) {
            last[nb - 1] = d;
        } else {
            if (nb == kMaxBands) return;  // too many bands: direct path
            first[nb] = last[nb] = d;
            ++nb;
        }
    }
    if (nb == p.nd && nb > 1) return;  // no offset sharing: staging buys nothing
    int h = 0;
    for (int bd = 0; bd < nb; ++bd) {
        p.center[bd] = first[bd] + (last[bd] - first[bd]) / 2;
        h = std::max<int>(h, (int)std::max(p.center[bd] - first[bd], last[bd] - p.center[bd]));
    }
    h = (h + 7) & ~7;  // keep the staged windows 128-byte aligned
    if (h > kMaxHalo) return;
    for (int i = 0; i < p.nd; ++i) {
        const int64_t d = p.dg[i].off;
        int bd = 0;
        while (bd + 1 < nb && d > last[bd]) ++bd;
        p.dg[i].band = bd;
        p.dg[i].resid = (int)(d - p.center[bd]);
    }
    p.nbands = nb;
    p.halo = h;
}

}  // namespace diaq

using namespace diaq;

// y rows [r0, r0 + nrows) of y = A x (whole x and matrix addressable)
static int spmv_rows(const diaq_matrix_t *a, const void *x, void *y, int64_t r0, int64_t nrows, cudaStream_t s) {
    const int64_t n = a->n;
    if (nrows <= 0) return DIAQ_OK;
    if (a->nd == 0) {
        // no stored diagonals: y = 0 (reference returns zeros)
        if (cudaMemsetAsync((double2 *)y + r0, 0, (size_t)nrows * 16, s) != cudaSuccess)
            return set_error(DIAQ_ERR_CUDA, "diaq_spmv: memset failed: %s", cudaGetErrorString(cudaGetLastError()));
        return DIAQ_OK;
    }
    int64_t ntiles, stride, nstrips;
    spmv_raster(nrows, a->nd, a->offs, &ntiles, &stride, &nstrips);
    const double2 *vals = (const double2 *)a->vals;
    if (a->nd <= kParamDiags) {
        SpmvParams<kParamDiags> p;
        p.n = n;
        p.r0 = r0;
        p.rend = r0 + nrows;
        p.ntiles = ntiles;
        p.stride_tiles = stride;
        p.nstrips = nstrips;
        p.raster = tuning().spmv_raster ? 1 : 0;
        p.chunk = tuning().spmv_chunk;
        p.nchunks = (nstrips + p.chunk - 1) / p.chunk;
        p.nitems = p.raster ? stride * p.nchunks : stride * nstrips;
        p.x = (const double2 *)x;
        p.y = (double2 *)y;
        p.nd = (int)a->nd;
        for (int64_t i = 0; i < a->nd; ++i) {
            const int64_t d = a->offs[i];
            p.dg[i].off = d;
            p.dg[i].row0 = vals + a->starts[i] + (d < 0 ? d : 0);
            p.dg[i].lo = d < 0 ? -d : 0;
            p.dg[i].hi = d > 0 ? n - d : n;
            p.dg[i].band = 0;
            p.dg[i].resid = 0;
        }
        plan_bands(p);
        switch (a->nd) {
            case 1: return launch_param<1>(p, s);
            case 2: return launch_param<2>(p, s);
            case 3: return launch_param<3>(p, s);
            case 4: return launch_param<4>(p, s);
            case 5: return launch_param<5>(p, s);
            case 6: return launch_param<6>(p, s);
            case 7: return launch_param<7>(p, s);
            case 8: return launch_param<8>(p, s);
            case 9: return launch_param<9>(p, s);
            case 10: return launch_param<10>(p, s);
            case 11: return launch_param<11>(p, s);
            case 12: return launch_param<12>(p, s);
            default: return launch_param<0>(p, s);
        }
    }
    // many diagonals: stage the table in device memory (stream-ordered, no
    // host sync: the pinned staging block is released once an event behind
    // its copy has completed -- polled on later calls)
    struct Staged {
        cudaEvent_t ev;
        void *host;
    };
    static thread_local std::vector<Staged> staged;
    for (size_t i = 0; i < staged.size();) {
        if (cudaEventQuery(staged[i].ev) == cudaSuccess) {
            cudaEventDestroy(staged[i].ev);
            cudaFreeHost(staged[i].host);
            staged[i] = staged.back();
            staged.pop_back();
        } else {
            cudaGetLastError();  // cudaErrorNotReady
            ++i;
        }
    }
    const size_t bytes = sizeof(SpmvDiag) * (size_t)a->nd;
    SpmvDiag *h = nullptr;
    if (cudaMallocHost((void **)&h, bytes) != cudaSuccess || !h) {
        cudaGetLastError();
        return set_error(DIAQ_ERR_RESOURCE, "diaq_spmv: pinned host alloc failed");
    }
    for (int64_t i = 0; i < a->nd; ++i) {
        const int64_t d = a->offs[i];
        h[i].off = d;
        h[i].row0 = vals + a->starts[i] + (d < 0 ? d : 0);
        h[i].lo = d < 0 ? -d : 0;
        h[i].hi = d > 0 ? n - d : n;
    }
    SpmvDiag *dtab = nullptr;
    if (cudaMallocAsync((void **)&dtab, bytes, s) != cudaSuccess) {
        cudaFreeHost(h);
        return set_error(DIAQ_ERR_CUDA, "diaq_spmv: device table alloc failed");
    }
    cudaMemcpyAsync(dtab, h, bytes, cudaMemcpyHostToDevice, s);
    Staged st{nullptr, h};
    if (cudaEventCreateWithFlags(&st.ev, cudaEventDisableTiming) != cudaSuccess || cudaEventRecord(st.ev, s) != cudaSuccess) {
        cudaGetLastError();
        cudaStreamSynchronize(s);  // cannot track the copy: wait for it instead
        cudaFreeHost(h);
        if (st.ev) cudaEventDestroy(st.ev);
    } else {
        staged.push_back(st);
    }
    const int grid = grid_for((const void *)spmv_kernel_global, stride * nstrips);
    spmv_kernel_global<<<grid, kThreads, 0, s>>>(r0, r0 + nrows, (int)a->nd, dtab, (const double2 *)x, (double2 *)y,
                                                 ntiles, stride, nstrips, stride * nstrips);
    count_launch();
    const int rc = check_launch("spmv_kernel_global");
    cudaFreeAsync(dtab, s);
    return rc;
}

// ---- sharded spmv: this rank's rows, x spread over the ranks ----
// Rank q holds x[q*2^B, (q+1)*2^B) (B = part_bits) and the rows [row0,
// row0 + nrows) of every diagonal (rows[i][j] = D_{d_i} at row row0 + j).
// x_parts are the ranks' x slices as seen from this process: its own, and
// partners' through CUDA IPC peer mappings (NVLink / NVSwitch) -- so an
// offset that crosses a shard boundary is a direct peer load inside the
// kernel, no halo copy.  Same per-row ascending-d arithmetic as diaq_spmv:
// the sharded product is bitwise the single-GPU one.
struct ShardSpmvParams {
    int64_t row0, nrows;
    int part_bits, nparts;
    int nd;
    double2 *y;
    const double2 *parts[kMaxParts];
    const double2 *rows[kParamDiags];
    int64_t off[kParamDiags];
    int64_t lo[kParamDiags], hi[kParamDiags];  // global rows where diagonal i exists
};

template <int ND>
__global__ void __launch_bounds__(kThreads) spmv_sharded_kernel(const __grid_constant__ ShardSpmvParams p) {
    const uint64_t pol = policy_evict_first();
    const uint64_t mask = (1ull << p.part_bits) - 1ull;
    const int nd = ND > 0 ? ND : p.nd;
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < p.nrows; j += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = p.row0 + j;
        double2 acc = make_double2(0.0, 0.0);
        if constexpr (ND > 0) {
            double2 v[ND], xv[ND];
#pragma unroll
            for (int i = 0; i < ND; ++i) {
                if (r >= p.lo[i] && r < p.hi[i]) {
                    const uint64_t c = (uint64_t)(r + p.off[i]);
                    v[i] = ld_stream(p.rows[i] + j, pol);
                    xv[i] = ld_reuse(p.parts[c >> p.part_bits] + (c & mask));
                }
            }
#pragma unroll
            for (int i = 0; i < ND; ++i)
                if (r >= p.lo[i] && r < p.hi[i]) acc = cadd(acc, cmul_plain(v[i], xv[i]));
        } else {
            for (int i = 0; i < nd; ++i) {
                if (r >= p.lo[i] && r < p.hi[i]) {
                    const uint64_t c = (uint64_t)(r + p.off[i]);
                    acc = cadd(acc, cmul_plain(ld_stream(p.rows[i] + j, pol),
                                               ld_reuse(p.parts[c >> p.part_bits] + (c & mask))));
                }
            }
        }
        st_stream(p.y + j, acc);
    }
}

extern "C" int diaq_spmv_sharded(int64_t n, int64_t nd, const int64_t *offs, const void *const *rows, int64_t row0,
                                 int64_t nrows, const void *const *x_parts, int part_bits, int nparts, void *y,
                                 void *stream) {
    if (nd < 0 || (nd > 0 && (!offs || !rows)) || !x_parts || !y)
        return set_error(DIAQ_ERR_VALUE, "diaq_spmv_sharded: null argument");
    if (nd > kParamDiags) return set_error(DIAQ_ERR_UNSUPPORTED, "diaq_spmv_sharded: more than %d diagonals", kParamDiags);
    if (nparts < 1 || nparts > kMaxParts || part_bits < 0 || part_bits > 62 || ((int64_t)nparts << part_bits) != n)
        return set_error(DIAQ_ERR_SHAPE, "diaq_spmv_sharded: %d parts of 2^%d do not tile n=%lld", nparts, part_bits,
                         (long long)n);
    if (row0 < 0 || nrows < 0 || row0 + nrows > n) return set_error(DIAQ_ERR_SHAPE, "diaq_spmv_sharded: rows outside n");
    ShardSpmvParams p;
    memset(&p, 0, sizeof(p));
    p.row0 = row0;
    p.nrows = nrows;
    p.part_bits = part_bits;
    p.nparts = nparts;
    p.nd = (int)nd;
    p.y = (double2 *)y;
    for (int q = 0; q < nparts; ++q) {
        if (!x_parts[q]) return set_error(DIAQ_ERR_VALUE, "diaq_spmv_sharded: x part %d missing", q);
        p.parts[q] = (const double2 *)x_parts[q];
    }
    for (int64_t i = 0; i < nd; ++i) {
        const int64_t d = offs[i];
        if (d <= -n || d >= n) return set_error(DIAQ_ERR_VALUE, "diagonal %lld out of range for n_dim=%lld", (long long)d, (long long)n);
        if (i > 0 && offs[i - 1] >= d) return set_error(DIAQ_ERR_VALUE, "offsets must be strictly ascending");
        if (!rows[i]) return set_error(DIAQ_ERR_VALUE, "diaq_spmv_sharded: diagonal %lld rows missing", (long long)i);
        p.rows[i] = (const double2 *)rows[i];
        p.off[i] = d;
        p.lo[i] = d < 0 ? -d : 0;
        p.hi[i] = d > 0 ? n - d : n;
    }
    if (nrows == 0) return DIAQ_OK;
    cudaStream_t s = (cudaStream_t)stream;
    if (nd > 0 && nd <= 12 && tuning().spmv_async) {
        // banded offsets: the cp.async kernel of diaq_spmv with its x windows
        // staged from the owning rank's slice (row pointers rebased so the
        // element of global row r is at row0ptr[r])
        SpmvParams<kParamDiags> q;
        memset(&q, 0, sizeof(q));
        q.n = n;
        q.r0 = row0;
        q.rend = row0 + nrows;
        int64_t ntiles, stride, nstrips;
        spmv_raster(nrows, nd, offs, &ntiles, &stride, &nstrips);
        q.ntiles = ntiles;
        q.stride_tiles = stride;
        q.nstrips = nstrips;
        q.y = (double2 *)y - row0;
        q.nd = (int)nd;
        q.part_bits = part_bits;
        for (int qq = 0; qq < nparts; ++qq) q.parts[qq] = p.parts[qq];
        for (int64_t i = 0; i < nd; ++i) {
            q.dg[i].off = p.off[i];
            q.dg[i].row0 = p.rows[i] - row0;
            q.dg[i].lo = p.lo[i];
            q.dg[i].hi = p.hi[i];
        }
        plan_bands(q);
        if (q.nbands > 0) {
            switch (nd) {
                case 1: return launch_async<1, true>(q, s);
                case 2: return launch_async<2, true>(q, s);
                case 3: return launch_async<3, true>(q, s);
                case 4: return launch_async<4, true>(q, s);
                case 5: return launch_async<5, true>(q, s);
                case 6: return launch_async<6, true>(q, s);
                case 7: return launch_async<7, true>(q, s);
                case 8: return launch_async<8, true>(q, s);
                case 9: return launch_async<9, true>(q, s);
                case 10: return launch_async<10, true>(q, s);
                case 11: return launch_async<11, true>(q, s);
                default: return launch_async<12, true>(q, s);
            }
        }
    }
    const int64_t grid = std::max<int64_t>(1, std::min<int64_t>((nrows + kThreads - 1) / kThreads, (int64_t)sm_count() * 8));
    switch (nd) {
#define DIAQ_SHARD_ND(K) \
    case K: spmv_sharded_kernel<K><<<(unsigned)grid, kThreads, 0, s>>>(p); break;
        DIAQ_SHARD_ND(1) DIAQ_SHARD_ND(2) DIAQ_SHARD_ND(3) DIAQ_SHARD_ND(4) DIAQ_SHARD_ND(5)
        DIAQ_SHARD_ND(6) DIAQ_SHARD_ND(7) DIAQ_SHARD_ND(8) DIAQ_SHARD_ND(9)
#undef DIAQ_SHARD_ND
        default: spmv_sharded_kernel<0><<<(unsigned)grid, kThreads, 0, s>>>(p); break;
    }
    count_launch();
    return check_launch("spmv_sharded_kernel");
}

extern "C" int diaq_spmv(const diaq_matrix_t *a, const void *x, void *y, void *stream) {
    if (!a || !x || !y) return set_error(DIAQ_ERR_VALUE, "diaq_spmv: null argument");
    if (a->n < 1) return set_error(DIAQ_ERR_SHAPE, "diaq_spmv: n_dim must be >= 1");
    SpmvLaunchCache &c = g_spmv_cache;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) {
        cudaGetLastError();
        dev = -1;
    }
    const bool small = a->nd >= 1 && a->nd <= 12;
    if (small && c.valid && c.dev == dev && c.epoch == tuning().epoch && c.vals == a->vals && c.n == a->n &&
        c.nd == a->nd && !memcmp(c.offs, a->offs, sizeof(int64_t) * (size_t)a->nd) &&
        !memcmp(c.starts, a->starts, sizeof(int64_t) * (size_t)a->nd))
        return c.fire(c, x, y, (cudaStream_t)stream);
    c.valid = false;
    c.pending = small;
    const int rc = spmv_rows(a, x, y, 0, a->n, (cudaStream_t)stream);
    c.pending = false;
    if (rc == DIAQ_OK && c.valid) {
        c.dev = dev;
        c.epoch = tuning().epoch;
        c.vals = a->vals;
        c.n = a->n;
        c.nd = a->nd;
        memcpy(c.offs, a->offs, sizeof(int64_t) * (size_t)a->nd);
        memcpy(c.starts, a->starts, sizeof(int64_t) * (size_t)a->nd);
    } else {
        c.valid = false;
    }
    return rc;
}

// Host-buffer spmv with copies and compute overlapped chunk by chunk: x
// chunks go up on one stream, each y chunk is computed as soon as the x
// window it reads (rows [r + d_min, r + d_max]) is resident, and goes down on
// a third stream -- so H2D and D2H share the PCIe link full-duplex instead
// of running back to back.  Synchronous: returns when y_host is complete.
extern "C" int diaq_spmv_host(const diaq_matrix_t *a, const void *x_host, void *y_host, void *x_dev, void *y_dev,
                              int64_t chunk_rows, void *stream) {
    if (!a || !x_host || !y_host || !x_dev || !y_dev) return set_error(DIAQ_ERR_VALUE, "diaq_spmv_host: null argument");
    const int64_t n = a->n;
    if (n < 1) return set_error(DIAQ_ERR_SHAPE, "diaq_spmv_host: n_dim must be >= 1");
    if (chunk_rows <= 0) chunk_rows = (int64_t)1 << 22;
    cudaStream_t s = (cudaStream_t)stream;
    static thread_local cudaStream_t up = nullptr, down = nullptr;
    if (!up && (cudaStreamCreateWithFlags(&up, cudaStreamNonBlocking) != cudaSuccess ||
                cudaStreamCreateWithFlags(&down, cudaStreamNonBlocking) != cudaSuccess))
        return set_error(DIAQ_ERR_CUDA, "diaq_spmv_host: stream create failed");
    int64_t dmin = 0, dmax = 0;
    for (int64_t i = 0; i < a->nd; ++i) {
        dmin = std::min(dmin, a->offs[i]);
        dmax = std::max(dmax, a->offs[i]);
    }
    const int64_t nchunks = (n + chunk_rows - 1) / chunk_rows;
    std::vector<cudaEvent_t> xev((size_t)nchunks), yev((size_t)nchunks);
    for (auto *v : {&xev, &yev})
        for (auto &e : *v)
            if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess)
                return set_error(DIAQ_ERR_CUDA, "diaq_spmv_host: event create failed");
    cudaEvent_t start;
    cudaEventCreateWithFlags(&start, cudaEventDisableTiming);
    cudaEventRecord(start, s);  // x_dev / y_dev may still be in use by earlier work on s
    cudaStreamWaitEvent(up, start, 0);
    cudaStreamWaitEvent(down, start, 0);
    int rc = DIAQ_OK;
    int64_t next_y = 0;
    for (int64_t j = 0; j < nchunks && rc == DIAQ_OK; ++j) {
        const int64_t r = j * chunk_rows, cnt = std::min(chunk_rows, n - r);
        if (cudaMemcpyAsync((double2 *)x_dev + r, (const double2 *)x_host + r, (size_t)cnt * 16,
                            cudaMemcpyHostToDevice, up) != cudaSuccess) {
            rc = set_error(DIAQ_ERR_CUDA, "diaq_spmv_host: H2D failed");
            break;
        }
        cudaEventRecord(xev[(size_t)j], up);
        const int64_t have = r + cnt;  // x rows [0, have) resident
        while (next_y < nchunks) {
            const int64_t yr = next_y * chunk_rows, ycnt = std::min(chunk_rows, n - yr);
            if (std::min(n, yr + ycnt + dmax) > have && have < n) break;
            cudaStreamWaitEvent(s, xev[(size_t)j], 0);
            rc = spmv_rows(a, x_dev, y_dev, yr, ycnt, s);
            if (rc) break;
            cudaEventRecord(yev[(size_t)next_y], s);
            cudaStreamWaitEvent(down, yev[(size_t)next_y], 0);
            if (cudaMemcpyAsync((double2 *)y_host + yr, (const double2 *)y_dev + yr, (size_t)ycnt * 16,
                                cudaMemcpyDeviceToHost, down) != cudaSuccess) {
                rc = set_error(DIAQ_ERR_CUDA, "diaq_spmv_host: D2H failed");
                break;
            }
            ++next_y;
        }
    }
    (void)dmin;
    if (cudaStreamSynchronize(down) != cudaSuccess && rc == DIAQ_OK)
        rc = set_error(DIAQ_ERR_CUDA, "diaq_spmv_host: %s", cudaGetErrorString(cudaGetLastError()));
    cudaStreamSynchronize(s);
    for (auto *v : {&xev, &yev})
        for (auto &e : *v) cudaEventDestroy(e);
    cudaEventDestroy(start);
    return rc;
}
