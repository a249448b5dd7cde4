// spgemm.cu -- DiaQ x DiaQ product C = A B on sm_100a (reference matrix.py:173-250).
//
// Two passes, as in the north star:
//   pass 1 (host, O(ndA*ndB) integers): the offset union -- every
//     dC = dA + dB with |dC| < n and a non-empty row range [lo, hi)
//     (matrix.py:173-178, 235-240), sorted ascending; and, per candidate,
//     its contributing pairs in ascending dA.  Exclusive scan of candidate
//     lengths lays out C (diaq_layout).
//   pass 2 (device): one thread per output element of every candidate
//     diagonal accumulates its pairs in ascending dA -- the order the
//     reference's `for dA: for dB:` loop produces for each dC -- from +0
//     with the reference rounding (acc += ar*br - ai*bi, each product
//     rounded).  The same kernel raises keep[dC] when any element has
//     |re|+|im| > PRUNE_EPS (matrix.py:246-249); the host drops the
//     others.  Bitwise equal to the reference, structure included.
#include <algorithm>
#include <cmath>
#include <vector>

#include "common.cuh"

namespace diaq {

struct SgPair {
    int64_t lo, hi;       // rows [lo, hi)
    int64_t a_row0;       // A element of row i: avals[a_row0 + i]
    int64_t b_row0;       // B element of row i: bvals[b_row0 + i]
};

struct SgCand {
    int64_t c_row0;       // C element of row i: cvals[c_row0 + i]
    int64_t row_lo, len;  // rows of this diagonal: [row_lo, row_lo + len)
    int32_t pbeg, pend;   // pairs [pbeg, pend)
};

// one output element: its pairs in ascending dA from +0 with the
// reference's rounding -- float64 (numpy float64 ufuncs), or float32 when
// both operands are single precision (matrix.py:231 result_type; the
// values are float32-representable, so the float32 products of the
// reference are reproduced exactly and stored widened)
template <bool SINGLE>
__device__ __forceinline__ double2 pair_term(double2 a, double2 b) {
    if constexpr (SINGLE) {
        const float ar = (float)a.x, ai = (float)a.y, br = (float)b.x, bi = (float)b.y;
        return make_double2((double)__fsub_rn(__fmul_rn(ar, br), __fmul_rn(ai, bi)),
                            (double)__fadd_rn(__fmul_rn(ar, bi), __fmul_rn(ai, br)));
    } else {
        return cmul_plain(a, b);
    }
}

template <bool SINGLE>
__device__ __forceinline__ double2 acc_add(double2 acc, double2 t) {
    if constexpr (SINGLE)
        return make_double2((double)__fadd_rn((float)acc.x, (float)t.x), (double)__fadd_rn((float)acc.y, (float)t.y));
    else
        return cadd(acc, t);
}

template <bool SINGLE>
__device__ __forceinline__ bool above_eps(double2 v, double eps) {
    if constexpr (SINGLE)
        return __fadd_rn(fabsf((float)v.x), fabsf((float)v.y)) > (float)eps;
    else
        return fabs(v.x) + fabs(v.y) > eps;
}

template <bool SINGLE>
__global__ void __launch_bounds__(kThreads)
spgemm_kernel(const double2 *__restrict__ av, const double2 *__restrict__ bv, double2 *cv,
              const SgCand *__restrict__ cands, const SgPair *__restrict__ pairs, uint8_t *keep,
              double prune_eps) {
    const SgCand cd = cands[blockIdx.y];
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t len_round = (cd.len + 31) & ~31ll;  // whole warps iterate together
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < len_round; k += stride) {
        const bool live = k < cd.len;
        double2 acc = make_double2(0.0, 0.0);
        if (live) {
            const int64_t i = cd.row_lo + k;
            for (int q = cd.pbeg; q < cd.pend; ++q) {
                const SgPair pr = pairs[q];
                if (i >= pr.lo && i < pr.hi)
                    acc = acc_add<SINGLE>(acc, pair_term<SINGLE>(ld_reuse(av + pr.a_row0 + i), ld_reuse(bv + pr.b_row0 + i)));
            }
            st_stream(cv + cd.c_row0 + cd.row_lo + k, acc);
        }
        const bool big = live && above_eps<SINGLE>(acc, prune_eps);
        const unsigned any = __ballot_sync(0xffffffffu, big);
        if (any && (threadIdx.x & 31) == 0) keep[blockIdx.y] = 1;
    }
}

// small plans travel in the kernel parameters (no H2D copy, no stream sync)
constexpr int kParamCands = 128;
constexpr int kParamPairs = 512;

struct SgParamPlan {
    SgCand cands[kParamCands];
    SgPair pairs[kParamPairs];
};

template <bool SINGLE>
__global__ void __launch_bounds__(kThreads)
spgemm_kernel_param(const double2 *__restrict__ av, const double2 *__restrict__ bv, double2 *cv,
                    const __grid_constant__ SgParamPlan plan, uint8_t *keep, double prune_eps) {
    const SgCand &cd = plan.cands[blockIdx.y];
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t len_round = (cd.len + 31) & ~31ll;
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < len_round; k += stride) {
        const bool live = k < cd.len;
        double2 acc = make_double2(0.0, 0.0);
        if (live) {
            const int64_t i = cd.row_lo + k;
            for (int q = cd.pbeg; q < cd.pend; ++q) {
                const SgPair &pr = plan.pairs[q];
                if (i >= pr.lo && i < pr.hi)
                    acc = acc_add<SINGLE>(acc, pair_term<SINGLE>(ld_reuse(av + pr.a_row0 + i), ld_reuse(bv + pr.b_row0 + i)));
            }
            st_stream(cv + cd.c_row0 + cd.row_lo + k, acc);
        }
        const bool big = live && above_eps<SINGLE>(acc, prune_eps);
        const unsigned any = __ballot_sync(0xffffffffu, big);
        if (any && (threadIdx.x & 31) == 0) keep[blockIdx.y] = 1;
    }
}

struct Plan {
    std::vector<int64_t> offc;
    std::vector<std::vector<std::pair<int64_t, int64_t>>> pairs;  // (ia, ib) per candidate
};

static void make_plan(int64_t n, int64_t nda, const int64_t *offa, int64_t ndb, const int64_t *offb,
                      Plan &pl) {
    std::vector<int64_t> c;
    c.reserve((size_t)(nda * ndb));
    for (int64_t ia = 0; ia < nda; ++ia)
        for (int64_t ib = 0; ib < ndb; ++ib) {
            const int64_t da = offa[ia], db = offb[ib], dc = da + db;
            if (dc >= n || -dc >= n) continue;
            const int64_t lo = std::max<int64_t>(0, std::max(-da, -dc));
            const int64_t hi = std::min<int64_t>(n, std::min(n - da, n - dc));
            if (lo >= hi) continue;
            c.push_back(dc);
        }
    std::sort(c.begin(), c.end());
    c.erase(std::unique(c.begin(), c.end()), c.end());
    pl.offc = c;
    pl.pairs.assign(c.size(), {});
    for (int64_t ia = 0; ia < nda; ++ia)
        for (int64_t ib = 0; ib < ndb; ++ib) {
            const int64_t da = offa[ia], db = offb[ib], dc = da + db;
            if (dc >= n || -dc >= n) continue;
            const int64_t lo = std::max<int64_t>(0, std::max(-da, -dc));
            const int64_t hi = std::min<int64_t>(n, std::min(n - da, n - dc));
            if (lo >= hi) continue;
            const size_t ic = (size_t)(std::lower_bound(c.begin(), c.end(), dc) - c.begin());
            pl.pairs[ic].push_back({ia, ib});  // ia ascending by construction
        }
}

}  // namespace diaq

using namespace diaq;

extern "C" int diaq_spgemm_plan(int64_t n, int64_t nda, const int64_t *offa, int64_t ndb, const int64_t *offb,
                                int64_t *offc, int64_t *nc) {
    if (!nc || (nda && !offa) || (ndb && !offb)) return set_error(DIAQ_ERR_VALUE, "diaq_spgemm_plan: null argument");
    Plan pl;
    make_plan(n, nda, offa, ndb, offb, pl);
    for (size_t i = 0; i < pl.offc.size(); ++i) offc[i] = pl.offc[i];
    *nc = (int64_t)pl.offc.size();
    return DIAQ_OK;
}

extern "C" int64_t diaq_spgemm_workspace(int64_t nda, int64_t ndb, int64_t nc) {
    return (int64_t)(sizeof(SgPair) * (size_t)(nda * ndb) + sizeof(SgCand) * (size_t)nc + 256);
}

extern "C" int diaq_spgemm(const diaq_matrix_t *a, const diaq_matrix_t *b, diaq_matrix_t *c, uint8_t *keep_dev,
                           double prune_eps, int single, void *workspace, int64_t workspace_bytes, void *stream) {
    if (!a || !b || !c || !keep_dev) return set_error(DIAQ_ERR_VALUE, "diaq_spgemm: null argument");
    if (a->n != b->n)
        return set_error(DIAQ_ERR_SHAPE, "not multiplyable: %lldx%lld by %lldx%lld", (long long)a->n,
                         (long long)a->n, (long long)b->n, (long long)b->n);
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t n = a->n;
    Plan pl;
    make_plan(n, a->nd, a->offs, b->nd, b->offs, pl);
    if ((int64_t)pl.offc.size() != c->nd || c->n != n)
        return set_error(DIAQ_ERR_SHAPE, "diaq_spgemm: output layout does not match the plan");
    for (int64_t i = 0; i < c->nd; ++i)
        if (c->offs[i] != pl.offc[i]) return set_error(DIAQ_ERR_SHAPE, "diaq_spgemm: output offsets mismatch");
    if (c->nd == 0) return DIAQ_OK;
    std::vector<SgPair> hp;
    std::vector<SgCand> hc(pl.offc.size());
    int64_t maxlen = 0;
    for (size_t ic = 0; ic < pl.offc.size(); ++ic) {
        const int64_t dc = pl.offc[ic];
        SgCand &cd = hc[ic];
        cd.row_lo = dc < 0 ? -dc : 0;
        cd.len = n - (dc < 0 ? -dc : dc);
        cd.c_row0 = c->starts[ic] + (dc < 0 ? dc : 0);
        cd.pbeg = (int32_t)hp.size();
        for (auto &pr : pl.pairs[ic]) {
            const int64_t da = a->offs[pr.first], db = b->offs[pr.second];
            SgPair q;
            q.lo = std::max<int64_t>(0, std::max(-da, -dc));
            q.hi = std::min<int64_t>(n, std::min(n - da, n - dc));
            q.a_row0 = a->starts[pr.first] + (da < 0 ? da : 0);
            q.b_row0 = b->starts[pr.second] + da + (db < 0 ? db : 0);
            hp.push_back(q);
        }
        cd.pend = (int32_t)hp.size();
        maxlen = std::max(maxlen, cd.len);
    }
    const int sms = sm_count();
    if (cudaMemsetAsync(keep_dev, 0, (size_t)c->nd, s) != cudaSuccess)
        return set_error(DIAQ_ERR_CUDA, "diaq_spgemm: memset failed");
    const int64_t want = (maxlen + kThreads - 1) / kThreads;
    const int64_t cap = std::max<int64_t>(1, (int64_t)sms * 8 / (int64_t)hc.size());
    if ((int)hc.size() <= kParamCands && (int)hp.size() <= kParamPairs) {
        static thread_local SgParamPlan pp;  // host staging of the by-value kernel argument
        std::copy(hc.begin(), hc.end(), pp.cands);
        std::copy(hp.begin(), hp.end(), pp.pairs);
        dim3 grid((unsigned)std::max<int64_t>(1, std::min(want, cap)), (unsigned)hc.size());
        if (single)
            spgemm_kernel_param<true><<<grid, kThreads, 0, s>>>((const double2 *)a->vals, (const double2 *)b->vals,
                                                                 (double2 *)c->vals, pp, keep_dev, prune_eps);
        else
            spgemm_kernel_param<false><<<grid, kThreads, 0, s>>>((const double2 *)a->vals, (const double2 *)b->vals,
                                                                  (double2 *)c->vals, pp, keep_dev, prune_eps);
        count_launch();
        return check_launch("spgemm_kernel_param");
    }
    const size_t need = sizeof(SgPair) * hp.size() + sizeof(SgCand) * hc.size();
    if (!workspace || workspace_bytes < (int64_t)need)
        return set_error(DIAQ_ERR_VALUE, "diaq_spgemm: workspace too small (%zu bytes needed)", need);
    SgCand *dcands = (SgCand *)workspace;
    SgPair *dpairs = (SgPair *)((char *)workspace + sizeof(SgCand) * hc.size());
    // pageable H2D copies stage the host tables before returning
    if (cudaMemcpyAsync(dcands, hc.data(), sizeof(SgCand) * hc.size(), cudaMemcpyHostToDevice, s) != cudaSuccess ||
        cudaMemcpyAsync(dpairs, hp.data(), sizeof(SgPair) * hp.size(), cudaMemcpyHostToDevice, s) != cudaSuccess)
        return set_error(DIAQ_ERR_CUDA, "diaq_spgemm: plan upload failed");
    for (int64_t base = 0; base < (int64_t)hc.size(); base += 65535) {
        const int cnt = (int)std::min<int64_t>(65535, (int64_t)hc.size() - base);
        dim3 grid((unsigned)std::max<int64_t>(1, std::min(want, cap)), cnt);
        if (single)
            spgemm_kernel<true><<<grid, kThreads, 0, s>>>((const double2 *)a->vals, (const double2 *)b->vals,
                                                           (double2 *)c->vals, dcands + base, dpairs, keep_dev + base,
                                                           prune_eps);
        else
            spgemm_kernel<false><<<grid, kThreads, 0, s>>>((const double2 *)a->vals, (const double2 *)b->vals,
                                                            (double2 *)c->vals, dcands + base, dpairs, keep_dev + base,
                                                            prune_eps);
        count_launch();
    }
    return check_launch("spgemm_kernel");
}

// ---- device pass 1: offset union, count and scan on the device -------------
//
// North-star form of the product (and its batched sweep): the structure of
// C is computed by a kernel from the device offset tables of A and B, so a
// product of device-resident matrices -- including a product of products --
// never waits for the host.  One CTA per product:
//   count: every pair (ia, ib) with |dC| < n and a non-empty row range;
//   union: a pair leads its dC if no earlier valid pair has the same dC;
//          candidate index = number of leading dC below it (ascending);
//   scan:  pair slot = valid pairs with smaller dC + earlier pairs with the
//          same dC (ascending dA within a candidate, as the reference's
//          `for dA: for dB:` loop accumulates); the candidates are laid out
//          by the diaq_layout rule (row-aligned starts).
// pass 2 is the same per-element multiply (one CTA row per candidate slot),
// and a compaction kernel writes the kept diagonals' offsets/starts (prune,
// matrix.py:246-249) into C's device table -- nothing is read back.

namespace diaq {

constexpr int kDevPlanMax = 1024;  // pairs per product planned on the device
constexpr int kDevBatch = 64;      // products per launch (kernel-parameter tables)

struct WsHdr {
    int64_t nc, total, err, pad;
};

__host__ __device__ inline size_t ws_stride_bytes(int64_t pair_cap) {
    const size_t b = sizeof(WsHdr) + (size_t)pair_cap * (sizeof(SgCand) + sizeof(SgPair) + 2 * sizeof(int64_t) + 1);
    return (b + 255) & ~(size_t)255;
}

struct DevBatch {
    int count;
    int single;
    int64_t pair_cap;
    double prune_eps;
    char *ws;
    diaq_dev_matrix_t a[kDevBatch];
    diaq_dev_matrix_t b[kDevBatch];
    diaq_dev_result_t c[kDevBatch];
};

struct WsView {
    WsHdr *hdr;
    SgCand *cand;
    SgPair *pair;
    int64_t *offc, *startc;
    uint8_t *keep;
};

__device__ __forceinline__ WsView ws_view(char *base, int64_t pair_cap) {
    WsView v;
    v.hdr = (WsHdr *)base;
    v.cand = (SgCand *)(base + sizeof(WsHdr));
    v.pair = (SgPair *)(v.cand + pair_cap);
    v.offc = (int64_t *)(v.pair + pair_cap);
    v.startc = v.offc + pair_cap;
    v.keep = (uint8_t *)(v.startc + pair_cap);
    return v;
}

__global__ void __launch_bounds__(kThreads) spgemm_plan_kernel(const __grid_constant__ DevBatch bp) {
    const int j = blockIdx.x;
    const diaq_dev_matrix_t &A = bp.a[j];
    const diaq_dev_matrix_t &B = bp.b[j];
    const WsView w = ws_view(bp.ws + (size_t)j * ws_stride_bytes(bp.pair_cap), bp.pair_cap);
    __shared__ int64_t sdc[kDevPlanMax];
    __shared__ uint8_t sok[kDevPlanMax], slead[kDevPlanMax];
    __shared__ int s_nc;
    const int64_t n = A.n;
    const int nda = (int)*A.nd, ndb = (int)*B.nd;
    const int P = nda * ndb;
    if (P > bp.pair_cap || P > kDevPlanMax || B.n != n) {
        if (threadIdx.x == 0) {
            w.hdr->err = 1;
            w.hdr->nc = 0;
        }
        return;
    }
    for (int p = threadIdx.x; p < P; p += blockDim.x) {
        const int64_t da = A.offs[p / ndb], db = B.offs[p % ndb], dc = da + db;
        const int64_t lo = max((int64_t)0, max(-da, -dc)), hi = min(n, min(n - da, n - dc));
        sdc[p] = dc;
        sok[p] = (dc < n && -dc < n && lo < hi) ? 1 : 0;
    }
    if (threadIdx.x == 0) s_nc = 0;
    __syncthreads();
    for (int p = threadIdx.x; p < P; p += blockDim.x) {
        bool lead = sok[p];
        for (int q = 0; q < p && lead; ++q) lead = !(sok[q] && sdc[q] == sdc[p]);
        slead[p] = lead ? 1 : 0;
        if (lead) atomicAdd(&s_nc, 1);
    }
    __syncthreads();
    for (int p = threadIdx.x; p < P; p += blockDim.x) {
        if (!sok[p]) continue;
        const int64_t dc = sdc[p];
        int less = 0, before = 0, same = 0, cidx = 0;
        for (int q = 0; q < P; ++q) {
            if (!sok[q]) continue;
            less += sdc[q] < dc;
            same += sdc[q] == dc;
            before += (sdc[q] == dc) & (q < p);
            cidx += slead[q] & (sdc[q] < dc);
        }
        const int ia = p / ndb, ib = p % ndb;
        const int64_t da = A.offs[ia], db = B.offs[ib];
        SgPair pr;
        pr.lo = max((int64_t)0, max(-da, -dc));
        pr.hi = min(n, min(n - da, n - dc));
        pr.a_row0 = A.starts[ia] + (da < 0 ? da : 0);
        pr.b_row0 = B.starts[ib] + da + (db < 0 ? db : 0);
        w.pair[less + before] = pr;
        if (slead[p]) {
            w.cand[cidx].pbeg = less;
            w.cand[cidx].pend = less + same;
            w.offc[cidx] = dc;
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {  // layout scan (diaq_layout rule), sequential over the candidates
        const int nc = s_nc;
        int64_t cur = 0;
        for (int c = 0; c < nc; ++c) {
            const int64_t d = w.offc[c];
            const int64_t want = (d < 0 ? -d : 0) & 7;
            const int64_t st = cur + ((want - (cur & 7)) & 7);
            const int64_t len = n - (d < 0 ? -d : d);
            w.startc[c] = st;
            w.cand[c].c_row0 = st + (d < 0 ? d : 0);
            w.cand[c].row_lo = d < 0 ? -d : 0;
            w.cand[c].len = len;
            w.keep[c] = 0;
            cur = st + len;
        }
        w.hdr->nc = nc;
        w.hdr->total = (cur + 7) & ~7ll;
        w.hdr->err = w.hdr->total > bp.c[j].capacity || nc > bp.c[j].nd_cap ? 2 : 0;
    }
}

template <bool SINGLE>
__global__ void __launch_bounds__(kThreads) spgemm_dev_kernel(const __grid_constant__ DevBatch bp) {
    const int j = blockIdx.z;
    const WsView w = ws_view(bp.ws + (size_t)j * ws_stride_bytes(bp.pair_cap), bp.pair_cap);
    const int64_t c_i = blockIdx.y;
    if (w.hdr->err || c_i >= w.hdr->nc) return;
    const double2 *av = (const double2 *)bp.a[j].vals, *bv = (const double2 *)bp.b[j].vals;
    double2 *cv = (double2 *)bp.c[j].vals;
    const SgCand cd = w.cand[c_i];
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t len_round = (cd.len + 31) & ~31ll;
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < len_round; k += stride) {
        const bool live = k < cd.len;
        double2 acc = make_double2(0.0, 0.0);
        if (live) {
            const int64_t i = cd.row_lo + k;
            for (int q = cd.pbeg; q < cd.pend; ++q) {
                const SgPair pr = w.pair[q];
                if (i >= pr.lo && i < pr.hi)
                    acc = acc_add<SINGLE>(acc, pair_term<SINGLE>(ld_reuse(av + pr.a_row0 + i), ld_reuse(bv + pr.b_row0 + i)));
            }
            st_stream(cv + cd.c_row0 + cd.row_lo + k, acc);
        }
        const bool big = live && above_eps<SINGLE>(acc, bp.prune_eps);
        const unsigned any = __ballot_sync(0xffffffffu, big);
        if (any && (threadIdx.x & 31) == 0) w.keep[c_i] = 1;
    }
}

// kept candidates, ascending, into C's device table; nd = -err on failure
__global__ void spgemm_compact_kernel(const __grid_constant__ DevBatch bp) {
    const int j = blockIdx.x;
    const WsView w = ws_view(bp.ws + (size_t)j * ws_stride_bytes(bp.pair_cap), bp.pair_cap);
    if (threadIdx.x != 0) return;
    const diaq_dev_result_t &C = bp.c[j];
    if (w.hdr->err) {
        *C.nd = -w.hdr->err;
        return;
    }
    int64_t k = 0;
    for (int64_t c = 0; c < w.hdr->nc; ++c)
        if (w.keep[c]) {
            C.offs[k] = w.offc[c];
            C.starts[k] = w.startc[c];
            ++k;
        }
    *C.nd = k;
}

// host-planned product: compact its keep flags into a device table the same way
__global__ void keep_compact_kernel(int64_t nc, const int64_t *cand_tab, const uint8_t *keep, int64_t *nd, int64_t *offs,
                                    int64_t *starts) {
    if (blockIdx.x != 0 || threadIdx.x != 0) return;
    int64_t k = 0;
    for (int64_t c = 0; c < nc; ++c)
        if (keep[c]) {
            offs[k] = cand_tab[c];
            starts[k] = cand_tab[nc + c];
            ++k;
        }
    *nd = k;
}

}  // namespace diaq (device plan)

extern "C" int64_t diaq_spgemm_dev_workspace(int count, int64_t pair_cap) {
    if (count < 1 || pair_cap < 1) return 0;
    return (int64_t)(ws_stride_bytes(pair_cap) * (size_t)count);
}

extern "C" int diaq_spgemm_dev(int count, const diaq_dev_matrix_t *a, const diaq_dev_matrix_t *b,
                               const diaq_dev_result_t *c, double prune_eps, int single, int64_t pair_cap,
                               void *workspace, int64_t workspace_bytes, void *stream) {
    if (count < 0 || (count && (!a || !b || !c || !workspace)))
        return set_error(DIAQ_ERR_VALUE, "diaq_spgemm_dev: bad arguments");
    if (pair_cap < 1 || pair_cap > kDevPlanMax)
        return set_error(DIAQ_ERR_VALUE, "diaq_spgemm_dev: pair capacity %lld outside 1..%d", (long long)pair_cap,
                         kDevPlanMax);
    if (workspace_bytes < diaq_spgemm_dev_workspace(count, pair_cap))
        return set_error(DIAQ_ERR_VALUE, "diaq_spgemm_dev: workspace too small");
    cudaStream_t s = (cudaStream_t)stream;
    static thread_local DevBatch bp;
    int64_t maxlen = 1;
    for (int base = 0; base < count; base += kDevBatch) {
        const int cnt = std::min(kDevBatch, count - base);
        bp.count = cnt;
        bp.single = single;
        bp.pair_cap = pair_cap;
        bp.prune_eps = prune_eps;
        bp.ws = (char *)workspace + ws_stride_bytes(pair_cap) * (size_t)base;
        for (int j = 0; j < cnt; ++j) {
            bp.a[j] = a[base + j];
            bp.b[j] = b[base + j];
            bp.c[j] = c[base + j];
            if (a[base + j].n != b[base + j].n)
                return set_error(DIAQ_ERR_SHAPE, "not multiplyable: %lldx%lld by %lldx%lld", (long long)a[base + j].n,
                                 (long long)a[base + j].n, (long long)b[base + j].n, (long long)b[base + j].n);
            maxlen = std::max(maxlen, a[base + j].n);
        }
        spgemm_plan_kernel<<<cnt, kThreads, 0, s>>>(bp);
        count_launch();
        const int64_t want = (maxlen + kThreads - 1) / kThreads;
        const int64_t cap = std::max<int64_t>(1, (int64_t)sm_count() * 8 / std::max<int64_t>(1, pair_cap * cnt));
        const dim3 grid((unsigned)std::max<int64_t>(1, std::min(want, cap)), (unsigned)pair_cap, (unsigned)cnt);
        if (single) spgemm_dev_kernel<true><<<grid, kThreads, 0, s>>>(bp);
        else spgemm_dev_kernel<false><<<grid, kThreads, 0, s>>>(bp);
        count_launch();
        spgemm_compact_kernel<<<cnt, 32, 0, s>>>(bp);
        count_launch();
        const int rc = check_launch("spgemm_dev");
        if (rc) return rc;
    }
    return DIAQ_OK;
}

extern "C" int diaq_spgemm_compact(int64_t nc, const int64_t *cand_tab_dev, const uint8_t *keep_dev, int64_t *nd_dev,
                                   int64_t *offs_dev, int64_t *starts_dev, void *stream) {
    if (nc < 0 || !nd_dev || (nc && (!cand_tab_dev || !keep_dev || !offs_dev || !starts_dev)))
        return set_error(DIAQ_ERR_VALUE, "diaq_spgemm_compact: bad arguments");
    keep_compact_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(nc, cand_tab_dev, keep_dev, nd_dev, offs_dev, starts_dev);
    count_launch();
    return check_launch("keep_compact_kernel");
}
