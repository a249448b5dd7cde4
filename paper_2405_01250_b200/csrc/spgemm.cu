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
                if (i >= pr.lo && i < pr.hi) {
                    const double2 a = ld_reuse(av + pr.a_row0 + i);
                    const double2 b = ld_reuse(bv + pr.b_row0 + i);
                    acc = cadd(acc, cmul_plain(a, b));
                }
            }
            st_stream(cv + cd.c_row0 + cd.row_lo + k, acc);
        }
        const bool big = live && (fabs(acc.x) + fabs(acc.y) > prune_eps);
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
                if (i >= pr.lo && i < pr.hi) {
                    const double2 a = ld_reuse(av + pr.a_row0 + i);
                    const double2 b = ld_reuse(bv + pr.b_row0 + i);
                    acc = cadd(acc, cmul_plain(a, b));
                }
            }
            st_stream(cv + cd.c_row0 + cd.row_lo + k, acc);
        }
        const bool big = live && (fabs(acc.x) + fabs(acc.y) > prune_eps);
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
                           double prune_eps, void *workspace, int64_t workspace_bytes, void *stream) {
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
        spgemm_kernel_param<<<grid, kThreads, 0, s>>>((const double2 *)a->vals, (const double2 *)b->vals,
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
        spgemm_kernel<<<grid, kThreads, 0, s>>>((const double2 *)a->vals, (const double2 *)b->vals,
                                                 (double2 *)c->vals, dcands + base, dpairs, keep_dev + base,
                                                 prune_eps);
        count_launch();
    }
    return check_launch("spgemm_kernel");
}
