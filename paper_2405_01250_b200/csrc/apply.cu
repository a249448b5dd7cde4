// apply.cu -- gate application on sm_100a (reference sim.py:53-105, 167-200).
//
// Two kernels:
//
// 1. gate_kernel<K>: the Kronecker-structured (compact) form.  A k-qubit
//    gate g on state bits s_0..s_{k-1} acts on disjoint groups of 2^k
//    amplitudes that differ only in those bits; each thread loads its group
//    once, multiplies by g and stores it (in place is legal: groups are
//    disjoint).  HBM traffic is the algorithmic 32 B per amplitude (x read +
//    y written) -- the reference instead walks 2^span-long stored diagonals
//    of the build_span_unitary embedding (gates.py:169-219).
//    Parity: for output row rg the reference (sim.py:69-78) adds the terms of
//    its stored diagonals in ascending offset d = embed(cg) - embed(rg),
//    i.e. in ascending embed(cg).  The host relabels the operands by
//    descending bit shift so that ascending relabelled column index IS
//    ascending embed(cg); the kernel then sums columns in natural order,
//    with numpy's complex multiply rounding (DIAQ_CMUL_*) and sequential
//    complex adds from +0 -- bitwise equal to the reference except for the
//    sign of exact zeros (exactly-zero gate entries, which the reference
//    stores as explicit zeros, are skipped).
//
// 2. placed_kernel: any Placement(dim_a, m, dim_b) over the stored
//    diagonals of m (reference _apply_diags_block, sim.py:69-78), one thread
//    per output amplitude, ascending d.  Used for user-built placements.
#include <algorithm>
#include <cstring>
#include <vector>

#include "common.cuh"

namespace diaq {

constexpr int kMaxGateK = 5;

template <int K>
struct GateParams {
    const double2 *x;
    double2 *y;
    int64_t ngroups;
    int sh_sorted[K > 0 ? K : 1];   // ascending bit shifts (zero-bit insertion)
    int64_t emb[1 << K];            // state offset of relabelled gate index c
    uint32_t nzmask[1 << K];        // bit c set iff g'[r][c] != 0
    double2 g[1 << K][1 << K];      // relabelled gate, row-major
};

template <int K, int MODE>
__global__ void __launch_bounds__(kThreads) gate_kernel(const __grid_constant__ GateParams<K> p) {
    constexpr int M = 1 << K;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t gi = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; gi < p.ngroups; gi += stride) {
        const uint64_t base = insert_zero_bits<K>((uint64_t)gi, p.sh_sorted);
        double2 xs[M];
#pragma unroll
        for (int c = 0; c < M; ++c) xs[c] = ld_plain(p.x + base + p.emb[c]);
#pragma unroll
        for (int r = 0; r < M; ++r) {
            double2 acc = make_double2(0.0, 0.0);
            const uint32_t nz = p.nzmask[r];
#pragma unroll
            for (int c = 0; c < M; ++c)
                if ((nz >> c) & 1u) acc = cadd(acc, cmul<MODE>(p.g[r][c], xs[c]));
            st_plain(p.y + base + p.emb[r], acc);
        }
    }
}

// ---- sharded state: multi-source gate kernel ---------------
// The state is split over its top log2(P) bits.  A gate's operands split
// into KL local bits and KG global (rank) bits.  After relabelling by
// descending shift the global operands are the top KG bits of the gate
// index, so for this rank only the 2^KL rows of block `vr` (its own global
// bit values) are produced, and column block v (global operand values v) is
// read from src[v]: this rank's shard for v == vr, a received partner shard
// otherwise.  Ascending relabelled column = ascending embedding in the full
// index, so per-amplitude summation order equals the single-GPU kernel's and
// the reference's.
template <int KL, int KG>
struct MultiParams {
    double2 *y;
    int64_t ngroups;
    int sh_sorted[KL > 0 ? KL : 1];
    int64_t emb[1 << KL];
    const double2 *src[1 << KG];
    uint32_t srcmask;
    uint32_t nzmask[1 << KL];
    double2 g[1 << KL][1 << (KL + KG)];
};

template <int KL, int KG, int MODE>
__global__ void __launch_bounds__(kThreads) gate_kernel_multi(const __grid_constant__ MultiParams<KL, KG> p) {
    constexpr int ML = 1 << KL;
    constexpr int MG = 1 << KG;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t gi = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; gi < p.ngroups; gi += stride) {
        const uint64_t base = insert_zero_bits<KL>((uint64_t)gi, p.sh_sorted);
        double2 xs[MG][ML];
#pragma unroll
        for (int v = 0; v < MG; ++v)
#pragma unroll
            for (int c = 0; c < ML; ++c)
                xs[v][c] = ((p.srcmask >> v) & 1u) ? ld_plain(p.src[v] + base + p.emb[c]) : make_double2(0.0, 0.0);
#pragma unroll
        for (int r = 0; r < ML; ++r) {
            double2 acc = make_double2(0.0, 0.0);
            const uint32_t nz = p.nzmask[r];
#pragma unroll
            for (int v = 0; v < MG; ++v)
#pragma unroll
                for (int c = 0; c < ML; ++c)
                    if ((nz >> (v * ML + c)) & 1u) acc = cadd(acc, cmul<MODE>(p.g[r][v * ML + c], xs[v][c]));
            st_plain(p.y + base + p.emb[r], acc);
        }
    }
}

struct PlacedDiag {
    const double2 *row0;  // m value for span row `row` is row0[row]
    int64_t lo, hi;       // valid span rows
    int64_t xoff;         // d * dim_b
};

struct PlacedParams {
    int64_t total, dim_b, n_m;
    const double2 *x;
    double2 *y;
    int nd;
    int accumulate;  // continue the sum already in y (a later chunk of > 64 diagonals)
    PlacedDiag dg[kParamDiags];
};

template <int MODE>
__global__ void __launch_bounds__(kThreads) placed_kernel(const __grid_constant__ PlacedParams p) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < p.total; e += stride) {
        const int64_t row = (e / p.dim_b) % p.n_m;
        double2 acc = p.accumulate ? ld_plain(p.y + e) : make_double2(0.0, 0.0);
        for (int i = 0; i < p.nd; ++i) {
            if (row >= p.dg[i].lo && row < p.dg[i].hi) {
                const double2 v = ld_reuse(p.dg[i].row0 + row);
                const double2 xv = ld_reuse(p.x + e + p.dg[i].xoff);
                acc = cadd(acc, cmul<MODE>(v, xv));
            }
        }
        st_stream(p.y + e, acc);
    }
}

__global__ void init_basis_kernel(double2 *x, int64_t n, int64_t index) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
        x[i] = make_double2(i == index ? 1.0 : 0.0, 0.0);
}

constexpr int kNormBlocks = 1024;

__global__ void __launch_bounds__(kThreads) norm2_partial(const double2 *x, int64_t n, double *part) {
    double s = 0.0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        const double2 v = ld_reuse(x + i);
        s = __fma_rn(v.x, v.x, s);
        s = __fma_rn(v.y, v.y, s);
    }
    __shared__ double red[kThreads / 32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x < 32) {
        s = threadIdx.x < kThreads / 32 ? red[threadIdx.x] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
        if (threadIdx.x == 0) part[blockIdx.x] = s;
    }
}

__global__ void norm2_final(const double *part, int nparts, double *out) {
    __shared__ double red[32];
    double s = 0.0;
    for (int i = threadIdx.x; i < nparts; i += blockDim.x) s += part[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x < 32) {
        s = threadIdx.x < (int)(blockDim.x / 32) ? red[threadIdx.x] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
        if (threadIdx.x == 0) out[0] = s;
    }
}

// Relabel a k-qubit gate so operand order follows descending state-bit
// shift (see file comment) and pack it for gate_kernel.
template <int K>
static int build_gate_params(GateParams<K> &p, int n_bits, const double *g, const int *shifts) {
    constexpr int M = 1 << K;
    int perm[kMaxGateK];  // perm[j] = original operand placed at relabelled position j
    for (int i = 0; i < K; ++i) perm[i] = i;
    std::sort(perm, perm + K, [&](int a, int b) { return shifts[a] > shifts[b]; });
    for (int i = 0; i < K; ++i) {
        if (shifts[i] < 0 || shifts[i] >= n_bits)
            return set_error(DIAQ_ERR_SHAPE, "gate shift %d outside state of %d qubits", shifts[i], n_bits);
        for (int j = 0; j < i; ++j)
            if (shifts[j] == shifts[i]) return set_error(DIAQ_ERR_SHAPE, "repeated gate bit %d", shifts[i]);
    }
    // relabelled index c' -> original gate index c (operand i is bit K-1-i)
    int orig[M];
    for (int cp = 0; cp < M; ++cp) {
        int c = 0;
        for (int j = 0; j < K; ++j) {
            const int bit = (cp >> (K - 1 - j)) & 1;
            c |= bit << (K - 1 - perm[j]);
        }
        orig[cp] = c;
    }
    for (int cp = 0; cp < M; ++cp) {
        int64_t e = 0;
        for (int j = 0; j < K; ++j) e |= (int64_t)((cp >> (K - 1 - j)) & 1) << shifts[perm[j]];
        p.emb[cp] = e;
    }
    for (int rp = 0; rp < M; ++rp) {
        uint32_t nz = 0;
        for (int cp = 0; cp < M; ++cp) {
            const double re = g[2 * (orig[rp] * M + orig[cp])];
            const double im = g[2 * (orig[rp] * M + orig[cp]) + 1];
            p.g[rp][cp] = make_double2(re, im);
            if (re != 0.0 || im != 0.0) nz |= 1u << cp;
        }
        p.nzmask[rp] = nz;
    }
    int s[kMaxGateK];
    for (int i = 0; i < K; ++i) s[i] = shifts[i];
    std::sort(s, s + K);
    for (int i = 0; i < K; ++i) p.sh_sorted[i] = s[i];
    p.ngroups = (int64_t)1 << (n_bits - K);
    return DIAQ_OK;
}

template <int K>
static int launch_gate(int n_bits, const double *g, const int *shifts, const void *x, void *y,
                       int cmul_mode, cudaStream_t s) {
    GateParams<K> p;
    int rc = build_gate_params<K>(p, n_bits, g, shifts);
    if (rc) return rc;
    p.x = (const double2 *)x;
    p.y = (double2 *)y;
    const int64_t want = (p.ngroups + kThreads - 1) / kThreads;
    const int grid = (int)std::max<int64_t>(
        1, std::min<int64_t>(want, (int64_t)sm_count() * tuning().gate_ctas_per_sm));
    if (cmul_mode != DIAQ_CMUL_PLAIN) gate_kernel<K, DIAQ_CMUL_FMA><<<grid, kThreads, 0, s>>>(p);
    else gate_kernel<K, DIAQ_CMUL_PLAIN><<<grid, kThreads, 0, s>>>(p);
    count_launch();
    return check_launch("gate_kernel");
}

int apply_gate(int n_bits, int k, const double *g, const int *shifts, const void *x, void *y,
               int cmul_mode, cudaStream_t s) {
    if (k < 1 || k > kMaxGateK) return set_error(DIAQ_ERR_UNSUPPORTED, "gate width %d outside 1..5", k);
    if (n_bits < k || n_bits > 62) return set_error(DIAQ_ERR_SHAPE, "state of %d bits too small for %d-qubit gate", n_bits, k);
    switch (k) {
        case 1: return launch_gate<1>(n_bits, g, shifts, x, y, cmul_mode, s);
        case 2: return launch_gate<2>(n_bits, g, shifts, x, y, cmul_mode, s);
        case 3: return launch_gate<3>(n_bits, g, shifts, x, y, cmul_mode, s);
        case 4: return launch_gate<4>(n_bits, g, shifts, x, y, cmul_mode, s);
        default: return launch_gate<5>(n_bits, g, shifts, x, y, cmul_mode, s);
    }
}


// Relabelled view of a gate for a sharded state: operands sorted by
// descending global shift (global operands first).  For rank `rank` returns
// the block value vr of its global operand bits and the mask of column blocks
// its rows read (nonzero entries).
struct ShardView {
    int k, kl, kg;
    int perm[kMaxGateK];     // relabelled position j -> original operand
    int shift[kMaxGateK];    // shift of relabelled operand j (descending)
    int orig[32];            // relabelled index -> original gate index
    uint32_t vr;             // this rank's global-operand block value
    uint32_t need;           // column blocks read by this rank's rows
};

static int shard_view(int n_bits, int local_bits, int k, const double *g, const int *shifts, int64_t rank,
                      ShardView &v) {
    if (k < 1 || k > kMaxGateK) return set_error(DIAQ_ERR_UNSUPPORTED, "gate width %d outside 1..5", k);
    if (local_bits < 1 || local_bits > n_bits) return set_error(DIAQ_ERR_SHAPE, "local_bits %d invalid", local_bits);
    for (int i = 0; i < k; ++i) {
        if (shifts[i] < 0 || shifts[i] >= n_bits)
            return set_error(DIAQ_ERR_SHAPE, "gate shift %d outside state of %d qubits", shifts[i], n_bits);
        for (int j = 0; j < i; ++j)
            if (shifts[j] == shifts[i]) return set_error(DIAQ_ERR_SHAPE, "repeated gate bit %d", shifts[i]);
    }
    v.k = k;
    for (int i = 0; i < k; ++i) v.perm[i] = i;
    std::sort(v.perm, v.perm + k, [&](int a, int b) { return shifts[a] > shifts[b]; });
    v.kg = 0;
    for (int j = 0; j < k; ++j) {
        v.shift[j] = shifts[v.perm[j]];
        if (v.shift[j] >= local_bits) ++v.kg;
    }
    v.kl = k - v.kg;
    const int M = 1 << k;
    for (int cp = 0; cp < M; ++cp) {
        int c = 0;
        for (int j = 0; j < k; ++j) c |= ((cp >> (k - 1 - j)) & 1) << (k - 1 - v.perm[j]);
        v.orig[cp] = c;
    }
    v.vr = 0;
    for (int j = 0; j < v.kg; ++j) v.vr |= (uint32_t)((rank >> (v.shift[j] - local_bits)) & 1) << (v.kg - 1 - j);
    v.need = 0;
    const int ML = 1 << v.kl;
    for (int rl = 0; rl < ML; ++rl) {
        const int rp = ((int)v.vr << v.kl) | rl;
        for (int cp = 0; cp < M; ++cp) {
            const double re = g[2 * (v.orig[rp] * M + v.orig[cp])], im = g[2 * (v.orig[rp] * M + v.orig[cp]) + 1];
            if (re != 0.0 || im != 0.0) v.need |= 1u << (cp >> v.kl);
        }
    }
    return DIAQ_OK;
}

template <int KL, int KG>
static int launch_multi(const ShardView &v, int local_bits, const double *g, const void *const *srcs, void *y,
                        int cmul_mode, cudaStream_t s) {
    constexpr int ML = 1 << KL;
    constexpr int M = 1 << (KL + KG);
    MultiParams<KL, KG> p;
    p.y = (double2 *)y;
    p.ngroups = (int64_t)1 << (local_bits - KL);
    int sl[kMaxGateK];
    for (int j = 0; j < KL; ++j) sl[j] = v.shift[KG + j];
    std::sort(sl, sl + KL);
    for (int j = 0; j < KL; ++j) p.sh_sorted[j] = sl[j];
    if (KL == 0) p.sh_sorted[0] = 0;
    for (int cl = 0; cl < ML; ++cl) {
        int64_t e = 0;
        for (int j = 0; j < KL; ++j) e |= (int64_t)((cl >> (KL - 1 - j)) & 1) << v.shift[KG + j];
        p.emb[cl] = e;
    }
    p.srcmask = v.need;
    for (int b = 0; b < (1 << KG); ++b) {
        p.src[b] = (const double2 *)srcs[b];
        if (((v.need >> b) & 1u) && !srcs[b])
            return set_error(DIAQ_ERR_VALUE, "sharded gate: source block %d is needed but missing", b);
    }
    for (int rl = 0; rl < ML; ++rl) {
        const int rp = ((int)v.vr << KL) | rl;
        uint32_t nz = 0;
        for (int cp = 0; cp < M; ++cp) {
            const double re = g[2 * (v.orig[rp] * M + v.orig[cp])], im = g[2 * (v.orig[rp] * M + v.orig[cp]) + 1];
            p.g[rl][cp] = make_double2(re, im);
            if (re != 0.0 || im != 0.0) nz |= 1u << cp;
        }
        p.nzmask[rl] = nz;
    }
    const int64_t want = (p.ngroups + kThreads - 1) / kThreads;
    const int grid = (int)std::max<int64_t>(
        1, std::min<int64_t>(want, (int64_t)sm_count() * tuning().gate_ctas_per_sm));
    if (cmul_mode != DIAQ_CMUL_PLAIN) gate_kernel_multi<KL, KG, DIAQ_CMUL_FMA><<<grid, kThreads, 0, s>>>(p);
    else gate_kernel_multi<KL, KG, DIAQ_CMUL_PLAIN><<<grid, kThreads, 0, s>>>(p);
    count_launch();
    return check_launch("gate_kernel_multi");
}

}  // namespace diaq

using namespace diaq;

extern "C" int diaq_apply_gate(int n_bits, int k, const double *g_host, const int *shifts, const void *x,
                               void *y, int cmul_mode, void *stream) {
    if (!g_host || !shifts || !x || !y) return set_error(DIAQ_ERR_VALUE, "diaq_apply_gate: null argument");
    return apply_gate(n_bits, k, g_host, shifts, x, y, cmul_mode, (cudaStream_t)stream);
}

extern "C" int diaq_run_gates(int n_bits, int ngates, const diaq_gate_t *gates, void *state, int cmul_mode,
                              void **events, void *stream) {
    cudaStream_t s = (cudaStream_t)stream;
    if (ngates < 0 || (ngates > 0 && !gates) || !state) return set_error(DIAQ_ERR_VALUE, "diaq_run_gates: bad arguments");
    if (events && timer_record(events[0], s) != cudaSuccess)
        return set_error(DIAQ_ERR_CUDA, "diaq_run_gates: event record failed");
    for (int i = 0; i < ngates; ++i) {
        const int rc = apply_gate(n_bits, gates[i].k, gates[i].g, gates[i].shifts, state, state, cmul_mode, s);
        if (rc) return rc;
        if (events && timer_record(events[i + 1], s) != cudaSuccess)
            return set_error(DIAQ_ERR_CUDA, "diaq_run_gates: event record failed");
    }
    return DIAQ_OK;
}

extern "C" int diaq_apply_placed(int64_t dim_a, const diaq_matrix_t *m, int64_t dim_b, const void *x, void *y,
                                 int cmul_mode, void *stream) {
    if (!m || !x || !y) return set_error(DIAQ_ERR_VALUE, "diaq_apply_placed: null argument");
    if (dim_a < 1 || dim_b < 1) return set_error(DIAQ_ERR_SHAPE, "dim_a and dim_b must be >= 1");
    if (x == y) return set_error(DIAQ_ERR_VALUE, "diaq_apply_placed: y must not alias x");
    cudaStream_t s = (cudaStream_t)stream;
    // Any number of stored diagonals: chunks of kParamDiags in ascending
    // order, each later chunk continuing the per-amplitude sum in y -- the
    // same sequence of additions as one pass over all of them (reference
    // _apply_diags_block, sim.py:69-78, has no cap).
    static thread_local PlacedParams p;
    p.total = dim_a * m->n * dim_b;
    p.dim_b = dim_b;
    p.n_m = m->n;
    p.x = (const double2 *)x;
    p.y = (double2 *)y;
    const double2 *vals = (const double2 *)m->vals;
    const int64_t want = (p.total + kThreads - 1) / kThreads;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)sm_count() * 8));
    for (int64_t c0 = 0; c0 == 0 || c0 < m->nd; c0 += kParamDiags) {
        p.nd = (int)std::min<int64_t>(kParamDiags, m->nd - c0);
        p.accumulate = c0 > 0;
        for (int i = 0; i < p.nd; ++i) {
            const int64_t d = m->offs[c0 + i];
            p.dg[i].row0 = vals + m->starts[c0 + i] + (d < 0 ? d : 0);
            p.dg[i].lo = d < 0 ? -d : 0;
            p.dg[i].hi = d > 0 ? m->n - d : m->n;
            p.dg[i].xoff = d * dim_b;
        }
        if (cmul_mode != DIAQ_CMUL_PLAIN) placed_kernel<DIAQ_CMUL_FMA><<<grid, kThreads, 0, s>>>(p);
        else placed_kernel<DIAQ_CMUL_PLAIN><<<grid, kThreads, 0, s>>>(p);
        count_launch();
        const int rc = check_launch("placed_kernel");
        if (rc) return rc;
    }
    return DIAQ_OK;
}

extern "C" int diaq_init_basis(int64_t n_amps, void *x, int64_t index, void *stream) {
    if (!x || n_amps < 1) return set_error(DIAQ_ERR_VALUE, "diaq_init_basis: bad arguments");
    const int64_t want = (n_amps + kThreads - 1) / kThreads;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)sm_count() * 8));
    init_basis_kernel<<<grid, kThreads, 0, (cudaStream_t)stream>>>((double2 *)x, n_amps, index);
    count_launch();
    return check_launch("init_basis_kernel");
}

extern "C" int diaq_norm2(int64_t n_amps, const void *x, double *work_dev, void *stream) {
    if (!x || !work_dev || n_amps < 0) return set_error(DIAQ_ERR_VALUE, "diaq_norm2: bad arguments");
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t want = (n_amps + kThreads - 1) / kThreads;
    const int nb = (int)std::max<int64_t>(1, std::min<int64_t>(want, kNormBlocks));
    norm2_partial<<<nb, kThreads, 0, s>>>((const double2 *)x, n_amps, work_dev + 1);
    norm2_final<<<1, 1024, 0, s>>>(work_dev + 1, nb, work_dev);
    count_launch(2);
    return check_launch("norm2");
}

namespace diaq {
// a gate that reads only this rank's own block (no partner data needed)
int apply_gate_sharded_own(int n_bits, int local_bits, int k, const double *g, const int *shifts, int64_t rank,
                           void *shard, int cmul_mode, cudaStream_t s) {
    ShardView v;
    int rc = shard_view(n_bits, local_bits, k, g, shifts, rank, v);
    if (rc) return rc;
    if (v.kg == 0) return apply_gate(local_bits, k, g, shifts, shard, shard, cmul_mode, s);
    if (v.need != (1u << v.vr)) return set_error(DIAQ_ERR_VALUE, "gate needs partner shards (need mask %u)", v.need);
    const void *srcs[8] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
    srcs[v.vr] = shard;
#define DIAQ_MULTI(KL_, KG_) \
    if (v.kl == KL_ && v.kg == KG_) return launch_multi<KL_, KG_>(v, local_bits, g, srcs, shard, cmul_mode, s);
    DIAQ_MULTI(0, 1) DIAQ_MULTI(1, 1) DIAQ_MULTI(2, 1) DIAQ_MULTI(3, 1) DIAQ_MULTI(4, 1)
    DIAQ_MULTI(0, 2) DIAQ_MULTI(1, 2) DIAQ_MULTI(2, 2) DIAQ_MULTI(3, 2)
    DIAQ_MULTI(0, 3) DIAQ_MULTI(1, 3) DIAQ_MULTI(2, 3)
#undef DIAQ_MULTI
    return set_error(DIAQ_ERR_UNSUPPORTED, "sharded gate with %d local + %d global operands", v.kl, v.kg);
}
}  // namespace diaq

extern "C" int diaq_shard_plan(int n_bits, int local_bits, int k, const double *g_host, const int *shifts,
                               int64_t rank, uint32_t *need_mask, int *n_global, uint32_t *own_block) {
    if (!g_host || !shifts || !need_mask) return set_error(DIAQ_ERR_VALUE, "diaq_shard_plan: null argument");
    ShardView v;
    const int rc = shard_view(n_bits, local_bits, k, g_host, shifts, rank, v);
    if (rc) return rc;
    *need_mask = v.need;
    if (n_global) *n_global = v.kg;
    if (own_block) *own_block = v.vr;
    return DIAQ_OK;
}

extern "C" int diaq_apply_gate_sharded(int n_bits, int local_bits, int k, const double *g_host, const int *shifts,
                                       int64_t rank, const void *const *srcs, void *y, int cmul_mode, void *stream) {
    if (!g_host || !shifts || !srcs || !y) return set_error(DIAQ_ERR_VALUE, "diaq_apply_gate_sharded: null argument");
    ShardView v;
    int rc = shard_view(n_bits, local_bits, k, g_host, shifts, rank, v);
    if (rc) return rc;
    cudaStream_t s = (cudaStream_t)stream;
    if (v.kg == 0) return apply_gate(local_bits, k, g_host, shifts, srcs[0], y, cmul_mode, s);
#define DIAQ_MULTI(KL_, KG_) \
    if (v.kl == KL_ && v.kg == KG_) return launch_multi<KL_, KG_>(v, local_bits, g_host, srcs, y, cmul_mode, s);
    DIAQ_MULTI(0, 1) DIAQ_MULTI(1, 1) DIAQ_MULTI(2, 1) DIAQ_MULTI(3, 1) DIAQ_MULTI(4, 1)
    DIAQ_MULTI(0, 2) DIAQ_MULTI(1, 2) DIAQ_MULTI(2, 2) DIAQ_MULTI(3, 2)
    DIAQ_MULTI(0, 3) DIAQ_MULTI(1, 3) DIAQ_MULTI(2, 3)
#undef DIAQ_MULTI
    return set_error(DIAQ_ERR_UNSUPPORTED, "sharded gate with %d local + %d global operands", v.kl, v.kg);
}
