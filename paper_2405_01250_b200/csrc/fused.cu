// fused.cu -- multi-gate passes over shared-memory tiles (sm_100a).
//
// The run loop (reference sim.py:193-199) applies gates one at a time; on the
// GPU each gate is a full 32*2^n-byte sweep of HBM.  A pass instead loads a
// tile of 2^T amplitudes -- every index that varies only in a chosen set B
// of T state bits (B always contains the low bits, so a tile row is a
// contiguous 128-byte run) -- into shared memory, applies a run of
// consecutive gates whose MIXING operand bits all lie in B, and writes the
// tile back: one HBM sweep for the whole run.
//
// Parity is unchanged: every gate is still applied on its own, in circuit
// order, with the gate kernel's arithmetic (relabelled ascending-embedding
// column order, numpy complex-multiply rounding, sequential adds from +0,
// exactly-zero entries skipped).  Operands a gate does not mix (controls,
// diagonal gates such as RZ/CZ) need not lie in B: within a group those bits
// are fixed, so they only select which sub-block of the gate applies
// (exactly the sharded-state argument, apply.cu).
#include <algorithm>
#include <cstring>
#include <vector>

#include "common.cuh"

namespace diaq {

constexpr int kMaxTileBits = 12;
constexpr int kMaxFusedK = 4;      // operands per gate on this path
constexpr int kLowBits = 3;        // tile rows are 2^3 amplitudes = 128 B

struct FusedGate {
    int kin, kout;                 // mixing operands (in the tile), block-selector operands
    int tsorted[kMaxFusedK];       // ascending tile positions of the mixing operands
    int emb[1 << kMaxFusedK];      // tile offset of relabelled mixing index c
    int osel[kMaxFusedK];          // selector j: 1 = bit from tile index, 0 = bit from tile base
    int opos[kMaxFusedK];          // tile position or state shift of selector j
    int coef_off;                  // coef[coef_off + (b << 2kin) + r * 2^kin + c]
    int nz_off;                    // nz[nz_off + (b << kin) + r]
};

struct PassParams {
    double2 *x;
    int64_t ntiles;
    int tbits;                     // T
    int tb[kMaxTileBits];          // ascending state bits of the tile
    int g0, g1;                    // gates [g0, g1) of the program
    const FusedGate *gates;
    const double2 *coef;
    const uint32_t *nz;
};

__device__ __forceinline__ uint64_t spread_tile(uint32_t e, const int *tb, int T) {
    uint64_t out = 0;
#pragma unroll
    for (int j = 0; j < kMaxTileBits; ++j)
        if (j < T) out |= (uint64_t)((e >> j) & 1u) << tb[j];
    return out;
}

__device__ __forceinline__ uint64_t insert_zero_bits_dyn(uint64_t g, const int *sh, int k) {
    for (int i = 0; i < k; ++i) {
        const uint64_t low = g & ((1ull << sh[i]) - 1ull);
        g = ((g >> sh[i]) << (sh[i] + 1)) | low;
    }
    return g;
}

__device__ __forceinline__ uint32_t block_of(const FusedGate &G, uint32_t te, uint64_t base) {
    uint32_t b = 0;
    for (int j = 0; j < G.kout; ++j) {
        const uint32_t bit = G.osel[j] ? (te >> G.opos[j]) & 1u : (uint32_t)((base >> G.opos[j]) & 1ull);
        b |= bit << (G.kout - 1 - j);
    }
    return b;
}

template <int KIN, int MODE>
__device__ __forceinline__ void apply_in_tile(double2 *tile, int T, const FusedGate &G, uint64_t base,
                                              const double2 *__restrict__ coef, const uint32_t *__restrict__ nz) {
    constexpr int M = 1 << KIN;
    const uint32_t ngroups = 1u << (T - KIN);
    for (uint32_t grp = threadIdx.x; grp < ngroups; grp += blockDim.x) {
        uint32_t tbase = grp;
#pragma unroll
        for (int i = 0; i < KIN; ++i) {
            const uint32_t low = tbase & ((1u << G.tsorted[i]) - 1u);
            tbase = ((tbase >> G.tsorted[i]) << (G.tsorted[i] + 1)) | low;
        }
        const uint32_t b = block_of(G, tbase, base);
        const double2 *cb = coef + G.coef_off + ((int)b << (2 * KIN));
        const uint32_t *nb = nz + G.nz_off + ((int)b << KIN);
        double2 xs[M];
#pragma unroll
        for (int c = 0; c < M; ++c) xs[c] = tile[tbase + G.emb[c]];
#pragma unroll
        for (int r = 0; r < M; ++r) {
            double2 acc = make_double2(0.0, 0.0);
            const uint32_t m = nb[r];
#pragma unroll
            for (int c = 0; c < M; ++c)
                if ((m >> c) & 1u) acc = cadd(acc, cmul<MODE>(cb[r * M + c], xs[c]));
            tile[tbase + G.emb[r]] = acc;
        }
    }
}

constexpr int kMaxPassGates = 64;   // gate records staged in shared memory per pass
constexpr int kBatch = 8;  // tile elements per thread per load/store batch

// Tile element e = tid + kThreads*k.  Its state offset is
// (e & lowmask) + hi_off[e >> lowbits]: the low tile bits are the low state
// bits (contiguous), the rest come from a per-CTA table built once.
template <int MODE, int MAXKIN>
__global__ void __launch_bounds__(kThreads, MAXKIN >= 3 ? 2 : 4) fused_pass_kernel(const __grid_constant__ PassParams p) {
    extern __shared__ double2 tile[];
    __shared__ uint64_t hi_off[1 << kMaxTileBits >> 3];
    __shared__ FusedGate sg[kMaxPassGates];
    const int T = p.tbits;
    const uint32_t tsize = 1u << T;
    int lowbits = 0;
    while (lowbits < T && p.tb[lowbits] == lowbits) ++lowbits;
    if (lowbits > 8) lowbits = 8;  // e >> 8 indexes the table; kThreads == 256
    const uint32_t lowmask = (1u << lowbits) - 1u;
    for (uint32_t h = threadIdx.x; h < (tsize >> lowbits); h += blockDim.x) {
        uint64_t off = 0;
        for (int j = lowbits; j < T; ++j) off |= (uint64_t)((h >> (j - lowbits)) & 1u) << p.tb[j];
        hi_off[h] = off;
    }
    const int ng = p.g1 - p.g0;
    const bool staged = ng <= kMaxPassGates;
    if (staged)
        for (int i = threadIdx.x; i < ng * (int)(sizeof(FusedGate) / 4); i += blockDim.x)
            reinterpret_cast<int *>(sg)[i] = reinterpret_cast<const int *>(p.gates + p.g0)[i];
    __syncthreads();
    const int per_thread = (int)(tsize >= kThreads ? tsize / kThreads : 1);
    for (int64_t t = blockIdx.x; t < p.ntiles; t += gridDim.x) {
        const uint64_t base = insert_zero_bits_dyn((uint64_t)t, p.tb, T);
        for (int k0 = 0; k0 < per_thread; k0 += kBatch) {
            double2 v[kBatch];
#pragma unroll
            for (int k = 0; k < kBatch; ++k) {
                const uint32_t e = threadIdx.x + (uint32_t)(k0 + k) * kThreads;
                if (k0 + k < per_thread && e < tsize)
                    v[k] = ld_reuse(p.x + base + (e & lowmask) + hi_off[e >> lowbits]);
            }
#pragma unroll
            for (int k = 0; k < kBatch; ++k) {
                const uint32_t e = threadIdx.x + (uint32_t)(k0 + k) * kThreads;
                if (k0 + k < per_thread && e < tsize) tile[e] = v[k];
            }
        }
        __syncthreads();
        for (int gi = 0; gi < ng; ++gi) {
            const FusedGate &G = staged ? sg[gi] : p.gates[p.g0 + gi];
            switch (G.kin) {
                case 0: {  // diagonal in every operand: element-wise
                    for (uint32_t e = threadIdx.x; e < tsize; e += blockDim.x) {
                        const uint32_t b = block_of(G, e, base);
                        double2 acc = make_double2(0.0, 0.0);
                        if (p.nz[G.nz_off + b] & 1u) acc = cadd(acc, cmul<MODE>(p.coef[G.coef_off + b], tile[e]));
                        tile[e] = acc;
                    }
                    break;
                }
                case 1: apply_in_tile<1, MODE>(tile, T, G, base, p.coef, p.nz); break;
                case 2: if constexpr (MAXKIN >= 2) apply_in_tile<2, MODE>(tile, T, G, base, p.coef, p.nz); break;
                case 3: if constexpr (MAXKIN >= 3) apply_in_tile<3, MODE>(tile, T, G, base, p.coef, p.nz); break;
                default: if constexpr (MAXKIN >= 4) apply_in_tile<4, MODE>(tile, T, G, base, p.coef, p.nz); break;
            }
            __syncthreads();
        }
        for (int k = 0; k < per_thread; ++k) {
            const uint32_t e = threadIdx.x + (uint32_t)k * kThreads;
            if (e < tsize) st_stream(p.x + base + (e & lowmask) + hi_off[e >> lowbits], tile[e]);
        }
        __syncthreads();
    }
}

// ---- host: analysis, scheduling, packing ------------------------------------

// operand i mixes iff some nonzero entry connects a row and a column that
// differ in bit (k-1-i) of the gate index
static uint32_t mixing_mask(int k, const double *g) {
    const int M = 1 << k;
    uint32_t mix = 0;
    for (int r = 0; r < M; ++r)
        for (int c = 0; c < M; ++c) {
            const double re = g[2 * (r * M + c)], im = g[2 * (r * M + c) + 1];
            if (re == 0.0 && im == 0.0) continue;
            const int diff = r ^ c;
            for (int i = 0; i < k; ++i)
                if ((diff >> (k - 1 - i)) & 1) mix |= 1u << i;
        }
    return mix;
}

struct Program {
    std::vector<FusedGate> gates;
    std::vector<double2> coef;
    std::vector<uint32_t> nz;
    struct Pass {
        int g0, g1;
        int maxkin = 1;
        std::vector<int> bits;  // ascending state bits of the tile
        std::vector<int> members;  // indices into the caller's gate list
    };
    std::vector<Pass> passes;
};

static int pack_gate(const diaq_gate_t &gt, const std::vector<int> &bits, Program &pr) {
    const int k = gt.k;
    const int M = 1 << k;
    const uint32_t mix = mixing_mask(k, gt.g);
    std::vector<int> mops, sops;  // mixing / selector operands
    for (int i = 0; i < k; ++i) ((mix >> i) & 1u ? mops : sops).push_back(i);
    std::sort(mops.begin(), mops.end(), [&](int a, int b) { return gt.shifts[a] > gt.shifts[b]; });
    std::sort(sops.begin(), sops.end(), [&](int a, int b) { return gt.shifts[a] > gt.shifts[b]; });
    FusedGate G;
    memset(&G, 0, sizeof(G));
    G.kin = (int)mops.size();
    G.kout = (int)sops.size();
    if (G.kin > kMaxFusedK || G.kout > kMaxFusedK) return set_error(DIAQ_ERR_UNSUPPORTED, "fused gate too wide");
    auto tpos = [&](int shift) {
        for (size_t j = 0; j < bits.size(); ++j)
            if (bits[j] == shift) return (int)j;
        return -1;
    };
    std::vector<int> tp;
    for (int j = 0; j < G.kin; ++j) {
        const int p = tpos(gt.shifts[mops[j]]);
        if (p < 0) return set_error(DIAQ_ERR_VALUE, "fused pass: mixing bit outside the tile");
        tp.push_back(p);
    }
    std::vector<int> ts = tp;
    std::sort(ts.begin(), ts.end());
    for (int j = 0; j < G.kin; ++j) G.tsorted[j] = ts[j];
    const int MI = 1 << G.kin;
    for (int c = 0; c < MI; ++c) {
        int e = 0;
        for (int j = 0; j < G.kin; ++j) e |= ((c >> (G.kin - 1 - j)) & 1) << tp[j];
        G.emb[c] = e;
    }
    for (int j = 0; j < G.kout; ++j) {
        const int s = gt.shifts[sops[j]];
        const int p = tpos(s);
        G.osel[j] = p >= 0 ? 1 : 0;
        G.opos[j] = p >= 0 ? p : s;
    }
    // original gate index from (selector value b, mixing value c)
    auto orig = [&](int b, int c) {
        int o = 0;
        for (int j = 0; j < G.kin; ++j) o |= ((c >> (G.kin - 1 - j)) & 1) << (k - 1 - mops[j]);
        for (int j = 0; j < G.kout; ++j) o |= ((b >> (G.kout - 1 - j)) & 1) << (k - 1 - sops[j]);
        return o;
    };
    G.coef_off = (int)pr.coef.size();
    G.nz_off = (int)pr.nz.size();
    for (int b = 0; b < (1 << G.kout); ++b)
        for (int r = 0; r < MI; ++r) {
            uint32_t m = 0;
            for (int c = 0; c < MI; ++c) {
                const int o_r = orig(b, r), o_c = orig(b, c);
                const double re = gt.g[2 * (o_r * M + o_c)], im = gt.g[2 * (o_r * M + o_c) + 1];
                pr.coef.push_back(make_double2(re, im));
                if (re != 0.0 || im != 0.0) m |= 1u << c;
            }
            pr.nz.push_back(m);
        }
    pr.gates.push_back(G);
    return DIAQ_OK;
}

// Greedy left-to-right: extend the current pass while the union of mixing
// bits (plus the low bits) fits in T; gates wider than kMaxFusedK or whose
// mixing bits alone exceed T become single-gate passes (tile empty: bits
// left empty, applied by gate_kernel).
static int schedule(int n_bits, int ngates, const diaq_gate_t *gates, int T, Program &pr) {
    const int low = std::min(kLowBits, n_bits);
    std::vector<int> cur_members;
    std::vector<char> inb(64, 0);
    int nb = 0;
    auto reset = [&]() {
        std::fill(inb.begin(), inb.end(), 0);
        nb = 0;
        for (int b = 0; b < low; ++b) { inb[b] = 1; ++nb; }
        cur_members.clear();
    };
    auto flush = [&]() -> int {
        if (cur_members.empty()) return DIAQ_OK;
        Program::Pass ps;
        std::vector<int> bits;
        for (int b = 0; b < 64; ++b)
            if (inb[b]) bits.push_back(b);
        // pad the tile to exactly T bits with the lowest unused bits
        for (int b = 0; (int)bits.size() < T && b < n_bits; ++b)
            if (!inb[b]) { bits.push_back(b); }
        std::sort(bits.begin(), bits.end());
        ps.bits = bits;
        ps.members = cur_members;
        ps.g0 = (int)pr.gates.size();
        for (int gi : cur_members) {
            const int rc = pack_gate(gates[gi], bits, pr);
            if (rc) return rc;
            ps.maxkin = std::max(ps.maxkin, pr.gates.back().kin);
        }
        ps.g1 = (int)pr.gates.size();
        pr.passes.push_back(ps);
        return DIAQ_OK;
    };
    reset();
    for (int i = 0; i < ngates; ++i) {
        const diaq_gate_t &gt = gates[i];
        if (gt.k < 1 || gt.k > 5) return set_error(DIAQ_ERR_UNSUPPORTED, "gate width %d outside 1..5", gt.k);
        const uint32_t mix = mixing_mask(gt.k, gt.g);
        int kin = 0, kout = 0, add = 0;
        for (int j = 0; j < gt.k; ++j) {
            if (gt.shifts[j] < 0 || gt.shifts[j] >= n_bits)
                return set_error(DIAQ_ERR_SHAPE, "gate shift %d outside state of %d qubits", gt.shifts[j], n_bits);
            if ((mix >> j) & 1u) { ++kin; add += inb[gt.shifts[j]] ? 0 : 1; }
            else ++kout;
        }
        if (kin > kMaxFusedK || kout > kMaxFusedK) {  // too wide for the tile path: its own pass
            int rc = flush();
            if (rc) return rc;
            reset();
            Program::Pass ps;
            ps.g0 = ps.g1 = -1;
            ps.members = {i};
            pr.passes.push_back(ps);
            continue;
        }
        if (nb + add > T) {
            int rc = flush();
            if (rc) return rc;
            reset();
            add = 0;
            for (int j = 0; j < gt.k; ++j)
                if (((mix >> j) & 1u) && !inb[gt.shifts[j]]) ++add;
        }
        for (int j = 0; j < gt.k; ++j)
            if (((mix >> j) & 1u) && !inb[gt.shifts[j]]) { inb[gt.shifts[j]] = 1; ++nb; }
        cur_members.push_back(i);
    }
    return flush();
}

int apply_gate(int n_bits, int k, const double *g, const int *shifts, const void *x, void *y, int cmul_mode,
               cudaStream_t s);

static int sm_count_f() {
    int dev = 0, sms = kSms;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaGetLastError();
    return sms;
}

}  // namespace diaq

using namespace diaq;

extern "C" int diaq_run_gates_fused(int n_bits, int ngates, const diaq_gate_t *gates, void *state, int cmul_mode,
                                    int tile_bits, void **events, int *npasses, void *stream) {
    if (ngates < 0 || (ngates > 0 && !gates) || !state)
        return set_error(DIAQ_ERR_VALUE, "diaq_run_gates_fused: bad arguments");
    cudaStream_t s = (cudaStream_t)stream;
    int T = tile_bits <= 0 ? 11 : tile_bits;
    T = std::min(std::min(T, kMaxTileBits), n_bits);
    Program pr;
    int rc = schedule(n_bits, ngates, gates, T, pr);
    if (rc) return rc;
    if (npasses) *npasses = (int)pr.passes.size();
    FusedGate *dg = nullptr;
    double2 *dc = nullptr;
    uint32_t *dn = nullptr;
    const size_t gb = sizeof(FusedGate) * std::max<size_t>(1, pr.gates.size());
    const size_t cb = sizeof(double2) * std::max<size_t>(1, pr.coef.size());
    const size_t nbytes = sizeof(uint32_t) * std::max<size_t>(1, pr.nz.size());
    if (cudaMallocAsync((void **)&dg, gb, s) != cudaSuccess || cudaMallocAsync((void **)&dc, cb, s) != cudaSuccess ||
        cudaMallocAsync((void **)&dn, nbytes, s) != cudaSuccess)
        return set_error(DIAQ_ERR_CUDA, "diaq_run_gates_fused: program alloc failed");
    if (!pr.gates.empty()) {
        cudaMemcpyAsync(dg, pr.gates.data(), sizeof(FusedGate) * pr.gates.size(), cudaMemcpyHostToDevice, s);
        cudaMemcpyAsync(dc, pr.coef.data(), sizeof(double2) * pr.coef.size(), cudaMemcpyHostToDevice, s);
        cudaMemcpyAsync(dn, pr.nz.data(), sizeof(uint32_t) * pr.nz.size(), cudaMemcpyHostToDevice, s);
    }
    const size_t smem_max = sizeof(double2) << kMaxTileBits;
    static bool attr_set = false;
    if (!attr_set) {
#define DIAQ_SMEM_ATTR(M_, K_) \
    cudaFuncSetAttribute(fused_pass_kernel<M_, K_>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_max);
        DIAQ_SMEM_ATTR(DIAQ_CMUL_FMA, 1) DIAQ_SMEM_ATTR(DIAQ_CMUL_FMA, 2) DIAQ_SMEM_ATTR(DIAQ_CMUL_FMA, 3)
        DIAQ_SMEM_ATTR(DIAQ_CMUL_FMA, 4) DIAQ_SMEM_ATTR(DIAQ_CMUL_PLAIN, 1) DIAQ_SMEM_ATTR(DIAQ_CMUL_PLAIN, 2)
        DIAQ_SMEM_ATTR(DIAQ_CMUL_PLAIN, 3) DIAQ_SMEM_ATTR(DIAQ_CMUL_PLAIN, 4)
#undef DIAQ_SMEM_ATTR
        attr_set = true;
    }
    int gate_idx = 0;
    if (events && cudaEventRecord((cudaEvent_t)events[0], s) != cudaSuccess)
        return set_error(DIAQ_ERR_CUDA, "diaq_run_gates_fused: event record failed");
    for (size_t pi = 0; pi < pr.passes.size() && rc == DIAQ_OK; ++pi) {
        const Program::Pass &ps = pr.passes[pi];
        if (ps.g0 < 0 || ps.members.size() == 1) {
            const diaq_gate_t &gt = gates[ps.members[0]];
            rc = apply_gate(n_bits, gt.k, gt.g, gt.shifts, state, state, cmul_mode, s);
        } else {
            PassParams p;
            p.x = (double2 *)state;
            p.tbits = (int)ps.bits.size();
            for (int j = 0; j < p.tbits; ++j) p.tb[j] = ps.bits[j];
            p.ntiles = (int64_t)1 << (n_bits - p.tbits);
            p.g0 = ps.g0;
            p.g1 = ps.g1;
            p.gates = dg;
            p.coef = dc;
            p.nz = dn;
            const size_t smem = sizeof(double2) << p.tbits;
            const int mk = std::min(4, std::max(1, ps.maxkin));
            const bool fma = cmul_mode == DIAQ_CMUL_FMA;
            const void *f = nullptr;
            switch (mk) {
                case 1: f = fma ? (const void *)fused_pass_kernel<DIAQ_CMUL_FMA, 1> : (const void *)fused_pass_kernel<DIAQ_CMUL_PLAIN, 1>; break;
                case 2: f = fma ? (const void *)fused_pass_kernel<DIAQ_CMUL_FMA, 2> : (const void *)fused_pass_kernel<DIAQ_CMUL_PLAIN, 2>; break;
                case 3: f = fma ? (const void *)fused_pass_kernel<DIAQ_CMUL_FMA, 3> : (const void *)fused_pass_kernel<DIAQ_CMUL_PLAIN, 3>; break;
                default: f = fma ? (const void *)fused_pass_kernel<DIAQ_CMUL_FMA, 4> : (const void *)fused_pass_kernel<DIAQ_CMUL_PLAIN, 4>; break;
            }
            int per_sm = 1;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, f, kThreads, smem);
            const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(p.ntiles, (int64_t)sm_count_f() * std::max(1, per_sm)));
            void *args[] = {(void *)&p};
            cudaLaunchKernel(f, dim3((unsigned)grid), dim3(kThreads), args, smem, s);
            count_launch();
            rc = check_launch("fused_pass_kernel");
        }
        gate_idx += (int)ps.members.size();
        // events[i]..events[i+1] bracket gate i; a fused pass's time lands on
        // its first gate, the others record zero-length intervals
        if (events && rc == DIAQ_OK)
            for (int gi : ps.members) cudaEventRecord((cudaEvent_t)events[gi + 1], s);
    }
    cudaFreeAsync(dg, s);
    cudaFreeAsync(dc, s);
    cudaFreeAsync(dn, s);
    (void)gate_idx;
    return rc;
}
