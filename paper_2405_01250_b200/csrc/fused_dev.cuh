// fused_dev.cuh -- device side of the multi-gate passes (see fused.cu for
// the design): pass records, register fast paths and the pass body.  Shared
// by the AOT interpreter kernel (fused.cu) and the NVRTC-specialised kernels
// (fused_jit.cu), which compile this same text with the structure constant.
#pragma once
#ifndef __CUDACC_RTC__
#include <stdint.h>

#include "dev_common.cuh"
#endif

// loops over pass structure: fully unrolled when the structure is a
// compile-time constant (NVRTC), left rolled in the interpreter
#ifdef DIAQ_JIT
#define DIAQ_SUNROLL _Pragma("unroll")
#else
#define DIAQ_SUNROLL
#endif

namespace diaq {

constexpr int kMaxTileBits = 12;
constexpr int kThreadBits = 8;      // 256 threads
constexpr int kLowBits = 3;         // tile rows are 2^3 amplitudes = 128 B
constexpr int kMaxRegKin = 2;       // mixing operands of a fused gate (2: shared-memory path; wider: own pass)
constexpr int kMaxSel = 4;          // selector (non-mixing) operands
constexpr int kMaxPassGates = 48;   // gate records per pass (kernel parameters)
constexpr int kMaxPhases = 24;
constexpr int kRetryNoDense2 = 1000;  // schedule(): internal, re-plan without register 2-qubit gates
constexpr int kMaxCoef = 256;       // coefficient entries per pass (kernel parameters)
constexpr int kMaxNz = 256;
constexpr int kPrePhases = 4;       // phases whose register slots are precomputed per CTA (R = 3; 3 at R = 4,
                                    // within the 48 KB of static shared memory)

static_assert(kThreads == (1 << kThreadBits), "thread layout");

struct RegGate {               // narrow fields: the records live in the kernel parameters
    int8_t kin;               // 0 or 1 mixing operands
    int8_t rb[kMaxRegKin];    // register bits of the mixing operands, descending (relabelled order)
    int8_t kout;              // selector operands
    int8_t osel[kMaxSel];     // 0: bit `opos` of the tile base; 1: thread bit at tile position opos;
                              // 2: register bit opos (varies between register groups)
    int8_t opos[kMaxSel];
    int8_t rsel;              // any osel == 2
    // fast-path classification (host): 0 generic, 1 dense 1-qubit (no selector),
    // 2 diagonal with one selector, 3 dense 2-qubit, 4 X / CX on register
    // bits rb[0] (target) and rb[1] (control, -1: none): an exchange of registers
    int8_t op;
    // dense 1-qubit coefficient shape (host): 0 complex, 1 all entries real
    // (RY, H), 2 real diagonal / imaginary off-diagonal (RX); contracted
    // arithmetic only: 3 / 4 = shapes 1 / 2 with both diagonal entries
    // exactly 1 (their common value factored out of the pass, fused.cu)
    int8_t shape;
    int8_t full;              // dense 1-qubit: all four entries nonzero (host) -- the branch-free form
    int8_t mpos[kMaxRegKin];  // generic phases: tile positions of the mixing bits (relabelled order)
    int16_t coef_off;         // coef[coef_off + (b << 2kin) + r * 2^kin + c]   (pass-relative)
    int16_t nz_off;           // nz[nz_off + (b << kin) + r]
    int16_t cls_off;          // host classification table (identity / swap blocks)
};

// Affine relabelling of tile indices, f -> A f ^ c ^ (XOR of b_i over the set
// full-state bits bbit_i): how a run of permutation gates (X, CX, SWAP, any
// gate whose matrix is a 0/1 permutation affine in the index bits) moves
// amplitudes.  Such runs are not executed: they are folded into the smem
// slot each amplitude is written to (phase store / tile load).
constexpr int kMaxPermBase = 8;

struct Affine {
    int8_t on;
    int8_t nb;
    uint16_t c;
    uint16_t a[kMaxTileBits];    // image of tile bit j
    int8_t bbit[kMaxPermBase];
    uint16_t b[kMaxPermBase];
};

__host__ __device__ __forceinline__ uint32_t aff_lin(const Affine &m, uint32_t f, int T) {
    uint32_t r = 0;
    DIAQ_SUNROLL
    for (int j = 0; j < T; ++j)
        if ((f >> j) & 1u) r ^= m.a[j];
    return r;
}

__device__ __forceinline__ uint32_t aff_const(const Affine &m, uint64_t sbase) {
    uint32_t r = m.c;
    DIAQ_SUNROLL
    for (int i = 0; i < m.nb; ++i)
        if ((sbase >> m.bbit[i]) & 1ull) r ^= m.b[i];
    return r;
}

struct Phase {
    int16_t g0, g1;           // gates [g0, g1) of the pass (pass-relative)
    int8_t generic;           // 1: gates applied in shared memory (no register bits)
    // sequence phase: its dense gates hit register bits 0, 1, ... in order
    // (register bits in first-use order), any other gate is a diagonal on a
    // non-register bit; nd_before[b] diagonals precede the dense gate on bit
    // b (nd_before[R]: trailing).  The kernel then unrolls over the register
    // bit, so every dense step has a compile-time pairing.
    int8_t seq, ndense;
    int8_t nd_before[5];
    int8_t kind[5];           // sequence phase: 1 = dense 1-qubit gate on bit b, 2 = dense 2-qubit on (b, b+1)
    int8_t rpos[4];           // tile positions of the register bits, ascending (R entries)
    int8_t tpos[kMaxTileBits];  // tile positions of the thread bits, ascending (T - R entries)
    Affine post;              // permutation run after the phase's gates, applied by its store
    // swizzled smem slot of register j's part of the index (swz is linear
    // over GF(2), and thread and register bits are disjoint): register j of
    // a thread lives at swz(tpart) ^ pj[j]; its post-permutation slot at
    // swz(A tpart ^ c) ^ ppj[j]
    uint16_t pj[16];
    uint16_t ppj[16];
};

// One pass = one launch; its whole gate program rides in the kernel
// parameters (__grid_constant__, < 32 KB): every thread reads the same
// phase / gate / coefficient at the same time, so these are uniform
// constant-bank loads, not per-thread shared-memory traffic.
struct TileParams {
    double2 *x;
    int64_t ntiles;
    int tbits;                // T
    int tb[kMaxTileBits];     // ascending state bits of the tile
    int nphases;
    int ngates;
    int ncoef, nnz;
    uint64_t gbase;           // sharded state: rank bits (rank << local_bits) for selector lookups
    uint64_t tmask;           // state bits of the tile
    uint64_t gstep;           // gridDim.x deposited into the non-tile bits (tile base stride)
    Affine pre;               // permutation run opening the pass, applied by the tile load
    double2 *y;               // destination (== x: in place)
    int gperm;                // store through the global map (out of place)
    int nbuf;                 // tile buffers in dynamic smem: 2 = prefetch the next tile during this one
    int gstore;               // global-map store: 0 streaming (.cs), 1 write-back default, 2 L2 evict_last
    int estore;               // pair passes: gather the store into registers, fetch the next unit, then store
    // pair passes with estore: units handed out in order by a global counter
    // (null: static blockIdx + k gridDim), so the units in flight are always
    // a contiguous window and adjacent DRAM runs are fetched together; the
    // last CTA to finish resets the counter pair for the slot's next launch
    unsigned long long *uctr;
    unsigned long long *udone;
    uint64_t gconst;          // its constant, rank bits folded in
    uint64_t gcol[64];        // image of local state bit j
    // Pair store of a global tail that splits 32-byte sectors (specialised
    // passes only): a tile and its partner across the extra state bit gpb[0]
    // run in one CTA, which writes whole destination sectors (rows, when the
    // map allows) gathered from both -- no partial-sector writes (DRAM
    // read-modify-write).  Pairs enumerate over eb[] (tile bits and gpb[0],
    // ascending; emask); the destination set of a pair is ab ^ span(gw[]),
    // gw[0..] = e0 (e1, e2) first, and gsrc[k] = tile offset | (half << 12)
    // of gw[k]'s source.  gnp = 0: per-element scatter store.
    int8_t gnp;
    // Plain pair (specialised passes, no global tail): the tile and its
    // partner across gpb[0] (the lowest non-tile bit, when that is bit 3)
    // are loaded, computed and stored together by one CTA, so every DRAM
    // access is a 256-byte run instead of two 128-byte halves visited by
    // different CTAs at different times (row-buffer locality: a pass over
    // high tile bits ran 1.98 ms against 1.50 ms with 256-byte runs, r02e)
    int8_t ppair;
    int8_t dstore;  // specialised passes: the last phase stores to HBM from registers (its register bits
                    // avoid tile positions 0-2, thread bits 0-2 sit on them: 128-byte rows per 8 lanes)
    int8_t ppipe;   // plain pair schedule: 0 both halves land before either computes, 1 half A computes
                    // while B lands, 2 half A is stored and the next A fetched while B computes,
                    // 3 the halves run on the two CTAs of a cluster (fetches aligned by a cluster barrier)
    int8_t gpb[3];
    int8_t eb[kMaxTileBits + 3];
    uint64_t emask;
    uint64_t gw[kMaxTileBits + 3];
    uint16_t gsrc[kMaxTileBits + 3];
    Phase ph[kMaxPhases];
    RegGate g[kMaxPassGates]; // pass-relative order
    double2 coef[kMaxCoef];
    uint32_t nz[kMaxNz];
};
static_assert(sizeof(TileParams) <= 32764, "kernel parameter space");

// base of tile t + gridDim.x from the base of tile t: add in the number
// system of the non-tile bits (tile bits forced to 1 carry straight through)
__device__ __forceinline__ uint64_t next_base(uint64_t base, const TileParams &p, const TileParams &S) {
    return ((base | S.tmask) + p.gstep) & ~S.tmask;
}

__host__ __device__ __forceinline__ uint32_t swz(uint32_t e) {
    return e ^ (((e >> 3) ^ (e >> 6) ^ (e >> 9)) & 7u);
}

template <class I>
__device__ __forceinline__ uint64_t insert_zero_bits_dyn(uint64_t g, const I *sh, int k) {
    DIAQ_SUNROLL
    for (int i = 0; i < k; ++i) {
        const uint64_t low = g & ((1ull << sh[i]) - 1ull);
        g = ((g >> sh[i]) << (sh[i] + 1)) | low;
    }
    return g;
}

template <int R>
__device__ __forceinline__ uint32_t reg_spread(int j, const int8_t *rpos) {
    uint32_t e = 0;
#pragma unroll
    for (int i = 0; i < R; ++i) e |= (uint32_t)((j >> i) & 1) << rpos[i];
    return e;
}

// ---- fast paths (R = 3 register bits) --------------------------------------

template <int R, int B1, int MODE>
__device__ __forceinline__ void dense1(double2 (&v)[1 << R], const double2 *c, uint32_t n0, uint32_t n1) {
    const double2 c00 = c[0], c01 = c[1], c10 = c[2], c11 = c[3];
#pragma unroll
    for (int g = 0; g < (1 << (R - 1)); ++g) {
        const int j0 = ((g >> B1) << (B1 + 1)) | (g & ((1 << B1) - 1));
        const int j1 = j0 | (1 << B1);
        const double2 x0 = v[j0], x1 = v[j1];
        // acc starts at +0; +0 + t == t except for the sign of an exact zero,
        // so the first term is taken as is (values unchanged, one add saved)
        double2 a0, a1;
        if ((n0 & 3u) == 3u) a0 = cadd(cmul<MODE>(c00, x0), cmul<MODE>(c01, x1));
        else if (n0 & 1u) a0 = cmul<MODE>(c00, x0);
        else if (n0 & 2u) a0 = cmul<MODE>(c01, x1);
        else a0 = make_double2(0.0, 0.0);
        if ((n1 & 3u) == 3u) a1 = cadd(cmul<MODE>(c10, x0), cmul<MODE>(c11, x1));
        else if (n1 & 1u) a1 = cmul<MODE>(c10, x0);
        else if (n1 & 2u) a1 = cmul<MODE>(c11, x1);
        else a1 = make_double2(0.0, 0.0);
        v[j0] = a0;
        v[j1] = a1;
    }
}

// all four entries nonzero (RX, RY, H, U3 ...): branch-free, so the
// compiler interleaves the 2^R independent multiply-add chains.
// SHAPE 1 (every entry real) / 2 (real diagonal, imaginary off-diagonal):
// an entry's zero part contributes an exact +-0 to each product, so
//   (vr + 0i) x = (vr xr, vr xi),   (0 + vi i) x = (-(vi xi), vi xr)
// in both numpy multiply forms (plain and FMA) up to the sign of an exact
// zero -- 6 instead of 10 FP64 operations per amplitude, same values.
template <int R, int B1, int MODE, int SHAPE = 0>
__device__ __forceinline__ void dense1_full(double2 (&v)[1 << R], const double2 *c) {
    const double2 c00 = c[0], c01 = c[1], c10 = c[2], c11 = c[3];
#pragma unroll
    for (int g = 0; g < (1 << (R - 1)); ++g) {
        const int j0 = ((g >> B1) << (B1 + 1)) | (g & ((1 << B1) - 1));
        const int j1 = j0 | (1 << B1);
        const double2 x0 = v[j0], x1 = v[j1];
        if constexpr (MODE == DIAQ_CMUL_CONTRACT) {  // 4 (shaped) / 8 FP64 operations per amplitude
            if constexpr (SHAPE == 3) {  // unit diagonal, real off-diagonal: 2 operations per amplitude
                v[j0] = cmac1_r(x0, c01.x, x1);
                v[j1] = cmac1_r(x1, c10.x, x0);
            } else if constexpr (SHAPE == 4) {  // unit diagonal, imaginary off-diagonal
                v[j0] = cmac1_i(x0, c01.y, x1);
                v[j1] = cmac1_i(x1, c10.y, x0);
            } else if constexpr (SHAPE == 1) {
                v[j0] = cmac2_rr(c00.x, x0, c01.x, x1);
                v[j1] = cmac2_rr(c10.x, x0, c11.x, x1);
            } else if constexpr (SHAPE == 2) {
                v[j0] = cmac2_ri(c00.x, x0, c01.y, x1);
                v[j1] = cmac2_ri(c11.x, x1, c10.y, x0);
            } else {
                v[j0] = cmac2_c(c00, x0, c01, x1);
                v[j1] = cmac2_c(c10, x0, c11, x1);
            }
        } else if constexpr (SHAPE == 1 || SHAPE == 3) {
            v[j0] = cadd(cmul_re(c00.x, x0), cmul_re(c01.x, x1));
            v[j1] = cadd(cmul_re(c10.x, x0), cmul_re(c11.x, x1));
        } else if constexpr (SHAPE == 2 || SHAPE == 4) {
            v[j0] = cadd(cmul_re(c00.x, x0), cmul_im(c01.y, x1));
            v[j1] = cadd(cmul_im(c10.y, x0), cmul_re(c11.x, x1));
        } else {
            v[j0] = cadd(cmul<MODE>(c00, x0), cmul<MODE>(c01, x1));
            v[j1] = cadd(cmul<MODE>(c10, x0), cmul<MODE>(c11, x1));
        }
    }
}

template <int R, int B1, int MODE>
__device__ __forceinline__ void dense1_shaped(double2 (&v)[1 << R], const double2 *c, int shape) {
    if (shape == 1) dense1_full<R, B1, MODE, 1>(v, c);
    else if (shape == 2) dense1_full<R, B1, MODE, 2>(v, c);
    else if (MODE == DIAQ_CMUL_CONTRACT && shape == 3) dense1_full<R, B1, MODE, 3>(v, c);  // host: contracted only
    else if (MODE == DIAQ_CMUL_CONTRACT && shape == 4) dense1_full<R, B1, MODE, 4>(v, c);
    else dense1_full<R, B1, MODE, 0>(v, c);
}

// dense two-qubit gate (all 16 entries nonzero) on register bits RA (its
// gate-index MSB, the operand with the larger state bit) and RB: four
// amplitude groups per 16 registers, ascending columns, first term as is
template <int R, int RA, int RB, int MODE>
__device__ __forceinline__ void dense2_full(double2 (&v)[1 << R], const double2 *c) {
    constexpr int LO = RA < RB ? RA : RB, HI = RA < RB ? RB : RA;
#pragma unroll
    for (int g = 0; g < (1 << (R - 2)); ++g) {
        int j0 = ((g >> LO) << (LO + 1)) | (g & ((1 << LO) - 1));
        j0 = ((j0 >> HI) << (HI + 1)) | (j0 & ((1 << HI) - 1));
        const int jq[4] = {j0, j0 | (1 << RB), j0 | (1 << RA), j0 | (1 << RA) | (1 << RB)};
        const double2 x0 = v[jq[0]], x1 = v[jq[1]], x2 = v[jq[2]], x3 = v[jq[3]];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            if constexpr (MODE == DIAQ_CMUL_CONTRACT) {
                v[jq[r]] = cfma_c(c[r * 4], x0, cfma_c(c[r * 4 + 1], x1, cmac2_c(c[r * 4 + 2], x2, c[r * 4 + 3], x3)));
                continue;
            }
            double2 a = cmul<MODE>(c[r * 4], x0);
            a = cadd(a, cmul<MODE>(c[r * 4 + 1], x1));
            a = cadd(a, cmul<MODE>(c[r * 4 + 2], x2));
            a = cadd(a, cmul<MODE>(c[r * 4 + 3], x3));
            v[jq[r]] = a;
        }
    }
}

// Diagonal factors are applied branch-free: an entry whose nz bit is clear is
// stored as exactly 0 + 0i, and 0 * x is the skipped term's +-0 (finite
// states), so values are unchanged; a uniform branch here would make ptxas
// copy the whole amplitude set at every iteration of the diagonal loops.
template <int R, int RB, int MODE>
__device__ __forceinline__ void diag_reg(double2 (&v)[1 << R], double2 d0, double2 d1) {
#pragma unroll
    for (int j = 0; j < (1 << R); ++j) v[j] = cmul<MODE>(((j >> RB) & 1) ? d1 : d0, v[j]);
}



// compile-time dispatch of a runtime register bit b in [0, R)
#define DIAQ_RB_DISPATCH(R_, b_, CALL)                              \
    do {                                                            \
        if ((b_) == 0) { constexpr int RB_ = 0; CALL; }             \
        else if ((b_) == 1) { constexpr int RB_ = 1; CALL; }        \
        else if ((R_) == 3 || (b_) == 2) { constexpr int RB_ = 2; CALL; } \
        else { constexpr int RB_ = (R_) >= 4 ? 3 : 2; CALL; }       \
    } while (0)


// the tile's full-state base lives in shared memory and is re-read where a
// selector needs it (an asm load: not hoisted into a register held across
// the gate loop, where it would push the fast paths into spills)
__device__ __forceinline__ uint64_t ld_base(const uint64_t *s) {
    uint64_t v;
    asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"(smem_u32(s)));
    return v;
}

// diagonal gate whose selector is a thread or base bit: one factor for all
// of this thread's amplitudes
template <int R, int MODE>
__device__ __forceinline__ void diag_uniform(double2 (&v)[1 << R], const RegGate &G, uint32_t tpart,
                                             const uint64_t *sbase_p, const double2 *sc, const uint32_t *snz) {
    const uint32_t b = G.osel[0] == 0 ? (uint32_t)((ld_base(sbase_p) >> G.opos[0]) & 1ull) : (tpart >> G.opos[0]) & 1u;
#ifdef DIAQ_JIT
    // constant record: two uniform loads and a select, not a per-thread indexed load
    const double2 d = b ? sc[G.coef_off + 1] : sc[G.coef_off];
#else
    const double2 d = sc[G.coef_off + (int)b];
#endif
    (void)snz;
#pragma unroll
    for (int j = 0; j < (1 << R); ++j) v[j] = cmul<MODE>(d, v[j]);
}

// a run of `count` diagonal gates whose selectors are thread or base bits
// (gates S.g[gi ..]): applied one by one, or under DIAQ_CMUL_CONTRACT
// folded into one factor per thread (their product, in gate order) and
// applied with one complex multiply per amplitude
template <int R, int MODE>
__device__ __forceinline__ void diag_run(double2 (&v)[1 << R], const TileParams &S, int &gi, int count, uint32_t tpart,
                                         const uint64_t *sbase_p, const double2 *sc, const uint32_t *snz) {
    if constexpr (MODE == DIAQ_CMUL_CONTRACT) {
        if (count <= 0) return;
        double2 d = make_double2(1.0, 0.0);
        for (int c = 0; c < count; ++c, ++gi) {
            const RegGate &G = S.g[gi];
            const uint32_t b =
                G.osel[0] == 0 ? (uint32_t)((ld_base(sbase_p) >> G.opos[0]) & 1ull) : (tpart >> G.opos[0]) & 1u;
#ifdef DIAQ_JIT
            const double2 f = b ? sc[G.coef_off + 1] : sc[G.coef_off];
#else
            const double2 f = sc[G.coef_off + (int)b];
#endif
            d = c == 0 ? f : cmul_fma(f, d);
        }
#pragma unroll
        for (int j = 0; j < (1 << R); ++j) v[j] = cmul_fma(d, v[j]);
        (void)snz;
    } else {
#ifdef DIAQ_JIT
#pragma unroll
#else
#pragma unroll 2
#endif
        for (int c = 0; c < count; ++c, ++gi) diag_uniform<R, MODE>(v, S.g[gi], tpart, sbase_p, sc, snz);
    }
}

// X / CX on register bits (RegGate::op 4): exchange of register pairs over
// target bit rt, for the indices whose control bit rc is set (rc < 0: all).
// Register indices are static and the exchange is predicated on the
// (uniform) record: no arithmetic, and a pure renaming when the record is a
// compile-time constant (the specialised kernels).
template <int R>
__device__ __forceinline__ void reg_cx(double2 (&v)[1 << R], int rt, int rc) {
#pragma unroll
    for (int t = 0; t < R; ++t) {
        if (t != rt) continue;
#pragma unroll
        for (int j = 0; j < (1 << R); ++j) {
            if ((j >> t) & 1) continue;
            if (rc >= 0 && !((j >> rc) & 1)) continue;
            const double2 a = v[j];
            v[j] = v[j | (1 << t)];
            v[j | (1 << t)] = a;
        }
    }
}

template <int R, int MODE>
__device__ __forceinline__ void dispatch_gate(double2 (&v)[1 << R], const RegGate &G, uint32_t tpart, const uint64_t *sbase_p,
                                              const double2 *sc, const uint32_t *snz) {
    // if-chains, not switches: a jump table would force v[] into local memory
    static_assert(R == 3 || R == 4, "register fast paths cover 8 or 16 amplitudes per thread");
    if (G.op == 1) {
        const double2 *c = sc + G.coef_off;
        if (G.full) {  // (a structure constant in the specialised kernels: one form compiled)
            DIAQ_RB_DISPATCH(R, G.rb[0], (dense1_shaped<R, RB_, MODE>(v, c, G.shape)));
        } else {
            const uint32_t n0 = snz[G.nz_off], n1 = snz[G.nz_off + 1];
            DIAQ_RB_DISPATCH(R, G.rb[0], (dense1<R, RB_, MODE>(v, c, n0, n1)));
        }
        return;
    }
    if (G.op == 4) {
        reg_cx<R>(v, G.rb[0], G.rb[1]);
        return;
    }
    if (G.op == 2) {
        const double2 d0 = sc[G.coef_off], d1 = sc[G.coef_off + 1];
        if (G.osel[0] == 2) {
            DIAQ_RB_DISPATCH(R, G.opos[0], (diag_reg<R, RB_, MODE>(v, d0, d1)));
        } else {
            const uint32_t b = G.osel[0] == 0 ? (uint32_t)((ld_base(sbase_p) >> G.opos[0]) & 1ull) : (tpart >> G.opos[0]) & 1u;
            const double2 d = b ? d1 : d0;
#pragma unroll
            for (int j = 0; j < (1 << R); ++j) v[j] = cmul<MODE>(d, v[j]);
        }
        return;
    }
}

// Generic gate (any selectors, <= 2 mixing bits) applied in the shared-memory
// tile: the cold path for gates the register fast paths do not cover (and
// dense two-qubit gates).  Same per-amplitude order as gate_kernel: ascending
// relabelled column, from +0, exactly-zero entries skipped.
template <int MODE>
__device__ __forceinline__ void smem_gate(double2 *tile, int T, const RegGate &G, uint64_t base, const double2 *sc,
                                          const uint32_t *snz) {
    const int kin = G.kin;
    const uint32_t ngroups = 1u << (T - kin);
    const int p0 = G.mpos[0], p1 = G.mpos[1];
    const int lo = p0 < p1 ? p0 : p1, hi = p0 < p1 ? p1 : p0;
    for (uint32_t grp = threadIdx.x; grp < ngroups; grp += blockDim.x) {
        uint32_t e0 = grp;
        if (kin == 1) {
            e0 = ((e0 >> p0) << (p0 + 1)) | (e0 & ((1u << p0) - 1u));
        } else if (kin == 2) {
            e0 = ((e0 >> lo) << (lo + 1)) | (e0 & ((1u << lo) - 1u));
            e0 = ((e0 >> hi) << (hi + 1)) | (e0 & ((1u << hi) - 1u));
        }
        uint32_t b = 0;
        for (int s = 0; s < G.kout; ++s) {
            const uint32_t bit = G.osel[s] ? (e0 >> G.opos[s]) & 1u : (uint32_t)((base >> G.opos[s]) & 1ull);
            b |= bit << (G.kout - 1 - s);
        }
        const double2 *c = sc + G.coef_off + ((int)b << (2 * kin));
        const uint32_t *nz = snz + G.nz_off + ((int)b << kin);
        if (kin == 0) {
            const uint32_t i0 = swz(e0);
            tile[i0] = (nz[0] & 1u) ? cadd(make_double2(0.0, 0.0), cmul<MODE>(c[0], tile[i0])) : make_double2(0.0, 0.0);
        } else if (kin == 1) {
            const uint32_t i0 = swz(e0), i1 = swz(e0 | (1u << p0));
            const double2 x0 = tile[i0], x1 = tile[i1];
            double2 a0 = make_double2(0.0, 0.0), a1 = make_double2(0.0, 0.0);
            if (nz[0] & 1u) a0 = cadd(a0, cmul<MODE>(c[0], x0));
            if (nz[0] & 2u) a0 = cadd(a0, cmul<MODE>(c[1], x1));
            if (nz[1] & 1u) a1 = cadd(a1, cmul<MODE>(c[2], x0));
            if (nz[1] & 2u) a1 = cadd(a1, cmul<MODE>(c[3], x1));
            tile[i0] = a0;
            tile[i1] = a1;
        } else {
            uint32_t idx[4];
            double2 x[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {  // gate column q = (bit at p0, bit at p1)
                idx[q] = swz(e0 | ((uint32_t)(q >> 1) << p0) | ((uint32_t)(q & 1) << p1));
                x[q] = tile[idx[q]];
            }
            if ((nz[0] & nz[1] & nz[2] & nz[3] & 15u) == 15u) {  // dense (Haar4 ...): branch-free
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    double2 a = cadd(make_double2(0.0, 0.0), cmul<MODE>(c[r * 4], x[0]));
#pragma unroll
                    for (int q = 1; q < 4; ++q) a = cadd(a, cmul<MODE>(c[r * 4 + q], x[q]));
                    tile[idx[r]] = a;
                }
            } else {
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    double2 a = make_double2(0.0, 0.0);
#pragma unroll
                    for (int q = 0; q < 4; ++q)
                        if ((nz[r] >> q) & 1u) a = cadd(a, cmul<MODE>(c[r * 4 + q], x[q]));
                    tile[idx[r]] = a;
                }
            }
        }
    }
}

// sequence phase, register bit RB onwards: the diagonals before the dense
// gate on RB, then that gate with its pairing fixed at compile time
template <int R, int MODE, int RB>
__device__ __forceinline__ void seq_steps(double2 (&v)[1 << R], const TileParams &S, const Phase &ph, int &gi,
                                          uint32_t tpart, const uint64_t *sbase_p, const double2 *sc,
                                          const uint32_t *snz) {
    // (diag_run unrolls by 2: a complex multiply cannot land in its input
    // registers, so a rolled loop pays a register copy of the amplitude set
    // per gate to return to the loop-carried assignment)
    diag_run<R, MODE>(v, S, gi, ph.nd_before[RB], tpart, sbase_p, sc, snz);
    if (ph.kind[RB] == 1) {
        dense1_shaped<R, RB, MODE>(v, sc + S.g[gi].coef_off, S.g[gi].shape);
        ++gi;
        if constexpr (RB + 1 < R) seq_steps<R, MODE, RB + 1>(v, S, ph, gi, tpart, sbase_p, sc, snz);
    } else if (ph.kind[RB] == 2) {
        if constexpr (RB + 1 < R) {
            dense2_full<R, RB, RB + 1, MODE>(v, sc + S.g[gi].coef_off);
            ++gi;
            if constexpr (RB + 2 < R) seq_steps<R, MODE, RB + 2>(v, S, ph, gi, tpart, sbase_p, sc, snz);
        }
    }
}

// One fused pass over the state.  `p` carries the data of the launch
// (buffers, tile count, grid stride, rank bits, coefficients); `S` carries
// the pass's STRUCTURE (tile bits, phases, gate records, permutations).  The
// AOT kernel passes the same object for both and interprets the structure;
// a runtime-specialised kernel (fused_jit.cu) binds S to a constant copy, so
// every loop over phases and gates unrolls and every branch on the gate
// records folds at compile time -- same arithmetic, same order, no decode.
template <int R, int MODE, int TB = kThreadBits>
__device__ __forceinline__ void tile_pass_body(const TileParams &p, const TileParams &S) {
    // dynamic smem: nbuf tiles, then the row-offset table, then (gperm) the
    // global-map table -- sized by T, so small tiles leave room for 3 CTAs
    extern __shared__ double2 tile[];
    const int T = S.tbits;
    const uint32_t tsize = 1u << T;
    uint64_t *hi_off = (uint64_t *)(tile + ((size_t)p.nbuf << T));
    uint64_t *s_ghi = hi_off + (tsize >> kLowBits);  // global map of each tile row offset
    // per-(phase, thread) index part of the thread bits, computed once per
    // CTA instead of once per tile (register parts ride in the phase record)
    constexpr int kPre = kPrePhases;
    constexpr int NT = 1 << TB;  // threads
    __shared__ uint16_t s_tpart[kPre][NT];
    __shared__ uint16_t s_pt[kPre][NT];  // folded permutations: swizzled image of the thread part
    __shared__ uint16_t s_lt[NT];
    __shared__ uint16_t s_lk[1 << (kMaxTileBits - TB)];
    __shared__ uint64_t s_sbase;  // current tile's base | rank bits (selector lookups)
    constexpr int NR = 1 << R;
    const double2 *sc = p.coef;
    const uint32_t *snz = p.nz;
    // tile element e -> state offset: low kLowBits tile bits are state bits 0..2
    for (uint32_t h = threadIdx.x; h < (tsize >> kLowBits); h += blockDim.x) {
        uint64_t off = 0;
        DIAQ_SUNROLL
        for (int j = kLowBits; j < T; ++j) off |= (uint64_t)((h >> (j - kLowBits)) & 1u) << S.tb[j];
        hi_off[h] = off;
    }
    __syncthreads();
    constexpr uint32_t lowmask = (1u << kLowBits) - 1u;
    const int npre = S.nphases < kPre ? S.nphases : kPre;
    DIAQ_SUNROLL
    for (int ph_i = 0; ph_i < npre; ++ph_i) {
        const Phase &ph = S.ph[ph_i];
        uint32_t tpart = 0;
        DIAQ_SUNROLL
        for (int i = 0; i < T - R; ++i) tpart |= ((threadIdx.x >> i) & 1u) << ph.tpos[i];
        s_tpart[ph_i][threadIdx.x] = (uint16_t)tpart;
        if (ph.post.on) s_pt[ph_i][threadIdx.x] = (uint16_t)swz(aff_lin(ph.post, tpart, T));
    }
    if (S.pre.on) {
        s_lt[threadIdx.x] = (uint16_t)swz(aff_lin(S.pre, threadIdx.x, T));
        if (threadIdx.x < (tsize >> TB)) s_lk[threadIdx.x] = (uint16_t)swz(aff_lin(S.pre, threadIdx.x << TB, T));
    }
    __shared__ uint64_t glo[1 << kLowBits];  // global map of the in-row offsets
#ifdef DIAQ_JIT
    // pair store (see TileParams::gnp): destination offsets / sources of the
    // high enumeration bits (uniform table) and of this thread's low bits
    const bool pairing = S.gnp > 0;
    __shared__ uint64_t s_pw[1 << (kMaxTileBits + 1 - TB)];
    __shared__ uint16_t s_ps[1 << (kMaxTileBits + 1 - TB)];
    uint64_t pw_t = 0;
    uint32_t ps_t = 0;
    if (pairing) {
        const int dims = T + S.gnp;
        DIAQ_SUNROLL
        for (int k = 0; k < TB; ++k)
            if ((threadIdx.x >> k) & 1u) {
                pw_t ^= S.gw[k];
                ps_t ^= S.gsrc[k];
            }
        if (threadIdx.x < (1u << (dims - TB))) {
            uint64_t w = 0;
            uint32_t sr = 0;
            DIAQ_SUNROLL
            for (int k = TB; k < dims; ++k)
                if ((threadIdx.x >> (k - TB)) & 1u) {
                    w ^= S.gw[k];
                    sr ^= S.gsrc[k];
                }
            s_pw[threadIdx.x] = w;
            s_ps[threadIdx.x] = (uint16_t)sr;
        }
    }
#else
    constexpr bool pairing = false;
#endif
    if (S.gperm && !pairing) {
        for (uint32_t h = threadIdx.x; h < (tsize >> kLowBits); h += blockDim.x) {
            uint64_t o = hi_off[h], r = 0;
            while (o) {
                r ^= p.gcol[__ffsll((long long)o) - 1];
                o &= o - 1;
            }
            s_ghi[h] = r;
        }
        if (threadIdx.x < (1u << kLowBits)) {
            uint64_t r = 0;
            for (int b = 0; b < kLowBits; ++b)
                if ((threadIdx.x >> b) & 1u) r ^= p.gcol[b];
            glo[threadIdx.x] = r;
        }
    }
    // HBM -> smem with cp.async, coalesced (consecutive e are consecutive
    // state indices in runs of 8); every element of the tile in flight at once
    auto fetch = [&](uint64_t b, double2 *buf) {
        const uint64_t pol = policy_evict_first();
        if (S.pre.on) {  // element e lands in the slot of its relabelled index
            const uint32_t lt = s_lt[threadIdx.x] ^ swz(aff_const(S.pre, b | p.gbase));
        #pragma unroll 1
            for (int k = 0; k < NR; ++k) {
                const uint32_t e = threadIdx.x + ((uint32_t)k << TB);
#ifdef DIAQ_JIT
                // (ptxas 12.9 emitted a malformed LDGSTS for the policy form of
                // this permuted-slot copy in specialised kernels: illegal
                // instruction at run time; the plain form is used here)
                cp_async16_nohint(buf + (lt ^ s_lk[k]), p.x + b + (e & lowmask) + hi_off[e >> kLowBits]);
#else
                cp_async16(buf + (lt ^ s_lk[k]), p.x + b + (e & lowmask) + hi_off[e >> kLowBits], pol);
#endif
            }
        } else {
        #pragma unroll 1
            for (int k = 0; k < NR; ++k) {
                const uint32_t e = threadIdx.x + ((uint32_t)k << TB);
                cp_async16(buf + swz(e), p.x + b + (e & lowmask) + hi_off[e >> kLowBits], pol);
            }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    __syncthreads();
    // one tile's phases, in place in its smem buffer (s_sbase: the tile's
    // full-state base, written by the caller before the barrier it passes)
    auto phases = [&](double2 *tl) {
        DIAQ_SUNROLL
        for (int ph_i = 0; ph_i < S.nphases; ++ph_i) {
            const Phase &ph = S.ph[ph_i];
            if (ph.generic) {
                DIAQ_SUNROLL
                for (int gi = ph.g0; gi < ph.g1; ++gi) {
                    smem_gate<MODE>(tl, T, S.g[gi], ld_base(&s_sbase), sc, snz);
                    __syncthreads();
                }
                continue;
            }
            double2 v[NR];
            uint32_t tpart;
            if (ph_i < kPre) {
                tpart = s_tpart[ph_i][threadIdx.x];
            } else {
                tpart = 0;
                DIAQ_SUNROLL
                for (int i = 0; i < T - R; ++i) tpart |= ((threadIdx.x >> i) & 1u) << ph.tpos[i];
            }
            const uint32_t tsw = swz(tpart);
#pragma unroll
            for (int j = 0; j < NR; ++j) v[j] = tl[tsw ^ ph.pj[j]];
            if (ph.seq) {
                int gi = ph.g0;
                seq_steps<R, MODE, 0>(v, S, ph, gi, tpart, &s_sbase, sc, snz);
                diag_run<R, MODE>(v, S, gi, ph.nd_before[R], tpart, &s_sbase, sc, snz);
            } else {
                // leading diagonals on non-register bits (nd_before[0] of them): one folded factor
                // under the contracted arithmetic, gate by gate otherwise (diag_run)
                int gd = ph.g0;
                diag_run<R, MODE>(v, S, gd, ph.nd_before[0], tpart, &s_sbase, sc, snz);
                DIAQ_SUNROLL
                for (int gi = ph.g0 + ph.nd_before[0]; gi < ph.g1; ++gi)
                    dispatch_gate<R, MODE>(v, S.g[gi], tpart, &s_sbase, sc, snz);
            }
            if (ph.post.on) {
                __syncthreads();  // relabelled slots belong to other threads' registers: all reads first
                const uint32_t bc = swz(aff_const(ph.post, ld_base(&s_sbase)));
                const uint32_t pt = (ph_i < kPre ? (uint32_t)s_pt[ph_i][threadIdx.x] : swz(aff_lin(ph.post, tpart, T))) ^ bc;
#pragma unroll
                for (int j = 0; j < NR; ++j) tl[pt ^ ph.ppj[j]] = v[j];
            } else {
#pragma unroll
                for (int j = 0; j < NR; ++j) tl[tsw ^ ph.pj[j]] = v[j];
            }
            __syncthreads();
        }
    };
#ifdef DIAQ_JIT
    if (pairing) {
        // Pair store: the tile and its partner across the extra bit gpb[0]
        // run in one CTA (both smem buffers), then every destination sector
        // (row) of the pair is written whole, gathered from the two buffers.
        // Units are pairs; their bases enumerate the bits outside emask.
        const uint64_t pbit = 1ull << S.gpb[0];
        const int64_t nunits = p.ntiles >> 1;
        uint64_t gb = insert_zero_bits_dyn((uint64_t)blockIdx.x, S.eb, T + 1);
        if ((int64_t)blockIdx.x < nunits) {
            fetch(gb, tile);
            fetch(gb | pbit, tile + ((size_t)1 << T));
        }
        for (int64_t t = blockIdx.x; t < nunits; t += gridDim.x) {
            const uint64_t ngb = ((gb | S.emask) + p.gstep) & ~S.emask;
            asm volatile("cp.async.wait_group 0;" ::: "memory");
        #pragma unroll 1
            for (int h = 0; h < 2; ++h) {
                if (threadIdx.x == 0) s_sbase = (gb | (h ? pbit : 0ull)) | p.gbase;
                __syncthreads();
                phases(tile + ((size_t)h << T));
            }
            __syncthreads();
            uint64_t ab = p.gconst, o = gb;
            while (o) {
                ab ^= p.gcol[__ffsll((long long)o) - 1];
                o &= o - 1;
            }
        #pragma unroll 4
            for (int i = 0; i < 2 * NR; ++i) {
                const uint32_t src = ps_t ^ s_ps[i];
                st_stream(p.y + (ab ^ pw_t ^ s_pw[i]), tile[((size_t)(src >> 12) << T) + swz(src & 0xfffu)]);
            }
            __syncthreads();
            gb = ngb;
            if (t + gridDim.x < nunits) {
                fetch(gb, tile);
                fetch(gb | pbit, tile + ((size_t)1 << T));
            }
        }
        return;
    }
#endif
    // nbuf 2: the next tile streams into the other buffer while this one is
    // computed (its latency hidden inside the CTA); nbuf 1: refill after the
    // store, latency hidden only by the other resident CTAs
    uint64_t base = insert_zero_bits_dyn((uint64_t)blockIdx.x, S.tb, T);
    if ((int64_t)blockIdx.x < p.ntiles) fetch(base, tile);
    int buf = 0;
    for (int64_t t = blockIdx.x; t < p.ntiles; t += gridDim.x) {
        const uint64_t nbase = next_base(base, p, S);
        const bool more = t + gridDim.x < p.ntiles;
        double2 *tl = tile + ((size_t)buf << T);
        if (threadIdx.x == 0) s_sbase = base | p.gbase;  // full-state index bits for selectors
        if (p.nbuf == 2 && more) {
            fetch(nbase, tile + ((size_t)(buf ^ 1) << T));
            asm volatile("cp.async.wait_group 1;" ::: "memory");
        } else {
            asm volatile("cp.async.wait_group 0;" ::: "memory");
        }
        __syncthreads();
        phases(tl);
        if (S.gperm) {  // trailing permutation run: element i goes to A i ^ c in the other buffer
            uint64_t ab = p.gconst, o = base;
            while (o) {
                ab ^= p.gcol[__ffsll((long long)o) - 1];
                o &= o - 1;
            }
        #pragma unroll 1
            for (int k = 0; k < NR; ++k) {
                const uint32_t e = threadIdx.x + ((uint32_t)k << TB);
                double2 *dst = p.y + (ab ^ s_ghi[e >> kLowBits] ^ glo[e & lowmask]);
                if (p.gstore == 0) st_stream(dst, tl[swz(e)]);
                else if (p.gstore == 1) st_plain(dst, tl[swz(e)]);
                else st_hint(dst, tl[swz(e)], policy_evict_last());
            }
        } else {
        #pragma unroll 1
            for (int k = 0; k < NR; ++k) {
                const uint32_t e = threadIdx.x + ((uint32_t)k << TB);
                st_stream(p.y + base + (e & lowmask) + hi_off[e >> kLowBits], tl[swz(e)]);
            }
        }
        __syncthreads();
        base = nbase;
        if (p.nbuf == 2) buf ^= 1;
        else if (more) fetch(base, tile);  // refill as soon as the tile is drained
    }
}

#ifdef DIAQ_JIT
// ---- specialised pass body (NVRTC; the structure S is a compile-time constant) --
//
// Same schedule, arithmetic and results as tile_pass_body; what changes is the
// address arithmetic, which the profile of the interpreted form put at about
// half of the pass's non-FP64 instructions and a third of its stall samples
// (r02b: the tile load/store loops waited on a shared-memory offset table):
//   * tile element e = tid + 256 k lies at state offset
//       b + (tid & 7) + dep(tid >> 3) + dep(32 k)
//     (dep deposits row bits into the tile's state bits): the thread part is
//     computed once per kernel, the k part is a constant of the pass, so a
//     tile load/store costs one 64-bit add per element -- no table lookups;
//   * the tile buffers are 1024-byte aligned, so for a slot s = sh | sl
//     (sl its low three bits) and a per-phase thread part T = th | tl whose
//     high bits are disjoint from sh, the byte address base + 16 (T ^ s) is
//     (base + 16 T) ^ 16 sl + 16 sh: one LOP3, and the rest is the load's
//     immediate offset.

__device__ __forceinline__ double2 lds128(uint32_t a) {
    double2 v;
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a) : "memory");
    return v;
}

__device__ __forceinline__ void sts128(uint32_t a, double2 v) {
    asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(a), "d"(v.x), "d"(v.y) : "memory");
}

__device__ __forceinline__ void cp_async16_s(uint32_t dst, const void *src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}

// byte address of slot s relative to a 128-byte aligned t16 = base + 16 T
// whose high part is disjoint from s's (see above)
__device__ __forceinline__ uint32_t slot_addr(uint32_t t16, uint32_t s) {
    return (t16 ^ ((s & 7u) << 4)) + ((s & ~7u) << 4);
}

// state offset of tile rows h (bits of h -> tile bits 3.. of S)
__device__ __forceinline__ uint64_t row_dep(const TileParams &S, uint32_t h) {
    uint64_t off = 0;
#pragma unroll
    for (int j = kLowBits; j < kMaxTileBits; ++j)
        if (j < S.tbits) off |= (uint64_t)((h >> (j - kLowBits)) & 1u) << S.tb[j];
    return off;
}

// image of state offset o under the global permutation map (columns S.gcol)
__device__ __forceinline__ uint64_t gmap(const TileParams &S, uint64_t o) {
    uint64_t r = 0;
#pragma unroll
    for (int j = 0; j < 64; ++j)
        if ((o >> j) & 1ull) r ^= S.gcol[j];
    return r;
}

template <int R, int MODE>
__device__ __forceinline__ void tile_pass_body_jit(const TileParams &p, const TileParams &S) {
    extern __shared__ __align__(1024) double2 tile[];
    const int T = S.tbits;
    const int TB = T - R;  // thread bits: 2^TB threads (a constant of the pass)
    constexpr int NR = 1 << R;
    constexpr uint32_t lowmask = (1u << kLowBits) - 1u;
    const uint32_t tid = threadIdx.x;
    const uint32_t tile0 = smem_u32(tile);
    constexpr int kPre = kPrePhases;
    __shared__ uint16_t s_t16[kPre][kThreads];  // 16 * swz(tpart) per phase (T <= 12: fits 16 bits)
    __shared__ uint16_t s_pt[kPre][kThreads];   // folded permutations: swizzled image of the thread part
    __shared__ uint16_t s_lt[kThreads];
    __shared__ uint64_t s_sbase;  // current tile's base | rank bits (selector lookups)
    __shared__ uint64_t s_ab;     // global-map image of the current tile / pair base
    __shared__ int64_t s_u[2];    // dynamic unit order: the next unit, double-buffered by parity
    const double2 *sc = p.coef;
    const uint32_t *snz = p.nz;
    const int npre = S.nphases < kPre ? S.nphases : kPre;
    DIAQ_SUNROLL
    for (int ph_i = 0; ph_i < npre; ++ph_i) {
        const Phase &ph = S.ph[ph_i];
        uint32_t tpart = 0;
        DIAQ_SUNROLL
        for (int i = 0; i < TB; ++i) tpart |= ((tid >> i) & 1u) << ph.tpos[i];
        s_t16[ph_i][tid] = (uint16_t)(swz(tpart) << 4);
        if (ph.post.on) s_pt[ph_i][tid] = (uint16_t)swz(aff_lin(ph.post, tpart, T));
    }
    if (S.pre.on) s_lt[tid] = (uint16_t)swz(aff_lin(S.pre, tid, T));
    // element k of this thread: state offset base + t_off + kdep(k)
    const uint64_t t_off = (tid & lowmask) + row_dep(S, tid >> kLowBits);
    auto kdep = [&](int k) -> uint64_t { return row_dep(S, (uint32_t)k << (TB - kLowBits)); };
    const uint32_t t16 = swz(tid) << 4;
    auto fetch = [&](uint64_t b, uint32_t buf) {
        const double2 *src = p.x + (b + t_off);
        if (S.pre.on) {  // element e lands in the slot of its relabelled index
            const uint32_t lt = s_lt[tid] ^ swz(aff_const(S.pre, b | p.gbase));
#pragma unroll
            for (int k = 0; k < NR; ++k)
                cp_async16_s(buf + ((lt ^ swz(aff_lin(S.pre, (uint32_t)k << TB, T))) << 4), src + kdep(k));
        } else {
            const uint32_t a = buf + t16;
#pragma unroll
            for (int k = 0; k < NR; ++k) cp_async16_s(slot_addr(a, swz((uint32_t)k << TB)), src + kdep(k));
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    // dynamic unit order (p.uctr): the first unit, and the end-of-pass reset
    auto first_unit = [&]() -> int64_t {
        if (!p.uctr) return (int64_t)blockIdx.x;
        if (tid == 0) s_u[0] = (int64_t)atomicAdd(p.uctr, 1ull);
        __syncthreads();
        return s_u[0];
    };
    auto units_done = [&]() {
        if (!p.uctr) return;
        __syncthreads();
        if (tid == 0) {
            __threadfence();
            if (atomicAdd(p.udone, 1ull) == (unsigned long long)gridDim.x - 1ull) {
                *p.uctr = 0ull;
                *p.udone = 0ull;
                __threadfence();
            }
        }
    };
    __syncthreads();
    // dbase / on_loaded: with S.dstore the last phase writes its registers
    // straight to y + dbase (no smem round trip), and on_loaded() runs once
    // every thread has read its last-phase registers (the tile buffers are
    // free from then on: the next unit's fetch can start under the compute)
    auto phases = [&](uint32_t buf, uint64_t dbase, auto &&on_loaded) {
        double2 *tl = tile + ((buf - tile0) >> 4);
        DIAQ_SUNROLL
        for (int ph_i = 0; ph_i < S.nphases; ++ph_i) {
            const Phase &ph = S.ph[ph_i];
            const bool direct = S.dstore && ph_i == S.nphases - 1;
            if (ph.generic) {
                DIAQ_SUNROLL
                for (int gi = ph.g0; gi < ph.g1; ++gi) {
                    smem_gate<MODE>(tl, T, S.g[gi], ld_base(&s_sbase), sc, snz);
                    __syncthreads();
                }
                continue;
            }
            double2 v[NR];
            // thread part of the phase's slots (dead code unless a selector or
            // a folded store needs it; the address comes from the table)
            uint32_t tpart = 0;
            DIAQ_SUNROLL
            for (int i = 0; i < TB; ++i) tpart |= ((tid >> i) & 1u) << ph.tpos[i];
            const uint32_t a = buf + (ph_i < kPre ? (uint32_t)s_t16[ph_i][tid] : (swz(tpart) << 4));
#pragma unroll
            for (int j = 0; j < NR; ++j) v[j] = lds128(slot_addr(a, ph.pj[j]));
            if (direct) {
                __syncthreads();  // every thread holds its registers: the buffers are free
                on_loaded();
            }
            if (ph.seq) {
                int gi = ph.g0;
                seq_steps<R, MODE, 0>(v, S, ph, gi, tpart, &s_sbase, sc, snz);
                diag_run<R, MODE>(v, S, gi, ph.nd_before[R], tpart, &s_sbase, sc, snz);
            } else {
                // leading diagonals on non-register bits (nd_before[0] of them): one folded factor
                // under the contracted arithmetic, gate by gate otherwise (diag_run)
                int gd = ph.g0;
                diag_run<R, MODE>(v, S, gd, ph.nd_before[0], tpart, &s_sbase, sc, snz);
                DIAQ_SUNROLL
                for (int gi = ph.g0 + ph.nd_before[0]; gi < ph.g1; ++gi)
                    dispatch_gate<R, MODE>(v, S.g[gi], tpart, &s_sbase, sc, snz);
            }
            if (direct) {
                // register j of this thread = tile position tpart | e_j: state
                // offset dep(tpart) + dep(e_j), the latter a constant
                uint64_t toff = 0;
                DIAQ_SUNROLL
                for (int i = 0; i < TB; ++i) toff |= (uint64_t)((tid >> i) & 1u) << S.tb[ph.tpos[i]];
                double2 *dst = p.y + (dbase + toff);
#pragma unroll
                for (int j = 0; j < NR; ++j) {
                    uint64_t roff = 0;
#pragma unroll
                    for (int q = 0; q < R; ++q)
                        if ((j >> q) & 1) roff |= 1ull << S.tb[ph.rpos[q]];
                    st_stream(dst + roff, v[j]);
                }
            } else if (ph.post.on) {
                __syncthreads();  // relabelled slots belong to other threads' registers: all reads first
                const uint32_t bc = swz(aff_const(ph.post, ld_base(&s_sbase)));
                const uint32_t pt = (ph_i < kPre ? (uint32_t)s_pt[ph_i][tid] : swz(aff_lin(ph.post, tpart, T))) ^ bc;
#pragma unroll
                for (int j = 0; j < NR; ++j) sts128(buf + ((pt ^ ph.ppj[j]) << 4), v[j]);
            } else {
#pragma unroll
                for (int j = 0; j < NR; ++j) sts128(slot_addr(a, ph.pj[j]), v[j]);
            }
            __syncthreads();
        }
    };
    if (S.gnp > 0) {
        // Pair store (see TileParams::gnp): the tile and its partner across
        // gpb[0] in both buffers, every destination sector written whole.
        // Destination / source of pair element i = tid + 256 m: pw_t ^ gw(m),
        // ps_t ^ gsrc(m) with the m parts constants of the pass.
        const int dims = T + S.gnp;
        uint64_t pw_t = 0;
        uint32_t ps_t = 0;
#pragma unroll
        for (int k = 0; k < TB; ++k)
            if ((tid >> k) & 1u) {
                pw_t ^= S.gw[k];
                ps_t ^= S.gsrc[k];
            }
        // smem slot of a source (tile offset | half << 12), linear over GF(2)
        auto pslot = [&](uint32_t src) -> uint32_t { return ((src >> 12) << T) ^ swz(src & 0xfffu); };
        const uint32_t ps_slot = pslot(ps_t);
        const uint64_t pbit = 1ull << S.gpb[0];
        const int64_t nunits = p.ntiles >> 1;
        const uint32_t buf1 = tile0 + (16u << T);
        const bool dyn = p.uctr && p.estore;
        const int64_t u0 = dyn ? first_unit() : (int64_t)blockIdx.x;
        uint64_t gb = insert_zero_bits_dyn((uint64_t)u0, S.eb, T + 1);
        if (u0 < nunits) {
            fetch(gb, tile0);
            fetch(gb | pbit, buf1);
        }
        int par = 1;
        for (int64_t t = u0; t < nunits; t += gridDim.x) {
            const uint64_t ngb = ((gb | S.emask) + p.gstep) & ~S.emask;
            if (dyn && tid == 0) s_u[par] = (int64_t)atomicAdd(p.uctr, 1ull);  // lands during the compute
            asm volatile("cp.async.wait_group 0;" ::: "memory");
#pragma unroll 1
            for (int h = 0; h < 2; ++h) {
                if (tid == 0) {
                    s_sbase = (gb | (h ? pbit : 0ull)) | p.gbase;
                    if (h == 0) s_ab = p.gconst ^ gmap(S, gb);
                }
                __syncthreads();
                phases(h ? buf1 : tile0, 0ull, [] {});
            }
            __syncthreads();
            const uint64_t ab = s_ab ^ pw_t;
            if (p.estore) {
                // the whole store gathered into registers first: the tile
                // buffers are free before any HBM write, so the next unit's
                // fetch is in flight while this unit's stores drain
                constexpr int NS = 2 * NR;
                double2 sv[NS];
#pragma unroll
                for (int i = 0; i < NS; ++i) {
                    if (i >= (1 << (dims - TB))) break;
                    uint32_t cs = 0;
#pragma unroll
                    for (int m = 0; m < dims - TB; ++m)
                        if ((i >> m) & 1) cs ^= S.gsrc[TB + m];
                    sv[i] = lds128(tile0 + ((ps_slot ^ pslot(cs)) << 4));
                }
                __syncthreads();
                int64_t nt = t + gridDim.x;
                if (dyn) {
                    nt = s_u[par];
                    par ^= 1;
                    gb = insert_zero_bits_dyn((uint64_t)nt, S.eb, T + 1);
                    t = nt - gridDim.x;  // the loop increment lands on nt
                } else {
                    gb = ngb;
                }
                if (nt < nunits) {
                    fetch(gb, tile0);
                    fetch(gb | pbit, buf1);
                }
#pragma unroll
                for (int i = 0; i < NS; ++i) {
                    if (i >= (1 << (dims - TB))) break;
                    uint64_t cw = 0;
#pragma unroll
                    for (int m = 0; m < dims - TB; ++m)
                        if ((i >> m) & 1) cw ^= S.gw[TB + m];
                    st_stream(p.y + (ab ^ cw), sv[i]);
                }
                continue;
            }
#pragma unroll
            for (int i = 0; i < 2 * NR; ++i) {
                if (i >= (1 << (dims - TB))) break;
                uint64_t cw = 0;
                uint32_t cs = 0;
#pragma unroll
                DIAQ_SUNROLL
                for (int m = 0; m < dims - TB; ++m)
                    if ((i >> m) & 1) {
                        cw ^= S.gw[TB + m];
                        cs ^= S.gsrc[TB + m];
                    }
                st_stream(p.y + (ab ^ cw), lds128(tile0 + ((ps_slot ^ pslot(cs)) << 4)));
            }
            __syncthreads();
            gb = ngb;
            if (t + gridDim.x < nunits) {
                fetch(gb, tile0);
                fetch(gb | pbit, buf1);
            }
        }
        if (dyn) units_done();
        return;
    }
    if (S.ppair && S.ppipe == 3) {
        // Plain pair across a CTA pair (thread-block cluster of 2): CTA rank h
        // owns half h of every pair unit.  Both CTAs pass a cluster barrier
        // before each fetch, so the two halves of every 256-byte DRAM run are
        // requested together (the locality of the one-CTA pair) while each
        // CTA holds one tile (32 KB) -- more resident CTAs per SM to hide the
        // fetch latency.
        uint32_t half;
        asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(half));
        const uint64_t hb = half ? (1ull << S.gpb[0]) : 0ull;
        const int64_t nunits = p.ntiles >> 1;
        const int64_t u0 = blockIdx.x >> 1, ustep = gridDim.x >> 1;
        const uint32_t a = tile0 + t16;
        uint64_t gb = insert_zero_bits_dyn((uint64_t)u0, S.eb, T + 1);
        for (int64_t t = u0; t < nunits; t += ustep) {
            const uint64_t ngb = ((gb | S.emask) + p.gstep) & ~S.emask;
            cluster_sync();
            fetch(gb | hb, tile0);
            if (tid == 0) s_sbase = (gb | hb) | p.gbase;
            asm volatile("cp.async.wait_group 0;" ::: "memory");
            __syncthreads();
            phases(tile0, 0ull, [] {});
            double2 *dst = p.y + ((gb | hb) + t_off);
#pragma unroll
            for (int k = 0; k < NR; ++k) st_stream(dst + kdep(k), lds128(slot_addr(a, swz((uint32_t)k << TB))));
            __syncthreads();
            gb = ngb;
        }
        cluster_sync();  // no CTA of a cluster exits while its partner may still arrive
        return;
    }
    if (S.ppair) {
        const uint64_t pbit = 1ull << S.gpb[0];
        const int64_t nunits = p.ntiles >> 1;
        const uint32_t buf1 = tile0 + (16u << T);
        const uint32_t a0 = tile0 + t16, a1 = buf1 + t16;
        // both halves' elements k interleaved: adjacent 128-byte rows in flight together
        auto fetch2 = [&](uint64_t b) {
            const double2 *src = p.x + (b + t_off);
            if (S.pre.on) {  // a permutation run opens the pass: each half lands relabelled (as fetch())
                const uint32_t lt0 = s_lt[tid] ^ swz(aff_const(S.pre, b | p.gbase));
                const uint32_t lt1 = s_lt[tid] ^ swz(aff_const(S.pre, (b | pbit) | p.gbase));
#pragma unroll
                for (int k = 0; k < NR; ++k) {
                    const uint32_t kl = swz(aff_lin(S.pre, (uint32_t)k << TB, T));
                    cp_async16_s(tile0 + ((lt0 ^ kl) << 4), src + kdep(k));
                    cp_async16_s(buf1 + ((lt1 ^ kl) << 4), src + (kdep(k) | pbit));
                }
                asm volatile("cp.async.commit_group;" ::: "memory");
                return;
            }
#pragma unroll
            for (int k = 0; k < NR; ++k) {
                const uint32_t sl = swz((uint32_t)k << TB);
                cp_async16_s(slot_addr(a0, sl), src + kdep(k));
                cp_async16_s(slot_addr(a1, sl), src + (kdep(k) | pbit));
            }
            asm volatile("cp.async.commit_group;" ::: "memory");
        };
        auto fetch1 = [&](uint64_t b, uint32_t a) {  // one half (its base b, buffer address a + t16), its own commit group
            if (S.pre.on) {
                fetch(b, a - t16);
                return;
            }
            const double2 *src = p.x + (b + t_off);
#pragma unroll
            for (int k = 0; k < NR; ++k) cp_async16_s(slot_addr(a, swz((uint32_t)k << TB)), src + kdep(k));
            asm volatile("cp.async.commit_group;" ::: "memory");
        };
        auto store1 = [&](uint64_t b, uint32_t a) {
            double2 *dst = p.y + (b + t_off);
#pragma unroll
            for (int k = 0; k < NR; ++k) st_stream(dst + kdep(k), lds128(slot_addr(a, swz((uint32_t)k << TB))));
        };
        uint64_t gb = insert_zero_bits_dyn((uint64_t)blockIdx.x, S.eb, T + 1);
        if (S.ppipe) {
            if ((int64_t)blockIdx.x < nunits) {
                fetch1(gb, a0);
                fetch1(gb | pbit, a1);
            }
            for (int64_t t = blockIdx.x; t < nunits; t += gridDim.x) {
                const uint64_t ngb = ((gb | S.emask) + p.gstep) & ~S.emask;
                const bool more = t + gridDim.x < nunits;
                asm volatile("cp.async.wait_group 1;" ::: "memory");  // half A landed (B may still fly)
                if (tid == 0) s_sbase = gb | p.gbase;
                __syncthreads();
                phases(tile0, 0ull, [] {});
                if (S.ppipe == 2) {  // A leaves now; its buffer takes the next A while B computes
                    store1(gb, a0);
                    __syncthreads();
                    if (more) fetch1(ngb, a0);
                    else asm volatile("cp.async.commit_group;" ::: "memory");  // keep the group count
                    asm volatile("cp.async.wait_group 1;" ::: "memory");      // half B landed
                } else {
                    asm volatile("cp.async.wait_group 0;" ::: "memory");
                }
                if (tid == 0) s_sbase = (gb | pbit) | p.gbase;
                __syncthreads();
                phases(buf1, 0ull, [] {});
                if (S.ppipe == 2) {
                    store1(gb | pbit, a1);
                    __syncthreads();
                    if (more) fetch1(ngb | pbit, a1);
                } else {
                    double2 *dst = p.y + (gb + t_off);
#pragma unroll
                    for (int k = 0; k < NR; ++k) {
                        const uint32_t sl = swz((uint32_t)k << TB);
                        st_stream(dst + kdep(k), lds128(slot_addr(a0, sl)));
                        st_stream(dst + (kdep(k) | pbit), lds128(slot_addr(a1, sl)));
                    }
                    __syncthreads();
                    if (more) {
                        fetch1(ngb, a0);
                        fetch1(ngb | pbit, a1);
                    }
                }
                gb = ngb;
            }
            return;
        }
        if (S.dstore) {  // both halves store from registers; the next pair lands under B's last phase
            if ((int64_t)blockIdx.x < nunits) fetch2(gb);
            for (int64_t t = blockIdx.x; t < nunits; t += gridDim.x) {
                const uint64_t ngb = ((gb | S.emask) + p.gstep) & ~S.emask;
                const bool more = t + gridDim.x < nunits;
                asm volatile("cp.async.wait_group 0;" ::: "memory");
#pragma unroll 1
                for (int h = 0; h < 2; ++h) {  // one copy of the phase code for both halves
                    const uint64_t hb = gb | (h ? pbit : 0ull);
                    if (tid == 0) s_sbase = hb | p.gbase;
                    __syncthreads();
                    phases(h ? buf1 : tile0, hb, [&] {
                        if (h && more) fetch2(ngb);
                    });
                }
                gb = ngb;
            }
            return;
        }
        // One loop for both unit orders (one copy of the phase code per
        // kernel: the unrolled gate program is most of its text): static
        // (unit t + gridDim.x next) or dynamic (p.uctr: units handed out in
        // order by a global counter, see TileParams::uctr).
        const bool dyn = p.uctr && p.estore;
        int64_t t = dyn ? first_unit() : (int64_t)blockIdx.x;
        gb = insert_zero_bits_dyn((uint64_t)t, S.eb, T + 1);
        if (t < nunits) fetch2(gb);
        int par = 1;
        while (t < nunits) {
            if (dyn && tid == 0) s_u[par] = (int64_t)atomicAdd(p.uctr, 1ull);  // lands during the compute
            asm volatile("cp.async.wait_group 0;" ::: "memory");
#pragma unroll 1
            for (int h = 0; h < 2; ++h) {
                if (tid == 0) s_sbase = (gb | (h ? pbit : 0ull)) | p.gbase;
                __syncthreads();
                phases(h ? buf1 : tile0, 0ull, [] {});
            }
            const uint64_t cgb = gb;
            if (p.estore) {  // gather to registers, fetch the next pair, then store (see the pair store)
                double2 sa[NR], sb[NR];
#pragma unroll
                for (int k = 0; k < NR; ++k) {
                    const uint32_t sl = swz((uint32_t)k << TB);
                    sa[k] = lds128(slot_addr(a0, sl));
                    sb[k] = lds128(slot_addr(a1, sl));
                }
                __syncthreads();
                t = dyn ? s_u[par] : t + gridDim.x;
                par ^= 1;
                gb = insert_zero_bits_dyn((uint64_t)t, S.eb, T + 1);
                if (t < nunits) fetch2(gb);
                double2 *dst = p.y + (cgb + t_off);
#pragma unroll
                for (int k = 0; k < NR; ++k) {
                    st_stream(dst + kdep(k), sa[k]);
                    st_stream(dst + (kdep(k) | pbit), sb[k]);
                }
                continue;
            }
            double2 *dst = p.y + (cgb + t_off);
#pragma unroll
            for (int k = 0; k < NR; ++k) {
                const uint32_t sl = swz((uint32_t)k << TB);
                st_stream(dst + kdep(k), lds128(slot_addr(a0, sl)));
                st_stream(dst + (kdep(k) | pbit), lds128(slot_addr(a1, sl)));
            }
            __syncthreads();
            t += gridDim.x;
            gb = insert_zero_bits_dyn((uint64_t)t, S.eb, T + 1);
            if (t < nunits) fetch2(gb);
        }
        if (dyn) units_done();
        return;
    }
    // gperm scatter store: element e -> gconst ^ G(base) ^ G(t_off) ^ G(kdep(k))
    const uint64_t g_t = S.gperm ? gmap(S, t_off) : 0ull;
    // one loop for both unit orders, as above (dynamic order: one buffer, estore)
    const bool dyn = p.uctr && p.estore && p.nbuf == 1;
    int64_t t = dyn ? first_unit() : (int64_t)blockIdx.x;
    uint64_t base = insert_zero_bits_dyn((uint64_t)t, S.tb, T);
    if (t < p.ntiles) fetch(base, tile0);
    uint32_t buf = tile0;
    const uint32_t tstride = 16u << T;
    int par = 1;
    while (t < p.ntiles) {
        const int64_t nt = t + gridDim.x;  // static order
        if (tid == 0) {
            if (dyn) s_u[par] = (int64_t)atomicAdd(p.uctr, 1ull);  // lands during the compute
            s_sbase = base | p.gbase;  // full-state index bits for selectors
            if (S.gperm) s_ab = p.gconst ^ gmap(S, base);
        }
        if (p.nbuf == 2 && nt < p.ntiles) {
            fetch(insert_zero_bits_dyn((uint64_t)nt, S.tb, T), buf == tile0 ? tile0 + tstride : tile0);
            asm volatile("cp.async.wait_group 1;" ::: "memory");
        } else {
            asm volatile("cp.async.wait_group 0;" ::: "memory");
        }
        __syncthreads();
        phases(buf, 0ull, [] {});
        const uint32_t a = buf + t16;
        if (p.estore && p.nbuf == 1) {
            // one buffer: gather this tile's store into registers, refill the
            // buffer with the next tile, then write -- the fetch is in flight
            // during the HBM writes instead of after them
            double2 sv[NR];
#pragma unroll
            for (int k = 0; k < NR; ++k) sv[k] = lds128(slot_addr(a, swz((uint32_t)k << TB)));
            const uint64_t ab = S.gperm ? (s_ab ^ g_t) : 0ull;
            __syncthreads();
            const uint64_t cbase = base;
            t = dyn ? s_u[par] : nt;
            par ^= 1;
            base = insert_zero_bits_dyn((uint64_t)t, S.tb, T);
            if (t < p.ntiles) fetch(base, buf);
            if (S.gperm) {
#pragma unroll
                for (int k = 0; k < NR; ++k) {
                    double2 *dst = p.y + (ab ^ gmap(S, kdep(k)));
                    if (p.gstore == 0) st_stream(dst, sv[k]);
                    else if (p.gstore == 1) st_plain(dst, sv[k]);
                    else st_hint(dst, sv[k], policy_evict_last());
                }
            } else {
                double2 *dst = p.y + (cbase + t_off);
#pragma unroll
                for (int k = 0; k < NR; ++k) st_stream(dst + kdep(k), sv[k]);
            }
            continue;
        }
        if (S.gperm) {  // trailing permutation run: element i goes to A i ^ c in the other buffer
            const uint64_t ab = s_ab ^ g_t;
#pragma unroll
            for (int k = 0; k < NR; ++k) {
                double2 *dst = p.y + (ab ^ gmap(S, kdep(k)));
                const double2 v = lds128(slot_addr(a, swz((uint32_t)k << TB)));
                if (p.gstore == 0) st_stream(dst, v);
                else if (p.gstore == 1) st_plain(dst, v);
                else st_hint(dst, v, policy_evict_last());
            }
        } else {
            double2 *dst = p.y + (base + t_off);
#pragma unroll
            for (int k = 0; k < NR; ++k) st_stream(dst + kdep(k), lds128(slot_addr(a, swz((uint32_t)k << TB))));
        }
        __syncthreads();
        t = nt;
        base = insert_zero_bits_dyn((uint64_t)t, S.tb, T);
        if (p.nbuf == 2) buf = (buf == tile0) ? tile0 + tstride : tile0;
        else if (t < p.ntiles) fetch(base, buf);  // refill as soon as the tile is drained
    }
    if (dyn) units_done();
}
#endif  // DIAQ_JIT

}  // namespace diaq
