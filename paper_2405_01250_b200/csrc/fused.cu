// fused.cu -- multi-gate passes: register-tiled, shared-memory staged (sm_100a).
//
// The run loop (reference sim.py:193-199) applies gates one at a time; on the
// GPU each gate alone is a full 32*2^n-byte sweep of HBM.  A pass instead
// moves a tile of 2^T amplitudes -- every index that varies only in a set B
// of T state bits (B contains the low bits, so tile rows are contiguous
// 128-byte runs) -- through the SM once and applies a run of consecutive
// gates whose MIXING operand bits all lie in B:
//
//   HBM --(coalesced)--> smem tile --> registers: phase 1 gates --> smem -->
//   registers: phase 2 gates --> ... --> smem --(coalesced)--> HBM
//
// Each thread holds 2^R amplitudes in registers (R = T - 8, 256 threads).  A
// phase picks R tile bits as "register bits" and applies every consecutive
// gate whose mixing bits are among them entirely in registers; shared memory
// is touched once per phase, not once per gate.  The smem tile is XOR-
// swizzled so any lane<->bit mapping stays (nearly) bank-conflict free.
//
// Parity is unchanged: every gate is still applied on its own, in circuit
// order, with the gate kernel's arithmetic (relabelled ascending-embedding
// column order, numpy complex-multiply rounding, sequential adds from +0,
// exactly-zero entries skipped).  Operands a gate does not mix (controls;
// diagonal gates such as RZ/CZ) may lie anywhere: within a register group
// those bits are fixed, so they only select which sub-block of the gate
// applies (the same argument as the sharded kernel, apply.cu).
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <functional>
#include <vector>

#include "common.cuh"
#include "fused_dev.cuh"
#include "fused_jit.cuh"

extern "C" const char *diaq_jit_last_error(void);

namespace diaq {

template <int R, int MODE>
__global__ void __launch_bounds__(kThreads, R >= 4 ? 2 : 3) tile_pass_kernel(const __grid_constant__ TileParams p) {
    tile_pass_body<R, MODE>(p, p);
}

// 128 threads x 16 amplitudes (T = 11, R = 4): the layout of the default
// specialised passes (fused_tbits 7), interpreted while they compile
template <int MODE>
__global__ void __launch_bounds__(128, 4) tile_pass_kernel_t7(const __grid_constant__ TileParams p) {
    tile_pass_body<4, MODE, 7>(p, p);
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

struct Packed {
    std::vector<double2> coef;
    std::vector<uint32_t> nz;
    std::vector<uint32_t> cls;
};

struct PassPlan {
    std::vector<int> bits;        // ascending state bits of the tile (empty: standalone gate)
    std::vector<int> members;     // caller gate indices, in order
    std::vector<Phase> phases;
    std::vector<RegGate> gates;   // pass-relative
    Packed pk;                    // pass-relative coefficient tables
    Affine pre;                   // permutation run opening the pass (pre.on = 0: none)
    // trailing permutation run leaving the tile, composed over the whole
    // local index and applied by the final store (out of place): new index =
    // XOR of gcol[j] over the set old bits j ^ gc ^ XOR of ggcol[g] over the
    // set global (rank) bits g
    int nrperm = 0;               // permutation members applied as register renamings (gate records, no arithmetic)
    int nrperm_records = 0;       // their gate records (a SWAP takes three)
    bool gon = false;
    size_t tail = SIZE_MAX;
    std::vector<uint64_t> gcol, ggcol;
    uint64_t gc = 0;
};

static int tile_pos(const std::vector<int> &bits, int shift) {
    for (size_t j = 0; j < bits.size(); ++j)
        if (bits[j] == shift) return (int)j;
    return -1;
}

// A gate whose matrix is a 0/1 permutation (entries exactly 1+0i or 0) that
// is affine over GF(2) in the gate-index bits: old index x moves to new
// index q(x) = XOR_{m: x_m} col[m] ^ d.  (X, CX in either orientation,
// SWAP, X on several operands, ...; CCX/CSWAP are not affine.)
struct PermGate {
    bool ok = false;
    uint32_t col[8] = {0};
    uint32_t d = 0;
};

static PermGate perm_affine(const diaq_gate_t &gt) {
    PermGate pg;
    const int k = gt.k, M = 1 << k;
    if (k < 1 || k > 8) return pg;
    std::vector<int> q(M, -1);
    for (int r = 0; r < M; ++r) {
        int c1 = -1;
        for (int c = 0; c < M; ++c) {
            const double re = gt.g[2 * (r * M + c)], im = gt.g[2 * (r * M + c) + 1];
            if (re == 1.0 && im == 0.0) {
                if (c1 >= 0) return pg;
                c1 = c;
            } else if (!(re == 0.0 && im == 0.0)) {
                return pg;
            }
        }
        if (c1 < 0 || q[c1] >= 0) return pg;
        q[c1] = r;  // new[r] = old[c1]: old index c1 moves to r
    }
    pg.d = (uint32_t)q[0];
    for (int m = 0; m < k; ++m) pg.col[m] = (uint32_t)q[1 << m] ^ pg.d;
    for (int x = 0; x < M; ++x) {
        uint32_t y = pg.d;
        for (int m = 0; m < k; ++m)
            if ((x >> m) & 1) y ^= pg.col[m];
        if (y != (uint32_t)q[x]) return pg;
    }
    pg.ok = true;
    return pg;
}

// Host form of an Affine map while a run of permutation gates is folded:
// row[o] is tile output bit o as a GF(2) combination of tile input bits
// (bits 0..T-1), base (non-tile) state bits (T + i, state bit base[i]) and
// the constant (bit 63).
struct HostAffine {
    int T = 0;
    bool on = false;
    std::vector<uint64_t> row;
    std::vector<int> base;

    void init(int t) {
        T = t;
        on = false;
        row.assign(t, 0);
        for (int o = 0; o < t; ++o) row[o] = 1ull << o;
        base.clear();
    }
    // this <- q o this for one permutation gate; false if the map would need
    // more than kMaxPermBase base bits
    bool fold(const diaq_gate_t &gt, const PermGate &pg, const std::vector<int> &bits) {
        const int k = gt.k;
        std::vector<uint64_t> in(k), out(k);
        std::vector<int> tp(k);
        for (int i = 0; i < k; ++i) {
            tp[i] = tile_pos(bits, gt.shifts[i]);
            if (tp[i] >= 0) {
                in[i] = row[tp[i]];
            } else {
                int idx = -1;
                for (size_t b = 0; b < base.size(); ++b)
                    if (base[b] == gt.shifts[i]) idx = (int)b;
                if (idx < 0) {
                    if ((int)base.size() >= kMaxPermBase) return false;
                    idx = (int)base.size();
                    base.push_back(gt.shifts[i]);
                }
                in[i] = 1ull << (T + idx);
            }
        }
        // operand i is gate-index bit k-1-i
        for (int i = 0; i < k; ++i) {
            const int gb = k - 1 - i;
            uint64_t e = ((pg.d >> gb) & 1u) ? (1ull << 63) : 0ull;
            for (int m = 0; m < k; ++m)
                if ((pg.col[m] >> gb) & 1u) e ^= in[k - 1 - m];
            out[i] = e;
        }
        for (int i = 0; i < k; ++i) {
            if (tp[i] >= 0) continue;
            if (out[i] != in[i]) return false;  // a bit outside the tile cannot move (mixing bits are in the tile)
        }
        for (int i = 0; i < k; ++i)
            if (tp[i] >= 0) row[tp[i]] = out[i];
        on = true;
        return true;
    }
    Affine pack() const {
        Affine a;
        memset(&a, 0, sizeof(a));
        a.on = on ? 1 : 0;
        if (!on) return a;
        for (int o = 0; o < T; ++o) {
            for (int j = 0; j < T; ++j)
                if ((row[o] >> j) & 1ull) a.a[j] |= 1u << o;
            for (size_t b = 0; b < base.size(); ++b)
                if ((row[o] >> (T + b)) & 1ull) a.b[b] |= 1u << o;
            if ((row[o] >> 63) & 1ull) a.c |= 1u << o;
        }
        a.nb = (int)base.size();
        for (size_t b = 0; b < base.size(); ++b) a.bbit[b] = base[b];
        return a;
    }
};

// A run of permutation gates composed over the whole local index (the
// trailing run of a pass whose targets leave the tile): old local index i
// moves to new index A i ^ c ^ (sum over set global (rank) bits of gcol).
// Applied by the pass's final store -- out of place, since amplitudes move
// between tiles.
struct GlobalAffine {
    struct Expr {
        uint64_t m = 0;  // local input bits
        uint64_t g = 0;  // global input bits (bit index - n)
        bool c = false;
        Expr operator^(const Expr &o) const { return Expr{m ^ o.m, g ^ o.g, c != o.c}; }
        bool operator!=(const Expr &o) const { return m != o.m || g != o.g || c != o.c; }
    };
    int n = 0;
    bool on = false;
    std::vector<Expr> row;  // new local bit o as a combination of old bits

    void init(int nbits) {
        n = nbits;
        on = false;
        row.assign(n, Expr{});
        for (int o = 0; o < n; ++o) row[o].m = 1ull << o;
    }
    bool fold(const diaq_gate_t &gt, const PermGate &pg) {
        const int k = gt.k;
        std::vector<Expr> in(k), out(k);
        for (int i = 0; i < k; ++i) {
            const int sh = gt.shifts[i];
            if (sh < n) {
                in[i] = row[sh];
            } else {
                if (sh - n >= 64) return false;
                in[i].g = 1ull << (sh - n);
            }
        }
        for (int i = 0; i < k; ++i) {  // operand i is gate-index bit k-1-i
            const int gb = k - 1 - i;
            Expr e;
            e.c = (pg.d >> gb) & 1u;
            for (int m = 0; m < k; ++m)
                if ((pg.col[m] >> gb) & 1u) e = e ^ in[k - 1 - m];
            out[i] = e;
        }
        for (int i = 0; i < k; ++i)
            if (gt.shifts[i] >= n && out[i] != in[i]) return false;  // a global bit cannot move
        for (int i = 0; i < k; ++i)
            if (gt.shifts[i] < n) row[gt.shifts[i]] = out[i];
        on = true;
        return true;
    }
};

static int pack_reg_gate(const diaq_gate_t &gt, const std::vector<int> &bits, const Phase &ph, int R, Packed &pk,
                         RegGate &G) {
    const int k = gt.k, M = 1 << k;
    const uint32_t mix = mixing_mask(k, gt.g);
    std::vector<int> mops, sops;
    for (int i = 0; i < k; ++i) ((mix >> i) & 1u ? mops : sops).push_back(i);
    std::sort(mops.begin(), mops.end(), [&](int a, int b) { return gt.shifts[a] > gt.shifts[b]; });
    std::sort(sops.begin(), sops.end(), [&](int a, int b) { return gt.shifts[a] > gt.shifts[b]; });
    memset(&G, 0, sizeof(G));
    G.kin = (int)mops.size();
    G.kout = (int)sops.size();
    if (G.kin > kMaxRegKin || G.kout > kMaxSel) return set_error(DIAQ_ERR_UNSUPPORTED, "fused gate too wide");
    for (int j = 0; j < G.kin; ++j) {
        const int tp = tile_pos(bits, gt.shifts[mops[j]]);
        int rb = -1;
        for (int i = 0; i < R; ++i)
            if (ph.rpos[i] == tp) rb = i;
        if (tp < 0 || rb < 0) return set_error(DIAQ_ERR_VALUE, "fused pass: mixing bit outside the phase registers");
        G.rb[j] = rb;  // descending shift -> descending register bit
    }
    G.rsel = 0;
    for (int j = 0; j < G.kout; ++j) {
        const int s = gt.shifts[sops[j]];
        const int tp = tile_pos(bits, s);
        if (tp < 0) {
            G.osel[j] = 0;
            G.opos[j] = s;
            continue;
        }
        int rb = -1;
        for (int i = 0; i < R; ++i)
            if (ph.rpos[i] == tp) rb = i;
        if (rb >= 0) {
            G.osel[j] = 2;
            G.opos[j] = rb;
            G.rsel = 1;
        } else {
            G.osel[j] = 1;
            G.opos[j] = tp;
        }
    }
    auto orig = [&](int b, int c) {
        int o = 0;
        for (int j = 0; j < G.kin; ++j) o |= ((c >> (G.kin - 1 - j)) & 1) << (k - 1 - mops[j]);
        for (int j = 0; j < G.kout; ++j) o |= ((b >> (G.kout - 1 - j)) & 1) << (k - 1 - sops[j]);
        return o;
    };
    const int MI = 1 << G.kin;
    G.coef_off = (int)pk.coef.size();
    G.nz_off = (int)pk.nz.size();
    G.cls_off = (int)pk.cls.size();
    for (int b = 0; b < (1 << G.kout); ++b) {
        bool ident = true, swap = (MI == 2);
        for (int r = 0; r < MI; ++r) {
            uint32_t m = 0;
            for (int c = 0; c < MI; ++c) {
                const int o_r = orig(b, r), o_c = orig(b, c);
                const double re = gt.g[2 * (o_r * M + o_c)], im = gt.g[2 * (o_r * M + o_c) + 1];
                pk.coef.push_back(make_double2(re, im));
                if (re != 0.0 || im != 0.0) m |= 1u << c;
                const bool one = (re == 1.0 && im == 0.0), zero = (re == 0.0 && im == 0.0);
                if (r == c ? !one : !zero) ident = false;
                if (r != c ? !one : !zero) swap = false;
            }
            pk.nz.push_back(m);
        }
        pk.cls.push_back(ident ? 1u : (swap ? 2u : 0u));
    }
    G.op = 0;
    G.shape = 0;
    if (G.kin == 1 && G.kout == 0) {
        G.op = 1;
        const double2 *c = &pk.coef[G.coef_off];
        bool real = true, rx = true;
        for (int e = 0; e < 4; ++e) {
            real = real && c[e].y == 0.0;
            rx = rx && ((e == 0 || e == 3) ? c[e].y == 0.0 : c[e].x == 0.0);
        }
        G.shape = real ? 1 : (rx ? 2 : 0);
        G.full = (pk.nz[(size_t)G.nz_off] & pk.nz[(size_t)G.nz_off + 1] & 3u) == 3u;
    }
    else if (G.kin == 0 && G.kout == 1) G.op = 2;
    else if (G.kin == 2 && G.kout == 0) {  // dense two-qubit: register path only when every entry is nonzero
        bool full = true;
        for (int r = 0; r < 4; ++r) full = full && (pk.nz[G.nz_off + r] & 15u) == 15u;
        if (full) G.op = 3;
    }
    return DIAQ_OK;
}

// gates the register fast paths handle: dense 1-qubit and 1-selector
// diagonal.  (Controlled swaps -- CX -- are permutations: folded into the
// pass addressing, see HostAffine; the shared-memory path takes the rest.)
static bool fast_op(const diaq_gate_t &gt) {
    const uint32_t mix = mixing_mask(gt.k, gt.g);
    int kin = 0;
    for (int i = 0; i < gt.k; ++i) kin += (mix >> i) & 1u;
    const int kout = gt.k - kin;
    if (kin > 1 || kout > 1) return false;
    if (kin == 1 && kout == 0) return true;
    if (kin == 0 && kout == 1) return true;
    return false;
}

static int pack_smem_gate(const diaq_gate_t &gt, const std::vector<int> &bits, Packed &pk, RegGate &G) {
    Phase ph;
    memset(&ph, 0, sizeof(ph));
    for (int i = 0; i < 4; ++i) ph.rpos[i] = -100;  // no register bits: selectors are tile or base bits
    const uint32_t mix = mixing_mask(gt.k, gt.g);
    int mshift = -1;
    for (int i = 0; i < gt.k; ++i)
        if ((mix >> i) & 1u) mshift = gt.shifts[i];
    // pack_reg_gate needs the mixing bits among the registers: give it fake ones
    int nm = 0;
    for (int i = 0; i < gt.k; ++i)
        if ((mix >> i) & 1u) ph.rpos[nm++] = (int8_t)tile_pos(bits, gt.shifts[i]);
    (void)mshift;
    const int rc = pack_reg_gate(gt, bits, ph, nm > 0 ? nm : 1, pk, G);
    if (rc) return rc;
    for (int j = 0; j < kMaxRegKin; ++j) G.mpos[j] = j < G.kin ? ph.rpos[G.rb[j]] : 0;
    for (int s = 0; s < G.kout; ++s)
        if (G.osel[s] == 2) return set_error(DIAQ_ERR_VALUE, "smem gate selector on a register bit");
    G.op = 0;
    return DIAQ_OK;
}

// Greedy, order preserving: a pass grows while the union of mixing bits
// (plus the low bits) fits in T; within a pass a phase grows while the
// union of its gates' mixing bits fits in R registers.  Gates that cannot
// be applied in registers (more than 2 mixing or 4 selector operands)
// become standalone single-gate passes (gate_kernel).
// set while re-planning a call without the out-of-place permutation tails
// (no room for the state-sized buffer they need)
static thread_local bool t_no_gperm = false;
// schedule with commutation-aware deferral (set for the contracted arithmetic;
// part of the program key)
static thread_local bool t_reorder = false;
// contracted arithmetic: rotations in unit-diagonal form (unit_forms below;
// part of the program key -- the coefficient tables differ)
static thread_local bool t_unit = false;

// thread bits of a tiled pass: 8 (256 threads; T = 11 -> R = 3, T = 12 -> R = 4)
// or 7 (128 threads, T = 11, R = 4: a phase covers one more qubit, so a pass
// needs fewer smem round trips, and CTAs are smaller -- the default)
static int pass_tbits() { return tuning().fused_tbits == 7 ? 7 : 8; }

// Shared-memory banks: a 16-byte access is served per quarter warp (lanes
// differing in thread bits 0-2); its 8 slots hit 8 distinct 16-byte bank
// groups iff the bank-group images (swz(e) & 7, linear in e) of the tile
// positions carrying thread bits 0-2 are independent.  Thread bits may sit
// on any tile positions (tpart is built from tpos; selectors test tile
// positions), so pick the three positions that minimise the conflict
// factors of the phase load (slot swz(tpart)) and, with a folded
// permutation, of its store (slot swz(A tpart ^ c)); the rest stay ascending.
static void spread_lane_bits(Phase &ph, int T, int R) {
    const int nt = T - R;
    if (nt < 4) return;
    auto distinct = [](uint32_t a, uint32_t b, uint32_t c) {
        uint32_t seen = 0;
        for (int m = 0; m < 8; ++m) seen |= 1u << (((m & 1) ? a : 0) ^ ((m & 2) ? b : 0) ^ ((m & 4) ? c : 0));
        return __builtin_popcount(seen);
    };
    auto ld = [&](int tp) { return swz(1u << tp) & 7u; };
    auto st = [&](int tp) { return swz(aff_lin(ph.post, 1u << tp, T)) & 7u; };
    int best[3] = {0, 1, 2};
    int best_cost = 1 << 30;
    for (int a = 0; a < nt; ++a)
        for (int b = a + 1; b < nt; ++b)
            for (int c = b + 1; c < nt; ++c) {
                const int pa = ph.tpos[a], pb = ph.tpos[b], pc = ph.tpos[c];
                int cost = 8 / distinct(ld(pa), ld(pb), ld(pc));
                if (ph.post.on) cost += 8 / distinct(st(pa), st(pb), st(pc));
                if (cost < best_cost) {
                    best_cost = cost;
                    best[0] = a, best[1] = b, best[2] = c;
                }
            }
    int8_t out[kMaxTileBits];
    int q = 0;
    for (int i = 0; i < 3; ++i) out[q++] = ph.tpos[best[i]];
    for (int i = 0; i < nt; ++i)
        if (i != best[0] && i != best[1] && i != best[2]) out[q++] = ph.tpos[i];
    for (int i = 0; i < nt; ++i) ph.tpos[i] = out[i];
}

// A permutation gate as controlled exchanges of register pairs: X (one
// operand), CX in either orientation, SWAP (three CX).  out: (control
// operand or -1, target operand) in application order; false: not of
// these kinds (the gate is folded into a phase store instead).
static bool rperm_ops(const diaq_gate_t &gt, const PermGate &pg, std::vector<std::pair<int, int>> &out) {
    out.clear();
    if (!pg.ok) return false;
    if (gt.k == 1) {
        if (pg.d != 1u || pg.col[0] != 1u) return false;
        out.push_back({-1, 0});
        return true;
    }
    if (gt.k != 2 || pg.d != 0u) return false;
    // gate-index bit m <-> operand 1 - m; col[m] = image of bit m
    const uint32_t c0 = pg.col[0], c1 = pg.col[1];
    if (c0 == 1u && c1 == 3u) out.push_back({0, 1});        // bit 1 (operand 0) controls bit 0 (operand 1)
    else if (c0 == 3u && c1 == 2u) out.push_back({1, 0});   // bit 0 (operand 1) controls bit 1 (operand 0)
    else if (c0 == 2u && c1 == 1u) out = {{0, 1}, {1, 0}, {0, 1}};  // SWAP
    else return false;
    return true;
}

static int pack_rperm(const diaq_gate_t &gt, const PermGate &pg, const std::vector<int> &bits, const Phase &ph, int R,
                      std::vector<RegGate> &out) {
    std::vector<std::pair<int, int>> ops;
    if (!rperm_ops(gt, pg, ops)) return set_error(DIAQ_ERR_VALUE, "fused pass: permutation is not a register exchange");
    auto regbit = [&](int operand) {
        const int tp = tile_pos(bits, gt.shifts[operand]);
        for (int i = 0; i < R; ++i)
            if (tp >= 0 && ph.rpos[i] == tp) return i;
        return -1;
    };
    for (const auto &op : ops) {
        RegGate G;
        memset(&G, 0, sizeof(G));
        G.op = 4;
        G.rb[0] = (int8_t)regbit(op.second);
        G.rb[1] = (int8_t)(op.first < 0 ? -1 : regbit(op.first));
        if (G.rb[0] < 0 || (op.first >= 0 && G.rb[1] < 0))
            return set_error(DIAQ_ERR_VALUE, "fused pass: register exchange outside the phase registers");
        out.push_back(G);
    }
    return DIAQ_OK;
}

// Contracted arithmetic: a rotation [[a, b], [c, a]] with a real (RX, RY)
// is applied as [[1, b/a], [c/a, 1]] -- one DFMA per part, 2 FP64
// operations per amplitude instead of 4 -- and the scalar a is carried to
// the pass's last such gate, which keeps its form with every entry scaled
// by the product of the scalars (a scalar commutes with every gate of the
// pass, so the pass computes the same operator; the rounding differs, as
// everywhere under this arithmetic).  |b/a| stays below 2^10.
static void unit_forms(PassPlan &ps) {
    std::vector<size_t> el;
    for (size_t gi = 0; gi < ps.gates.size(); ++gi) {
        const RegGate &G = ps.gates[gi];
        if (G.op != 1 || (G.shape != 1 && G.shape != 2)) continue;
        const double2 *c = &ps.pk.coef[(size_t)G.coef_off];
        if ((ps.pk.nz[(size_t)G.nz_off] & ps.pk.nz[(size_t)G.nz_off + 1] & 3u) != 3u) continue;
        if (c[0].x != c[3].x || !(fabs(c[0].x) >= 0x1p-10) || !(fabs(c[0].x) <= 1.0)) continue;
        el.push_back(gi);
    }
    if (el.size() < 2) return;
    double scale = 1.0;
    for (size_t e = 0; e + 1 < el.size(); ++e) {
        RegGate &G = ps.gates[el[e]];
        double2 *c = &ps.pk.coef[(size_t)G.coef_off];
        const double a = c[0].x;
        scale *= a;
        c[1] = make_double2(c[1].x / a, c[1].y / a);
        c[2] = make_double2(c[2].x / a, c[2].y / a);
        c[0] = c[3] = make_double2(1.0, 0.0);
        G.shape = (int8_t)(G.shape + 2);
    }
    double2 *c = &ps.pk.coef[(size_t)ps.gates[el.back()].coef_off];
    for (int e = 0; e < 4; ++e) c[e] = make_double2(c[e].x * scale, c[e].y * scale);
}

static int schedule_once(int n_bits, int n_total, int ngates, const diaq_gate_t *gates, int T, int R,
                         std::vector<PassPlan> &plan, bool allow_d2) {
    const bool reorder = t_reorder;
    const int low = std::min(kLowBits, n_bits);
    std::vector<char> fast((size_t)ngates);  // register fast-path classification, once per gate
    std::vector<PermGate> perm((size_t)ngates);
    std::vector<char> d2((size_t)ngates, 0);  // dense two-qubit gate for the register path (sequence phases)
    for (int i = 0; i < ngates; ++i) {
        fast[(size_t)i] = (gates[i].k >= 1 && gates[i].k <= 5) ? fast_op(gates[i]) : 0;
        if (tuning().fused_perm && gates[i].k >= 1 && gates[i].k <= 5) perm[(size_t)i] = perm_affine(gates[i]);
        if (allow_d2 && tuning().fused_dense2 && tuning().fused_seq && !perm[(size_t)i].ok && gates[i].k >= 2 &&
            gates[i].k <= 5) {
            const diaq_gate_t &gt = gates[i];
            const uint32_t mix = mixing_mask(gt.k, gt.g);
            int kin = 0;
            for (int o = 0; o < gt.k; ++o) kin += (mix >> o) & 1u;
            bool full = kin == 2 && gt.k == 2;  // no selectors: every entry of the 4x4 nonzero
            for (int e = 0; full && e < 16; ++e) full = !(gt.g[2 * e] == 0.0 && gt.g[2 * e + 1] == 0.0);
            d2[(size_t)i] = full;
        }
    }
    std::vector<int> members;
    std::vector<char> inb(64, 0);
    int nb = 0;
    int ncoef = 0, nnz = 0;  // the pass's coefficient / mask table entries (kernel parameter bound)
    size_t tail = SIZE_MAX;  // members[tail..]: permutation run folded over the whole index (final store)
    GlobalAffine tail_map;   // that run's composition so far
    auto reset = [&]() {
        std::fill(inb.begin(), inb.end(), 0);
        nb = 0;
        for (int b = 0; b < low; ++b) { inb[b] = 1; ++nb; }
        members.clear();
        ncoef = nnz = 0;
        tail = SIZE_MAX;
    };
    // phase specs: register phases (<= R mixing bits), generic smem phases,
    // and permutation runs folded into the previous phase's store (or the
    // tile load when the pass opens with one)
    struct Spec {
        int generic = 0;
        std::vector<int> mem;
        std::vector<char> rperm;  // parallel to mem (may be shorter: 0): permutation applied in registers
        std::vector<int> used;
        HostAffine post;
        bool seq_ok = true;  // still a sequence phase (dense steps on fresh register bits in order)
        bool has_d2 = false;
    };
    std::function<int(PassPlan &, std::vector<Spec> &, HostAffine &, const std::vector<int> &)> finish;
    auto tile_bits_of = [&](PassPlan &ps) {
        for (int b = 0; b < 64; ++b)
            if (inb[b]) ps.bits.push_back(b);
        for (int b = 0; (int)ps.bits.size() < T && b < n_bits; ++b)
            if (!inb[b]) ps.bits.push_back(b);
        std::sort(ps.bits.begin(), ps.bits.end());
    };
    auto flush = [&]() -> int {
        if (members.empty()) return DIAQ_OK;
        PassPlan ps;
        tile_bits_of(ps);
        ps.members = members;
        std::vector<Spec> specs;
        HostAffine pre;
        pre.init((int)ps.bits.size());
        bool open = false;
        const size_t body = std::min(tail, members.size());
        for (size_t i = 0; i < body; ++i) {
            const int gi = members[i];
            const diaq_gate_t &gt = gates[gi];
            if (perm[(size_t)gi].ok) {
                HostAffine *tgt;
                if (specs.empty()) {
                    tgt = &pre;
                } else if (!specs.back().generic) {
                    tgt = &specs.back().post;
                } else {  // after a shared-memory phase: an empty register phase carries it
                    Spec sp;
                    sp.post.init((int)ps.bits.size());
                    specs.push_back(sp);
                    tgt = &specs.back().post;
                }
                open = false;
                if (!tgt->fold(gt, perm[(size_t)gi], ps.bits))
                    return set_error(DIAQ_ERR_VALUE, "fused pass: permutation fold overflow");
                continue;
            }
            if (fast[(size_t)gi] || d2[(size_t)gi]) {
                const uint32_t mix = mixing_mask(gt.k, gt.g);
                const bool isd2 = d2[(size_t)gi] != 0;
                int kin = 0;
                for (int o = 0; o < gt.k; ++o) kin += (mix >> o) & 1u;
                // mixing bits in relabelled order (descending state bit): a two-qubit
                // gate's gate-index MSB takes the lower register bit of its pair
                std::vector<int> mops;
                for (int o = 0; o < gt.k; ++o)
                    if ((mix >> o) & 1u) mops.push_back(o);
                std::sort(mops.begin(), mops.end(), [&](int a, int b) { return gt.shifts[a] > gt.shifts[b]; });
                std::vector<int> add;
                for (int o : mops) {
                    const int tp = tile_pos(ps.bits, gt.shifts[o]);
                    if ((!open || std::find(specs.back().used.begin(), specs.back().used.end(), tp) ==
                                      specs.back().used.end()) &&
                        std::find(add.begin(), add.end(), tp) == add.end())
                        add.push_back(tp);
                }
                // does the gate keep the open phase a sequence phase?
                bool keeps = (int)add.size() == kin;  // dense steps on fresh bits only
                if (kin == 0 && open) {               // a diagonal must not select a register bit
                    for (int o = 0; o < gt.k; ++o) {
                        const int tp = tile_pos(ps.bits, gt.shifts[o]);
                        if (tp >= 0 && std::find(specs.back().used.begin(), specs.back().used.end(), tp) !=
                                           specs.back().used.end())
                            keeps = false;
                    }
                }
                const bool fits = open && (int)(specs.back().used.size() + add.size()) <= R;
                const bool join = fits && (keeps || (!specs.back().has_d2 && !isd2)) &&
                                  (!isd2 || specs.back().seq_ok);
                if (join) {
                    specs.back().mem.push_back(gi);
                    specs.back().used.insert(specs.back().used.end(), add.begin(), add.end());
                    specs.back().seq_ok = specs.back().seq_ok && keeps;
                    specs.back().has_d2 = specs.back().has_d2 || isd2;
                } else {
                    Spec sp;
                    sp.mem = {gi};
                    std::vector<int> all;
                    for (int o : mops) all.push_back(tile_pos(ps.bits, gt.shifts[o]));
                    sp.used = all;
                    sp.post.init((int)ps.bits.size());
                    sp.has_d2 = isd2;
                    specs.push_back(sp);
                    open = true;
                }
                continue;
            }
            Spec sp;  // cold path: its own shared-memory phase
            sp.generic = 1;
            sp.mem = {gi};
            specs.push_back(sp);
            open = false;
        }
        const std::vector<int> tailm(members.begin() + (long)body, members.end());
        return finish(ps, specs, pre, tailm);
    };
    // the pass from its phase specs: global tail map, packed phases and gate records
    finish = [&](PassPlan &ps, std::vector<Spec> &specs, HostAffine &pre, const std::vector<int> &tailm) -> int {
        ps.pre = pre.pack();
        if (!tailm.empty()) {  // trailing run leaving the tile: one map over the whole local index
            GlobalAffine ga;
            ga.init(n_bits);
            for (const int gi : tailm)
                if (!ga.fold(gates[gi], perm[(size_t)gi]))
                    return set_error(DIAQ_ERR_VALUE, "fused pass: permutation moves a global bit");
            ps.tail = ps.members.size() - tailm.size();
            ps.gon = true;
            ps.gcol.assign((size_t)n_bits, 0);
            ps.ggcol.assign(64, 0);
            for (int o = 0; o < n_bits; ++o) {
                for (int j = 0; j < n_bits; ++j)
                    if ((ga.row[o].m >> j) & 1ull) ps.gcol[j] |= 1ull << o;
                for (int g = 0; g < 64; ++g)
                    if ((ga.row[o].g >> g) & 1ull) ps.ggcol[g] |= 1ull << o;
                if (ga.row[o].c) ps.gc |= 1ull << o;
            }
        }
        // 2. pack
        for (const Spec &sp : specs) {
            Phase ph;
            memset(&ph, 0, sizeof(ph));
            if (sp.generic) {
                ph.generic = 1;
                ph.g0 = (int)ps.gates.size();
                RegGate G;
                const int rc = pack_smem_gate(gates[sp.mem[0]], ps.bits, ps.pk, G);
                if (rc) return rc;
                ps.gates.push_back(G);
                ph.g1 = (int)ps.gates.size();
                ps.phases.push_back(ph);
                continue;
            }
            std::vector<int> rp = sp.used;  // first-use order of the mixing bits
            const bool seq_try = tuning().fused_seq != 0;
            if (seq_try) {  // pad with positions no diagonal of the phase selects on
                std::vector<int> sel;
                for (int gi : sp.mem) {
                    const diaq_gate_t &gt = gates[gi];
                    const uint32_t mix = mixing_mask(gt.k, gt.g);
                    for (int o = 0; o < gt.k; ++o)
                        if (!((mix >> o) & 1u)) sel.push_back(tile_pos(ps.bits, gt.shifts[o]));
                }
                for (int tp = 0; (int)rp.size() < R && tp < (int)ps.bits.size(); ++tp)
                    if (std::find(rp.begin(), rp.end(), tp) == rp.end() &&
                        std::find(sel.begin(), sel.end(), tp) == sel.end())
                        rp.push_back(tp);
            }
            for (int tp = 0; (int)rp.size() < R; ++tp)
                if (std::find(rp.begin(), rp.end(), tp) == rp.end()) rp.push_back(tp);
            if (!seq_try) std::sort(rp.begin(), rp.end());
            for (int q = 0; q < R; ++q) ph.rpos[q] = rp[q];
            int tq = 0;
            for (int tp = 0; tp < (int)ps.bits.size(); ++tp)
                if (std::find(rp.begin(), rp.end(), tp) == rp.end()) ph.tpos[tq++] = tp;
            ph.g0 = (int)ps.gates.size();
            for (size_t mi = 0; mi < sp.mem.size(); ++mi) {
                const int gi = sp.mem[mi];
                if (mi < sp.rperm.size() && sp.rperm[mi]) {
                    const int before = (int)ps.gates.size();
                    const int rc = pack_rperm(gates[gi], perm[(size_t)gi], ps.bits, ph, R, ps.gates);
                    if (rc) return rc;
                    ++ps.nrperm;
                    ps.nrperm_records += (int)ps.gates.size() - before;
                    continue;
                }
                RegGate G;
                const int rc = pack_reg_gate(gates[gi], ps.bits, ph, R, ps.pk, G);
                if (rc) return rc;
                ps.gates.push_back(G);
            }
            ph.g1 = (int)ps.gates.size();
            ph.post = sp.post.pack();
            if (tuning().fused_bank_spread) spread_lane_bits(ph, (int)ps.bits.size(), R);
            for (int j = 0; j < 16; ++j) {
                uint32_t e = 0;
                for (int q = 0; q < R; ++q) e |= (uint32_t)((j >> q) & 1) << ph.rpos[q];
                ph.pj[j] = j < (1 << R) ? (uint16_t)swz(e) : 0;
                ph.ppj[j] = (j < (1 << R) && ph.post.on) ? (uint16_t)swz(aff_lin(ph.post, e, (int)ps.bits.size())) : 0;
            }
            if (seq_try) {  // sequence form?
                int nd = 0, cnt = 0;
                bool ok = true;
                for (int b = 0; b < 5; ++b) ph.kind[b] = 0;
                for (int g = ph.g0; g < ph.g1 && ok; ++g) {
                    const RegGate &G = ps.gates[g];
                    if (G.op == 1 && G.rb[0] == nd && nd < R) {
                        ph.kind[nd] = 1;
                        ph.nd_before[nd++] = (int8_t)cnt;
                        cnt = 0;
                    } else if (G.op == 3 && G.rb[0] == nd && G.rb[1] == nd + 1 && nd + 1 < R) {
                        ph.kind[nd] = 2;
                        ph.nd_before[nd] = (int8_t)cnt;
                        ph.nd_before[nd + 1] = 0;
                        nd += 2;
                        cnt = 0;
                    } else if (G.op == 2 && G.osel[0] != 2 && cnt < 127) {
                        ++cnt;
                    } else {
                        ok = false;
                    }
                }
                if (ok) {
                    ph.seq = 1;
                    ph.ndense = (int8_t)nd;
                    for (int b = nd; b <= R; ++b) ph.nd_before[b] = 0;
                    ph.nd_before[R] = (int8_t)cnt;
                }
            }
            if (!ph.seq) {  // a dense two-qubit gate runs only in a sequence phase
                for (int g = ph.g0; g < ph.g1; ++g)
                    if (ps.gates[g].op == 3) return kRetryNoDense2;
                int lead = 0;  // leading diagonals on non-register bits: applied as one run (diag_run)
                while (ph.g0 + lead < ph.g1 && lead < 127 && ps.gates[(size_t)(ph.g0 + lead)].op == 2 &&
                       ps.gates[(size_t)(ph.g0 + lead)].osel[0] != 2)
                    ++lead;
                for (int b = 0; b < 5; ++b) ph.nd_before[b] = 0;
                ph.nd_before[0] = (int8_t)lead;
            }
            ps.phases.push_back(ph);
        }
        if ((int)ps.phases.size() > kMaxPhases || (int)ps.gates.size() > kMaxPassGates)
            return set_error(DIAQ_ERR_VALUE, "fused pass too long");
        if (t_unit) unit_forms(ps);
        plan.push_back(ps);
        return DIAQ_OK;
    };
    // per-gate facts the sweep needs (once per schedule)
    std::vector<uint32_t> gmix((size_t)ngates, 0);
    std::vector<uint64_t> gqm((size_t)ngates, 0);
    for (int i = 0; i < ngates; ++i) {
        const diaq_gate_t &gt = gates[i];
        if (gt.k < 1 || gt.k > 5) return set_error(DIAQ_ERR_UNSUPPORTED, "gate width %d outside 1..5", gt.k);
        gmix[(size_t)i] = mixing_mask(gt.k, gt.g);
        for (int j = 0; j < gt.k; ++j) {
            if (gt.shifts[j] < 0 || gt.shifts[j] >= n_total || gt.shifts[j] >= 64)
                return set_error(DIAQ_ERR_SHAPE, "gate shift %d outside state of %d qubits", gt.shifts[j], n_total);
            gqm[(size_t)i] |= 1ull << gt.shifts[j];
            if (((gmix[(size_t)i] >> j) & 1u) && gt.shifts[j] >= n_bits)
                return set_error(DIAQ_ERR_VALUE, "gate mixes global bit %d: it needs the partner shard", gt.shifts[j]);
        }
    }
    const uint64_t allq = n_total >= 64 ? ~0ull : ((1ull << n_total) - 1ull);
    // One sweep over `pending` builds one pass (program order: every pass).
    // reorder (contracted arithmetic only): a gate that does not fit the open
    // pass is deferred instead of closing it, and the scan goes on -- later
    // gates on other qubits commute with it and may still join.  Any gate
    // sharing a qubit with a deferred one is deferred too (program order per
    // qubit is kept), and the deferred gates, in order, form the next sweep.
    // Reordering gates on disjoint qubits is exact in real arithmetic but
    // changes the rounding, so the bitwise modes keep the program order.
    //   preset != 0 (lookahead): the pass's tile bits are fixed before the
    // sweep, and a gate whose mixing bits are not among them is deferred.
    //   dry: a lookahead trial -- nothing is flushed or emitted; *score is
    // the value of the pass this sweep would build.
    // reorder: phases per pass are capped where the shared-memory round trips
    // stop hiding under the pass's HBM time (each phase moves every amplitude
    // through shared memory once: ncu r02u shows deep passes at 73-81% of the
    // shared-memory pipe); a gate that would open one more phase is deferred
    const int maxph = reorder ? std::max(1, std::min(tuning().fused_maxph, kMaxPhases)) : kMaxPhases;
    uint64_t preset = 0;
    uint64_t tailq = 0;      // qubits of the tail's permutation gates
    int nrec = 0;            // gate records of the open pass (its non-permutation members)
    // phases the open pass needs so far -- the count flush() will arrive at
    // (exact without dense two-qubit gates, an upper bound with them)
    int nph = 0;
    bool ph_open = false, ph_generic = false, has_d2 = false;
    uint64_t ph_used = 0;
    std::vector<int> run_base;  // operands outside the tile of the open permutation run (one folded map)
    auto reset2 = [&]() {
        reset();
        if (preset) {
            nb = 0;
            for (int b = 0; b < 64; ++b) {
                inb[b] = (char)((preset >> b) & 1ull);
                nb += inb[b];
            }
        }
        tailq = 0;
        nrec = nph = 0;
        ph_open = ph_generic = has_d2 = false;
        ph_used = 0;
        run_base.clear();
    };
    auto sweep = [&](const std::vector<int> &pending, std::vector<int> *deferred_out, bool dry, int *score) -> int {
        uint64_t blocked = 0;
        int sc = 0;
        const bool fixed = preset != 0;
        for (size_t pi = 0; pi < pending.size(); ++pi) {
            const int i = pending[pi];
            if (reorder && blocked == allq) {  // nothing further can join
                if (deferred_out) deferred_out->insert(deferred_out->end(), pending.begin() + (long)pi, pending.end());
                break;
            }
            const diaq_gate_t &gt = gates[i];
            const uint64_t qmask = gqm[(size_t)i];
            auto defer = [&]() {
                if (deferred_out) deferred_out->push_back(i);
                blocked |= qmask;
            };
            if (reorder && (qmask & blocked)) {
                defer();
                continue;
            }
            const uint32_t mix = gmix[(size_t)i];
            uint64_t mixq = 0;
            int kin = 0, kout = 0, add = 0;
            for (int j = 0; j < gt.k; ++j) {
                if ((mix >> j) & 1u) {
                    ++kin;
                    add += inb[gt.shifts[j]] ? 0 : 1;
                    mixq |= 1ull << gt.shifts[j];
                } else {
                    ++kout;
                }
            }
            const bool pg = perm[(size_t)i].ok;
            // reorder: an open pass never closes inside a sweep; a fixed tile also defers from an empty pass
            const bool can_defer = reorder && (!members.empty() || fixed || dry);
            bool before_tail = false;
            if (!pg && tail != SIZE_MAX) {  // a gate after a global permutation tail opens the next pass ...
                if (reorder) {
                    if (qmask & tailq) {
                        defer();
                        continue;
                    }
                    before_tail = true;  // ... unless it shares no qubit with the tail: it commutes exactly, and joins the body
                } else {
                    int rc = flush();
                    if (rc) return rc;
                    reset2();
                    add = kin;
                    for (int j = 0; j < gt.k; ++j)
                        if (((mix >> j) & 1u) && inb[gt.shifts[j]]) --add;
                }
            }
            // operands outside the tile this permutation adds to the open run's folded map
            int padd = 0;
            if (pg)
                for (int j = 0; j < gt.k; ++j)
                    if (!((mix >> j) & 1u) && !inb[gt.shifts[j]] &&
                        std::find(run_base.begin(), run_base.end(), gt.shifts[j]) == run_base.end())
                        ++padd;
            // phases after this gate
            const bool isd2 = d2[(size_t)i] != 0;
            const bool fastg = fast[(size_t)i] || isd2;
            int nph_after = nph;
            if (pg) {
                nph_after += ph_generic ? 1 : 0;
            } else if (!fastg) {
                nph_after += 1;
            } else if (has_d2 || isd2) {
                nph_after += 1;
            } else if (!(ph_open && __builtin_popcountll(ph_used | mixq) <= R)) {
                nph_after += 1;
            }
            const bool room = nrec + (pg ? 0 : 1) <= kMaxPassGates && nph_after <= maxph;
            if (pg && !members.empty() && tuning().fused_gperm && !t_no_gperm) {
                // a permutation that does not fit the tile (or follows one that did
                // not) joins the pass's global tail instead of opening a pass
                if (tail != SIZE_MAX || kin > T - low || nb + add > T || (int)run_base.size() + padd > kMaxPermBase || !room) {
                    // the tail must keep 128-byte rows whole (its store writes whole
                    // rows): no output bit above the row may depend on a row bit,
                    // else partial-sector writes cost read-modify-write traffic
                    GlobalAffine trial;
                    if (tail == SIZE_MAX) trial.init(n_bits);
                    else trial = tail_map;
                    bool rows = trial.fold(gt, perm[(size_t)i]);
                    for (int o = low; o < n_bits && rows && tuning().fused_gperm_rows; ++o)
                        if (trial.row[o].m & ((1ull << low) - 1ull)) rows = false;
                    if (rows) {
                        tail_map = trial;
                        if (tail == SIZE_MAX) tail = members.size();
                        members.push_back(i);
                        tailq |= qmask;
                        sc += 1;
                        continue;
                    }
                    // it opens the next pass, where its bits can join the tile
                    if (reorder) {
                        defer();
                        continue;
                    }
                    int rc = flush();
                    if (rc) return rc;
                    reset2();
                    add = kin;
                    for (int j = 0; j < gt.k; ++j)
                        if (((mix >> j) & 1u) && inb[gt.shifts[j]]) --add;
                    padd = 0;
                    for (int j = 0; j < gt.k; ++j)
                        if (!((mix >> j) & 1u) && !inb[gt.shifts[j]]) ++padd;
                    nph_after = 0;
                }
            }
            if (pg ? (kin > T - low) : (kin > kMaxRegKin || kin > R || kout > kMaxSel)) {  // standalone pass
                if (can_defer) {  // its own pass, after the open one
                    defer();
                    continue;
                }
                int rc = flush();
                if (rc) return rc;
                reset2();
                PassPlan ps;
                ps.members = {i};
                plan.push_back(ps);
                continue;
            }
            const int gcoef = pg ? 0 : (1 << kout) << (2 * kin), gnz = pg ? 0 : (1 << kout) << kin;
            if (nb + add > T || nrec + (pg ? 0 : 1) > kMaxPassGates || nph_after > maxph ||
                (int)run_base.size() + padd > kMaxPermBase || ncoef + gcoef > kMaxCoef || nnz + gnz > kMaxNz) {
                if (can_defer) {
                    defer();
                    continue;
                }
                int rc = flush();
                if (rc) return rc;
                reset2();
                before_tail = false;
                add = kin;
                for (int j = 0; j < gt.k; ++j)
                    if (((mix >> j) & 1u) && inb[gt.shifts[j]]) --add;
            }
            for (int j = 0; j < gt.k; ++j)
                if (((mix >> j) & 1u) && !inb[gt.shifts[j]]) { inb[gt.shifts[j]] = 1; ++nb; }
            // bookkeeping as flush() will build the phases
            if (pg) {
                for (int j = 0; j < gt.k; ++j)
                    if (!((mix >> j) & 1u) && !inb[gt.shifts[j]] &&
                        std::find(run_base.begin(), run_base.end(), gt.shifts[j]) == run_base.end())
                        run_base.push_back(gt.shifts[j]);
                if (ph_generic) ++nph;  // an empty register phase carries the run
                ph_generic = false;
                ph_open = false;
                sc += 1;
            } else {
                run_base.clear();  // the next permutation run is a new map
                ++nrec;
                if (!fastg) {
                    ++nph;
                    ph_open = false;
                    ph_generic = true;
                } else {
                    ph_generic = false;
                    if (has_d2 || isd2) {
                        ++nph;
                        has_d2 = true;
                        ph_open = false;
                    } else if (ph_open && __builtin_popcountll(ph_used | mixq) <= R) {
                        ph_used |= mixq;
                    } else {
                        ++nph;
                        ph_open = true;
                        ph_used = mixq;
                    }
                }
                sc += kin > 0 ? 4 : 1;
            }
            ncoef += gcoef;
            nnz += gnz;
            if (before_tail) {
                members.insert(members.begin() + (long)tail, i);
                ++tail;
            } else {
                members.push_back(i);
            }
        }
        if (score) *score = sc;
        return DIAQ_OK;
    };
    // ---- slot sweep (reorder only, knob fused_slots) ------------------------
    // The pass is built as a list of phase slots instead of one open phase:
    // a gate goes into the EARLIEST slot that follows the last gate on each
    // of its qubits and has register bits left for it (gates on other
    // qubits in later slots commute with it), so one phase takes several
    // layers' gates on its four qubits.  An X / CX / SWAP whose operands are
    // register bits of its slot is applied there as a register exchange
    // (no arithmetic, a renaming in the specialised kernels) and the slot
    // stays open; any other permutation is folded into its slot's store.
    struct Slot {
        std::vector<int> body;
        std::vector<char> rperm;
        std::vector<int> post;      // folded permutations, in order
        std::vector<int> base;      // their operands outside the tile (one folded map)
        uint64_t used = 0;          // state bits taken as register bits
        int ndiag = 0;              // one-selector diagonal gates of the body (most lead it as one run)
        bool generic = false, has_d2 = false, seq_ok = true;
    };
    std::vector<Slot> slots;
    std::vector<int> prev, prebase, tailv;  // permutations opening the pass / their outside operands / global tail
    int lastph[64];
    bool lastpost[64];
    int barrier = -1;  // slot of the last shared-memory (generic) gate: every later gate follows it
    const bool use_slots = reorder && tuning().fused_slots != 0;
    auto reset_slots = [&]() {
        reset2();
        slots.clear();
        prev.clear();
        prebase.clear();
        tailv.clear();
        for (int b = 0; b < 64; ++b) { lastph[b] = -2; lastpost[b] = false; }
        barrier = -1;
    };
    auto sweep_slots = [&](const std::vector<int> &pending, std::vector<int> *deferred_out, bool dry, int *score) -> int {
        uint64_t blocked = 0;
        int sc = 0;
        bool any = false;  // the pass has a member
        std::vector<std::pair<int, int>> rops;
        for (size_t pi = 0; pi < pending.size(); ++pi) {
            const int i = pending[pi];
            if (blocked == allq) {
                if (deferred_out) deferred_out->insert(deferred_out->end(), pending.begin() + (long)pi, pending.end());
                break;
            }
            const diaq_gate_t &gt = gates[i];
            const uint64_t qmask = gqm[(size_t)i];
            auto defer = [&]() {
                if (deferred_out) deferred_out->push_back(i);
                blocked |= qmask;
            };
            if (qmask & blocked) {
                defer();
                continue;
            }
            const uint32_t mix = gmix[(size_t)i];
            uint64_t mixq = 0;
            int kin = 0, kout = 0, add = 0;
            for (int j = 0; j < gt.k; ++j) {
                if ((mix >> j) & 1u) {
                    ++kin;
                    add += inb[gt.shifts[j]] ? 0 : 1;
                    mixq |= 1ull << gt.shifts[j];
                } else {
                    ++kout;
                }
            }
            const bool pg = perm[(size_t)i].ok;
            const bool standalone = pg ? (kin > T - low) : (kin > kMaxRegKin || kin > R || kout > kMaxSel);
            if (standalone) {
                if (any || preset || dry) {
                    defer();
                    continue;
                }
                PassPlan ps;  // first in order and nothing open: its own pass now
                ps.members = {i};
                plan.push_back(ps);
                continue;
            }
            // the slot this gate must follow on each of its qubits
            int kmin = barrier + 1;
            bool after_post = false;
            for (int j = 0; j < gt.k; ++j) {
                const int q = gt.shifts[j];
                if (lastph[q] == -2) continue;
                const int need = (pg || !lastpost[q]) ? lastph[q] : lastph[q] + 1;  // a permutation may join the same store
                if (need > kmin) kmin = need;
            }
            if (pg) {
                // global tail: its target leaves the tile (or it follows the tail on a shared qubit)
                const bool fits_tile = tailv.empty() && kin <= T - low && nb + add <= T;
                if (!fits_tile || (qmask & tailq)) {
                    if (!any || !tuning().fused_gperm || t_no_gperm) {
                        defer();
                        continue;
                    }
                    GlobalAffine trial_map;
                    if (tailv.empty()) trial_map.init(n_bits);
                    else trial_map = tail_map;
                    bool rows = trial_map.fold(gt, perm[(size_t)i]);
                    for (int o = low; o < n_bits && rows && tuning().fused_gperm_rows; ++o)
                        if (trial_map.row[o].m & ((1ull << low) - 1ull)) rows = false;
                    if (!rows) {
                        defer();
                        continue;
                    }
                    tail_map = trial_map;
                    tailv.push_back(i);
                    tailq |= qmask;
                    sc += 1;
                    continue;
                }
                // in the tile: a register exchange in slot kmin, or folded into its store
                for (int j = 0; j < gt.k; ++j) after_post = after_post || (lastph[gt.shifts[j]] == kmin && lastpost[gt.shifts[j]]);
                bool done = false;
                if (kmin >= 0 && kmin < (int)slots.size() && !after_post && rperm_ops(gt, perm[(size_t)i], rops)) {
                    Slot &sl = slots[(size_t)kmin];
                    bool in_tile = true;
                    for (int j = 0; j < gt.k; ++j) in_tile = in_tile && inb[gt.shifts[j]];
                    if (in_tile && !sl.generic && !sl.has_d2 && __builtin_popcountll(sl.used | qmask) <= R &&
                        nrec + (int)rops.size() <= kMaxPassGates &&
                        (int)sl.body.size() - sl.ndiag + (int)rops.size() <= tuning().fused_slot_gates) {
                        sl.body.push_back(i);
                        sl.rperm.push_back(1);
                        sl.used |= qmask;
                        sl.seq_ok = false;
                        nrec += (int)rops.size();
                        for (int j = 0; j < gt.k; ++j) { lastph[gt.shifts[j]] = kmin; lastpost[gt.shifts[j]] = false; }
                        done = true;
                    }
                }
                if (!done) {
                    int k = kmin;
                    if (k >= (int)slots.size()) k = (int)slots.size() - 1;  // (barrier + 1 past the end: the last slot's store)
                    if (k >= 0 && slots[(size_t)k].generic) {  // a shared-memory phase has no store map: an empty register phase carries it
                        if (k + 1 < (int)slots.size()) {
                            k = k + 1;
                        } else {
                            if ((int)slots.size() + 1 > maxph) {
                                defer();
                                continue;
                            }
                            slots.emplace_back();
                            k = (int)slots.size() - 1;
                        }
                    }
                    std::vector<int> &base = k < 0 ? prebase : slots[(size_t)k].base;
                    int padd = 0;
                    for (int j = 0; j < gt.k; ++j)
                        if (!((mix >> j) & 1u) && !inb[gt.shifts[j]] &&
                            std::find(base.begin(), base.end(), gt.shifts[j]) == base.end())
                            ++padd;
                    if ((int)base.size() + padd > kMaxPermBase) {
                        defer();
                        continue;
                    }
                    for (int j = 0; j < gt.k; ++j)
                        if (!((mix >> j) & 1u) && !inb[gt.shifts[j]] &&
                            std::find(base.begin(), base.end(), gt.shifts[j]) == base.end())
                            base.push_back(gt.shifts[j]);
                    (k < 0 ? prev : slots[(size_t)k].post).push_back(i);
                    for (int j = 0; j < gt.k; ++j) { lastph[gt.shifts[j]] = k; lastpost[gt.shifts[j]] = true; }
                }
                for (int j = 0; j < gt.k; ++j)
                    if (((mix >> j) & 1u) && !inb[gt.shifts[j]]) { inb[gt.shifts[j]] = 1; ++nb; }
                any = true;
                sc += 1;
                continue;
            }
            // arithmetic gates
            if (qmask & tailq) {  // after the tail on a shared qubit
                defer();
                continue;
            }
            const int gcoef = (1 << kout) << (2 * kin), gnz = (1 << kout) << kin;
            if (nb + add > T || nrec + 1 > kMaxPassGates || ncoef + gcoef > kMaxCoef || nnz + gnz > kMaxNz) {
                defer();
                continue;
            }
            const bool isd2 = d2[(size_t)i] != 0;
            const bool fastg = fast[(size_t)i] || isd2;
            if (kmin < 0) kmin = 0;
            int k = -1;
            if (fastg) {
                for (int c = kmin; c < (int)slots.size() && k < 0; ++c) {
                    const Slot &sl = slots[(size_t)c];
                    if (sl.generic) continue;
                    // (the specialised kernels unroll a phase's gate loop only up to a size)
                    if ((int)sl.body.size() - sl.ndiag >= tuning().fused_slot_gates) continue;
                    const int fresh = __builtin_popcountll(mixq & ~sl.used);
                    if (__builtin_popcountll(sl.used | mixq) > R) continue;
                    // as flush(): dense two-qubit gates only in sequence phases
                    bool keeps = fresh == kin;
                    if (kin == 0 && (qmask & sl.used)) keeps = false;
                    if (!(keeps || (!sl.has_d2 && !isd2)) || (isd2 && !sl.seq_ok)) continue;
                    k = c;
                }
            }
            if (k < 0) {  // a new slot at the end
                if ((int)slots.size() + 1 > maxph) {
                    defer();
                    continue;
                }
                slots.emplace_back();
                k = (int)slots.size() - 1;
                if (!fastg) {
                    slots.back().generic = true;
                    barrier = k;
                }
            }
            Slot &sl = slots[(size_t)k];
            if (fastg) {
                const int fresh = __builtin_popcountll(mixq & ~sl.used);
                bool keeps = fresh == kin;
                if (kin == 0 && (qmask & sl.used)) keeps = false;
                sl.seq_ok = sl.seq_ok && keeps;
                sl.has_d2 = sl.has_d2 || isd2;
                sl.used |= mixq;
            }
            sl.body.push_back(i);
            sl.rperm.push_back(0);
            if (fastg && kin == 0) ++sl.ndiag;
            for (int j = 0; j < gt.k; ++j) {
                lastph[gt.shifts[j]] = k;
                lastpost[gt.shifts[j]] = sl.generic;  // nothing joins a shared-memory phase
            }
            for (int j = 0; j < gt.k; ++j)
                if (((mix >> j) & 1u) && !inb[gt.shifts[j]]) { inb[gt.shifts[j]] = 1; ++nb; }
            ++nrec;
            ncoef += gcoef;
            nnz += gnz;
            any = true;
            sc += kin > 0 ? 4 : 1;
        }
        if (score) *score = sc;
        if (dry) return DIAQ_OK;
        // members in execution order, for flush_slots()
        members.clear();
        members.insert(members.end(), prev.begin(), prev.end());
        for (const Slot &sl : slots) {
            members.insert(members.end(), sl.body.begin(), sl.body.end());
            members.insert(members.end(), sl.post.begin(), sl.post.end());
        }
        members.insert(members.end(), tailv.begin(), tailv.end());
        return DIAQ_OK;
    };
    auto flush_slots = [&]() -> int {
        if (members.empty()) return DIAQ_OK;
        PassPlan ps;
        tile_bits_of(ps);
        ps.members = members;
        const int TT = (int)ps.bits.size();
        HostAffine pre;
        pre.init(TT);
        for (const int gi : prev)
            if (!pre.fold(gates[gi], perm[(size_t)gi], ps.bits))
                return set_error(DIAQ_ERR_VALUE, "fused pass: permutation fold overflow");
        std::vector<Spec> specs;
        for (const Slot &sl : slots) {
            Spec sp;
            sp.generic = sl.generic ? 1 : 0;
            // diagonal gates on bits that are not register bits of the slot commute with every
            // other gate of its body (those act on register bits): they lead it, as one run
            if (!sl.generic) {
                for (int part = 0; part < 2; ++part)
                    for (size_t mi = 0; mi < sl.body.size(); ++mi) {
                        const diaq_gate_t &gt = gates[sl.body[mi]];
                        const bool lead = !sl.rperm[mi] && gmix[(size_t)sl.body[mi]] == 0u && gt.k == 1 &&
                                          fast[(size_t)sl.body[mi]] && !(gqm[(size_t)sl.body[mi]] & sl.used);
                        if (lead == (part == 0)) {
                            sp.mem.push_back(sl.body[mi]);
                            sp.rperm.push_back(sl.rperm[mi]);
                        }
                    }
            } else {
                sp.mem = sl.body;
                sp.rperm = sl.rperm;
            }
            sp.has_d2 = sl.has_d2;
            sp.post.init(TT);
            for (size_t mi = 0; mi < sp.mem.size(); ++mi) {  // register bits in first-use order
                const diaq_gate_t &gt = gates[sp.mem[mi]];
                const uint32_t mix = gmix[(size_t)sp.mem[mi]];
                std::vector<int> ops;
                for (int o = 0; o < gt.k; ++o)
                    if (sp.rperm[mi] || ((mix >> o) & 1u)) ops.push_back(o);
                std::sort(ops.begin(), ops.end(), [&](int a, int b) { return gt.shifts[a] > gt.shifts[b]; });
                for (const int o : ops) {
                    const int tp = tile_pos(ps.bits, gt.shifts[o]);
                    if (!sl.generic && std::find(sp.used.begin(), sp.used.end(), tp) == sp.used.end()) sp.used.push_back(tp);
                }
            }
            for (const int gi : sl.post)
                if (!sp.post.fold(gates[gi], perm[(size_t)gi], ps.bits))
                    return set_error(DIAQ_ERR_VALUE, "fused pass: permutation fold overflow");
            specs.push_back(sp);
        }
        return finish(ps, specs, pre, tailv);
    };
    std::vector<int> pending((size_t)ngates);
    for (int i = 0; i < ngates; ++i) pending[(size_t)i] = i;
    if (!reorder) {
        reset2();
        int rc = sweep(pending, nullptr, false, nullptr);
        if (rc) return rc;
        return flush();
    }
    // Lookahead (reorder only): first fit takes tile bits in the order the
    // gates ask for them; a pass is worth more when its tile holds qubits
    // whose CX partners are in the tile too, so their next layers' gates can
    // join.  Start from the first-fit tile and exchange one bit at a time
    // while the trial sweep's score grows.
    const bool look = tuning().fused_lookahead != 0 && n_bits > T;
    auto trial = [&](uint64_t bits) -> int {
        int sc = 0;
        preset = bits;
        if (use_slots) {
            reset_slots();
            if (sweep_slots(pending, nullptr, true, &sc) != DIAQ_OK) sc = -1;
        } else {
            reset2();
            if (sweep(pending, nullptr, true, &sc) != DIAQ_OK) sc = -1;
        }
        return sc;
    };
    auto real_sweep = [&](std::vector<int> &deferred) -> int {
        if (use_slots) {
            reset_slots();
            return sweep_slots(pending, &deferred, false, nullptr);
        }
        reset2();
        return sweep(pending, &deferred, false, nullptr);
    };
    while (!pending.empty()) {
        uint64_t choice = 0;
        if (look) {
            const int sc0 = trial(0);
            uint64_t bits = 0;
            int nbits = 0;
            for (int b = 0; b < 64; ++b)
                if (inb[b]) { bits |= 1ull << b; ++nbits; }
            for (int b = 0; nbits < T && b < n_bits; ++b)
                if (!((bits >> b) & 1ull)) { bits |= 1ull << b; ++nbits; }
            int best = nbits == T ? trial(bits) : -1;
            bool improved = best >= 0;
            for (int it = 0; improved && it < 64; ++it) {
                improved = false;
                for (int out = low; out < n_bits && !improved; ++out) {
                    if (!((bits >> out) & 1ull)) continue;
                    for (int in = low; in < n_bits && !improved; ++in) {
                        if ((bits >> in) & 1ull) continue;
                        const uint64_t cand = (bits & ~(1ull << out)) | (1ull << in);
                        const int sc = trial(cand);
                        if (sc > best) {
                            best = sc;
                            bits = cand;
                            improved = true;
                        }
                    }
                }
            }
            if (best > sc0) choice = bits;
        }
        std::vector<int> deferred;
        preset = choice;
        const size_t plan0 = plan.size();
        int rc = real_sweep(deferred);
        if (rc) return rc;
        if (members.empty() && plan.size() == plan0) {
            if (!choice) return set_error(DIAQ_ERR_VALUE, "fused schedule made no progress");
            deferred.clear();  // the fixed tile admitted nothing: first fit
            preset = 0;
            rc = real_sweep(deferred);
            if (rc) return rc;
        }
        rc = use_slots ? flush_slots() : flush();
        if (rc) return rc;
        pending.swap(deferred);
    }
    preset = 0;
    return DIAQ_OK;
}

static int schedule(int n_bits, int n_total, int ngates, const diaq_gate_t *gates, int T, int R,
                    std::vector<PassPlan> &plan) {
    int rc = schedule_once(n_bits, n_total, ngates, gates, T, R, plan, true);
    if (rc == kRetryNoDense2) {  // a two-qubit gate landed outside a sequence phase: shared-memory path for all
        plan.clear();
        rc = schedule_once(n_bits, n_total, ngates, gates, T, R, plan, false);
    }
    return rc;
}

int apply_gate(int n_bits, int k, const double *g, const int *shifts, const void *x, void *y, int cmul_mode,
               cudaStream_t s);
int apply_gate_sharded_own(int n_bits, int local_bits, int k, const double *g, const int *shifts, int64_t rank,
                           void *shard, int cmul_mode, cudaStream_t s);

template <int R>
static const void *tile_kernel_ptr(int cmul_mode) {
    return cmul_mode == DIAQ_CMUL_CONTRACT ? (const void *)tile_pass_kernel<R, DIAQ_CMUL_CONTRACT>
           : cmul_mode == DIAQ_CMUL_FMA    ? (const void *)tile_pass_kernel<R, DIAQ_CMUL_FMA>
                                           : (const void *)tile_pass_kernel<R, DIAQ_CMUL_PLAIN>;
}

static const void *tile_kernel_t7_ptr(int cmul_mode) {
    return cmul_mode == DIAQ_CMUL_CONTRACT ? (const void *)tile_pass_kernel_t7<DIAQ_CMUL_CONTRACT>
           : cmul_mode == DIAQ_CMUL_FMA    ? (const void *)tile_pass_kernel_t7<DIAQ_CMUL_FMA>
                                           : (const void *)tile_pass_kernel_t7<DIAQ_CMUL_PLAIN>;
}

}  // namespace diaq

using namespace diaq;

// A scheduled and packed gate program.  Scheduling 10^3 gates costs about a
// millisecond of host time -- as much as the passes themselves at n = 20 --
// so the last few programs are kept per thread, keyed by the exact gate data,
// each pass already in its launch-parameter form.
struct Program {
    std::vector<char> key;
    std::vector<PassPlan> plan;
    std::vector<TileParams> params;  // per tiled pass (x, gbase and the grid are filled in at launch)
    // specialised kernels of the tiled passes (fused_jit.cu), per cmul mode:
    // looked up once per program, then read on every call
    mutable std::mutex jit_mu;
    mutable std::vector<std::shared_ptr<JitPass>> jit[3];
    mutable bool jit_requested[3] = {false, false, false};

    std::vector<const TileParams *> tiled() const {
        std::vector<const TileParams *> v(plan.size(), nullptr);
        for (size_t i = 0; i < plan.size(); ++i)
            if (!(plan[i].bits.empty() || plan[i].members.size() == 1)) v[i] = &params[i];
        return v;
    }
};

static void debug_plan(const std::vector<PassPlan> &plan) {
    {
        for (size_t i = 0; i < plan.size(); ++i) {
            const PassPlan &ps = plan[i];
            fprintf(stderr, "pass %zu: %zu gates, bits", i, ps.members.size());
            for (int b : ps.bits) fprintf(stderr, " %d", b);
            fprintf(stderr, "%s\n", ps.pre.on ? " [pre-perm]" : "");
            for (const Phase &ph : ps.phases)
                fprintf(stderr, "  phase g[%d,%d) generic=%d seq=%d ndense=%d post=%d rpos %d %d %d %d\n", ph.g0, ph.g1,
                        ph.generic, ph.seq, ph.ndense, ph.post.on, ph.rpos[0], ph.rpos[1], ph.rpos[2], ph.rpos[3]);
        }
    }
}

static std::vector<char> program_key(int n_total, int n_bits, int T, int ngates, const diaq_gate_t *gates) {
    std::vector<char> key;
    auto put = [&](const void *p, size_t n) {
        const char *c = (const char *)p;
        key.insert(key.end(), c, c + n);
    };
    // every tuning switch the schedule depends on is part of the key
    const int head[18] = {n_total, n_bits, T, pass_tbits(), ngates, (int)t_reorder, (int)t_unit,
                          t_reorder ? tuning().fused_lookahead + 2 * tuning().fused_slots + 256 * tuning().fused_maxph +
                                          65536 * tuning().fused_slot_gates
                                    : 0,
                          tuning().fused_perm,
                          tuning().fused_gperm && !t_no_gperm, tuning().fused_seq, tuning().fused_dense2,
                          tuning().fused_gperm_rows, tuning().fused_pair_store, tuning().fused_bank_spread, tuning().fused_plain_pair, tuning().fused_ppipe, tuning().fused_dstore};
    put(head, sizeof(head));
    for (int i = 0; i < ngates; ++i) {
        const diaq_gate_t &gt = gates[i];
        put(&gt.k, sizeof(int));
        if (gt.k < 1 || gt.k > 5) continue;  // rejected by schedule()
        put(gt.shifts, sizeof(int) * gt.k);
        put(gt.g, sizeof(double) * 2 * ((size_t)1 << (2 * gt.k)));
    }
    return key;
}

// Linear algebra over GF(2) on 64-bit vectors: span membership and
// solutions of A x = v for A given by its columns.
struct Gf2 {
    std::vector<std::pair<uint64_t, uint64_t>> rows;  // (reduced vector, combination of inputs), distinct top bits
    // reduce v against the rows (highest pivots first); c tracks the combination
    void reduce(uint64_t &v, uint64_t &c) const {
        for (const auto &r : rows)
            if (v & (1ull << (63 - __builtin_clzll(r.first)))) {
                v ^= r.first;
                c ^= r.second;
            }
    }
    bool add(uint64_t v, uint64_t tag) {  // false if v is in the span already
        uint64_t c = tag;
        reduce(v, c);
        if (!v) return false;
        rows.emplace_back(v, c);
        std::sort(rows.begin(), rows.end(), [](const auto &a, const auto &b) { return a.first > b.first; });
        // keep the rows fully reduced against each other's pivots (a new pivot
        // may sit inside an older row)
        for (size_t i = 0; i < rows.size(); ++i)
            for (size_t j = 0; j < rows.size(); ++j)
                if (i != j && (rows[j].first & (1ull << (63 - __builtin_clzll(rows[i].first))))) {
                    rows[j].first ^= rows[i].first;
                    rows[j].second ^= rows[i].second;
                }
        std::sort(rows.begin(), rows.end(), [](const auto &a, const auto &b) { return a.first > b.first; });
        return true;
    }
    bool solve(uint64_t v, uint64_t &x) const {
        uint64_t c = 0;
        reduce(v, c);
        x = c;
        return v == 0;
    }
};

// Pair store of a pass's global tail (TileParams::gnp): the extra bit G
// whose tiles must be stored together so every 32-byte destination sector
// (rows, when cheap) is written whole by one CTA.  gcol = A's columns.
static void plan_pair_store(const PassPlan &ps, int n_bits, TileParams &p) {
    p.gnp = 0;
    if (!ps.gon || n_bits > 63) return;
    Gf2 a;
    for (int j = 0; j < n_bits; ++j) a.add(ps.gcol[(size_t)j], 1ull << j);
    if ((int)a.rows.size() != n_bits) return;  // not invertible (cannot happen for permutations)
    uint64_t tmask = 0;
    for (int b : ps.bits) tmask |= 1ull << b;
    uint64_t x[3];
    for (int j = 0; j < 3; ++j)
        if (!a.solve(1ull << j, x[j])) return;
    uint64_t G = (x[0] | x[1] | x[2]) & ~tmask;         // whole rows
    if (__builtin_popcountll(G) > 1) G = x[0] & ~tmask;  // whole sectors
    if (__builtin_popcountll(G) != 1) return;           // rows whole already / a pair does not close them
    const int T = (int)ps.bits.size();
    p.gnp = (int8_t)__builtin_popcountll(G);
    for (int k = 0, b = 0; b < 64; ++b)
        if ((G >> b) & 1ull) p.gpb[k++] = (int8_t)b;
    p.emask = tmask | G;
    for (int k = 0, b = 0; b < 64; ++b)
        if ((p.emask >> b) & 1ull) p.eb[k++] = (int8_t)b;
    // destination basis: e0 (e1, e2 when in the span) first, then images of the group bits
    Gf2 span, basis;
    std::vector<int> gbits;
    for (int b = 0; b < 64; ++b)
        if ((p.emask >> b) & 1ull) gbits.push_back(b);
    for (int b : gbits) span.add(ps.gcol[(size_t)b], 0);
    std::vector<uint64_t> w;
    for (int j = 0; j < 3; ++j) {
        uint64_t dummy;
        if (span.solve(1ull << j, dummy) && basis.add(1ull << j, 0)) w.push_back(1ull << j);
    }
    for (int b : gbits)
        if ((int)w.size() < T + p.gnp && basis.add(ps.gcol[(size_t)b], 0)) w.push_back(ps.gcol[(size_t)b]);
    if ((int)w.size() != T + p.gnp) {
        p.gnp = 0;
        return;
    }
    for (int k = 0; k < T + p.gnp; ++k) {
        uint64_t src;
        if (!a.solve(w[(size_t)k], src) || (src & ~p.emask)) {
            p.gnp = 0;
            return;
        }
        uint32_t off = 0, rank = 0;
        for (int j = 0; j < T; ++j)
            if ((src >> ps.bits[(size_t)j]) & 1ull) off |= 1u << j;
        for (int j = 0; j < p.gnp; ++j)
            if ((src >> p.gpb[j]) & 1ull) rank |= 1u << j;
        p.gw[k] = w[(size_t)k];
        p.gsrc[k] = (uint16_t)(off | (rank << 12));
    }
    // lanes 1-2 (thread bits 1-2; bit 0 keeps the sector partner e0): the
    // destination basis vectors whose sources spread the quarter warp's
    // gather reads over the most smem bank groups (fused_bank_spread & 2)
    if (!(tuning().fused_bank_spread & 2) || T + p.gnp < 4) return;
    auto bank = [&](int k) { return swz(p.gsrc[k] & 0xfffu) & 7u; };
    auto distinct = [](uint32_t a, uint32_t b, uint32_t c) {
        uint32_t seen = 0;
        for (int m = 0; m < 8; ++m) seen |= 1u << (((m & 1) ? a : 0) ^ ((m & 2) ? b : 0) ^ ((m & 4) ? c : 0));
        return __builtin_popcount(seen);
    };
    const int nw = T + p.gnp;
    int b1 = 1, b2 = 2, best = distinct(bank(0), bank(1), bank(2));
    for (int i = 1; i < nw && best < 8; ++i)
        for (int j = i + 1; j < nw && best < 8; ++j) {
            const int d = distinct(bank(0), bank(i), bank(j));
            if (d > best) best = d, b1 = i, b2 = j;
        }
    if (b1 == 1 && b2 == 2) return;
    uint64_t gw[kMaxTileBits + 3];
    uint16_t gs[kMaxTileBits + 3];
    int q = 0;
    gw[q] = p.gw[0], gs[q++] = p.gsrc[0];
    gw[q] = p.gw[b1], gs[q++] = p.gsrc[b1];
    gw[q] = p.gw[b2], gs[q++] = p.gsrc[b2];
    for (int k = 1; k < nw; ++k)
        if (k != b1 && k != b2) gw[q] = p.gw[k], gs[q++] = p.gsrc[k];
    for (int k = 0; k < nw; ++k) p.gw[k] = gw[k], p.gsrc[k] = gs[k];
}

static std::shared_ptr<const Program> build_program(int n_total, int n_bits, int T, int ngates, const diaq_gate_t *gates,
                                                    int &rc) {
    auto prog = std::make_shared<Program>();
    std::vector<PassPlan> &plan = prog->plan;
    if (n_bits >= T) {
        rc = schedule(n_bits, n_total, ngates, gates, T, T - pass_tbits(), plan);
        if (rc) return nullptr;
    } else {  // state smaller than a tile: gate by gate (standalone path)
        for (int i = 0; i < ngates; ++i) {
            PassPlan ps;
            ps.members = {i};
            plan.push_back(ps);
        }
    }
    if (getenv("DIAQ_PLAN_DEBUG")) debug_plan(plan);
    prog->params.resize(plan.size());
    for (size_t i = 0; i < plan.size(); ++i) {
        const PassPlan &ps = plan[i];
        if (ps.bits.empty() || ps.members.size() == 1) continue;  // standalone gate
        if ((int)ps.phases.size() > kMaxPhases || (int)ps.gates.size() > kMaxPassGates ||
            (int)ps.pk.coef.size() > kMaxCoef || (int)ps.pk.nz.size() > kMaxNz) {
            rc = set_error(DIAQ_ERR_VALUE, "fused pass exceeds its parameter tables");
            return nullptr;
        }
        TileParams &p = prog->params[i];
        memset(&p, 0, sizeof(p));
        p.tbits = (int)ps.bits.size();
        for (int j = 0; j < p.tbits; ++j) {
            p.tb[j] = ps.bits[j];
            p.tmask |= 1ull << ps.bits[j];
        }
        p.ntiles = (int64_t)1 << (n_bits - p.tbits);
        p.nphases = (int)ps.phases.size();
        p.ngates = (int)ps.gates.size();
        p.ncoef = (int)ps.pk.coef.size();
        p.nnz = (int)ps.pk.nz.size();
        p.pre = ps.pre;
        p.gperm = ps.gon ? 1 : 0;
        if (ps.gon) {
            for (size_t j = 0; j < ps.gcol.size() && j < 64; ++j) p.gcol[j] = ps.gcol[j];
            p.gconst = ps.gc;  // rank bits folded in at launch
            // a pair of 12-bit tiles needs 128 KB of smem (one CTA per SM):
            // per pass it beats the scatter store's partial-sector writes or
            // not (6.4-27 ms vs 8.2-14 ms at n=30, tools/pass_times.py);
            // over the config-5 program it wins (knob 2: 453 vs 471 ms)
            const int pst = tuning().fused_pair_store;
            if (pst >= 2 || (pst == 1 && (int)ps.bits.size() <= 11)) plan_pair_store(ps, n_bits, p);
        }
        if (!ps.gon && tuning().fused_plain_pair && n_bits > p.tbits) {
            int lowest = 0;  // lowest state bit outside the tile: tile rows are 2^lowest amplitudes
            while (lowest < n_bits && ((p.tmask >> lowest) & 1ull)) ++lowest;
            if (lowest == kLowBits) {
                p.ppair = 1;
                p.ppipe = (int8_t)tuning().fused_ppipe;

                p.gpb[0] = (int8_t)lowest;
                p.emask = p.tmask | (1ull << lowest);
                for (int k = 0, b = 0; b < 64; ++b)
                    if ((p.emask >> b) & 1ull) p.eb[k++] = (int8_t)b;
            }
        }
        std::copy(ps.phases.begin(), ps.phases.end(), p.ph);
        if (p.ppair && p.ppipe == 0 && tuning().fused_dstore && p.nphases > 0) {
            Phase &lp = p.ph[p.nphases - 1];
            const int R = p.tbits - pass_tbits();
            bool ok = !lp.generic && !lp.post.on && p.tbits - R >= kLowBits;
            for (int q = 0; q < R && ok; ++q) ok = lp.rpos[q] >= kLowBits;
            if (ok) {  // thread bits 0-2 on tile positions 0-2 (the lane-contiguous rows), the rest as before
                int8_t tp[kMaxTileBits];
                int m = 0;
                for (int b = 0; b < kLowBits; ++b) tp[m++] = (int8_t)b;
                for (int k = 0; k < p.tbits - R; ++k)
                    if (lp.tpos[k] >= kLowBits) tp[m++] = lp.tpos[k];
                for (int k = 0; k < p.tbits - R; ++k) lp.tpos[k] = tp[k];
                p.dstore = 1;
            }
        }
        std::copy(ps.gates.begin(), ps.gates.end(), p.g);
        std::copy(ps.pk.coef.begin(), ps.pk.coef.end(), p.coef);
        std::copy(ps.pk.nz.begin(), ps.pk.nz.end(), p.nz);
    }
    rc = DIAQ_OK;
    return prog;
}

static std::shared_ptr<const Program> cached_program(int n_total, int n_bits, int T, int ngates,
                                                     const diaq_gate_t *gates, int &rc) {
    constexpr size_t kKeep = 8;
    thread_local std::vector<std::shared_ptr<const Program>> cache;  // most recent first
    std::vector<char> key = program_key(n_total, n_bits, T, ngates, gates);
    for (size_t i = 0; i < cache.size(); ++i)
        if (cache[i]->key == key) {
            std::shared_ptr<const Program> hit = cache[i];
            cache.erase(cache.begin() + (long)i);
            cache.insert(cache.begin(), hit);
            rc = DIAQ_OK;
            return hit;
        }
    std::shared_ptr<const Program> prog = build_program(n_total, n_bits, T, ngates, gates, rc);
    if (!prog) return nullptr;
    const_cast<Program &>(*prog).key = std::move(key);
    cache.insert(cache.begin(), prog);
    if (cache.size() > kKeep) cache.pop_back();
    return prog;
}

// The out-of-place permutation buffer is as large as the state (4 GiB at
// n = 28) and is taken from the device's default stream-ordered pool on
// every call; the pool would hand that memory back to the driver at each
// synchronisation and re-map it on the next call (milliseconds).  Keep freed
// pool memory reserved instead (once per device); diaq_trim_pool releases it.
static void keep_pool_reserved() {
    static bool done[64] = {false};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) {
        cudaGetLastError();
        return;
    }
    if (done[dev]) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t thr = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    cudaGetLastError();
    done[dev] = true;
}

static int run_fused(int n_total, int n_bits, int64_t rank, int ngates, const diaq_gate_t *gates, void *state,
                     int cmul_mode, int tile_bits, void **events, int *npasses, void *stream) {
    if (ngates < 0 || (ngates > 0 && !gates) || !state)
        return set_error(DIAQ_ERR_VALUE, "diaq_run_gates_fused: bad arguments");
    if (cmul_mode < DIAQ_CMUL_PLAIN || cmul_mode > DIAQ_CMUL_CONTRACT)
        return set_error(DIAQ_ERR_VALUE, "diaq_run_gates_fused: cmul_mode %d", cmul_mode);
    t_reorder = cmul_mode == DIAQ_CMUL_CONTRACT && tuning().fused_reorder;
    t_unit = cmul_mode == DIAQ_CMUL_CONTRACT && tuning().fused_unit;
    const bool sharded = n_total > n_bits;
    cudaStream_t s = (cudaStream_t)stream;
    // tile_bits 12 -> 16 amplitudes per thread (R = 4), 11 -> 8 (R = 3); 256
    // threads.  tile_bits <= 0: schedule both and keep the cheaper: a 12-bit
    // pass costs ~1.14x an 11-bit one (2 vs 3 CTAs per SM; measured 1.13-1.14
    // over 20-layer programs at n=24/28/30), so 12 wins only with >12% fewer passes
    int T = tile_bits >= kThreadBits + 4 ? kThreadBits + 4 : kThreadBits + 3;
    if (pass_tbits() == 7) T = kThreadBits + 3;  // 128 threads x 16 amplitudes (R = 4 is the widest phase)
    int rc = DIAQ_OK;
    std::shared_ptr<const Program> prog = cached_program(n_total, n_bits, T, ngates, gates, rc);
    if (!prog) return rc;
    if (t_reorder) {
        // the reordered schedule only where it saves passes: at equal counts
        // program order keeps the work spread evenly (the reordered first
        // pass of an n=28 layer took 514M FP64 instructions against 268M
        // for the second, 1.85 + 1.45 ms, vs 371M / 442M and 1.52 + 1.70)
        t_reorder = false;
        std::shared_ptr<const Program> inorder = cached_program(n_total, n_bits, T, ngates, gates, rc);
        if (!inorder) return rc;
        if (inorder->plan.size() <= prog->plan.size()) prog = inorder;
        else t_reorder = true;
    }
    if (tile_bits <= 0 && pass_tbits() == 8) {
        T = kThreadBits + 3;
        std::shared_ptr<const Program> big = cached_program(n_total, n_bits, kThreadBits + 4, ngates, gates, rc);
        if (!big) return rc;
        if (114 * big->plan.size() < 100 * prog->plan.size()) {
            prog = big;
            T = kThreadBits + 4;
        }
    }
    const int R = T - pass_tbits();
    const int tbits = T - R;
    const std::vector<PassPlan> &plan = prog->plan;
    if (npasses) *npasses = (int)plan.size();
    // specialised kernels: requested once per (program, mode); passes whose
    // kernel is not compiled yet run the AOT interpreter (bitwise the same)
    std::vector<std::shared_ptr<JitPass>> jit;
    const int jit_knob = tuning().fused_jit;
    if (jit_knob != 0 && cmul_mode >= 0 && cmul_mode <= 2) {
        std::lock_guard<std::mutex> lk(prog->jit_mu);
        if (!prog->jit_requested[cmul_mode]) {
            jit_request(prog->tiled(), R, cmul_mode, jit_knob == 2, prog->jit[cmul_mode]);
            prog->jit_requested[cmul_mode] = true;
        }
        jit = prog->jit[cmul_mode];
    }
    const size_t smem_max = 2 * (sizeof(double2) << kMaxTileBits) + 2 * (sizeof(uint64_t) << (kMaxTileBits - kLowBits));
    static bool attr_set[64] = {false};  // per device (one process may drive several)
    int cur_dev = 0;
    if (cudaGetDevice(&cur_dev) != cudaSuccess || cur_dev < 0 || cur_dev >= 64) {
        cudaGetLastError();
        cur_dev = 0;
    }
    if (!attr_set[cur_dev]) {
        cudaFuncSetAttribute(tile_pass_kernel<3, DIAQ_CMUL_FMA>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_max);
        cudaFuncSetAttribute(tile_pass_kernel<3, DIAQ_CMUL_PLAIN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_max);
        cudaFuncSetAttribute(tile_pass_kernel<4, DIAQ_CMUL_FMA>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_max);
        cudaFuncSetAttribute(tile_pass_kernel<4, DIAQ_CMUL_PLAIN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_max);
        cudaFuncSetAttribute(tile_pass_kernel_t7<DIAQ_CMUL_FMA>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_max);
        cudaFuncSetAttribute(tile_pass_kernel_t7<DIAQ_CMUL_PLAIN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_max);
        cudaFuncSetAttribute(tile_pass_kernel<3, DIAQ_CMUL_CONTRACT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_max);
        cudaFuncSetAttribute(tile_pass_kernel<4, DIAQ_CMUL_CONTRACT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_max);
        cudaFuncSetAttribute(tile_pass_kernel_t7<DIAQ_CMUL_CONTRACT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_max);
        cudaGetLastError();
        attr_set[cur_dev] = true;
    }
    if (events && timer_record(events[0], s) != cudaSuccess)
        return set_error(DIAQ_ERR_CUDA, "diaq_run_gates_fused: event record failed");
    thread_local TileParams tparams;
    // Buffers: a pass with a global permutation tail writes the other buffer
    // (amplitudes move between tiles); every other pass may run in place or
    // out of place.  Flip one flexible pass when the forced flips are odd,
    // so the result lands in `state` (else copy it back at the end).
    const size_t np = plan.size();
    std::vector<char> flip(np, 0);
    int nflip = 0, flexible = -1;
    for (size_t pi = 0; pi < np; ++pi) {
        const PassPlan &ps = plan[pi];
        const bool tiled_pass = !(ps.bits.empty() || ps.members.size() == 1);
        if (tiled_pass && ps.gon) {
            flip[pi] = 1;
            ++nflip;
        } else if (tiled_pass || !sharded) {
            flexible = (int)pi;
        }
    }
    if ((nflip & 1) && flexible >= 0) {
        flip[(size_t)flexible] = 1;
        ++nflip;
    }
    double2 *bufs[2] = {(double2 *)state, nullptr};
    if (nflip > 0) {
        keep_pool_reserved();
        if (cudaMallocAsync((void **)&bufs[1], (size_t)16 << n_bits, s) != cudaSuccess) {
            cudaGetLastError();
            if (t_no_gperm)
                return set_error(DIAQ_ERR_RESOURCE, "diaq_run_gates_fused: no room for a %llu-byte buffer",
                                 (unsigned long long)((size_t)16 << n_bits));
            // no room for the state-sized buffer: plan without global permutation
            // tails (they become in-tile folds or their own passes), all in place
            t_no_gperm = true;
            rc = run_fused(n_total, n_bits, rank, ngates, gates, state, cmul_mode, tile_bits, events, npasses, stream);
            t_no_gperm = false;
            return rc;
        }
    }
    int cur = 0;
    int ev_hi = -1;  // highest gate applied so far (reordered programs: events stay monotone)
    for (size_t pi = 0; pi < np && rc == DIAQ_OK; ++pi) {
        const int nxt = flip[pi] ? 1 - cur : cur;
        const PassPlan &ps = plan[pi];
        for (int m : ps.members) ev_hi = std::max(ev_hi, m);
        if (ps.bits.empty() || ps.members.size() == 1) {
            const diaq_gate_t &gt = gates[ps.members[0]];
            if (sharded) rc = apply_gate_sharded_own(n_total, n_bits, gt.k, gt.g, gt.shifts, rank, bufs[cur], cmul_mode, s);
            else rc = apply_gate(n_bits, gt.k, gt.g, gt.shifts, bufs[cur], bufs[nxt], cmul_mode, s);
        } else {
            TileParams &p = tparams;  // thread-local scratch: the launch copies it
            p = prog->params[pi];
            p.x = bufs[cur];
            p.y = bufs[nxt];
            p.gbase = sharded ? ((uint64_t)rank << n_bits) : 0ull;
            p.estore = tuning().fused_estore;
            if (p.gperm && sharded)  // controls on global bits: constants of this rank
                for (int g = 0; g < 64 && g < n_total - n_bits; ++g)
                    if (((uint64_t)rank >> g) & 1ull) p.gconst ^= ps.ggcol[(size_t)g];
            const void *f = tbits == 7 ? tile_kernel_t7_ptr(cmul_mode)
                            : R >= 4 ? tile_kernel_ptr<4>(cmul_mode) : tile_kernel_ptr<3>(cmul_mode);
            const int nthreads = 1 << tbits;
            auto smem_for = [&](int nb) {
                return ((sizeof(double2) * nb) << p.tbits) + ((sizeof(uint64_t) * (p.gperm ? 2 : 1)) << (p.tbits - kLowBits));
            };
            if (pi < jit.size() && jit[pi] &&
                jit_launch(jit[pi], p, R, smem_for(1), smem_for(2), tuning().fused_nbuf, s, rc)) {
                if (events && rc == DIAQ_OK) timer_record(events[ev_hi + 1], s);
                cur = nxt;
                continue;
            }
            // two tile buffers (prefetch) unless that costs a resident CTA
            const int knob = tuning().fused_nbuf;
            int per_sm = occupancy(f, nthreads, smem_for(1));
            p.nbuf = 1;
            if (knob != 1) {
                const int per_sm2 = occupancy(f, nthreads, smem_for(2));
                if (knob == 2 || per_sm2 >= per_sm) {
                    p.nbuf = 2;
                    per_sm = per_sm2;
                }
            }
            const size_t smem = smem_for(p.nbuf);
            p.gstore = tuning().fused_gstore;
            const int64_t grid =
                std::max<int64_t>(1, std::min<int64_t>(p.ntiles, (int64_t)sm_count() * std::max(1, per_sm)));
            p.gstep = 0;  // deposit grid into the non-tile bits, low to high
            for (int b = 0, k = 0; b < 64 && ((uint64_t)grid >> k) != 0; ++b)
                if (!((p.tmask >> b) & 1ull)) p.gstep |= (((uint64_t)grid >> k++) & 1ull) << b;
            void *args[] = {(void *)&p};
            cudaLaunchKernel(f, dim3((unsigned)grid), dim3((unsigned)nthreads), args, smem, s);
            count_launch();
            rc = check_launch("tile_pass_kernel");
        }
        // events[i]..events[i+1] bracket gate i; a fused pass records only its
        // last gate's event (one record per pass, not per gate), so the pass's
        // time lands on that gate and diaq_timer_elapsed reads the others as 0
        if (events && rc == DIAQ_OK) timer_record(events[ev_hi + 1], s);
        cur = nxt;
    }
    if (rc == DIAQ_OK && cur != 0 &&
        cudaMemcpyAsync(state, bufs[1], (size_t)16 << n_bits, cudaMemcpyDeviceToDevice, s) != cudaSuccess)
        rc = set_error(DIAQ_ERR_CUDA, "diaq_run_gates_fused: copy back failed");
    if (bufs[1]) cudaFreeAsync(bufs[1], s);
    return rc;
}

extern "C" int diaq_trim_pool(void) {
    int dev = 0;
    cudaMemPool_t pool;
    if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetDefaultMemPool(&pool, dev) != cudaSuccess ||
        cudaDeviceSynchronize() != cudaSuccess || cudaMemPoolTrimTo(pool, 0) != cudaSuccess) {
        const cudaError_t e = cudaGetLastError();
        return set_error(DIAQ_ERR_CUDA, "diaq_trim_pool: %s", cudaGetErrorString(e));
    }
    return DIAQ_OK;
}

extern "C" int diaq_run_gates_fused(int n_bits, int ngates, const diaq_gate_t *gates, void *state, int cmul_mode,
                                    int tile_bits, void **events, int *npasses, void *stream) {
    return run_fused(n_bits, n_bits, 0, ngates, gates, state, cmul_mode, tile_bits, events, npasses, stream);
}

extern "C" int diaq_fused_plan_mode(int n_bits, int local_bits, int ngates, const diaq_gate_t *gates, int tile_bits,
                                    int cmul_mode, int *stats) {
    if (ngates < 0 || (ngates > 0 && !gates) || !stats) return set_error(DIAQ_ERR_VALUE, "diaq_fused_plan: bad arguments");
    if (cmul_mode < DIAQ_CMUL_PLAIN || cmul_mode > DIAQ_CMUL_CONTRACT)
        return set_error(DIAQ_ERR_VALUE, "diaq_fused_plan: cmul_mode %d", cmul_mode);
    if (local_bits < 1 || local_bits > n_bits) return set_error(DIAQ_ERR_SHAPE, "local_bits %d invalid", local_bits);
    const int T = (tile_bits >= kThreadBits + 4 && pass_tbits() == 8) ? kThreadBits + 4 : kThreadBits + 3;
    for (int i = 0; i < 5; ++i) stats[i] = 0;
    if (local_bits < T) {  // gate by gate
        stats[0] = stats[1] = ngates;
        return DIAQ_OK;
    }
    std::vector<PassPlan> plan;
    t_reorder = false;  // the program-order schedule (the bitwise modes')
    t_unit = cmul_mode == DIAQ_CMUL_CONTRACT && tuning().fused_unit;
    int rc = schedule(local_bits, n_bits, ngates, gates, T, T - pass_tbits(), plan);
    if (rc) return rc;
    if (cmul_mode == DIAQ_CMUL_CONTRACT && tuning().fused_reorder) {  // as run_fused: reordered only when it saves passes
        std::vector<PassPlan> re;
        t_reorder = true;
        rc = schedule(local_bits, n_bits, ngates, gates, T, T - pass_tbits(), re);
        t_reorder = false;
        if (rc) return rc;
        if (re.size() < plan.size()) plan.swap(re);
    }
    if (getenv("DIAQ_PLAN_DEBUG")) debug_plan(plan);
    for (const PassPlan &ps : plan) {
        ++stats[0];
        if (ps.bits.empty() || ps.members.size() == 1) {
            ++stats[1];
            continue;
        }
        stats[2] += (int)ps.phases.size();
        stats[3] += (int)(ps.members.size() - ps.gates.size()) + ps.nrperm_records;
        for (const Phase &ph : ps.phases) stats[4] += ph.generic;
    }
    return DIAQ_OK;
}

extern "C" int diaq_fused_plan(int n_bits, int local_bits, int ngates, const diaq_gate_t *gates, int tile_bits,
                               int *stats) {
    return diaq_fused_plan_mode(n_bits, local_bits, ngates, gates, tile_bits, DIAQ_CMUL_PLAIN, stats);
}

// Host-only: schedule the program and compile its specialised passes now
// (NVRTC, no device); *seconds the compile time, *kernels the pass count.
extern "C" int diaq_fused_jit_compile(int n_bits, int local_bits, int ngates, const diaq_gate_t *gates, int tile_bits,
                                      int cmul_mode, double *seconds, int *kernels) {
    if (ngates < 0 || (ngates > 0 && !gates) || !kernels)
        return set_error(DIAQ_ERR_VALUE, "diaq_fused_jit_compile: bad arguments");
    if (local_bits < 1 || local_bits > n_bits) return set_error(DIAQ_ERR_SHAPE, "local_bits %d invalid", local_bits);
    if (cmul_mode < 0 || cmul_mode > 2) return set_error(DIAQ_ERR_VALUE, "cmul_mode %d", cmul_mode);
    t_reorder = cmul_mode == DIAQ_CMUL_CONTRACT && tuning().fused_reorder;
    t_unit = cmul_mode == DIAQ_CMUL_CONTRACT && tuning().fused_unit;
    const int T = (tile_bits >= kThreadBits + 4 && pass_tbits() == 8) ? kThreadBits + 4 : kThreadBits + 3;
    int rc = DIAQ_OK;
    std::shared_ptr<const Program> prog = build_program(n_bits, local_bits, T, ngates, gates, rc);
    if (!prog) return rc;
    if (t_reorder) {  // the schedule run_fused would pick (reordered only when it saves passes)
        t_reorder = false;
        std::shared_ptr<const Program> inorder = build_program(n_bits, local_bits, T, ngates, gates, rc);
        if (!inorder) return rc;
        if (inorder->plan.size() <= prog->plan.size()) prog = inorder;
    }
    if (!seconds) {  // submit to the background compile queue (as a first run_gates call would)
        std::vector<std::shared_ptr<JitPass>> out;
        jit_request(prog->tiled(), T - pass_tbits(), cmul_mode, false, out);
        *kernels = 0;
        for (auto &e : out) *kernels += e ? 1 : 0;
        return DIAQ_OK;
    }
    return jit_compile_now(prog->tiled(), T - pass_tbits(), cmul_mode, *seconds, *kernels);
}

extern "C" int diaq_run_gates_local(int n_bits, int local_bits, int64_t rank, int ngates, const diaq_gate_t *gates,
                                    void *shard, int cmul_mode, int tile_bits, void **events, int *npasses,
                                    void *stream) {
    if (local_bits < 1 || local_bits > n_bits) return set_error(DIAQ_ERR_SHAPE, "local_bits %d invalid", local_bits);
    return run_fused(n_bits, local_bits, rank, ngates, gates, shard, cmul_mode, tile_bits, events, npasses, stream);
}
