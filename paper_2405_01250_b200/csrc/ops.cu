// ops.cu -- the DiaQ matrix algebra around the hot path, on the device
// (reference matrix.py:281-355): conjugate (adjoint), scale, add and the
// general Kronecker product.  Transpose needs no kernel: position k of
// diagonal d and of -d are transposes of each other (matrix.py:281-290), so
// the Python mirror relabels the same arena.
//
// Every value is computed with the reference's rounding in the reference's
// result precision: float64 (numpy float64 ufuncs, products rounded, no FMA)
// or, when the result dtype is single, float32 arithmetic on the
// float32-representable values (numpy's weak Python-float scalars keep a
// float32 array float32), widened exactly into the complex128 arena.
#include <algorithm>
#include <vector>

#include "common.cuh"

namespace diaq {

__device__ __forceinline__ double rnd(double v, bool single) { return single ? (double)(float)v : v; }

__device__ __forceinline__ double mul_p(double a, double b, bool single) {
    return single ? (double)__fmul_rn((float)a, (float)b) : __dmul_rn(a, b);
}
__device__ __forceinline__ double add_p(double a, double b, bool single) {
    return single ? (double)__fadd_rn((float)a, (float)b) : __dadd_rn(a, b);
}
__device__ __forceinline__ double sub_p(double a, double b, bool single) {
    return single ? (double)__fsub_rn((float)a, (float)b) : __dsub_rn(a, b);
}

// re' = sr*re - si*im, im' = sr*im + si*re over a whole arena (same layout);
// conj: (re, -im)
__global__ void __launch_bounds__(kThreads) arena_map_kernel(const double2 *src, double2 *dst, int64_t total, int op,
                                                              double sr, double si, int single) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += stride) {
        const double2 v = src[e];
        double2 o;
        if (op == 0) {
            o = make_double2(v.x, -v.y);
        } else {
            o.x = sub_p(mul_p(sr, v.x, single), mul_p(si, v.y, single), single);
            o.y = add_p(mul_p(sr, v.y, single), mul_p(si, v.x, single), single);
        }
        dst[e] = o;
    }
}

struct AddDiag {
    const double2 *a, *b;  // null: absent in that operand
    double2 *dst;
    int64_t len;
};

struct AddParams {
    int nd;
    int single;
    AddDiag dg[kParamDiags];
};

// out_d = (+0 + a_d) + b_d element by element (matrix.py:301-315)
__global__ void __launch_bounds__(kThreads) add_kernel(const __grid_constant__ AddParams p) {
    const AddDiag g = p.dg[blockIdx.y];
    const bool single = p.single;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < g.len; k += stride) {
        double2 acc = make_double2(0.0, 0.0);
        if (g.a) {
            const double2 v = g.a[k];
            acc = make_double2(add_p(acc.x, v.x, single), add_p(acc.y, v.y, single));
        }
        if (g.b) {
            const double2 v = g.b[k];
            acc = make_double2(add_p(acc.x, v.x, single), add_p(acc.y, v.y, single));
        }
        g.dst[k] = acc;
    }
}

struct KronTab {  // device: offsets then starts of A (nda) and B (ndb)
    const int64_t *offa, *sta, *offb, *stb;
    int64_t nda, ndb;
};

struct KronGenDiag {
    int64_t d;
    double2 *dst;
    int64_t len;
};

struct KronGenParams {
    int64_t na, nb;
    const double2 *av, *bv;
    KronTab t;
    int nd;
    int single;
    KronGenDiag dg[kParamDiags];
};

__device__ __forceinline__ int64_t find_off(const int64_t *offs, int64_t nd, int64_t d) {
    int64_t lo = 0, hi = nd;  // ascending offsets: binary search
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (offs[mid] < d) lo = mid + 1;
        else hi = mid;
    }
    return (lo < nd && offs[lo] == d) ? lo : -1;
}

// element (r, r + d) of A (x) B: rows/cols split into (A, B) parts; the
// unique source pair (dA, dB) = (cA - rA, cB - rB) contributes
// (ar*br - ai*bi, ar*bi + ai*br) if both diagonals are stored, else 0
// (matrix.py:329-355: every result diagonal's uncovered positions stay 0)
__global__ void __launch_bounds__(kThreads) kron_general_kernel(const __grid_constant__ KronGenParams p) {
    const KronGenDiag g = p.dg[blockIdx.y];
    const bool single = p.single;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < g.len; k += stride) {
        const int64_t r = k - (g.d < 0 ? g.d : 0), c = r + g.d;
        const int64_t ra = r / p.nb, rb = r - ra * p.nb, ca = c / p.nb, cb = c - ca * p.nb;
        const int64_t da = ca - ra, db = cb - rb;
        double2 o = make_double2(0.0, 0.0);
        const int64_t ia = find_off(p.t.offa, p.t.nda, da);
        const int64_t ib = ia >= 0 ? find_off(p.t.offb, p.t.ndb, db) : -1;
        if (ib >= 0) {
            const double2 a = p.av[p.t.sta[ia] + ra + (da < 0 ? da : 0)];
            const double2 b = p.bv[p.t.stb[ib] + rb + (db < 0 ? db : 0)];
            o.x = sub_p(mul_p(a.x, b.x, single), mul_p(a.y, b.y, single), single);
            o.y = add_p(mul_p(a.x, b.y, single), mul_p(a.y, b.x, single), single);
        }
        g.dst[k] = o;
    }
}

static int grid_for(int64_t len, int nd) {
    const int64_t want = (len + kThreads - 1) / kThreads;
    const int64_t cap = std::max<int64_t>(1, (int64_t)sm_count() * 8 / std::max(1, nd));
    return (int)std::max<int64_t>(1, std::min<int64_t>(want, cap));
}

}  // namespace diaq

using namespace diaq;

extern "C" int diaq_arena_map(int64_t total, const void *src, void *dst, int op, double sr, double si, int single,
                              void *stream) {
    if (total < 0 || (total && (!src || !dst)) || op < 0 || op > 1)
        return set_error(DIAQ_ERR_VALUE, "diaq_arena_map: bad arguments");
    if (total == 0) return DIAQ_OK;
    arena_map_kernel<<<grid_for(total, 1), kThreads, 0, (cudaStream_t)stream>>>((const double2 *)src, (double2 *)dst,
                                                                                  total, op, sr, si, single);
    count_launch();
    return check_launch("arena_map_kernel");
}

extern "C" int diaq_add(const diaq_matrix_t *a, const diaq_matrix_t *b, diaq_matrix_t *out, int single, void *stream) {
    if (!a || !b || !out) return set_error(DIAQ_ERR_VALUE, "diaq_add: null argument");
    if (a->n != b->n || out->n != a->n)
        return set_error(DIAQ_ERR_SHAPE, "shape mismatch: %lld vs %lld", (long long)a->n, (long long)b->n);
    cudaStream_t s = (cudaStream_t)stream;
    static thread_local AddParams p;
    p.single = single;
    int64_t ia = 0, ib = 0;
    for (int64_t base = 0; base < out->nd; base += kParamDiags) {
        const int cnt = (int)std::min<int64_t>(kParamDiags, out->nd - base);
        p.nd = cnt;
        int64_t maxlen = 0;
        for (int j = 0; j < cnt; ++j) {
            const int64_t d = out->offs[base + j];
            while (ia < a->nd && a->offs[ia] < d) ++ia;
            while (ib < b->nd && b->offs[ib] < d) ++ib;
            AddDiag &g = p.dg[j];
            g.a = (ia < a->nd && a->offs[ia] == d) ? (const double2 *)a->vals + a->starts[ia] : nullptr;
            g.b = (ib < b->nd && b->offs[ib] == d) ? (const double2 *)b->vals + b->starts[ib] : nullptr;
            g.dst = (double2 *)out->vals + out->starts[base + j];
            g.len = out->n - (d < 0 ? -d : d);
            maxlen = std::max(maxlen, g.len);
        }
        add_kernel<<<dim3(grid_for(maxlen, cnt), cnt), kThreads, 0, s>>>(p);
        count_launch();
        const int rc = check_launch("add_kernel");
        if (rc) return rc;
    }
    return DIAQ_OK;
}

// tables_dev: [offa[nda], sta[nda], offb[ndb], stb[ndb]] in device memory
extern "C" int diaq_kron(const diaq_matrix_t *a, const diaq_matrix_t *b, const int64_t *tables_dev, diaq_matrix_t *out,
                         int single, void *stream) {
    if (!a || !b || !out || (a->nd && b->nd && !tables_dev)) return set_error(DIAQ_ERR_VALUE, "diaq_kron: bad arguments");
    if (out->n != a->n * b->n) return set_error(DIAQ_ERR_SHAPE, "diaq_kron: output n mismatch");
    cudaStream_t s = (cudaStream_t)stream;
    static thread_local KronGenParams p;
    p.na = a->n;
    p.nb = b->n;
    p.av = (const double2 *)a->vals;
    p.bv = (const double2 *)b->vals;
    p.t.offa = tables_dev;
    p.t.sta = tables_dev + a->nd;
    p.t.offb = tables_dev + 2 * a->nd;
    p.t.stb = tables_dev + 2 * a->nd + b->nd;
    p.t.nda = a->nd;
    p.t.ndb = b->nd;
    p.single = single;
    for (int64_t base = 0; base < out->nd; base += kParamDiags) {
        const int cnt = (int)std::min<int64_t>(kParamDiags, out->nd - base);
        p.nd = cnt;
        int64_t maxlen = 0;
        for (int j = 0; j < cnt; ++j) {
            const int64_t d = out->offs[base + j];
            p.dg[j].d = d;
            p.dg[j].dst = (double2 *)out->vals + out->starts[base + j];
            p.dg[j].len = out->n - (d < 0 ? -d : d);
            maxlen = std::max(maxlen, p.dg[j].len);
        }
        kron_general_kernel<<<dim3(grid_for(maxlen, cnt), cnt), kThreads, 0, s>>>(p);
        count_launch();
        const int rc = check_launch("kron_general_kernel");
        if (rc) return rc;
    }
    return DIAQ_OK;
}
