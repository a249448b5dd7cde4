// construct.cu -- building DiaQ matrices on the device (sm_100a).
//
//  * kron_identity (reference matrix.py:358-387): closed form.  Output
//    diagonal d*R, element k: with block = n_m*R and run = len(m_d)*R,
//    value m_d[(k mod block) / R] if (k mod block) < run else 0 (explicit
//    zeros kept, never pruned).  Pure streaming writes; m stays in L1/L2.
//  * build_span_unitary (reference gates.py:169-219): closed form.  For
//    output diagonal d, row r, column c = r + d: value g[gather(r),
//    gather(c)] when r and c agree on every non-gate bit and that gate entry
//    is nonzero (|re|+|im| > 0, gates.py:203-204), else 0.
//  * from_dense (reference matrix.py:135-153): pass 1 flags every diagonal
//    holding some |re|+|im| > eps (coalesced row-major read of the dense
//    matrix); the host lays out the kept set; pass 2 gathers them.
//  * to_dense (reference matrix.py:156-167): scatter at stride n+1.
#include <algorithm>
#include <cmath>
#include <vector>

#include "common.cuh"

namespace diaq {

struct KronDiag {
    const double2 *src;  // m diagonal (k = 0)
    double2 *dst;        // output diagonal (k = 0)
    int64_t len;         // output length n - |d*R|
    int64_t run;         // len(m_d) * R
};

struct KronParams {
    int64_t block, right;
    int pow2;
    int block_shift, right_shift;
    int nd;
    KronDiag dg[kParamDiags];
    int64_t beg[kParamDiags];  // arena offset of each output diagonal from dg[0].dst (flat mode)
    int64_t end;               // beg[nd-1] + dg[nd-1].len
};

__device__ __forceinline__ double2 kron_value(const KronParams &p, const KronDiag &dg, int64_t k) {
    int64_t pos, src;
    if (p.pow2) {
        pos = k & (p.block - 1);
        src = pos >> p.right_shift;
    } else {
        pos = k % p.block;
        src = pos / p.right;
    }
    return pos < dg.run ? ld_reuse(dg.src + src) : make_double2(0.0, 0.0);
}

// Two adjacent output elements per thread and iteration, written with one
// 256-bit store; an element left over at either end of a diagonal (odd
// arena start / odd remaining length) is written singly by one thread.
__global__ void __launch_bounds__(kThreads) kron_identity_kernel(const __grid_constant__ KronParams p) {
    const KronDiag &dg = p.dg[blockIdx.y];
    const int64_t k0 = ((uintptr_t)dg.dst & 31) ? 1 : 0;
    const int64_t pairs = dg.len > k0 ? (dg.len - k0) >> 1 : 0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < pairs; j += stride) {
        const int64_t k = k0 + 2 * j;
        st_stream2(dg.dst + k, kron_value(p, dg, k), kron_value(p, dg, k + 1));
    }
    if (blockIdx.x == 0 && threadIdx.x == 0 && dg.len > 0) {
        if (k0) st_stream(dg.dst, kron_value(p, dg, 0));
        if (k0 + 2 * pairs < dg.len) st_stream(dg.dst + dg.len - 1, kron_value(p, dg, dg.len - 1));
    }
}

// Arena-linear variant: the batch's output diagonals are one contiguous
// arena range (gaps only the < 8-element alignment padding of diaq_layout,
// which receives zeros), written front to back as a single 256-bit store
// stream like a fill -- no per-diagonal grid rows competing for DRAM pages.
// A thread's pairs advance monotonically, so it keeps the current
// diagonal's fields in registers and re-reads the table only on crossing a
// diagonal boundary (a pair straddling one takes the generic lookup).
__device__ __forceinline__ double2 kron_flat_value(const KronParams &p, int i, int64_t e) {
    const int64_t k = e - p.beg[i];
    if (k < 0 || k >= p.dg[i].len) return make_double2(0.0, 0.0);
    return kron_value(p, p.dg[i], k);
}

__device__ __forceinline__ int kron_flat_find(const KronParams &p, int64_t e) {
    int i = 0;
    while (i + 1 < p.nd && e >= p.beg[i + 1]) ++i;
    return i;
}

template <bool kPow2>
struct KronCursor {
    const double2 *src;
    int64_t lo, hi;  // [lo, hi): arena range of the cached diagonal's elements
    int64_t run, block, right;
    int block_shift, right_shift;
    uint64_t pol;  // L2 evict_last: the source diagonal is re-read once per left block, between
                   // which a whole block of output streams through L2 and would evict it

    __device__ __forceinline__ void load(const KronParams &p, int i) {
        src = p.dg[i].src;
        lo = p.beg[i];
        hi = lo + p.dg[i].len;
        run = p.dg[i].run;
        block = p.block;
        right = p.right;
        block_shift = p.block_shift;
        right_shift = p.right_shift;
    }
    __device__ __forceinline__ double2 at(int64_t k) const {
        int64_t pos, idx;
        if (kPow2) {
            pos = k & (block - 1);
            idx = pos >> right_shift;
        } else {
            pos = k % block;
            idx = pos / right;
        }
        return pos < run ? ld_reuse_hint(src + idx, pol) : make_double2(0.0, 0.0);
    }
    // elements k and k+1; one load when both read the same source element
    // (right >= 2 and the pair inside one run of R), the common case
    __device__ __forceinline__ void at2(int64_t k, double2 &a, double2 &b) const {
        int64_t pos, idx;
        if (kPow2) {
            pos = k & (block - 1);
            idx = pos >> right_shift;
        } else {
            pos = k % block;
            idx = pos / right;
        }
        const int64_t pos1 = pos + 1 == block ? 0 : pos + 1;
        const int64_t idx1 = kPow2 ? (pos1 >> right_shift) : pos1 / right;
        a = pos < run ? ld_reuse_hint(src + idx, pol) : make_double2(0.0, 0.0);
        if (idx1 == idx && pos1 < run) b = a;
        else b = pos1 < run ? ld_reuse_hint(src + idx1, pol) : make_double2(0.0, 0.0);
    }
};

template <bool kPow2>
__global__ void __launch_bounds__(kThreads) kron_identity_flat_kernel(const __grid_constant__ KronParams p) {
    double2 *base = p.dg[0].dst;
    const int64_t first = ((uintptr_t)base & 31) ? 1 : 0;
    const int64_t pairs = p.end > first ? (p.end - first) >> 1 : 0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= pairs) return;
    int i = kron_flat_find(p, first + 2 * j);
    KronCursor<kPow2> c;
    c.pol = policy_evict_last();
    c.load(p, i);
    constexpr int U = 4;  // pairs in flight per thread (all loads issued before the stores)
    for (; j < pairs; j += U * stride) {
        double2 v[2 * U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t e = first + 2 * (j + u * stride);
            if (j + u * stride >= pairs) break;
            if (e >= c.hi && i + 1 < p.nd && e >= p.beg[i + 1]) {
                i = kron_flat_find(p, e);
                c.load(p, i);
            }
            if (e >= c.lo && e + 1 < c.hi) {
                c.at2(e - c.lo, v[2 * u], v[2 * u + 1]);
            } else {  // padding or a diagonal boundary inside the pair
                v[2 * u] = kron_flat_value(p, kron_flat_find(p, e), e);
                v[2 * u + 1] = kron_flat_value(p, kron_flat_find(p, e + 1), e + 1);
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (j + u * stride < pairs) st_stream2(base + first + 2 * (j + u * stride), v[2 * u], v[2 * u + 1]);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        if (first && p.end > 0) st_stream(base, kron_flat_value(p, 0, 0));
        if (first + 2 * pairs < p.end) st_stream(base + p.end - 1, kron_flat_value(p, p.nd - 1, p.end - 1));
    }
}

struct SpanParams {
    int k, span;
    int shifts[kParamDiags];   // state bit of gate operand i (operand 0 = MSB)
    uint64_t free_mask;        // bits of the span that are not gate bits
    int nd;
    int64_t off[kParamDiags];
    double2 *dst[kParamDiags];
    int64_t len[kParamDiags];
    const double2 *gdev;       // k > 4: the dense gate in device memory (else in g below)
    double2 g[256];            // dense gate, k <= 4
};

__device__ __forceinline__ int gather_bits(uint64_t r, const int *shifts, int k) {
    int out = 0;
    for (int i = 0; i < k; ++i) out |= (int)((r >> shifts[i]) & 1ull) << (k - 1 - i);
    return out;
}

__global__ void __launch_bounds__(kThreads) span_expand_kernel(const __grid_constant__ SpanParams p) {
    const int i = blockIdx.y;
    const int64_t d = p.off[i];
    const int64_t len = p.len[i];
    const int M = 1 << p.k;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t kk = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; kk < len; kk += stride) {
        const uint64_t r = (uint64_t)(kk - (d < 0 ? d : 0));
        const uint64_t c = r + (uint64_t)d;
        double2 v = make_double2(0.0, 0.0);
        if (((r ^ c) & p.free_mask) == 0) {
            const int rg = gather_bits(r, p.shifts, p.k);
            const int cg = gather_bits(c, p.shifts, p.k);
            const double2 gv = p.gdev ? ld_reuse(p.gdev + (int64_t)rg * M + cg) : p.g[rg * M + cg];
            if (fabs(gv.x) + fabs(gv.y) > 0.0) v = gv;
        }
        st_stream(p.dst[i] + kk, v);
    }
}

__global__ void __launch_bounds__(kThreads)
from_dense_scan_kernel(const double2 *m, int64_t n, double eps, uint8_t *keep) {
    const int64_t total = n * n;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += stride) {
        const double2 v = ld_stream(m + e, policy_evict_first());
        if (fabs(v.x) + fabs(v.y) > eps) {
            const int64_t r = e / n, c = e - r * n;
            keep[c - r + n - 1] = 1;
        }
    }
}

struct GatherDiag {
    double2 *dst;
    int64_t len, base;  // dense flat index of k = 0
};

__global__ void __launch_bounds__(kThreads)
from_dense_fill_kernel(const double2 *m, int64_t n, const GatherDiag *__restrict__ dg) {
    const GatherDiag g = dg[blockIdx.y];
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < g.len; k += stride)
        g.dst[k] = m[g.base + k * (n + 1)];
}

__global__ void __launch_bounds__(kThreads)
to_dense_kernel(double2 *m, int64_t n, const GatherDiag *__restrict__ dg) {
    const GatherDiag g = dg[blockIdx.y];
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < g.len; k += stride)
        m[g.base + k * (n + 1)] = g.dst[k];
}

static int grid_x(int64_t len, int nd) {
    const int sms = sm_count();
    const int64_t want = (len + kThreads - 1) / kThreads;
    const int64_t cap = std::max<int64_t>(1, (int64_t)sms * 8 / std::max(1, nd));
    return (int)std::max<int64_t>(1, std::min<int64_t>(want, cap));
}

static bool is_pow2(int64_t v) { return v > 0 && (v & (v - 1)) == 0; }
static int log2i(int64_t v) { int s = 0; while ((1ll << s) < v) ++s; return s; }

static int64_t embed_idx(int64_t idx, int k, const int *shifts) {
    int64_t out = 0;
    for (int i = 0; i < k; ++i) out |= ((idx >> (k - 1 - i)) & 1) << shifts[i];
    return out;
}

// temporary device table, freed stream-ordered
template <typename T>
static T *upload_table(const std::vector<T> &h, cudaStream_t s) {
    T *d = nullptr;
    if (cudaMallocAsync((void **)&d, sizeof(T) * h.size(), s) != cudaSuccess) return nullptr;
    if (cudaMemcpyAsync(d, h.data(), sizeof(T) * h.size(), cudaMemcpyHostToDevice, s) != cudaSuccess) {
        cudaFreeAsync(d, s);
        return nullptr;
    }
    return d;
}

}  // namespace diaq

using namespace diaq;

extern "C" int diaq_kron_identity(int64_t left, const diaq_matrix_t *m, int64_t right, diaq_matrix_t *out,
                                  void *stream) {
    if (!m || !out) return set_error(DIAQ_ERR_VALUE, "diaq_kron_identity: null argument");
    if (left < 1 || right < 1) return set_error(DIAQ_ERR_SHAPE, "left_dim and right_dim must be >= 1");
    if (out->n != left * m->n * right || out->nd != m->nd)
        return set_error(DIAQ_ERR_SHAPE, "diaq_kron_identity: output layout mismatch");
    if (m->nd == 0) return DIAQ_OK;
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t block = m->n * right;
    for (int64_t base = 0; base < m->nd; base += kParamDiags) {
        const int cnt = (int)std::min<int64_t>(kParamDiags, m->nd - base);
        KronParams p;
        p.block = block;
        p.right = right;
        p.pow2 = is_pow2(block) && is_pow2(right);
        p.block_shift = p.pow2 ? log2i(block) : 0;
        p.right_shift = p.pow2 ? log2i(right) : 0;
        p.nd = cnt;
        int64_t maxlen = 0;
        bool flat = tuning().kron_flat != 0;
        for (int j = 0; j < cnt; ++j) {
            const int64_t i = base + j;
            const int64_t d = m->offs[i];
            if (out->offs[i] != d * right) return set_error(DIAQ_ERR_SHAPE, "diaq_kron_identity: offset table mismatch");
            const int64_t dout = d * right;
            p.dg[j].src = (const double2 *)m->vals + m->starts[i];
            p.dg[j].dst = (double2 *)out->vals + out->starts[i];
            p.dg[j].len = out->n - (dout < 0 ? -dout : dout);
            p.dg[j].run = (m->n - (d < 0 ? -d : d)) * right;
            maxlen = std::max(maxlen, p.dg[j].len);
            p.beg[j] = p.dg[j].dst - p.dg[0].dst;
            if (j > 0) {
                const int64_t gap = p.beg[j] - (p.beg[j - 1] + p.dg[j - 1].len);
                if (gap < 0 || gap >= 8) flat = false;  // not a diaq_layout arena: keep to the diagonals
            }
        }
        p.end = p.beg[cnt - 1] + p.dg[cnt - 1].len;
        if (flat) {
            const int sms = sm_count();
            const int64_t want = (p.end / 2 + kThreads - 1) / kThreads;
            const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)sms * tuning().kron_ctas_per_sm));
            if (p.pow2)
                kron_identity_flat_kernel<true><<<grid, kThreads, 0, s>>>(p);
            else
                kron_identity_flat_kernel<false><<<grid, kThreads, 0, s>>>(p);
        } else {
            dim3 grid(grid_x((maxlen + 1) / 2, cnt), cnt);
            kron_identity_kernel<<<grid, kThreads, 0, s>>>(p);
        }
        count_launch();
        const int rc = check_launch("kron_identity_kernel");
        if (rc) return rc;
    }
    return DIAQ_OK;
}

extern "C" int diaq_span_plan(int k, const double *g, const int *positions, int span, int64_t *offs_out,
                              int64_t *nd_out) {
    if (!g || !positions || !offs_out || !nd_out) return set_error(DIAQ_ERR_VALUE, "diaq_span_plan: null argument");
    if (k < 1 || k > 16) return set_error(DIAQ_ERR_UNSUPPORTED, "diaq_span_plan: gate width %d outside 1..16", k);
    if (span < k || span > 62) return set_error(DIAQ_ERR_SHAPE, "diaq_span_plan: span %d", span);
    int shifts[64];
    for (int i = 0; i < k; ++i) {
        if (positions[i] < 0 || positions[i] >= span)
            return set_error(DIAQ_ERR_SHAPE, "positions outside span of %d qubits", span);
        for (int j = 0; j < i; ++j)
            if (positions[j] == positions[i]) return set_error(DIAQ_ERR_SHAPE, "need %d distinct positions", k);
        shifts[i] = span - 1 - positions[i];
    }
    const int64_t M = 1ll << k;
    std::vector<int64_t> v;
    for (int64_t rg = 0; rg < M; ++rg)
        for (int64_t cg = 0; cg < M; ++cg) {
            const double re = g[2 * (rg * M + cg)], im = g[2 * (rg * M + cg) + 1];
            if (!(std::fabs(re) + std::fabs(im) > 0.0)) continue;
            v.push_back(embed_idx(cg, k, shifts) - embed_idx(rg, k, shifts));
        }
    std::sort(v.begin(), v.end());
    v.erase(std::unique(v.begin(), v.end()), v.end());
    for (size_t i = 0; i < v.size(); ++i) offs_out[i] = v[i];
    *nd_out = (int64_t)v.size();
    return DIAQ_OK;
}

extern "C" int diaq_span_expand(int k, const double *g, const int *positions, int span, diaq_matrix_t *out,
                                void *stream) {
    if (!g || !positions || !out) return set_error(DIAQ_ERR_VALUE, "diaq_span_expand: null argument");
    if (k < 1 || k > 16) return set_error(DIAQ_ERR_UNSUPPORTED, "diaq_span_expand: gate width %d outside 1..16", k);
    if (out->n != (1ll << span)) return set_error(DIAQ_ERR_SHAPE, "diaq_span_expand: output n mismatch");
    cudaStream_t s = (cudaStream_t)stream;
    static thread_local SpanParams p;
    p.k = k;
    p.span = span;
    uint64_t gate_mask = 0;
    for (int i = 0; i < k; ++i) {
        p.shifts[i] = span - 1 - positions[i];
        gate_mask |= 1ull << p.shifts[i];
    }
    p.free_mask = (span >= 64 ? ~0ull : ((1ull << span) - 1ull)) & ~gate_mask;
    const int M = 1 << k;
    double2 *gdev = nullptr;
    p.gdev = nullptr;
    if (k <= 4) {
        for (int i = 0; i < M * M; ++i) p.g[i] = make_double2(g[2 * i], g[2 * i + 1]);
    } else {  // 4^k entries: too many for the kernel parameters, staged in device memory
        const size_t bytes = sizeof(double2) * (size_t)M * (size_t)M;
        if (cudaMallocAsync((void **)&gdev, bytes, s) != cudaSuccess ||
            cudaMemcpyAsync(gdev, g, bytes, cudaMemcpyHostToDevice, s) != cudaSuccess) {
            cudaGetLastError();
            if (gdev) cudaFreeAsync(gdev, s);
            return set_error(DIAQ_ERR_CUDA, "diaq_span_expand: staging a %d-qubit gate failed", k);
        }
        p.gdev = gdev;
    }
    int rc = DIAQ_OK;
    for (int64_t base = 0; base < out->nd && rc == DIAQ_OK; base += kParamDiags) {
        const int cnt = (int)std::min<int64_t>(kParamDiags, out->nd - base);
        p.nd = cnt;
        int64_t maxlen = 0;
        for (int j = 0; j < cnt; ++j) {
            const int64_t d = out->offs[base + j];
            p.off[j] = d;
            p.len[j] = out->n - (d < 0 ? -d : d);
            p.dst[j] = (double2 *)out->vals + out->starts[base + j];
            maxlen = std::max(maxlen, p.len[j]);
        }
        dim3 grid(grid_x(maxlen, cnt), cnt);
        span_expand_kernel<<<grid, kThreads, 0, s>>>(p);
        count_launch();
        rc = check_launch("span_expand_kernel");
    }
    if (gdev) cudaFreeAsync(gdev, s);
    return rc;
}

extern "C" int diaq_from_dense_scan(int64_t n, const void *dense, double eps, uint8_t *keep_dev, void *stream) {
    if (!dense || !keep_dev || n < 1) return set_error(DIAQ_ERR_VALUE, "diaq_from_dense_scan: bad arguments");
    cudaStream_t s = (cudaStream_t)stream;
    if (cudaMemsetAsync(keep_dev, 0, (size_t)(2 * n - 1), s) != cudaSuccess)
        return set_error(DIAQ_ERR_CUDA, "diaq_from_dense_scan: memset failed");
    const int grid = grid_x(n * n, 1);
    from_dense_scan_kernel<<<grid, kThreads, 0, s>>>((const double2 *)dense, n, eps, keep_dev);
    count_launch();
    return check_launch("from_dense_scan_kernel");
}

static int gather_launch(const void *dense, diaq_matrix_t *a, bool to_dense, cudaStream_t s) {
    if (a->nd == 0) return DIAQ_OK;
    std::vector<GatherDiag> h((size_t)a->nd);
    int64_t maxlen = 0;
    const int64_t n = a->n;
    for (int64_t i = 0; i < a->nd; ++i) {
        const int64_t d = a->offs[i];
        h[i].dst = (double2 *)a->vals + a->starts[i];
        h[i].len = n - (d < 0 ? -d : d);
        h[i].base = d >= 0 ? d : -d * n;
        maxlen = std::max(maxlen, h[i].len);
    }
    GatherDiag *dt = upload_table(h, s);
    if (!dt) return set_error(DIAQ_ERR_CUDA, "gather table upload failed");
    for (int64_t base = 0; base < a->nd; base += 65535) {
        const int cnt = (int)std::min<int64_t>(65535, a->nd - base);
        dim3 grid(grid_x(maxlen, cnt), cnt);
        if (to_dense) to_dense_kernel<<<grid, kThreads, 0, s>>>((double2 *)dense, n, dt + base);
        else from_dense_fill_kernel<<<grid, kThreads, 0, s>>>((const double2 *)dense, n, dt + base);
        count_launch();
    }
    const int rc = check_launch(to_dense ? "to_dense_kernel" : "from_dense_fill_kernel");
    cudaFreeAsync(dt, s);
    return rc;
}

extern "C" int diaq_from_dense_fill(const void *dense, diaq_matrix_t *out, void *stream) {
    if (!dense || !out) return set_error(DIAQ_ERR_VALUE, "diaq_from_dense_fill: null argument");
    return gather_launch(dense, out, false, (cudaStream_t)stream);
}

extern "C" int diaq_to_dense(const diaq_matrix_t *a, void *dense, void *stream) {
    if (!dense || !a) return set_error(DIAQ_ERR_VALUE, "diaq_to_dense: null argument");
    return gather_launch(dense, const_cast<diaq_matrix_t *>(a), true, (cudaStream_t)stream);
}

// ---- accounting on the device (reference nnz matrix.py:393-400, memory.py:29-46) ----

struct CountDiag {
    const double2 *vals;  // k = 0
    int64_t len, d;
};

__global__ void __launch_bounds__(kThreads)
count_nonzero_kernel(const CountDiag *__restrict__ dg, double eps, unsigned long long *count) {
    const CountDiag g = dg[blockIdx.y];
    unsigned long long c = 0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < g.len; k += stride) {
        const double2 v = g.vals[k];
        c += (fabs(v.x) + fabs(v.y) > eps) ? 1ull : 0ull;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_down_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(count, c);
}

// 2x2 blocks holding a nonzero: one bit per block, then a popcount
__global__ void __launch_bounds__(kThreads)
bsr_mark_kernel(const CountDiag *__restrict__ dg, double eps, int64_t nb, unsigned int *bitmap) {
    const CountDiag g = dg[blockIdx.y];
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < g.len; k += stride) {
        const double2 v = g.vals[k];
        if (fabs(v.x) + fabs(v.y) > eps) {
            const int64_t row = k - (g.d < 0 ? g.d : 0), col = row + g.d;
            const int64_t blk = (row >> 1) * nb + (col >> 1);
            atomicOr(bitmap + (blk >> 5), 1u << (blk & 31));
        }
    }
}

__global__ void __launch_bounds__(kThreads) popcount_kernel(const unsigned int *bitmap, int64_t words,
                                                            unsigned long long *count) {
    unsigned long long c = 0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < words; i += stride) c += __popc(bitmap[i]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_down_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(count, c);
}

static int count_common(const diaq_matrix_t *a, double eps, int64_t *nnz_out, int64_t *bsr_out, void *stream) {
    cudaStream_t s = (cudaStream_t)stream;
    if (nnz_out) *nnz_out = 0;
    if (bsr_out) *bsr_out = 0;
    if (a->nd == 0) return DIAQ_OK;
    std::vector<CountDiag> h((size_t)a->nd);
    int64_t maxlen = 0;
    for (int64_t i = 0; i < a->nd; ++i) {
        const int64_t d = a->offs[i];
        h[i].vals = (const double2 *)a->vals + a->starts[i];
        h[i].len = a->n - (d < 0 ? -d : d);
        h[i].d = d;
        maxlen = std::max(maxlen, h[i].len);
    }
    CountDiag *dt = upload_table(h, s);
    if (!dt) return set_error(DIAQ_ERR_CUDA, "count table upload failed");
    unsigned long long *cnt = nullptr;
    unsigned int *bitmap = nullptr;
    const int64_t nb = (a->n + 1) / 2;
    const int64_t words = (nb * nb + 31) / 32;
    int rc = DIAQ_OK;
    unsigned long long hc[2] = {0, 0};
    if (cudaMallocAsync((void **)&cnt, 2 * sizeof(unsigned long long), s) != cudaSuccess) {
        cudaFreeAsync(dt, s);
        return set_error(DIAQ_ERR_CUDA, "count alloc failed");
    }
    cudaMemsetAsync(cnt, 0, 2 * sizeof(unsigned long long), s);
    for (int64_t base = 0; base < a->nd; base += 65535) {
        const int cntd = (int)std::min<int64_t>(65535, a->nd - base);
        dim3 grid(grid_x(maxlen, cntd), cntd);
        if (nnz_out) {
            count_nonzero_kernel<<<grid, kThreads, 0, s>>>(dt + base, eps, cnt);
            count_launch();
        }
    }
    if (bsr_out) {
        if (cudaMallocAsync((void **)&bitmap, sizeof(unsigned int) * (size_t)words, s) != cudaSuccess) {
            rc = set_error(DIAQ_ERR_RESOURCE, "bsr bitmap of %lld words does not fit", (long long)words);
        } else {
            cudaMemsetAsync(bitmap, 0, sizeof(unsigned int) * (size_t)words, s);
            for (int64_t base = 0; base < a->nd; base += 65535) {
                const int cntd = (int)std::min<int64_t>(65535, a->nd - base);
                dim3 grid(grid_x(maxlen, cntd), cntd);
                bsr_mark_kernel<<<grid, kThreads, 0, s>>>(dt + base, eps, nb, bitmap);
                count_launch();
            }
            popcount_kernel<<<grid_x(words, 1), kThreads, 0, s>>>(bitmap, words, cnt + 1);
            count_launch();
        }
    }
    if (rc == DIAQ_OK) rc = check_launch("count kernels");
    if (rc == DIAQ_OK) {
        cudaMemcpyAsync(hc, cnt, sizeof(hc), cudaMemcpyDeviceToHost, s);
        if (cudaStreamSynchronize(s) != cudaSuccess)
            rc = set_error(DIAQ_ERR_CUDA, "count sync: %s", cudaGetErrorString(cudaGetLastError()));
    }
    if (bitmap) cudaFreeAsync(bitmap, s);
    cudaFreeAsync(cnt, s);
    cudaFreeAsync(dt, s);
    if (nnz_out) *nnz_out = (int64_t)hc[0];
    if (bsr_out) *bsr_out = (int64_t)hc[1];
    return rc;
}

extern "C" int diaq_count_nonzero(const diaq_matrix_t *a, double eps, int64_t *nnz_out, int64_t *bsr_blocks_out,
                                  void *stream) {
    if (!a || eps < 0) return set_error(DIAQ_ERR_VALUE, "diaq_count_nonzero: bad arguments");
    return count_common(a, eps, nnz_out, bsr_blocks_out, stream);
}
