/*
 * diaq_b200.h -- C-ABI of the B200-native DiaQ hot path (arXiv 2405.01250).
 *
 * The reference (/root/reference/pkg/src/diaqsim) is a pure Python package
 * with no native ABI; its drop-in boundary is the Python API re-exported by
 * diaqsim/__init__.py:5-70 (and the `kernel` JSON protocol, cli.py:251-287).
 * Every entry point below replaces one reference function; the Python host
 * mirror (paper_2405_01250_b200/) binds them with ctypes exactly the way
 * INTEGRATION.md shows a diaqsim maintainer would.
 *
 * Conventions (reference matrix.py:1-14): d = col - row; diagonal d holds
 * n-|d| values; element (r, r+d) is at storage position k = r + min(d,0).
 * On the device a matrix is one complex128 arena (interleaved re,im = one
 * 16-byte load per element) plus a host offset table:
 *   - offs[i]   ascending diagonal offsets (int64),
 *   - starts[i] element index of k=0 of diagonal i inside the arena, chosen
 *     by diaq_layout() so that row r of every diagonal sits at a 128-byte
 *     aligned address whenever r % 8 == 0 ("row-aligned" padding),
 *   - vals      device pointer to the arena (cudaMalloc / torch storage).
 * State vectors are device complex128 arrays (reference sim.py:36).
 *
 * All functions are stream-ordered (cudaStream_t passed as void*), never
 * synchronise unless documented, are reentrant per stream, and return a
 * diaq_status (0 = OK).  No CPU fallback exists: without a CUDA device
 * every compute entry point returns DIAQ_ERR_CUDA.
 */
#ifndef DIAQ_B200_H
#define DIAQ_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes; the Python mirror maps them onto the reference exception
 * types (reference errors.py:9-46) */
typedef enum {
    DIAQ_OK = 0,
    DIAQ_ERR_SHAPE = 1,     /* -> ShapeError ("not multiplyable: ..."), matrix.py:227-229,262-263 */
    DIAQ_ERR_VALUE = 2,     /* -> ValueError (bad offset / argument), matrix.py:33-34 */
    DIAQ_ERR_RESOURCE = 3,  /* -> ResourceError (size guard), sim.py:55-56, gates.py:237-240 */
    DIAQ_ERR_CUDA = 4,      /* CUDA runtime failure (no device, launch error, OOM) */
    DIAQ_ERR_UNSUPPORTED = 5
} diaq_status;

/* complex-multiply rounding of the gate apply: numpy's complex128 multiply
 * on AVX-512 hosts is re=fma(vr,xr,-(vi*xi)), im=fma(vr,xi,vi*xr)
 * (reference sim.py:76-78); PLAIN is the textbook four-product form. */
#define DIAQ_CMUL_PLAIN 0
#define DIAQ_CMUL_FMA 1
/* CONTRACT: not the reference's rounding but fused multiply-add chains
 * (a 2x2 rotation costs 4 FP64 operations per amplitude instead of 6, runs
 * of diagonal gates on non-register bits fold into one factor); results
 * agree with the reference within 1e-12 relative L2 (north_star tolerance),
 * not bitwise.  Standalone gate kernels use the FMA form under it. */
#define DIAQ_CMUL_CONTRACT 2

/* a device-resident DiaQ matrix (replaces reference DiaqMatrix,
 * matrix.py:50-123; the dict of Diagonal objects becomes offs/starts/vals) */
typedef struct {
    int64_t n;              /* n_dim */
    int64_t nd;             /* number of stored diagonals */
    const int64_t *offs;    /* host, ascending, nd entries */
    const int64_t *starts;  /* host, element start of diagonal i in vals */
    void *vals;             /* device complex128 arena */
} diaq_matrix_t;

/* ---- library / diagnostics ------------------------------------------- */
int diaq_version(void);
const char *diaq_last_error(void);               /* thread-local message */
int diaq_device_count(int *count);
uint64_t diaq_launch_count(void);                /* kernels launched by this library */
void diaq_reset_launch_count(void);
/* launch-geometry knobs (never change results): "spmv_raster" (0 strip-
 * fastest, 1 column chunks), "spmv_chunk", "spmv_xpol" (0 normal, 1 L2
 * evict_last for x), "spmv_ctas_per_sm" (0 = occupancy max),
 * "gate_ctas_per_sm"; the "fused_*" switches of the multi-gate passes
 * (csrc/common.cuh lists them) never change results in the bitwise
 * numerics modes.  Under DIAQ_CMUL_CONTRACT the schedule switches
 * ("fused_reorder", "fused_lookahead", "fused_slots", "fused_maxph",
 * "fused_slot_gates", "fused_unit") pick which gates share a pass and in
 * which form they are applied: the state stays within the mode's 1e-12
 * tolerance, and is deterministic for a given setting */
int diaq_tune(const char *key, int64_t value);

/* ---- layout (host only) ----------------------------------------------
 * Row-aligned storage starts for a diagonal set; returns total arena
 * elements in *total.  Replaces the per-diagonal aligned_zeros of
 * reference alloc.py:15-24 / matrix.py:75-76.  Offsets must be strictly
 * ascending with |d| <= n-1 (reference diag_len, matrix.py:31-35). */
int diaq_layout(int64_t n, int64_t nd, const int64_t *offs, int64_t *starts, int64_t *total);

/* ---- construction ----------------------------------------------------- */
/* I_left (x) m (x) I_right into a pre-laid-out `out` whose offs are
 * m.offs * right (reference kron_identity, matrix.py:358-387). */
int diaq_kron_identity(int64_t left, const diaq_matrix_t *m, int64_t right, diaq_matrix_t *out,
                       void *stream);

/* offsets of build_span_unitary(g, positions, span) (reference
 * gates.py:169-219): g is a HOST dense 2^k x 2^k complex128 row-major
 * matrix; offs_out has room for 4^k entries. */
int diaq_span_plan(int k, const double *g_host, const int *positions, int span, int64_t *offs_out,
                   int64_t *nd_out);
/* fill a pre-laid-out span matrix on the device */
int diaq_span_expand(int k, const double *g_host, const int *positions, int span,
                     diaq_matrix_t *out, void *stream);

/* from_dense (reference matrix.py:135-153), device dense n x n complex128
 * row-major.  Pass 1 writes keep[d+n-1] in {0,1} for all 2n-1 diagonals
 * (|re|+|im| > eps anywhere); pass 2 gathers the kept diagonals into `out`. */
int diaq_from_dense_scan(int64_t n, const void *dense, double eps, uint8_t *keep_dev,
                         void *stream);
int diaq_from_dense_fill(const void *dense, diaq_matrix_t *out, void *stream);
/* to_dense (reference matrix.py:156-167) into a zeroed device n x n buffer */
int diaq_to_dense(const diaq_matrix_t *a, void *dense, void *stream);

/* ---- accounting (reference nnz matrix.py:393-400, memory.py:29-46) --------
 * entries with |re|+|im| > eps, and (optional, NULL to skip) the number of
 * distinct 2x2 blocks holding such an entry (BSR model).  Synchronous. */
int diaq_count_nonzero(const diaq_matrix_t *a, double eps, int64_t *nnz_out, int64_t *bsr_blocks_out,
                       void *stream);

/* ---- matrix algebra around the hot path (reference matrix.py:281-355) ----
 * All in the reference's result precision (single != 0: float32 arithmetic
 * on float32-representable values, widened into the complex128 arena).
 * transpose needs no call: it relabels the arena (d -> -d).
 * diaq_arena_map: op 0 -> conj (adjoint's values), op 1 -> scale by sr+i*si,
 *   over `total` arena elements (same layout in and out). */
int diaq_arena_map(int64_t total, const void *src, void *dst, int op, double sr, double si, int single,
                   void *stream);
/* out = a + b over the union of stored diagonals (out laid out by the caller
 * with that union); per element (+0 + a) + b (matrix.py:301-315) */
int diaq_add(const diaq_matrix_t *a, const diaq_matrix_t *b, diaq_matrix_t *out, int single, void *stream);
/* out = a (x) b (matrix.py:329-355); out's offsets are {dA*nB + dB}; the
 * operands' offset/start tables also in device memory: tables_dev =
 * [offa, starta, offb, startb] */
int diaq_kron(const diaq_matrix_t *a, const diaq_matrix_t *b, const int64_t *tables_dev, diaq_matrix_t *out,
              int single, void *stream);

/* ---- spmv (reference matrix.py:253-278) -------------------------------
 * y = A x, bitwise equal to the reference (ascending d, no FMA). */
int diaq_spmv(const diaq_matrix_t *a, const void *x, void *y, void *stream);
/* y_host = A x_host with the H2D of x, the spmv and the D2H of y pipelined
 * in chunks of chunk_rows rows over three streams (host buffers should be
 * pinned).  x_dev / y_dev are n-element device scratch vectors.  Returns
 * when y_host is complete; bitwise equal to diaq_spmv. */
int diaq_spmv_host(const diaq_matrix_t *a, const void *x_host, void *y_host, void *x_dev, void *y_dev,
                   int64_t chunk_rows, void *stream);

/* ---- spgemm (reference matrix.py:173-250) -----------------------------
 * plan (host): candidate result offsets (sorted), nc <= nda*ndb. */
int diaq_spgemm_plan(int64_t n, int64_t nda, const int64_t *offa, int64_t ndb, const int64_t *offb,
                     int64_t *offc, int64_t *nc);
/* device workspace bytes needed by diaq_spgemm for these operands (plans with
 * <= 128 candidates and <= 512 pairs travel in the kernel parameters; the
 * workspace may then be NULL) */
int64_t diaq_spgemm_workspace(int64_t nda, int64_t ndb, int64_t nc);
/* multiply into the candidate layout `c` and flag keep_dev[i] = 1 iff
 * candidate i has an element with |re|+|im| > prune_eps (matrix.py:246-249).
 * single != 0: both operands are single precision -- products, sums and the
 * prune test in float32 (reference result_type, matrix.py:231). */
int diaq_spgemm(const diaq_matrix_t *a, const diaq_matrix_t *b, diaq_matrix_t *c,
                uint8_t *keep_dev, double prune_eps, int single, void *workspace, int64_t workspace_bytes,
                void *stream);
/* compact a host-planned product's keep flags into a device structure table:
 * cand_tab_dev = [offc[nc], startc[nc]]; writes *nd_dev and the kept
 * offsets/starts, ascending (no readback). */
int diaq_spgemm_compact(int64_t nc, const int64_t *cand_tab_dev, const uint8_t *keep_dev, int64_t *nd_dev,
                        int64_t *offs_dev, int64_t *starts_dev, void *stream);

/* ---- device-resident structure: spgemm with the plan on the device ----------
 * A matrix whose offset/start table lives in device memory (e.g. a product
 * whose pruned structure was never read back). */
typedef struct {
    int64_t n;
    int64_t nd_cap;         /* capacity of offs/starts (>= *nd) */
    const int64_t *nd;      /* device: number of stored diagonals */
    const int64_t *offs;    /* device: ascending offsets */
    const int64_t *starts;  /* device: element starts in vals */
    const void *vals;       /* device complex128 arena */
} diaq_dev_matrix_t;
typedef struct {
    int64_t *nd;            /* device outputs: count (negative: plan error), */
    int64_t *offs;          /*   kept offsets, ascending,                      */
    int64_t *starts;        /*   their element starts                          */
    void *vals;             /* arena of capacity elements                      */
    int64_t capacity;       /* >= nc * (n + 7) + 7 for nc candidates           */
    int64_t nd_cap;         /* entries of offs/starts                          */
} diaq_dev_result_t;
/* count products C[i] = A[i] B[i] (matmul, matrix.py:218-250): pass 1 (the
 * offset union count and scan) runs on the device from the operands' device
 * tables, pass 2 multiplies, a compaction pass prunes -- one launch of each
 * per 64 products, no host round trip.  pair_cap >= nd(A[i]) * nd(B[i])
 * (<= 1024).  Bitwise diaq_spgemm, structure included. */
int64_t diaq_spgemm_dev_workspace(int count, int64_t pair_cap);
int diaq_spgemm_dev(int count, const diaq_dev_matrix_t *a, const diaq_dev_matrix_t *b, const diaq_dev_result_t *c,
                    double prune_eps, int single, int64_t pair_cap, void *workspace, int64_t workspace_bytes,
                    void *stream);

/* ---- gate application (reference sim.py:69-105) -----------------------
 * Generic placement: y = (I_dim_a (x) m (x) I_dim_b) x over the stored
 * diagonals of m (any m, any number of diagonals: chunks of 64 continue
 * the per-amplitude sum in y, the reference's order).  y must not alias x. */
int diaq_apply_placed(int64_t dim_a, const diaq_matrix_t *m, int64_t dim_b, const void *x, void *y,
                      int cmul_mode, void *stream);

/* Compact Kronecker-structured gate: a k-qubit gate g (HOST dense 2^k x 2^k,
 * row-major complex128) acting on state bits shifts[0..k-1] (operand 0 =
 * most significant gate-index bit) of an N = 2^n_bits state.  Equals
 * apply_placed of the placement compile_circuit builds for it (incl. the
 * build_span_unitary embedding, gates.py:169-219, 242-245) with the same
 * per-element summation order.  In place allowed (x == y).  k <= 5. */
int diaq_apply_gate(int n_bits, int k, const double *g_host, const int *shifts, const void *x,
                    void *y, int cmul_mode, void *stream);

/* a compiled gate for the native program runner */
typedef struct {
    int k;                  /* gate qubits (<= 5) */
    int shifts[5];          /* state bit of operand i (operand 0 = MSB) */
    const double *g;        /* HOST dense 2^k x 2^k complex128 */
} diaq_gate_t;

/* Apply `ngates` compact gates in order to `state` (in place) on one
 * stream: the device loop of reference run(), sim.py:193-199.  If events
 * is non-NULL it must hold ngates+1 cudaEvent_t recorded around each gate
 * (per-gate timings, resolved by the caller after the loop). */
int diaq_run_gates(int n_bits, int ngates, const diaq_gate_t *gates, void *state, int cmul_mode,
                   void **events, void *stream);

/* ---- sharded state ------------------------------------------
 * The 2^n_bits state is split over P = 2^(n_bits-local_bits) ranks by its
 * top bits; rank r holds indices [r*2^local_bits, (r+1)*2^local_bits).
 * A gate's operands on bits >= local_bits are "global".  Relabel the
 * operands by descending shift; the global ones form the top kg bits of the
 * gate index.  Rank r produces only its own row block vr (its global operand
 * bit values) and reads column block v from srcs[v] (v = values of the
 * global operands, first = highest shift = most significant).
 * diaq_shard_plan (host only) reports which blocks rank r reads; the caller
 * exchanges the partner shards for those blocks, then calls
 * diaq_apply_gate_sharded (srcs[v] may be NULL for unread blocks; y may
 * alias srcs[vr], the rank's own shard). */
int diaq_shard_plan(int n_bits, int local_bits, int k, const double *g_host, const int *shifts,
                    int64_t rank, uint32_t *need_mask, int *n_global, uint32_t *own_block);
int diaq_apply_gate_sharded(int n_bits, int local_bits, int k, const double *g_host, const int *shifts,
                            int64_t rank, const void *const *srcs, void *y, int cmul_mode, void *stream);
/* diaq_run_gates_fused on one rank's shard for a run of gates that need no
 * partner data (every mixing operand local; selectors may be global bits,
 * read from `rank`).  Shifts are in the full n_bits index space. */
int diaq_run_gates_local(int n_bits, int local_bits, int64_t rank, int ngates, const diaq_gate_t *gates,
                         void *shard, int cmul_mode, int tile_bits, void **events, int *npasses, void *stream);

/* Sharded spmv: y[j] = row row0+j of A x, where x is split over
 * nparts ranks in slices of 2^part_bits (x_parts[q]: rank q's slice as
 * addressable here -- own memory or a peer mapping from diaq_ipc_open) and
 * rows[i] holds diagonal offs[i] for this rank's rows (rows[i][j] = the
 * element of row row0+j; entries of rows where the diagonal does not exist
 * are ignored).  Offsets crossing a shard boundary read the partner's x
 * in the kernel.  Bitwise diaq_spmv. */
int diaq_spmv_sharded(int64_t n, int64_t nd, const int64_t *offs, const void *const *rows, int64_t row0,
                      int64_t nrows, const void *const *x_parts, int part_bits, int nparts, void *y, void *stream);

/* ---- peer memory between the ranks of a sharded state --------
 * diaq_alloc: a cudaMalloc'd buffer (an allocation base, so exportable);
 * diaq_ipc_handle: its CUDA IPC handle (DIAQ_IPC_HANDLE_BYTES bytes) for the
 * other ranks; diaq_ipc_open maps a partner's handle into this process
 * (NVLink/NVSwitch peer access enabled lazily), so diaq_apply_gate_sharded
 * can take partner shard pointers as `srcs` and read them in the pass. */
#define DIAQ_IPC_HANDLE_BYTES 64
int diaq_alloc(int64_t bytes, void **ptr);
int diaq_free(void *ptr);
int diaq_ipc_handle(const void *ptr, void *handle_out);
int diaq_ipc_open(const void *handle, void **ptr_out);
int diaq_ipc_close(void *ptr);
/* Cross-rank ordering of the peer transport without host synchronisation:
 * an interprocess event per rank (cudaEventInterprocess), exported with
 * diaq_ipc_event_handle (DIAQ_IPC_HANDLE_BYTES bytes) and opened by the
 * partners; a rank records its event before a cross-shard gate, the ranks
 * pass a host barrier (which orders the enqueueing only), and each stream
 * waits on the partners' events before the multi-source kernel. */
int diaq_ipc_event_create(void **ev);
int diaq_ipc_event_handle(void *ev, void *handle_out);
int diaq_ipc_event_open(const void *handle, void **ev_out);
int diaq_event_record(void *ev, void *stream);
int diaq_stream_wait_event(void *stream, void *ev);
int diaq_event_destroy(void *ev);

/* ---- sampling (reference measure_all_sample, sim.py:142-161) -------------
 * hits[k] = min(#{i : cdf_i <= u_k}, N-1) with cdf = sequential float64
 * cumsum of round(|x_i|^2, 12), reproduced exactly (binade-segmented exact
 * integer scans); *norm2_out = sum |x_i|^2.  u_host: `shots` uniforms. */
int diaq_sample_hits(int64_t n_amps, const void *x, const double *u_host, int64_t shots, int64_t *hits_host,
                     double *norm2_out, void *stream);

/* ---- timing (per-gate CUDA events, resolved after the loop) ---------------- */
int diaq_timer_create(int n, void **events);
int diaq_timer_record(void *event, void *stream);
/* waits for events[n-1]; ms_out[i] = milliseconds from events[i] to events[i+1]
 * (from the last recorded event before i+1; 0 if events[i+1] was never recorded) */
int diaq_timer_elapsed(int n, void **events, float *ms_out);
int diaq_timer_destroy(int n, void **events);

/* Same result as diaq_run_gates (bitwise), but consecutive gates whose
 * mixing operand bits fit in a tile of 2^tile_bits amplitudes (low bits
 * included) are applied in ONE pass over HBM through shared memory.
 * Operands a gate does not mix (controls, diagonal gates) may lie outside
 * the tile.  tile_bits 11 or 12; <= 0 schedules both and keeps the one
 * with fewer passes (ties: 11); *npasses (optional)
 * receives the number of HBM passes.  events: as diaq_run_gates, except
 * that a pass records only its last gate's event (its time lands on that
 * gate; diaq_timer_elapsed reads the unrecorded intervals as 0). */
int diaq_run_gates_fused(int n_bits, int ngates, const diaq_gate_t *gates, void *state, int cmul_mode,
                         int tile_bits, void **events, int *npasses, void *stream);

/* The fused passes take a state-sized permutation buffer from the device's
 * default stream-ordered pool and keep freed pool memory reserved for the
 * next call; diaq_trim_pool synchronises the device and returns it. */
int diaq_trim_pool(void);

/* Host-only view of the fused schedule (no device work): stats[0] HBM
 * passes, [1] of them single-gate (gate kernel), [2] register/smem phases
 * in the tiled passes, [3] permutation gates folded into pass addressing,
 * [4] shared-memory (generic) phases.  local_bits < n_bits: one rank's
 * shard, as diaq_run_gates_local. */
int diaq_fused_plan(int n_bits, int local_bits, int ngates, const diaq_gate_t *gates, int tile_bits, int *stats);
/* The same for the schedule a numerics mode runs: DIAQ_CMUL_CONTRACT takes
 * the commutation-aware schedule when it needs fewer passes. */
int diaq_fused_plan_mode(int n_bits, int local_bits, int ngates, const diaq_gate_t *gates, int tile_bits,
                         int cmul_mode, int *stats);

/* ---- specialised fused passes (NVRTC) ------------------------------------
 * Each tiled pass is also compiled at run time with its structure (tile
 * bits, phases, gate records) constant -- the same device code as the AOT
 * pass kernel, bitwise the same results, without the per-gate decode.
 * Compiles run on a background thread (knob fused_jit: 0 off, 1 async,
 * 2 compile before the first launch); until a pass's kernel is ready the
 * AOT kernel runs it. */
/* wait until no specialised pass is compiling (timeout_s < 0: no limit) */
int diaq_jit_wait(double timeout_s);
/* stats[0] passes compiled, [1] failed, [2] specialised launches,
 * [3] modules loaded, [4] pending, [5] total compile milliseconds */
int diaq_jit_stats(int64_t *stats);
/* last compile / load error text ("" if none) */
const char *diaq_jit_last_error(void);
/* host-only: schedule and compile a program's specialised passes now (no
 * device, no cache); *seconds compile time, *kernels passes compiled.
 * seconds == NULL: submit them to the background compile queue instead
 * (as the first diaq_run_gates_fused call of the program would) and return. */
int diaq_fused_jit_compile(int n_bits, int local_bits, int ngates, const diaq_gate_t *gates, int tile_bits,
                           int cmul_mode, double *seconds, int *kernels);

/* ---- state helpers ------------------------------------------------------ */
/* |index> (reference init_state, sim.py:53-59) */
int diaq_init_basis(int64_t n_amps, void *x, int64_t index, void *stream);
/* sum |x_i|^2 (reference StateVector.norm, sim.py:38-39, squared) into
 * work_dev[0]; work_dev holds DIAQ_NORM_WORK device doubles (partials in
 * 1..); fixed two-pass order, so repeated calls are bitwise identical. */
#define DIAQ_NORM_WORK 1025
int diaq_norm2(int64_t n_amps, const void *x, double *work_dev, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* DIAQ_B200_H */
