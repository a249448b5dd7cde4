// common.cuh -- shared device helpers for the DiaQ sm_100a kernels.
//
// Device helpers live in dev_common.cuh (also compiled by the NVRTC path).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/diaq_b200.h"
#include "dev_common.cuh"

// ---- host-side error plumbing (defined in abi.cu) ------------------------
namespace diaq {
// launch-geometry knobs (diaq_tune); results never depend on them
struct Tuning {
    int spmv_raster = 1;       // 0: strips fastest per tile, 1: column chunks
    int spmv_chunk = 8;        // strips per work item in raster 1
    int spmv_xpol = 0;         // 0: x evict_normal, 1: x evict_last
    int spmv_ctas_per_sm = 0;  // 0: occupancy maximum
    int spmv_banded = 1;       // stage banded x windows in shared memory
    int spmv_strips = 1;       // strip raster for far offsets (0: plain row order)
    int spmv_tma = 0;          // banded path through the TMA bulk-copy pipeline (opt-in: measured slower)
    int spmv_tma_stages = 4;   // tiles in flight per CTA
    int spmv_async = 1;        // banded path through cp.async (LDGSTS) staging (default: fastest)
    int gate_ctas_per_sm = 32;
    int fused_dense2 = 1;      // dense two-qubit gates in registers (sequence phases)
    int fused_gperm_rows = 0;  // 1: global tails only while they keep 128-byte rows whole (measured slower: an extra pass costs more than partial-row writes)
    int fused_gperm = 1;       // trailing permutation runs leaving the tile folded into the pass's store
    int fused_seq = 1;         // sequence phases (compile-time register bit per dense step)
    int fused_nbuf = 0;        // fused pass tile buffers: 0 auto (2 unless it costs occupancy), 1, 2
    int fused_tbits = 7;       // thread bits of the fused passes (8: 256 threads; 7: 128 threads x 16 amplitudes, T = 11)
    int fused_jit = 1;         // fused passes specialised per structure (NVRTC): 0 off, 1 async, 2 compile first
    int fused_gstore = 0;      // global-map (out-of-place permuted) store policy: 0 .cs, 1 default, 2 evict_last
    int fused_bank_spread = 3;  // fused passes, quarter-warp lanes on bank-spreading positions: 1 phase
                                // thread bits, 2 pair-store destination basis (bitmask)
    int fused_dstore = 0;      // plain-pair passes: last phase stored from registers (TileParams::dstore; measured 1.72 vs 1.68 ms, r02o)
    int fused_ppipe = 0;       // plain-pair schedule (TileParams::ppipe)
    int fused_plain_pair = 1;  // specialised passes over 128-byte tile rows: tiles paired across bit 3 (256-byte DRAM runs)
    int fused_pair_store = 2;  // specialised passes: sector-splitting global tails stored as tile pairs
                               // (2: any tile, 1: 11-bit tiles only, 0: off)
    int fused_perm = 1;        // fold permutation gates (X/CX/SWAP) into the fused passes' smem addressing
    int kron_flat = 1;         // kron_identity as one arena-linear store stream
    int kron_ctas_per_sm = 32;  // CTAs per SM launched (4 resident; later ones refill)
    int fused_estore = 1;      // pair passes: store gathered into registers, next fetch issued before the HBM writes
                               // (n=28 layer, contracted: 1.615 -> 1.574 ms per pass, r02f)
    int fused_reorder = 1;     // contracted arithmetic: schedule passes with commutation-aware deferral
    int fused_dyn = 1;         // units handed out in order by a global counter (TileParams::uctr): adjacent DRAM runs fetched
                               // together (n=28 layer 1.554 -> 1.434 ms per contracted pass, config 5 339 -> 305 ms, r02n)
    int fused_lookahead = 1;   // contracted arithmetic: each pass's tile bits chosen by trial sweeps (fused.cu schedule_once)
    int fused_maxph = 5;       // contracted arithmetic: phases (shared-memory round trips) per pass at most (config 5 n=30 with slots: 204/182/178/193 ms at 3/4/5/6; without: 237/223/214/198/215/286 ms at 3..8, r02u)
    int fused_slots = 1;       // contracted arithmetic: gates placed into the earliest phase slot, X/CX/SWAP on register bits as exchanges
    int fused_slot_gates = 6;  // ... at most this many non-diagonal gate records per slot (the specialised kernels unroll longer gate loops only partly: 8 left 3 of 23 config-5 kernels with run-time dispatch)
    int fused_unit = 1;        // contracted arithmetic: rotations in unit-diagonal form, 2 FP64 operations per amplitude
    uint64_t epoch = 0;         // bumped by every diaq_tune (launch caches key on it)
};
Tuning &tuning();
// SM count of the current device and resident CTAs per SM of a kernel,
// asked of the runtime once per (device, kernel, block, smem) -- each query
// costs microseconds, which is the whole budget of a small launch
int sm_count();
int occupancy(const void *kernel, int threads, size_t smem);
int set_error(int code, const char *fmt, ...);
void count_launch(int n = 1);
int check_launch(const char *what);
// record a per-gate timer event and mark it as recorded for the next
// diaq_timer_elapsed (events of gates inside a fused pass are not recorded)
cudaError_t timer_record(void *event, cudaStream_t s);
}  // namespace diaq
