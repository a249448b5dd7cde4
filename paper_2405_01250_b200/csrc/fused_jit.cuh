// fused_jit.cuh -- host interface of the runtime-specialised fused passes
// (fused_jit.cu) used by the pass driver in fused.cu.
#pragma once
#include <memory>
#include <vector>

#include "fused_dev.cuh"

namespace diaq {
struct JitPass;
// Look up or submit (asynchronously unless sync) the specialised kernels of a
// program's passes; out[i] is null for untiled passes (null inputs).
void jit_request(const std::vector<const TileParams *> &passes, int R, int mode, bool sync,
                 std::vector<std::shared_ptr<JitPass>> &out);
// Launch pass `ps` if its kernel is ready on this device (sets p.nbuf and
// p.gstep like the AOT launch); false: not ready, launch the AOT kernel.
bool jit_launch(const std::shared_ptr<JitPass> &ps, TileParams &p, int R, size_t smem_for_nbuf1,
                size_t smem_for_nbuf2, int knob_nbuf, cudaStream_t s, int &rc);
// Host-only compile of the given passes (no cache, no device)
int jit_compile_now(const std::vector<const TileParams *> &passes, int R, int mode, double &seconds, int &kernels);
}  // namespace diaq
