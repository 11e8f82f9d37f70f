// SH-3 fast path kernels for GS_MODE_ADAMW_CONST (explicit instantiation; see gs_step_sh3.cuh).
#include "gs_step_sh3.cuh"

namespace gs {
template void launch_fixed<LayoutSH3, GS_MODE_ADAMW_CONST, false>(const FixedParams&, const TmaMaps*, int64_t, int,
                                                              cudaStream_t);
template void launch_fixed<LayoutSH3, GS_MODE_ADAMW_CONST, true>(const FixedParams&, const TmaMaps*, int64_t, int,
                                                              cudaStream_t);
template void launch_fixed_masked<LayoutSH3, GS_MODE_ADAMW_CONST>(const FixedParams&, const TmaMaps&, int64_t, int,
                                                                const void*, bool, cudaStream_t);
}  // namespace gs
