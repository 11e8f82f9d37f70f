// SH-3 fast path kernels for GS_MODE_SPARSE_ADAM (explicit instantiation; see gs_step_sh3.cuh).
#include "gs_step_sh3.cuh"

namespace gs {
template void launch_fixed<LayoutSH3, GS_MODE_SPARSE_ADAM, false>(const FixedParams&, const TmaMaps*, int64_t, int,
                                                              cudaStream_t);
template void launch_fixed<LayoutSH3, GS_MODE_SPARSE_ADAM, true>(const FixedParams&, const TmaMaps*, int64_t, int,
                                                              cudaStream_t);
template void launch_fixed_masked<LayoutSH3, GS_MODE_SPARSE_ADAM>(const FixedParams&, const TmaMaps&, int64_t, int,
                                                                const void*, bool, cudaStream_t);
}  // namespace gs
