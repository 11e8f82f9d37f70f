// The SH-3 fast path: variant switch, dispatch over the step modes and the
// C-ABI hook.  The kernels are in gs_step_sh3.cuh; each mode is instantiated
// in its own translation unit (gs_step_sh3_m<mode>.cu).
#include <cstring>
#include "gs_step_sh3.cuh"

namespace gs {

extern template void launch_fixed<LayoutSH3, GS_MODE_COUPLED_ADAM, false>(const FixedParams&, const TmaMaps*,
                                                          int64_t, int, cudaStream_t);
extern template void launch_fixed<LayoutSH3, GS_MODE_COUPLED_ADAM, true>(const FixedParams&, const TmaMaps*,
                                                          int64_t, int, cudaStream_t);
extern template void launch_fixed<LayoutSH3, GS_MODE_SPARSE_ADAM, false>(const FixedParams&, const TmaMaps*,
                                                          int64_t, int, cudaStream_t);
extern template void launch_fixed<LayoutSH3, GS_MODE_SPARSE_ADAM, true>(const FixedParams&, const TmaMaps*,
                                                          int64_t, int, cudaStream_t);
extern template void launch_fixed<LayoutSH3, GS_MODE_ADAMW_CONST, false>(const FixedParams&, const TmaMaps*,
                                                          int64_t, int, cudaStream_t);
extern template void launch_fixed<LayoutSH3, GS_MODE_ADAMW_CONST, true>(const FixedParams&, const TmaMaps*,
                                                          int64_t, int, cudaStream_t);
extern template void launch_fixed<LayoutSH3, GS_MODE_ADAMW_CONST_CLIP, false>(const FixedParams&, const TmaMaps*,
                                                          int64_t, int, cudaStream_t);
extern template void launch_fixed<LayoutSH3, GS_MODE_ADAMW_CONST_CLIP, true>(const FixedParams&, const TmaMaps*,
                                                          int64_t, int, cudaStream_t);
extern template void launch_fixed<LayoutSH3, GS_MODE_ADAMW_GS, false>(const FixedParams&, const TmaMaps*,
                                                          int64_t, int, cudaStream_t);
extern template void launch_fixed<LayoutSH3, GS_MODE_ADAMW_GS, true>(const FixedParams&, const TmaMaps*,
                                                          int64_t, int, cudaStream_t);

extern template void launch_fixed_masked<LayoutSH3, GS_MODE_SPARSE_ADAM>(
    const FixedParams&, const TmaMaps&, int64_t, int, const void*, bool, cudaStream_t);
extern template void launch_fixed_masked<LayoutSH3, GS_MODE_ADAMW_CONST>(
    const FixedParams&, const TmaMaps&, int64_t, int, const void*, bool, cudaStream_t);
extern template void launch_fixed_masked<LayoutSH3, GS_MODE_ADAMW_CONST_CLIP>(
    const FixedParams&, const TmaMaps&, int64_t, int, const void*, bool, cudaStream_t);
extern template void launch_fixed_masked<LayoutSH3, GS_MODE_ADAMW_GS>(
    const FixedParams&, const TmaMaps&, int64_t, int, const void*, bool, cudaStream_t);

static int g_fixed_variant = -1;

static bool g_fixed_variant_set = false;

int fixed_variant() {
  if (!g_fixed_variant_set) {
    const char* e = getenv("GS_FIXED_VARIANT");
    g_fixed_variant = e ? atoi(e) : 0;
    g_fixed_variant_set = true;
  }
  return g_fixed_variant;
}

template <class L, bool STRICT>
void dispatch_fixed(int mode, const FixedParams& P, const TmaMaps* M, int64_t max_rows, int kind,
                    cudaStream_t s) {
  switch (mode) {
    case GS_MODE_COUPLED_ADAM:
      launch_fixed<L, GS_MODE_COUPLED_ADAM, STRICT>(P, M, max_rows, kind, s);
      break;
    case GS_MODE_SPARSE_ADAM:
      launch_fixed<L, GS_MODE_SPARSE_ADAM, STRICT>(P, M, max_rows, kind, s);
      break;
    case GS_MODE_ADAMW_CONST:
      launch_fixed<L, GS_MODE_ADAMW_CONST, STRICT>(P, M, max_rows, kind, s);
      break;
    case GS_MODE_ADAMW_CONST_CLIP:
      launch_fixed<L, GS_MODE_ADAMW_CONST_CLIP, STRICT>(P, M, max_rows, kind, s);
      break;
    default: launch_fixed<L, GS_MODE_ADAMW_GS, STRICT>(P, M, max_rows, kind, s); break;
  }
}

// 0 dense, 1 strided, 2 records (see launch_fixed); -1 if 32-bit element
// offsets could overflow
template <class L>
int rows_kind(const gs_group* groups, int64_t max_rows, FixedParams& P) {
  constexpr int PL = WsStage<L, 32>::kPL;
  bool dense = true, prec = true, grec = true;
  int64_t smax = 1;
  const int64_t ps0 = groups[0].param_stride ? groups[0].param_stride : groups[0].width;
  const int64_t gs0 = groups[0].grad_stride ? groups[0].grad_stride : groups[0].width;
  for (int i = 0; i < L::G; ++i) {
    const gs_group& g = groups[i];
    const int64_t ps = g.param_stride ? g.param_stride : g.width;
    const int64_t gs = g.grad_stride ? g.grad_stride : g.width;
    dense = dense && ps == g.width && gs == g.width;
    prec = prec && ps == ps0 && g.param == groups[0].param + L::OFF(i);
    grec = grec && gs == gs0 && g.grad == groups[0].grad + L::OFF(i);
    smax = std::max(smax, std::max(ps, gs));
  }
  // past 2^32 elements of row offset only the record ring kernel runs, with
  // 64-bit offsets (P.wide); everything else falls back to the generic kernels
  const bool wide = max_rows * smax + smax >= (int64_t)UINT32_MAX;
  if (dense && !wide) return 0;
  prec = prec && ps0 >= PL && ps0 % 4 == 0 && (reinterpret_cast<uintptr_t>(groups[0].param) & 15u) == 0;
  grec = grec && gs0 >= PL && gs0 % 4 == 0 && (reinterpret_cast<uintptr_t>(groups[0].grad) & 15u) == 0;
  if (prec && grec) {
    P.prec = groups[0].param;
    P.grec = groups[0].grad;
    P.prs = (uint32_t)ps0;
    P.grs = (uint32_t)gs0;
    cudaPointerAttributes a{};
    const bool host = cudaPointerGetAttributes(&a, groups[0].grad) == cudaSuccess &&
                      a.type == cudaMemoryTypeHost;
    (void)cudaGetLastError();
    const char* e = getenv("GS_GREC_CA");
    P.grec_ca = e ? atoi(e) : (host ? 1 : 0);
    P.wide = wide ? 1 : 0;
    return 2;
  }
  return wide ? -1 : 1;
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
  static std::atomic<EncodeTiledFn> fn{nullptr};
  EncodeTiledFn f = fn.load(std::memory_order_acquire);
  if (f == nullptr) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || p == nullptr) {
      (void)cudaGetLastError();
      return nullptr;
    }
    f = reinterpret_cast<EncodeTiledFn>(p);
    fn.store(f, std::memory_order_release);
  }
  return f;
}

// 2-D fp32 map [n_rows, stride] with a one-row box of `box` columns (the
// gather4 / scatter4 operations move four such rows); rows past n_rows are
// out of bounds (zero-filled on load, dropped on store).
static bool encode_rows(CUtensorMap* m, const float* base, int64_t n_rows, int64_t stride, int box) {
  EncodeTiledFn enc = encode_fn();
  if (enc == nullptr || n_rows < 1 || n_rows > INT32_MAX) return false;
  const cuuint64_t dim[2] = {(cuuint64_t)stride, (cuuint64_t)n_rows};
  const cuuint64_t str[1] = {(cuuint64_t)stride * 4};
  const cuuint32_t boxd[2] = {(cuuint32_t)box, 1};
  const cuuint32_t es[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dim, str, boxd, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool encode_tma_maps(const FixedParams& P, int64_t n_rows, int rec_box, TmaMaps* out) {
  // the last encoding per host thread is reused when the records did not
  // move (three cuTensorMapEncodeTiled calls cost a few us of the host's
  // per-step time, which small clouds feel)
  struct Key {
    const void *rec, *prm, *grd;
    int64_t n, st, ps, gs;
    int box;
    int dev;
  };
  static thread_local Key last{};
  static thread_local TmaMaps cached;
  static thread_local bool valid = false;
  int dev = 0;
  cudaGetDevice(&dev);
  const Key k{P.record, P.prec, P.grec, n_rows, P.stride, (int64_t)P.prs, (int64_t)P.grs, rec_box,
              dev};
  if (valid && std::memcmp(&k, &last, sizeof(Key)) == 0) {
    *out = cached;
    return true;
  }
  valid = false;
  const bool ok = encode_rows(&out->rec, P.record, n_rows, P.stride, rec_box) &&
                  encode_rows(&out->prm, P.prec, n_rows, P.prs, Tma4Stage<LayoutSH3, 32>::kPT) &&
                  encode_rows(&out->grd, P.grec, n_rows, P.grs, Tma4Stage<LayoutSH3, 32>::kPT);
  if (ok) {
    last = k;
    cached = *out;
    valid = true;
  }
  return ok;
}

template <class L>
bool layout_matches(const gs_group* groups, int n_groups) {
  if (n_groups != L::G) return false;
  for (int i = 0; i < L::G; ++i) {
    if (groups[i].width != L::W(i) || groups[i].role != L::ROLE(i)) return false;
  }
  return true;
}

}  // namespace gs

extern "C" int32_t gs_set_fixed_variant(int32_t variant) {
  const int32_t prev = gs::fixed_variant();
  gs::g_fixed_variant = variant;
  return prev;
}

namespace gs {

// The launch parameters of the fixed-layout kernels; false if the layout or
// the record does not fit them.  tma4: the 2-D TMA kernel may run.
static bool fixed_setup(const gs_group* groups, int32_t n_groups, const gs_step_cfg* cfg,
                        const int32_t* rows, const int32_t* n_rows_dev, int64_t max_rows,
                        float* record, int64_t record_stride, double* stats_out, double* partials,
                        unsigned int* counter, FixedParams& P, int& kind, bool& tma4) {
  if (fixed_variant() < 0) return false;  // fixed-layout path disabled
  if (!layout_matches<LayoutSH3>(groups, n_groups)) return false;
  // every fixed-layout kernel copies the state record in 16-byte pieces
  if (record_stride % 4 != 0 || (reinterpret_cast<uintptr_t>(record) & 15u) != 0) return false;
  P = FixedParams{};
  kind = rows_kind<LayoutSH3>(groups, max_rows, P);
  if (kind < 0) return false;  // 32-bit element offsets
  P.tma_ok = kind == 2 && P.grec_ca == 0 && record_stride % 4 == 0 &&
             (reinterpret_cast<uintptr_t>(record) & 15u) == 0;
  // 2-D TMA kernel: device-resident records, 16-byte row strides, whole
  // 64-float parameter / gradient rows and a state row of >= 2(P+1) floats
  constexpr int kPT = Tma4Stage<LayoutSH3, 32>::kPT;
  tma4 = P.tma_ok && P.prs >= kPT && P.grs >= kPT && P.prs % 4 == 0 && P.grs % 4 == 0 &&
         record_stride >= 2 * (LayoutSH3::P + 1) && max_rows <= INT32_MAX;
  for (int i = 0; i < n_groups; ++i)
    P.g[i] = FixedGroup{
        groups[i].param, groups[i].grad, groups[i].lr,
        (uint32_t)(groups[i].param_stride ? groups[i].param_stride : groups[i].width),
        (uint32_t)(groups[i].grad_stride ? groups[i].grad_stride : groups[i].width)};
  P.active_logit = cfg->active_logit;
  P.K = make_consts(cfg);
  P.lut = cfg->bias_lut;
  P.lut_len = cfg->lut_len;
  P.global_t = cfg->global_t;
  P.nv_dev = cfg->n_visible_norm;
  P.nv_host = cfg->n_visible_host;
  P.abort_flag = cfg->abort_flag;
  P.D = DensifyArgs{cfg->densify_accum, cfg->densify_count, cfg->densify_scale,
                    cfg->densify_group};
  P.rows = rows;
  P.n_rows_dev = n_rows_dev;
  P.max_rows = max_rows;
  P.record = record;
  P.stride = record_stride;
  P.stats_out = stats_out;
  P.partials = partials;
  P.counter = counter;
  return true;
}

}  // namespace gs

// Called by gs_step_rows (gs_step_rows.cu) after argument validation; returns
// 1 if a compiled fixed layout handled the launch, 0 otherwise.
int gs_step_fixed_try(const gs_group* groups, int32_t n_groups, const gs_step_cfg* cfg,
                      const int32_t* rows, const int32_t* n_rows_dev, int64_t max_rows,
                      float* record, int64_t record_stride, double* stats_out, double* partials,
                      unsigned int* counter, void* stream) {
  using namespace gs;
  FixedParams P;
  int kind = 0;
  bool tma4 = false;
  if (!fixed_setup(groups, n_groups, cfg, rows, n_rows_dev, max_rows, record, record_stride,
                   stats_out, partials, counter, P, kind, tma4))
    return 0;
  cudaStream_t s = (cudaStream_t)stream;
  TmaMaps maps;
  const TmaMaps* M = nullptr;
  if (tma4 && encode_tma_maps(P, max_rows, 2 * (LayoutSH3::P + 1), &maps)) M = &maps;
  if (cfg->check == GS_CHECK_STRICT)
    dispatch_fixed<LayoutSH3, true>(cfg->mode, P, M, max_rows, kind, s);
  else
    dispatch_fixed<LayoutSH3, false>(cfg->mode, P, M, max_rows, kind, s);
  return 1;
}

// The fused compaction + step (gs_step_rows_masked): 1 if launched.  Needs
// the TMA record kernel, the fused check and a mode whose step does not
// depend on the global visible count (not the coupled normaliser N_v).
constexpr int kFusedMinTilesPerSlot = 16;

int gs_step_fixed_masked_try(const gs_group* groups, int32_t n_groups, const gs_step_cfg* cfg,
                             const uint8_t* mask, const int32_t* radii, int64_t n_rows,
                             float* record, int64_t record_stride, double* stats_out,
                             double* partials, unsigned int* counter, unsigned int* tp_bar,
                             int32_t* tp_counts, int32_t* tp_ids, unsigned int* tile_ctr,
                             int32_t flags, void* stream) {
  using namespace gs;
  if (cfg->check != GS_CHECK_FUSED || cfg->mode == GS_MODE_COUPLED_ADAM) return 0;
  if (fixed_variant() == 21 || n_rows < 1) return 0;
  // GS_FUSED_MODE (measurement): 1 = the streaming loader, 2 = two-phase
  static const int fm = getenv("GS_FUSED_MODE") ? atoi(getenv("GS_FUSED_MODE")) : 0;
  const bool tp_ok = tp_ids != nullptr && tp_counts != nullptr;
  // small clouds (under 16 one-KB mask tiles per CTA slot): the streaming
  // loader gives every CTA its own mask slice (dealt whole tiles, a few
  // tiles would idle most SMs); index-coherent masks (the caller's
  // GS_MASKED_COHERENT hint) pile their visible rows into a few slices, and
  // the coupled normaliser needs N_v first: both take the two-phase kernel,
  // which balances the visible rows and counts them
  // (profiles/r02/small_clouds.txt)
  const int64_t tile_rows = radii ? 256 : 1024;
  const bool small =
      (n_rows + tile_rows - 1) / tile_rows < kFusedMinTilesPerSlot * 2 * (int64_t)gs_sm_count();
  const bool coupled_nv = cfg->mode == GS_MODE_SPARSE_ADAM &&
                          (cfg->lambda_opacity != 0.0 || cfg->lambda_scale != 0.0) &&
                          cfg->n_visible_norm == nullptr;
  bool two;
  if (fm == 2) two = tp_ok;
  else if (fm == 1) two = false;
  else two = tp_ok && small && ((flags & GS_MASKED_COHERENT) != 0 || coupled_nv);
  // the streaming kernels need N_v on the device before the step
  if (!two && coupled_nv) return 0;
  // the loader streams 2-KB mask tiles with 16-byte bulk copies
  if ((reinterpret_cast<uintptr_t>(radii ? static_cast<const void*>(radii)
                                         : static_cast<const void*>(mask)) & 15u) != 0)
    return 0;
  FixedParams P;
  int kind = 0;
  bool tma4 = false;
  if (!fixed_setup(groups, n_groups, cfg, nullptr, nullptr, n_rows, record, record_stride,
                   stats_out, partials, counter, P, kind, tma4) ||
      kind != 2 || !tma4)
    return 0;
  TmaMaps maps;
  if (!encode_tma_maps(P, n_rows, 2 * (LayoutSH3::P + 1), &maps)) return 0;
  static const int slices = getenv("GS_MASK_SLICES") ? atoi(getenv("GS_MASK_SLICES")) : 0;
  P.mask_slices = slices;  // measurement override of the streaming kernel's mask dealing
  // the streaming kernel deals the last eighth of its mask tiles dynamically
  // when the caller's hint says the mask is not very sparse (>= 2 % visible:
  // c5 30% 4.22 against 4.34 ms, 3% 0.452 against 0.479, c3 0.5345 against
  // 0.5366; at 1% the claims cost more than the balance gains, 0.198 against
  // 0.185; profiles/r02/small_clouds.txt).  GS_DYN_TAIL=0/k forces off /
  // k eighths (measurement).
  static const int dyn_env = getenv("GS_DYN_TAIL") ? atoi(getenv("GS_DYN_TAIL")) : -1;
  const int dyn = dyn_env >= 0 ? dyn_env : ((flags & GS_MASKED_BALANCE_TAIL) ? 1 : 0);
  P.tile_ctr = (!two && dyn >= 1) ? tile_ctr : nullptr;
  P.dyn_eighths = dyn >= 1 ? (dyn < 8 ? dyn : 7) : 0;
  const int mk = (radii ? 2 : 1) + (two ? 2 : 0);
  if (two) {
    P.tp_ids = tp_ids;
    P.tp_counts = tp_counts;
    P.tp_bar = tp_bar;
  }
  const bool low = (flags & GS_MASKED_LOW_VISIBILITY) != 0;
  const void* m = radii ? static_cast<const void*>(radii) : static_cast<const void*>(mask);
  cudaStream_t s = (cudaStream_t)stream;
  switch (cfg->mode) {
    case GS_MODE_SPARSE_ADAM:
      launch_fixed_masked<LayoutSH3, GS_MODE_SPARSE_ADAM>(P, maps, n_rows, mk, m, low, s);
      break;
    case GS_MODE_ADAMW_CONST:
      launch_fixed_masked<LayoutSH3, GS_MODE_ADAMW_CONST>(P, maps, n_rows, mk, m, low, s);
      break;
    case GS_MODE_ADAMW_CONST_CLIP:
      launch_fixed_masked<LayoutSH3, GS_MODE_ADAMW_CONST_CLIP>(P, maps, n_rows, mk, m, low, s);
      break;
    default: launch_fixed_masked<LayoutSH3, GS_MODE_ADAMW_GS>(P, maps, n_rows, mk, m, low, s); break;
  }
  return 1;
}
