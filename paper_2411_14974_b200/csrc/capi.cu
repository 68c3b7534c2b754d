// extern "C" boundary of libconvexsplat_sm100.so (include/convexsplat_b200.h).
#include <cstring>

#include "common.cuh"

namespace cs {
struct Scratch;
}

namespace {

int validate(const cs_camera *cam, const cs_settings *set, int64_t n, int32_t k) {
  if (!cam || !set) return CS_ERR_ARG;
  if (n < 0 || n > (int64_t)0x7fffffff) return CS_ERR_ARG;
  if (k < 3 || k > 16) return CS_ERR_ARG;
  if (cam->width <= 0 || cam->height <= 0) return CS_ERR_ARG;
  if (cam->width > 32767 || cam->height > 32767) return CS_ERR_UNSUPPORTED;  // 16-bit bbox packing
  if (set->tile != cs::kTile) return CS_ERR_UNSUPPORTED;
  if (set->sh_degree < 0 || set->sh_degree > 3) return CS_ERR_UNSUPPORTED;
  if (set->scaling_mode < 0 || set->scaling_mode > 3) return CS_ERR_ARG;
  return CS_OK;
}

}  // namespace

extern "C" {

int cs_abi_version(void) { return CS_ABI_VERSION; }

const char *cs_error_string(int code) {
  switch (code) {
    case CS_OK: return "ok";
    case CS_ERR_ARG: return "bad argument";
    case CS_ERR_CUDA: return "CUDA launch failure";
    case CS_ERR_WORKSPACE: return "workspace too small";
    case CS_ERR_NONFINITE: return "non-finite gradient";
    case CS_ERR_UNSUPPORTED: return "unsupported setting (tile size must be 16, sh_degree 0..3)";
    default: return "unknown error";
  }
}

int cs_workspace_layout(const cs_camera *cam, const cs_settings *set, int64_t n, int32_t k,
                        int64_t pair_capacity, cs_layout *out) {
  int rc = validate(cam, set, n, k);
  if (rc) return rc;
  if (!out || pair_capacity < 0 || pair_capacity > (int64_t)0x3fffffff) return CS_ERR_ARG;
  cs_layout L;
  std::memset(&L, 0, sizeof(L));
  L.max_k = k <= 8 ? 8 : 16;
  L.rec_floats = cs::R_HEADER;
  L.acc_floats = cs::A_LINES + 3 * L.max_k;
  L.tiles_x = (cam->width + cs::kTile - 1) / cs::kTile;
  L.tiles_y = (cam->height + cs::kTile - 1) / cs::kTile;
  const int tiles = L.tiles_x * L.tiles_y;
  const int pp = cs::pair_sort_passes(tiles);
  if (pp > 3) return CS_ERR_UNSUPPORTED;
  const size_t npix = (size_t)cam->width * cam->height;
  const size_t un = (size_t)n, cap = (size_t)pair_capacity;
  size_t off = 0;
  auto take = [&](size_t bytes) { size_t o = off; off = cs::align_up(off + bytes, 256); return o; };
  L.counters = take(sizeof(uint32_t) * cs::C_COUNT);
  L.records = take(sizeof(float) * un * L.rec_floats);
  L.lines = take(sizeof(double) * un * 4 * L.max_k);
  L.hull = take(un * L.max_k);
  L.bbox = take(sizeof(int32_t) * 4 * un);
  L.depth_keys = take(sizeof(uint64_t) * un);
  L.order = take(sizeof(uint32_t) * un);
  L.tiles_touched = take(sizeof(uint32_t) * un);
  L.pair_offsets = take(sizeof(uint32_t) * (un + 1));
  L.pair_tiles = take(sizeof(uint32_t) * cap);
  L.pair_ids = take(sizeof(uint32_t) * cap);
  L.tile_ranges = take(sizeof(uint32_t) * 2 * tiles);
  L.pixel_last = take(sizeof(int32_t) * npix);
  L.pixel_T = take(sizeof(float) * npix);
  L.pixel_clamp = take(npix);
  L.grad_accum = take(sizeof(cs::AccT) * un * L.acc_floats);
  L.scratch_bytes = cs::scratch_bytes(n, pair_capacity, pp, tiles, nullptr, nullptr);
  L.scratch = take(L.scratch_bytes);
  L.total_bytes = off;
  *out = L;
  return CS_OK;
}

int cs_forward_ex(const cs_camera *cam, const cs_settings *set, const cs_params *params, void *workspace,
                  size_t workspace_bytes, int64_t pair_capacity, const cs_frame *frame, uint32_t flags,
                  int32_t first_stage, int32_t last_stage, void *stream) {
  if (!params || !frame || !workspace) return CS_ERR_ARG;
  if (flags & ~(uint32_t)CS_WORK_COUNTERS) return CS_ERR_ARG;
  if (first_stage < 0 || last_stage > 2 || first_stage > last_stage) return CS_ERR_ARG;
  cs_layout L;
  int rc = cs_workspace_layout(cam, set, params->n, params->k, pair_capacity, &L);
  if (rc) return rc;
  if (workspace_bytes < L.total_bytes) return CS_ERR_WORKSPACE;
  if (!frame->image || !frame->final_T || !frame->count || !frame->weight_sum) return CS_ERR_ARG;
  if (params->n > 0 && (!params->points || !params->raw_delta || !params->raw_sigma || !params->raw_opacity ||
                        !params->raw_mask || !params->sh))
    return CS_ERR_ARG;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  char *ws = static_cast<char *>(workspace);
  if (first_stage <= 0 && last_stage >= 0) {
    cudaMemsetAsync(ws + L.counters, 0, sizeof(uint32_t) * cs::C_COUNT, s);
    if ((rc = cs::launch_preprocess(*cam, *set, *params, L, ws, s))) return rc;
  }
  if (first_stage <= 1 && last_stage >= 1)
    if ((rc = cs::launch_binning(*cam, *set, *params, L, ws, pair_capacity, s))) return rc;
  if (first_stage <= 2 && last_stage >= 2)
    if ((rc = cs::launch_forward_blend(*cam, *set, *params, L, ws, *frame, (flags & CS_WORK_COUNTERS) != 0, s)))
      return rc;
  return CS_OK;
}

int cs_forward_record(const cs_camera *cam, const cs_settings *set, const cs_params *params, void *workspace,
                      size_t workspace_bytes, int64_t pair_capacity, const cs_frame *frame, const int64_t *offsets,
                      int32_t *positions, void *stream) {
  if (!params || !frame || !workspace || !offsets || !positions) return CS_ERR_ARG;
  cs_layout L;
  int rc = cs_workspace_layout(cam, set, params->n, params->k, pair_capacity, &L);
  if (rc) return rc;
  if (workspace_bytes < L.total_bytes) return CS_ERR_WORKSPACE;
  if (!frame->image || !frame->final_T || !frame->count || !frame->weight_sum) return CS_ERR_ARG;
  return cs::launch_forward_blend(*cam, *set, *params, L, static_cast<char *>(workspace), *frame, false,
                                  reinterpret_cast<cudaStream_t>(stream), offsets, positions);
}

int cs_prepare_view_export(const cs_camera *cam, const cs_settings *set, const cs_params *params,
                           const void *workspace, size_t workspace_bytes, int64_t pair_capacity,
                           const cs_view_export *out, void *stream) {
  if (!params || !workspace || !out) return CS_ERR_ARG;
  cs_layout L;
  int rc = cs_workspace_layout(cam, set, params->n, params->k, pair_capacity, &L);
  if (rc) return rc;
  if (workspace_bytes < L.total_bytes) return CS_ERR_WORKSPACE;
  if (params->n > 0 && (!out->pixels || !out->point_depths || !out->normals || !out->offsets || !out->delta_s ||
                        !out->sigma_s || !out->opacity || !out->scale || !out->view_dir || !out->view_dist ||
                        !out->color || !params->points || !params->sh))
    return CS_ERR_ARG;
  return cs::launch_export_view(*cam, *set, *params, L, static_cast<const char *>(workspace), *out,
                                reinterpret_cast<cudaStream_t>(stream));
}

int cs_read_status(const void *workspace, void *stream) {
  if (!workspace) return CS_ERR_ARG;
  uint32_t c[cs::C_COUNT];
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (cudaMemcpyAsync(c, workspace, sizeof(c), cudaMemcpyDeviceToHost, s) != cudaSuccess) return CS_ERR_CUDA;
  if (cudaStreamSynchronize(s) != cudaSuccess) return CS_ERR_CUDA;
  if (c[cs::C_NONFINITE]) return CS_ERR_NONFINITE;
  if (c[cs::C_OVERFLOW]) return CS_ERR_WORKSPACE;
  return CS_OK;
}

int cs_forward_stages(const cs_camera *cam, const cs_settings *set, const cs_params *params, void *workspace,
                      size_t workspace_bytes, int64_t pair_capacity, const cs_frame *frame, int32_t first_stage,
                      int32_t last_stage, void *stream) {
  return cs_forward_ex(cam, set, params, workspace, workspace_bytes, pair_capacity, frame, 0, first_stage, last_stage,
                       stream);
}

int cs_forward(const cs_camera *cam, const cs_settings *set, const cs_params *params, void *workspace,
               size_t workspace_bytes, int64_t pair_capacity, const cs_frame *frame, void *stream) {
  return cs_forward_stages(cam, set, params, workspace, workspace_bytes, pair_capacity, frame, 0, 2, stream);
}

static int backward_impl(const cs_camera *cam, const cs_settings *set, const cs_params *params, void *workspace,
                         size_t workspace_bytes, int64_t pair_capacity, const float *d_image, const cs_grads *grads,
                         const cs_view_signal *sig, uint32_t flags, int32_t first_stage, int32_t last_stage,
                         void *stream) {
  if (!params || !grads || !workspace || !d_image) return CS_ERR_ARG;
  if (flags & ~(uint32_t)(CS_GRADS_OVERWRITE | CS_WORK_COUNTERS | CS_ACCUM_ZEROED)) return CS_ERR_ARG;
  if (sig && (!sig->sigma_signal || !sig->sigma_views || !sig->visible)) return CS_ERR_ARG;
  if (first_stage < 0 || last_stage > 1 || first_stage > last_stage) return CS_ERR_ARG;
  cs_layout L;
  int rc = cs_workspace_layout(cam, set, params->n, params->k, pair_capacity, &L);
  if (rc) return rc;
  if (workspace_bytes < L.total_bytes) return CS_ERR_WORKSPACE;
  if (params->n > 0 && (!grads->d_points || !grads->d_raw_delta || !grads->d_raw_sigma ||
                        !grads->d_raw_opacity || !grads->d_raw_mask || !grads->d_sh))
    return CS_ERR_ARG;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  char *ws = static_cast<char *>(workspace);
  if (first_stage == 0) {
    cudaMemsetAsync(ws + L.counters + sizeof(uint32_t) * cs::C_NONFINITE, 0, sizeof(uint32_t), s);
    if ((rc = cs::launch_backward_blend(*cam, *set, *params, L, ws, d_image, (flags & CS_WORK_COUNTERS) != 0,
                                        (flags & CS_ACCUM_ZEROED) == 0, s)))
      return rc;
  }
  if (last_stage == 1)
    return cs::launch_chain(*cam, *set, *params, L, ws, *grads, sig, (flags & CS_GRADS_OVERWRITE) != 0, s);
  return CS_OK;
}

int cs_zero_accumulators(const cs_camera *cam, const cs_settings *set, const cs_params *params, void *workspace,
                         size_t workspace_bytes, int64_t pair_capacity, void *stream) {
  if (!params || !workspace) return CS_ERR_ARG;
  cs_layout L;
  int rc = cs_workspace_layout(cam, set, params->n, params->k, pair_capacity, &L);
  if (rc) return rc;
  if (workspace_bytes < L.total_bytes) return CS_ERR_WORKSPACE;
  return cs::launch_zero_accumulators(*params, L, static_cast<char *>(workspace), reinterpret_cast<cudaStream_t>(stream));
}

int cs_backward_chain_range(const cs_camera *cam, const cs_settings *set, const cs_params *params, void *workspace,
                            size_t workspace_bytes, int64_t pair_capacity, const cs_grads *grads,
                            const cs_view_signal *signal, uint32_t flags, int64_t first, int64_t last, void *stream) {
  if (!params || !grads || !workspace) return CS_ERR_ARG;
  if (flags & ~(uint32_t)CS_GRADS_OVERWRITE) return CS_ERR_ARG;
  if (signal && (!signal->sigma_signal || !signal->sigma_views || !signal->visible)) return CS_ERR_ARG;
  if (first < 0 || last < first || last > params->n) return CS_ERR_ARG;
  cs_layout L;
  int rc = cs_workspace_layout(cam, set, params->n, params->k, pair_capacity, &L);
  if (rc) return rc;
  if (workspace_bytes < L.total_bytes) return CS_ERR_WORKSPACE;
  if (params->n > 0 && (!grads->d_points || !grads->d_raw_delta || !grads->d_raw_sigma || !grads->d_raw_opacity ||
                        !grads->d_raw_mask || !grads->d_sh))
    return CS_ERR_ARG;
  return cs::launch_chain(*cam, *set, *params, L, static_cast<char *>(workspace), *grads, signal,
                          (flags & CS_GRADS_OVERWRITE) != 0, reinterpret_cast<cudaStream_t>(stream), first, last);
}

int cs_backward_stages(const cs_camera *cam, const cs_settings *set, const cs_params *params, void *workspace,
                       size_t workspace_bytes, int64_t pair_capacity, const float *d_image, const cs_grads *grads,
                       int32_t first_stage, int32_t last_stage, void *stream) {
  return backward_impl(cam, set, params, workspace, workspace_bytes, pair_capacity, d_image, grads, nullptr, 0,
                       first_stage, last_stage, stream);
}

int cs_backward(const cs_camera *cam, const cs_settings *set, const cs_params *params, void *workspace,
                size_t workspace_bytes, int64_t pair_capacity, const float *d_image, const cs_grads *grads,
                void *stream) {
  return backward_impl(cam, set, params, workspace, workspace_bytes, pair_capacity, d_image, grads, nullptr, 0, 0, 1,
                       stream);
}

int cs_backward_signal(const cs_camera *cam, const cs_settings *set, const cs_params *params, void *workspace,
                       size_t workspace_bytes, int64_t pair_capacity, const float *d_image, const cs_grads *grads,
                       const cs_view_signal *signal, void *stream) {
  return backward_impl(cam, set, params, workspace, workspace_bytes, pair_capacity, d_image, grads, signal, 0, 0, 1,
                       stream);
}

int cs_backward_ex(const cs_camera *cam, const cs_settings *set, const cs_params *params, void *workspace,
                   size_t workspace_bytes, int64_t pair_capacity, const float *d_image, const cs_grads *grads,
                   const cs_view_signal *signal, uint32_t flags, int32_t first_stage, int32_t last_stage,
                   void *stream) {
  return backward_impl(cam, set, params, workspace, workspace_bytes, pair_capacity, d_image, grads, signal, flags,
                       first_stage, last_stage, stream);
}

int cs_image_loss_workspace(int32_t height, int32_t width, size_t *bytes) {
  if (!bytes || height < 11 || width < 11) return CS_ERR_ARG;   // losses.py:60-63
  *bytes = sizeof(float) * 9 * (size_t)(height - 10) * (size_t)(width - 10);
  return CS_OK;
}

int cs_image_loss(int32_t height, int32_t width, const float *rendered, const float *target, const float *raw_mask,
                  int64_t n, double lambda_dssim, double beta_mask, float *d_image, float *d_raw_mask,
                  double *stats, void *workspace, size_t workspace_bytes, void *stream) {
  size_t need = 0;
  int rc = cs_image_loss_workspace(height, width, &need);
  if (rc) return rc;
  if (!rendered || !target || !d_image || !stats || !workspace || n < 0 || (n > 0 && !raw_mask)) return CS_ERR_ARG;
  if (workspace_bytes < need) return CS_ERR_WORKSPACE;
  return cs::launch_image_loss(height, width, rendered, target, raw_mask, n, lambda_dssim, beta_mask, d_image,
                               d_raw_mask, stats, workspace, reinterpret_cast<cudaStream_t>(stream));
}

int cs_adam_step(int32_t count, const cs_adam_tensor *tensors, double beta1, double beta2, double eps, int32_t step,
                 double grad_scale, void *stream) {
  if (count < 0 || count > 8 || (count > 0 && !tensors) || step < 1) return CS_ERR_ARG;
  for (int k = 0; k < count; k++)
    if (tensors[k].numel < 0 || (tensors[k].numel > 0 && (!tensors[k].param || !tensors[k].grad ||
                                                          !tensors[k].m || !tensors[k].v)))
      return CS_ERR_ARG;
  return cs::launch_adam(count, tensors, beta1, beta2, eps, step, grad_scale, reinterpret_cast<cudaStream_t>(stream));
}

int cs_read_counters(const void *workspace, uint32_t *host_out4, void *stream) {
  if (!workspace || !host_out4) return CS_ERR_ARG;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (cudaMemcpyAsync(host_out4, workspace, 4 * sizeof(uint32_t), cudaMemcpyDeviceToHost, s) != cudaSuccess)
    return CS_ERR_CUDA;
  return cudaStreamSynchronize(s) == cudaSuccess ? CS_OK : CS_ERR_CUDA;
}

int cs_graham_scan_batch(int32_t m, int32_t npts, const int32_t *counts, const double *pts, int32_t *hull,
                         int32_t *hull_n, void *stream) {
  if (m < 0 || npts < 0 || npts > 32 || (m > 0 && (!pts || !hull || !hull_n))) return CS_ERR_ARG;
  return cs::launch_hull_batch(m, npts, counts, pts, hull, hull_n, reinterpret_cast<cudaStream_t>(stream));
}

static bool scene_out_ok(const cs_scene_out *o) {
  return o && o->points && o->raw_delta && o->raw_sigma && o->raw_opacity && o->raw_mask && o->sh;
}

int cs_checkpoint_unpack(int32_t precision, int64_t n, int32_t k, const void *rows, const cs_scene_out *out,
                         void *stream) {
  if ((precision != 16 && precision != 32) || n < 0 || k < 3 || k > 16) return CS_ERR_ARG;
  if (n > 0 && (!rows || !scene_out_ok(out))) return CS_ERR_ARG;
  return cs::launch_checkpoint_rows(false, precision, n, k, const_cast<void *>(rows), *out,
                                    reinterpret_cast<cudaStream_t>(stream));
}

int cs_checkpoint_pack(int32_t precision, int64_t n, int32_t k, const cs_scene_out *scene, void *rows,
                       void *stream) {
  if ((precision != 16 && precision != 32) || n < 0 || k < 3 || k > 16) return CS_ERR_ARG;
  if (n > 0 && (!rows || !scene_out_ok(scene))) return CS_ERR_ARG;
  return cs::launch_checkpoint_rows(true, precision, n, k, rows, *scene, reinterpret_cast<cudaStream_t>(stream));
}

static bool params_ok(const cs_params *p) {
  return p && p->n >= 0 && p->k >= 3 && p->k <= 16 &&
         (p->n == 0 || (p->points && p->raw_delta && p->raw_sigma && p->raw_opacity && p->raw_mask && p->sh));
}

int cs_density_flags(const cs_params *params, const float *signal, const cs_density_config *cfg, uint8_t *flags,
                     uint32_t *child_keep, int64_t *surv_count, int64_t *child_count, void *stream) {
  if (!params_ok(params) || !cfg) return CS_ERR_ARG;
  if (params->n > 0 && (!signal || !flags || !child_keep || !surv_count || !child_count)) return CS_ERR_ARG;
  return cs::launch_density_flags(*params, signal, *cfg, flags, child_keep, surv_count, child_count,
                                  reinterpret_cast<cudaStream_t>(stream));
}

int cs_density_scatter(const cs_params *params, const cs_density_config *cfg, const uint8_t *flags,
                       const uint32_t *child_keep, const int64_t *surv_pos, const int64_t *child_pos,
                       const int64_t *n_surv, const cs_scene_out *out, int64_t *index_map, void *stream) {
  if (!params_ok(params) || !cfg) return CS_ERR_ARG;
  if (params->n > 0 && (!flags || !child_keep || !surv_pos || !child_pos || !n_surv || !index_map ||
                        !scene_out_ok(out)))
    return CS_ERR_ARG;
  return cs::launch_density_scatter(*params, *cfg, flags, child_keep, surv_pos, child_pos, n_surv, *out, index_map,
                                    reinterpret_cast<cudaStream_t>(stream));
}

}  // extern "C"
