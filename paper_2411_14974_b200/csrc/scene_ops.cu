// Scene-level operations on the SoA parameters:
//
//   checkpoint rows  sceneio.save/load_checkpoint (sceneio.py:251-320): the
//                    .3dcs payload is rows `points | raw_delta raw_sigma
//                    raw_opacity | sh | raw_mask` of float32 or float16;
//                    unpack_rows / pack_rows convert between it and the SoA
//                    tensors on the device (one thread per value, the host
//                    only moves the raw bytes).
//   densify/prune    density.densify_and_prune (density.py:54-105) with
//                    split_convex (density.py:19-43): per-convex decisions in
//                    float64 (the reference's arithmetic, so the discrete
//                    outcome matches), then an order-preserving scatter into
//                    the new arrays (survivors in index order, then the K
//                    children of every split parent).
#include <cuda_fp16.h>

#include "common.cuh"

namespace cs {

// ------------------------------------------------------------------ .3dcs rows
__device__ __forceinline__ int row_floats(int k) { return 3 * k + 3 + 3 * kShCoeffs + 1; }

template <typename T>
__device__ __forceinline__ float to_f(T v);
template <> __device__ __forceinline__ float to_f<float>(float v) { return v; }
template <> __device__ __forceinline__ float to_f<__half>(__half v) { return __half2float(v); }
template <typename T>
__device__ __forceinline__ T from_f(float v);
template <> __device__ __forceinline__ float from_f<float>(float v) { return v; }
template <> __device__ __forceinline__ __half from_f<__half>(float v) { return __float2half_rn(v); }

// element j of a row -> destination array and index (sceneio.py:262-268 layout)
__device__ __forceinline__ float *soa_slot(const cs_scene_out &o, int64_t i, int k, int j) {
  const int k3 = 3 * k;
  if (j < k3) return o.points + i * k3 + j;
  if (j == k3) return o.raw_delta + i;
  if (j == k3 + 1) return o.raw_sigma + i;
  if (j == k3 + 2) return o.raw_opacity + i;
  if (j < k3 + 3 + 3 * kShCoeffs) return o.sh + i * 3 * kShCoeffs + (j - k3 - 3);
  return o.raw_mask + i;
}

template <typename T>
__global__ void unpack_rows_kernel(const T *rows, int64_t n, int k, cs_scene_out o) {
  const int rf = row_floats(k);
  const int64_t total = n * rf;
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < total; g += (int64_t)gridDim.x * blockDim.x)
    *soa_slot(o, g / rf, k, (int)(g % rf)) = to_f<T>(rows[g]);
}

template <typename T>
__global__ void pack_rows_kernel(cs_scene_out o, int64_t n, int k, T *rows) {
  const int rf = row_floats(k);
  const int64_t total = n * rf;
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < total; g += (int64_t)gridDim.x * blockDim.x)
    rows[g] = from_f<T>(*soa_slot(o, g / rf, k, (int)(g % rf)));
}

int launch_checkpoint_rows(bool pack, int precision, int64_t n, int k, void *rows, const cs_scene_out &o,
                           cudaStream_t s) {
  if (n == 0) return CS_OK;
  const int64_t total = n * (3 * k + 3 + 3 * kShCoeffs + 1);
  const int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 32);
  if (precision == 32) {
    if (pack) pack_rows_kernel<float><<<blocks, 256, 0, s>>>(o, n, k, static_cast<float *>(rows));
    else unpack_rows_kernel<float><<<blocks, 256, 0, s>>>(static_cast<const float *>(rows), n, k, o);
  } else {
    if (pack) pack_rows_kernel<__half><<<blocks, 256, 0, s>>>(o, n, k, static_cast<__half *>(rows));
    else unpack_rows_kernel<__half><<<blocks, 256, 0, s>>>(static_cast<const __half *>(rows), n, k, o);
  }
  return cudaGetLastError() == cudaSuccess ? CS_OK : CS_ERR_CUDA;
}

// ------------------------------------------------------------------ densify / prune
constexpr double kMaskGateD = 0.01;   // rasterize.py:26 MASK_GATE

__device__ __forceinline__ double expit_d(double x) { return 1.0 / (1.0 + exp(-x)); }

// SmoothConvex.diameter (model.py:113-116): max pairwise distance,
// sqrt((dx*dx + dy*dy) + dz*dz) in float64.
template <int MAXK>
__device__ __forceinline__ double diameter(const double (&p)[MAXK][3], int k) {
  double best = 0.0;
  for (int a = 0; a < k; a++)
    for (int b = 0; b < k; b++) {
      const double dx = p[a][0] - p[b][0], dy = p[a][1] - p[b][1], dz = p[a][2] - p[b][2];
      const double d = sqrt((dx * dx + dy * dy) + dz * dz);
      best = d > best ? d : best;
    }
  return best;
}

// density.py:96-102: kept iff opacity >= prune_opacity, diameter <= limit, mask > MASK_GATE
__device__ __forceinline__ bool keep_row(double opacity, double diam, double mask, const cs_density_config &c) {
  return !(opacity < c.prune_opacity) && !(diam > c.size_limit) && !(mask <= kMaskGateD);
}

// split_convex (density.py:19-43) child c, in float64
template <int MAXK>
__device__ __forceinline__ void child_points(const double (&p)[MAXK][3], const double (&cen)[3], int k, int c,
                                             double scale, double (&q)[MAXK][3]) {
  for (int j = 0; j < k; j++)
    for (int d = 0; d < 3; d++) q[j][d] = p[c][d] + scale * (p[j][d] - cen[d]);
}

template <int MAXK>
__device__ __forceinline__ void load_convex(const cs_params &P, int64_t i, double (&p)[MAXK][3], double (&cen)[3]) {
  const int k = P.k;
  for (int j = 0; j < k; j++)
    for (int d = 0; d < 3; d++) p[j][d] = P.points[(i * k + j) * 3 + d];
  for (int d = 0; d < 3; d++) {   // points.mean(axis=0): rows summed in order
    double s = 0.0;
    for (int j = 0; j < k; j++) s += p[j][d];
    cen[d] = s / k;
  }
}

// flags[i]: bit0 = kept survivor, bit1 = split; child_keep[i]: kept children bits
template <int MAXK>
__global__ void density_flags_kernel(cs_params P, const float *signal, cs_density_config c, uint8_t *flags,
                                     uint32_t *child_keep, int64_t *surv_count, int64_t *child_count) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= P.n) return;
  const int k = P.k;
  double p[MAXK][3], cen[3];
  load_convex<MAXK>(P, i, p, cen);
  const double mask = expit_d((double)P.raw_mask[i]);
  const double opacity = expit_d((double)P.raw_opacity[i]);
  const bool split = c.allow_split && (double)signal[i] > c.sigma_threshold;   // density.py:81
  uint8_t f = split ? 2 : 0;
  uint32_t ck = 0;
  if (!split) {
    if (keep_row(opacity, diameter<MAXK>(p, k), mask, c)) f |= 1;
  } else {
    // children share delta, mask; sigma += log(boost); opacity = logit(o * factor)
    const double co = opacity * c.split_opacity_factor;
    const double craw = log(co / (1.0 - co));                    // scipy.special.logit
    const double copacity = expit_d(craw);
    double q[MAXK][3];
    for (int ch = 0; ch < k; ch++) {
      child_points<MAXK>(p, cen, k, ch, c.split_scale, q);
      if (keep_row(copacity, diameter<MAXK>(q, k), mask, c)) ck |= 1u << ch;
    }
  }
  flags[i] = f;
  child_keep[i] = ck;
  surv_count[i] = f & 1;
  child_count[i] = __popc(ck);
}

// surv_pos / child_pos: exclusive scans of surv_count / child_count;
// n_surv = kept survivors (children start there).
template <int MAXK>
__global__ void density_scatter_kernel(cs_params P, cs_density_config c, const uint8_t *flags,
                                       const uint32_t *child_keep, const int64_t *surv_pos,
                                       const int64_t *child_pos, const int64_t *n_surv, cs_scene_out o,
                                       int64_t *index_map) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= P.n) return;
  const int k = P.k;
  const uint8_t f = flags[i];
  if (f & 1) {   // survivor row, copied unchanged
    const int64_t r = surv_pos[i];
    for (int j = 0; j < 3 * k; j++) o.points[r * 3 * k + j] = P.points[i * 3 * k + j];
    o.raw_delta[r] = P.raw_delta[i];
    o.raw_sigma[r] = P.raw_sigma[i];
    o.raw_opacity[r] = P.raw_opacity[i];
    o.raw_mask[r] = P.raw_mask[i];
    for (int j = 0; j < 3 * kShCoeffs; j++) o.sh[r * 3 * kShCoeffs + j] = P.sh[i * 3 * kShCoeffs + j];
    index_map[r] = i;
  }
  const uint32_t ck = child_keep[i];
  if (!(f & 2) || ck == 0) return;
  double p[MAXK][3], cen[3];
  load_convex<MAXK>(P, i, p, cen);
  const double opacity = expit_d((double)P.raw_opacity[i]);
  const double co = opacity * c.split_opacity_factor;
  const float craw = (float)log(co / (1.0 - co));
  const float csig = (float)((double)P.raw_sigma[i] + log(c.split_sigma_boost));
  int64_t r = *n_surv + child_pos[i];
  double q[MAXK][3];
  for (int ch = 0; ch < k; ch++) {
    if (!((ck >> ch) & 1u)) continue;
    child_points<MAXK>(p, cen, k, ch, c.split_scale, q);
    for (int j = 0; j < k; j++)
      for (int d = 0; d < 3; d++) o.points[(r * k + j) * 3 + d] = (float)q[j][d];
    o.raw_delta[r] = P.raw_delta[i];
    o.raw_sigma[r] = csig;
    o.raw_opacity[r] = craw;
    o.raw_mask[r] = P.raw_mask[i];
    for (int j = 0; j < 3 * kShCoeffs; j++) o.sh[r * 3 * kShCoeffs + j] = P.sh[i * 3 * kShCoeffs + j];
    index_map[r] = -1;
    r++;
  }
}

int launch_density_flags(const cs_params &P, const float *signal, const cs_density_config &c, uint8_t *flags,
                         uint32_t *child_keep, int64_t *surv_count, int64_t *child_count, cudaStream_t s) {
  if (P.n == 0) return CS_OK;
  const int blocks = (int)((P.n + 127) / 128);
  if (P.k <= 8)
    density_flags_kernel<8><<<blocks, 128, 0, s>>>(P, signal, c, flags, child_keep, surv_count, child_count);
  else
    density_flags_kernel<16><<<blocks, 128, 0, s>>>(P, signal, c, flags, child_keep, surv_count, child_count);
  return cudaGetLastError() == cudaSuccess ? CS_OK : CS_ERR_CUDA;
}

int launch_density_scatter(const cs_params &P, const cs_density_config &c, const uint8_t *flags,
                           const uint32_t *child_keep, const int64_t *surv_pos, const int64_t *child_pos,
                           const int64_t *n_surv, const cs_scene_out &o, int64_t *index_map, cudaStream_t s) {
  if (P.n == 0) return CS_OK;
  const int blocks = (int)((P.n + 127) / 128);
  if (P.k <= 8)
    density_scatter_kernel<8><<<blocks, 128, 0, s>>>(P, c, flags, child_keep, surv_pos, child_pos, n_surv, o, index_map);
  else
    density_scatter_kernel<16><<<blocks, 128, 0, s>>>(P, c, flags, child_keep, surv_pos, child_pos, n_surv, o,
                                                      index_map);
  return cudaGetLastError() == cudaSuccess ? CS_OK : CS_ERR_CUDA;
}

}  // namespace cs
