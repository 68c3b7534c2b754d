// K3 forward blend and K4a backward blend over 16x16 tiles.
//
// Forward (rasterize.py:178-209, field.py:51-72, rasterize.py:147-153): one
// thread per pixel, candidates staged in shared memory in batches; per
// candidate whose bbox holds the pixel:
//   z_j = delta_s L_j, phi = LSE(z), I = sigmoid(-sigma_s phi),
//   alpha = min(o I, ALPHA_MAX); blend iff (T >= floor if floor > 0) and
//   alpha >= cutoff: C += T alpha c, W += T alpha, T *= 1 - alpha, count++.
// Evaluated in base 2: z2 = log2(e) z, phi2 = max z2 + log2 sum 2^(z2-max),
// I = 1 / (1 + 2^(sigma_s phi2)); 1 - alpha = (1-o) + o (1-I) avoids the
// fp32 cancellation near ALPHA_MAX.  Pixels whose T fell below the floor
// stop; the block leaves a tile when all its pixels stopped.
//
// Backward (backward.py:110-205): walks each tile back to front from every
// pixel's last blended candidate, reconstructs T_prev = T/(1-alpha) and the
// colour behind, and produces per-candidate screen-space gradients
// (d_colour, d_opacity_eff, d_sigma_s, d_delta_s, and per hull line
// sum dL*(q-a), sum dL).  The warp reduces those 32 values with a
// transpose-reduce (31 shuffles, lane L ends with value L) and issues a single
// vector of global float atomics.
#include "common.cuh"

namespace cs {

constexpr int kBlendThreads = 256;
constexpr int kBatch = 128;

struct BlendArgs {
  const float *records;
  const uint32_t *pair_ids;
  const uint2 *ranges;
  int width, height, tiles_x;
  float cutoff, floor;
  float bg[3];
  // forward outputs
  float *image, *final_T, *weight_sum, *depth;
  int32_t *count;
  uint8_t *visible;
  int32_t *pixel_last;
  float *pixel_T;
  uint8_t *pixel_clamp;
  // backward
  const float *d_image;
  float *accum;
  unsigned long long *stats;
};

template <int MAXK>
__device__ __forceinline__ void stage_batch(const BlendArgs &a, uint32_t start, int nb, float4 *s_rec,
                                            uint32_t *s_id) {
  constexpr int Q = Rec<MAXK>::kFloats / 4;
  if (threadIdx.x < nb) s_id[threadIdx.x] = a.pair_ids[start + threadIdx.x];
  __syncthreads();
  const float4 *src = reinterpret_cast<const float4 *>(a.records);
  for (int q = threadIdx.x; q < nb * Q; q += kBlendThreads) {
    int r = q / Q, part = q - r * Q;
    s_rec[q] = __ldg(src + (size_t)s_id[r] * Q + part);
  }
  __syncthreads();
}

struct Eval {
  float I, J, alpha, alpha_raw, phi2, m, s;
};

// field value of record `rec` at anchor-relative pixel (dx, dy); keeps the
// per-line z2 in z[] for the backward.
template <int MAXK>
__device__ __forceinline__ Eval eval_field(const float *rec, int nl, float dx, float dy, float *z) {
  Eval e;
  float m = -INFINITY;
#pragma unroll
  for (int l = 0; l < MAXK; l++) {
    if (l < nl) {
      z[l] = fmaf(rec[R_HEADER + 3 * l], dx, fmaf(rec[R_HEADER + 3 * l + 1], dy, rec[R_HEADER + 3 * l + 2]));
      m = fmaxf(m, z[l]);
    }
  }
  float s = 0.f;
#pragma unroll
  for (int l = 0; l < MAXK; l++)
    if (l < nl) s += ex2(z[l] - m);
  const float phi2 = m + lg2(s);
  const float u = ex2(rec[R_SIGMA] * phi2);
  e.I = rcp(1.f + u);
  // 1 - I without cancellation: u*I while I >= 1/2, else 1 - I (also covers
  // u so large that I flushes to zero)
  e.J = u > 1.f ? 1.f - e.I : u * e.I;
  e.alpha_raw = rec[R_OPACITY] * e.I;
  e.alpha = fminf(e.alpha_raw, (float)kAlphaMaxD);
  e.phi2 = phi2;
  e.m = m;
  e.s = s;
  return e;
}

__device__ __forceinline__ bool in_bbox(const float *rec, int px, int py) {
  uint32_t bx = __float_as_uint(rec[R_BBX]), by = __float_as_uint(rec[R_BBY]);
  return px >= (int)(bx & 0xffffu) && px < (int)(bx >> 16) && py >= (int)(by & 0xffffu) && py < (int)(by >> 16);
}

template <int MAXK>
__global__ void __launch_bounds__(kBlendThreads) forward_kernel(BlendArgs a) {
  constexpr int Q = Rec<MAXK>::kFloats / 4;
  constexpr int RF = Rec<MAXK>::kFloats;
  __shared__ float4 s_rec[kBatch * Q];
  __shared__ uint32_t s_id[kBatch];
  __shared__ int s_vis[kBatch];
  const int tile = blockIdx.x;
  const int tx = tile % a.tiles_x, ty = tile / a.tiles_x;
  int lx, ly;
  tile_pixel(threadIdx.x, lx, ly);
  const int px = tx * kTile + lx, py = ty * kTile + ly;
  const bool inside = px < a.width && py < a.height;
  const uint2 range = a.ranges[tile];
  const float qx = px + 0.5f, qy = py + 0.5f;
  float T = 1.f, C0 = 0.f, C1 = 0.f, C2 = 0.f, Wsum = 0.f, D = 0.f;
  int cnt = 0, last = -1;
  unsigned n_eval = 0, n_lines = 0;
  bool done = !inside;
  const bool use_floor = a.floor > 0.f;
  float z[MAXK];
  for (uint32_t start = range.x; start < range.y; start += kBatch) {
    if (__syncthreads_count(!done) == 0) break;
    const int nb = min((uint32_t)kBatch, range.y - start);
    if (threadIdx.x < kBatch) s_vis[threadIdx.x] = 0;
    stage_batch<MAXK>(a, start, nb, s_rec, s_id);
    for (int j = 0; j < nb && !done; j++) {
      const float *rec = reinterpret_cast<const float *>(s_rec) + j * RF;
      if (!in_bbox(rec, px, py)) continue;
      const int nl = __float_as_int(rec[R_NLINES]);
      const Eval e = eval_field<MAXK>(rec, nl, qx - rec[R_AX], qy - rec[R_AY], z);
      n_eval++;
      n_lines += nl;
      if (!(e.alpha >= a.cutoff)) continue;
      const float w = T * e.alpha;
      C0 = fmaf(w, rec[R_R], C0);
      C1 = fmaf(w, rec[R_G], C1);
      C2 = fmaf(w, rec[R_B], C2);
      Wsum += w;
      D = fmaf(w, rec[R_DEPTH], D);
      T *= fmaxf(fmaf(rec[R_OPACITY], e.J, rec[R_ONE_MINUS_O]), 1e-6f);
      cnt++;
      last = (int)(start + j);
      s_vis[j] = 1;
      if (use_floor && T < a.floor) done = true;
    }
    __syncthreads();
    if (a.visible && threadIdx.x < nb && s_vis[threadIdx.x]) a.visible[s_id[threadIdx.x]] = 1;
  }
  block_add_u64(a.stats + S_FWD_EVALS, n_eval);
  block_add_u64(a.stats + S_FWD_LINES, n_lines);
  block_add_u64(a.stats + S_FWD_BLENDS, (unsigned)cnt);
  if (!inside) return;
  const size_t p = (size_t)py * a.width + px;
  const float v0 = fmaf(T, a.bg[0], C0), v1 = fmaf(T, a.bg[1], C1), v2 = fmaf(T, a.bg[2], C2);
  a.image[3 * p] = fminf(fmaxf(v0, 0.f), 1.f);
  a.image[3 * p + 1] = fminf(fmaxf(v1, 0.f), 1.f);
  a.image[3 * p + 2] = fminf(fmaxf(v2, 0.f), 1.f);
  a.final_T[p] = T;
  a.pixel_T[p] = T;
  a.weight_sum[p] = Wsum;
  a.count[p] = cnt;
  if (a.depth) a.depth[p] = D;
  a.pixel_last[p] = last;
  a.pixel_clamp[p] = (uint8_t)((v0 >= 0.f && v0 <= 1.f) | ((v1 >= 0.f && v1 <= 1.f) << 1) |
                               ((v2 >= 0.f && v2 <= 1.f) << 2));
}

// 32 per-lane values -> lane L holds the warp sum of value L.
__device__ __forceinline__ float transpose_reduce32(float (&v)[32]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int k = 16; k >= 1; k >>= 1) {
    const bool upper = lane & k;
#pragma unroll
    for (int i = 0; i < k; i++) {
      float send = upper ? v[i] : v[i + k];
      float keep = upper ? v[i + k] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, k);
    }
  }
  return v[0];
}

template <int MAXK>
__global__ void __launch_bounds__(kBlendThreads) backward_kernel(BlendArgs a) {
  constexpr int Q = Rec<MAXK>::kFloats / 4;
  constexpr int RF = Rec<MAXK>::kFloats;
  constexpr int AF = Acc<MAXK>::kFloats;
  constexpr int NG = (AF + 31) / 32;  // 32-value groups
  __shared__ float4 s_rec[kBatch * Q];
  __shared__ uint32_t s_id[kBatch];
  const int tile = blockIdx.x;
  const int tx = tile % a.tiles_x, ty = tile / a.tiles_x;
  int lx, ly;
  tile_pixel(threadIdx.x, lx, ly);
  const int px = tx * kTile + lx, py = ty * kTile + ly;
  const bool inside = px < a.width && py < a.height;
  const uint2 range = a.ranges[tile];
  if (range.y <= range.x) return;
  const float qx = px + 0.5f, qy = py + 0.5f;
  unsigned n_eval = 0, n_lines = 0;
  float T = 1.f, g0 = 0.f, g1 = 0.f, g2 = 0.f, S0 = 0.f, S1 = 0.f, S2 = 0.f;
  int last = -1;
  if (inside) {
    const size_t p = (size_t)py * a.width + px;
    T = a.pixel_T[p];
    last = a.pixel_last[p];
    const uint32_t cm = a.pixel_clamp[p];
    g0 = (cm & 1) ? a.d_image[3 * p] : 0.f;
    g1 = (cm & 2) ? a.d_image[3 * p + 1] : 0.f;
    g2 = (cm & 4) ? a.d_image[3 * p + 2] : 0.f;
    S0 = T * a.bg[0];
    S1 = T * a.bg[1];
    S2 = T * a.bg[2];
  }
  const int lane = threadIdx.x & 31;
  float z[MAXK];
  for (int64_t end = range.y; end > (int64_t)range.x; end -= kBatch) {
    const uint32_t start = (uint32_t)max((int64_t)range.x, end - kBatch);
    if (__syncthreads_count(last >= (int)start) == 0) continue;
    const int nb = (int)(end - start);
    stage_batch<MAXK>(a, start, nb, s_rec, s_id);
    for (int j = nb - 1; j >= 0; j--) {
      const float *rec = reinterpret_cast<const float *>(s_rec) + j * RF;
      const int nl = __float_as_int(rec[R_NLINES]);
      bool contrib = (int)(start + j) <= last && in_bbox(rec, px, py);
      float v[NG * 32];
#pragma unroll
      for (int f = 0; f < NG * 32; f++) v[f] = 0.f;
      if (contrib) {
        const float dx = qx - rec[R_AX], dy = qy - rec[R_AY];
        const Eval e = eval_field<MAXK>(rec, nl, dx, dy, z);
        n_eval++;
        n_lines += nl;
        contrib = e.alpha >= a.cutoff;
        if (contrib) {
          const float o = rec[R_OPACITY], sig = rec[R_SIGMA], dls = rec[R_DLS];
          const float om = fmaxf(fmaf(o, e.J, rec[R_ONE_MINUS_O]), 1e-6f);
          const float rom = 1.f / om;
          const float Tp = T * rom;
          const float w = Tp * e.alpha;
          const float c0 = rec[R_R], c1 = rec[R_G], c2 = rec[R_B];
          v[A_DC] = g0 * w;
          v[A_DC + 1] = g1 * w;
          v[A_DC + 2] = g2 * w;
          float dA = g0 * (Tp * c0 - S0 * rom) + g1 * (Tp * c1 - S1 * rom) + g2 * (Tp * c2 - S2 * rom);
          if (!(e.alpha_raw < (float)kAlphaMaxD)) dA = 0.f;
          v[A_DOEFF] = dA * e.I;
          const float dI = dA * o;
          const float slope = e.I * e.J;
          const float dphi = -sig * slope * dI;         // d loss / d phi (natural units)
          v[A_DSIG] = -(e.phi2 * kLn2) * slope * dI;
          const float rs = 1.f / e.s;
          float wz = 0.f;
#pragma unroll
          for (int l = 0; l < MAXK; l++) {
            if (l < nl) {
              const float wl = ex2(z[l] - e.m) * rs;    // softmax_over_lines (field.py:62-67)
              wz = fmaf(wl, z[l], wz);
              const float dL = dphi * (dls * kLn2) * wl;  // dphi * delta_s * w_l
              v[A_LINES + 3 * l] = dL * dx;
              v[A_LINES + 3 * l + 1] = dL * dy;
              v[A_LINES + 3 * l + 2] = dL;
            }
          }
          v[A_DDEL] = dphi * wz / dls;                   // dphi * sum_l w_l L_l
          S0 = fmaf(w, c0, S0);
          S1 = fmaf(w, c1, S1);
          S2 = fmaf(w, c2, S2);
          T = Tp;
        }
      }
      if (__any_sync(0xffffffffu, contrib)) {
        float *dst = a.accum + (size_t)s_id[j] * AF;
#pragma unroll
        for (int gi = 0; gi < NG; gi++) {
          float (&vv)[32] = *reinterpret_cast<float (*)[32]>(v + 32 * gi);
          const float sum = transpose_reduce32(vv);
          const int f = gi * 32 + lane;
          if (f < AF && sum != 0.f) atomicAdd(dst + f, sum);
        }
      }
    }
    __syncthreads();
  }
  block_add_u64(a.stats + S_BWD_EVALS, n_eval);
  block_add_u64(a.stats + S_BWD_LINES, n_lines);
}

static BlendArgs make_args(const cs_camera &cam, const cs_settings &set, const cs_layout &L, char *ws) {
  BlendArgs a;
  a.records = reinterpret_cast<const float *>(ws + L.records);
  a.pair_ids = reinterpret_cast<const uint32_t *>(ws + L.pair_ids);
  a.ranges = reinterpret_cast<const uint2 *>(ws + L.tile_ranges);
  a.width = cam.width;
  a.height = cam.height;
  a.tiles_x = L.tiles_x;
  a.cutoff = (float)set.cutoff;
  a.floor = (float)set.floor;
  for (int c = 0; c < 3; c++) a.bg[c] = (float)set.background[c];
  a.pixel_last = reinterpret_cast<int32_t *>(ws + L.pixel_last);
  a.pixel_T = reinterpret_cast<float *>(ws + L.pixel_T);
  a.pixel_clamp = reinterpret_cast<uint8_t *>(ws + L.pixel_clamp);
  a.accum = reinterpret_cast<float *>(ws + L.grad_accum);
  a.stats = reinterpret_cast<unsigned long long *>(ws + L.counters + sizeof(uint32_t) * C_STATS);
  a.image = a.final_T = a.weight_sum = a.depth = nullptr;
  a.count = nullptr;
  a.visible = nullptr;
  a.d_image = nullptr;
  return a;
}

int launch_forward_blend(const cs_camera &cam, const cs_settings &set, const cs_params &p,
                         const cs_layout &L, char *ws, const cs_frame &f, cudaStream_t s) {
  BlendArgs a = make_args(cam, set, L, ws);
  a.image = f.image;
  a.final_T = f.final_T;
  a.weight_sum = f.weight_sum;
  a.depth = f.depth;
  a.count = f.count;
  a.visible = f.visible;
  if (f.visible && p.n > 0) cudaMemsetAsync(f.visible, 0, (size_t)p.n, s);
  const int tiles = L.tiles_x * L.tiles_y;
  if (L.max_k == 8)
    forward_kernel<8><<<tiles, kBlendThreads, 0, s>>>(a);
  else
    forward_kernel<16><<<tiles, kBlendThreads, 0, s>>>(a);
  return cudaGetLastError() == cudaSuccess ? CS_OK : CS_ERR_CUDA;
}

int launch_backward_blend(const cs_camera &cam, const cs_settings &set, const cs_params &p,
                          const cs_layout &L, char *ws, const float *d_image, cudaStream_t s) {
  BlendArgs a = make_args(cam, set, L, ws);
  a.d_image = d_image;
  if (p.n > 0) cudaMemsetAsync(a.accum, 0, (size_t)p.n * L.acc_floats * sizeof(float), s);
  const int tiles = L.tiles_x * L.tiles_y;
  if (L.max_k == 8)
    backward_kernel<8><<<tiles, kBlendThreads, 0, s>>>(a);
  else
    backward_kernel<16><<<tiles, kBlendThreads, 0, s>>>(a);
  return cudaGetLastError() == cudaSuccess ? CS_OK : CS_ERR_CUDA;
}

}  // namespace cs
