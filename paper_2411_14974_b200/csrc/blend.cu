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

constexpr int kBlendThreads = 256;  // 8 warps; warp w owns the 8x4 pixel block of tile_pixel()

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

struct Eval {
  float I, J, alpha, alpha_raw, phi2, m, s;
};

__device__ __forceinline__ bool in_box(uint32_t bx, uint32_t by, int px, int py) {
  return px >= (int)(bx & 0xffffu) && px < (int)(bx >> 16) && py >= (int)(by & 0xffffu) && py < (int)(by >> 16);
}

// Does the bbox of candidate id overlap the warp's 8x4 pixel block?
__device__ __forceinline__ uint2 load_bbox(const float *records, uint32_t id, int rf) {
  return __ldg(reinterpret_cast<const uint2 *>(records + (size_t)id * rf + R_BBX));
}
__device__ __forceinline__ bool box_overlaps(uint2 b, int rx0, int ry0) {
  return (int)(b.x & 0xffffu) < rx0 + 8 && (int)(b.x >> 16) > rx0 && (int)(b.y & 0xffffu) < ry0 + 4 &&
         (int)(b.y >> 16) > ry0;
}

// Candidate record held in registers (loaded with warp-broadcast 128-bit
// loads: every lane reads the same address, one request per load).
template <int MAXK>
struct RecRegs {
  float4 h0, h1, h2;            // ax ay sigma o | r g b depth | 1-o dls nl -
  float ln[3 * MAXK];           // A_j B_j C_j
  __device__ __forceinline__ void load(const float *records, uint32_t id) {
    const float4 *r = reinterpret_cast<const float4 *>(records + (size_t)id * Rec<MAXK>::kFloats);
    h0 = __ldg(r);
    h1 = __ldg(r + 1);
    h2 = __ldg(r + 2);
#pragma unroll
    for (int q = 0; q < 3 * MAXK / 4; q++) {
      const float4 v = __ldg(r + R_HEADER / 4 + q);
      ln[4 * q] = v.x; ln[4 * q + 1] = v.y; ln[4 * q + 2] = v.z; ln[4 * q + 3] = v.w;
    }
  }
  __device__ __forceinline__ void load_smem(const float4 *r) {
    h0 = r[0];
    h1 = r[1];
    h2 = r[2];
#pragma unroll
    for (int q = 0; q < 3 * MAXK / 4; q++) {
      const float4 v = r[R_HEADER / 4 + q];
      ln[4 * q] = v.x; ln[4 * q + 1] = v.y; ln[4 * q + 2] = v.z; ln[4 * q + 3] = v.w;
    }
  }
  __device__ __forceinline__ int nl() const { return __float_as_int(h2.z); }
};

constexpr int kBatch = 128;  // candidates staged per block iteration (4 ballots per warp)

// Stage the records of pair indices [start, start+nb) into shared memory
// (coalesced 16-byte gathers; consecutive threads read consecutive pieces of
// one record) and cull them against this warp's 8x4 pixel block: bit j of
// mask[q] is set iff candidate 32q+j's bbox overlaps the block.
template <int MAXK>
__device__ __forceinline__ void stage_and_cull(const float *records, const uint32_t *pair_ids, uint32_t start,
                                               int nb, float4 *s_rec, uint32_t *s_id, int rx0, int ry0,
                                               bool warp_live, uint32_t (&mask)[kBatch / 32]) {
  constexpr int Q = Rec<MAXK>::kFloats / 4;
  if (threadIdx.x < nb) s_id[threadIdx.x] = __ldg(pair_ids + start + threadIdx.x);
  __syncthreads();
  const float4 *src = reinterpret_cast<const float4 *>(records);
  for (int q = threadIdx.x; q < nb * Q; q += kBlendThreads) {
    const int r = q / Q, part = q - r * Q;
    s_rec[q] = __ldg(src + (size_t)s_id[r] * Q + part);
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int q = 0; q < kBatch / 32; q++) {
    const int c = 32 * q + lane;
    bool hit = false;
    if (warp_live && c < nb) {
      const float4 bb = s_rec[c * Q + R_BBX / 4];
      hit = box_overlaps(make_uint2(__float_as_uint(bb.x), __float_as_uint(bb.y)), rx0, ry0);
    }
    mask[q] = __ballot_sync(0xffffffffu, hit);
  }
}

// smooth field of a candidate at anchor-relative pixel (dx, dy):
// z2_j = A_j dx + B_j dy + C_j, phi2 = max z2 + log2 sum 2^(z2 - max),
// I = 1 / (1 + 2^(sigma_s phi2)), alpha = min(o I, ALPHA_MAX)
// (field.py:51-72, rasterize.py:147-153 in log2 units).
template <int MAXK>
__device__ __forceinline__ Eval eval_field(const RecRegs<MAXK> &r, float dx, float dy, float *z) {
  Eval e;
  const int nl = r.nl();
  float m = -INFINITY;
#pragma unroll
  for (int l = 0; l < MAXK; l++) {
    if (l < nl) {
      z[l] = fmaf(r.ln[3 * l], dx, fmaf(r.ln[3 * l + 1], dy, r.ln[3 * l + 2]));
      m = fmaxf(m, z[l]);
    }
  }
  float s = 0.f;
#pragma unroll
  for (int l = 0; l < MAXK; l++)
    if (l < nl) s += ex2(z[l] - m);
  const float phi2 = m + lg2(s);
  const float u = ex2(r.h0.z * phi2);
  e.I = rcp(1.f + u);
  // 1 - I without cancellation: u*I while I >= 1/2, else 1 - I (also covers
  // u so large that I flushes to zero)
  e.J = u > 1.f ? 1.f - e.I : u * e.I;
  e.alpha_raw = r.h0.w * e.I;
  e.alpha = fminf(e.alpha_raw, (float)kAlphaMaxD);
  e.phi2 = phi2;
  e.m = m;
  e.s = s;
  return e;
}

// Forward blend, one tile per block.  Batches of 128 candidates are staged in
// shared memory; each warp culls the batch with four ballots against its 8x4
// pixel block and evaluates only the overlapping candidates, per pixel, in
// list order.  A warp stops evaluating once its 32 pixels are done; the block
// leaves the tile when all are.
template <int MAXK>
__global__ void __launch_bounds__(kBlendThreads) forward_kernel(BlendArgs a) {
  constexpr int RF = Rec<MAXK>::kFloats;
  const int tile = blockIdx.x;
  const int tx = tile % a.tiles_x, ty = tile / a.tiles_x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int lx, ly;
  tile_pixel(threadIdx.x, lx, ly);
  const int px = tx * kTile + lx, py = ty * kTile + ly;
  const int rx0 = tx * kTile + ((warp & 1) << 3), ry0 = ty * kTile + ((warp >> 1) << 2);
  const bool inside = px < a.width && py < a.height;
  const uint2 range = a.ranges[tile];
  const float qx = px + 0.5f, qy = py + 0.5f;
  float T = 1.f, C0 = 0.f, C1 = 0.f, C2 = 0.f, Wsum = 0.f, D = 0.f;
  int cnt = 0, last = -1;
  unsigned n_eval = 0, n_lines = 0;
  bool done = !inside;
  const bool use_floor = a.floor > 0.f;
  float z[MAXK];
  RecRegs<MAXK> r;
  __shared__ float4 s_rec[kBatch * (RF / 4)];
  __shared__ uint32_t s_id[kBatch];
  __shared__ uint8_t s_vis[kBatch];
  for (uint32_t start = range.x; start < range.y; start += kBatch) {
    if (__syncthreads_count(!done) == 0) break;
    const int nb = (int)min((uint32_t)kBatch, range.y - start);
    if (threadIdx.x < kBatch) s_vis[threadIdx.x] = 0;
    uint32_t mask[kBatch / 32];
    stage_and_cull<MAXK>(a.records, a.pair_ids, start, nb, s_rec, s_id, rx0, ry0,
                         !__all_sync(0xffffffffu, done), mask);
    bool warp_done = false;
#pragma unroll
    for (int q = 0; q < kBatch / 32; q++) {
      uint32_t m = warp_done ? 0u : mask[q];
      while (m) {
        const int j = 32 * q + __ffs(m) - 1;
        m &= m - 1;
        r.load_smem(s_rec + j * (RF / 4));
        const uint2 bb = make_uint2(__float_as_uint(s_rec[j * (RF / 4) + R_BBX / 4].x),
                                    __float_as_uint(s_rec[j * (RF / 4) + R_BBX / 4].y));
        if (!done && in_box(bb.x, bb.y, px, py)) {
          const Eval e = eval_field<MAXK>(r, qx - r.h0.x, qy - r.h0.y, z);
          n_eval++;
          n_lines += r.nl();
          if (e.alpha >= a.cutoff) {
            const float w = T * e.alpha;
            C0 = fmaf(w, r.h1.x, C0);
            C1 = fmaf(w, r.h1.y, C1);
            C2 = fmaf(w, r.h1.z, C2);
            Wsum += w;
            D = fmaf(w, r.h1.w, D);
            T *= fmaxf(fmaf(r.h0.w, e.J, r.h2.x), 1e-6f);
            cnt++;
            last = (int)(start + j);
            s_vis[j] = 1;
            if (use_floor && T < a.floor) done = true;
          }
        }
        if (__all_sync(0xffffffffu, done)) {  // this warp is finished with the tile
          warp_done = true;
          m = 0;
        }
      }
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

// Backward blend (backward.py:110-205): the block walks the tile list back
// to front from the largest `last` of its pixels in staged batches; each warp
// culls a batch by ballot, reconstructs T_prev = T / (1 - alpha) per pixel
// and reduces the 32 screen-space gradient values of each candidate across
// the warp (transpose-reduce) into one vector of float atomics.
template <int MAXK>
__global__ void __launch_bounds__(kBlendThreads) backward_kernel(BlendArgs a) {
  constexpr int RF = Rec<MAXK>::kFloats;
  constexpr int AF = Acc<MAXK>::kFloats;
  constexpr int NG = (AF + 31) / 32;  // 32-value groups
  const int tile = blockIdx.x;
  const int tx = tile % a.tiles_x, ty = tile / a.tiles_x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int lx, ly;
  tile_pixel(threadIdx.x, lx, ly);
  const int px = tx * kTile + lx, py = ty * kTile + ly;
  const int rx0 = tx * kTile + ((warp & 1) << 3), ry0 = ty * kTile + ((warp >> 1) << 2);
  const bool inside = px < a.width && py < a.height;
  const uint2 range = a.ranges[tile];
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
  // nothing behind the last blended candidate of the block matters
  const int warp_last = __reduce_max_sync(0xffffffffu, last);
  __shared__ int s_wl[kBlendThreads / 32];
  if (lane == 0) s_wl[warp] = warp_last;
  __syncthreads();
  int block_last = s_wl[0];
#pragma unroll
  for (int w = 1; w < kBlendThreads / 32; w++) block_last = max(block_last, s_wl[w]);
  float z[MAXK];
  RecRegs<MAXK> r;
  __shared__ float4 s_rec[kBatch * (RF / 4)];
  __shared__ uint32_t s_id[kBatch];
  for (int64_t end = (int64_t)block_last + 1; end > (int64_t)range.x; end -= kBatch) {
    const uint32_t start = (uint32_t)max((int64_t)range.x, end - kBatch);
    const int nb = (int)(end - start);
    uint32_t mask[kBatch / 32];
    __syncthreads();  // previous batch fully consumed before restaging
    stage_and_cull<MAXK>(a.records, a.pair_ids, start, nb, s_rec, s_id, rx0, ry0,
                         warp_last >= (int)start, mask);
#pragma unroll
    for (int q = kBatch / 32 - 1; q >= 0; q--) {
      uint32_t m = mask[q];
      while (m) {
        const int jj = 31 - __clz(m);   // back to front
        m &= ~(1u << jj);
        const int j = 32 * q + jj;
        const int e_idx = (int)start + j;
        r.load_smem(s_rec + j * (RF / 4));
        const uint2 bb = make_uint2(__float_as_uint(s_rec[j * (RF / 4) + R_BBX / 4].x),
                                    __float_as_uint(s_rec[j * (RF / 4) + R_BBX / 4].y));
        bool contrib = e_idx <= last && in_box(bb.x, bb.y, px, py);
        float v[NG * 32];
#pragma unroll
        for (int f = 0; f < NG * 32; f++) v[f] = 0.f;
        if (contrib) {
          const float dx = qx - r.h0.x, dy = qy - r.h0.y;
          const Eval e = eval_field<MAXK>(r, dx, dy, z);
          n_eval++;
          n_lines += r.nl();
          contrib = e.alpha >= a.cutoff;
          if (contrib) {
            const float o = r.h0.w, sig = r.h0.z, dls = r.h2.y;
            const float om = fmaxf(fmaf(o, e.J, r.h2.x), 1e-6f);
            const float rom = 1.f / om;
            const float Tp = T * rom;
            const float w = Tp * e.alpha;
            const float c0 = r.h1.x, c1 = r.h1.y, c2 = r.h1.z;
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
            const int nl = r.nl();
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
    }
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
