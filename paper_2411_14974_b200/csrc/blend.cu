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

// ---------------------------------------------------------------------------
// Producer/consumer pipeline shared by both blend kernels.  Warp kConsumers
// (the producer) streams the tile's candidate records into a ring of kStages
// shared-memory stages of kStageCands records, one TMA bulk copy
// (cp.async.bulk) per 16-byte-aligned record row, completion counted on the
// stage's `full` mbarrier (expect_tx).  The 8 consumer warps (8x4 pixels each)
// take stages at their own pace and release them on the `empty` mbarrier:
// no block-wide barrier, a slow warp never stalls a fast one by more than the
// ring depth.  When every consumer is done (all pixels terminated) the
// producer stops streaming and releases the waiting consumers with `stop`.
constexpr int kConsumers = 8;
constexpr int kPipeThreads = 32 * (kConsumers + 1);
constexpr int kStages = 4;
constexpr int kStageCands = 32;

template <int MAXK>
struct PipeSmem {
  float4 rec[kStages][kStageCands][Rec<MAXK>::kFloats / 4];
  uint32_t id[kStages][kStageCands];
  uint64_t full[kStages];
  uint64_t empty[kStages];
  int ndone;
  int stop;
};

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Producer warp: batch b covers pair indices first(b) .. first(b)+count(b)-1.
template <int MAXK, typename Batch>
__device__ __forceinline__ void pipe_produce(PipeSmem<MAXK> &sm, const float *records, const uint32_t *pair_ids,
                                             int nbatch, Batch batch, bool allow_stop) {
  constexpr int RB = Rec<MAXK>::kFloats * 4;
  const int lane = threadIdx.x & 31;
  int issued = 0;
  bool stopped = false;
  for (int b = 0; b < nbatch; b++) {
    const int s = b % kStages, u = b / kStages;
    if (u > 0) mbar_wait(&sm.empty[s], (u - 1) & 1);
    if (allow_stop && *reinterpret_cast<volatile int *>(&sm.ndone) == kConsumers) {
      if (lane == 0) {
        *reinterpret_cast<volatile int *>(&sm.stop) = 1;
        mbar_arrive(&sm.full[s]);          // wake consumers waiting on batch b; they see stop
      }
      stopped = true;
      break;
    }
    uint32_t first, count;
    batch(b, first, count);
    uint32_t id = 0;
    if (lane < (int)count) {
      id = __ldg(pair_ids + first + lane);
      sm.id[s][lane] = id;
    }
    __syncwarp();
    if (lane == 0) mbar_expect_tx(&sm.full[s], count * RB);
    __syncwarp();
    if (lane < (int)count) tma_bulk_g2s(&sm.rec[s][lane][0], records + (size_t)id * Rec<MAXK>::kFloats, RB, &sm.full[s]);
    issued = b + 1;
  }
  // drain: no bulk copy may still target this CTA's shared memory at exit.
  // After a stop at batch `issued` the stop arrival completed the next phase
  // of stage issued % kStages, whose previous batch was already consumed
  // (the empty wait above), so that batch must not be waited on again (its
  // parity would now name a phase that has not completed).
  const int lo = stopped ? issued - kStages + 1 : issued - kStages;
  for (int b = max(0, lo); b < issued; b++) mbar_wait(&sm.full[b % kStages], (b / kStages) & 1);
}

template <int MAXK>
__device__ __forceinline__ void pipe_init(PipeSmem<MAXK> &sm) {
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; s++) {
      mbar_init(&sm.full[s], 1);
      mbar_init(&sm.empty[s], kConsumers);
    }
    sm.ndone = 0;
    sm.stop = 0;
    fence_mbar_init();
  }
  __syncthreads();
}

// Forward blend (rasterize.py:178-209), one 16x16 tile per block.
template <int MAXK>
__global__ void __launch_bounds__(kPipeThreads) forward_kernel(BlendArgs a) {
  constexpr int Q = Rec<MAXK>::kFloats / 4;
  __shared__ PipeSmem<MAXK> sm;
  const int tile = blockIdx.x;
  const int tx = tile % a.tiles_x, ty = tile / a.tiles_x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint2 range = a.ranges[tile];
  const int nbatch = (int)((range.y - range.x + kStageCands - 1) / kStageCands);
  pipe_init(sm);
  unsigned n_eval = 0, n_lines = 0, n_blend = 0;
  if (warp == kConsumers) {
    pipe_produce<MAXK>(sm, a.records, a.pair_ids, nbatch,
                       [&](int b, uint32_t &first, uint32_t &count) {
                         first = range.x + (uint32_t)b * kStageCands;
                         count = min((uint32_t)kStageCands, range.y - first);
                       }, true);
  } else {
    int lx, ly;
    tile_pixel(threadIdx.x, lx, ly);
    const int px = tx * kTile + lx, py = ty * kTile + ly;
    const int rx0 = tx * kTile + ((warp & 1) << 3), ry0 = ty * kTile + ((warp >> 1) << 2);
    const bool inside = px < a.width && py < a.height;
    const float qx = px + 0.5f, qy = py + 0.5f;
    float T = 1.f, C0 = 0.f, C1 = 0.f, C2 = 0.f, Wsum = 0.f, D = 0.f;
    int last = -1;
    bool done = !inside;
    bool warp_done = __all_sync(0xffffffffu, done);
    if (warp_done && lane == 0) atomicAdd(&sm.ndone, 1);
    const bool use_floor = a.floor > 0.f;
    float z[MAXK];
    RecRegs<MAXK> r;
    for (int b = 0; b < nbatch; b++) {
      const int s = b % kStages;
      mbar_wait(&sm.full[s], (b / kStages) & 1);
      if (*reinterpret_cast<volatile int *>(&sm.stop)) break;
      if (!warp_done) {
        const uint32_t first = range.x + (uint32_t)b * kStageCands;
        const int count = (int)min((uint32_t)kStageCands, range.y - first);
        bool hit = false;
        if (lane < count) {
          const float4 bb = sm.rec[s][lane][R_BBX / 4];
          hit = box_overlaps(make_uint2(__float_as_uint(bb.x), __float_as_uint(bb.y)), rx0, ry0);
        }
        uint32_t m = __ballot_sync(0xffffffffu, hit);
        while (m) {
          const int j = __ffs(m) - 1;
          m &= m - 1;
          r.load_smem(sm.rec[s][j]);
          const float4 bb = sm.rec[s][j][R_BBX / 4];
          bool blended = false;
          if (!done && in_box(__float_as_uint(bb.x), __float_as_uint(bb.y), px, py)) {
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
              n_blend++;
              last = (int)(first + j);
              blended = true;
              if (use_floor && T < a.floor) done = true;
            }
          }
          if (__any_sync(0xffffffffu, blended)) {
            if (lane == 0 && a.visible) a.visible[sm.id[s][j]] = 1;
            if (__all_sync(0xffffffffu, done)) {
              warp_done = true;
              if (lane == 0) atomicAdd(&sm.ndone, 1);
              break;
            }
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.empty[s]);
    }
    if (inside) {
      const size_t p = (size_t)py * a.width + px;
      const float v0 = fmaf(T, a.bg[0], C0), v1 = fmaf(T, a.bg[1], C1), v2 = fmaf(T, a.bg[2], C2);
      a.image[3 * p] = fminf(fmaxf(v0, 0.f), 1.f);
      a.image[3 * p + 1] = fminf(fmaxf(v1, 0.f), 1.f);
      a.image[3 * p + 2] = fminf(fmaxf(v2, 0.f), 1.f);
      a.final_T[p] = T;
      a.pixel_T[p] = T;
      a.weight_sum[p] = Wsum;
      a.count[p] = (int)n_blend;
      if (a.depth) a.depth[p] = D;
      a.pixel_last[p] = last;
      a.pixel_clamp[p] = (uint8_t)((v0 >= 0.f && v0 <= 1.f) | ((v1 >= 0.f && v1 <= 1.f) << 1) |
                                   ((v2 >= 0.f && v2 <= 1.f) << 2));
    }
  }
  block_add_u64(a.stats + S_FWD_EVALS, n_eval);
  block_add_u64(a.stats + S_FWD_LINES, n_lines);
  block_add_u64(a.stats + S_FWD_BLENDS, n_blend);
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

// Backward blend (backward.py:110-205): the producer streams the tile list
// back to front from the block's largest `last`; each consumer warp culls a
// stage by ballot, reconstructs T_prev = T / (1 - alpha) per pixel and
// reduces the 32 screen-space gradient values of each candidate across the
// warp (transpose-reduce) into one vector of float atomics.
template <int MAXK>
__global__ void __launch_bounds__(kPipeThreads, 3) backward_kernel(BlendArgs a) {
  constexpr int AF = Acc<MAXK>::kFloats;
  constexpr int NG = (AF + 31) / 32;  // 32-value groups
  __shared__ PipeSmem<MAXK> sm;
  __shared__ int s_last[kConsumers];
  const int tile = blockIdx.x;
  const int tx = tile % a.tiles_x, ty = tile / a.tiles_x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint2 range = a.ranges[tile];
  // consumer pixel state
  int lx = 0, ly = 0;
  if (warp < kConsumers) tile_pixel(threadIdx.x, lx, ly);
  const int px = tx * kTile + lx, py = ty * kTile + ly;
  const bool inside = warp < kConsumers && px < a.width && py < a.height;
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
  const int warp_last = __reduce_max_sync(0xffffffffu, last);
  if (warp < kConsumers && lane == 0) s_last[warp] = warp_last;
  pipe_init(sm);  // (its __syncthreads also publishes s_last)
  int block_last = s_last[0];
#pragma unroll
  for (int w = 1; w < kConsumers; w++) block_last = max(block_last, s_last[w]);
  // batches back to front over [range.x, block_last]
  const int64_t end = (int64_t)block_last + 1;
  const int nbatch = end > (int64_t)range.x ? (int)((end - range.x + kStageCands - 1) / kStageCands) : 0;
  auto batch = [&](int b, uint32_t &first, uint32_t &count) {
    const int64_t hi = end - (int64_t)b * kStageCands;
    const int64_t lo = max((int64_t)range.x, hi - kStageCands);
    first = (uint32_t)lo;
    count = (uint32_t)(hi - lo);
  };
  unsigned n_eval = 0, n_lines = 0;
  if (warp == kConsumers) {
    pipe_produce<MAXK>(sm, a.records, a.pair_ids, nbatch, batch, false);
  } else {
    const int rx0 = tx * kTile + ((warp & 1) << 3), ry0 = ty * kTile + ((warp >> 1) << 2);
    const float qx = px + 0.5f, qy = py + 0.5f;
    float z[MAXK];
    RecRegs<MAXK> r;
    for (int b = 0; b < nbatch; b++) {
      const int s = b % kStages;
      mbar_wait(&sm.full[s], (b / kStages) & 1);
      uint32_t first, count;
      batch(b, first, count);
      if ((int)first <= warp_last) {
        bool hit = false;
        if (lane < (int)count && (int)(first + lane) <= warp_last) {
          const float4 bb = sm.rec[s][lane][R_BBX / 4];
          hit = box_overlaps(make_uint2(__float_as_uint(bb.x), __float_as_uint(bb.y)), rx0, ry0);
        }
        uint32_t m = __ballot_sync(0xffffffffu, hit);
        while (m) {
          const int j = 31 - __clz(m);   // back to front
          m &= ~(1u << j);
          const int e_idx = (int)first + j;
          r.load_smem(sm.rec[s][j]);
          const float4 bb = sm.rec[s][j][R_BBX / 4];
          bool contrib = e_idx <= last && in_box(__float_as_uint(bb.x), __float_as_uint(bb.y), px, py);
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
            float *dst = a.accum + (size_t)sm.id[s][j] * AF;
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
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.empty[s]);
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
    forward_kernel<8><<<tiles, kPipeThreads, 0, s>>>(a);
  else
    forward_kernel<16><<<tiles, kPipeThreads, 0, s>>>(a);
  return cudaGetLastError() == cudaSuccess ? CS_OK : CS_ERR_CUDA;
}

int launch_backward_blend(const cs_camera &cam, const cs_settings &set, const cs_params &p,
                          const cs_layout &L, char *ws, const float *d_image, cudaStream_t s) {
  BlendArgs a = make_args(cam, set, L, ws);
  a.d_image = d_image;
  if (p.n > 0) cudaMemsetAsync(a.accum, 0, (size_t)p.n * L.acc_floats * sizeof(float), s);
  const int tiles = L.tiles_x * L.tiles_y;
  if (L.max_k == 8)
    backward_kernel<8><<<tiles, kPipeThreads, 0, s>>>(a);
  else
    backward_kernel<16><<<tiles, kPipeThreads, 0, s>>>(a);
  return cudaGetLastError() == cudaSuccess ? CS_OK : CS_ERR_CUDA;
}

}  // namespace cs
