// K3 forward blend and K4a backward blend over 16x16 tiles.
//
// Forward (rasterize.py:178-209, field.py:51-72, rasterize.py:147-153): two
// pixels per thread (forward2_kernel; forward_kernel, one pixel per thread,
// with -DCS_FWD_PPL1), candidates staged in shared memory in batches; per
// candidate whose bbox holds the pixel:
//   z_j = delta_s L_j, phi = LSE(z), I = sigmoid(-sigma_s phi),
//   alpha = min(o I, ALPHA_MAX); blend iff (T >= floor if floor > 0) and
//   alpha >= cutoff: C += T alpha c, W += T alpha, T *= 1 - alpha, count++.
// Evaluated in base 2: z2 = log2(e) z, phi2 = log2 sum 2^z2,
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
//
// The hull line count of a candidate is uniform across the warp (every lane
// evaluates the same candidate), so the evaluation is dispatched to a
// specialisation per count (no per-line predicates).
#include <algorithm>

#include "common.cuh"


namespace cs {

#ifdef CS_WAIT_STATS
// diagnostics (tools/wait_stats.py): SM cycles of the forward / backward
// consumer warps [0]/[4] and of their waits on `full` [1]/[5]; producer
// cycles [2]/[6] and its waits on `empty` [3]/[7]
__device__ unsigned long long g_wait_stats[12];   // [8]: forward consumers' wait on batch 0
#define WS_T0(v) const long long v = clock64()
#define WS_ADD(i, t0) atomicAdd(&g_wait_stats[i], (unsigned long long)(clock64() - (t0)))
#else
#define WS_T0(v)
#define WS_ADD(i, t0)
#endif

struct BlendArgs {
  const float *records;
  const double *lines;
  const uint32_t *pair_ids;
  const uint2 *ranges;
  const uint32_t *tile_order;   // heaviest tiles first (null: index order)
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
  AccT *accum;
  unsigned long long *stats;
  // blend masks: word (range.x / 32 + tile + b) of array q = which of the
  // 32 candidates of forward batch b some pixel of the tile's 8x4 block q
  // blended (8 arrays of mask_words words in the scratch); the backward
  // skips the others
  uint32_t *blend_mask;
  uint32_t mask_words;
  int ahead;   // forward: blocks resident at once (the block `ahead` after this one starts about when it ends)
  // decision record (forward, REC instantiation only): pixel p's blended
  // pair indices, in blend order, at rec_pos[rec_off[p] ...]
  const int64_t *rec_off;
  int32_t *rec_pos;
};

struct Eval {
  float I, J, alpha, alpha_raw, phi2;
};

// Warp block [rx0, rx0+8) x [ry0, ry0+4) vs a candidate's half-open bbox.
__device__ __forceinline__ bool box_overlaps(int4 b, int rx0, int ry0) {
  return b.x < rx0 + 8 && b.y > rx0 && b.z < ry0 + 4 && b.w > ry0;
}
__device__ __forceinline__ bool in_box(int4 b, int px, int py) {
  return px >= b.x && px < b.y && py >= b.z && py < b.w;
}
// Pixels of the warp's 8x4 block (bit = 8 * row + column, the lane order of
// tile_pixel) inside a candidate's half-open bbox.
__device__ __forceinline__ uint32_t block_mask(int4 b, int rx0, int ry0) {
  const int c0 = max(b.x - rx0, 0), c1 = min(b.y - rx0, 8);
  const int r0 = max(b.z - ry0, 0), r1 = min(b.w - ry0, 4);
  if (c1 <= c0 || r1 <= r0) return 0u;
  const uint32_t cols = (1u << c1) - (1u << c0);                                  // < 256
  const uint32_t rows = (0x01010101u >> (8 * (4 - (r1 - r0)))) << (8 * r0);         // 0x01 per row byte
  return cols * rows;
}
__device__ __forceinline__ int4 rec_bbox(const float4 *rec) {
  const float4 v = rec[R_BBOX / 4];
  return make_int4(__float_as_int(v.x), __float_as_int(v.y), __float_as_int(v.z), __float_as_int(v.w));
}

// Line coefficients of a candidate record in shared memory.  NL > 0: the
// warp-uniform line count is a compile-time constant (the hot path, one
// instantiation per count); NL == 0: runtime count nl <= MAXK (fallback).
template <int NL, int MAXK, bool Z64 = false>
struct LineSet {
  static constexpr int kN = NL > 0 ? NL : MAXK;
  static constexpr bool kPrecise = false;
  float c[3 * kN];
  int nl;
  // stage record planes A[MAXK] | B[MAXK] | C'[MAXK] after the header
  __device__ __forceinline__ void load(const float4 *rec, int nl_rt) {
    nl = NL > 0 ? NL : nl_rt;
#pragma unroll
    for (int p = 0; p < 3; p++)
#pragma unroll
      for (int q = 0; q < (kN + 3) / 4; q++) {
        const float4 v = rec[(R_HEADER + p * MAXK) / 4 + q];
        const float e[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int r = 0; r < 4; r++)
          if (4 * q + r < kN) c[3 * (4 * q + r) + p] = e[r];
      }
  }
  __device__ __forceinline__ bool has(int l) const { return NL > 0 ? true : l < nl; }
  // z_l at (dx, dy) relative to the tile's re-basing point
  __device__ __forceinline__ float z(int l, float dx, float dy) const {
    return fmaf(c[3 * l], dx, fmaf(c[3 * l + 1], dy, c[3 * l + 2]));
  }
};
// Float64 planes (StageRec<MAXK, true>): z formed in float64 from the staged
// coefficients (read from shared memory at each use, so no float64 registers
// stay live) and rounded once.  The float32 fma chain loses ~2^-24 of its
// largest intermediate, |C' + B dy|, which steep lines (the NONE and
// DEPTH_SQUARED scalings of the bench scenes) make large against z.
template <int NL, int MAXK>
struct LineSet<NL, MAXK, true> {
  static constexpr int kN = NL > 0 ? NL : MAXK;
  static constexpr bool kPrecise = true;
  const double *p;   // A[MAXK] | B[MAXK] | C'[MAXK]
  int nl;
  __device__ __forceinline__ void load(const float4 *rec, int nl_rt) {
    nl = NL > 0 ? NL : nl_rt;
    p = reinterpret_cast<const double *>(rec + R_HEADER / 4);
  }
  __device__ __forceinline__ bool has(int l) const { return NL > 0 ? true : l < nl; }
  __device__ __forceinline__ float z(int l, float dx, float dy) const {
    return (float)fma(p[l], (double)dx, fma(p[MAXK + l], (double)dy, p[2 * MAXK + l]));
  }
};

// Smooth field of a candidate at pixel (dx, dy) relative to the tile's
// re-basing point, in log2 units (field.py:51-72, rasterize.py:147-153):
//   z_l = A_l dx + B_l dy + C_l, phi2 = log2 sum 2^z_l,
//   I = 1 / (1 + 2^(sigma_s phi2)), alpha = min(o I, ALPHA_MAX).
// The sum is formed without the max shift (4 instructions per line); when it
// leaves [2^-100, 2^100] (denormal flush / overflow would bias phi) it is
// recomputed with the shift.  Softmax weights are w_l = 2^(z_l - phi2).
#ifdef CS_BWD_ACCURATE
__device__ __forceinline__ float acc_ex2(float x) { return exp2f(x); }
__device__ __forceinline__ float acc_lg2(float x) { return log2f(x); }
__device__ __forceinline__ float acc_rcp(float x) { return 1.f / x; }
#else
__device__ __forceinline__ float acc_ex2(float x) { return ex2(x); }
__device__ __forceinline__ float acc_lg2(float x) { return lg2(x); }
__device__ __forceinline__ float acc_rcp(float x) { return rcp(x); }
#endif
// P: correctly rounded exp2 / log2 / reciprocal (the float64-line kernels:
// their scalings put many more alphas next to the cutoff), else the
// approximations (ACC: the backward's acc_* choice)
template <bool P, bool ACC = false> __device__ __forceinline__ float fx2(float x) {
  return P ? exp2f(x) : (ACC ? acc_ex2(x) : ex2(x));
}
template <bool P, bool ACC = false> __device__ __forceinline__ float flg2(float x) {
  return P ? log2f(x) : (ACC ? acc_lg2(x) : lg2(x));
}
template <bool P, bool ACC = false> __device__ __forceinline__ float frcp(float x) {
  return P ? 1.f / x : (ACC ? acc_rcp(x) : rcp(x));
}

template <bool ACC = false, typename LS>
__device__ __forceinline__ Eval eval_field(const LS &L, float sig, float o, float dx, float dy, float (&z)[LS::kN]) {
  constexpr int N = LS::kN;
  float ex[N];
#pragma unroll
  for (int l = 0; l < N; l++) {
    if (L.has(l)) {
      z[l] = L.z(l, dx, dy);
      ex[l] = fx2<LS::kPrecise, ACC>(z[l]);
    } else {
      ex[l] = 0.f;
    }
  }
  // pairwise sum (log-depth dependency chain instead of N-1 serial adds)
#pragma unroll
  for (int w = 1; w < N; w *= 2)
#pragma unroll
    for (int l = 0; l + w < N; l += 2 * w) ex[l] += ex[l + w];
  const float s = ex[0];
  float phi2;
#ifdef CS_MAX_SHIFT
  if (false) {
#else
  if (s >= 0x1p-100f && s <= 0x1p100f) {
#endif
    phi2 = flg2<LS::kPrecise, ACC>(s);
  } else {
    float m = -INFINITY;
#pragma unroll
    for (int l = 0; l < N; l++)
      if (L.has(l)) m = fmaxf(m, z[l]);
    float s2 = 0.f;
#pragma unroll
    for (int l = 0; l < N; l++)
      if (L.has(l)) s2 += fx2<LS::kPrecise, ACC>(z[l] - m);
    phi2 = m + flg2<LS::kPrecise, ACC>(s2);
  }
  Eval e;
  const float u = fx2<LS::kPrecise, ACC>(sig * phi2);
  e.I = frcp<LS::kPrecise, ACC>(1.f + u);
  // 1 - I without cancellation: u*I while I >= 1/2, else 1 - I (also covers
  // u so large that I flushes to zero)
  e.J = u > 1.f ? 1.f - e.I : u * e.I;
  e.alpha_raw = o * e.I;
  e.alpha = fminf(e.alpha_raw, (float)kAlphaMaxD);
  e.phi2 = phi2;
  return e;
}

// ---------------------------------------------------------------------------
// Producer/consumer pipeline shared by both blend kernels.  Warp NC
// (the producer) streams the tile's candidate records into a ring of kStages
// shared-memory stages of kStageCands records, one TMA bulk copy
// (cp.async.bulk) per 16-byte-aligned record row, completion counted on the
// stage's `full` mbarrier (expect_tx).  The 8 consumer warps (8x4 pixels each)
// take stages at their own pace and release them on the `empty` mbarrier:
// no block-wide barrier, a slow warp never stalls a fast one by more than the
// ring depth.  When every consumer is done (all pixels terminated) the
// producer stops streaming and releases the waiting consumers with `stop`.
// Forward only: consumers OR the stage's candidates that blended somewhere
// into `vis`; the producer writes visible[] for them when it recycles the
// stage (rasterize.py:203 `visible[idx] = True`).
// Consumer warps per block: 8 cover a whole 16x16 tile; 4 cover half of it
// (two blocks per tile, each streaming the tile's list) -- smaller blocks
// finish sooner and leave fewer idle warps behind (measured per kernel).
#ifndef CS_FWD_NC
#define CS_FWD_NC 8
#endif
template <int NC> __host__ __device__ constexpr int pipe_threads() { return 32 * (NC + 1); }
// Ring depth: the forward stops early (saturated pixels), so a deep ring
// mostly prefetches records nobody evaluates; the backward walks the whole
// list up to each warp's last candidate and profits from more lookahead
// (measured per kernel: the counts below).
#ifndef CS_FWD_STAGES
#define CS_FWD_STAGES 3   // forward2: 3 / 4 / 5 / 6 stages 327 / 329 / 335 / 351 us
#endif
#ifndef CS_BWD_STAGES
#define CS_BWD_STAGES 5   // paired backward: 3 / 4 / 5 / 6 / 7 / 8 stages 620 / 672 / 622 / 632 / 650 / 736 us
#endif
constexpr int kStageCands = 32;
// longest back-off sleep of the producer waiting for a free stage
#ifndef CS_PROD_SLEEP_NS
#define CS_PROD_SLEEP_NS 512
#endif


template <int MAXK, int kStages, bool Z64 = false>
struct PipeSmem {
  static constexpr int kRing = kStages;
  float4 rec[kStages][kStageCands][StageRec<MAXK, Z64>::kFloats / 4];
  uint32_t id[kStages][kStageCands];
  uint8_t bmask[kStages][kStageCands];   // forward: 8x4 blocks that may reach the cutoff (bit = warp)
  uint32_t vis[kStages];
  uint64_t full[kStages];
  uint64_t empty[kStages];
  int ndone;
  int stop;
};

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

template <int MAXK, int kStages, bool Z64>
__device__ __forceinline__ void flush_visible(PipeSmem<MAXK, kStages, Z64> &sm, int s, uint8_t *visible) {
  const int lane = threadIdx.x & 31;
  const uint32_t vm = *reinterpret_cast<volatile uint32_t *>(&sm.vis[s]);
  if (visible && ((vm >> lane) & 1u)) visible[sm.id[s][lane]] = 1;
  __syncwarp();
  if (lane == 0) *reinterpret_cast<volatile uint32_t *>(&sm.vis[s]) = 0u;
  __syncwarp();
}

// Per-tile line staging by the producer warp (lane j = candidate j of the
// batch): every line of the candidate re-based onto the tile's re-basing
// point T (float64: C' = A (Tx - ax) + B (Ty - ay) + C, then rounded once),
// written to the stage's A / B / C' planes.
//
// Forward block culling (the producer is otherwise idle between stage
// fills): for the tile's 8x4 block q, the LSE is at least the largest line
// value, and each line's minimum over the block's pixel centres is at a
// corner, so phi2 >= max_l min_corner z_l.  When even that bound keeps o I
// below the cutoff at every pixel of the block -- sig * lb >
// log2(o / cutoff - 1), with a margin far above the float32 evaluation's
// error -- the block cannot blend the candidate and its warp skips it.
struct TileLines {
  double tx, ty;    // re-basing point (pixel coordinates)
  float cutoff;     // > 0: compute the forward cull mask
};
template <int MAXK, bool Z64 = false>
__device__ __forceinline__ uint32_t stage_lines(const float *rec_g, const double *lines_g, float4 *rec_s,
                                                const TileLines &tl) {
  const float4 h0 = __ldg(reinterpret_cast<const float4 *>(rec_g)), h2 = __ldg(reinterpret_cast<const float4 *>(rec_g) + 2);
  const int nl = min(__float_as_int(h2.z), MAXK);
  const double X = tl.tx - (double)h0.x, Y = tl.ty - (double)h0.y;
  float *As = reinterpret_cast<float *>(rec_s) + R_HEADER, *Bs = As + MAXK, *Cs = As + 2 * MAXK;
  const bool cull = tl.cutoff > 0.f;
  const float thr = cull ? __log2f(h0.w / tl.cutoff - 1.f) : 0.f;
  // block q's pixel-centre corners relative to T: x in {c0, c0 + 7}, y in {r0, r0 + 3}
  constexpr float d0 = 0.5f - (float)kRebase;
  float lb[8];
#pragma unroll
  for (int q = 0; q < 8; q++) lb[q] = -INFINITY;
  float mag = 0.f;   // largest |C'| + 8 |A| + 8 |B|: the float32 evaluation error of z is ~2^-23 of it
#pragma unroll
  for (int l = 0; l < MAXK; l++) {
    if (l < nl) {
      double A, B, C, pad;
      ld_global_nc_v4d(lines_g + 4 * l, A, B, C, pad);
      const double Cr = fma(A, X, fma(B, Y, C));   // re-based onto T
      const float Af = (float)A, Bf = (float)B, Cf = (float)Cr;
      if (Z64) {   // float64 planes A | B | C' (StageRec<MAXK, true>)
        double *D = reinterpret_cast<double *>(As);
        D[l] = A;
        D[MAXK + l] = B;
        D[2 * MAXK + l] = Cr;
      } else {
        As[l] = Af;
        Bs[l] = Bf;
        Cs[l] = Cf;
      }
      if (cull) {
        mag = fmaxf(mag, fabsf(Cf) + 8.f * (fabsf(Af) + fabsf(Bf)));
#pragma unroll
        for (int q = 0; q < 8; q++) {
          const float xl = d0 + (float)((q & 1) * 8), yl = d0 + (float)((q >> 1) * 4);
          const float zx = fminf(Af * xl, Af * (xl + 7.f)), zy = fminf(Bf * yl, Bf * (yl + 3.f));
          lb[q] = fmaxf(lb[q], Cf + zx + zy);
        }
      }
    }
  }
  uint32_t m = 0xffu;
  if (cull) {
#pragma unroll
    for (int q = 0; q < 8; q++) {
      const float v = h0.z * lb[q];
      if (v - thr > 1e-3f * (1.f + fabsf(thr) + fabsf(v)) + h0.z * mag * 0x1p-18f) m &= ~(1u << q);
    }
  }
  return m;
}

// Producer warp: batch b covers pair indices first(b) .. first(b)+count(b)-1.
// Per batch: the candidates' headers by coalesced cp.async gathers (4
// 16-byte chunks per record, 8 records per warp instruction; `full` counts
// their completion per lane), their lines re-based onto the tile by
// stage_lines (plain shared stores, then an explicit release arrive per lane
// on `full`, which therefore expects 64 arrivals).
struct NoLookAhead {
  __device__ __forceinline__ void operator()(int) const {}
};
template <int MAXK, int kStages, int NC, bool Z64, typename Batch, typename LookAhead = NoLookAhead>
__device__ __forceinline__ void pipe_produce(PipeSmem<MAXK, kStages, Z64> &sm, const float *records, const double *lines,
                                             const uint32_t *pair_ids, int nbatch, Batch batch, bool forward,
                                             uint8_t *visible, const TileLines &tl, bool cull,
                                             LookAhead look_ahead = LookAhead()) {
  constexpr int RG = Rec<MAXK>::kGlobal;
  const int lane = threadIdx.x & 31;
  WS_T0(tp);
  int issued = 0;
  bool stopped = false;
  // candidate ids are loaded one batch ahead (their latency hides behind the
  // wait for the next free stage)
  uint32_t next_id = 0;
  if (nbatch > 0) {
    uint32_t f0, c0;
    batch(0, f0, c0);
    if (lane < (int)c0) next_id = __ldg(pair_ids + f0 + lane);
  }
  // Forward consumers leave the pipeline when their pixels are done
  // (arrive_drop into the phases of the next kStages batches): once every
  // consumer has left, those drops can complete phases of batches this warp
  // never issues, and a stage's barrier may run two phases past the one
  // waited for -- its parity then reads "not complete" again.  So the
  // forward's waits on `empty` also end as soon as every consumer has left
  // (sm.ndone == NC): nothing reads the stages any more.
  auto wait_empty = [&](int y) -> bool {   // false: every consumer left
    uint64_t *bar = &sm.empty[y % kStages];
    const uint32_t par = (y / kStages) & 1;
    if (!forward) {
      if (CS_PROD_SLEEP_NS > 0) mbar_wait_backoff(bar, par, CS_PROD_SLEEP_NS);
      else mbar_wait(bar, par);
      return true;
    }
    const uint64_t t0 = globaltimer_ns();
    uint32_t ns = 32;
    for (int it = 0;; it++) {
      if (mbar_try_wait(bar, par)) return true;
      if (*reinterpret_cast<volatile int *>(&sm.ndone) == NC) return false;
      if (CS_PROD_SLEEP_NS > 0) {
        __nanosleep(ns);
        ns = min(2u * ns, (uint32_t)CS_PROD_SLEEP_NS);
      }
      if ((it & 63) == 63 && globaltimer_ns() - t0 > 2000000000ull) __trap();
    }
  };
  bool all_left = false;
  for (int b = 0; b < nbatch; b++) {
    const int s = b % kStages, u = b / kStages;
    if (u > 0) {
      // batch b - kStages released by every consumer
      WS_T0(tw);
      const bool ok = wait_empty(b - kStages);
      if (lane == 0) WS_ADD(forward ? 3 : 7, tw);
      if (!ok) {
        all_left = true;
        break;
      }
      if (forward) flush_visible(sm, s, visible);
    }
    if (forward && *reinterpret_cast<volatile int *>(&sm.ndone) == NC) {
      // every consumer left: stop streaming (stop = b + 1 releases any
      // consumer still waiting for batch b -- none with the drop-out)
      if (lane == 0) *reinterpret_cast<volatile int *>(&sm.stop) = b + 1;
      __syncwarp();
      mbar_arrive(&sm.full[s]);                  // all 32 lanes, twice: the barrier counts 64
      mbar_arrive(&sm.full[s]);
      stopped = true;
      break;
    }
    uint32_t first, count;
    batch(b, first, count);
    const uint32_t id = next_id;
    if (b + 1 < nbatch) {
      uint32_t f1, c1;
      batch(b + 1, f1, c1);
      next_id = lane < (int)c1 ? __ldg(pair_ids + f1 + lane) : 0u;
    }
    if (lane < (int)count) sm.id[s][lane] = id;
    {
      // coalesced header gather: each round copies 8 whole headers, one
      // 16-byte chunk per lane (cp.async.cg), so every header is read as
      // contiguous sectors; the lanes then arrive on `full` when their
      // copies land.
      constexpr int CPR = R_HEADER / 4, RPR = 32 / CPR;
      const int r_in = lane / CPR, c = lane % CPR;
      for (int r0 = 0; r0 < (int)count; r0 += RPR) {
        const int r = r0 + r_in;
        const uint32_t rid = __shfl_sync(0xffffffffu, id, min(r, 31));
        if (r < (int)count) {
          const float4 *src = reinterpret_cast<const float4 *>(records + (size_t)rid * RG) + c;
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(&sm.rec[s][r][c])), "l"(src)
                       : "memory");
        }
      }
      asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(&sm.full[s])) : "memory");
    }
    uint32_t bm = 0xffu;
    if (lane < (int)count)
      bm = stage_lines<MAXK, Z64>(records + (size_t)id * RG, lines + (size_t)id * Rec<MAXK>::kLines64, sm.rec[s][lane],
                             TileLines{tl.tx, tl.ty, cull ? tl.cutoff : 0.f});
    sm.bmask[s][lane] = (uint8_t)bm;
    mbar_arrive(&sm.full[s]);   // release: this lane's shared stores
    issued = b + 1;
    look_ahead(b);
  }
  // drain: wait until the consumers released the last issued batches (their
  // copies have landed, so nothing targets this CTA's shared memory after
  // exit) and publish their visibility.  After a stop, batch issued - kStages
  // was already waited on and flushed above.  Once every (forward) consumer
  // has left, the producer's own copies are waited for instead and every
  // stage's remaining visibility bits are published.
  const int lo = stopped ? issued - kStages + 1 : issued - kStages;
  for (int b = max(0, lo); b < issued && !all_left; b++) {
    if (!wait_empty(b)) {
      all_left = true;
      break;
    }
    if (forward) flush_visible(sm, b % kStages, visible);
  }
  if (all_left || stopped) {
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncwarp();
    if (forward)
      for (int st = 0; st < kStages; st++) flush_visible(sm, st, visible);
  }
  if (lane == 0) WS_ADD(forward ? 2 : 6, tp);
}

template <int MAXK, int kStages, int NC, bool Z64>
__device__ __forceinline__ void pipe_init(PipeSmem<MAXK, kStages, Z64> &sm) {
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; s++) {
      mbar_init(&sm.full[s], 64);   // per producer lane: its cp.async completion + its line stores
      mbar_init(&sm.empty[s], NC);
      sm.vis[s] = 0u;
    }
    sm.ndone = 0;
    sm.stop = 0;
    fence_mbar_init();
  }
  __syncthreads();
}

#define P_T_LT(t, thr) ((t) < (thr))
// Per-pixel forward state (rasterize.py:178-204).  A pixel is done when
// T < thr: thr = the transmittance floor (or 0 without one), and pixels
// outside the image start at T = -1 -- no separate flag.
struct FwdPixel {
  float T, C0, C1, C2, D;
  int last, nblend;
  __device__ __forceinline__ bool done(float thr) const { return P_T_LT(T, thr); }
};

// One candidate at one pixel: evaluate, and blend iff (T >= floor if floor >
// 0) and alpha >= cutoff (rasterize.py:194-204).  Returns whether it blended.
// (dqx, dqy): the pixel centre relative to the tile's re-basing point.
template <int NL, int MAXK, bool STATS, bool Z64 = false>
__device__ __forceinline__ bool fwd_candidate(const float4 *rec, float dqx, float dqy, float cutoff, float floor_,
                                              bool use_floor, int pos, FwdPixel &P, unsigned &n_lines) {
  const float4 h0 = rec[0], h2 = rec[2];
  LineSet<NL, MAXK, Z64> L;
  L.load(rec, __float_as_int(h2.z));
  float z[LineSet<NL, MAXK, Z64>::kN];
  const Eval e = eval_field<false>(L, h0.z, h0.w, dqx, dqy, z);
  if (STATS) n_lines += L.nl;
#ifdef CS_FWD_BRANCHY
  if (!(e.alpha >= cutoff)) return false;
  const float4 h1 = rec[1];
  const float w = P.T * e.alpha;
  P.C0 = fmaf(w, h1.x, P.C0);
  P.C1 = fmaf(w, h1.y, P.C1);
  P.C2 = fmaf(w, h1.z, P.C2);
  P.D = fmaf(w, h1.w, P.D);
  P.T *= fmaxf(fmaf(h0.w, e.J, h2.x), 1e-6f);   // 1 - alpha = (1-o) + o (1-I)
  P.nblend++;
  P.last = pos;
  return true;
#else
  // predicated (no divergent branch): a rejected candidate adds w = 0 and
  // multiplies T by 1, which leaves the state bit-identical
  const bool ok = e.alpha >= cutoff;
  const float4 h1 = rec[1];
  const float w = ok ? P.T * e.alpha : 0.f;
  P.C0 = fmaf(w, h1.x, P.C0);
  P.C1 = fmaf(w, h1.y, P.C1);
  P.C2 = fmaf(w, h1.z, P.C2);
  P.D = fmaf(w, h1.w, P.D);
  P.T *= ok ? fmaxf(fmaf(h0.w, e.J, h2.x), 1e-6f) : 1.f;   // 1 - alpha = (1-o) + o (1-I)
  P.nblend += ok ? 1 : 0;
  P.last = ok ? pos : P.last;
  return ok;
#endif
}

// Forward blend (rasterize.py:178-209), one 16x16 tile per block.  REC:
// also record every blend decision (diagnostics, cs_forward_record).
template <int MAXK, bool STATS, bool REC = false>
#ifndef CS_FWD_MINB
#define CS_FWD_MINB (CS_FWD_NC == 8 ? 4 : 7)
#endif
__global__ void __launch_bounds__(pipe_threads<CS_FWD_NC>(), CS_FWD_MINB) forward_kernel(BlendArgs a) {
  constexpr int kStages = CS_FWD_STAGES;
  constexpr int NC = CS_FWD_NC;
  const int half = NC == 8 ? 0 : (int)(blockIdx.x & 1);   // which half of the tile (NC == 4)
  const int unit = NC == 8 ? (int)blockIdx.x : (int)(blockIdx.x >> 1);
  extern __shared__ __align__(16) unsigned char pipe_dyn_smem[];
  PipeSmem<MAXK, kStages> &sm = *reinterpret_cast<PipeSmem<MAXK, kStages> *>(pipe_dyn_smem);
  const int tile = a.tile_order ? (int)a.tile_order[unit] : unit;
  const int tx = tile % a.tiles_x, ty = tile / a.tiles_x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint2 range = a.ranges[tile];
  const int nbatch = (int)((range.y - range.x + kStageCands - 1) / kStageCands);
  pipe_init<MAXK, kStages, NC>(sm);
  unsigned n_eval = 0, n_lines = 0, n_blend = 0, n_warp_evals = 0;
  if (warp == NC) {
#ifndef CS_NO_BLOCK_CULL
    // (a counting run evaluates every candidate: its work counts are the
    // algorithmic E_fwd of the roofline accounting)
    const bool cull = !STATS && NC == 8 && a.cutoff > 0.f;
#else
    const bool cull = false;
#endif
    const TileLines tl{(double)(tx * kTile + kRebase), (double)(ty * kTile + kRebase), a.cutoff};
    // A block's first batch waits for a chain of dependent loads (tile ->
    // range -> pair ids -> records): 12% of the consumers' cycles.  The
    // block `ahead` units later in launch order starts about when this one
    // ends, so this producer walks that chain for it, one step per issued
    // batch, and leaves its first candidates' records in L2.
    const int total = (int)gridDim.x;
    int f_tile = -1;
    uint2 f_range = make_uint2(0u, 0u);
    uint32_t f_id = 0u;
    auto look_ahead = [&](int step) {
      const int fu = unit + a.ahead;
      if (a.ahead <= 0 || fu >= total) return;
      const int lane = threadIdx.x & 31;
      if (step == 0) f_tile = a.tile_order ? (int)__ldg(a.tile_order + fu) : fu;
      else if (step == 1) f_range = __ldg(a.ranges + f_tile);
      else if (step == 2) f_id = f_range.x + lane < f_range.y ? __ldg(a.pair_ids + f_range.x + lane) : 0xffffffffu;
      else if (step == 3 && f_id != 0xffffffffu) {
        asm volatile("prefetch.global.L2 [%0];" ::"l"(a.records + (size_t)f_id * Rec<MAXK>::kGlobal) : "memory");
        asm volatile("prefetch.global.L2 [%0];" ::"l"(a.lines + (size_t)f_id * Rec<MAXK>::kLines64) : "memory");
        asm volatile("prefetch.global.L2 [%0];" ::"l"(a.lines + (size_t)f_id * Rec<MAXK>::kLines64 + 16) : "memory");
      }
    };
    pipe_produce<MAXK, kStages, NC>(sm, a.records, a.lines, a.pair_ids, nbatch,
                       [&](int b, uint32_t &first, uint32_t &count) {
                         first = range.x + (uint32_t)b * kStageCands;
                         count = min((uint32_t)kStageCands, range.y - first);
                       }, true, a.visible, tl, cull, look_ahead);
  } else {
    int lx, ly;
    tile_pixel(threadIdx.x, lx, ly);
    ly += half * 8;
    const int px = tx * kTile + lx, py = ty * kTile + ly;
    const int rx0 = tx * kTile + ((warp & 1) << 3), ry0 = ty * kTile + ((warp >> 1) << 2) + half * 8;
    bool inside = px < a.width && py < a.height;
    const float qx = (float)(lx - kRebase) + 0.5f, qy = (float)(ly - kRebase) + 0.5f;   // relative to T
    int32_t *rec_dst = nullptr;
    if (REC && inside) rec_dst = a.rec_pos + a.rec_off[(size_t)py * a.width + px];
    FwdPixel P;
    P.T = 1.f; P.C0 = P.C1 = P.C2 = P.D = 0.f;
    P.last = -1; P.nblend = 0;
    if (!inside) P.T = -1.f;
    const float thr = a.floor > 0.f ? a.floor : 0.f;   // rasterize.py:194: alive while T >= floor
    bool warp_done = __all_sync(0xffffffffu, P.done(thr));
    // A warp whose pixels all terminated leaves the pipeline for good
    // instead of waiting on every remaining stage: before arriving for
    // batch b it arrive_drops on the phases of batches b .. b + kStages - 1
    // (the phase of batch x is current once every consumer released batch
    // x - kStages; this warp's own arrival for that one is already in), so
    // the producer's later phases no longer expect it.
    auto leave = [&](int b) {
      if (lane == 0) {
        __threadfence_block();   // this warp's visibility bits before the count the producer reads
        atomicAdd(&sm.ndone, 1);
#pragma unroll 1
        for (int i = 0; i < kStages; i++) {
          const int x = b + i;
          if (i > 0 && x >= kStages) mbar_wait(&sm.empty[x % kStages], ((x - kStages) / kStages) & 1);
          mbar_arrive_drop(&sm.empty[x % kStages]);
        }
      }
      __syncwarp();
    };
    WS_T0(tc);
    if (warp_done) leave(0);
    const bool use_floor = a.floor > 0.f;
    for (int b = 0; b < nbatch && !warp_done; b++) {
      const int s = b % kStages;
      {
        WS_T0(tw);
        mbar_wait(&sm.full[s], (b / kStages) & 1);
        if (lane == 0) WS_ADD(1, tw);
        if (lane == 0 && b == 0) WS_ADD(8, tw);
      }
      if (*reinterpret_cast<volatile int *>(&sm.stop) == b + 1) break;
      {
        const uint32_t first = range.x + (uint32_t)b * kStageCands;
        const int count = (int)min((uint32_t)kStageCands, range.y - first);
        // lane j: pixels of this warp's block inside candidate j's bbox and alive
        const uint32_t alive = __ballot_sync(0xffffffffu, !P.done(thr));
#ifndef CS_NO_BLOCK_CULL
        const bool may = STATS || NC != 8 || !(a.cutoff > 0.f) || ((sm.bmask[s][lane] >> warp) & 1u);
#else
        const bool may = true;
#endif
        const uint32_t pm = lane < count && may ? block_mask(rec_bbox(sm.rec[s][lane]), rx0, ry0) & alive : 0u;
        uint32_t m = __ballot_sync(0xffffffffu, pm != 0u);
        uint32_t vis = 0;
        while (m) {
          const int j = __ffs(m) - 1;
          m &= m - 1;
          const float4 *rec = sm.rec[s][j];
          bool blended = false;
          const uint32_t pj = __shfl_sync(0xffffffffu, pm, j);
          const bool act = !P.done(thr) && ((pj >> lane) & 1u);
          if (!__any_sync(0xffffffffu, act)) continue;   // its pixels died earlier in this stage
          if (STATS) n_warp_evals++;
#ifdef CS_NO_EVAL
          if (false) {
#else
          if (act) {
#endif
            if (STATS) n_eval++;
            const int pos = (int)first + j;
            if (MAXK == 8) {
              const int nl = __float_as_int(rec[2].z);   // warp-uniform line count (an if chain: a switch became a jump table)
              if (nl == 5) blended = fwd_candidate<5, MAXK, STATS>(rec, qx, qy, a.cutoff, a.floor, use_floor, pos, P, n_lines);
              else if (nl == 6) blended = fwd_candidate<6, MAXK, STATS>(rec, qx, qy, a.cutoff, a.floor, use_floor, pos, P, n_lines);
              else if (nl == 4) blended = fwd_candidate<4, MAXK, STATS>(rec, qx, qy, a.cutoff, a.floor, use_floor, pos, P, n_lines);
              else blended = fwd_candidate<0, MAXK, STATS>(rec, qx, qy, a.cutoff, a.floor, use_floor, pos, P, n_lines);
            } else {
              blended = fwd_candidate<0, MAXK, STATS>(rec, qx, qy, a.cutoff, a.floor, use_floor, pos, P, n_lines);
            }
            if (REC && blended) rec_dst[P.nblend - 1] = pos;
          }
          if (__any_sync(0xffffffffu, blended)) {
            vis |= 1u << j;
            if (__all_sync(0xffffffffu, P.done(thr))) {
              warp_done = true;
              break;
            }
          }
        }
        if (lane == 0) {
          if (vis) atomicOr(&sm.vis[s], vis);
          // word (range.x / 32 + tile + b) of this block's mask: unique per
          // (tile, batch), written for every batch the warp processed
          a.blend_mask[(size_t)(warp + (NC == 8 ? 0 : 4 * half)) * a.mask_words + (range.x >> 5) + tile + b] = vis;
        }
      }
      __syncwarp();
      if (warp_done) {
        leave(b);
      } else if (lane == 0) {
        mbar_arrive(&sm.empty[s]);
      }
    }
    if (lane == 0) WS_ADD(0, tc);
    n_blend = (unsigned)P.nblend;
    inside = px < a.width && py < a.height;
    if (inside) {
      const size_t p = (size_t)py * a.width + px;
      const float v0 = fmaf(P.T, a.bg[0], P.C0), v1 = fmaf(P.T, a.bg[1], P.C1), v2 = fmaf(P.T, a.bg[2], P.C2);
      a.image[3 * p] = fminf(fmaxf(v0, 0.f), 1.f);
      a.image[3 * p + 1] = fminf(fmaxf(v1, 0.f), 1.f);
      a.image[3 * p + 2] = fminf(fmaxf(v2, 0.f), 1.f);
      a.final_T[p] = P.T;
      a.pixel_T[p] = P.T;
      // blend_weight_sum = sum T_prev alpha telescopes to 1 - T (rasterize.py:198-200;
      // the compositing identity of test_rasterize.py:108-116): no running sum
      a.weight_sum[p] = 1.f - P.T;
      a.count[p] = P.nblend;
      if (a.depth) a.depth[p] = P.D;
      a.pixel_last[p] = P.last;
      a.pixel_clamp[p] = (uint8_t)((v0 >= 0.f && v0 <= 1.f) | ((v1 >= 0.f && v1 <= 1.f) << 1) |
                                   ((v2 >= 0.f && v2 <= 1.f) << 2));
    }
  }
  if (STATS) {
    block_add_u64(a.stats + S_FWD_EVALS, n_eval);
    block_add_u64(a.stats + S_FWD_LINES, n_lines);
    block_add_u64(a.stats + S_FWD_BLENDS, n_blend);
    block_add_u64(a.stats + S_FWD_WARP_EVALS, lane == 0 ? n_warp_evals : 0u);
  }
}

// ---------------------------------------------------------------------------
// Forward blend, two pixels per lane (8x8 pixels per warp, 4 consumer warps
// per 16x16 tile).  Per candidate the warp-level work -- the loop step, the
// record address, the line-count dispatch, the line loads and the votes --
// is shared by two pixels (rows r and r + 4 of the lane's column), and the
// two evaluations are independent chains the scheduler interleaves.  Every
// pixel sees the same candidates in the same order with the same arithmetic
// as in forward_kernel, so the outputs are bit-identical; the blend masks are
// still per 8x4 block (a warp writes the words of its two blocks).
// ---------------------------------------------------------------------------

// 2^z summed over the lines at (dx, dy): eval_field's expression and order.
template <typename LS>
__device__ __forceinline__ float line_sum(const LS &L, float dx, float dy) {
  constexpr int N = LS::kN;
  float ex[N];
#pragma unroll
  for (int l = 0; l < N; l++)
    ex[l] = L.has(l) ? fx2<LS::kPrecise>(L.z(l, dx, dy)) : 0.f;
#pragma unroll
  for (int w = 1; w < N; w *= 2)
#pragma unroll
    for (int l = 0; l + w < N; l += 2 * w) ex[l] += ex[l + w];
  return ex[0];
}
__device__ __forceinline__ bool lse_in_range(float s) { return s >= 0x1p-100f && s <= 0x1p100f; }
// eval_field's max-shifted log-sum-exp (a sum outside [2^-100, 2^100]; rare):
// the lines are re-read from the stage
template <int NL, int MAXK, bool Z64>
__device__ __noinline__ float lse_shifted(const float4 *rec, float dx, float dy) {
  constexpr int N = LineSet<NL, MAXK, Z64>::kN;
  LineSet<NL, MAXK, Z64> L;
  L.load(rec, __float_as_int(rec[2].z));
  float z[N];
  float m = -INFINITY;
#pragma unroll
  for (int l = 0; l < N; l++)
    if (L.has(l)) {
      z[l] = L.z(l, dx, dy);
      m = fmaxf(m, z[l]);
    }
  float s2 = 0.f;
#pragma unroll
  for (int l = 0; l < N; l++)
    if (L.has(l)) s2 += fx2<Z64>(z[l] - m);
  return m + flg2<Z64>(s2);
}
template <bool P = false>
__device__ __forceinline__ Eval eval_finish(float phi2, float sig, float o) {
  Eval e;
  const float u = fx2<P>(sig * phi2);
  e.I = frcp<P>(1.f + u);
  e.J = u > 1.f ? 1.f - e.I : u * e.I;
  e.alpha_raw = o * e.I;
  e.alpha = fminf(e.alpha_raw, (float)kAlphaMaxD);
  e.phi2 = phi2;
  return e;
}
// the predicated blend update of fwd_candidate
__device__ __forceinline__ void blend_update(FwdPixel &P, const Eval &e, bool ok, float4 h0, float4 h1, float4 h2,
                                             int pos) {
  const float w = ok ? P.T * e.alpha : 0.f;
  P.C0 = fmaf(w, h1.x, P.C0);
  P.C1 = fmaf(w, h1.y, P.C1);
  P.C2 = fmaf(w, h1.z, P.C2);
  P.D = fmaf(w, h1.w, P.D);
  P.T *= ok ? fmaxf(fmaf(h0.w, e.J, h2.x), 1e-6f) : 1.f;
  P.nblend += ok ? 1 : 0;
  P.last = ok ? pos : P.last;
}
// One candidate at both pixels of the lane (act0 / act1: which of them to blend).
template <int NL, int MAXK, bool STATS, bool Z64 = false>
__device__ __forceinline__ void fwd_pair(const float4 *rec, float qx, float qy0, bool act0, bool act1, float cutoff,
                                         int pos, FwdPixel &P0, FwdPixel &P1, unsigned &n_lines, bool &bl0, bool &bl1) {
  const float4 h0 = rec[0], h2 = rec[2];
  float s0, s1;
  {
    LineSet<NL, MAXK, Z64> L;
    L.load(rec, __float_as_int(h2.z));
    s0 = line_sum(L, qx, qy0);
    s1 = line_sum(L, qx, qy0 + 4.f);
    if (STATS) n_lines += (unsigned)L.nl * ((act0 ? 1u : 0u) + (act1 ? 1u : 0u));
  }
  float phi0 = flg2<Z64>(s0), phi1 = flg2<Z64>(s1);
  if (!(lse_in_range(s0) && lse_in_range(s1))) {
    if (!lse_in_range(s0)) phi0 = lse_shifted<NL, MAXK, Z64>(rec, qx, qy0);
    if (!lse_in_range(s1)) phi1 = lse_shifted<NL, MAXK, Z64>(rec, qx, qy0 + 4.f);
  }
  const Eval e0 = eval_finish<Z64>(phi0, h0.z, h0.w), e1 = eval_finish<Z64>(phi1, h0.z, h0.w);
  const float4 h1 = rec[1];
  bl0 = act0 && e0.alpha >= cutoff;
  bl1 = act1 && e1.alpha >= cutoff;
  blend_update(P0, e0, bl0, h0, h1, h2, pos);
  blend_update(P1, e1, bl1, h0, h1, h2, pos);
}

#ifndef CS_FWD2_MINB
#define CS_FWD2_MINB 5
#endif
template <int MAXK, bool STATS, bool REC = false, bool Z64 = false>
__global__ void __launch_bounds__(pipe_threads<4>(), CS_FWD2_MINB) forward2_kernel(BlendArgs a) {
  constexpr int kStages = CS_FWD_STAGES;
  constexpr int NC = 4;
  extern __shared__ __align__(16) unsigned char pipe_dyn_smem[];
  PipeSmem<MAXK, kStages, Z64> &sm = *reinterpret_cast<PipeSmem<MAXK, kStages, Z64> *>(pipe_dyn_smem);
  const int unit = (int)blockIdx.x;
  const int tile = a.tile_order ? (int)a.tile_order[unit] : unit;
  const int tx = tile % a.tiles_x, ty = tile / a.tiles_x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint2 range = a.ranges[tile];
  const int nbatch = (int)((range.y - range.x + kStageCands - 1) / kStageCands);
  pipe_init<MAXK, kStages, NC>(sm);
  unsigned n_eval = 0, n_lines = 0, n_blend = 0, n_warp_evals = 0;
  if (warp == NC) {
#ifndef CS_NO_BLOCK_CULL
    const bool cull = !STATS && a.cutoff > 0.f;
#else
    const bool cull = false;
#endif
    const TileLines tl{(double)(tx * kTile + kRebase), (double)(ty * kTile + kRebase), a.cutoff};
    const int total = (int)gridDim.x;
    int f_tile = -1;
    uint2 f_range = make_uint2(0u, 0u);
    uint32_t f_id = 0u;
    auto look_ahead = [&](int step) {   // as in forward_kernel
      const int fu = unit + a.ahead;
      if (a.ahead <= 0 || fu >= total) return;
      const int lane = threadIdx.x & 31;
      if (step == 0) f_tile = a.tile_order ? (int)__ldg(a.tile_order + fu) : fu;
      else if (step == 1) f_range = __ldg(a.ranges + f_tile);
      else if (step == 2) f_id = f_range.x + lane < f_range.y ? __ldg(a.pair_ids + f_range.x + lane) : 0xffffffffu;
      else if (step == 3 && f_id != 0xffffffffu) {
        asm volatile("prefetch.global.L2 [%0];" ::"l"(a.records + (size_t)f_id * Rec<MAXK>::kGlobal) : "memory");
        asm volatile("prefetch.global.L2 [%0];" ::"l"(a.lines + (size_t)f_id * Rec<MAXK>::kLines64) : "memory");
        asm volatile("prefetch.global.L2 [%0];" ::"l"(a.lines + (size_t)f_id * Rec<MAXK>::kLines64 + 16) : "memory");
      }
    };
    pipe_produce<MAXK, kStages, NC>(sm, a.records, a.lines, a.pair_ids, nbatch,
                       [&](int b, uint32_t &first, uint32_t &count) {
                         first = range.x + (uint32_t)b * kStageCands;
                         count = min((uint32_t)kStageCands, range.y - first);
                       }, true, a.visible, tl, cull, look_ahead);
  } else {
    // warp: columns (warp & 1) * 8 + 0..7, rows (warp >> 1) * 8 + 0..7; lane:
    // column lane & 7, rows lane >> 3 and (lane >> 3) + 4 (pixel h = 0, 1,
    // in the 8x4 blocks q0 and q1 = q0 + 2)
    const int lx = ((warp & 1) << 3) | (lane & 7), ly0 = ((warp >> 1) << 3) | (lane >> 3);
    const int px = tx * kTile + lx, py0 = ty * kTile + ly0;
    const int rx0 = tx * kTile + ((warp & 1) << 3), ry0 = ty * kTile + ((warp >> 1) << 3);
    const int q0 = (warp & 1) | ((warp >> 1) << 2);
    const float qx = (float)(lx - kRebase) + 0.5f, qy0 = (float)(ly0 - kRebase) + 0.5f;
    FwdPixel P0, P1;
    P0.T = P1.T = 1.f;
    P0.C0 = P0.C1 = P0.C2 = P0.D = 0.f;
    P1.C0 = P1.C1 = P1.C2 = P1.D = 0.f;
    P0.last = P1.last = -1;
    P0.nblend = P1.nblend = 0;
    const bool in0 = px < a.width && py0 < a.height, in1 = px < a.width && py0 + 4 < a.height;
    if (!in0) P0.T = -1.f;
    if (!in1) P1.T = -1.f;
    int32_t *rec0 = nullptr, *rec1 = nullptr;
    if (REC && in0) rec0 = a.rec_pos + a.rec_off[(size_t)py0 * a.width + px];
    if (REC && in1) rec1 = a.rec_pos + a.rec_off[(size_t)(py0 + 4) * a.width + px];
    const float thr = a.floor > 0.f ? a.floor : 0.f;   // rasterize.py:194: alive while T >= floor
    bool warp_done = __all_sync(0xffffffffu, P0.done(thr) && P1.done(thr));
    auto leave = [&](int b) {   // as in forward_kernel
      if (lane == 0) {
        __threadfence_block();
        atomicAdd(&sm.ndone, 1);
#pragma unroll 1
        for (int i = 0; i < kStages; i++) {
          const int x = b + i;
          if (i > 0 && x >= kStages) mbar_wait(&sm.empty[x % kStages], ((x - kStages) / kStages) & 1);
          mbar_arrive_drop(&sm.empty[x % kStages]);
        }
      }
      __syncwarp();
    };
    WS_T0(tc);
    if (warp_done) leave(0);
    const bool cull = !STATS && a.cutoff > 0.f;
    for (int b = 0; b < nbatch && !warp_done; b++) {
      const int s = b % kStages;
      {
        WS_T0(tw);
        mbar_wait(&sm.full[s], (b / kStages) & 1);
        if (lane == 0) WS_ADD(1, tw);
        if (lane == 0 && b == 0) WS_ADD(8, tw);
      }
      if (*reinterpret_cast<volatile int *>(&sm.stop) == b + 1) break;
      {
        const uint32_t first = range.x + (uint32_t)b * kStageCands;
        const int count = (int)min((uint32_t)kStageCands, range.y - first);
        const uint32_t alive0 = __ballot_sync(0xffffffffu, !P0.done(thr));
        const uint32_t alive1 = __ballot_sync(0xffffffffu, !P1.done(thr));
        uint32_t pm0 = 0u, pm1 = 0u;
        if (lane < count) {
          const uint32_t bm = cull ? sm.bmask[s][lane] : 0xffu;
          const int4 bb = rec_bbox(sm.rec[s][lane]);
          if ((bm >> q0) & 1u) pm0 = block_mask(bb, rx0, ry0) & alive0;
          if ((bm >> (q0 + 2)) & 1u) pm1 = block_mask(bb, rx0, ry0 + 4) & alive1;
        }
        uint32_t m = __ballot_sync(0xffffffffu, (pm0 | pm1) != 0u);
        uint32_t vis0 = 0, vis1 = 0;
        while (m) {
          const int j = __ffs(m) - 1;
          m &= m - 1;
          const float4 *rec = sm.rec[s][j];
          const uint32_t pj0 = __shfl_sync(0xffffffffu, pm0, j), pj1 = __shfl_sync(0xffffffffu, pm1, j);
          const bool act0 = !P0.done(thr) && ((pj0 >> lane) & 1u);
          const bool act1 = !P1.done(thr) && ((pj1 >> lane) & 1u);
          const bool any0 = __any_sync(0xffffffffu, act0), any1 = __any_sync(0xffffffffu, act1);
          if (!(any0 || any1)) continue;
          if (STATS) {
            n_warp_evals += (any0 ? 1u : 0u) + (any1 ? 1u : 0u);
            n_eval += (act0 ? 1u : 0u) + (act1 ? 1u : 0u);
          }
          const int pos = (int)first + j;
          bool bl0 = false, bl1 = false;
          if (any0 && any1) {
            if (MAXK == 8) {
              const int nl = __float_as_int(rec[2].z);   // warp-uniform line count
              if (nl == 5) fwd_pair<5, MAXK, STATS, Z64>(rec, qx, qy0, act0, act1, a.cutoff, pos, P0, P1, n_lines, bl0, bl1);
              else if (nl == 6) fwd_pair<6, MAXK, STATS, Z64>(rec, qx, qy0, act0, act1, a.cutoff, pos, P0, P1, n_lines, bl0, bl1);
#ifndef CS_FWD_NO_NL4
              else if (nl == 4) fwd_pair<4, MAXK, STATS, Z64>(rec, qx, qy0, act0, act1, a.cutoff, pos, P0, P1, n_lines, bl0, bl1);
#endif
              else fwd_pair<0, MAXK, STATS, Z64>(rec, qx, qy0, act0, act1, a.cutoff, pos, P0, P1, n_lines, bl0, bl1);
            } else {
              fwd_pair<0, MAXK, STATS, Z64>(rec, qx, qy0, act0, act1, a.cutoff, pos, P0, P1, n_lines, bl0, bl1);
            }
          } else {
            // one of the two 8x4 blocks: the single-pixel evaluation
            FwdPixel &P = any0 ? P0 : P1;
            const bool act = any0 ? act0 : act1;
            const float qy = any0 ? qy0 : qy0 + 4.f;
            bool bl = false;
            if (act) {
              if (MAXK == 8) {
                const int nl = __float_as_int(rec[2].z);
                if (nl == 5) bl = fwd_candidate<5, MAXK, STATS, Z64>(rec, qx, qy, a.cutoff, a.floor, false, pos, P, n_lines);
                else if (nl == 6) bl = fwd_candidate<6, MAXK, STATS, Z64>(rec, qx, qy, a.cutoff, a.floor, false, pos, P, n_lines);
#ifndef CS_FWD_NO_NL4
                else if (nl == 4) bl = fwd_candidate<4, MAXK, STATS, Z64>(rec, qx, qy, a.cutoff, a.floor, false, pos, P, n_lines);
#endif
                else bl = fwd_candidate<0, MAXK, STATS, Z64>(rec, qx, qy, a.cutoff, a.floor, false, pos, P, n_lines);
              } else {
                bl = fwd_candidate<0, MAXK, STATS, Z64>(rec, qx, qy, a.cutoff, a.floor, false, pos, P, n_lines);
              }
            }
            if (any0) bl0 = bl; else bl1 = bl;
          }
          if (REC && bl0) rec0[P0.nblend - 1] = pos;
          if (REC && bl1) rec1[P1.nblend - 1] = pos;
          const bool b0 = __any_sync(0xffffffffu, bl0), b1 = __any_sync(0xffffffffu, bl1);
          if (b0) vis0 |= 1u << j;
          if (b1) vis1 |= 1u << j;
          if ((b0 || b1) && __all_sync(0xffffffffu, P0.done(thr) && P1.done(thr))) {
            warp_done = true;
            break;
          }
        }
        if (lane == 0) {
          if (vis0 | vis1) atomicOr(&sm.vis[s], vis0 | vis1);
          const size_t word = (size_t)(range.x >> 5) + tile + b;
          a.blend_mask[(size_t)q0 * a.mask_words + word] = vis0;
          a.blend_mask[(size_t)(q0 + 2) * a.mask_words + word] = vis1;
        }
      }
      __syncwarp();
      if (warp_done) {
        leave(b);
      } else if (lane == 0) {
        mbar_arrive(&sm.empty[s]);
      }
    }
    if (lane == 0) WS_ADD(0, tc);
    n_blend = (unsigned)(P0.nblend + P1.nblend);
#pragma unroll
    for (int h = 0; h < 2; h++) {
      const FwdPixel &P = h ? P1 : P0;
      const int py = py0 + 4 * h;
      if (px < a.width && py < a.height) {
        const size_t p = (size_t)py * a.width + px;
        const float v0 = fmaf(P.T, a.bg[0], P.C0), v1 = fmaf(P.T, a.bg[1], P.C1), v2 = fmaf(P.T, a.bg[2], P.C2);
        a.image[3 * p] = fminf(fmaxf(v0, 0.f), 1.f);
        a.image[3 * p + 1] = fminf(fmaxf(v1, 0.f), 1.f);
        a.image[3 * p + 2] = fminf(fmaxf(v2, 0.f), 1.f);
        a.final_T[p] = P.T;
        a.pixel_T[p] = P.T;
        a.weight_sum[p] = 1.f - P.T;
        a.count[p] = P.nblend;
        if (a.depth) a.depth[p] = P.D;
        a.pixel_last[p] = P.last;
        a.pixel_clamp[p] = (uint8_t)((v0 >= 0.f && v0 <= 1.f) | ((v1 >= 0.f && v1 <= 1.f) << 1) |
                                     ((v2 >= 0.f && v2 <= 1.f) << 2));
      }
    }
  }
  if (STATS) {
    block_add_u64(a.stats + S_FWD_EVALS, n_eval);
    block_add_u64(a.stats + S_FWD_LINES, n_lines);
    block_add_u64(a.stats + S_FWD_BLENDS, n_blend);
    block_add_u64(a.stats + S_FWD_WARP_EVALS, lane == 0 ? n_warp_evals : 0u);
  }
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

// Per-pixel backward state (backward.py:133-205).
// GS = g . S, the upstream gradient dotted with the colour composited
// behind (backward.py:163-205 keeps S per channel; only g . S enters
// d alpha, and g is constant per pixel): one running scalar instead of three.
struct BwdPixel {
  float T, g0, g1, g2, GS;
  int last;
};

// One candidate at one pixel of the reverse walk: recompute the field,
// reconstruct T_prev = T / (1 - alpha), and add the pixel's 32 screen-space
// gradient terms to v (unchanged when it did not blend).  Returns whether
// it did.
template <int NL, int MAXK, bool STATS, int VN, bool Z64 = false>
__device__ __forceinline__ bool bwd_candidate(const float4 *rec, float qx, float qy, float cutoff, BwdPixel &P,
                                              float (&v)[VN], unsigned &n_lines) {
  const float4 h0 = rec[0], h2 = rec[2];
  LineSet<NL, MAXK, Z64> L;
  L.load(rec, __float_as_int(h2.z));
  constexpr int N = LineSet<NL, MAXK, Z64>::kN;
  float z[N];
  const float dx = qx, dy = qy;   // relative to the tile's re-basing point
  const float o = h0.w, sig = h0.z, dls = h2.y, inv_dls = h2.w;
  const Eval e = eval_field<true>(L, sig, o, dx, dy, z);
  if (STATS) n_lines += L.nl;
  if (!(e.alpha >= cutoff)) return false;
  const float4 h1 = rec[1];
  const float om = fmaxf(fmaf(o, e.J, h2.x), 1e-6f);  // 1 - alpha
#ifdef CS_EXACT_RECIP
  const float rom = 1.f / om;
#else
  const float rom = frcp<Z64>(om);
#endif
  const float Tp = P.T * rom;
  const float w = Tp * e.alpha;
  const float c0 = h1.x, c1 = h1.y, c2 = h1.z;
  v[A_DC] += P.g0 * w;
  v[A_DC + 1] += P.g1 * w;
  v[A_DC + 2] += P.g2 * w;
  const float gc = fmaf(P.g0, c0, fmaf(P.g1, c1, P.g2 * c2));   // g . c
  float dA = fmaf(Tp, gc, -P.GS * rom);                            // g . (T_prev c - S / (1 - alpha))
  if (!(e.alpha_raw < (float)kAlphaMaxD)) dA = 0.f;
  v[A_DOEFF] += dA * e.I;
  const float dI = dA * o;
  const float slope = e.I * e.J;
  const float dphi = -sig * slope * dI;          // d loss / d phi (natural units)
  v[A_DSIG] += -(e.phi2 * kLn2) * slope * dI;
  const float dscale = dphi * (dls * kLn2);      // dphi * delta_s
  float wz = 0.f;
#pragma unroll
  for (int l = 0; l < N; l++) {
    if (L.has(l)) {
      const float wl = fx2<Z64, true>(z[l] - e.phi2);   // softmax_over_lines (field.py:62-67)
      wz = fmaf(wl, z[l], wz);
      const float dL = dscale * wl;
      v[A_LINES + 3 * l] += dL * dx;
      v[A_LINES + 3 * l + 1] += dL * dy;
      v[A_LINES + 3 * l + 2] += dL;
    }
  }
  v[A_DDEL] += dphi * wz * inv_dls;               // dphi * sum_l w_l L_l
  P.GS = fmaf(w, gc, P.GS);
  P.T = Tp;
  return true;
}

// The gradient terms of one pixel (bwd_candidate after its evaluation), with
// the blend decision as a predicate: a pixel that did not blend adds exact
// zeros (v never holds -0, so v + 0 == v) and keeps its state -- the same
// sums, in the same order, as the branch in bwd_candidate.
template <typename LS, int VN>
__device__ __forceinline__ void bwd_terms(const LS &L, const float (&z)[LS::kN],
                                          const Eval &e, bool ok, float dx, float dy, float4 h0, float4 h1,
                                          float4 h2, BwdPixel &P, float (&v)[VN]) {
  constexpr int N = LS::kN;
  const float o = h0.w, sig = h0.z, dls = h2.y, inv_dls = h2.w;
  const float om = fmaxf(fmaf(o, e.J, h2.x), 1e-6f);  // 1 - alpha
#ifdef CS_EXACT_RECIP
  const float rom = 1.f / om;
#else
  const float rom = frcp<LS::kPrecise>(om);
#endif
  const float Tp = P.T * rom;
  const float w = ok ? Tp * e.alpha : 0.f;
  v[A_DC] += P.g0 * w;
  v[A_DC + 1] += P.g1 * w;
  v[A_DC + 2] += P.g2 * w;
  const float gc = fmaf(P.g0, h1.x, fmaf(P.g1, h1.y, P.g2 * h1.z));   // g . c
  float dA = fmaf(Tp, gc, -P.GS * rom);
  if (!ok || !(e.alpha_raw < (float)kAlphaMaxD)) dA = 0.f;
  v[A_DOEFF] += dA * e.I;
  const float dI = dA * o;
  const float slope = e.I * e.J;
  const float dphi = -sig * slope * dI;
  v[A_DSIG] += ok ? -(e.phi2 * kLn2) * slope * dI : 0.f;
  const float dscale = dphi * (dls * kLn2);
  float wz = 0.f;
#pragma unroll
  for (int l = 0; l < N; l++) {
    if (L.has(l)) {
      const float wl = fx2<LS::kPrecise, true>(z[l] - e.phi2);
      wz = fmaf(wl, z[l], wz);
      const float dL = dscale * wl;
      v[A_LINES + 3 * l] += dL * dx;
      v[A_LINES + 3 * l + 1] += dL * dy;
      v[A_LINES + 3 * l + 2] += dL;
    }
  }
  v[A_DDEL] += ok ? dphi * wz * inv_dls : 0.f;
  P.GS = fmaf(w, gc, P.GS);
  if (ok) P.T = Tp;
}
// z_l and sum 2^z_l at (dx, dy): eval_field's expressions (ACC) and order.
template <typename LS>
__device__ __forceinline__ float line_sum_z(const LS &L, float dx, float dy, float (&z)[LS::kN]) {
  constexpr int N = LS::kN;
  float ex[N];
#pragma unroll
  for (int l = 0; l < N; l++) {
    if (L.has(l)) {
      z[l] = L.z(l, dx, dy);
      ex[l] = fx2<LS::kPrecise, true>(z[l]);
    } else {
      ex[l] = 0.f;
    }
  }
#pragma unroll
  for (int w = 1; w < N; w *= 2)
#pragma unroll
    for (int l = 0; l + w < N; l += 2 * w) ex[l] += ex[l + w];
  return ex[0];
}
template <typename LS>
__device__ __forceinline__ float lse_shifted_z(const LS &L, const float (&z)[LS::kN]) {
  constexpr int N = LS::kN;
  float m = -INFINITY;
#pragma unroll
  for (int l = 0; l < N; l++)
    if (L.has(l)) m = fmaxf(m, z[l]);
  float s2 = 0.f;
#pragma unroll
  for (int l = 0; l < N; l++)
    if (L.has(l)) s2 += fx2<LS::kPrecise, true>(z[l] - m);
  return m + flg2<LS::kPrecise, true>(s2);
}
template <bool P = false>
__device__ __forceinline__ Eval eval_finish_acc(float phi2, float sig, float o) {
  Eval e;
  const float u = fx2<P, true>(sig * phi2);
  e.I = frcp<P, true>(1.f + u);
  e.J = u > 1.f ? 1.f - e.I : u * e.I;
  e.alpha_raw = o * e.I;
  e.alpha = fminf(e.alpha_raw, (float)kAlphaMaxD);
  e.phi2 = phi2;
  return e;
}
// One candidate at both pixels of the lane (rows r and r + 4): one line load,
// two independent evaluation chains, the terms added pixel 0 then pixel 1
// (the order of the per-pixel calls).
template <int NL, int MAXK, bool STATS, int VN, bool Z64 = false>
__device__ __forceinline__ void bwd_pair(const float4 *rec, float qx, float qy0, bool act0, bool act1, float cutoff,
                                         BwdPixel &P0, BwdPixel &P1, float (&v)[VN], unsigned &n_lines, bool &ok0,
                                         bool &ok1) {
  constexpr int N = LineSet<NL, MAXK, Z64>::kN;
  const float4 h0 = rec[0], h2 = rec[2];
  LineSet<NL, MAXK, Z64> L;
  L.load(rec, __float_as_int(h2.z));
  float z0[N], z1[N];
  const float s0 = line_sum_z(L, qx, qy0, z0), s1 = line_sum_z(L, qx, qy0 + 4.f, z1);
  float phi0 = flg2<Z64, true>(s0), phi1 = flg2<Z64, true>(s1);
  if (!(lse_in_range(s0) && lse_in_range(s1))) {
    if (!lse_in_range(s0)) phi0 = lse_shifted_z(L, z0);
    if (!lse_in_range(s1)) phi1 = lse_shifted_z(L, z1);
  }
  const Eval e0 = eval_finish_acc<Z64>(phi0, h0.z, h0.w), e1 = eval_finish_acc<Z64>(phi1, h0.z, h0.w);
  if (STATS) n_lines += (unsigned)L.nl * ((act0 ? 1u : 0u) + (act1 ? 1u : 0u));
  ok0 = act0 && e0.alpha >= cutoff;
  ok1 = act1 && e1.alpha >= cutoff;
  const float4 h1 = rec[1];
  bwd_terms(L, z0, e0, ok0, qx, qy0, h0, h1, h2, P0, v);
  bwd_terms(L, z1, e1, ok1, qx, qy0 + 4.f, h0, h1, h2, P1, v);
}

// Backward blend (backward.py:110-205): the producer streams the tile list
// back to front from the block's largest `last`; each consumer warp culls a
// stage by ballot, reconstructs T_prev = T / (1 - alpha) per pixel and
// reduces the 32 screen-space gradient values of each candidate across the
// warp (transpose-reduce) into one vector of float atomics.
// PPL pixels per lane: 8 / PPL consumer warps of 8 x (4 PPL) pixels (lane =
// column + 8 * row of the top 8x4 block, pixel h another 4 h rows down).
// The lane sums its pixels' gradient terms before the transpose-reduce, so
// PPL = 2 halves the reductions per evaluated pixel (853 -> 775 us at 1M
// @1080p; PPL = 4: 929 us, the coarser 8x16 culling loses).
#ifndef CS_BWD_MINB
#define CS_BWD_MINB 6   // PPL 2: 5 -> 777 us, 6 -> 775, 7 -> 941 (spills)
#endif
#ifndef CS_BWD_PPL
#define CS_BWD_PPL 2
#endif
template <int MAXK, int PPL, bool STATS, bool Z64 = false>
__global__ void __launch_bounds__(pipe_threads<8 / PPL>(), CS_BWD_MINB) backward_kernel(BlendArgs a) {
  constexpr int NC = 8 / PPL;   // warps of 8 x (4 PPL) pixels
  constexpr int AF = Acc<MAXK>::kFloats;
  constexpr int NG = (AF + 31) / 32;
  constexpr int kStages = CS_BWD_STAGES;
  extern __shared__ __align__(16) unsigned char pipe_dyn_smem[];
  PipeSmem<MAXK, kStages, Z64> &sm = *reinterpret_cast<PipeSmem<MAXK, kStages, Z64> *>(pipe_dyn_smem);
  __shared__ int s_last[NC];
#ifdef CS_BWD_SMEM_REDUCE
  // per-warp transpose scratch: lane L's 32 values at row L (stride 36
  // floats: conflict-free 128-bit row stores and 32-bit column loads)
  __shared__ __align__(16) float s_red[NC][32 * 36];
#endif
  const int tile = a.tile_order ? (int)a.tile_order[blockIdx.x] : (int)blockIdx.x;
  const int tx = tile % a.tiles_x, ty = tile / a.tiles_x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint2 range = a.ranges[tile];
  const int rx0 = tx * kTile + ((warp & 1) << 3), ry0 = ty * kTile + (warp >> 1) * 4 * PPL;
  BwdPixel P[PPL];
  // pixel h of the lane, relative to the tile's re-basing point: (qx, qy0 + 4 h)
  const float qx = (float)(rx0 + (lane & 7) - tx * kTile - kRebase) + 0.5f;
  const float qy0 = (float)(ry0 + (lane >> 3) - ty * kTile - kRebase) + 0.5f;
#pragma unroll
  for (int h = 0; h < PPL; h++) {
    const int px = rx0 + (lane & 7), py = ry0 + (lane >> 3) + 4 * h;
    P[h].T = 1.f; P[h].g0 = P[h].g1 = P[h].g2 = P[h].GS = 0.f;
    P[h].last = -1;
    if (warp < NC && px < a.width && py < a.height) {
      const size_t p = (size_t)py * a.width + px;
      P[h].T = a.pixel_T[p];
      P[h].last = a.pixel_last[p];
      const uint32_t cm = a.pixel_clamp[p];
      P[h].g0 = (cm & 1) ? a.d_image[3 * p] : 0.f;
      P[h].g1 = (cm & 2) ? a.d_image[3 * p + 1] : 0.f;
      P[h].g2 = (cm & 4) ? a.d_image[3 * p + 2] : 0.f;
      P[h].GS = P[h].T * fmaf(P[h].g0, a.bg[0], fmaf(P[h].g1, a.bg[1], P[h].g2 * a.bg[2]));   // S = T_final bg
    }
  }
  // last blended position of each of the warp's 8x4 blocks (the forward
  // wrote a blend-mask word for every batch up to it) and of the warp
  int sub_last[PPL];
#pragma unroll
  for (int h = 0; h < PPL; h++) sub_last[h] = __reduce_max_sync(0xffffffffu, P[h].last);
  int lmax = sub_last[0];
#pragma unroll
  for (int h = 1; h < PPL; h++) lmax = max(lmax, sub_last[h]);
  const int warp_last = lmax;
  if (warp < NC && lane == 0) s_last[warp] = warp_last;
  pipe_init<MAXK, kStages, NC>(sm);
  int block_last = s_last[0];
#pragma unroll
  for (int w = 1; w < NC; w++) block_last = max(block_last, s_last[w]);
  const int64_t end = (int64_t)block_last + 1;
  const int nbatch = end > (int64_t)range.x ? (int)((end - range.x + kStageCands - 1) / kStageCands) : 0;
  auto batch = [&](int b, uint32_t &first, uint32_t &count) {
    const int64_t hi = end - (int64_t)b * kStageCands;
    const int64_t lo = max((int64_t)range.x, hi - kStageCands);
    first = (uint32_t)lo;
    count = (uint32_t)(hi - lo);
  };
  unsigned n_eval = 0, n_lines = 0, n_warp_evals = 0, n_bblend = 0;
  if (warp == NC) {
    const TileLines tl{(double)(tx * kTile + kRebase), (double)(ty * kTile + kRebase), 0.f};
    pipe_produce<MAXK, kStages, NC>(sm, a.records, a.lines, a.pair_ids, nbatch, batch, false, nullptr, tl, false);
  } else {
    WS_T0(tc);
    for (int b = 0; b < nbatch; b++) {
      const int s = b % kStages;
      uint32_t first, count;
      batch(b, first, count);
      // the forward's blend masks of this warp's 8x4 blocks for the batch
      // (loaded before the wait): candidates none of a block's pixels
      // blended are skipped for it
      uint32_t fm[PPL];
      if ((int)first <= warp_last) {
#pragma unroll
        for (int h = 0; h < PPL; h++) {
          const int sub = ((((ry0 - ty * kTile) >> 2) + h) << 1) | ((rx0 - tx * kTile) >> 3);
          const uint32_t rel = first - range.x;   // forward batch rel / 32, bit rel % 32
          const uint32_t *mk = a.blend_mask + (size_t)sub * a.mask_words + (range.x >> 5) + tile + (rel >> 5);
          const uint32_t sh = rel & 31u;
          // only words of forward batches that hold a position <= the
          // block's last were written (and can matter)
          const uint32_t w0 = (int)first <= sub_last[h] ? __ldg(mk) : 0u;
          const uint32_t w1 = sh && (int)(first + 32u - sh) <= sub_last[h] ? __ldg(mk + 1) : 0u;
          fm[h] = sh ? (w0 >> sh) | (w1 << (32u - sh)) : w0;
        }
      }
      {
        WS_T0(tw);
        mbar_wait(&sm.full[s], (b / kStages) & 1);
        if (lane == 0) WS_ADD(5, tw);
      }
      if ((int)first <= warp_last) {
        const uint32_t pos = first + lane;
        uint32_t pm[PPL], any = 0u;
#pragma unroll
        for (int h = 0; h < PPL; h++) pm[h] = 0u;
        if (lane < (int)count && (int)pos <= warp_last) {
          const int4 bb = rec_bbox(sm.rec[s][lane]);
#pragma unroll
          for (int h = 0; h < PPL; h++) {
            pm[h] = ((fm[h] >> lane) & 1u) ? block_mask(bb, rx0, ry0 + 4 * h) : 0u;
            any |= pm[h];
          }
        }
        uint32_t m = __ballot_sync(0xffffffffu, any != 0u);
        while (m) {
          const int j = 31 - __clz(m);   // back to front
          m &= ~(1u << j);
          const float4 *rec = sm.rec[s][j];
          float v[NG * 32];
#pragma unroll
          for (int f = 0; f < NG * 32; f++) v[f] = 0.f;
          const int cpos = (int)first + j;
          bool act[PPL], any_act = false;
#pragma unroll
          for (int h = 0; h < PPL; h++) {
            const uint32_t pj = __shfl_sync(0xffffffffu, pm[h], j);
            act[h] = cpos <= P[h].last && ((pj >> lane) & 1u);
            if (STATS) n_eval += (unsigned)act[h];
            any_act |= act[h];
          }
          bool contrib = false;
#ifndef CS_BWD_NO_PAIR
#ifdef CS_BWD_PAIR_ONLY
          const bool pair = PPL == 2;   // one code path (the idle pixel's terms are predicated off)
#else
          bool pair = PPL == 2 && __any_sync(0xffffffffu, act[0]) && __any_sync(0xffffffffu, act[PPL - 1]);
#ifndef CS_BWD_PAIR_NL0   // MAXK = 8: pair only the specialised line counts (the generic
                          // instance's registers spilled everywhere: 652 -> 641 us without it)
          if (MAXK == 8) {
            const int nl_ = __float_as_int(rec[2].z);
            pair = pair && nl_ >= 4 && nl_ <= 6;
          }
#endif
#endif
#else
          const bool pair = false;
#endif
#define CS_BWD2_PX(NLV, H)                                                                       \
  if (H < PPL && act[H % PPL]) {                                                                   \
    const bool c_ = bwd_candidate<NLV, MAXK, STATS, NG * 32, Z64>(rec, qx, qy0 + (float)(4 * (H % PPL)), a.cutoff, P[H % PPL], v, n_lines); \
    contrib |= c_;                                                                                 \
    if (STATS) n_bblend += (unsigned)c_;                                                           \
  }
#define CS_BWD2_CASE(NLV) CS_BWD2_PX(NLV, 0) CS_BWD2_PX(NLV, 1) CS_BWD2_PX(NLV, 2) CS_BWD2_PX(NLV, 3)
#define CS_BWD2_PAIR(NLV)                                                                        \
  {                                                                                                \
    bool o0_, o1_;                                                                                 \
    bwd_pair<NLV, MAXK, STATS, NG * 32, Z64>(rec, qx, qy0, act[0], act[PPL - 1], a.cutoff, P[0], P[PPL - 1], v, n_lines, o0_, o1_); \
    contrib = o0_ || o1_;                                                                          \
    if (STATS) n_bblend += (unsigned)o0_ + (unsigned)o1_;                                         \
  }
          if (pair) {
            if (MAXK == 8) {
              const int nl = __float_as_int(rec[2].z);   // warp-uniform line count
              if (nl == 5) CS_BWD2_PAIR(5)
              else if (nl == 6) CS_BWD2_PAIR(6)
#ifndef CS_BWD_NO_NL4   // (without the 4-line instance: 639 vs 647 us at the 1080p bench view,
                        // but 129 vs 114 ms per config-5 step, whose views hold more 4-line hulls)
              else if (nl == 4) CS_BWD2_PAIR(4)
#endif
              else CS_BWD2_PAIR(0)
            } else {
              CS_BWD2_PAIR(0)
            }
          } else if (MAXK == 8) {
            const int nl = __float_as_int(rec[2].z);   // warp-uniform line count
            if (nl == 5) { CS_BWD2_CASE(5) }
            else if (nl == 6) { CS_BWD2_CASE(6) }
#ifndef CS_BWD_NO_NL4
            else if (nl == 4) { CS_BWD2_CASE(4) }
#endif
            else { CS_BWD2_CASE(0) }
          } else {
            CS_BWD2_CASE(0)
          }
#undef CS_BWD2_PAIR
#undef CS_BWD2_CASE
#undef CS_BWD2_PX
          if (STATS) n_warp_evals += __any_sync(0xffffffffu, any_act) ? 1u : 0u;
          if (__any_sync(0xffffffffu, contrib)) {
            // the line sums are kept relative to the record's anchor a (the
            // chain's frame): sum dL (q - a) = sum dL (q - T) + (T - a) sum dL
            {
              const float2 an = *reinterpret_cast<const float2 *>(rec);
              const float ox = (float)(tx * kTile + kRebase) - an.x, oy = (float)(ty * kTile + kRebase) - an.y;
#pragma unroll
              for (int l = 0; l < MAXK; l++) {
                v[A_LINES + 3 * l] = fmaf(ox, v[A_LINES + 3 * l + 2], v[A_LINES + 3 * l]);
                v[A_LINES + 3 * l + 1] = fmaf(oy, v[A_LINES + 3 * l + 2], v[A_LINES + 3 * l + 1]);
              }
            }
            AccT *dst = a.accum + (size_t)sm.id[s][j] * AF;
#pragma unroll
            for (int gi = 0; gi < NG; gi++) {
              float (&vv)[32] = *reinterpret_cast<float (*)[32]>(v + 32 * gi);
#ifdef CS_BWD_SMEM_REDUCE
              float *red = s_red[warp];
              {
                float4 *row = reinterpret_cast<float4 *>(red + lane * 36);
#pragma unroll
                for (int q = 0; q < 8; q++) row[q] = make_float4(vv[4 * q], vv[4 * q + 1], vv[4 * q + 2], vv[4 * q + 3]);
              }
              __syncwarp();
              float sum = 0.f;
#pragma unroll
              for (int r = 0; r < 32; r++) sum += red[r * 36 + lane];
              __syncwarp();
#else
              const float sum = transpose_reduce32(vv);
#endif
              const int f = gi * 32 + lane;
              if (f < AF && sum != 0.f) atomicAdd(dst + f, (AccT)sum);
            }
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.empty[s]);
    }
    if (lane == 0) WS_ADD(4, tc);
  }
  if (STATS) {
    block_add_u64(a.stats + S_BWD_EVALS, n_eval);
    block_add_u64(a.stats + S_BWD_LINES, n_lines);
    block_add_u64(a.stats + S_BWD_WARP_EVALS, lane == 0 ? n_warp_evals : 0u);
    block_add_u64(a.stats + S_BWD_BLENDS, n_bblend);
  }
}

// Blend lines staged and evaluated in float64 for the scalings whose line
// slopes the float32 evaluation cannot hold at scale (NONE: no depth factor,
// DEPTH_SQUARED: its square); DEPTH and SQRT_DEPTH (the
// configs' scaling) keep the float32 planes.
static bool lines_f64(const cs_settings &set) {
#ifdef CS_LINES_F32_ONLY
  (void)set;
  return false;
#else
  return set.scaling_mode == CS_SCALE_NONE || set.scaling_mode == CS_SCALE_DEPTH2;
#endif
}

static BlendArgs make_args(const cs_camera &cam, const cs_settings &set, const cs_layout &L, char *ws) {
  BlendArgs a;
  a.records = reinterpret_cast<const float *>(ws + L.records);
  a.lines = reinterpret_cast<const double *>(ws + L.lines);
  a.pair_ids = reinterpret_cast<const uint32_t *>(ws + L.pair_ids);
  a.ranges = reinterpret_cast<const uint2 *>(ws + L.tile_ranges);
  a.tile_order = L.tiles_x * L.tiles_y <= kMaxTileOrder ? reinterpret_cast<const uint32_t *>(ws + L.scratch) : nullptr;
  a.width = cam.width;
  a.height = cam.height;
  a.tiles_x = L.tiles_x;
  a.cutoff = (float)set.cutoff;
  a.floor = (float)set.floor;
  for (int c = 0; c < 3; c++) a.bg[c] = (float)set.background[c];
  a.pixel_last = reinterpret_cast<int32_t *>(ws + L.pixel_last);
  a.pixel_T = reinterpret_cast<float *>(ws + L.pixel_T);
  a.pixel_clamp = reinterpret_cast<uint8_t *>(ws + L.pixel_clamp);
  a.blend_mask = reinterpret_cast<uint32_t *>(ws + L.scratch + blend_mask_offset());
  a.mask_words = blend_mask_words((int64_t)((L.pair_ids - L.pair_tiles) / sizeof(uint32_t)), L.tiles_x * L.tiles_y);
  a.accum = reinterpret_cast<AccT *>(ws + L.grad_accum);
  a.stats = reinterpret_cast<unsigned long long *>(ws + L.counters + sizeof(uint32_t) * C_STATS);
  a.image = a.final_T = a.weight_sum = a.depth = nullptr;
  a.count = nullptr;
  a.visible = nullptr;
  a.d_image = nullptr;
  a.rec_off = nullptr;
  a.rec_pos = nullptr;
  a.ahead = 0;
  return a;
}

int launch_forward_blend(const cs_camera &cam, const cs_settings &set, const cs_params &p,
                         const cs_layout &L, char *ws, const cs_frame &f, bool stats, cudaStream_t s,
                         const int64_t *rec_off, int32_t *rec_pos) {
  BlendArgs a = make_args(cam, set, L, ws);
  a.rec_off = rec_off;
  a.rec_pos = rec_pos;
  const bool rec = rec_off != nullptr;
  a.image = f.image;
  a.final_T = f.final_T;
  a.weight_sum = f.weight_sum;
  a.depth = f.depth;
  a.count = f.count;
  a.visible = f.visible;
  if (f.visible && p.n > 0) cudaMemsetAsync(f.visible, 0, (size_t)p.n, s);
  const int tiles = L.tiles_x * L.tiles_y;
  {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    a.ahead = sms * CS_FWD_MINB;   // resident blocks (the launch bound's blocks per SM)
#ifdef CS_NO_LOOK_AHEAD
    a.ahead = 0;
#endif
  }
#ifndef CS_FWD_PPL1
  a.ahead = a.ahead / CS_FWD_MINB * CS_FWD2_MINB;
  auto go = [&](auto kernel, size_t smem) {
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kernel<<<tiles, pipe_threads<4>(), smem, s>>>(a);
  };
  if (lines_f64(set)) {
    if (L.max_k == 8)
      go(rec ? forward2_kernel<8, false, true, true> : stats ? forward2_kernel<8, true, false, true>
                                                             : forward2_kernel<8, false, false, true>,
         sizeof(PipeSmem<8, CS_FWD_STAGES, true>));
    else
      go(rec ? forward2_kernel<16, false, true, true> : stats ? forward2_kernel<16, true, false, true>
                                                              : forward2_kernel<16, false, false, true>,
         sizeof(PipeSmem<16, CS_FWD_STAGES, true>));
  } else {
    if (L.max_k == 8)
      go(rec ? forward2_kernel<8, false, true> : stats ? forward2_kernel<8, true> : forward2_kernel<8, false>,
         sizeof(PipeSmem<8, CS_FWD_STAGES>));
    else
      go(rec ? forward2_kernel<16, false, true> : stats ? forward2_kernel<16, true> : forward2_kernel<16, false>,
         sizeof(PipeSmem<16, CS_FWD_STAGES>));
  }
  return cudaGetLastError() == cudaSuccess ? CS_OK : CS_ERR_CUDA;
#endif
  if (L.max_k == 8) {
    auto k = rec ? forward_kernel<8, false, true> : stats ? forward_kernel<8, true> : forward_kernel<8, false>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(PipeSmem<8, CS_FWD_STAGES>));
    k<<<tiles * (8 / CS_FWD_NC), pipe_threads<CS_FWD_NC>(), sizeof(PipeSmem<8, CS_FWD_STAGES>), s>>>(a);
  } else {
    auto k = rec ? forward_kernel<16, false, true> : stats ? forward_kernel<16, true> : forward_kernel<16, false>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(PipeSmem<16, CS_FWD_STAGES>));
    k<<<tiles * (8 / CS_FWD_NC), pipe_threads<CS_FWD_NC>(), sizeof(PipeSmem<16, CS_FWD_STAGES>), s>>>(a);
  }
  return cudaGetLastError() == cudaSuccess ? CS_OK : CS_ERR_CUDA;
}

// Zeroing the screen-space accumulators (128 MB at 1M convexes):
// 16-byte streaming stores over a grid of 8 blocks per SM.
__global__ void __launch_bounds__(512) zero_kernel(float4 *p, size_t n4) {
  const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
  for (size_t i = (size_t)blockIdx.x * 512 + threadIdx.x; i < n4; i += (size_t)gridDim.x * 512) __stcs(p + i, z);
}

int launch_zero_accumulators(const cs_params &p, const cs_layout &L, char *ws, cudaStream_t s) {
  if (p.n > 0) {
    AccT *acc = reinterpret_cast<AccT *>(ws + L.grad_accum);
#ifdef CS_MEMSET_ACCUM
    cudaMemsetAsync(acc, 0, (size_t)p.n * L.acc_floats * sizeof(AccT), s);
#else
    const size_t n4 = (size_t)p.n * L.acc_floats * sizeof(AccT) / 16;   // acc_floats is a multiple of 4
    zero_kernel<<<(int)std::min<size_t>((n4 + 511) / 512, 148 * 8), 512, 0, s>>>(reinterpret_cast<float4 *>(acc), n4);
#endif
  }
  return cudaGetLastError() == cudaSuccess ? CS_OK : CS_ERR_CUDA;
}

int launch_backward_blend(const cs_camera &cam, const cs_settings &set, const cs_params &p,
                          const cs_layout &L, char *ws, const float *d_image, bool stats, bool zero, cudaStream_t s) {
  BlendArgs a = make_args(cam, set, L, ws);
  a.d_image = d_image;
  if (zero) launch_zero_accumulators(p, L, ws, s);
  const int tiles = L.tiles_x * L.tiles_y;
  auto go = [&](auto kernel, size_t smem) {
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kernel<<<tiles, pipe_threads<8 / CS_BWD_PPL>(), smem, s>>>(a);
  };
  if (lines_f64(set)) {
    if (L.max_k == 8)
      go(stats ? backward_kernel<8, CS_BWD_PPL, true, true> : backward_kernel<8, CS_BWD_PPL, false, true>,
         sizeof(PipeSmem<8, CS_BWD_STAGES, true>));
    else
      go(stats ? backward_kernel<16, CS_BWD_PPL, true, true> : backward_kernel<16, CS_BWD_PPL, false, true>,
         sizeof(PipeSmem<16, CS_BWD_STAGES, true>));
  } else {
    if (L.max_k == 8)
      go(stats ? backward_kernel<8, CS_BWD_PPL, true> : backward_kernel<8, CS_BWD_PPL, false>,
         sizeof(PipeSmem<8, CS_BWD_STAGES>));
    else
      go(stats ? backward_kernel<16, CS_BWD_PPL, true> : backward_kernel<16, CS_BWD_PPL, false>,
         sizeof(PipeSmem<16, CS_BWD_STAGES>));
  }
  return cudaGetLastError() == cudaSuccess ? CS_OK : CS_ERR_CUDA;
}

}  // namespace cs

#ifdef CS_WAIT_STATS
extern "C" CS_API int cs_debug_wait_stats(unsigned long long *host12, int reset) {
  cudaDeviceSynchronize();
  if (cudaMemcpyFromSymbol(host12, cs::g_wait_stats, sizeof(unsigned long long) * 12) != cudaSuccess) return 2;
  if (reset) {
    unsigned long long z[12] = {0};
    cudaMemcpyToSymbol(cs::g_wait_stats, z, sizeof(z));
  }
  return 0;
}
#endif
