// Shared definitions of the sm_100a convex-splatting kernels.
#pragma once
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#include "../../include/convexsplat_b200.h"

namespace cs {

constexpr int kTile = 16;                 // rasterize.py:23 TILE_SIZE (only 16 supported)
constexpr int kTilePixels = kTile * kTile;
constexpr int kShCoeffs = 16;             // model.py:15
constexpr double kMaskGate = 0.01;        // rasterize.py:26
constexpr double kCrossTol = 1e-9;        // projection.py:19
constexpr double kAlphaMaxD = 1.0 - 1e-6; // rasterize.py:30
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;
constexpr uint64_t kCulledKey = ~0ull;
// tiles ordered heaviest first for the blends (scratch + 0); larger frames use index order
constexpr int kMaxTileOrder = 1 << 17;

// ---------------------------------------------------------------------------
// Per-convex blend record, written by the preprocess kernel:
//   header (float32, 16 floats, global `records`):
//     float4 0: ax ay sigma_s o | 1: r g b depth | 2: 1-o dls nl 1/dls
//     float4 3: bbox x0 x1 y0 y1 (int32 bits, half-open)
//   lines (float64, global `lines`, [MAXK][4] = (A, B, C, 0) per line, one
//   256-bit store / load each):
//     z2_j(q) = A_j*(qx-ax) + B_j*(qy-ay) + C_j = delta_s*log2(e)*L_j(q)
//   where L_j = n_j.q + off_j is the reference's signed line distance
//   (projection.py:131-133) and (ax, ay) an integer anchor (the pixel at hull
//   vertex 0).
// The blend kernels' producer warp re-bases every line of a candidate onto
// the tile it streams it to -- C'_j = z2_j at the tile's centre point
// (tx*16+8, ty*16+8), formed in float64 -- and stages float32 (A, B, C') in
// shared memory next to the header: the per-pixel float32 evaluation then
// only sees |dx|, |dy| <= 8 and |C'| = |z| near the tile, instead of
// cancelling offsets of the size of the convex (a 300-pixel convex at
// delta_s*log2(e) ~ 7 carried ~1e-4 of absolute error in z2 with one anchor).
// Stage record in shared memory: header (16 floats) | A[MAXK] | B[MAXK] | C'[MAXK].
enum RecField {
  R_AX = 0, R_AY = 1, R_SIGMA = 2, R_OPACITY = 3, R_R = 4, R_G = 5, R_B = 6, R_DEPTH = 7,
  R_ONE_MINUS_O = 8, R_DLS = 9, R_NLINES = 10, R_INV_DLS = 11, R_BBOX = 12, R_HEADER = 16
};
template <int MAXK> struct Rec {
  static constexpr int kGlobal = R_HEADER;               // floats per convex in `records`
  static constexpr int kFloats = R_HEADER + 3 * MAXK;   // stage record: 40 for MAXK=8, multiple of 4
  static constexpr int kLines64 = 4 * MAXK;             // doubles per convex in `lines`
  static_assert(kFloats % 4 == 0 && MAXK % 4 == 0, "record planes must be float4 aligned");
};
// A candidate's record in a blend stage: the header, then its hull lines
// re-based onto the tile as planes A | B | C' -- float32, or float64 (Z64:
// the scalings whose line slopes the float32 field evaluation cannot hold,
// DESIGN.md section 2).
template <int MAXK, bool Z64 = false> struct StageRec {
  static constexpr int kFloats = R_HEADER + (Z64 ? 6 : 3) * MAXK;
  static_assert(kFloats % 4 == 0, "stage records are float4 rows");
};
// Tile re-basing point: pixel (tx*16 + kRebase, ty*16 + kRebase).
constexpr int kRebase = 8;

// Screen-space gradient accumulators per convex (backward.py:102-108):
//   d_color(3), d_opacity_eff, d_sigma_s, d_delta_s, pad(2), then per line
//   (sum dL*(qx-ax), sum dL*(qy-ay), sum dL).
enum AccField { A_DC = 0, A_DOEFF = 3, A_DSIG = 4, A_DDEL = 5, A_LINES = 8 };
template <int MAXK> struct Acc {
  static constexpr int kFloats = A_LINES + 3 * MAXK;
};
// Accumulator element type: the per-warp float32 partial sums of the
// backward blend are added into AccT by global atomics.  float64 (native
// red.global.add.f64): the order of those additions varies from run to run,
// and in float32 a convex spread over thousands of tiles changed its
// near-cancelling sums by up to ~7e-4 relative between runs; in float64 the
// order costs ~1e-16.  -DCS_ACC_F32 for the float32 accumulators.
#ifdef CS_ACC_F32
typedef float AccT;
#else
typedef double AccT;
#endif

// Counters at the head of the workspace.
// C_KMINC / C_KMAX: uint64 complement of the smallest / the largest depth key
// of the visible convexes (word offsets, 8-byte aligned), for the 32-bit
// depth-sort keys.
enum Counter {
  C_NVISIBLE = 0, C_NPAIRS = 1, C_OVERFLOW = 2, C_NSORT = 3, C_CHUNK0 = 4, C_STATS = 16, C_KMINC = 32, C_KMAX = 34,
  C_NONFINITE = 36, C_COUNT = 40
};
// uint64 work statistics at word C_STATS (roofline accounting, read by the benchmark)
enum Stat {
  S_FWD_EVALS = 0, S_FWD_LINES = 1, S_FWD_BLENDS = 2, S_BWD_EVALS = 3, S_BWD_LINES = 4, S_FWD_WARP_EVALS = 5,
  S_BWD_WARP_EVALS = 6, S_BWD_BLENDS = 7, S_COUNT = 8
};

// Block-wide sum of a per-thread count, added once per block to a global u64.
__device__ __forceinline__ void block_add_u64(unsigned long long *dst, unsigned v) {
  __shared__ unsigned long long s_acc;
  if (threadIdx.x == 0) s_acc = 0;
  __syncthreads();
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0 && v) atomicAdd(&s_acc, (unsigned long long)v);
  __syncthreads();
  if (threadIdx.x == 0 && s_acc) atomicAdd(dst, s_acc);
}

struct Layout {
  cs_layout l;
};

constexpr size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// Order-preserving map of a double to uint64 (ascending).
__device__ __forceinline__ uint64_t orderable_bits(double d) {
  if (d == 0.0) d = 0.0;  // -0.0 ties +0.0 as in Python's sort
  uint64_t b = (uint64_t)__double_as_longlong(d);
  return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}

// 256-bit global accesses (sm_100): four doubles at a 32-byte aligned address.
__device__ __forceinline__ void st_global_v4d(double *p, double a, double b, double c, double d) {
  asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(a), "d"(b), "d"(c), "d"(d) : "memory");
}
__device__ __forceinline__ void ld_global_nc_v4d(const double *p, double &a, double &b, double &c, double &d) {
  asm volatile("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];" : "=d"(a), "=d"(b), "=d"(c), "=d"(d) : "l"(p));
}

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float lg2(float x) {
  float y;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float rcp(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// ---------------------------------------------------------------------------
// TMA 1-D bulk copies (cp.async.bulk global -> shared, completion on an
// mbarrier).  Addresses and sizes must be 16-byte aligned.
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tma_bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
// shared -> global bulk store / bulk float reduction (+=), bulk-group
// completion; the generic-proxy writes to the source must be fenced first.
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tma_bulk_s2g(void *dst, const void *src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void tma_bulk_s2g_add(float *dst, const float *src, uint32_t bytes) {
  asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;" ::"l"(dst),
               "r"(smem_u32(src)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void tma_bulk_commit_and_wait_read() {
  asm volatile("cp.async.bulk.commit_group;\n cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t *bar, uint32_t phase) {
  uint32_t done;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
      : "=r"(done)
      : "r"(smem_u32(bar)), "r"(phase)
      : "memory");
  return done != 0;
}
// Wait for the phase of parity `phase` to complete.  A wait longer than 2 s
// can only be a protocol bug: trap (the launch fails with an error the host
// reports) instead of hanging the device.
// try_wait with a suspend-time hint: the waiting warp sleeps until the phase
// completes (or the hint elapses) instead of spinning on issue slots.
__device__ __forceinline__ bool mbar_try_wait_sleep(uint64_t *bar, uint32_t phase) {
  uint32_t done;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n selp.u32 %0, 1, 0, p;\n}"
      : "=r"(done)
      : "r"(smem_u32(bar)), "r"(phase), "r"(1000000u)
      : "memory");
  return done != 0;
}
// Wait for the phase of parity `phase` to complete: suspend-hinted
// try_wait (the warp sleeps until a barrier event of the CTA), the 2 s
// watchdog read once per 64 polls (a wait that long is a protocol bug: trap
// instead of hanging the device).
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t phase) {
  if (mbar_try_wait(bar, phase)) return;
  const uint64_t t0 = globaltimer_ns();
  for (;;) {
#pragma unroll 1
    for (int it = 0; it < 64; it++)
      if (mbar_try_wait_sleep(bar, phase)) return;
    if (globaltimer_ns() - t0 > 2000000000ull) {
#ifdef CS_WAIT_DEBUG
      printf("mbar_wait timeout: block %d thread %d bar smem+%u parity %u\n", (int)blockIdx.x, (int)threadIdx.x,
             smem_u32(bar), phase);
#endif
      __trap();
    }
  }
}
// The same with an exponential __nanosleep back-off (up to max_ns): for a
// waiter that expects a long wait (the producer warp waiting for the
// consumers to release a stage), so that it stays off the issue slots
// instead of waking on every barrier event of the CTA.
__device__ __forceinline__ void mbar_wait_backoff(uint64_t *bar, uint32_t phase, uint32_t max_ns) {
  if (mbar_try_wait(bar, phase)) return;
  const uint64_t t0 = globaltimer_ns();
  uint32_t ns = 32;
  for (;;) {
#pragma unroll 1
    for (int it = 0; it < 16; it++) {
      __nanosleep(ns);
      if (mbar_try_wait(bar, phase)) return;
      ns = min(2u * ns, max_ns);
    }
    if (globaltimer_ns() - t0 > 2000000000ull) {
#ifdef CS_WAIT_DEBUG
      printf("mbar_wait_backoff timeout: block %d thread %d bar smem+%u parity %u\n", (int)blockIdx.x,
             (int)threadIdx.x, smem_u32(bar), phase);
#endif
      __trap();
    }
  }
}
// Leave a barrier for good: arrive on its current phase and drop this
// thread's arrival from the expected count of every later phase.
__device__ __forceinline__ void mbar_arrive_drop(uint64_t *bar) {
  asm volatile("mbarrier.arrive_drop.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Pixel of a 16x16 tile handled by thread t: warps cover 8x4 sub-blocks so
// a warp's pixels form a compact square (better bbox culling per warp).
__device__ __forceinline__ void tile_pixel(int t, int &lx, int &ly) {
  int warp = t >> 5, lane = t & 31;
  lx = ((warp & 1) << 3) | (lane & 7);
  ly = ((warp >> 1) << 2) | (lane >> 3);
}

}  // namespace cs

// Entry points implemented in the .cu files (host side, C++ linkage).
namespace cs {
int launch_preprocess(const cs_camera &cam, const cs_settings &set, const cs_params &p,
                      const cs_layout &L, char *ws, cudaStream_t s);
int launch_binning(const cs_camera &cam, const cs_settings &set, const cs_params &p,
                   const cs_layout &L, char *ws, int64_t cap, cudaStream_t s);
int launch_forward_blend(const cs_camera &cam, const cs_settings &set, const cs_params &p,
                         const cs_layout &L, char *ws, const cs_frame &f, bool stats, cudaStream_t s,
                         const int64_t *rec_off = nullptr, int32_t *rec_pos = nullptr);
int launch_backward_blend(const cs_camera &cam, const cs_settings &set, const cs_params &p,
                          const cs_layout &L, char *ws, const float *d_image, bool stats, bool zero, cudaStream_t s);
int launch_zero_accumulators(const cs_params &p, const cs_layout &L, char *ws, cudaStream_t s);
int launch_chain(const cs_camera &cam, const cs_settings &set, const cs_params &p,
                 const cs_layout &L, char *ws, const cs_grads &g, const cs_view_signal *sig, bool overwrite,
                 cudaStream_t s, int64_t first = 0, int64_t last = -1);
int launch_image_loss(int H, int W, const float *img, const float *tgt, const float *raw_mask, int64_t n,
                      double lam, double beta, float *d_image, float *d_raw_mask, double *stats, void *ws,
                      cudaStream_t s);
int launch_adam(int count, const cs_adam_tensor *tensors, double b1, double b2, double eps, int step,
                double gscale, cudaStream_t s);
int launch_checkpoint_rows(bool pack, int precision, int64_t n, int k, void *rows, const cs_scene_out &o,
                           cudaStream_t s);
int launch_density_flags(const cs_params &P, const float *signal, const cs_density_config &c, uint8_t *flags,
                         uint32_t *child_keep, int64_t *surv_count, int64_t *child_count, cudaStream_t s);
int launch_density_scatter(const cs_params &P, const cs_density_config &c, const uint8_t *flags,
                           const uint32_t *child_keep, const int64_t *surv_pos, const int64_t *child_pos,
                           const int64_t *n_surv, const cs_scene_out &o, int64_t *index_map, cudaStream_t s);
int launch_export_view(const cs_camera &cam, const cs_settings &set, const cs_params &p, const cs_layout &L,
                       const char *ws, const cs_view_export &out, cudaStream_t s);
int launch_hull_batch(int32_t m, int32_t npts, const int32_t *counts, const double *pts,
                      int32_t *hull, int32_t *hull_n, cudaStream_t s);
size_t scratch_bytes(int64_t n, int64_t cap, int pair_passes, int tiles, struct Scratch *sc, char *base);
// forward blend masks (8 bit arrays of blend_mask_words words) in the scratch, after the tile order
uint32_t blend_mask_words(int64_t cap, int tiles);
constexpr size_t blend_mask_offset() { return align_up(sizeof(uint32_t) * kMaxTileOrder, 256); }
int pair_sort_passes(int tiles);
}  // namespace cs
