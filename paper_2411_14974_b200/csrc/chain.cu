// K4b: per-convex gradient chain (backward.py:215-282), one thread per convex.
//
// Turns the screen-space accumulators of the backward blend into gradients of
// the raw parameters (reciprocals instead of divisions; float32 unless
// built with -DCS_CHAIN_F64):
//   hull lines -> hull vertices (normalisation Jacobian, backward.py:231-246)
//   -> projection Jacobian -> 3-D points (backward.py:248-261)
//   delta/sigma activations + the depth path (backward.py:263-269)
//   opacity and straight-through mask (backward.py:271-275)
//   SH VJP + view-direction path (backward.py:277-282, harmonics.py:112-128)
// Discrete state (hull cycle, anchor) is read from the forward workspace;
// projection, depth, scale and view direction are recomputed from the
// parameters.  Gradients are accumulated (+=) into the caller's buffers, or
// written (CS_GRADS_OVERWRITE).
#include "common.cuh"

namespace cs {

// harmonics.py:7-24 constants (fp32: the SH VJP is continuous and small)
constexpr float kC0 = 0.28209479177387814f, kC1 = 0.4886025119029199f;
constexpr float kC20 = 1.0925484305920792f, kC21 = -1.0925484305920792f, kC22 = 0.31539156525252005f,
                kC23 = -1.0925484305920792f, kC24 = 0.5462742152960396f;
constexpr float kC30 = -0.5900435899266435f, kC31 = 2.890611442640554f, kC32 = -0.4570457994644658f,
                kC33 = 0.3731763325901154f, kC34 = -0.4570457994644658f, kC35 = 1.445305721320277f,
                kC36 = -0.5900435899266435f;

struct ChainArgs {
  cs_camera cam;
  int64_t n;
  int k, sh_degree, mode;
  double cam_center[3];
  const float *points, *raw_delta, *raw_sigma, *raw_opacity, *raw_mask, *sh;
  const float *records;
  const AccT *accum;
  const uint8_t *hull;
  const uint32_t *touched;
  cs_grads g;
  cs_view_signal sig;   // sigma_signal == nullptr: no densification signal
  uint32_t *nonfinite;  // workspace counter C_NONFINITE: set when a gradient row is not finite
  int64_t first;        // convexes [first, n) (a range: cs_backward_chain_range)
};

#ifndef CS_CHAIN_THREADS
#define CS_CHAIN_THREADS 64   // 64 / 128 threads: 235 / 238 us (also keeps CS_CHAIN_F64's smem under 48 KB)
#endif
template <int MAXK> __host__ __device__ constexpr int chain_threads() {
  return MAXK <= 8 ? CS_CHAIN_THREADS : CS_CHAIN_THREADS / 2;
}
#ifndef CS_CHAIN_MINB
#define CS_CHAIN_MINB (640 / CS_CHAIN_THREADS)   // the SH staging limits it anyway
#endif

// Accumulation into the caller's gradient buffers (+=, GradientBuffer.add).
// Every convex has one owning thread, so these need no atomicity; they are
// issued as fire-and-forget L2 reductions (RED) so the SM never waits for the
// read half of a read-modify-write of ~0.7 KB per convex.
__device__ __forceinline__ void red_add(float *p, float v) {
  asm volatile("red.global.add.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
}
// Gradient output: += (RED) or, with CS_GRADS_OVERWRITE, a plain store (the
// caller's buffers are written, not read: no zeroing pass, no read half).
template <bool OW> __device__ __forceinline__ void grad_out(float *p, float v) {
  if (OW) *p = v; else red_add(p, v);
}

// d(Y_b)/d(dir) . v_b added into (gx, gy, gz): eval_sh_basis_grad
// (harmonics.py:62-98) row b, written out (b is a compile-time constant).
__device__ __forceinline__ void add_basis_grad(int b, float v, float x, float y, float z, float &gx, float &gy,
                                               float &gz) {
  const float xx = x * x, yy = y * y, zz = z * z;
  switch (b) {
    case 1: gy -= kC1 * v; break;
    case 2: gz += kC1 * v; break;
    case 3: gx -= kC1 * v; break;
    case 4: gx += kC20 * y * v; gy += kC20 * x * v; break;
    case 5: gy += kC21 * z * v; gz += kC21 * y * v; break;
    case 6: gx += -2.0f * kC22 * x * v; gy += -2.0f * kC22 * y * v; gz += 4.0f * kC22 * z * v; break;
    case 7: gx += kC23 * z * v; gz += kC23 * x * v; break;
    case 8: gx += 2.0f * kC24 * x * v; gy += -2.0f * kC24 * y * v; break;
    case 9: gx += kC30 * 6.0f * x * y * v; gy += kC30 * 3.0f * (xx - yy) * v; break;
    case 10: gx += kC31 * y * z * v; gy += kC31 * x * z * v; gz += kC31 * x * y * v; break;
    case 11:
      gx += -2.0f * kC32 * x * y * v; gy += kC32 * (4.0f * zz - xx - 3.0f * yy) * v; gz += 8.0f * kC32 * y * z * v;
      break;
    case 12:
      gx += -6.0f * kC33 * x * z * v; gy += -6.0f * kC33 * y * z * v; gz += kC33 * (6.0f * zz - 3.0f * xx - 3.0f * yy) * v;
      break;
    case 13:
      gx += kC34 * (4.0f * zz - 3.0f * xx - yy) * v; gy += -2.0f * kC34 * x * y * v; gz += 8.0f * kC34 * x * z * v;
      break;
    case 14: gx += 2.0f * kC35 * x * z * v; gy += -2.0f * kC35 * y * z * v; gz += kC35 * (xx - yy) * v; break;
    case 15: gx += kC36 * 3.0f * (xx - yy) * v; gy += -6.0f * kC36 * x * y * v; break;
    default: break;
  }
}

// SH colour VJP (harmonics.py:112-128): d_sh = Y (x) d_eff and the
// direction gradient dY/ddir^T (sh . d_eff), on the convex's SH row staged
// in shared memory (`row`, 48 floats, loaded by a bulk copy at kernel
// start): d_sh is written back into the row in place and leaves by one bulk
// store (overwrite) or bulk float reduction (+=).
__device__ __forceinline__ void sh_vjp_row(float x, float y, float z, int deg, float *row, const float *d_color,
                                           float *ddir) {
  float Y[kShCoeffs];
  Y[0] = kC0;
  const float xx = x * x, yy = y * y, zz = z * z;
#pragma unroll
  for (int b = 1; b < kShCoeffs; b++) Y[b] = 0.f;
  if (deg >= 1) { Y[1] = -kC1 * y; Y[2] = kC1 * z; Y[3] = -kC1 * x; }
  if (deg >= 2) {
    Y[4] = kC20 * x * y; Y[5] = kC21 * y * z; Y[6] = kC22 * (2.0f * zz - xx - yy);
    Y[7] = kC23 * x * z; Y[8] = kC24 * (xx - yy);
  }
  if (deg >= 3) {
    Y[9] = kC30 * y * (3.0f * xx - yy); Y[10] = kC31 * x * y * z; Y[11] = kC32 * y * (4.0f * zz - xx - yy);
    Y[12] = kC33 * z * (2.0f * zz - 3.0f * xx - 3.0f * yy); Y[13] = kC34 * x * (4.0f * zz - xx - yy);
    Y[14] = kC35 * z * (xx - yy); Y[15] = kC36 * x * (xx - 3.0f * yy);
  }
  const int nb = (deg + 1) * (deg + 1);
  float4 *row4 = reinterpret_cast<float4 *>(row);
  float raw[3] = {0.5f, 0.5f, 0.5f};
#pragma unroll
  for (int q = 0; q < kShCoeffs * 3 / 4; q++) {
    if (4 * q < 3 * nb) {
      const float4 v = row4[q];
      const float e[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int r = 0; r < 4; r++) {
        const int f = 4 * q + r, b = f / 3, c = f % 3;
        if (b < nb) raw[c] = fmaf(Y[b], e[r], raw[c]);
      }
    }
  }
  float deff[3];
#pragma unroll
  for (int c = 0; c < 3; c++) deff[c] = raw[c] > 0.f ? d_color[c] : 0.f;
  float gx = 0.0f, gy = 0.0f, gz = 0.0f, vb = 0.0f;
#pragma unroll
  for (int q = 0; q < kShCoeffs * 3 / 4; q++) {
    float de[4] = {0.f, 0.f, 0.f, 0.f};
    if (4 * q < 3 * nb) {
      const float4 v = row4[q];
      const float e[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int r = 0; r < 4; r++) {
        const int f = 4 * q + r, b = f / 3, c = f % 3;
        if (b < nb) {
          de[r] = Y[b] * deff[c];
          vb = fmaf(e[r], deff[c], vb);
          if (c == 2) {
            add_basis_grad(b, vb, x, y, z, gx, gy, gz);
            vb = 0.0f;
          }
        }
      }
    }
    row4[q] = make_float4(de[0], de[1], de[2], de[3]);   // zeros above sh_degree
  }
  ddir[0] = gx; ddir[1] = gy; ddir[2] = gz;
}

// Geometry precision of the chain.  float32 by default; -DCS_CHAIN_F64 for A/B.
#ifdef CS_CHAIN_F64
typedef double G;
__device__ __forceinline__ G g_rcp(G x) { return __drcp_rn(x); }
__device__ __forceinline__ G g_rsqrt(G x) { return rsqrt(x); }
#else
typedef float G;
__device__ __forceinline__ G g_rcp(G x) { return __frcp_rn(x); }
__device__ __forceinline__ G g_rsqrt(G x) { return rsqrtf(x); }
#endif

#if defined(CS_CHAIN_ACC_F64) && !defined(CS_ACC_F32)
typedef double AccR;
#else
typedef float AccR;
#endif

template <int MAXK, bool OW>
__global__ void __launch_bounds__(chain_threads<MAXK>(), CS_CHAIN_MINB) chain_kernel(ChainArgs a) {
  constexpr int kChainThreads = chain_threads<MAXK>();
  // per-thread slots for the dynamically indexed per-point arrays
  __shared__ G s_x[MAXK][kChainThreads], s_y[MAXK][kChainThreads];
  __shared__ G s_dx[MAXK][kChainThreads], s_dy[MAXK][kChainThreads];
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const int64_t i = a.first + (int64_t)blockIdx.x * kChainThreads + t;
  constexpr int RF = Rec<MAXK>::kGlobal;
  constexpr int AF = Acc<MAXK>::kFloats;
  constexpr int kShRow = kShCoeffs * 3;
  // SH rows: one 192-byte bulk copy per prepared convex, issued first so it
  // lands while the geometry is recomputed; 208-byte slots keep the per-lane
  // float4 reads free of bank conflicts
  constexpr int kShStride = kShRow + 4;
  __shared__ __align__(16) float s_sh[kChainThreads * kShStride];
  __shared__ __align__(8) uint64_t s_shbar[kChainThreads / 32];
  float *const shrow = s_sh + t * kShStride;
  const bool active = i < a.n && a.touched[i] != 0;
  {
    const uint32_t act = __ballot_sync(0xffffffffu, active);
    if (lane == 0) {
      mbar_init(&s_shbar[w], 1);
      fence_mbar_init();
      if (act) mbar_expect_tx(&s_shbar[w], (uint32_t)__popc(act) * kShRow * 4);
    }
    __syncwarp();
    if (active) tma_bulk_g2s(shrow, a.sh + i * kShRow, kShRow * 4, &s_shbar[w]);
  }
  if (i >= a.n) return;
  if (!active) {   // not prepared for this view: zero gradient
    if (OW) {
      for (int q = 0; q < 3 * a.k; q++) a.g.d_points[i * 3 * a.k + q] = 0.f;
      float4 *dsh4 = reinterpret_cast<float4 *>(a.g.d_sh + i * kShRow);
#pragma unroll
      for (int q = 0; q < kShRow / 4; q++) dsh4[q] = make_float4(0.f, 0.f, 0.f, 0.f);
      a.g.d_raw_delta[i] = 0.f; a.g.d_raw_sigma[i] = 0.f; a.g.d_raw_opacity[i] = 0.f; a.g.d_raw_mask[i] = 0.f;
    }
    return;
  }
  const int k = a.k;
  const G inv_k = G(1) / (G)k;
  // the convex's screen-space accumulators, loaded up front (float64 sums
  // rounded once to the chain's float32 arithmetic; -DCS_CHAIN_ACC_F64 keeps
  // them in float64)
  AccR acc[AF];
  {
#ifndef CS_ACC_F32
    const double2 *acc2 = reinterpret_cast<const double2 *>(a.accum + i * AF);
#pragma unroll
    for (int q = 0; q < AF / 2; q++) {
      const double2 v = __ldg(acc2 + q);
      acc[2 * q] = (AccR)v.x; acc[2 * q + 1] = (AccR)v.y;
    }
#else
    const float4 *acc4 = reinterpret_cast<const float4 *>(a.accum + i * AF);
#pragma unroll
    for (int q = 0; q < AF / 4; q++) {
      const float4 v = __ldg(acc4 + q);
      acc[4 * q] = v.x; acc[4 * q + 1] = v.y; acc[4 * q + 2] = v.z; acc[4 * q + 3] = v.w;
    }
#endif
  }
  // every other per-convex input is loaded up front too (one exposed
  // latency instead of a chain of them)
  float pts[MAXK * 3];
  {
    const float *pp = a.points + i * k * 3;
    if ((k & 1) == 0) {   // rows of 12k bytes: 8-byte aligned for even k, 6k float2 loads
      const float2 *pp2 = reinterpret_cast<const float2 *>(pp);
#pragma unroll
      for (int q = 0; q < MAXK * 3 / 2; q++) {
        const float2 v = 2 * q < 3 * k ? __ldg(pp2 + q) : make_float2(0.f, 0.f);
        pts[2 * q] = v.x;
        pts[2 * q + 1] = v.y;
      }
    } else {
#pragma unroll
      for (int q = 0; q < MAXK * 3; q++) pts[q] = q < 3 * k ? __ldg(pp + q) : 0.f;
    }
  }
  const float raw_delta = __ldg(a.raw_delta + i), raw_sigma = __ldg(a.raw_sigma + i);
  const float raw_opacity = __ldg(a.raw_opacity + i), raw_mask = __ldg(a.raw_mask + i);
  uint8_t hb[MAXK];
  if (MAXK == 8) {
    const uint2 hw = __ldg(reinterpret_cast<const uint2 *>(a.hull + i * MAXK));
#pragma unroll
    for (int j = 0; j < 4; j++) { hb[j] = (hw.x >> (8 * j)) & 0xff; hb[j + 4] = (hw.y >> (8 * j)) & 0xff; }
  } else {
#pragma unroll
    for (int j = 0; j < MAXK; j++) hb[j] = a.hull[i * MAXK + j];
  }
  const float2 anchor = __ldg(reinterpret_cast<const float2 *>(a.records + i * RF));
  G R[9];
#pragma unroll
  for (int q = 0; q < 9; q++) R[q] = (G)a.cam.R[q];
  const G fx = (G)a.cam.fx, fy = (G)a.cam.fy;
  // recompute the projection (projection.py:22-40) in float64 and keep the
  // projected points RELATIVE TO THE ANCHOR (ax, ay): the hull normals and
  // the line -> vertex Jacobian then see small coordinates, so float32 keeps
  // ~1e-6 px where absolute 1080p coordinates would only keep ~6e-5 px.
  const double *Rd = a.cam.R;
  const double ox = a.cam.cx - (double)anchor.x, oy = a.cam.cy - (double)anchor.y;
  G zsum = 0, cx = 0, cy = 0, cz = 0;
  G izc[MAXK];
#pragma unroll
  for (int j = 0; j < MAXK; j++) {
    if (j < k) {
      const float q0 = pts[3 * j], q1 = pts[3 * j + 1], q2 = pts[3 * j + 2];
      cx += q0; cy += q1; cz += q2;
      const double p0 = q0, p1 = q1, p2 = q2;
      const double xc = fma(p2, Rd[2], fma(p1, Rd[1], p0 * Rd[0])) + a.cam.t[0];
      const double yc = fma(p2, Rd[5], fma(p1, Rd[4], p0 * Rd[3])) + a.cam.t[1];
      const double zc = fma(p2, Rd[8], fma(p1, Rd[7], p0 * Rd[6])) + a.cam.t[2];
      zsum += (G)zc;
      if (a.cam.ortho) {
        s_x[j][t] = (G)fma(a.cam.fx, xc, ox);
        s_y[j][t] = (G)fma(a.cam.fy, yc, oy);
        izc[j] = 0;
      } else {
        const double iz = __drcp_rn(zc);
        izc[j] = (G)iz;
        s_x[j][t] = (G)fma(a.cam.fx * xc, iz, ox);
        s_y[j][t] = (G)fma(a.cam.fy * yc, iz, oy);
      }
      s_dx[j][t] = 0;
      s_dy[j][t] = 0;
    }
  }
  int h = 0;
#pragma unroll
  for (int j = 0; j < MAXK; j++) h += hb[j] != 0xff;
  // lines -> hull vertices (backward.py:231-246)
#pragma unroll
  for (int j = 0; j < MAXK; j++) {
    if (j < h) {
      int v = hb[0];
#pragma unroll
      for (int q = 1; q < MAXK; q++)
        if (q == j + 1) v = q < h ? hb[q] : hb[0];
      const int u = hb[j];
      const G ux = s_x[u][t], uy = s_y[u][t];
      const G ex = s_x[v][t] - ux, ey = s_y[v][t] - uy;
      const G il = g_rsqrt(fma(ex, ex, ey * ey));
      const G nx = ey * il, ny = -ex * il;
      const G gs = (G)acc[A_LINES + 3 * j + 2];
      // reference gn = sum dL*q - gs*v = sum dL*(q-a) - gs*(v-a); u is anchor-relative
      // (the cancellation of the two sums is formed in the accumulator type)
      const G gx = (G)fma(-acc[A_LINES + 3 * j + 2], (AccR)ux, acc[A_LINES + 3 * j]);
      const G gy = (G)fma(-acc[A_LINES + 3 * j + 2], (AccR)uy, acc[A_LINES + 3 * j + 1]);
      const G nd = fma(nx, gx, ny * gy);
      const G rx = (gx - nx * nd) * il, ry = (gy - ny * nd) * il;
      s_dx[v][t] += -ry;
      s_dy[v][t] += rx;
      s_dx[u][t] += ry - nx * gs;
      s_dy[u][t] += -rx - ny * gs;
    }
  }
  const float dcol[3] = {(float)acc[A_DC], (float)acc[A_DC + 1], (float)acc[A_DC + 2]};
  // depth, scale and activations (rasterize.py:99-103, field.py:26-48)
  const G depth = zsum * inv_k;
  const G dsc = a.cam.ortho ? G(1) : depth;
  G s, sgrad;
  switch (a.mode) {
    case CS_SCALE_NONE: s = 1; sgrad = 0; break;
    case CS_SCALE_SQRT: s = sqrt(dsc); sgrad = G(0.5) * g_rsqrt(depth); break;
    case CS_SCALE_DEPTH: s = dsc; sgrad = 1; break;
    default: s = dsc * dsc; sgrad = G(2) * depth; break;
  }
  const G delta = exp((G)raw_delta), sigma = exp((G)raw_sigma);
  const G ddel = (G)acc[A_DDEL], dsig = (G)acc[A_DSIG];
  const G d_depth = a.cam.ortho ? G(0) : (ddel * delta + dsig * sigma) * sgrad;
  // view direction (rasterize.py:110-113) and SH VJP (harmonics.py:112-128)
  const float fk = 1.f / (float)k;
  const float vx = (float)cx * fk - (float)a.cam_center[0], vy = (float)cy * fk - (float)a.cam_center[1],
              vz = (float)cz * fk - (float)a.cam_center[2];
  const float d2 = fmaf(vx, vx, fmaf(vy, vy, vz * vz));
  const float idist = d2 > 0.f ? rsqrtf(d2) : 0.f;
  float dir[3] = {0.f, 0.f, 1.f};
  if (d2 > 0.f) { dir[0] = vx * idist; dir[1] = vy * idist; dir[2] = vz * idist; }
  float ddirf[3];
  mbar_wait(&s_shbar[w], 0);
  sh_vjp_row(dir[0], dir[1], dir[2], a.sh_degree, shrow, dcol, ddirf);
  fence_proxy_async_smem();
  if (OW) tma_bulk_s2g(a.g.d_sh + i * kShRow, shrow, kShRow * 4);
  else tma_bulk_s2g_add(a.g.d_sh + i * kShRow, shrow, kShRow * 4);
  const float dot = dir[0] * ddirf[0] + dir[1] * ddirf[1] + dir[2] * ddirf[2];
  // projection Jacobian + depth + centre paths into d_points (backward.py:248-269, 281-282)
  G common[3];
#pragma unroll
  for (int c = 0; c < 3; c++) common[c] = (d_depth * R[6 + c] + (G)((ddirf[c] - dir[c] * dot) * idist)) * inv_k;
  float *dp = a.g.d_points + i * k * 3;
  // non-finite check: inf/NaN in any input reaches the
  // accumulators or the per-point terms, and then this sum
  float chk = 0.f;
#pragma unroll
  for (int q = 0; q < AF; q++) chk += (float)acc[q];
#pragma unroll
  for (int j = 0; j < MAXK; j++) {
    if (j < k) {
      const G gx = s_dx[j][t], gy = s_dy[j][t];
      G d0, d1, dz;
      if (a.cam.ortho) {
        d0 = fx * gx; d1 = fy * gy; dz = 0;
      } else {
        d0 = fx * izc[j] * gx;
        d1 = fy * izc[j] * gy;
        // fx x / z^2 = (px - cx) / z, px - cx = (px - ax) - (cx - ax)
        dz = -((s_x[j][t] - (G)ox) * gx + (s_y[j][t] - (G)oy) * gy) * izc[j];
      }
#pragma unroll
      for (int c = 0; c < 3; c++) {
        const float g = (float)fma(d0, R[c], fma(d1, R[3 + c], fma(dz, R[6 + c], common[c])));
        chk += g;
        grad_out<OW>(dp + 3 * j + c, g);
      }
    }
  }
  grad_out<OW>(a.g.d_raw_delta + i, (float)(ddel * s * delta));
  const float d_rs = (float)(dsig * s * sigma);
  grad_out<OW>(a.g.d_raw_sigma + i, d_rs);
  if (a.sig.sigma_signal) {   // trainer.py:192-193, this view's contribution only
    const float vis = a.sig.visible[i] ? 1.f : 0.f;
    red_add(a.sig.sigma_signal + i, fabsf(d_rs) * vis);
    red_add(a.sig.sigma_views + i, vis);
  }
  const float o = 1.f / (1.f + __expf(-raw_opacity));
  const float m = 1.f / (1.f + __expf(-raw_mask));
  const float doe = (float)acc[A_DOEFF];
  grad_out<OW>(a.g.d_raw_opacity + i, doe * o * (1.f - o));
  grad_out<OW>(a.g.d_raw_mask + i, doe * o * m * (1.f - m));
  chk += d_rs + (float)(ddel * s * delta) + o + m + dot;
  if (!isfinite(chk)) atomicOr(a.nonfinite, 1u);
  tma_bulk_commit_and_wait_read();   // the d_sh row has left shared memory
}

int launch_chain(const cs_camera &cam, const cs_settings &set, const cs_params &p,
                 const cs_layout &L, char *ws, const cs_grads &g, const cs_view_signal *sig, bool overwrite,
                 cudaStream_t s, int64_t first, int64_t last) {
  if (last < 0 || last > p.n) last = p.n;
  if (first < 0) first = 0;
  if (last <= first) return CS_OK;
  ChainArgs a;
  a.cam = cam;
  a.n = last;
  a.first = first;
  a.k = p.k;
  a.sh_degree = set.sh_degree;
  a.mode = set.scaling_mode;
  for (int j = 0; j < 3; j++) {
    double c = 0.0;
    for (int r = 0; r < 3; r++) c += (-cam.R[3 * r + j]) * cam.t[r];
    a.cam_center[j] = c;
  }
  a.points = p.points; a.raw_delta = p.raw_delta; a.raw_sigma = p.raw_sigma;
  a.raw_opacity = p.raw_opacity; a.raw_mask = p.raw_mask; a.sh = p.sh;
  a.records = reinterpret_cast<const float *>(ws + L.records);
  a.accum = reinterpret_cast<const AccT *>(ws + L.grad_accum);
  a.hull = reinterpret_cast<const uint8_t *>(ws + L.hull);
  a.touched = reinterpret_cast<const uint32_t *>(ws + L.tiles_touched);
  a.g = g;
  a.sig = sig ? *sig : cs_view_signal{nullptr, nullptr, nullptr};
  a.nonfinite = reinterpret_cast<uint32_t *>(ws + L.counters) + C_NONFINITE;
  if (L.max_k == 8) {
    if (overwrite) chain_kernel<8, true><<<(int)((last - first + chain_threads<8>() - 1) / chain_threads<8>()), chain_threads<8>(), 0, s>>>(a);
    else chain_kernel<8, false><<<(int)((last - first + chain_threads<8>() - 1) / chain_threads<8>()), chain_threads<8>(), 0, s>>>(a);
  } else {
    if (overwrite) chain_kernel<16, true><<<(int)((last - first + chain_threads<16>() - 1) / chain_threads<16>()), chain_threads<16>(), 0, s>>>(a);
    else chain_kernel<16, false><<<(int)((last - first + chain_threads<16>() - 1) / chain_threads<16>()), chain_threads<16>(), 0, s>>>(a);
  }
  return cudaGetLastError() == cudaSuccess ? CS_OK : CS_ERR_CUDA;
}

}  // namespace cs
