// K4b: per-convex gradient chain (backward.py:215-282), one thread per convex.
//
// Turns the screen-space accumulators of the backward blend into gradients of
// the raw parameters, in float64:
//   hull lines -> hull vertices (normalisation Jacobian, backward.py:231-246)
//   -> projection Jacobian -> 3-D points (backward.py:248-261)
//   delta/sigma activations + the depth path (backward.py:263-269)
//   opacity and straight-through mask (backward.py:271-275)
//   SH VJP + view-direction path (backward.py:277-282, harmonics.py:112-128)
// Discrete state (hull cycle, anchor) is read from the forward workspace;
// projection, depth, scale and view direction are recomputed from the
// parameters.  Gradients are accumulated (+=) into the caller's buffers.
#include "common.cuh"

namespace cs {

__constant__ double kC0 = 0.28209479177387814;
__constant__ double kC1 = 0.4886025119029199;
__constant__ double kC2[5] = {1.0925484305920792, -1.0925484305920792, 0.31539156525252005,
                              -1.0925484305920792, 0.5462742152960396};
__constant__ double kC3[7] = {-0.5900435899266435, 2.890611442640554, -0.4570457994644658,
                              0.3731763325901154, -0.4570457994644658, 1.445305721320277,
                              -0.5900435899266435};

// harmonics.py:33-59 (basis) and :62-98 (gradient rows)
__device__ void sh_basis_and_grad(double x, double y, double z, int deg, double *b, double (*g)[3]) {
  for (int i = 0; i < kShCoeffs; i++) { b[i] = 0.0; g[i][0] = g[i][1] = g[i][2] = 0.0; }
  b[0] = kC0;
  if (deg >= 1) {
    b[1] = -kC1 * y; b[2] = kC1 * z; b[3] = -kC1 * x;
    g[1][1] = -kC1; g[2][2] = kC1; g[3][0] = -kC1;
  }
  const double xx = x * x, yy = y * y, zz = z * z;
  if (deg >= 2) {
    b[4] = kC2[0] * x * y;
    b[5] = kC2[1] * y * z;
    b[6] = kC2[2] * (2.0 * zz - xx - yy);
    b[7] = kC2[3] * x * z;
    b[8] = kC2[4] * (xx - yy);
    g[4][0] = kC2[0] * y; g[4][1] = kC2[0] * x;
    g[5][1] = kC2[1] * z; g[5][2] = kC2[1] * y;
    g[6][0] = -2.0 * kC2[2] * x; g[6][1] = -2.0 * kC2[2] * y; g[6][2] = 4.0 * kC2[2] * z;
    g[7][0] = kC2[3] * z; g[7][2] = kC2[3] * x;
    g[8][0] = 2.0 * kC2[4] * x; g[8][1] = -2.0 * kC2[4] * y;
  }
  if (deg >= 3) {
    b[9] = kC3[0] * y * (3.0 * xx - yy);
    b[10] = kC3[1] * x * y * z;
    b[11] = kC3[2] * y * (4.0 * zz - xx - yy);
    b[12] = kC3[3] * z * (2.0 * zz - 3.0 * xx - 3.0 * yy);
    b[13] = kC3[4] * x * (4.0 * zz - xx - yy);
    b[14] = kC3[5] * z * (xx - yy);
    b[15] = kC3[6] * x * (xx - 3.0 * yy);
    g[9][0] = kC3[0] * 6.0 * x * y; g[9][1] = kC3[0] * 3.0 * (xx - yy);
    g[10][0] = kC3[1] * y * z; g[10][1] = kC3[1] * x * z; g[10][2] = kC3[1] * x * y;
    g[11][0] = -2.0 * kC3[2] * x * y; g[11][1] = kC3[2] * (4.0 * zz - xx - 3.0 * yy); g[11][2] = 8.0 * kC3[2] * y * z;
    g[12][0] = -6.0 * kC3[3] * x * z; g[12][1] = -6.0 * kC3[3] * y * z;
    g[12][2] = kC3[3] * (6.0 * zz - 3.0 * xx - 3.0 * yy);
    g[13][0] = kC3[4] * (4.0 * zz - 3.0 * xx - yy); g[13][1] = -2.0 * kC3[4] * x * y; g[13][2] = 8.0 * kC3[4] * x * z;
    g[14][0] = 2.0 * kC3[5] * x * z; g[14][1] = -2.0 * kC3[5] * y * z; g[14][2] = kC3[5] * (xx - yy);
    g[15][0] = kC3[6] * 3.0 * (xx - yy); g[15][1] = -6.0 * kC3[6] * x * y;
  }
}

struct ChainArgs {
  cs_camera cam;
  int64_t n;
  int k, sh_degree, mode;
  double cam_center[3];
  const float *points, *raw_delta, *raw_sigma, *raw_opacity, *raw_mask, *sh;
  const float *records, *accum;
  const uint8_t *hull;
  const uint32_t *touched;
  cs_grads g;
};

template <int MAXK>
__global__ void __launch_bounds__(128) chain_kernel(ChainArgs a) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.n || a.touched[i] == 0) return;  // not prepared for this view
  constexpr int RF = Rec<MAXK>::kFloats;
  constexpr int AF = Acc<MAXK>::kFloats;
  const int k = a.k;
  const float *acc = a.accum + i * AF;
  const float *rec = a.records + i * RF;
  const uint8_t *hull = a.hull + i * MAXK;
  const double *R = a.cam.R;
  // recompute the projection (projection.py:22-40)
  double X[MAXK], Y[MAXK], xc[MAXK], yc[MAXK], zc[MAXK];
  double zsum = 0.0, cx = 0.0, cy = 0.0, cz = 0.0;
  for (int j = 0; j < k; j++) {
    const float *pp = a.points + (i * k + j) * 3;
    double p0 = pp[0], p1 = pp[1], p2 = pp[2];
    cx += p0; cy += p1; cz += p2;
    xc[j] = fma(p2, R[2], fma(p1, R[1], p0 * R[0])) + a.cam.t[0];
    yc[j] = fma(p2, R[5], fma(p1, R[4], p0 * R[3])) + a.cam.t[1];
    zc[j] = fma(p2, R[8], fma(p1, R[7], p0 * R[6])) + a.cam.t[2];
    zsum += zc[j];
    if (a.cam.ortho) {
      X[j] = a.cam.fx * xc[j] + a.cam.cx;
      Y[j] = a.cam.fy * yc[j] + a.cam.cy;
    } else {
      X[j] = (a.cam.fx * xc[j]) / zc[j] + a.cam.cx;
      Y[j] = (a.cam.fy * yc[j]) / zc[j] + a.cam.cy;
    }
  }
  int h = 0;
  while (h < MAXK && hull[h] != 0xff) h++;
  const double ax = rec[R_AX], ay = rec[R_AY];
  // lines -> hull vertices (backward.py:231-246)
  double dpx[MAXK], dpy[MAXK];
  for (int j = 0; j < k; j++) dpx[j] = dpy[j] = 0.0;
  for (int j = 0; j < h; j++) {
    const int u = hull[j], v = hull[(j + 1) % h];
    const double ex = X[v] - X[u], ey = Y[v] - Y[u];
    const double len = hypot(ey, ex);
    const double nx = ey / len, ny = -ex / len;
    const double gs = acc[A_LINES + 3 * j + 2];
    // reference gn = sum dL*q - gs*v = sum dL*(q-a) + gs*(a - v)
    const double gx = acc[A_LINES + 3 * j] + gs * (ax - X[u]);
    const double gy = acc[A_LINES + 3 * j + 1] + gs * (ay - Y[u]);
    const double nd = nx * gx + ny * gy;
    const double rx = (gx - nx * nd) / len, ry = (gy - ny * nd) / len;
    const double dex = -ry, dey = rx;
    dpx[v] += dex; dpy[v] += dey;
    dpx[u] += -dex - nx * gs; dpy[u] += -dey - ny * gs;
  }
  // depth, scale and activations (rasterize.py:99-103, field.py:26-48)
  const double depth = zsum / k;
  const double dsc = a.cam.ortho ? 1.0 : depth;
  double s, sgrad;
  switch (a.mode) {
    case CS_SCALE_NONE: s = 1.0; sgrad = 0.0; break;
    case CS_SCALE_SQRT: s = sqrt(dsc); sgrad = 0.5 / sqrt(depth); break;
    case CS_SCALE_DEPTH: s = dsc; sgrad = 1.0; break;
    default: s = dsc * dsc; sgrad = 2.0 * depth; break;
  }
  const double delta = exp((double)a.raw_delta[i]), sigma = exp((double)a.raw_sigma[i]);
  const double ddel = acc[A_DDEL], dsig = acc[A_DSIG];
  const double d_depth = a.cam.ortho ? 0.0 : (ddel * delta + dsig * sigma) * sgrad;
  // view direction (rasterize.py:110-113)
  const double vx = cx / k - a.cam_center[0], vy = cy / k - a.cam_center[1], vz = cz / k - a.cam_center[2];
  const double dist = sqrt(vx * vx + vy * vy + vz * vz);
  double dir[3] = {0.0, 0.0, 1.0};
  if (dist > 0.0) { dir[0] = vx / dist; dir[1] = vy / dist; dir[2] = vz / dist; }
  // SH VJP (harmonics.py:112-128)
  double basis[kShCoeffs], bg[kShCoeffs][3];
  sh_basis_and_grad(dir[0], dir[1], dir[2], a.sh_degree, basis, bg);
  const int nb = (a.sh_degree + 1) * (a.sh_degree + 1);
  const float *sh = a.sh + i * kShCoeffs * 3;
  double deff[3];
  for (int c = 0; c < 3; c++) {
    double raw = 0.0;
    for (int b = 0; b < nb; b++) raw += basis[b] * (double)sh[3 * b + c];
    deff[c] = (0.5 + raw) > 0.0 ? (double)acc[A_DC + c] : 0.0;
  }
  float *dsh = a.g.d_sh + i * kShCoeffs * 3;
  double ddir[3] = {0.0, 0.0, 0.0};
  for (int b = 0; b < nb; b++) {
    double vb = 0.0;
    for (int c = 0; c < 3; c++) {
      dsh[3 * b + c] += (float)(basis[b] * deff[c]);
      vb += (double)sh[3 * b + c] * deff[c];
    }
    for (int q = 0; q < 3; q++) ddir[q] += bg[b][q] * vb;
  }
  const double dot = dir[0] * ddir[0] + dir[1] * ddir[1] + dir[2] * ddir[2];
  double dcen[3];
  for (int q = 0; q < 3; q++) dcen[q] = dist > 0.0 ? (ddir[q] - dir[q] * dot) / dist : 0.0;
  // projection Jacobian + depth + centre paths into d_points (backward.py:248-269, 281-282)
  float *dp = a.g.d_points + i * k * 3;
  for (int j = 0; j < k; j++) {
    double d0, d1, d2;
    if (a.cam.ortho) {
      d0 = a.cam.fx * dpx[j]; d1 = a.cam.fy * dpy[j]; d2 = 0.0;
    } else {
      const double z = zc[j];
      d0 = a.cam.fx / z * dpx[j];
      d1 = a.cam.fy / z * dpy[j];
      d2 = -(a.cam.fx * xc[j] / (z * z)) * dpx[j] - (a.cam.fy * yc[j] / (z * z)) * dpy[j];
    }
    for (int c = 0; c < 3; c++) {
      double v = d0 * R[c] + d1 * R[3 + c] + d2 * R[6 + c];
      v += d_depth * R[6 + c] / k;
      v += dcen[c] / k;
      dp[3 * j + c] += (float)v;
    }
  }
  a.g.d_raw_delta[i] += (float)(ddel * s * delta);
  a.g.d_raw_sigma[i] += (float)(dsig * s * sigma);
  const double o = 1.0 / (1.0 + exp(-(double)a.raw_opacity[i]));
  const double m = 1.0 / (1.0 + exp(-(double)a.raw_mask[i]));
  const double doe = acc[A_DOEFF];
  a.g.d_raw_opacity[i] += (float)(doe * o * (1.0 - o));
  a.g.d_raw_mask[i] += (float)(doe * o * m * (1.0 - m));
}

int launch_chain(const cs_camera &cam, const cs_settings &set, const cs_params &p,
                 const cs_layout &L, char *ws, const cs_grads &g, cudaStream_t s) {
  if (p.n == 0) return CS_OK;
  ChainArgs a;
  a.cam = cam;
  a.n = p.n;
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
  a.accum = reinterpret_cast<const float *>(ws + L.grad_accum);
  a.hull = reinterpret_cast<const uint8_t *>(ws + L.hull);
  a.touched = reinterpret_cast<const uint32_t *>(ws + L.tiles_touched);
  a.g = g;
  const int blocks = (int)((p.n + 127) / 128);
  if (L.max_k == 8)
    chain_kernel<8><<<blocks, 128, 0, s>>>(a);
  else
    chain_kernel<16><<<blocks, 128, 0, s>>>(a);
  return cudaGetLastError() == cudaSuccess ? CS_OK : CS_ERR_CUDA;
}

}  // namespace cs
