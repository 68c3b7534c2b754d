// Training-step kernels on either side of the rasterizer:
//
//   image loss  losses.image_loss (losses.py:129-155) with ssim_with_grad
//               (losses.py:58-101): L1 + D-SSIM (11x11, sigma 1.5, valid
//               window) + mask sparsity, value and d_image in two passes:
//                 ssim_moments_kernel  windowed moments -> SSIM map (summed)
//                                      and the three adjoint coefficient maps
//                 ssim_adjoint_kernel  transposed window over the maps, plus
//                                      the L1 sign term -> d_image; L1 sum
//               The moments are taken of x - 1/2, y - 1/2 (variances are
//               shift-invariant; float32 then keeps ~4x more bits of sxx).
//   mask term   mean(sigmoid(raw_mask)) and its gradient (losses.py:146-151)
//   Adam        optim.Adam.step (optim.py:22-35), one launch for all tensors
#include <cmath>

#include "common.cuh"

namespace cs {

constexpr int kWin = 11;              // losses.py:16 SSIM_WINDOW
constexpr int kHalo = kWin - 1;
constexpr float kC1 = 0.01f * 0.01f;  // losses.py:18-19
constexpr float kC2 = 0.03f * 0.03f;
// gaussian_window() (losses.py:22-25), passed by value (no per-device state)
struct Win {
  float w[kWin];
};

constexpr int kLossTW = 32, kLossTH = 16, kLossThreads = 256;

__device__ __forceinline__ void atomic_add_block_sum(double *dst, double v) {
  __shared__ double s_part[kLossThreads / 32];
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) s_part[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < kLossThreads / 32; w++) t += s_part[w];
    atomicAdd(dst, t);
  }
}

// One 32x16 tile of the valid grid of one channel (blockIdx.z).  maps:
// [3 channels][3: dMx, dVxx, dVxy][Hv*Wv], scaled by 1/(3 Hv Wv).
__global__ void __launch_bounds__(kLossThreads) ssim_moments_kernel(int H, int W, const float *img, const float *tgt,
                                                                    float *maps, double *stats, Win win) {
  constexpr int RW = kLossTW + kHalo, RH = kLossTH + kHalo;
  __shared__ float sx[RH][RW], sy[RH][RW];
  __shared__ float hs[5][RH][kLossTW];
  const int c = blockIdx.z;
  const int Hv = H - kHalo, Wv = W - kHalo;
  const int ox = blockIdx.x * kLossTW, oy = blockIdx.y * kLossTH;
  for (int q = threadIdx.x; q < RH * RW; q += kLossThreads) {
    const int r = q / RW, col = q % RW;
    const int gy = oy + r, gx = ox + col;
    float xv = 0.f, yv = 0.f;
    if (gy < H && gx < W) {
      const size_t p = ((size_t)gy * W + gx) * 3 + c;
      xv = img[p] - 0.5f;
      yv = tgt[p] - 0.5f;
    }
    sx[r][col] = xv;
    sy[r][col] = yv;
  }
  __syncthreads();
  for (int q = threadIdx.x; q < RH * kLossTW; q += kLossThreads) {  // horizontal window
    const int r = q / kLossTW, col = q % kLossTW;
    float mx = 0.f, my = 0.f, vxx = 0.f, vyy = 0.f, vxy = 0.f;
#pragma unroll
    for (int u = 0; u < kWin; u++) {
      const float w = win.w[u], xv = sx[r][col + u], yv = sy[r][col + u];
      mx = fmaf(w, xv, mx);
      my = fmaf(w, yv, my);
      vxx = fmaf(w, xv * xv, vxx);
      vyy = fmaf(w, yv * yv, vyy);
      vxy = fmaf(w, xv * yv, vxy);
    }
    hs[0][r][col] = mx; hs[1][r][col] = my; hs[2][r][col] = vxx; hs[3][r][col] = vyy; hs[4][r][col] = vxy;
  }
  __syncthreads();
  const float scale = 1.f / (3.f * (float)Hv * (float)Wv);
  double ssum = 0.0;
  for (int q = threadIdx.x; q < kLossTH * kLossTW; q += kLossThreads) {  // vertical window
    const int r = q / kLossTW, col = q % kLossTW;
    const int gy = oy + r, gx = ox + col;
    if (gy >= Hv || gx >= Wv) continue;
    float M[5] = {0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int u = 0; u < kWin; u++) {
      const float w = win.w[u];
#pragma unroll
      for (int f = 0; f < 5; f++) M[f] = fmaf(w, hs[f][r + u][col], M[f]);
    }
    const float Mx = M[0], My = M[1];
    const float mux = Mx + 0.5f, muy = My + 0.5f;
    const float sxx = M[2] - Mx * Mx, syy = M[3] - My * My, sxy = M[4] - Mx * My;
    const float a1 = 2.f * mux * muy + kC1, a2 = 2.f * sxy + kC2;
    const float b1 = mux * mux + muy * muy + kC1, b2 = sxx + syy + kC2;
    const float inv = 1.f / (b1 * b2);
    const float smap = a1 * a2 * inv;
    ssum += smap;
    // d smap / d (Mx, Vxx, Vxy) of the shifted statistics (same derivative
    // as losses.py:86-94 in exact arithmetic)
    const float dMx = 2.f * muy * a2 * inv - 2.f * mux * smap / b1 + 2.f * Mx * smap / b2 - 2.f * My * a1 * inv;
    const float dVxx = -smap / b2;
    const float dVxy = 2.f * a1 * inv;
    const size_t o = (size_t)gy * Wv + gx, plane = (size_t)Hv * Wv;
    float *mc = maps + (size_t)c * 3 * plane;
    mc[o] = scale * dMx;
    mc[plane + o] = scale * dVxx;
    mc[2 * plane + o] = scale * dVxy;
  }
  atomic_add_block_sum(stats + 1, ssum);
}

// d_image for one 32x16 tile of the full image, one channel: transposed
// window over the coefficient maps (losses.py:45-55), combined with the
// pixel (losses.py:96-100), plus the L1 term; accumulates sum |diff|.
__global__ void __launch_bounds__(kLossThreads) ssim_adjoint_kernel(int H, int W, const float *img, const float *tgt,
                                                                    const float *maps, float lam, float *d_image,
                                                                    double *stats, Win win) {
  constexpr int RW = kLossTW + kHalo, RH = kLossTH + kHalo;
  __shared__ float sm[3][RH][RW];
  __shared__ float hs[3][RH][kLossTW];
  const int c = blockIdx.z;
  const int Hv = H - kHalo, Wv = W - kHalo;
  const int ox = blockIdx.x * kLossTW, oy = blockIdx.y * kLossTH;
  const size_t plane = (size_t)Hv * Wv;
  const float *mc = maps + (size_t)c * 3 * plane;
  for (int q = threadIdx.x; q < RH * RW; q += kLossThreads) {   // map rows oy-10.., cols ox-10..
    const int r = q / RW, col = q % RW;
    const int my = oy - kHalo + r, mx = ox - kHalo + col;
    const bool in = my >= 0 && my < Hv && mx >= 0 && mx < Wv;
    const size_t o = in ? (size_t)my * Wv + mx : 0;
#pragma unroll
    for (int f = 0; f < 3; f++) sm[f][r][col] = in ? mc[f * plane + o] : 0.f;
  }
  __syncthreads();
  for (int q = threadIdx.x; q < RH * kLossTW; q += kLossThreads) {  // out col x takes map cols x-10..x
    const int r = q / kLossTW, col = q % kLossTW;
    float a[3] = {0.f, 0.f, 0.f};
#pragma unroll
    for (int v = 0; v < kWin; v++) {
      const float w = win.w[v];
#pragma unroll
      for (int f = 0; f < 3; f++) a[f] = fmaf(w, sm[f][r][col + kHalo - v], a[f]);
    }
#pragma unroll
    for (int f = 0; f < 3; f++) hs[f][r][col] = a[f];
  }
  __syncthreads();
  const float l1s = (1.f - lam) / (3.f * (float)H * (float)W);
  double asum = 0.0;
  for (int q = threadIdx.x; q < kLossTH * kLossTW; q += kLossThreads) {
    const int r = q / kLossTW, col = q % kLossTW;
    const int gy = oy + r, gx = ox + col;
    if (gy >= H || gx >= W) continue;
    float a[3] = {0.f, 0.f, 0.f};
#pragma unroll
    for (int u = 0; u < kWin; u++) {
      const float w = win.w[u];
#pragma unroll
      for (int f = 0; f < 3; f++) a[f] = fmaf(w, hs[f][r + kHalo - u][col], a[f]);
    }
    const size_t p = ((size_t)gy * W + gx) * 3 + c;
    const float x = img[p], y = tgt[p];
    const float d_ssim = a[0] + 2.f * (x - 0.5f) * a[1] + (y - 0.5f) * a[2];
    const float diff = x - y;
    asum += fabsf(diff);
    const float sgn = diff > 0.f ? 1.f : (diff < 0.f ? -1.f : 0.f);   // np.sign
    d_image[p] = l1s * sgn - 0.5f * lam * d_ssim;                       // losses.py:154
  }
  atomic_add_block_sum(stats + 0, asum);
}

// mask_term = mean sigmoid(raw_mask); d_raw_mask += beta m (1-m) / n (losses.py:146-151)
__global__ void __launch_bounds__(kLossThreads) mask_term_kernel(const float *raw_mask, int64_t n, float beta,
                                                                 float *d_raw_mask, double *stats) {
  double s = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * kLossThreads + threadIdx.x; i < n; i += (int64_t)gridDim.x * kLossThreads) {
    const float m = 1.f / (1.f + __expf(-raw_mask[i]));
    s += m;
    if (d_raw_mask) d_raw_mask[i] += beta * m * (1.f - m) / (float)n;
  }
  atomic_add_block_sum(stats + 2, s);
}

__global__ void loss_stats_init_kernel(double *stats, double valid) {
  stats[0] = 0.0; stats[1] = 0.0; stats[2] = 0.0; stats[3] = valid;
}

// The loss values from the sums (losses.py:129-155), one thread: the caller
// reads device scalars without further kernels.
__global__ void loss_finalize_kernel(double *stats, int H, int W, int64_t n, double lam, double beta) {
  const double l1 = stats[0] / (3.0 * H * W);
  const double ssim = stats[1] / (3.0 * stats[3]);
  const double dssim = (1.0 - ssim) / 2.0;
  const double mask_term = n ? stats[2] / (double)n : 0.0;
  stats[4] = (1.0 - lam) * l1 + lam * dssim + beta * mask_term;
  stats[5] = l1; stats[6] = ssim; stats[7] = dssim; stats[8] = mask_term;
}

// ------------------------------------------------------------------ Adam
struct AdamArgs {
  cs_adam_tensor t[8];
  int64_t start[9];     // prefix of numel over tensors (flattened index space)
  int count;
  float b1, b2, omb1, omb2, eps, bc1, bc2, gscale;   // omb = 1 - b, formed in float64
};

__global__ void __launch_bounds__(256) adam_kernel(AdamArgs a) {
  const int64_t total = a.start[a.count];
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < total; g += (int64_t)gridDim.x * blockDim.x) {
    int k = 0;
    while (g >= a.start[k + 1]) k++;
    const cs_adam_tensor &T = a.t[k];
    const int64_t i = g - a.start[k];
    const float gr = a.gscale * T.grad[i];
    float m = T.m[i], v = T.v[i];
    m = m * a.b1 + a.omb1 * gr;                   // optim.py:30-31
    v = v * a.b2 + a.omb2 * gr * gr;              // optim.py:32-33
    T.m[i] = m;
    T.v[i] = v;
    T.param[i] -= (float)T.lr * (m / a.bc1) / (sqrtf(v / a.bc2) + a.eps);   // optim.py:34
  }
}

int launch_image_loss(int H, int W, const float *img, const float *tgt, const float *raw_mask, int64_t n,
                      double lam, double beta, float *d_image, float *d_raw_mask, double *stats, void *ws,
                      cudaStream_t s) {
  Win win;
  {
    double g[kWin], sum = 0.0;
    for (int u = 0; u < kWin; u++) {
      const double off = u - (kWin - 1) / 2.0;
      g[u] = std::exp(-(off * off) / (2.0 * 1.5 * 1.5));
      sum += g[u];
    }
    for (int u = 0; u < kWin; u++) win.w[u] = (float)(g[u] / sum);
  }
  const int Hv = H - kHalo, Wv = W - kHalo;
  loss_stats_init_kernel<<<1, 1, 0, s>>>(stats, (double)Hv * (double)Wv);
  float *maps = static_cast<float *>(ws);
  dim3 gv((Wv + kLossTW - 1) / kLossTW, (Hv + kLossTH - 1) / kLossTH, 3);
  ssim_moments_kernel<<<gv, kLossThreads, 0, s>>>(H, W, img, tgt, maps, stats, win);
  dim3 gf((W + kLossTW - 1) / kLossTW, (H + kLossTH - 1) / kLossTH, 3);
  ssim_adjoint_kernel<<<gf, kLossThreads, 0, s>>>(H, W, img, tgt, maps, (float)lam, d_image, stats, win);
  if (n > 0) {
    const int blocks = (int)std::min<int64_t>((n + kLossThreads - 1) / kLossThreads, 148 * 8);
    mask_term_kernel<<<blocks, kLossThreads, 0, s>>>(raw_mask, n, (float)beta, d_raw_mask, stats);
  }
  loss_finalize_kernel<<<1, 1, 0, s>>>(stats, H, W, n, lam, beta);
  return cudaGetLastError() == cudaSuccess ? CS_OK : CS_ERR_CUDA;
}

int launch_adam(int count, const cs_adam_tensor *tensors, double b1, double b2, double eps, int step,
                double gscale, cudaStream_t s) {
  AdamArgs a;
  a.count = count;
  a.start[0] = 0;
  for (int k = 0; k < count; k++) {
    a.t[k] = tensors[k];
    a.start[k + 1] = a.start[k] + tensors[k].numel;
  }
  for (int k = count + 1; k < 9; k++) a.start[k] = a.start[count];
  a.b1 = (float)b1; a.b2 = (float)b2; a.eps = (float)eps; a.gscale = (float)gscale;
  a.omb1 = (float)(1.0 - b1); a.omb2 = (float)(1.0 - b2);
  a.bc1 = (float)(1.0 - std::pow(b1, step));
  a.bc2 = (float)(1.0 - std::pow(b2, step));
  const int64_t total = a.start[count];
  if (total == 0) return CS_OK;
  const int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 16);
  adam_kernel<<<blocks, 256, 0, s>>>(a);
  return cudaGetLastError() == cudaSuccess ? CS_OK : CS_ERR_CUDA;
}

}  // namespace cs
