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

constexpr int kLossThreads = 256;

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

// One 32x32 tile of the valid grid of one channel (blockIdx.z).  maps:
// [3 channels][3: dMx, dVxx, dVxy][Hv*Wv], scaled by 1/(3 Hv Wv).
// Register-blocked separable window: the horizontal pass gives each thread
// 4 adjacent outputs of a row (14 inputs loaded once), the vertical pass 4
// adjacent outputs of a column (14 rows of the 5 moments loaded once).
constexpr int kSsimT = 32;            // output tile side
constexpr int kSsimR = kSsimT + kHalo;
constexpr int kSsimB = 4;             // outputs per thread and pass

__global__ void __launch_bounds__(kLossThreads) ssim_moments_kernel(int H, int W, const float *img, const float *tgt,
                                                                    float *maps, double *stats, Win win) {
  __shared__ float sx[kSsimR][kSsimR], sy[kSsimR][kSsimR];
  __shared__ float hs[5][kSsimR][kSsimT];
  const int c = blockIdx.z;
  const int Hv = H - kHalo, Wv = W - kHalo;
  const int ox = blockIdx.x * kSsimT, oy = blockIdx.y * kSsimT;
  for (int q = threadIdx.x; q < kSsimR * kSsimR; q += kLossThreads) {
    const int r = q / kSsimR, col = q % kSsimR;
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
  // horizontal: item = (row, 4-column group)
  for (int q = threadIdx.x; q < kSsimR * (kSsimT / kSsimB); q += kLossThreads) {
    const int r = q / (kSsimT / kSsimB), c0 = (q % (kSsimT / kSsimB)) * kSsimB;
    float xv[kSsimB + kHalo], yv[kSsimB + kHalo], xx[kSsimB + kHalo], yy[kSsimB + kHalo], xy[kSsimB + kHalo];
#pragma unroll
    for (int u = 0; u < kSsimB + kHalo; u++) {   // products once per input, not once per tap
      xv[u] = sx[r][c0 + u]; yv[u] = sy[r][c0 + u];
      xx[u] = xv[u] * xv[u]; yy[u] = yv[u] * yv[u]; xy[u] = xv[u] * yv[u];
    }
#pragma unroll
    for (int o = 0; o < kSsimB; o++) {
      float mx = 0.f, my = 0.f, vxx = 0.f, vyy = 0.f, vxy = 0.f;
#pragma unroll
      for (int u = 0; u < kWin; u++) {
        const float w = win.w[u];
        mx = fmaf(w, xv[o + u], mx);
        my = fmaf(w, yv[o + u], my);
        vxx = fmaf(w, xx[o + u], vxx);
        vyy = fmaf(w, yy[o + u], vyy);
        vxy = fmaf(w, xy[o + u], vxy);
      }
      hs[0][r][c0 + o] = mx; hs[1][r][c0 + o] = my; hs[2][r][c0 + o] = vxx; hs[3][r][c0 + o] = vyy;
      hs[4][r][c0 + o] = vxy;
    }
  }
  __syncthreads();
  // vertical: item = (column, 4-row group)
  const float scale = 1.f / (3.f * (float)Hv * (float)Wv);
  const size_t plane = (size_t)Hv * Wv;
  float *mc = maps + (size_t)c * 3 * plane;
  double ssum = 0.0;
  for (int q = threadIdx.x; q < kSsimT * (kSsimT / kSsimB); q += kLossThreads) {
    const int col = q % kSsimT, r0 = (q / kSsimT) * kSsimB;
    float M[kSsimB][5];
#pragma unroll
    for (int o = 0; o < kSsimB; o++)
#pragma unroll
      for (int f = 0; f < 5; f++) M[o][f] = 0.f;
#pragma unroll
    for (int u = 0; u < kSsimB + kHalo; u++) {
      float h[5];
#pragma unroll
      for (int f = 0; f < 5; f++) h[f] = hs[f][r0 + u][col];
#pragma unroll
      for (int o = 0; o < kSsimB; o++) {
        const int t = u - o;   // window tap of output row r0 + o
        if (t >= 0 && t < kWin) {
#pragma unroll
          for (int f = 0; f < 5; f++) M[o][f] = fmaf(win.w[t], h[f], M[o][f]);
        }
      }
    }
#pragma unroll
    for (int o = 0; o < kSsimB; o++) {
      const int gy = oy + r0 + o, gx = ox + col;
      if (gy >= Hv || gx >= Wv) continue;
      const float Mx = M[o][0], My = M[o][1];
      const float mux = Mx + 0.5f, muy = My + 0.5f;
      const float sxx = M[o][2] - Mx * Mx, syy = M[o][3] - My * My, sxy = M[o][4] - Mx * My;
      const float a1 = 2.f * mux * muy + kC1, a2 = 2.f * sxy + kC2;
      const float b1 = mux * mux + muy * muy + kC1, b2 = sxx + syy + kC2;
      const float inv = 1.f / (b1 * b2);
      const float smap = a1 * a2 * inv;
      ssum += smap;
      // d smap / d (Mx, Vxx, Vxy) of the shifted statistics (same derivative
      // as losses.py:86-94 in exact arithmetic); 1/b1 = b2 inv, 1/b2 = b1 inv
      const float sb1 = smap * (b2 * inv), sb2 = smap * (b1 * inv);
      const float dMx = 2.f * muy * a2 * inv - 2.f * mux * sb1 + 2.f * Mx * sb2 - 2.f * My * a1 * inv;
      const float dVxx = -sb2;
      const float dVxy = 2.f * a1 * inv;
      const size_t oo = (size_t)gy * Wv + gx;
      mc[oo] = scale * dMx;
      mc[plane + oo] = scale * dVxx;
      mc[2 * plane + oo] = scale * dVxy;
    }
  }
  atomic_add_block_sum(stats + 1, ssum);
}

// d_image for one 32x32 tile of the full image, one channel: transposed
// window over the coefficient maps (losses.py:45-55; the Gaussian is
// symmetric, so the transposed window is the window), combined with the
// pixel (losses.py:96-100), plus the L1 term; accumulates sum |diff|.
__global__ void __launch_bounds__(kLossThreads) ssim_adjoint_kernel(int H, int W, const float *img, const float *tgt,
                                                                    const float *maps, float lam, float *d_image,
                                                                    double *stats, Win win) {
  __shared__ float sm[3][kSsimR][kSsimR];
  __shared__ float hs[3][kSsimR][kSsimT];
  const int c = blockIdx.z;
  const int Hv = H - kHalo, Wv = W - kHalo;
  const int ox = blockIdx.x * kSsimT, oy = blockIdx.y * kSsimT;
  const size_t plane = (size_t)Hv * Wv;
  const float *mc = maps + (size_t)c * 3 * plane;
  for (int q = threadIdx.x; q < kSsimR * kSsimR; q += kLossThreads) {   // map rows oy-10.., cols ox-10..
    const int r = q / kSsimR, col = q % kSsimR;
    const int my = oy - kHalo + r, mx = ox - kHalo + col;
    const bool in = my >= 0 && my < Hv && mx >= 0 && mx < Wv;
    const size_t o = in ? (size_t)my * Wv + mx : 0;
#pragma unroll
    for (int f = 0; f < 3; f++) sm[f][r][col] = in ? mc[f * plane + o] : 0.f;
  }
  __syncthreads();
  for (int q = threadIdx.x; q < kSsimR * (kSsimT / kSsimB); q += kLossThreads) {   // horizontal
    const int r = q / (kSsimT / kSsimB), c0 = (q % (kSsimT / kSsimB)) * kSsimB;
#pragma unroll
    for (int f = 0; f < 3; f++) {
      float v[kSsimB + kHalo];
#pragma unroll
      for (int u = 0; u < kSsimB + kHalo; u++) v[u] = sm[f][r][c0 + u];
#pragma unroll
      for (int o = 0; o < kSsimB; o++) {
        float acc = 0.f;
#pragma unroll
        for (int u = 0; u < kWin; u++) acc = fmaf(win.w[kHalo - u], v[o + u], acc);
        hs[f][r][c0 + o] = acc;
      }
    }
  }
  __syncthreads();
  const float l1s = (1.f - lam) / (3.f * (float)H * (float)W);
  double asum = 0.0;
  for (int q = threadIdx.x; q < kSsimT * (kSsimT / kSsimB); q += kLossThreads) {   // vertical + pixel terms
    const int col = q % kSsimT, r0 = (q / kSsimT) * kSsimB;
    float A[kSsimB][3];
#pragma unroll
    for (int o = 0; o < kSsimB; o++) { A[o][0] = 0.f; A[o][1] = 0.f; A[o][2] = 0.f; }
#pragma unroll
    for (int u = 0; u < kSsimB + kHalo; u++) {
      const float h0 = hs[0][r0 + u][col], h1 = hs[1][r0 + u][col], h2 = hs[2][r0 + u][col];
#pragma unroll
      for (int o = 0; o < kSsimB; o++) {
        const int t = u - o;
        if (t >= 0 && t < kWin) {
          const float w = win.w[kHalo - t];
          A[o][0] = fmaf(w, h0, A[o][0]);
          A[o][1] = fmaf(w, h1, A[o][1]);
          A[o][2] = fmaf(w, h2, A[o][2]);
        }
      }
    }
#pragma unroll
    for (int o = 0; o < kSsimB; o++) {
      const int gy = oy + r0 + o, gx = ox + col;
      if (gy >= H || gx >= W) continue;
      const size_t p = ((size_t)gy * W + gx) * 3 + c;
      const float x = img[p], y = tgt[p];
      const float d_ssim = A[o][0] + 2.f * (x - 0.5f) * A[o][1] + (y - 0.5f) * A[o][2];
      const float diff = x - y;
      asum += fabsf(diff);
      const float sgn = diff > 0.f ? 1.f : (diff < 0.f ? -1.f : 0.f);   // np.sign
      d_image[p] = l1s * sgn - 0.5f * lam * d_ssim;                       // losses.py:154
    }
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
    // a reduction, not a read-modify-write: the chain stages of other views
    // (other streams) accumulate into the same gradient row concurrently
    if (d_raw_mask) atomicAdd(d_raw_mask + i, beta * m * (1.f - m) / (float)n);
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
  dim3 gv((Wv + kSsimT - 1) / kSsimT, (Hv + kSsimT - 1) / kSsimT, 3);
  ssim_moments_kernel<<<gv, kLossThreads, 0, s>>>(H, W, img, tgt, maps, stats, win);
  dim3 gf((W + kSsimT - 1) / kSsimT, (H + kSsimT - 1) / kSsimT, 3);
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
