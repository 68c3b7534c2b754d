// K1: per-convex preprocess (one thread per convex).
//
// Replaces the Python loop of rasterize.prepare_view (rasterize.py:88-120):
// mask gate (model.py:105-107), projection (projection.py:22-40), Graham-scan
// hull (projection.py:47-113), hull lines (projection.py:116-128), depth and
// depth scaling (rasterize.py:99-103, field.py:26-35), screen bbox with the
// cutoff margin (projection.py:136-177) and SH colour (harmonics.py:101-109).
//
// Everything that feeds a DISCRETE decision (cull, hull cycle, bbox, depth
// order) is computed in float64 with the reference's operation order; this
// translation unit is compiled with --fmad=false so that only the explicit
// fma() of the projection (OpenBLAS dgemm order of `points @ R.T`) fuses.
// Outputs are a float32 blend record per convex plus the discrete results.
#include <type_traits>

#include "common.cuh"

namespace cs {

struct PreArgs {
  cs_camera cam;
  int64_t n;
  int k;
  int sh_degree;
  int mode;
  double cutoff;
  const float *points, *raw_delta, *raw_sigma, *raw_opacity, *raw_mask, *sh;
  float *records;
  double *lines;
  uint8_t *hull;
  int4 *bbox;
  uint64_t *depth_keys;
  uint32_t *touched;
  uint32_t *counters;
  double cam_center[3];
};

// projection.py:43-44 -- no contraction (TU built with --fmad=false)
__device__ __forceinline__ double cross_d(const double *X, const double *Y, int o, int a, int b) {
  return (X[a] - X[o]) * (Y[b] - Y[o]) - (Y[a] - Y[o]) * (X[b] - X[o]);
}

// comparator of projection.py:73-85 reduced to "cmp(a, b) < 0"
__device__ __forceinline__ bool hull_lt(const double *X, const double *Y, int ref, int a, int b) {
  double c = cross_d(X, Y, ref, a, b);
  if (c > kCrossTol) return true;
  if (c < -kCrossTol) return false;
  double ax = X[a] - X[ref], ay = Y[a] - Y[ref];
  double bx = X[b] - X[ref], by = Y[b] - Y[ref];
  return (ax * ax + ay * ay) < (bx * bx + by * by);
}

// projection.py:47-113.  The sort reproduces CPython's list.sort for fewer
// than 64 items (count_run + binary insertion), because the tolerance
// comparator is not a strict weak order and the result depends on the
// algorithm.  Returns the hull size (0 == None); out[] gets the CCW cycle
// starting at the reference point.
template <int NP>
__device__ int graham_scan_dev(int n, const double *X, const double *Y, int *out) {
  if (n < 3) return 0;
  int uq[NP];
  int nu = 0;
  for (int i = 0; i < n; i++) {
    bool dup = false;
    for (int j = 0; j < nu; j++) {
      int u = uq[j];
      if (X[u] == X[i] && Y[u] == Y[i]) { dup = true; break; }
    }
    if (!dup) uq[nu++] = i;
  }
  if (nu < 3) return 0;
  int ref = uq[0];
  for (int j = 1; j < nu; j++) {
    int u = uq[j];
    if (Y[u] < Y[ref] || (Y[u] == Y[ref] && X[u] < X[ref])) ref = u;
  }
  int rest[NP];
  int m = 0;
  for (int j = 0; j < nu; j++)
    if (uq[j] != ref) rest[m++] = uq[j];
  if (m >= 2) {
    int run = 2;
    if (hull_lt(X, Y, ref, rest[1], rest[0])) {
      while (run < m && hull_lt(X, Y, ref, rest[run], rest[run - 1])) run++;
      for (int a = 0, b = run - 1; a < b; a++, b--) { int t = rest[a]; rest[a] = rest[b]; rest[b] = t; }
    } else {
      while (run < m && !hull_lt(X, Y, ref, rest[run], rest[run - 1])) run++;
    }
    for (int start = run; start < m; start++) {
      int pivot = rest[start];
      int l = 0, r = start;
      do {
        int p = l + ((r - l) >> 1);
        if (hull_lt(X, Y, ref, pivot, rest[p])) r = p; else l = p + 1;
      } while (l < r);
      for (int p = start; p > l; p--) rest[p] = rest[p - 1];
      rest[l] = pivot;
    }
  }
  int st[NP];
  int sn = 0;
  st[sn++] = ref;
  for (int j = 0; j < m; j++) {
    int c = rest[j];
    while (sn >= 2 && cross_d(X, Y, st[sn - 2], st[sn - 1], c) <= kCrossTol) sn--;
    st[sn++] = c;
  }
  bool changed = true;
  while (changed && sn >= 3) {
    changed = false;
    for (int q = 0; q < sn; q++) {
      int a = st[(q - 1 + sn) % sn], b = st[q], c = st[(q + 1) % sn];
      if (cross_d(X, Y, a, b, c) <= kCrossTol) {
        for (int r = q; r < sn - 1; r++) st[r] = st[r + 1];
        sn--;
        changed = true;
        break;
      }
    }
  }
  if (sn < 3) return 0;
  int start = 0;
  for (int q = 0; q < sn; q++)
    if (st[q] == ref) { start = q; break; }
  for (int q = 0; q < sn; q++) out[q] = st[(start + q) % sn];
  return sn;
}

// harmonics.py:7-24 constants
__constant__ double kSH_C0 = 0.28209479177387814;
__constant__ double kSH_C1 = 0.4886025119029199;
__constant__ double kSH_C2[5] = {1.0925484305920792, -1.0925484305920792, 0.31539156525252005,
                                 -1.0925484305920792, 0.5462742152960396};
__constant__ double kSH_C3[7] = {-0.5900435899266435, 2.890611442640554, -0.4570457994644658,
                                 0.3731763325901154, -0.4570457994644658, 1.445305721320277,
                                 -0.5900435899266435};

// harmonics.py:33-59
__device__ __forceinline__ void sh_basis(double x, double y, double z, int deg, double *b) {
  b[0] = kSH_C0;
  if (deg >= 1) { b[1] = -kSH_C1 * y; b[2] = kSH_C1 * z; b[3] = -kSH_C1 * x; }
  if (deg >= 2) {
    double xx = x * x, yy = y * y, zz = z * z;
    b[4] = kSH_C2[0] * x * y;
    b[5] = kSH_C2[1] * y * z;
    b[6] = kSH_C2[2] * (2.0 * zz - xx - yy);
    b[7] = kSH_C2[3] * x * z;
    b[8] = kSH_C2[4] * (xx - yy);
  }
  if (deg >= 3) {
    double xx = x * x, yy = y * y, zz = z * z;
    b[9] = kSH_C3[0] * y * (3.0 * xx - yy);
    b[10] = kSH_C3[1] * x * y * z;
    b[11] = kSH_C3[2] * y * (4.0 * zz - xx - yy);
    b[12] = kSH_C3[3] * z * (2.0 * zz - 3.0 * xx - 3.0 * yy);
    b[13] = kSH_C3[4] * x * (4.0 * zz - xx - yy);
    b[14] = kSH_C3[5] * z * (xx - yy);
    b[15] = kSH_C3[6] * x * (xx - 3.0 * yy);
  }
}

__device__ __forceinline__ double depth_scale(int mode, double d) {  // field.py:26-35
  switch (mode) {
    case CS_SCALE_NONE: return 1.0;
    case CS_SCALE_SQRT: return sqrt(d);
    case CS_SCALE_DEPTH: return d;
    default: return d * d;
  }
}

#ifndef CS_PRE_THREADS
#define CS_PRE_THREADS 64   // 64 / 128 / 256 threads (12 / 6 / 3 blocks per SM): 182 / 184 / 191 us
#endif
constexpr int kPreThreads = CS_PRE_THREADS;
#ifndef CS_PRE_LINES_UNROLL
#define CS_PRE_LINES_UNROLL 2   // code size: 1 / 2 / 8: 184 / 183 / 192 us (instruction-cache misses)
#endif
constexpr int kPreLinesUnroll = CS_PRE_LINES_UNROLL;
#ifndef CS_PRE_BLOCKS
#define CS_PRE_BLOCKS (768 / CS_PRE_THREADS)   // resident blocks per SM (register budget 85)
#endif

// Index list of up to 16 entries packed as 4-bit nibbles in a register, so
// the Graham scan's insert / erase / pop keep no per-thread local memory.
template <typename W>
struct NibbleListT {
  static constexpr int kCap = (int)sizeof(W) * 2;   // 4-bit entries per word
  W w = 0;
  int n = 0;
  __device__ __forceinline__ static W low(int i) { return i >= kCap ? ~W(0) : ((W(1) << (4 * i)) - W(1)); }
  __device__ __forceinline__ int get(int i) const { return (int)((w >> (4 * i)) & W(15)); }
  __device__ __forceinline__ void set(int i, int v) { w = (w & ~(W(15) << (4 * i))) | ((W)v << (4 * i)); }
  __device__ __forceinline__ void push(int v) { w |= (W)v << (4 * n); n++; }
  __device__ __forceinline__ void pop() { n--; w &= low(n); }
  __device__ __forceinline__ void insert(int i, int v) {
    w = (w & low(i)) | ((W)v << (4 * i)) | ((w & ~low(i)) << 4);
    n++;
  }
  __device__ __forceinline__ void erase(int i) {
    w = (w & low(i)) | ((w >> 4) & ~low(i));
    n--;
  }
  // entries start, start+1, ..., n-1, 0, ..., start-1 (cyclic rotation)
  __device__ __forceinline__ NibbleListT rotated(int start) const {
    NibbleListT r;
    r.n = n;
    r.w = start == 0 ? w : (((w >> (4 * start)) | (w << (4 * (n - start)))) & low(n));
    return r;
  }
};
// 8 entries fit a 32-bit word (the K <= 8 kernels: cheaper shifts than 64-bit)
using NibbleList = NibbleListT<uint64_t>;

// projection.py:47-113 on points X[j*stride], Y[j*stride] (shared memory),
// n <= 16.  Same algorithm as graham_scan_dev (CPython list.sort
// count_run + binary insertion for the tolerance comparator), with the
// index lists held in registers.
template <typename NL>
__device__ int graham_scan_packed(int n, const double *X, const double *Y, int stride, NL &out) {
#define GX(i) X[(i) * stride]
#define GY(i) Y[(i) * stride]
  if (n < 3) return 0;
  int ref = 0;
  NL rest;
#ifndef CS_NO_HULL_FAST
  bool sorted = false;
  // Fast sort for n <= 8.  When every pair of the other points has a cross
  // product around ref (the comparator's own float64 expression) beyond
  // both the 1e-9 tolerance and its rounding bound (4.5e-16 (|ax by| +
  // |ay bx|), so its sign is the exact one), the comparator is the strict
  // total order of the points' angles around ref: there are no duplicates
  // (a duplicate pair gives 0), the dedupe is the identity, and any sort --
  // CPython's binarysort included -- yields the one order, each point's
  // position being the number of points before it.  The C(n-1, 2) products
  // are independent, where binary insertion is a chain of dependent
  // comparisons.  Otherwise fall through to the CPython-order sort.
  if (n <= 8) {
    for (int j = 1; j < n; j++)
      if (GY(j) < GY(ref) || (GY(j) == GY(ref) && GX(j) < GX(ref))) ref = j;
    const double rx = GX(ref), ry = GY(ref);
    for (int j = 0; j < n; j++)
      if (j != ref) rest.push(j);
    const int m = n - 1;
    uint32_t rank = 0;   // 4-bit position per rest entry
    bool decisive = true;
    for (int q = 1; q < m; q++) {
      const int b = rest.get(q);
      const double bx = GX(b) - rx, by = GY(b) - ry;
#pragma unroll
      for (int p = 0; p < 7; p++)
        if (p < q) {
          const int a = rest.get(p);
          const double ax = GX(a) - rx, ay = GY(a) - ry;
          const double s = ax * by, t = ay * bx, c = s - t;
          decisive &= fabs(c) > fmax(kCrossTol, 1e-15 * (fabs(s) + fabs(t)));
          rank += c > 0.0 ? (1u << (4 * q)) : (1u << (4 * p));   // a before b : b before a
        }
    }
    if (decisive) {
      NL order;
      order.n = m;
      for (int j = 0; j < m; j++) order.set((int)((rank >> (4 * j)) & 15u), rest.get(j));
      rest = order;
      sorted = true;
    } else {
      rest = NL();
      ref = 0;
    }
  }
  if (!sorted) {
#endif
  NL uq;
  for (int i = 0; i < n; i++) {
    const double xi = GX(i), yi = GY(i);
    bool dup = false;
    for (int j = 0; j < uq.n; j++) {
      const int u = uq.get(j);
      if (GX(u) == xi && GY(u) == yi) { dup = true; break; }
    }
    if (!dup) uq.push(i);
  }
  if (uq.n < 3) return 0;
  ref = uq.get(0);
  for (int j = 1; j < uq.n; j++) {
    const int u = uq.get(j);
    if (GY(u) < GY(ref) || (GY(u) == GY(ref) && GX(u) < GX(ref))) ref = u;
  }
  const double rx = GX(ref), ry = GY(ref);
  auto lt = [&](int a, int b) -> bool {  // cmp(a, b) < 0, projection.py:73-85
    const double ax = GX(a) - rx, ay = GY(a) - ry, bx = GX(b) - rx, by = GY(b) - ry;
    const double c = ax * by - ay * bx;
    if (c > kCrossTol) return true;
    if (c < -kCrossTol) return false;
    return (ax * ax + ay * ay) < (bx * bx + by * by);
  };
  for (int j = 0; j < uq.n; j++)
    if (uq.get(j) != ref) rest.push(uq.get(j));
  const int m = rest.n;
  if (m >= 2) {
    int run = 2;
    if (lt(rest.get(1), rest.get(0))) {
      while (run < m && lt(rest.get(run), rest.get(run - 1))) run++;
      for (int a = 0, b = run - 1; a < b; a++, b--) {
        const int t = rest.get(a);
        rest.set(a, rest.get(b));
        rest.set(b, t);
      }
    } else {
      while (run < m && !lt(rest.get(run), rest.get(run - 1))) run++;
    }
    for (int start = run; start < m; start++) {
      const int pivot = rest.get(start);
      int l = 0, r = start;
      do {
        const int p = l + ((r - l) >> 1);
        if (lt(pivot, rest.get(p))) r = p; else l = p + 1;
      } while (l < r);
      rest.erase(start);
      rest.insert(l, pivot);
    }
  }
#ifndef CS_NO_HULL_FAST
  }
#endif
  const int nrest = rest.n;
  auto cross = [&](int o, int a, int b) -> double {  // projection.py:43-44
    return (GX(a) - GX(o)) * (GY(b) - GY(o)) - (GY(a) - GY(o)) * (GX(b) - GX(o));
  };
  NL st;
  st.push(ref);
  for (int j = 0; j < nrest; j++) {
    const int c = rest.get(j);
    while (st.n >= 2 && cross(st.get(st.n - 2), st.get(st.n - 1), c) <= kCrossTol) st.pop();
    st.push(c);
  }
  bool changed = true;
  while (changed && st.n >= 3) {
    changed = false;
    const int sn = st.n;
    for (int q = 0; q < sn; q++) {   // neighbours without integer modulo
      if (cross(st.get(q == 0 ? sn - 1 : q - 1), st.get(q), st.get(q + 1 == sn ? 0 : q + 1)) <= kCrossTol) {
        st.erase(q);
        changed = true;
        break;
      }
    }
  }
  if (st.n < 3) return 0;
  int start = 0;
  for (int q = 0; q < st.n; q++)
    if (st.get(q) == ref) { start = q; break; }
  out = st.rotated(start);
  return out.n;
#undef GX
#undef GY
}

// SH colour in float32 (harmonics.py:33-59, 101-109): continuous output,
// checked at 1e-4, so it needs no float64.  sh: the convex's 16x3 floats.
__device__ __forceinline__ void sh_colour(float x, float y, float z, int deg, const float *sh, float *col) {
  float b[kShCoeffs];
  b[0] = 0.28209479177387814f;
  const float c1 = 0.4886025119029199f;
  const float xx = x * x, yy = y * y, zz = z * z;
  if (deg >= 1) { b[1] = -c1 * y; b[2] = c1 * z; b[3] = -c1 * x; }
  if (deg >= 2) {
    b[4] = 1.0925484305920792f * x * y;
    b[5] = -1.0925484305920792f * y * z;
    b[6] = 0.31539156525252005f * (2.f * zz - xx - yy);
    b[7] = -1.0925484305920792f * x * z;
    b[8] = 0.5462742152960396f * (xx - yy);
  }
  if (deg >= 3) {
    b[9] = -0.5900435899266435f * y * (3.f * xx - yy);
    b[10] = 2.890611442640554f * x * y * z;
    b[11] = -0.4570457994644658f * y * (4.f * zz - xx - yy);
    b[12] = 0.3731763325901154f * z * (2.f * zz - 3.f * xx - 3.f * yy);
    b[13] = -0.4570457994644658f * x * (4.f * zz - xx - yy);
    b[14] = 1.445305721320277f * z * (xx - yy);
    b[15] = -0.5900435899266435f * x * (xx - 3.f * yy);
  }
  const int nb = (deg + 1) * (deg + 1);
  float acc[3] = {0.f, 0.f, 0.f};
  const float4 *sh4 = reinterpret_cast<const float4 *>(sh);
#pragma unroll
  for (int q = 0; q < kShCoeffs * 3 / 4; q++) {  // 4 coefficients of 3 channels = 3 float4
    if (4 * q < 3 * nb) {
      const float4 v = sh4[q];
      const float e[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int r = 0; r < 4; r++) {
        const int f = 4 * q + r, qb = f / 3, c = f % 3;
        if (qb < nb) acc[c] = fmaf(b[qb], e[r], acc[c]);
      }
    }
  }
#pragma unroll
  for (int c = 0; c < 3; c++) col[c] = fmaxf(0.5f + acc[c], 0.f);
}

// One convex.  pts_s: this convex's points staged in smem by TMA; X, Y:
// this thread's projected-pixel slots in smem (stride kPreThreads).
//
// Order of work: projection + cull, hull, then depth / activations / margin,
// then ONE loop over the hull edges that computes each line (hull_lines),
// writes its blend coefficients and inflates the vertex it starts at
// (bbox_with_margin) -- the per-line arrays never exist, which keeps the
// register footprint (and so the occupancy of this latency-bound float64
// kernel) in check.  Every value is computed by the same expression as in the
// reference, so the discrete results are unchanged.  The anchor of the
// anchor-relative line offsets is the integer pixel at hull vertex 0.
#ifdef CS_PRE_PHASES
// diagnostics: SM cycles per preprocess phase, summed over threads (tools/pre_phases.py)
__device__ unsigned long long g_pre_phase[8];
#define PH(n) do { const long long t_ = clock64(); atomicAdd(&g_pre_phase[n], (unsigned long long)(t_ - ph_t)); ph_t = t_; } while (0)
#else
#define PH(n) do {} while (0)
#endif

// What the colour pass (after the block's geometry) needs of a visible convex.
struct ColourJob {
  float dx, dy, dz, depth;
};

template <int MAXK>
__device__ __forceinline__ bool preprocess_one(const PreArgs &a, int64_t i, const float *pts_s, double *X,
                                               double *Y, ColourJob &cj, uint64_t &key) {
#ifdef CS_PRE_PHASES
  long long ph_t = clock64();
#endif
  const int k = a.k;
  // the scalar parameters are loaded up front (their latency overlaps)
  const float r_mask = __ldg(a.raw_mask + i), r_delta = __ldg(a.raw_delta + i);
  const float r_sigma = __ldg(a.raw_sigma + i), ro = __ldg(a.raw_opacity + i);
  a.touched[i] = 0u;
  a.depth_keys[i] = kCulledKey;
  // rasterize.py:89 mask gate (model.py:105-107, expit = 1/(1+exp(-x)))
  const double mask = 1.0 / (1.0 + exp(-(double)r_mask));
  if (mask <= kMaskGate) return false;
  PH(0);
  // projection.py:22-40
  const double *R = a.cam.R;
  double zsum = 0.0, cx = 0.0, cy = 0.0, cz = 0.0;
  bool culled = false;
  for (int j = 0; j < k; j++) {
    const double p0 = pts_s[3 * j], p1 = pts_s[3 * j + 1], p2 = pts_s[3 * j + 2];
    const double xc = fma(p2, R[2], fma(p1, R[1], p0 * R[0])) + a.cam.t[0];
    const double yc = fma(p2, R[5], fma(p1, R[4], p0 * R[3])) + a.cam.t[1];
    const double zc = fma(p2, R[8], fma(p1, R[7], p0 * R[6])) + a.cam.t[2];
    culled |= zc <= a.cam.z_near;
    zsum = zsum + zc;  // rasterize.py:99 mean, left to right
    cx = cx + p0;      // model.py:109-111 centre, left to right
    cy = cy + p1;
    cz = cz + p2;
    if (a.cam.ortho) {
      X[j * kPreThreads] = a.cam.fx * xc + a.cam.cx;
      Y[j * kPreThreads] = a.cam.fy * yc + a.cam.cy;
    } else {
      X[j * kPreThreads] = (a.cam.fx * xc) / zc + a.cam.cx;
      Y[j * kPreThreads] = (a.cam.fy * yc) / zc + a.cam.cy;
    }
  }
  if (culled) return false;
  PH(1);
  NibbleListT<typename std::conditional<(MAXK <= 8), uint32_t, uint64_t>::type> hull;
  const int h = graham_scan_packed(k, X, Y, kPreThreads, hull);
  if (h == 0) return false;
  PH(2);
  // rasterize.py:99-103
  const double depth = zsum / k;
  const double s = depth_scale(a.mode, a.cam.ortho ? 1.0 : depth);
  const double delta_s = s * exp((double)r_delta);
  const double sigma_s = s * exp((double)r_sigma);
  const double o = 1.0 / (1.0 + exp(-(double)ro));
  // projection.py:157-163
  if (o <= a.cutoff) return false;
  const bool full_frame = a.cutoff <= 0.0;
  double margin = 0.0;
  if (!full_frame) {
    double eps = a.cutoff / o;
    if (0.5 < eps) eps = 0.5;
    margin = log((1.0 - eps) / eps) / (sigma_s * delta_s);
  }
  const int v0 = hull.get(0);
  const double axd = floor(X[v0 * kPreThreads]), ayd = floor(Y[v0 * kPreThreads]);
  const double dls = delta_s * 1.4426950408889634;  // delta_s * log2(e)
  constexpr int RF = Rec<MAXK>::kGlobal;
  float4 *dst = reinterpret_cast<float4 *>(a.records + i * RF);
  double *lines = a.lines + i * Rec<MAXK>::kLines64;   // (A, B, C, 0) per line
  // line of edge j (projection.py:116-128): from vertex hull[j] to hull[j+1]
  auto line = [&](int j, double &nx, double &ny, double &off) {
    const int u = hull.get(j), v = hull.get(j + 1 < h ? j + 1 : 0);
    const double ux = X[u * kPreThreads], uy = Y[u * kPreThreads];
    const double ex = X[v * kPreThreads] - ux, ey = Y[v * kPreThreads] - uy;
    const double rx = ey, ry = -ex;
    const double len = sqrt(rx * rx + ry * ry);
    nx = rx / len;
    ny = ry / len;
    off = -(nx * ux + ny * uy);
  };
  double pnx, pny;  // normal of the line ending at the current vertex (projection.py:167)
  {
    double poff;
    line(h - 1, pnx, pny, poff);
  }
  double xmin = INFINITY, xmax = -INFINITY, ymin = INFINITY, ymax = -INFINITY;
#pragma unroll kPreLinesUnroll
  for (int j = 0; j < MAXK; j++) {
    if (j < h) {
      double nx, ny, off;
      line(j, nx, ny, off);
      // blend coefficients in float64, anchor-relative offset (the blends'
      // producer re-bases them per tile)
      st_global_v4d(lines + 4 * j, dls * nx, dls * ny, dls * (off + nx * axd + ny * ayd), 0.0);
      if (!full_frame) {  // projection.py:167-169, vertex j
        const int u = hull.get(j);
        double den = 1.0 + (pnx * nx + pny * ny);
        if (!(den >= 1e-12)) den = 1e-12;
        const double ix = X[u * kPreThreads] + (margin * (pnx + nx)) / den;
        const double iy = Y[u * kPreThreads] + (margin * (pny + ny)) / den;
        xmin = fmin(xmin, ix); xmax = fmax(xmax, ix);
        ymin = fmin(ymin, iy); ymax = fmax(ymax, iy);
      }
      pnx = nx;
      pny = ny;
    }
  }
  PH(3);
  // projection.py:170-177
  int x0, x1, y0, y1;
  if (full_frame) {
    x0 = 0; x1 = a.cam.width; y0 = 0; y1 = a.cam.height;
  } else {
    double fx0 = ceil(xmin - 0.5), fx1 = floor(xmax - 0.5) + 1.0;
    double fy0 = ceil(ymin - 0.5), fy1 = floor(ymax - 0.5) + 1.0;
    fx0 = fmax(fx0, 0.0); fy0 = fmax(fy0, 0.0);
    fx1 = fmin(fx1, (double)a.cam.width); fy1 = fmin(fy1, (double)a.cam.height);
    if (!(fx0 < fx1) || !(fy0 < fy1)) return false;
    x0 = (int)fx0; x1 = (int)fx1; y0 = (int)fy0; y1 = (int)fy1;
  }
  // ---- outputs: discrete state, then the float32 record header ----
  uint8_t hb[MAXK];
#pragma unroll
  for (int j = 0; j < MAXK; j++) hb[j] = (uint8_t)(j < h ? hull.get(j) : 0xff);
  if (MAXK == 8) {
    *reinterpret_cast<uint2 *>(a.hull + i * MAXK) =
        make_uint2(hb[0] | hb[1] << 8 | hb[2] << 16 | (uint32_t)hb[3] << 24,
                   hb[4] | hb[5] << 8 | hb[6] << 16 | (uint32_t)hb[7] << 24);
  } else {
#pragma unroll
    for (int j = 0; j < MAXK; j++) a.hull[i * MAXK + j] = hb[j];
  }
  a.bbox[i] = make_int4(x0, x1, y0, y1);
  a.touched[i] = (uint32_t)(((x1 - 1) / kTile - x0 / kTile + 1) * ((y1 - 1) / kTile - y0 / kTile + 1));
  key = orderable_bits(depth);
  a.depth_keys[i] = key;
  // rasterize.py:110-114 view direction; harmonics.py:101-109 colour (float32,
  // SH rows read straight from global: 12 x 16-byte loads per thread).  The
  // direction only feeds the continuous colour: centre offset in float64
  // (no cancellation), normalisation in float32 (no float64 divisions).
  const double ik = 1.0 / k;
  const float vx = (float)(cx * ik - a.cam_center[0]), vy = (float)(cy * ik - a.cam_center[1]),
              vz = (float)(cz * ik - a.cam_center[2]);
  const float d2 = vx * vx + vy * vy + vz * vz;
  float dx = 0.f, dy = 0.f, dz = 1.f;
  if (d2 > 0.f) { const float rs = rsqrtf(d2); dx = vx * rs; dy = vy * rs; dz = vz * rs; }
  cj.dx = dx; cj.dy = dy; cj.dz = dz; cj.depth = (float)depth;
  PH(4);
  dst[0] = make_float4((float)axd, (float)ayd, (float)sigma_s, (float)o);
  dst[2] = make_float4(1.f / (1.f + __expf(ro)), (float)dls, __int_as_float(h), __frcp_rn((float)dls));
  dst[3] = make_float4(__int_as_float(x0), __int_as_float(x1), __int_as_float(y0), __int_as_float(y1));
  PH(5);
  return true;
}

template <int MAXK>
__global__ void __launch_bounds__(kPreThreads, CS_PRE_BLOCKS) preprocess_kernel(PreArgs a) {
  // dynamic smem: X[MAXK][threads], Y[MAXK][threads] (f64), points[threads][k*3] (f32)
  extern __shared__ __align__(16) double pre_smem[];
  __shared__ __align__(8) uint64_t bars[1];
  double *Xs = pre_smem, *Ys = pre_smem + MAXK * kPreThreads;
  float *pts_smem = reinterpret_cast<float *>(pre_smem + 2 * MAXK * kPreThreads);
  const int64_t base = (int64_t)blockIdx.x * kPreThreads;
  const int rowf = a.k * 3;
  const int64_t nblk = min((int64_t)kPreThreads, a.n - base);
  const bool full = nblk == kPreThreads;  // full blocks: 16B-aligned, in-bounds bulk copies
  if (threadIdx.x == 0) {
    mbar_init(&bars[0], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (full) {
    if (threadIdx.x == 0) {
      const uint32_t pbytes = kPreThreads * rowf * 4;
      mbar_expect_tx(&bars[0], pbytes);
      tma_bulk_g2s(pts_smem, a.points + base * rowf, pbytes, &bars[0]);
      // the block's SH rows are read at the very end of each thread (colour):
      // start pulling them into L2 now so that read does not wait on DRAM
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a.sh + base * kShCoeffs * 3),
                   "r"((uint32_t)(kPreThreads * kShCoeffs * 3 * 4)) : "memory");
    }
    mbar_wait(&bars[0], 0);
  } else {  // tail block: plain coalesced loads
    for (int q = threadIdx.x; q < nblk * rowf; q += kPreThreads) pts_smem[q] = a.points[base * rowf + q];
    __syncthreads();
  }
  const int64_t i = base + threadIdx.x;
  bool vis = false;
  ColourJob cj;
  uint64_t key = 0ull;
  if (i < a.n)
    vis = preprocess_one<MAXK>(a, i, pts_smem + threadIdx.x * rowf, Xs + threadIdx.x, Ys + threadIdx.x, cj, key);
  // Colour (harmonics.py:101-109) after the block's geometry: its SH rows
  // (48 floats per convex, prefetched into L2 at the start) are copied by
  // one bulk TMA into the smem the geometry no longer needs, so the
  // per-thread 192-byte rows are not gathered from L2 by 12 strided loads
  // per thread each waiting on its own round trip.
  {
    float *sh_smem = reinterpret_cast<float *>(pre_smem);
    __syncthreads();   // every thread is done with X, Y and its points
    if (full) {
      if (threadIdx.x == 0) {
        const uint32_t sbytes = kPreThreads * kShCoeffs * 3 * 4;
        fence_proxy_async_smem();   // the generic reads above precede the async-proxy writes
        mbar_expect_tx(&bars[0], sbytes);
        tma_bulk_g2s(sh_smem, a.sh + base * kShCoeffs * 3, sbytes, &bars[0]);
      }
      mbar_wait(&bars[0], 1);
    } else {
      for (int q = threadIdx.x; q < nblk * kShCoeffs * 3; q += kPreThreads) sh_smem[q] = a.sh[base * kShCoeffs * 3 + q];
      __syncthreads();
    }
    if (vis) {
      float col[3];
      sh_colour(cj.dx, cj.dy, cj.dz, a.sh_degree, sh_smem + threadIdx.x * kShCoeffs * 3, col);
      reinterpret_cast<float4 *>(a.records + i * Rec<MAXK>::kGlobal)[1] = make_float4(col[0], col[1], col[2], cj.depth);
    }
  }
  unsigned b = __ballot_sync(0xffffffffu, vis);
  if ((threadIdx.x & 31) == 0 && b) atomicAdd(&a.counters[C_NVISIBLE], (unsigned)__popc(b));
  // range of the visible depth keys (block reduce, one atomic pair per block)
  {
    __shared__ unsigned long long s_kminc, s_kmax;
    if (threadIdx.x == 0) { s_kminc = 0ull; s_kmax = 0ull; }
    __syncthreads();
    unsigned long long kc = 0ull, kx = 0ull;
    if (vis) { kx = key; kc = ~kx; }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      kc = max(kc, (unsigned long long)__shfl_xor_sync(0xffffffffu, kc, o));
      kx = max(kx, (unsigned long long)__shfl_xor_sync(0xffffffffu, kx, o));
    }
    if ((threadIdx.x & 31) == 0 && b) { atomicMax(&s_kminc, kc); atomicMax(&s_kmax, kx); }
    __syncthreads();
    if (threadIdx.x == 0 && s_kmax) {
      atomicMax(reinterpret_cast<unsigned long long *>(a.counters + C_KMINC), s_kminc);
      atomicMax(reinterpret_cast<unsigned long long *>(a.counters + C_KMAX), s_kmax);
    }
  }
}

// cs_graham_scan_batch: one thread per point set.
__global__ void hull_batch_kernel(int m, int npts, const int32_t *counts, const double *pts,
                                  int32_t *hull, int32_t *hull_n) {
  int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= m) return;
  int n = counts ? counts[s] : npts;
  double X[32], Y[32];
  for (int j = 0; j < n; j++) {
    X[j] = pts[((int64_t)s * npts + j) * 2];
    Y[j] = pts[((int64_t)s * npts + j) * 2 + 1];
  }
  int out[32];
  int h;
  if (n <= 16) {  // the scan the preprocess kernel runs
    NibbleList l;
    h = graham_scan_packed(n, X, Y, 1, l);
    for (int j = 0; j < h; j++) out[j] = l.get(j);
  } else {
    h = graham_scan_dev<32>(n, X, Y, out);
  }
  for (int j = 0; j < npts; j++) hull[(int64_t)s * npts + j] = j < h ? out[j] : -1;
  hull_n[s] = h;
}

static void camera_center(const cs_camera &cam, double *c) {  // model.py:164-166
  for (int j = 0; j < 3; j++) {
    double s = 0.0;
    for (int r = 0; r < 3; r++) s += (-cam.R[3 * r + j]) * cam.t[r];
    c[j] = s;
  }
}

// ---------------------------------------------------------------------------
// cs_prepare_view_export: the full per-view state of every prepared convex
// in float64 (projection.ProjectedConvex, projection.py:180-203, and
// rasterize.ViewPrimitive, rasterize.py:56-65) for the drop-in prepare_view.
// Not on the hot path: one thread per convex after a forward's stage 0
// (hull cycle and visibility from the workspace), the projection and
// hull_lines re-evaluated with the preprocess's expressions in this
// --fmad=false translation unit (bit-exact with the reference), delta_s /
// sigma_s / opacity, and the view direction and colour in float64
// (rasterize.py:110-114, harmonics.py:33-59, 101-109).
struct ExportArgs {
  cs_camera cam;
  int64_t n;
  int k, max_k, sh_degree, mode;
  double cam_center[3];
  const float *points, *raw_delta, *raw_sigma, *raw_opacity, *sh;
  const uint8_t *hull;
  const uint32_t *touched;
  cs_view_export out;
};

__global__ void __launch_bounds__(128) export_view_kernel(ExportArgs a) {
  const int64_t i = (int64_t)blockIdx.x * 128 + threadIdx.x;
  if (i >= a.n || a.touched[i] == 0) return;
  const int k = a.k;
  const double *R = a.cam.R;
  double X[16], Y[16];
  double cx = 0.0, cy = 0.0, cz = 0.0, zsum = 0.0;
  for (int j = 0; j < k; j++) {
    const double p0 = a.points[(i * k + j) * 3], p1 = a.points[(i * k + j) * 3 + 1], p2 = a.points[(i * k + j) * 3 + 2];
    const double xc = fma(p2, R[2], fma(p1, R[1], p0 * R[0])) + a.cam.t[0];
    const double yc = fma(p2, R[5], fma(p1, R[4], p0 * R[3])) + a.cam.t[1];
    const double zc = fma(p2, R[8], fma(p1, R[7], p0 * R[6])) + a.cam.t[2];
    zsum = zsum + zc;
    cx = cx + p0; cy = cy + p1; cz = cz + p2;
    if (a.cam.ortho) {
      X[j] = a.cam.fx * xc + a.cam.cx;
      Y[j] = a.cam.fy * yc + a.cam.cy;
    } else {
      X[j] = (a.cam.fx * xc) / zc + a.cam.cx;
      Y[j] = (a.cam.fy * yc) / zc + a.cam.cy;
    }
    a.out.pixels[(i * k + j) * 2] = X[j];
    a.out.pixels[(i * k + j) * 2 + 1] = Y[j];
    a.out.point_depths[i * k + j] = zc;
  }
  int hidx[16], h = 0;
  for (int j = 0; j < a.max_k; j++) {
    const int v = a.hull[i * a.max_k + j];
    if (v != 0xff) hidx[h++] = v;
  }
  for (int j = 0; j < k; j++) {   // projection.py:116-128 over the hull cycle; unused rows NaN
    double nx = NAN, ny = NAN, off = NAN;
    if (j < h) {
      const int u = hidx[j], v = hidx[j + 1 < h ? j + 1 : 0];
      const double ex = X[v] - X[u], ey = Y[v] - Y[u];
      const double rx = ey, ry = -ex;
      const double len = sqrt(rx * rx + ry * ry);
      nx = rx / len;
      ny = ry / len;
      off = -(nx * X[u] + ny * Y[u]);
    }
    a.out.normals[(i * k + j) * 2] = nx;
    a.out.normals[(i * k + j) * 2 + 1] = ny;
    a.out.offsets[i * k + j] = off;
  }
  const double depth = zsum / k;
  const double s = depth_scale(a.mode, a.cam.ortho ? 1.0 : depth);
  a.out.delta_s[i] = s * exp((double)a.raw_delta[i]);
  a.out.sigma_s[i] = s * exp((double)a.raw_sigma[i]);
  a.out.opacity[i] = 1.0 / (1.0 + exp(-(double)a.raw_opacity[i]));
  a.out.scale[i] = s;
  const double vx = cx / k - a.cam_center[0], vy = cy / k - a.cam_center[1], vz = cz / k - a.cam_center[2];
  const double dist = sqrt(vx * vx + vy * vy + vz * vz);
  double d[3] = {0.0, 0.0, 1.0};
  if (dist > 0.0) { d[0] = vx / dist; d[1] = vy / dist; d[2] = vz / dist; }
  a.out.view_dir[i * 3] = d[0]; a.out.view_dir[i * 3 + 1] = d[1]; a.out.view_dir[i * 3 + 2] = d[2];
  a.out.view_dist[i] = dist;
  // harmonics.py:33-59 basis, 101-109 colour
  const double x = d[0], y = d[1], z = d[2], xx = x * x, yy = y * y, zz = z * z;
  double b[16];
  b[0] = 0.28209479177387814;
  b[1] = -0.4886025119029199 * y; b[2] = 0.4886025119029199 * z; b[3] = -0.4886025119029199 * x;
  b[4] = 1.0925484305920792 * x * y; b[5] = -1.0925484305920792 * y * z;
  b[6] = 0.31539156525252005 * (2.0 * zz - xx - yy); b[7] = -1.0925484305920792 * x * z;
  b[8] = 0.5462742152960396 * (xx - yy);
  b[9] = -0.5900435899266435 * y * (3.0 * xx - yy); b[10] = 2.890611442640554 * x * y * z;
  b[11] = -0.4570457994644658 * y * (4.0 * zz - xx - yy);
  b[12] = 0.3731763325901154 * z * (2.0 * zz - 3.0 * xx - 3.0 * yy);
  b[13] = -0.4570457994644658 * x * (4.0 * zz - xx - yy); b[14] = 1.445305721320277 * z * (xx - yy);
  b[15] = -0.5900435899266435 * x * (xx - 3.0 * yy);
  const int nb = (a.sh_degree + 1) * (a.sh_degree + 1);
  for (int c = 0; c < 3; c++) {
    double acc = 0.0;
    for (int q = 0; q < nb; q++) acc += b[q] * (double)a.sh[(i * kShCoeffs + q) * 3 + c];
    const double v = 0.5 + acc;
    a.out.color[i * 3 + c] = v > 0.0 ? v : 0.0;
  }
}

#ifdef CS_PRE_PHASES
extern "C" CS_API int cs_debug_pre_phases(unsigned long long *host8, int reset) {
  cudaDeviceSynchronize();
  if (cudaMemcpyFromSymbol(host8, g_pre_phase, sizeof(unsigned long long) * 8) != cudaSuccess) return 2;
  if (reset) {
    unsigned long long z[8] = {0};
    cudaMemcpyToSymbol(g_pre_phase, z, sizeof(z));
  }
  return 0;
}
#endif

int launch_export_view(const cs_camera &cam, const cs_settings &set, const cs_params &p, const cs_layout &L,
                       const char *ws, const cs_view_export &out, cudaStream_t s) {
  if (p.n == 0) return CS_OK;
  ExportArgs a;
  a.cam = cam;
  a.n = p.n;
  a.k = p.k;
  a.max_k = L.max_k;
  a.sh_degree = set.sh_degree;
  a.mode = set.scaling_mode;
  camera_center(cam, a.cam_center);
  a.points = p.points; a.raw_delta = p.raw_delta; a.raw_sigma = p.raw_sigma; a.raw_opacity = p.raw_opacity;
  a.sh = p.sh;
  a.hull = reinterpret_cast<const uint8_t *>(ws + L.hull);
  a.touched = reinterpret_cast<const uint32_t *>(ws + L.tiles_touched);
  a.out = out;
  export_view_kernel<<<(int)((p.n + 127) / 128), 128, 0, s>>>(a);
  return cudaGetLastError() == cudaSuccess ? CS_OK : CS_ERR_CUDA;
}

int launch_preprocess(const cs_camera &cam, const cs_settings &set, const cs_params &p,
                      const cs_layout &L, char *ws, cudaStream_t s) {
  if (p.n == 0) return CS_OK;
  PreArgs a;
  a.cam = cam;
  a.n = p.n;
  a.k = p.k;
  a.sh_degree = set.sh_degree;
  a.mode = set.scaling_mode;
  a.cutoff = set.cutoff;
  a.points = p.points; a.raw_delta = p.raw_delta; a.raw_sigma = p.raw_sigma;
  a.raw_opacity = p.raw_opacity; a.raw_mask = p.raw_mask; a.sh = p.sh;
  a.records = reinterpret_cast<float *>(ws + L.records);
  a.lines = reinterpret_cast<double *>(ws + L.lines);
  a.hull = reinterpret_cast<uint8_t *>(ws + L.hull);
  a.bbox = reinterpret_cast<int4 *>(ws + L.bbox);
  a.depth_keys = reinterpret_cast<uint64_t *>(ws + L.depth_keys);
  a.touched = reinterpret_cast<uint32_t *>(ws + L.tiles_touched);
  a.counters = reinterpret_cast<uint32_t *>(ws + L.counters);
  camera_center(cam, a.cam_center);
  const int blocks = (int)((p.n + kPreThreads - 1) / kPreThreads);
  // geometry staging (X, Y, points), later reused for the block's SH rows
  const size_t smem = (size_t)kPreThreads * std::max(2 * L.max_k * sizeof(double) + p.k * 3 * sizeof(float),
                                                     (size_t)kShCoeffs * 3 * sizeof(float));
  if (L.max_k == 8) {
    cudaFuncSetAttribute(preprocess_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    preprocess_kernel<8><<<blocks, kPreThreads, smem, s>>>(a);
  } else {
    cudaFuncSetAttribute(preprocess_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    preprocess_kernel<16><<<blocks, kPreThreads, smem, s>>>(a);
  }
  return cudaGetLastError() == cudaSuccess ? CS_OK : CS_ERR_CUDA;
}

int launch_hull_batch(int32_t m, int32_t npts, const int32_t *counts, const double *pts,
                      int32_t *hull, int32_t *hull_n, cudaStream_t s) {
  if (m <= 0) return CS_OK;
  hull_batch_kernel<<<(m + 127) / 128, 128, 0, s>>>(m, npts, counts, pts, hull, hull_n);
  return cudaGetLastError() == cudaSuccess ? CS_OK : CS_ERR_CUDA;
}

}  // namespace cs
