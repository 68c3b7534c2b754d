// K2: depth order + tile binning (rasterize.py:121 sort, rasterize.py:134-144).
//
//   depth sort   stable LSD radix sort of 24-bit keys monotone in the
//                orderable f64 depth bits + exact fix-up of equal-key runs
//                == Python's sort by (depth, index) (rasterize.py:121)
//   duplicate    one fused kernel: exclusive scan of tiles_touched in depth
//                order (decoupled look-back between 1024-rank chunks) and
//                the (tile, id) pairs of every convex's bbox tiles, written
//                in depth order (the append loop of bin_tiles), plus the
//                digit histograms of the pair sort
//   pair sort    stable radix sort by tile id only: since pairs are emitted in
//                depth order, a stable sort by tile gives exactly the reference
//                per-tile lists in (depth, index) order
//   ranges       [start, end) of every tile in the sorted pairs
//
// Both radix sorts are onesweep (Adinets & Merrill): the digit histograms
// come from the producing kernel, then one kernel per 8-bit digit ranks keys
// with warp ballots, publishes per-chunk digit counts and resolves its
// prefix by decoupled look-back.
#include <algorithm>

#include "common.cuh"

namespace cs {

constexpr int kRadixBits = 8;
constexpr int kRadix = 1 << kRadixBits;
#ifndef CS_SORT_THREADS
#define CS_SORT_THREADS 512
#endif
#ifndef CS_SORT_ITEMS
#define CS_SORT_ITEMS 8
#endif
#ifndef CS_SORT_MINB
#define CS_SORT_MINB 3
#endif
constexpr int kSortThreads = CS_SORT_THREADS;
constexpr int kSortWarps = kSortThreads / 32;
constexpr int kSortItems = CS_SORT_ITEMS;
constexpr int kSortChunk = kSortThreads * kSortItems;  // 4096 keys per chunk (the pair sort)
// keys per thread of the depth sort's chunks (binning at 1M @1080p with 1 /
// 2 / 4 / 8 / 16: 283 / 261 / 246 / 236 / 238 us -- smaller chunks, more
// blocks for the 1M keys, lose more to the longer look-back than they win;
// the pair sort at 8 / 12 / 16: 236 / 241 / 244 us)
#ifndef CS_DEPTH_SORT_ITEMS
#define CS_DEPTH_SORT_ITEMS 8
#endif
constexpr int kDepthSortItems = CS_DEPTH_SORT_ITEMS;
constexpr int kDepthChunk = kSortThreads * kDepthSortItems;
constexpr uint32_t kFlagAgg = 1u << 30;
constexpr uint32_t kFlagPrefix = 2u << 30;
constexpr uint32_t kValueMask = (1u << 30) - 1;


// ------------------------------------------------------------------ hist
template <typename KeyT>
__global__ void __launch_bounds__(kSortThreads) radix_hist_kernel(const KeyT *keys, const uint32_t *count,
                                                                   uint32_t n_fixed, int passes, int shift0,
                                                                   uint32_t *hist) {
  __shared__ uint32_t h[8][kRadix];
  for (int q = threadIdx.x; q < passes * kRadix; q += kSortThreads) h[q / kRadix][q % kRadix] = 0;
  __syncthreads();
  const uint32_t n = count ? *count : n_fixed;
  for (uint32_t idx = blockIdx.x * kSortThreads + threadIdx.x; idx < n; idx += gridDim.x * kSortThreads) {
    KeyT k = keys[idx];
    for (int p = 0; p < passes; p++) atomicAdd(&h[p][(uint32_t)(k >> (shift0 + p * kRadixBits)) & (kRadix - 1)], 1u);
  }
  __syncthreads();
  for (int q = threadIdx.x; q < passes * kRadix; q += kSortThreads) {
    uint32_t v = h[q / kRadix][q % kRadix];
    if (v) atomicAdd(&hist[q], v);
  }
}

// exclusive scan of each pass's 256-bin histogram (one block per pass)
__global__ void radix_offsets_kernel(const uint32_t *hist, uint32_t *offsets) {
  __shared__ uint32_t s[kRadix];
  const int p = blockIdx.x, t = threadIdx.x;
  s[t] = hist[p * kRadix + t];
  __syncthreads();
  for (int d = 1; d < kRadix; d <<= 1) {
    uint32_t v = t >= d ? s[t - d] : 0;
    __syncthreads();
    s[t] += v;
    __syncthreads();
  }
  offsets[p * kRadix + t] = s[t] - hist[p * kRadix + t];
}

// ------------------------------------------------------------------ onesweep pass
template <typename KeyT>
struct PassArgs {
  const KeyT *keys_in;
  KeyT *keys_out;
  const uint32_t *vals_in;
  uint32_t *vals_out;
  const uint32_t *count;  // device item count (or null -> n_fixed)
  uint32_t n_fixed;
  int shift;
  int bits;                 // significant bits of this pass's digit (<= 8): fewer ballots
  const uint32_t *offsets;  // [256] global exclusive digit offsets of this pass
  uint32_t *lookback;       // [chunks][256]
  uint32_t *chunk_counter;
};

// exclusive scan of one value per thread over the block (threads >= 256 add 0)
__device__ __forceinline__ uint32_t block_exclusive_scan256(uint32_t v, uint32_t *s_warp) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t u = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += u;
  }
  if (lane == 31) s_warp[w] = inc;
  __syncthreads();
  if (w == 0) {
    const uint32_t x = lane < kSortWarps ? s_warp[lane] : 0;
    uint32_t y = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t u = __shfl_up_sync(0xffffffffu, y, o);
      if (lane >= o) y += u;
    }
    if (lane < kSortWarps) s_warp[lane] = y - x;
  }
  __syncthreads();
  return s_warp[w] + inc - v;
}

template <typename KeyT, int ITEMS>
constexpr size_t onesweep_dyn_smem() { return (size_t)kSortThreads * ITEMS * (sizeof(KeyT) + sizeof(uint32_t)); }

// One LSD digit.  Items are ranked per warp with __match_any_sync, the
// chunk's digit counts are published for decoupled look-back, and the chunk
// is first scattered into shared memory in digit order so that the global
// writes come out as contiguous runs per digit (coalesced).
template <typename KeyT, int ITEMS>
__global__ void __launch_bounds__(kSortThreads, CS_SORT_MINB) onesweep_kernel(PassArgs<KeyT> a) {
  constexpr int kChunk = kSortThreads * ITEMS;
  extern __shared__ __align__(16) unsigned char onesweep_dyn[];
  KeyT *s_keys = reinterpret_cast<KeyT *>(onesweep_dyn);
  uint32_t *s_vals = reinterpret_cast<uint32_t *>(onesweep_dyn + sizeof(KeyT) * kChunk);
  __shared__ uint32_t s_hist[kSortWarps][kRadix];
  __shared__ uint32_t s_dexcl[kRadix];
  __shared__ uint32_t s_base[kRadix];
  __shared__ uint32_t s_warp[kSortWarps];
  __shared__ uint32_t s_chunk;
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  if (t == 0) s_chunk = atomicAdd(a.chunk_counter, 1u);
  for (int q = t; q < kSortWarps * kRadix; q += kSortThreads) s_hist[q / kRadix][q % kRadix] = 0;
  __syncthreads();
  const uint32_t chunk = s_chunk;
  const uint32_t n = a.count ? *a.count : a.n_fixed;
  const uint32_t start = chunk * kChunk;
  if (start >= n) return;  // no later chunk holds items, nobody looks back here
  const uint32_t nvalid = min((uint32_t)kChunk, n - start);

  const uint32_t lt_mask = (1u << lane) - 1u;
  KeyT key[ITEMS];
  uint32_t val[ITEMS];
  uint32_t dig[ITEMS];
  uint32_t rank[ITEMS];
  const uint32_t wbase = start + w * (32 * ITEMS);
#pragma unroll
  for (int i = 0; i < ITEMS; i++) {
    const uint32_t idx = wbase + i * 32 + lane;
    const bool valid = idx < n;
    key[i] = valid ? a.keys_in[idx] : (KeyT)0;
    val[i] = valid ? a.vals_in[idx] : 0u;
    dig[i] = valid ? (uint32_t)(key[i] >> a.shift) & (kRadix - 1) : kRadix;
  }
#pragma unroll
  for (int i = 0; i < ITEMS; i++) {
    const uint32_t d = dig[i];
    // lanes holding the same digit: AND of 8 bit ballots (cheaper than MATCH)
    uint32_t peers = __ballot_sync(0xffffffffu, d < kRadix);
#pragma unroll
    for (int b = 0; b < kRadixBits; b++) {
      if (b >= a.bits) break;            // higher digit bits are zero for every key
      const uint32_t bal = __ballot_sync(0xffffffffu, (d >> b) & 1u);
      peers &= ((d >> b) & 1u) ? bal : ~bal;
    }
    uint32_t prev = 0;
    if (d < kRadix) prev = s_hist[w][d];
    __syncwarp();
    if (d < kRadix && lane == __ffs(peers) - 1) s_hist[w][d] = prev + __popc(peers);
    __syncwarp();
    rank[i] = prev + __popc(peers & lt_mask);
  }
  __syncthreads();
  // digit t (t < 256): exclusive offsets across warps and the chunk total
  const int d = t;
  const bool owner = t < kRadix;
  uint32_t sum = 0;
  if (owner) {
#pragma unroll
    for (int ww = 0; ww < kSortWarps; ww++) {
      const uint32_t v = s_hist[ww][d];
      s_hist[ww][d] = sum;
      sum += v;
    }
  }
  // publish early, then resolve the prefix from the preceding chunks
  volatile uint32_t *lb = a.lookback;
  if (owner) {
    if (chunk == 0) lb[d] = kFlagPrefix | sum;
    else lb[chunk * kRadix + d] = kFlagAgg | sum;
  }
  const uint32_t dex = block_exclusive_scan256(sum, s_warp);
  if (owner) s_dexcl[d] = dex;
  __syncthreads();
  // local scatter into digit order first: the predecessors' prefixes get
  // the scatter's time to appear before the look-back reads them
#pragma unroll
  for (int i = 0; i < ITEMS; i++) {
    const uint32_t dd = dig[i];
    if (dd < kRadix) {
      const uint32_t pos = s_dexcl[dd] + s_hist[w][dd] + rank[i];
      s_keys[pos] = key[i];
      s_vals[pos] = val[i];
    }
  }
  uint32_t excl = 0;
  if (owner && chunk > 0) {
    // windowed decoupled look-back: kLookback independent loads per round, so
    // the walk over not-yet-resolved predecessors costs one L2 round trip per
    // kLookback chunks instead of one per chunk (4: wider windows re-read
    // more unpublished entries; binning 4 / 8 / 16 / 32: 243 / 243 / 251 /
    // 264 us)
#ifndef CS_LOOKBACK
#define CS_LOOKBACK 4
#endif
    constexpr int kLookback = CS_LOOKBACK;
    int c = (int)chunk - 1;
    bool done = false;
    while (!done) {
      uint32_t v[kLookback];
#pragma unroll
      for (int q = 0; q < kLookback; q++) v[q] = c - q >= 0 ? lb[(c - q) * kRadix + d] : (2u << 30);
      int used = 0;
#pragma unroll
      for (int q = 0; q < kLookback; q++) {
        if (done || used < q) continue;              // stopped earlier in this window
        const uint32_t flag = v[q] & ~kValueMask;
        if (flag == 0) continue;                     // not published yet: re-read from here
        excl += v[q] & kValueMask;
        used = q + 1;
        done = flag == kFlagPrefix;
      }
      c -= used;
    }
    lb[chunk * kRadix + d] = kFlagPrefix | (excl + sum);
  }
  if (owner) s_base[d] = a.offsets[d] + excl;
  __syncthreads();
  for (uint32_t q = t; q < nvalid; q += kSortThreads) {
    const KeyT kk = s_keys[q];
    const uint32_t dd = (uint32_t)(kk >> a.shift) & (kRadix - 1);
    const uint32_t gpos = s_base[dd] + (q - s_dexcl[dd]);
    a.keys_out[gpos] = kk;
    a.vals_out[gpos] = s_vals[q];
  }
}

// Full LSD sort over `passes` digits starting at bit shift0.  Ping-pongs
// (k0,v0) <-> (k1,v1); returns true when the result ends in (k1,v1).  With
// hist_ready the caller has already accumulated the digit histograms.
template <typename KeyT, int ITEMS>
static bool radix_sort(KeyT *k0, uint32_t *v0, KeyT *k1, uint32_t *v1, const uint32_t *count, int key_bits,
                       uint32_t n_fixed, uint32_t n_cap, int passes, int shift0, uint32_t *hist,
                       uint32_t *offsets, uint32_t *lookback, uint32_t *chunk_counters, bool hist_ready,
                       cudaStream_t s) {
  constexpr int kChunk = kSortThreads * ITEMS;
  const int chunks = (int)((n_cap + kChunk - 1) / kChunk);
  if (chunks == 0) return false;
  if (!hist_ready) {
    const int hist_blocks = min(chunks * 4, 148 * 8);
    radix_hist_kernel<KeyT><<<hist_blocks, kSortThreads, 0, s>>>(k0, count, n_fixed, passes, shift0, hist);
  }
  radix_offsets_kernel<<<passes, kRadix, 0, s>>>(hist, offsets);
  constexpr size_t dyn = onesweep_dyn_smem<KeyT, ITEMS>();
  cudaFuncSetAttribute(onesweep_kernel<KeyT, ITEMS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
  for (int p = 0; p < passes; p++) {
    PassArgs<KeyT> a;
    bool odd = p & 1;
    a.keys_in = odd ? k1 : k0;
    a.vals_in = odd ? v1 : v0;
    a.keys_out = odd ? k0 : k1;
    a.vals_out = odd ? v0 : v1;
    a.count = count;
    a.n_fixed = n_fixed;
    a.shift = shift0 + p * kRadixBits;
    a.bits = min(kRadixBits, key_bits - a.shift);
    a.offsets = offsets + p * kRadix;
    a.lookback = lookback + (size_t)p * chunks * kRadix;
    a.chunk_counter = chunk_counters + p;
    onesweep_kernel<KeyT, ITEMS><<<chunks, kSortThreads, dyn, s>>>(a);
  }
  return passes & 1;
}

// ------------------------------------------------------------------ duplicate
// A warp takes 32 consecutive depth ranks; their pairs occupy one contiguous
// range of the pair arrays, which the warp writes cooperatively (coalesced).
// The 8-bit digit histograms of the tile keys for the pair sort are
// accumulated on the way (shared-memory atomics, one global add per bin).
constexpr int kDupThreads = 256;
#ifndef CS_DUP_ROUNDS
#define CS_DUP_ROUNDS 2   // with CS_SORT_MINB 3: binning 236 -> 228 us (rounds 1 / 2 / 3 / 4 / 8 at MINB 2: 240 / 231 / 234 / 236 / 247)
#endif
constexpr int kDupRounds = CS_DUP_ROUNDS;   // ranks per block = kDupRounds * kDupThreads (fewer histogram flushes)

// Fused scan + duplicate: every block takes the next 1024 depth ranks (a
// dynamic chunk id, so predecessors are always resident), sums their tile
// counts, resolves its offset by decoupled look-back over the preceding
// chunks (one warp, 32 predecessors per round) and emits its pairs.  This
// replaces the three-kernel scan of tiles_touched (rasterize.py:134-144
// append order == exclusive scan in depth order).
constexpr uint64_t kDupFlagAgg = 1ull << 62, kDupFlagPrefix = 2ull << 62, kDupValue = (1ull << 62) - 1;

__global__ void __launch_bounds__(kDupThreads) duplicate_scan_kernel(
    const uint32_t *order, const uint32_t *touched, const int4 *bbox, uint32_t n, uint32_t cap, int tiles_x,
    int passes, uint32_t *pair_tiles, uint32_t *pair_ids, uint32_t *hist, uint32_t *offsets_out,
    unsigned long long *lookback, uint32_t *chunk_counter, uint32_t *counters) {
  constexpr int kRanks = kDupThreads * kDupRounds;
  __shared__ uint32_t s_h[3][kRadix];
  __shared__ uint32_t s_wtot[kDupRounds][kDupThreads / 32];
  __shared__ uint32_t s_chunk;
  __shared__ unsigned long long s_base;
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  if (t == 0) s_chunk = atomicAdd(chunk_counter, 1u);
  for (int q = t; q < passes * kRadix; q += kDupThreads) s_h[q / kRadix][q % kRadix] = 0;
  __syncthreads();
  const uint32_t chunk = s_chunk;
  const uint32_t nchunks = (n + kRanks - 1) / kRanks;
  uint32_t id[kDupRounds], cnt[kDupRounds], inc[kDupRounds];
#pragma unroll
  for (int k = 0; k < kDupRounds; k++) {
    const uint32_t r = chunk * kRanks + k * kDupThreads + t;
    id[k] = r < n ? order[r] : 0u;
  }
#pragma unroll
  for (int k = 0; k < kDupRounds; k++) {
    const uint32_t r = chunk * kRanks + k * kDupThreads + t;
    cnt[k] = r < n ? touched[id[k]] : 0u;
    uint32_t v = cnt[k];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t u = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += u;
    }
    inc[k] = v;
    if (lane == 31) s_wtot[k][w] = v;
  }
  __syncthreads();
  // exclusive offset of each warp-round inside the chunk (rounds in order)
  uint32_t before[kDupRounds];
  uint32_t run = 0;
#pragma unroll
  for (int k = 0; k < kDupRounds; k++) {
    uint32_t wb = run;
    for (int ww = 0; ww < kDupThreads / 32; ww++) {
      if (ww == w) wb = run;
      run += s_wtot[k][ww];
    }
    before[k] = wb;
  }
  const uint32_t total = run;   // chunk total (<= 1024 * tiles, fits 32 bits)
  if (w == 0) {
    volatile unsigned long long *lb = lookback;
    if (lane == 0) lb[chunk] = (chunk == 0 ? kDupFlagPrefix : kDupFlagAgg) | (unsigned long long)total;
    unsigned long long excl = 0;
    if (chunk > 0) {
      int c = (int)chunk - 1;
      while (true) {
        const unsigned long long v = c - lane >= 0 ? lb[c - lane] : kDupFlagPrefix;
        const uint64_t flag = v & ~kDupValue;
        const uint32_t notready = __ballot_sync(0xffffffffu, flag == 0);
        const uint32_t prefix = __ballot_sync(0xffffffffu, flag == kDupFlagPrefix);
        const int fp = prefix ? __ffs(prefix) - 1 : 32;
        const int nr = notready ? __ffs(notready) - 1 : 32;
        if (nr <= fp && nr < 32) continue;   // a nearer predecessor has not published yet
        unsigned long long part = lane <= fp ? (v & kDupValue) : 0ull;
#pragma unroll
        for (int o = 16; o; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
        excl += part;
        if (fp < 32) break;
        c -= 32;
      }
      if (lane == 0) lb[chunk] = kDupFlagPrefix | (excl + total);
    }
    if (lane == 0) {
      s_base = excl;
      if (chunk + 1 == nchunks) {   // the grand total: pair count and capacity check
        const unsigned long long all = excl + total;
        counters[C_NPAIRS] = all > 0xffffffffull ? 0xffffffffu : (uint32_t)all;
        counters[C_OVERFLOW] = all > cap ? 1u : 0u;
        counters[C_NSORT] = all > cap ? 0u : (uint32_t)all;
      }
    }
  }
  __syncthreads();
  const unsigned long long cbase = s_base;
#pragma unroll 1
  for (int k = 0; k < kDupRounds; k++) {
    const uint32_t r = chunk * kRanks + k * kDupThreads + t;
    const unsigned long long off64 = cbase + before[k] + (inc[k] - cnt[k]);
    const uint32_t off = off64 > 0xffffffffull ? 0xffffffffu : (uint32_t)off64;
    if (r < n) offsets_out[r] = off;
    int tx0 = 0, ty0 = 0, wdt = 1;
    float inv_wdt = 1.f;
    if (cnt[k]) {
      const int4 b = bbox[id[k]];
      tx0 = b.x / kTile;
      ty0 = b.z / kTile;
      wdt = (b.y - 1) / kTile - tx0 + 1;
      inv_wdt = 1.f / (float)wdt;
      if (passes > 1 && off64 + cnt[k] <= cap) {   // higher-digit histograms, per run of equal digits
        const int ty1 = (b.w - 1) / kTile;
        for (int ty = ty0; ty <= ty1; ty++) {
          const uint32_t t0 = (uint32_t)(ty * tiles_x + tx0), t1 = t0 + (uint32_t)wdt - 1;
          for (int ps = 1; ps < passes; ps++) {
            const int sh = ps * kRadixBits;
            uint32_t seg = t0;
            while (seg <= t1) {
              const uint32_t blk_end = min(t1, ((seg >> sh) + 1) * (1u << sh) - 1);
              atomicAdd(&s_h[ps][(seg >> sh) & (kRadix - 1)], blk_end - seg + 1);
              seg = blk_end + 1;
            }
          }
        }
      }
    }
    // the warp's 32 ranks are contiguous: write its pairs cooperatively
    const uint32_t wtotal = __shfl_sync(0xffffffffu, inc[k], 31);
    const uint64_t wbase = cbase + before[k];
    const uint32_t excl = inc[k] - cnt[k];
    for (uint32_t p0 = 0; p0 < wtotal; p0 += 32) {
      const uint32_t p = p0 + lane;
      int lo = 0;
#pragma unroll
      for (int step = 16; step >= 1; step >>= 1) {
        const uint32_t e = __shfl_sync(0xffffffffu, excl, (lo + step) & 31);
        if (lo + step < 32 && e <= p) lo += step;
      }
      const uint32_t q = p - __shfl_sync(0xffffffffu, excl, lo);
      const int w_o = __shfl_sync(0xffffffffu, wdt, lo);
      // q / w_o by a float reciprocal plus a one-step correction (exact for
      // any q < 2^24), instead of an integer division
      int qy = (int)(((float)q + 0.5f) * __shfl_sync(0xffffffffu, inv_wdt, lo));
      if (qy * w_o > (int)q) qy--;
      else if ((qy + 1) * w_o <= (int)q) qy++;
      const int tx = __shfl_sync(0xffffffffu, tx0, lo) + ((int)q - qy * w_o);
      const int ty = __shfl_sync(0xffffffffu, ty0, lo) + qy;
      const uint32_t owner_id = __shfl_sync(0xffffffffu, id[k], lo);
      const uint64_t pos = wbase + p;
      if (p < wtotal && pos < cap) {
        const uint32_t tile = (uint32_t)(ty * tiles_x + tx);
        pair_tiles[pos] = tile;
        pair_ids[pos] = owner_id;
        // low-digit histogram here, one pair per lane (a per-convex loop
        // over its tiles diverged across the warp)
        atomicAdd(&s_h[0][tile & (kRadix - 1)], 1u);
      }
    }
  }
  __syncthreads();
  for (int q = t; q < passes * kRadix; q += kDupThreads) {
    const uint32_t v = s_h[q / kRadix][q % kRadix];
    if (v) atomicAdd(&hist[q], v);
  }
}

// [start, end) of every tile in the sorted pair keys: each pair position
// that starts or ends a run of equal tiles writes that bound (one coalesced
// pass over the keys; empty tiles keep the zeroed (0, 0)).
__global__ void __launch_bounds__(256) ranges_kernel(const uint32_t *pair_tiles, const uint32_t *counters,
                                                     uint2 *ranges) {
  const uint32_t P = counters[C_NSORT];
  // four positions per thread: one 16-byte load plus the two neighbours
  for (uint32_t p0 = 4 * (blockIdx.x * blockDim.x + threadIdx.x); p0 < P; p0 += 4 * gridDim.x * blockDim.x) {
    uint32_t t[6];
    t[0] = p0 > 0 ? __ldg(pair_tiles + p0 - 1) : ~0u;
    if (p0 + 4 <= P) {
      const uint4 v = __ldg(reinterpret_cast<const uint4 *>(pair_tiles + p0));
      t[1] = v.x; t[2] = v.y; t[3] = v.z; t[4] = v.w;
    } else {
      for (int q = 0; q < 4; q++) t[1 + q] = p0 + q < P ? pair_tiles[p0 + q] : ~0u;
    }
    t[5] = p0 + 4 < P ? __ldg(pair_tiles + p0 + 4) : ~0u;
#pragma unroll
    for (int q = 0; q < 4; q++) {
      const uint32_t p = p0 + q;
      if (p >= P) break;
      if (t[q] != t[q + 1]) ranges[t[q + 1]].x = p;
      if (t[q + 2] != t[q + 1]) ranges[t[q + 1]].y = p + 1;
    }
  }
}

// ------------------------------------------------------------------ depth order
// The depth order sorts (f64 depth, index) (rasterize.py:121).  Instead of a
// 64-bit radix sort (8 passes) the keys are reduced to 23 bits,
//   key32 = (key64 - kmin) >> shift,   shift = max(0, bits(kmax - kmin) - 23),
// which is monotone in key64; a stable 3-pass sort by key32 then orders
// (key32, index).  Only runs of EQUAL key32 can be out of (key64, index)
// order, and only when shift > 0; depth_fixup_kernel re-sorts those runs by
// the full key (they are a few items long on real scenes).  Culled convexes
// get key32 = 0xffffff and stay at the end, in index order.
constexpr int kDepthBits = 23, kDepthPasses = 3;
constexpr uint32_t kDepthCulled = (1u << (kDepthBits + 1)) - 1;

__device__ __forceinline__ void depth_range(const uint32_t *counters, uint64_t &kmin, int &shift, bool &any) {
  const uint64_t kminc = *reinterpret_cast<const unsigned long long *>(counters + C_KMINC);
  const uint64_t kmax = *reinterpret_cast<const unsigned long long *>(counters + C_KMAX);
  any = kmax != 0ull;
  kmin = ~kminc;
  const uint64_t range = any ? kmax - kmin : 0ull;
  const int bits = range ? 64 - __clzll((long long)range) : 0;
  shift = bits > kDepthBits ? bits - kDepthBits : 0;
}

__global__ void __launch_bounds__(kSortThreads) depth_key32_kernel(const uint64_t *keys64, const uint32_t *counters,
                                                                   uint32_t n, uint32_t *keys32, uint32_t *order,
                                                                   uint32_t *hist) {
  __shared__ uint32_t h[kDepthPasses][kRadix];
  for (int q = threadIdx.x; q < kDepthPasses * kRadix; q += kSortThreads) h[q / kRadix][q % kRadix] = 0;
  __syncthreads();
  uint64_t kmin;
  int shift;
  bool any;
  depth_range(counters, kmin, shift, any);
  for (uint32_t idx = blockIdx.x * kSortThreads + threadIdx.x; idx < n; idx += gridDim.x * kSortThreads) {
    const uint64_t k = keys64[idx];
    const uint32_t k32 = k == kCulledKey ? kDepthCulled : (uint32_t)((k - kmin) >> shift);
    keys32[idx] = k32;
    order[idx] = idx;
#pragma unroll
    for (int p = 0; p < kDepthPasses; p++) {   // one shared atomic when the whole warp shares the digit (depths cluster)
      const uint32_t d = (k32 >> (p * kRadixBits)) & (kRadix - 1);
      const uint32_t act = __activemask();
      const uint32_t d0 = __shfl_sync(act, d, __ffs(act) - 1);
      if (__all_sync(act, d == d0)) {
        if ((threadIdx.x & 31) == __ffs(act) - 1) atomicAdd(&h[p][d], (uint32_t)__popc(act));
      } else {
        atomicAdd(&h[p][d], 1u);
      }
    }
  }
  __syncthreads();
  for (int q = threadIdx.x; q < kDepthPasses * kRadix; q += kSortThreads) {
    const uint32_t v = h[q / kRadix][q % kRadix];
    if (v) atomicAdd(&hist[q], v);
  }
}

// Re-sort runs of equal key32 by (key64, index).  One thread per run start;
// insertion sort for short runs, heap sort beyond (pathological clustering).
__device__ __forceinline__ bool depth_less(const uint64_t *keys64, uint32_t a, uint32_t b) {
  const uint64_t ka = keys64[a], kb = keys64[b];
  return ka < kb || (ka == kb && a < b);
}

__global__ void depth_fixup_kernel(const uint64_t *keys64, const uint32_t *counters, const uint32_t *keys32,
                                   uint32_t *order) {
  uint64_t kmin;
  int shift;
  bool any;
  depth_range(counters, kmin, shift, any);
  if (!any || shift == 0) return;  // key32 exact: nothing to fix
  const uint32_t V = counters[C_NVISIBLE];
  const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r + 1 >= V) return;
  const uint32_t k = keys32[r];
  if ((r > 0 && keys32[r - 1] == k) || keys32[r + 1] != k) return;  // not the start of a run of >= 2
  uint32_t e = r + 2;
  while (e < V && keys32[e] == k) e++;
  uint32_t *o = order + r;
  const uint32_t len = e - r;
  if (len <= 32) {
    for (uint32_t x = 1; x < len; x++) {
      const uint32_t v = o[x];
      uint32_t y = x;
      while (y > 0 && depth_less(keys64, v, o[y - 1])) { o[y] = o[y - 1]; y--; }
      o[y] = v;
    }
    return;
  }
  auto sift = [&](uint32_t root, uint32_t end) {
    while (2 * root + 1 < end) {
      uint32_t c = 2 * root + 1;
      if (c + 1 < end && depth_less(keys64, o[c], o[c + 1])) c++;
      if (!depth_less(keys64, o[root], o[c])) return;
      const uint32_t t = o[root]; o[root] = o[c]; o[c] = t;
      root = c;
    }
  };
  for (uint32_t st = len / 2; st-- > 0;) sift(st, len);
  for (uint32_t end = len - 1; end > 0; end--) {
    const uint32_t t = o[0]; o[0] = o[end]; o[end] = t;
    sift(0, end);
  }
}

// ------------------------------------------------------------------ tile order
// The blend kernels take tiles heaviest first (candidate-list length, log
// buckets): the long tiles start in the first wave instead of forming the
// grid's tail.  One block: bucket histogram, scan, scatter.
__global__ void __launch_bounds__(1024) tile_order_kernel(const uint2 *ranges, int tiles, uint32_t *order) {
  __shared__ uint32_t h[256], base[256];
  const int t = threadIdx.x;
  if (t < 256) h[t] = 0;
  __syncthreads();
  auto bucket = [&](int tile) {   // 255 - ~20 log2(len + 1): heavy tiles get small buckets
    const uint2 r = ranges[tile];
    const uint32_t len = r.y > r.x ? r.y - r.x : 0u;
    return 255 - min(255, (int)(20.f * __log2f((float)len + 1.f)));
  };
  for (int q = t; q < tiles; q += 1024) atomicAdd(&h[bucket(q)], 1u);
  __syncthreads();
  if (t < 32) {   // exclusive scan of the 256 buckets, 8 per lane
    uint32_t v[8], sum = 0;
#pragma unroll
    for (int i = 0; i < 8; i++) { v[i] = h[t * 8 + i]; sum += v[i]; }
    uint32_t inc = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t u = __shfl_up_sync(0xffffffffu, inc, o);
      if (t >= o) inc += u;
    }
    uint32_t run = inc - sum;
#pragma unroll
    for (int i = 0; i < 8; i++) { base[t * 8 + i] = run; run += v[i]; }
  }
  __syncthreads();
  for (int q = t; q < tiles; q += 1024) order[atomicAdd(&base[bucket(q)], 1u)] = (uint32_t)q;
}

// ------------------------------------------------------------------ orchestration
struct Scratch {
  uint64_t *dkeys_alt;
  uint32_t *dvals_alt;
  uint32_t *ptiles_alt;
  uint32_t *pids_alt;
  uint32_t *hist;       // [16][256]
  uint32_t *offsets;    // [16][256]
  uint32_t *lookback;   // depth passes then pair passes
  uint32_t *block_sums;
  size_t lookback_words;
};

uint32_t blend_mask_words(int64_t cap, int tiles) {
  return (uint32_t)(align_up((size_t)cap * sizeof(uint32_t), 256) / sizeof(uint32_t) / 32 + tiles + 2);
}

size_t scratch_bytes(int64_t n, int64_t cap, int pair_passes, int tiles, Scratch *sc, char *base) {
  size_t off = 0;
  auto take = [&](size_t bytes) { size_t o = off; off = align_up(off + bytes, 256); return base ? base + o : nullptr; };
  const size_t dchunks = (size_t)((n + kDepthChunk - 1) / kDepthChunk);
  const size_t pchunks = (size_t)((cap + kSortChunk - 1) / kSortChunk);
  const size_t lb_words = (8 * dchunks + pair_passes * pchunks) * kRadix;
  take(sizeof(uint32_t) * kMaxTileOrder);   // tile_order first: the blends find it at scratch + 0
  take(sizeof(uint32_t) * 8 * (size_t)blend_mask_words(cap, tiles));   // then the blend masks (blend_mask_offset)
  char *p0 = take(sizeof(uint64_t) * n);
  char *p1 = take(sizeof(uint32_t) * n);
  char *p2 = take(sizeof(uint32_t) * cap);
  char *p3 = take(sizeof(uint32_t) * cap);
  char *p4 = take(sizeof(uint32_t) * 16 * kRadix);
  char *p5 = take(sizeof(uint32_t) * 16 * kRadix);
  char *p6 = take(sizeof(uint32_t) * lb_words);
  char *p7 = take(sizeof(uint64_t) * ((n + kDupThreads * kDupRounds - 1) / (kDupThreads * kDupRounds) + 2));   // duplicate-scan look-back
  if (sc) {
    sc->dkeys_alt = (uint64_t *)p0; sc->dvals_alt = (uint32_t *)p1;
    sc->ptiles_alt = (uint32_t *)p2; sc->pids_alt = (uint32_t *)p3;
    sc->hist = (uint32_t *)p4; sc->offsets = (uint32_t *)p5; sc->lookback = (uint32_t *)p6;
    sc->block_sums = (uint32_t *)p7; sc->lookback_words = lb_words;
  }
  return off;
}

struct ClearList {
  uint2 *p[5];
  uint64_t n[5];   // 8-byte words
};
__global__ void __launch_bounds__(256) clear_kernel(ClearList c) {
  const uint64_t stride = (uint64_t)gridDim.x * 256;
  uint64_t i = (uint64_t)blockIdx.x * 256 + threadIdx.x;
#pragma unroll
  for (int r = 0; r < 5; r++) {
    for (; i < c.n[r]; i += stride) c.p[r][i] = make_uint2(0u, 0u);
    i -= c.n[r];
  }
}

int pair_sort_passes(int tiles) {
  int bits = 0;
  while ((1 << bits) < tiles) bits++;
  return bits == 0 ? 1 : (bits + kRadixBits - 1) / kRadixBits;
}

int launch_binning(const cs_camera &cam, const cs_settings &set, const cs_params &p,
                   const cs_layout &L, char *ws, int64_t cap, cudaStream_t s) {
  (void)cam; (void)set;
  const uint32_t n = (uint32_t)p.n;
  const int tiles = L.tiles_x * L.tiles_y;
  const int pp = pair_sort_passes(tiles);
  Scratch sc;
  scratch_bytes(p.n, cap, pp, tiles, &sc, ws + L.scratch);
  uint32_t *counters = reinterpret_cast<uint32_t *>(ws + L.counters);
  uint64_t *dkeys = reinterpret_cast<uint64_t *>(ws + L.depth_keys);
  uint32_t *order = reinterpret_cast<uint32_t *>(ws + L.order);
  uint32_t *touched = reinterpret_cast<uint32_t *>(ws + L.tiles_touched);
  uint32_t *offs = reinterpret_cast<uint32_t *>(ws + L.pair_offsets);
  uint32_t *ptiles = reinterpret_cast<uint32_t *>(ws + L.pair_tiles);
  uint32_t *pids = reinterpret_cast<uint32_t *>(ws + L.pair_ids);
  uint2 *ranges = reinterpret_cast<uint2 *>(ws + L.tile_ranges);

  // one clearing kernel instead of five memsets: digit histograms, look-back
  // flags, tile ranges (empty tiles and n == 0 read (0, 0)), scan block sums
  // and the sorts' dynamic chunk counters (so stage 1 can run again on its
  // own, e.g. a replayed stage-1 graph, without stage 0's counter reset)
  const uint32_t dchunks = (n + kDupThreads * kDupRounds - 1) / (kDupThreads * kDupRounds);
  {
    ClearList cl;
    cl.p[0] = reinterpret_cast<uint2 *>(sc.hist); cl.n[0] = sizeof(uint32_t) * 16 * kRadix / 8;
    cl.p[1] = reinterpret_cast<uint2 *>(sc.lookback); cl.n[1] = sizeof(uint32_t) * sc.lookback_words / 8;
    cl.p[2] = ranges; cl.n[2] = (uint64_t)tiles;
    cl.p[3] = reinterpret_cast<uint2 *>(sc.block_sums); cl.n[3] = dchunks;
    static_assert(C_CHUNK0 % 2 == 0 && (C_STATS - C_CHUNK0) % 2 == 0, "chunk counters: whole 8-byte words");
    cl.p[4] = reinterpret_cast<uint2 *>(counters + C_CHUNK0); cl.n[4] = (C_STATS - C_CHUNK0) / 2;
    const uint64_t total = cl.n[0] + cl.n[1] + cl.n[2] + cl.n[3] + cl.n[4];
    clear_kernel<<<(int)std::min<uint64_t>((total + 255) / 256, 148 * 8), 256, 0, s>>>(cl);
  }
  if (n > 0) {
    // depth order: 24-bit keys, 3 passes (odd: start in the alternate
    // buffers so the result ends in (keys32, order)), then the exact fix-up
    // of equal-key runs
    static_assert(kDepthPasses == 3, "odd pass count assumed below");
    uint32_t *k32 = reinterpret_cast<uint32_t *>(sc.dkeys_alt), *k32b = k32 + n;
#ifndef CS_KEY_BLOCKS_PER_SM
#define CS_KEY_BLOCKS_PER_SM 2   // fewer blocks, fewer histogram flushes: binning 243 -> 237 us (4: 238)
#endif
    const int kb = min((int)((n + kSortThreads - 1) / kSortThreads), 148 * CS_KEY_BLOCKS_PER_SM);
    depth_key32_kernel<<<kb, kSortThreads, 0, s>>>(dkeys, counters, n, k32b, sc.dvals_alt, sc.hist);
    radix_sort<uint32_t, kDepthSortItems>(k32b, sc.dvals_alt, k32, order, nullptr, kDepthBits + 1, n, n, kDepthPasses, 0, sc.hist,
                         sc.offsets, sc.lookback, counters + C_CHUNK0, true, s);
    depth_fixup_kernel<<<(n + 255) / 256, 256, 0, s>>>(dkeys, counters, k32, order);
    // pairs land in the buffer that makes the sorted result end in (ptiles, pids)
    uint32_t *dt = (pp & 1) ? sc.ptiles_alt : ptiles;
    uint32_t *di = (pp & 1) ? sc.pids_alt : pids;
    duplicate_scan_kernel<<<dchunks, kDupThreads, 0, s>>>(
        order, touched, reinterpret_cast<const int4 *>(ws + L.bbox), n, (uint32_t)cap, L.tiles_x, pp, dt, di,
        sc.hist + 8 * kRadix, offs, reinterpret_cast<unsigned long long *>(sc.block_sums), counters + C_CHUNK0 + 6,
        counters);
    if (cap > 0) {
      uint32_t *ka = (pp & 1) ? sc.ptiles_alt : ptiles, *va = (pp & 1) ? sc.pids_alt : pids;
      uint32_t *kb = (pp & 1) ? ptiles : sc.ptiles_alt, *vb = (pp & 1) ? pids : sc.pids_alt;
      int tile_bits = 0;
      while ((1 << tile_bits) < tiles) tile_bits++;
      radix_sort<uint32_t, kSortItems>(ka, va, kb, vb, counters + C_NSORT, tile_bits, 0, (uint32_t)cap, pp, 0, sc.hist + 8 * kRadix,
                           sc.offsets + 8 * kRadix, sc.lookback + 8 * ((n + kDepthChunk - 1) / kDepthChunk) * kRadix,
                           counters + C_CHUNK0 + 8, true, s);
    }
    const int rb = (int)std::min<int64_t>((cap + 1023) / 1024, 148 * 16);
    if (rb > 0) ranges_kernel<<<rb, 256, 0, s>>>(ptiles, counters, ranges);
  }
  if (tiles <= kMaxTileOrder)
    tile_order_kernel<<<1, 1024, 0, s>>>(ranges, tiles, reinterpret_cast<uint32_t *>(ws + L.scratch));
  return cudaGetLastError() == cudaSuccess ? CS_OK : CS_ERR_CUDA;
}

}  // namespace cs
