// tm_sort.cu — stable LSD radix sort of (uint64 key, uint32 value) pairs and
// an exclusive scan, hand-written for sm_100a.
//
// This replaces the reference's np.lexsort calls (txgraph.py:135-136,151):
// lexsort((eid, time, node)) is a stable sort by the packed key
// (node << rank_bits | rank) of an input already in eid order, which is what
// an LSD radix sort computes.  Only the bits the key actually uses are
// sorted (8 bits per pass).
//
// Per pass: (1) per-tile digit histogram (warp __match_any_sync aggregation
// into shared memory), (2) exclusive scan of the digit-major
// [256 x tiles] count matrix -> every (digit, tile) output offset,
// (3) stable scatter: each warp ranks its 32-item steps with
// __match_any_sync + popc, warps are ordered by a shared-memory prefix, so
// the global order is (digit, tile, warp, step, lane) = stable.
#include "tm_internal.cuh"

namespace tmb {
namespace {

constexpr int kSortThreads = 256;
constexpr int kSortItems = 16;
constexpr int kTile = kSortThreads * kSortItems;  // 4096
constexpr int kWarps = kSortThreads / 32;
constexpr int kRadix = 256;

__global__ void __launch_bounds__(kSortThreads) k_digit_hist(const uint64_t *__restrict__ keys,
                                                             int64_t n, int shift, int64_t ntiles,
                                                             uint32_t *__restrict__ counts) {
  __shared__ uint32_t hist[kRadix];
  for (int i = threadIdx.x; i < kRadix; i += kSortThreads) hist[i] = 0;
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * kTile;
  const int lane = threadIdx.x & 31;
#pragma unroll 4
  for (int it = 0; it < kSortItems; ++it) {
    int64_t i = base + (int64_t)it * kSortThreads + threadIdx.x;
    bool valid = i < n;
    unsigned vmask = __ballot_sync(0xffffffffu, valid);
    if (valid) {
      unsigned d = (unsigned)(keys[i] >> shift) & 0xffu;
      unsigned peers = __match_any_sync(vmask, d);
      if ((peers & ((1u << lane) - 1)) == 0) atomicAdd(&hist[d], __popc(peers));
    }
  }
  __syncthreads();
  for (int d = threadIdx.x; d < kRadix; d += kSortThreads)
    counts[(int64_t)d * ntiles + blockIdx.x] = hist[d];
}

// Stable scatter, onesweep-style: every item's rank within its digit is
// computed as before (warp match + shared per-warp counts), the tile is then
// regrouped by digit in shared memory, and the digit runs leave in
// consecutive addresses (the direct scatter wrote 12 bytes per item into up
// to 256 regions per warp step).
__global__ void __launch_bounds__(kSortThreads) k_digit_scatter(
    const uint64_t *__restrict__ kin, const uint32_t *__restrict__ vin, uint64_t *__restrict__ kout,
    uint32_t *__restrict__ vout, int64_t n, int shift, int64_t ntiles,
    const uint32_t *__restrict__ offsets) {
  __shared__ uint32_t wcnt[kWarps][kRadix];
  __shared__ uint32_t goff[kRadix];
  __shared__ uint32_t loff[kRadix];  // digit's first slot in the regrouped tile
  extern __shared__ unsigned char scatter_smem[];
  uint64_t *sk = reinterpret_cast<uint64_t *>(scatter_smem);  // [kTile]
  uint32_t *sv = reinterpret_cast<uint32_t *>(sk + kTile);    // [kTile]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < kWarps * kRadix; i += kSortThreads) (&wcnt[0][0])[i] = 0;
  for (int d = threadIdx.x; d < kRadix; d += kSortThreads)
    goff[d] = offsets[(int64_t)d * ntiles + blockIdx.x];
  __syncthreads();

  // warp w owns items [w*512, (w+1)*512) of the tile, in 16 steps of 32
  const int64_t wbase = (int64_t)blockIdx.x * kTile + (int64_t)warp * (32 * kSortItems);
  uint64_t k[kSortItems];
  uint32_t v[kSortItems];
  uint32_t pos[kSortItems];
#pragma unroll
  for (int it = 0; it < kSortItems; ++it) {
    int64_t i = wbase + it * 32 + lane;
    bool valid = i < n;
    unsigned vmask = __ballot_sync(0xffffffffu, valid);
    pos[it] = 0xffffffffu;
    if (valid) {
      k[it] = kin[i];
      v[it] = vin[i];
      unsigned d = (unsigned)(k[it] >> shift) & 0xffu;
      unsigned peers = __match_any_sync(vmask, d);
      unsigned before = __popc(peers & ((1u << lane) - 1));
      pos[it] = wcnt[warp][d] + before;
      __syncwarp(vmask);
      if (before == 0) wcnt[warp][d] += __popc(peers);
    }
    __syncwarp();
  }
  __syncthreads();
  // per digit: exclusive prefix over warps (stable order) and the digit's
  // total -> loff = exclusive prefix of the totals over digits
  for (int d = threadIdx.x; d < kRadix; d += kSortThreads) {
    uint32_t run = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
      uint32_t c = wcnt[w][d];
      wcnt[w][d] = run;
      run += c;
    }
    loff[d] = run;  // total, scanned below
  }
  __syncthreads();
  if (threadIdx.x < 32) {  // exclusive scan of the 256 digit totals by warp 0
    uint32_t carry = 0;
    for (int c0 = 0; c0 < kRadix; c0 += 32) {
      const uint32_t x = loff[c0 + lane];
      uint32_t inc = x;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
      }
      loff[c0 + lane] = carry + inc - x;
      carry += __shfl_sync(0xffffffffu, inc, 31);
    }
  }
  __syncthreads();
#pragma unroll
  for (int it = 0; it < kSortItems; ++it) {
    if (pos[it] != 0xffffffffu) {
      unsigned d = (unsigned)(k[it] >> shift) & 0xffu;
      const uint32_t q = loff[d] + wcnt[warp][d] + pos[it];
      sk[q] = k[it];
      sv[q] = v[it];
    }
  }
  __syncthreads();
  const int64_t tile0 = (int64_t)blockIdx.x * kTile;
  const int nt = (int)(n - tile0 < kTile ? n - tile0 : kTile);
  for (int q = threadIdx.x; q < nt; q += kSortThreads) {
    const uint64_t key = sk[q];
    const unsigned d = (unsigned)(key >> shift) & 0xffu;
    const uint32_t o = goff[d] + (q - loff[d]);
    kout[o] = key;
    vout[o] = sv[q];
  }
}

// ------------------------------------------------------------------ scan

constexpr int kScanThreads = 1024;
constexpr int kScanItems = 4;
constexpr int kScanTile = kScanThreads * kScanItems;

__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t x, uint32_t *total) {
  __shared__ uint32_t warp_sums[kScanThreads / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t inc = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) warp_sums[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    uint32_t s = lane < kScanThreads / 32 ? warp_sums[lane] : 0;
    uint32_t si = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t y = __shfl_up_sync(0xffffffffu, si, o);
      if (lane >= o) si += y;
    }
    if (lane < kScanThreads / 32) warp_sums[lane] = si - s;
    if (lane == 31) *total = si;
  }
  __syncthreads();
  return warp_sums[warp] + inc - x;
}

__global__ void __launch_bounds__(kScanThreads) k_scan_tiles(const uint32_t *__restrict__ in,
                                                             uint32_t *__restrict__ out, int64_t n,
                                                             uint32_t *__restrict__ tile_sums) {
  __shared__ uint32_t total;
  const int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
  uint32_t x[kScanItems];
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    x[i] = base + i < n ? in[base + i] : 0;
    s += x[i];
  }
  uint32_t run = block_exclusive_scan(s, &total);
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    if (base + i < n) out[base + i] = run;
    run += x[i];
  }
  if (threadIdx.x == 0 && tile_sums) tile_sums[blockIdx.x] = total;
}

__global__ void k_scan_add(uint32_t *__restrict__ out, int64_t n, const uint32_t *__restrict__ add) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] += add[i / kScanTile];
}

}  // namespace

int exclusive_scan_u32(const uint32_t *in, uint32_t *out, int64_t n, cudaStream_t s) {
  if (n <= 0) return TM_OK;
  const int64_t tiles = (n + kScanTile - 1) / kScanTile;
  if (tiles == 1) {
    k_scan_tiles<<<1, kScanThreads, 0, s>>>(in, out, n, nullptr);
    TM_LAUNCHED("k_scan_tiles");
    return TM_OK;
  }
  uint32_t *sums = nullptr;
  TM_CUDA(pool_malloc((void **)&sums, sizeof(uint32_t) * tiles, s));
  k_scan_tiles<<<(unsigned)tiles, kScanThreads, 0, s>>>(in, out, n, sums);
  TM_LAUNCHED("k_scan_tiles");
  int rc = exclusive_scan_u32(sums, sums, tiles, s);
  if (rc) return rc;
  k_scan_add<<<grid_for(n, 256), 256, 0, s>>>(out, n, sums);
  TM_LAUNCHED("k_scan_add");
  TM_CUDA(cudaFreeAsync(sums, s));
  return TM_OK;
}

int radix_sort_pairs(uint64_t *keys, uint32_t *vals, uint64_t *ktmp, uint32_t *vtmp, int64_t n,
                     int nbits, cudaStream_t s, uint64_t **kout, uint32_t **vout) {
  *kout = keys;
  *vout = vals;
  if (n <= 1 || nbits <= 0) return TM_OK;
  const int64_t ntiles = (n + kTile - 1) / kTile;
  uint32_t *counts = nullptr;
  TM_CUDA(pool_malloc((void **)&counts, sizeof(uint32_t) * kRadix * ntiles, s));
  constexpr int kScatterSmem = kTile * (sizeof(uint64_t) + sizeof(uint32_t));  // 48 KB
  TM_CUDA(cudaFuncSetAttribute(k_digit_scatter, cudaFuncAttributeMaxDynamicSharedMemorySize, kScatterSmem));
  uint64_t *ka = keys, *kb = ktmp;
  uint32_t *va = vals, *vb = vtmp;
  for (int shift = 0; shift < nbits; shift += 8) {
    k_digit_hist<<<(unsigned)ntiles, kSortThreads, 0, s>>>(ka, n, shift, ntiles, counts);
    TM_LAUNCHED("k_digit_hist");
    int rc = exclusive_scan_u32(counts, counts, kRadix * ntiles, s);
    if (rc) return rc;
    k_digit_scatter<<<(unsigned)ntiles, kSortThreads, kScatterSmem, s>>>(ka, va, kb, vb, n, shift, ntiles,
                                                                         counts);
    TM_LAUNCHED("k_digit_scatter");
    uint64_t *kt = ka; ka = kb; kb = kt;
    uint32_t *vt = va; va = vb; vb = vt;
  }
  TM_CUDA(cudaFreeAsync(counts, s));
  *kout = ka;
  *vout = va;
  return TM_OK;
}

}  // namespace tmb
