// tm_slab.cu — the time-slab view of the dual CSR for one window length.
//
// The reference answers every windowed-neighbour question with
// np.searchsorted over a node's WHOLE time-sorted run (kernels.py:251-276,
// txgraph.py:357-381).  On a B200 those runs are the problem: at the
// HI-Large shape (97-day horizon, 1-day windows) a node's run spans the whole
// horizon, so a window is a small piece of it — the bisection walks log2(run)
// dependent loads, and each 32-byte sector it touches holds entries from
// other days, so the windows of the ~150 K triggers in flight spread over the
// full 2 x 1.4 GB of CSR arrays (L2: 126 MB).
//
// The slab view cuts the time axis into n_slabs slabs of width W >= delta.
// Slab s owns the triggers with time in [t0 + s W, t0 + (s+1) W) — ranks
// [S_s, S_{s+1}) — and stores, per node, the sub-run of its edges with rank
// in [L_s, S_{s+1}), L_s = the first window start of those triggers
// (lo_tab[S_s]).  Every window of a slab-s trigger is a contiguous piece of
// that short sub-run, so the mining kernels (tm_mine.cu) read one slab's
// arrays — about (W + delta) / horizon of the edges, L2-resident — and bisect
// runs of a few entries.  With W >= delta an edge lands in at most two slabs
// (its own and, inside the halo, the next), so the view costs <= 2 E entries
// of 12 bytes per direction plus two [n_slabs][N+1] int32 tables.
//
// Build (streaming passes, no sort — the global runs are already sorted by
// (owner, rank, eid) and a slab run is a contiguous piece of a global run).
// The per-cell tables are written and read in owner-major [N+1][n_slabs]
// layout ("T"), where the slots of one owner touch adjacent cells; the
// slab-major [n_slabs][N+1] offsets ("S") the mining kernels use are
// produced tile by tile (32 owners x all slabs):
//   k_slab_bounds     S_s = lower_bound(uniq_time, t0 + s W), L_s = lo_tab[S_s]
//   k_slab_of         slab of every rank
//   k_slab_edges      per global CSR slot: the first / last slot of each slab
//                     run it opens / closes -> startT[x][s], endT[x][s]
//   k_slab_tile_sums  per tile and slab: entries (end - start) -> exclusive
//                     scan over (slab, tile) = every tile's offset
//   k_slab_tile_ptrs  per-slab prefix inside the tile -> ptrS, startS
//                     (slab-major) and deltaT = ptrS - startS (owner-major)
//   k_slab_fill       per global slot: its copies (nbr, prev, rank) at
//                     slot + deltaT[x][s] for its (at most two) slabs
#include <algorithm>
#include <cstdlib>

#include "tm_internal.cuh"

namespace tmb {
namespace {

constexpr int kB = 256;

__global__ void k_slab_bounds(const int64_t *__restrict__ uniq, int64_t R, long long t0, long long W,
                              int n_slabs, const uint32_t *__restrict__ lo_tab, uint32_t *__restrict__ S,
                              uint32_t *__restrict__ L) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s > n_slabs) return;
  int64_t r = R;
  if (s < n_slabs) {
    const long long x = t0 + (long long)s * W;
    int64_t a = 0, b = R;
    while (a < b) {
      const int64_t m = (a + b) >> 1;
      if (uniq[m] < x) a = m + 1; else b = m;
    }
    r = a;
  }
  S[s] = (uint32_t)r;
  L[s] = r < R ? lo_tab[r] : (uint32_t)R;
}

__global__ void k_slab_of(const uint32_t *__restrict__ S, int n_slabs, int64_t R, uint16_t *__restrict__ slab_of) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= R) return;
  int a = 0, b = n_slabs;  // last s with S[s] <= r
  while (b - a > 1) {
    const int m = (a + b) >> 1;
    if (__ldg(S + m) <= (uint32_t)r) a = m; else b = m;
  }
  slab_of[r] = (uint16_t)a;
}

// The slab of a rank from the slab starts staged in shared memory instead
// of the rank-indexed slab_of table: global slots are (owner, rank)-sorted,
// so slab_of[rank] is a random 2-byte load (a DRAM sector per slot) in the
// build kernels.  sS[i] = S[sb + i] for slabs sb .. s1 + 1; the result is
// the last s in [sb, s1] with S[s] <= r (callers pass r >= S[sb]).
#ifndef TM_EDGES_HOIST  // 1: full-view edge passes load the 4 owners with the 4 ranks
#define TM_EDGES_HOIST 1
#endif
#ifndef TM_FILL_HOIST  // 1: full-view fills load owner / (nbr, prev) with the rank
#define TM_FILL_HOIST 1
#endif
#ifndef TM_SLAB_SEARCH
#define TM_SLAB_SEARCH 1
#endif
__device__ __forceinline__ int slab_in_smem(const uint32_t *sS, int sb, int s1, uint32_t r) {
  int a = 0, b = s1 - sb + 1;  // answer index in [a, b)
  while (b - a > 1) {
    const int m = (a + b) >> 1;
    if (sS[m] <= r) a = m; else b = m;
  }
  return sb + a;
}
// stage S[sb .. s1 + 1] (sb = max(s0 - 1, 0): a slot's home slab can be the
// one before s0 when only its halo copy is built)
__device__ __forceinline__ int stage_slab_starts(uint32_t *sS, const uint32_t *__restrict__ S, int s0, int s1) {
  const int sb = s0 > 0 ? s0 - 1 : 0;
  for (int i = threadIdx.x; i <= s1 + 1 - sb; i += blockDim.x) sS[i] = __ldg(S + sb + i);
  return sb;
}

// slab s holds global slot j (rank r) iff L_s <= r < S_{s+1}; the slabs of
// r are [slab_of(r), ...) while L_s <= r (two at most when W >= delta).
// Cells are owner-major: cell (x, s) = x * ns + s.
// Only slabs [s0, s1] are built (a prepared view covers the slabs of one
// rank's trigger range); cell column of slab s = s - s0, ns = s1 - s0 + 1.
// One thread per 4 consecutive global slots (one 16-byte rank load): a
// prepared view of 1/N of the slabs skips most slots after that load.
__device__ __forceinline__ void slab_edge_slot(int64_t j, uint32_t r, const int32_t *__restrict__ owner,
                                               const uint32_t *__restrict__ rnk, const int32_t *__restrict__ ptr,
                                               int s0, int s1, const uint16_t *__restrict__ slab_of,
                                               const uint32_t *__restrict__ S, const uint32_t *__restrict__ L,
                                               int32_t *__restrict__ startT, int32_t *__restrict__ endT,
                                               const uint32_t *sS, int sb, int x) {
#if TM_SLAB_SEARCH
  int s = slab_in_smem(sS, sb, s1, r);
#else
  int s = __ldg(slab_of + r);
#endif
  if (x < 0) x = __ldg(owner + j);
  const int a = __ldg(ptr + x), b = __ldg(ptr + x + 1);
  const uint32_t rp = j > a ? __ldg(rnk + j - 1) : 0u;
  const uint32_t rn = j + 1 < b ? __ldg(rnk + j + 1) : 0xffffffffu;
  const int ns = s1 - s0 + 1;
  int32_t *st = startT + (int64_t)x * ns - s0, *en = endT + (int64_t)x * ns - s0;
  for (s = max(s, s0); s <= s1 && __ldg(L + s) <= r; ++s) {
    if (j == a || rp < __ldg(L + s)) st[s] = (int32_t)j;          // opens x's run in slab s
    if (j + 1 == b || rn >= __ldg(S + s + 1)) en[s] = (int32_t)(j + 1);  // closes it
  }
}

__global__ void k_slab_edges(const int32_t *__restrict__ owner, const uint32_t *__restrict__ rnk,
                             const int32_t *__restrict__ ptr, int64_t E, int s0, int s1,
                             const uint16_t *__restrict__ slab_of, const uint32_t *__restrict__ S,
                             const uint32_t *__restrict__ L, int32_t *__restrict__ startT,
                             int32_t *__restrict__ endT) {
  __shared__ uint32_t sS[kMaxSlabs + 2];
  const int sb = stage_slab_starts(sS, S, s0, s1);
  __syncthreads();
  const int64_t j0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4;
  if (j0 >= E) return;
  const uint32_t r_lo = __ldg(L + s0), r_hi = __ldg(S + s1 + 1);  // ranks held by slabs s0..s1
  uint32_t r4[4];
  int x4[4] = {-1, -1, -1, -1};  // owners (-1: loaded per slot)
  if (j0 + 4 <= E) {  // rank arrays are 16-byte aligned (device buffers)
    const uint4 q = __ldg(reinterpret_cast<const uint4 *>(rnk + j0));
    r4[0] = q.x; r4[1] = q.y; r4[2] = q.z; r4[3] = q.w;
    if (TM_EDGES_HOIST && s0 == 0) {  // a full view: every slot is in range
      const int4 o = __ldg(reinterpret_cast<const int4 *>(owner + j0));
      x4[0] = o.x; x4[1] = o.y; x4[2] = o.z; x4[3] = o.w;
    }
  } else {
#pragma unroll
    for (int k = 0; k < 4; ++k) r4[k] = j0 + k < E ? __ldg(rnk + j0 + k) : 0xffffffffu;
  }
#pragma unroll
  for (int k = 0; k < 4; ++k)
    if (j0 + k < E && r4[k] >= r_lo && r4[k] < r_hi)
      slab_edge_slot(j0 + k, r4[k], owner, rnk, ptr, s0, s1, slab_of, S, L, startT, endT, sS, sb, x4[k]);
}

// The slab-major offsets ptrS[s][x] = (entries of slabs < s) + (entries of
// slab s owned by nodes < x) are computed straight from the owner-major
// start / end tables, tile by tile (32 owners x all slabs, one contiguous
// block of each table): k_slab_tile_sums sums each slab column of a tile,
// one exclusive scan over the (slab, tile) sums gives every tile's offset,
// and k_slab_tile_ptrs runs the per-column prefix inside the tile and
// writes ptrS / startS (slab-major, through shared memory) and deltaT
// (owner-major) = ptr - start, the shift of a slot's copy in slab s.
constexpr int kTX = 32;            // owners per tile
constexpr int kTileThreads = 256;
__global__ void __launch_bounds__(kTileThreads) k_slab_tile_sums(const int32_t *__restrict__ startT,
                                                                 const int32_t *__restrict__ endT, int64_t rows,
                                                                 int ns, int64_t ntiles,
                                                                 uint32_t *__restrict__ tsum) {
  __shared__ uint32_t col[128];
  for (int i = threadIdx.x; i < ns; i += kTileThreads) col[i] = 0;
  __syncthreads();
  const int64_t x0 = (int64_t)blockIdx.x * kTX;
  const int nr = (int)(rows - x0 < kTX ? rows - x0 : kTX);
  const int64_t base = x0 * ns;
  for (int k = threadIdx.x; k < nr * ns; k += kTileThreads) {
    const int32_t len = endT[base + k] - startT[base + k];
    if (len) atomicAdd(&col[k % ns], (uint32_t)len);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < ns; i += kTileThreads) tsum[(int64_t)i * ntiles + blockIdx.x] = col[i];
}

__global__ void __launch_bounds__(kTileThreads) k_slab_tile_ptrs(
    const int32_t *__restrict__ startT, const int32_t *__restrict__ endT, int64_t rows, int ns, int64_t ntiles,
    const uint32_t *__restrict__ toff, int32_t *__restrict__ ptrS, int32_t *__restrict__ startS,
    int32_t *__restrict__ deltaT) {
  __shared__ int32_t st[kTX][129], pt[kTX][129];
  const int64_t x0 = (int64_t)blockIdx.x * kTX;
  const int nr = (int)(rows - x0 < kTX ? rows - x0 : kTX);
  const int64_t base = x0 * ns;
  for (int k = threadIdx.x; k < nr * ns; k += kTileThreads) {  // coalesced block reads
    const int r = k / ns, c = k - r * ns;
    const int32_t a = startT[base + k];
    st[r][c] = a;
    pt[r][c] = endT[base + k] - a;
  }
  __syncthreads();
  for (int c = threadIdx.x; c < ns; c += kTileThreads) {  // per-slab prefix over the tile's owners
    int32_t run = (int32_t)toff[(int64_t)c * ntiles + blockIdx.x];
    for (int r = 0; r < nr; ++r) {
      const int32_t len = pt[r][c];
      pt[r][c] = run;
      run += len;
    }
  }
  __syncthreads();
  for (int k = threadIdx.x; k < nr * ns; k += kTileThreads) {  // owner-major shift, coalesced
    const int r = k / ns, c = k - r * ns;
    deltaT[base + k] = pt[r][c] - st[r][c];
  }
  for (int k = threadIdx.x; k < kTX * ns; k += kTileThreads) {  // slab-major rows, owners fastest
    const int c = k / kTX, r = k - c * kTX;
    if (r < nr) {
      ptrS[(int64_t)c * rows + x0 + r] = pt[r][c];
      startS[(int64_t)c * rows + x0 + r] = st[r][c];
    }
  }
}

// The copies of a tile of consecutive global slots that land in one slab
// form ONE contiguous range of that slab's output (slab runs keep the global
// (owner, rank) order), so the tile is regrouped by slab in shared memory —
// position = chunk offset of the slab + (dest - first dest of the slab) — and
// every slab chunk leaves in coalesced stores (the direct per-slot scatter
// wrote 12-byte pieces into ~100 slab regions per warp: 7.5 ms per direction
// at HI-Large).
#ifndef TM_FILL_THREADS
#define TM_FILL_THREADS 1024  // measured: 1024 x 2 slots 80.7 ms, 512 x 4 81.7, 256 x 8 83.3, 1024 x 4 83.0 (HI-Large call)
#endif
#ifndef TM_FILL_PER
#define TM_FILL_PER 2
#endif
constexpr int kFillThreads = TM_FILL_THREADS;
constexpr int kFillPer = TM_FILL_PER;                 // global slots per thread
constexpr int kFillTile = kFillThreads * kFillPer;   // 2048 global slots per block
constexpr int kFillItems = 2 * kFillTile;    // at most two copies per slot
constexpr int kMaxSlabBins = 128;            // kMaxSlabs
__global__ void __launch_bounds__(kFillThreads) k_slab_fill(
    const int32_t *__restrict__ owner, const uint32_t *__restrict__ rnk, const int2 *__restrict__ np,
    int64_t E, int s0, int s1, const uint16_t *__restrict__ slab_of, const uint32_t *__restrict__ L,
    const uint32_t *__restrict__ S_next, const int32_t *__restrict__ deltaT, int2 *__restrict__ snp,
    uint32_t *__restrict__ srnk) {
  const int ns = s1 - s0 + 1;  // bins / cell columns: slab - s0
  extern __shared__ unsigned char fill_smem[];
  int2 *b_np = reinterpret_cast<int2 *>(fill_smem);                       // [kFillItems]
  uint32_t *b_rk = reinterpret_cast<uint32_t *>(b_np + kFillItems);      // [kFillItems]
  int32_t *b_dst = reinterpret_cast<int32_t *>(b_rk + kFillItems);       // [kFillItems]
  __shared__ int32_t cnt[kMaxSlabBins], first[kMaxSlabBins], off[kMaxSlabBins + 1];
  __shared__ uint32_t sS[kMaxSlabBins + 2];
  const int sb = stage_slab_starts(sS, S_next - 1, s0, s1);
  for (int i = threadIdx.x; i < ns; i += kFillThreads) {
    cnt[i] = 0;
    first[i] = INT32_MAX;
  }
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * kFillTile;
  const uint32_t r_lo = __ldg(L + s0), r_hi = __ldg(S_next + s1);  // ranks held by slabs s0..s1
  // pass 1: load the thread's slots (kept in registers), per-slab counts and
  // first destinations; a slot's copies: home slab s0 and, inside the next
  // slab's halo, s0 + 1
  int2 e[kFillPer];
  uint32_t r[kFillPer];
  int b0[kFillPer], d0[kFillPer], d1[kFillPer];  // bin of the first copy, its / the next bin's destination
  int xo[kFillPer];
  // a full view (s0 == 0) copies every slot: its owner and (nbr, prev) are
  // loaded with its rank, off the rank -> slab -> offset chain
  const bool hoist = TM_FILL_HOIST && s0 == 0;
#pragma unroll
  for (int k = 0; k < kFillPer; ++k) {
    const int64_t j = base + k * kFillThreads + threadIdx.x;
    r[k] = j < E ? __ldg(rnk + j) : 0xffffffffu;
    if (hoist && j < E) {
      xo[k] = __ldg(owner + j);
      e[k] = __ldg(np + j);
    }
  }
#pragma unroll
  for (int k = 0; k < kFillPer; ++k) {
    const int64_t j = base + k * kFillThreads + threadIdx.x;
    b0[k] = -1;
    if (j < E) {
      if (r[k] < r_lo || r[k] >= r_hi) continue;  // in no built slab
#if TM_SLAB_SEARCH
      const int s = slab_in_smem(sS, sb, s1, r[k]);
#else
      const int s = __ldg(slab_of + r[k]);
#endif
      // copies in slabs s (home) and s + 1 (inside its halo), clipped to [s0, s1]
      const bool home = s >= s0 && s <= s1;
      const bool next = s + 1 >= s0 && s + 1 <= s1 && __ldg(L + s + 1) <= r[k];
      if (home || next) {
        int x;
        if (hoist) {
          x = xo[k];
        } else {
          x = __ldg(owner + j);
          e[k] = __ldg(np + j);
        }
        const int32_t *dt = deltaT + (int64_t)x * ns - s0;
        if (home) {
          b0[k] = s - s0;
          d0[k] = (int32_t)(j + __ldg(dt + s));
          d1[k] = next ? (int32_t)(j + __ldg(dt + s + 1)) : -1;
        } else {  // only the halo copy
          b0[k] = s + 1 - s0;
          d0[k] = (int32_t)(j + __ldg(dt + s + 1));
          d1[k] = -1;
        }
      }
    }
  }
  bool any = false;
#pragma unroll
  for (int k = 0; k < kFillPer; ++k) any |= b0[k] >= 0;
  if (!__syncthreads_or(any)) return;  // a tile outside the prepared range
#pragma unroll
  for (int k = 0; k < kFillPer; ++k) {
    if (b0[k] < 0) continue;
    atomicAdd(&cnt[b0[k]], 1);
    atomicMin(&first[b0[k]], d0[k]);
    if (d1[k] >= 0) {
      atomicAdd(&cnt[b0[k] + 1], 1);
      atomicMin(&first[b0[k] + 1], d1[k]);
    }
  }
  __syncthreads();
  if (threadIdx.x < 32) {  // exclusive scan of the (<= 128) slab counts by warp 0
    int run = 0;
    for (int c0 = 0; c0 < ns; c0 += 32) {
      const int s = c0 + threadIdx.x;
      const int v = s < ns ? cnt[s] : 0;
      int inc = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, inc, o);
        if ((int)threadIdx.x >= o) inc += y;
      }
      if (s < ns) off[s] = run + inc - v;
      run += __shfl_sync(0xffffffffu, inc, 31);
    }
    if (threadIdx.x == 0) off[ns] = run;
  }
  __syncthreads();
  // pass 2: stage every copy at off[s] + (dest - first[s])
#pragma unroll
  for (int k = 0; k < kFillPer; ++k) {
    if (b0[k] < 0) continue;
    int q = off[b0[k]] + (d0[k] - first[b0[k]]);
    b_np[q] = e[k];
    b_rk[q] = r[k];
    b_dst[q] = d0[k];
    if (d1[k] >= 0) {
      q = off[b0[k] + 1] + (d1[k] - first[b0[k] + 1]);
      b_np[q] = e[k];
      b_rk[q] = r[k];
      b_dst[q] = d1[k];
    }
  }
  __syncthreads();
  // pass 3: consecutive staged copies of one slab have consecutive destinations
  const int total = off[ns];
  for (int q = threadIdx.x; q < total; q += kFillThreads) {
    const int32_t d = b_dst[q];
    snp[d] = b_np[q];
    srnk[d] = b_rk[q];
  }
}

}  // namespace

int build_slab_view(tm_graph *g, SlabIndex &si, int64_t delta, const uint32_t *lo_tab, cudaStream_t s,
                    int64_t trig_lo, int64_t trig_hi, bool restrict_range, DevGraph *view,
                    const uint16_t **slab_of, int64_t *stride) {
  *view = g->dev();
  *slab_of = nullptr;
  *stride = 0;
  const char *env = getenv("TM_SLABS");  // TM_SLABS=0 / 1: force the global / slab view (A/B)
  if (env && env[0] == '0') return TM_OK;
  const bool force = env && env[0] == '1';
  const int64_t E = g->n_edges, N = g->n_nodes, R = g->n_ranks;
  if (E == 0 || R == 0) return TM_OK;
  // The view pays off when the global runs are long (the bisections and the
  // L2 footprint it saves grow with the mean run length E/N): measured a
  // win at the HI-Large shape (E/N = 85: 144 -> 100 ms per call), a loss at
  // HI-Small / HI-Medium (E/N = 10 / 15: 2.9 -> 3.6, 17.4 -> 19.3 ms) and
  // at short windows (many slabs: 1-h windows on HI-Medium 1.2 -> 10 ms).
  if (!force && E < kSlabMinRun * N) return TM_OK;
  const int64_t span = g->t_span + 1;  // ticks covered by the distinct times
  // slab width >= delta (an edge then lands in at most two slabs);
  // TM_SLAB_WMULT=k widens slabs to >= k delta (A/B: fewer cells, larger views)
  int64_t wmult = 1;
  if (const char *wm = getenv("TM_SLAB_WMULT")) wmult = std::max<int64_t>(1, atoll(wm));
  const int64_t w_min = std::max<int64_t>(delta, 1) * wmult;
  int64_t n = span / w_min;
  if (n > kMaxSlabs) n = kMaxSlabs;
  if (n < kMinSlabs) return TM_OK;
  const int n_slabs = (int)n;
  const int64_t W = (span + n_slabs - 1) / n_slabs;  // >= delta
  const int64_t N1 = N + 1;
  if (!force && (int64_t)n_slabs * N1 > 2 * E) return TM_OK;  // cell tables would outweigh the entries
  // entries are addressed by int32 offsets: at most 2 E of them when W >= delta
  if (2 * E >= (int64_t)INT32_MAX || (int64_t)n_slabs * N1 >= (int64_t)INT32_MAX) return TM_OK;
  si.n_slabs = n_slabs;
  int rc;
  if ((rc = si.slab_of.ensure_pooled(sizeof(uint16_t) * (size_t)R, s, g->stream)) ||
      (rc = si.bounds.ensure_pooled(sizeof(uint32_t) * 2 * (size_t)(n_slabs + 1), s, g->stream)))
    return rc;
  uint32_t *S = si.bounds.as<uint32_t>(), *L = S + (n_slabs + 1);
  k_slab_bounds<<<grid_for(n_slabs + 1, kB), kB, 0, s>>>(g->uniq_time.as<int64_t>(), R, (long long)g->t_min,
                                                         (long long)W, n_slabs, lo_tab, S, L);
  TM_LAUNCHED("k_slab_bounds");
  k_slab_of<<<grid_for(R, kB), kB, 0, s>>>(S, n_slabs, R, si.slab_of.as<uint16_t>());
  TM_LAUNCHED("k_slab_of");
  // slabs built: all, or (a prepared view of time-ordered triggers [trig_lo,
  // trig_hi)) only those holding them — a rank of a multi-GPU run builds
  // the ~1/world of the view its triggers read (one host sync)
  int s0 = 0, s1 = n_slabs - 1;
  if (restrict_range && g->ids_time_ordered && trig_hi > trig_lo) {
    uint32_t r01[2];
    TM_CUDA(cudaMemcpyAsync(&r01[0], g->e_rank.as<uint32_t>() + trig_lo, 4, cudaMemcpyDeviceToHost, s));
    TM_CUDA(cudaMemcpyAsync(&r01[1], g->e_rank.as<uint32_t>() + trig_hi - 1, 4, cudaMemcpyDeviceToHost, s));
    uint16_t sl[2];
    TM_CUDA(cudaStreamSynchronize(s));  // r01 is needed to address slab_of
    TM_CUDA(cudaMemcpyAsync(&sl[0], si.slab_of.as<uint16_t>() + r01[0], 2, cudaMemcpyDeviceToHost, s));
    TM_CUDA(cudaMemcpyAsync(&sl[1], si.slab_of.as<uint16_t>() + r01[1], 2, cudaMemcpyDeviceToHost, s));
    TM_CUDA(cudaStreamSynchronize(s));
    s0 = sl[0];
    s1 = sl[1];
  }
  const int ns = s1 - s0 + 1;
  const int64_t cells = (int64_t)ns * N1;
  si.s0 = s0;
  // owner-major scratch, shared by both directions (stream-ordered)
  if ((rc = si.scratch.ensure_pooled(sizeof(int32_t) * 2 * (size_t)cells, s, g->stream))) return rc;
  int32_t *startT = si.scratch.as<int32_t>(), *endT = startT + cells;
  constexpr int kFillSmem = kFillItems * (sizeof(int2) + 2 * sizeof(int32_t));  // 64 KB
  TM_CUDA(cudaFuncSetAttribute(k_slab_fill, cudaFuncAttributeMaxDynamicSharedMemorySize, kFillSmem));
  for (int d = 0; d < 2; ++d) {
    if ((rc = si.start[d].ensure_pooled(sizeof(int32_t) * (size_t)cells, s, g->stream)) ||
        (rc = si.ptr[d].ensure_pooled(sizeof(int32_t) * (size_t)cells, s, g->stream)))
      return rc;
    int32_t *startS = si.start[d].as<int32_t>(), *ptr = si.ptr[d].as<int32_t>();
    // cells of owners without entries in a slab stay 0 - 0 (empty runs)
    TM_CUDA(cudaMemsetAsync(startT, 0, sizeof(int32_t) * 2 * (size_t)cells, s));
    k_slab_edges<<<grid_for((E + 3) / 4, kB), kB, 0, s>>>(g->owner[d].as<int32_t>(), g->rnk[d].as<uint32_t>(),
                                                g->ptr[d].as<int32_t>(), E, s0, s1,
                                                si.slab_of.as<uint16_t>(), S, L, startT, endT);
    TM_LAUNCHED("k_slab_edges");
    const int64_t ntiles = (N1 + kTX - 1) / kTX;
    uint32_t *tsum = nullptr;
    TM_CUDA(pool_malloc((void **)&tsum, sizeof(uint32_t) * (size_t)(ntiles * ns), s));
    k_slab_tile_sums<<<(unsigned)ntiles, kTileThreads, 0, s>>>(startT, endT, N1, ns, ntiles, tsum);
    TM_LAUNCHED("k_slab_tile_sums");
    if ((rc = exclusive_scan_u32(tsum, tsum, ntiles * ns, s))) return rc;
    int32_t *deltaT = startT;  // each tile reads its start / end block before writing it back
    k_slab_tile_ptrs<<<(unsigned)ntiles, kTileThreads, 0, s>>>(startT, endT, N1, ns, ntiles, tsum, ptr,
                                                                startS, deltaT);
    TM_LAUNCHED("k_slab_tile_ptrs");
    TM_CUDA(cudaFreeAsync(tsum, s));
    // W >= delta: an edge lands in at most two slabs, so 2 E entries bound
    // the view without reading the scan's total back (no host sync)
    si.entries[d] = 2 * E;
    if ((rc = si.np[d].ensure_pooled(sizeof(int2) * (size_t)(2 * E), s, g->stream)) ||
        (rc = si.rnk[d].ensure_pooled(sizeof(uint32_t) * (size_t)(2 * E), s, g->stream)))
      return rc;
    k_slab_fill<<<grid_for(E, kFillTile), kFillThreads, kFillSmem, s>>>(g->owner[d].as<int32_t>(), g->rnk[d].as<uint32_t>(),
                                               g->npk[d].as<int2>(), E, s0, s1, si.slab_of.as<uint16_t>(),
                                               L, S + 1, deltaT, si.np[d].as<int2>(), si.rnk[d].as<uint32_t>());
    TM_LAUNCHED("k_slab_fill");
    view->ptr[d] = ptr - (int64_t)s0 * N1;  // rows of slabs s0..s1, addressed by slab * (N + 1)
    view->np[d] = si.np[d].as<int2>();
    view->rnk[d] = si.rnk[d].as<uint32_t>();
    // only the global-CSR helpers may touch these in a slab view
    view->nbr[d] = nullptr;
    view->prev[d] = nullptr;
    view->eid[d] = nullptr;
    view->peid[d] = nullptr;
    view->owner[d] = nullptr;
  }
  *slab_of = si.slab_of.as<uint16_t>();
  *stride = N1;
  return TM_OK;
}

}  // namespace tmb
