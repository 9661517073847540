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
// layout ("T"), where the slots of one owner touch adjacent cells, and
// transposed through shared memory to the slab-major [n_slabs][N+1] layout
// ("S") the scan and the mining kernels use:
//   k_slab_bounds     S_s = lower_bound(uniq_time, t0 + s W), L_s = lo_tab[S_s]
//   k_slab_of         slab of every rank
//   k_slab_edges      per global CSR slot: the first / last slot of each slab
//                     run it opens / closes -> startT[x][s], endT[x][s]
//   k_slab_transpose  lenS = endT - startT, startS = startT (slab-major)
//   exclusive scan    lenS -> ptrS (slab run offsets)
//   k_slab_delta      deltaT[x][s] = ptrS - startS (owner-major again)
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

// slab s holds global slot j (rank r) iff L_s <= r < S_{s+1}; the slabs of
// r are [slab_of(r), ...) while L_s <= r (two at most when W >= delta).
// Cells are owner-major: cell (x, s) = x * ns + s.
__global__ void k_slab_edges(const int32_t *__restrict__ owner, const uint32_t *__restrict__ rnk,
                             const int32_t *__restrict__ ptr, int64_t E, int ns,
                             const uint16_t *__restrict__ slab_of, const uint32_t *__restrict__ S,
                             const uint32_t *__restrict__ L, int32_t *__restrict__ startT,
                             int32_t *__restrict__ endT) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= E) return;
  const int x = __ldg(owner + j);
  const uint32_t r = __ldg(rnk + j);
  const int a = __ldg(ptr + x), b = __ldg(ptr + x + 1);
  const uint32_t rp = j > a ? __ldg(rnk + j - 1) : 0u;
  const uint32_t rn = j + 1 < b ? __ldg(rnk + j + 1) : 0xffffffffu;
  int32_t *st = startT + (int64_t)x * ns, *en = endT + (int64_t)x * ns;
  for (int s = __ldg(slab_of + r); s < ns && __ldg(L + s) <= r; ++s) {
    if (j == a || rp < __ldg(L + s)) st[s] = (int32_t)j;          // opens x's run in slab s
    if (j + 1 == b || rn >= __ldg(S + s + 1)) en[s] = (int32_t)(j + 1);  // closes it
  }
}

// owner-major [rows][ns] -> slab-major [ns][rows] through a 32 x 32 shared tile:
// lenS = endT - startT, startS = startT
constexpr int kTT = 32;
__global__ void k_slab_transpose(const int32_t *__restrict__ startT, const int32_t *__restrict__ endT,
                                 int64_t rows, int ns, uint32_t *__restrict__ lenS,
                                 int32_t *__restrict__ startS) {
  __shared__ int32_t ts[kTT][kTT + 1], tl[kTT][kTT + 1];
  const int64_t x0 = (int64_t)blockIdx.x * kTT;
  const int s0 = blockIdx.y * kTT;
  for (int i = threadIdx.y; i < kTT; i += blockDim.y) {  // read rows x0 + i, columns s0 + tx
    const int64_t x = x0 + i;
    const int s = s0 + threadIdx.x;
    if (x < rows && s < ns) {
      const int32_t a = startT[x * ns + s];
      ts[i][threadIdx.x] = a;
      tl[i][threadIdx.x] = endT[x * ns + s] - a;
    }
  }
  __syncthreads();
  for (int i = threadIdx.y; i < kTT; i += blockDim.y) {  // write rows s0 + i, columns x0 + tx
    const int s = s0 + i;
    const int64_t x = x0 + threadIdx.x;
    if (x < rows && s < ns) {
      lenS[(int64_t)s * rows + x] = (uint32_t)tl[threadIdx.x][i];
      startS[(int64_t)s * rows + x] = ts[threadIdx.x][i];
    }
  }
}

// deltaT[x][s] = ptrS[s][x] - startS[s][x]: a slot j of x in slab s lands at j + deltaT
__global__ void k_slab_delta(const int32_t *__restrict__ ptrS, const int32_t *__restrict__ startS,
                             int64_t rows, int ns, int32_t *__restrict__ deltaT) {
  __shared__ int32_t td[kTT][kTT + 1];
  const int64_t x0 = (int64_t)blockIdx.x * kTT;
  const int s0 = blockIdx.y * kTT;
  for (int i = threadIdx.y; i < kTT; i += blockDim.y) {  // read rows s0 + i, columns x0 + tx
    const int s = s0 + i;
    const int64_t x = x0 + threadIdx.x;
    if (x < rows && s < ns) {
      const int64_t c = (int64_t)s * rows + x;
      td[i][threadIdx.x] = ptrS[c] - startS[c];
    }
  }
  __syncthreads();
  for (int i = threadIdx.y; i < kTT; i += blockDim.y) {  // write rows x0 + i, columns s0 + tx
    const int64_t x = x0 + i;
    const int s = s0 + threadIdx.x;
    if (x < rows && s < ns) deltaT[x * ns + s] = td[threadIdx.x][i];
  }
}

// The copies of a tile of consecutive global slots that land in one slab
// form ONE contiguous range of that slab's output (slab runs keep the global
// (owner, rank) order), so the tile is regrouped by slab in shared memory —
// position = chunk offset of the slab + (dest - first dest of the slab) — and
// every slab chunk leaves in coalesced stores (the direct per-slot scatter
// wrote 12-byte pieces into ~100 slab regions per warp: 7.5 ms per direction
// at HI-Large).
constexpr int kFillThreads = 512;
constexpr int kFillPer = 4;                           // global slots per thread
constexpr int kFillTile = kFillThreads * kFillPer;   // 2048 global slots per block
constexpr int kFillItems = 2 * kFillTile;    // at most two copies per slot
constexpr int kMaxSlabBins = 128;            // kMaxSlabs
__global__ void __launch_bounds__(kFillThreads) k_slab_fill(
    const int32_t *__restrict__ owner, const uint32_t *__restrict__ rnk, const int2 *__restrict__ np,
    int64_t E, int ns, const uint16_t *__restrict__ slab_of, const uint32_t *__restrict__ L,
    const int32_t *__restrict__ deltaT, int2 *__restrict__ snp, uint32_t *__restrict__ srnk) {
  extern __shared__ unsigned char fill_smem[];
  int2 *b_np = reinterpret_cast<int2 *>(fill_smem);                       // [kFillItems]
  uint32_t *b_rk = reinterpret_cast<uint32_t *>(b_np + kFillItems);      // [kFillItems]
  int32_t *b_dst = reinterpret_cast<int32_t *>(b_rk + kFillItems);       // [kFillItems]
  __shared__ int32_t cnt[kMaxSlabBins], first[kMaxSlabBins], off[kMaxSlabBins + 1];
  for (int i = threadIdx.x; i < ns; i += kFillThreads) {
    cnt[i] = 0;
    first[i] = INT32_MAX;
  }
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * kFillTile;
  // pass 1: load the thread's slots (kept in registers), per-slab counts and
  // first destinations; a slot's copies: home slab s0 and, inside the next
  // slab's halo, s0 + 1
  int2 e[kFillPer];
  uint32_t r[kFillPer];
  int s0[kFillPer], d0[kFillPer], d1[kFillPer];
#pragma unroll
  for (int k = 0; k < kFillPer; ++k) {
    const int64_t j = base + k * kFillThreads + threadIdx.x;
    s0[k] = -1;
    if (j < E) {
      const int x = __ldg(owner + j);
      r[k] = __ldg(rnk + j);
      e[k] = __ldg(np + j);
      const int32_t *dt = deltaT + (int64_t)x * ns;
      const int s = __ldg(slab_of + r[k]);
      s0[k] = s;
      d0[k] = (int32_t)(j + __ldg(dt + s));
      d1[k] = (s + 1 < ns && __ldg(L + s + 1) <= r[k]) ? (int32_t)(j + __ldg(dt + s + 1)) : -1;
    }
  }
#pragma unroll
  for (int k = 0; k < kFillPer; ++k) {
    if (s0[k] < 0) continue;
    atomicAdd(&cnt[s0[k]], 1);
    atomicMin(&first[s0[k]], d0[k]);
    if (d1[k] >= 0) {
      atomicAdd(&cnt[s0[k] + 1], 1);
      atomicMin(&first[s0[k] + 1], d1[k]);
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
    if (s0[k] < 0) continue;
    int q = off[s0[k]] + (d0[k] - first[s0[k]]);
    b_np[q] = e[k];
    b_rk[q] = r[k];
    b_dst[q] = d0[k];
    if (d1[k] >= 0) {
      q = off[s0[k] + 1] + (d1[k] - first[s0[k] + 1]);
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

int build_slab_view(tm_graph *g, int k, int64_t delta, const uint32_t *lo_tab, cudaStream_t s,
                    DevGraph *view, const uint16_t **slab_of, int64_t *stride) {
  *view = g->dev();
  *slab_of = nullptr;
  *stride = 0;
  const char *env = getenv("TM_SLABS");  // TM_SLABS=0: global view (A/B)
  if (env && env[0] == '0') return TM_OK;
  const int64_t E = g->n_edges, N = g->n_nodes, R = g->n_ranks;
  if (E == 0 || R == 0) return TM_OK;
  const int64_t span = g->t_span + 1;  // ticks covered by the distinct times
  const int64_t w_min = std::max<int64_t>(delta, 1);
  int64_t n = span / w_min;
  if (n > kMaxSlabs) n = kMaxSlabs;
  if (n < kMinSlabs) return TM_OK;
  const int n_slabs = (int)n;
  const int64_t W = (span + n_slabs - 1) / n_slabs;  // >= delta
  const int64_t N1 = N + 1;
  const int64_t cells = (int64_t)n_slabs * N1;
  // entries are addressed by int32 offsets: at most 2 E of them when W >= delta
  if (2 * E >= (int64_t)INT32_MAX || cells >= (int64_t)INT32_MAX) return TM_OK;
  SlabIndex &si = g->slabs[k];
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
  // owner-major scratch, shared by both directions (stream-ordered)
  if ((rc = si.scratch.ensure_pooled(sizeof(int32_t) * 2 * (size_t)cells, s, g->stream))) return rc;
  int32_t *startT = si.scratch.as<int32_t>(), *endT = startT + cells;
  constexpr int kFillSmem = kFillItems * (sizeof(int2) + 2 * sizeof(int32_t));  // 64 KB
  TM_CUDA(cudaFuncSetAttribute(k_slab_fill, cudaFuncAttributeMaxDynamicSharedMemorySize, kFillSmem));
  const dim3 tgrid((unsigned)((N1 + kTT - 1) / kTT), (unsigned)((n_slabs + kTT - 1) / kTT)), tblock(kTT, 8);
  for (int d = 0; d < 2; ++d) {
    if ((rc = si.start[d].ensure_pooled(sizeof(int32_t) * (size_t)cells, s, g->stream)) ||
        (rc = si.ptr[d].ensure_pooled(sizeof(int32_t) * (size_t)cells, s, g->stream)))
      return rc;
    int32_t *startS = si.start[d].as<int32_t>(), *ptr = si.ptr[d].as<int32_t>();
    // cells of owners without entries in a slab stay 0 - 0 (empty runs)
    TM_CUDA(cudaMemsetAsync(startT, 0, sizeof(int32_t) * 2 * (size_t)cells, s));
    k_slab_edges<<<grid_for(E, kB), kB, 0, s>>>(g->owner[d].as<int32_t>(), g->rnk[d].as<uint32_t>(),
                                                g->ptr[d].as<int32_t>(), E, n_slabs,
                                                si.slab_of.as<uint16_t>(), S, L, startT, endT);
    TM_LAUNCHED("k_slab_edges");
    k_slab_transpose<<<tgrid, tblock, 0, s>>>(startT, endT, N1, n_slabs, reinterpret_cast<uint32_t *>(ptr), startS);
    TM_LAUNCHED("k_slab_transpose");
    if ((rc = exclusive_scan_u32(reinterpret_cast<uint32_t *>(ptr), reinterpret_cast<uint32_t *>(ptr), cells, s)))
      return rc;
    int32_t *deltaT = startT;  // startT / endT are consumed
    k_slab_delta<<<tgrid, tblock, 0, s>>>(ptr, startS, N1, n_slabs, deltaT);
    TM_LAUNCHED("k_slab_delta");
    // W >= delta: an edge lands in at most two slabs, so 2 E entries bound
    // the view without reading the scan's total back (no host sync)
    si.entries[d] = 2 * E;
    if ((rc = si.np[d].ensure_pooled(sizeof(int2) * (size_t)(2 * E), s, g->stream)) ||
        (rc = si.rnk[d].ensure_pooled(sizeof(uint32_t) * (size_t)(2 * E), s, g->stream)))
      return rc;
    k_slab_fill<<<grid_for(E, kFillTile), kFillThreads, kFillSmem, s>>>(g->owner[d].as<int32_t>(), g->rnk[d].as<uint32_t>(),
                                               g->npk[d].as<int2>(), E, n_slabs, si.slab_of.as<uint16_t>(),
                                               L, deltaT, si.np[d].as<int2>(), si.rnk[d].as<uint32_t>());
    TM_LAUNCHED("k_slab_fill");
    view->ptr[d] = ptr;
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
