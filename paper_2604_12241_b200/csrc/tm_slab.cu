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
// Build (all streaming, no sort — the global runs are already sorted by
// (owner, rank, eid) and a slab run is a contiguous piece of a global run):
//   k_slab_bounds   S_s = lower_bound(uniq_time, t0 + s W), L_s = lo_tab[S_s]
//   k_slab_of       slab of every rank
//   k_slab_edges    per global CSR slot: the first / last slot of each slab
//                   run it opens / closes -> start[s][x], end[s][x]
//   k_slab_count    run lengths end - start, then an exclusive scan -> ptr
//   k_slab_fill     per global slot: its copies (nbr, prev, rank) at
//                   ptr[s][x] + (slot - start[s][x])
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
// r are [slab_of(r), ...) while L_s <= r (two at most when W >= delta)
__global__ void k_slab_edges(const int32_t *__restrict__ owner, const uint32_t *__restrict__ rnk,
                             const int32_t *__restrict__ ptr, int64_t E, int64_t N1, int n_slabs,
                             const uint16_t *__restrict__ slab_of, const uint32_t *__restrict__ S,
                             const uint32_t *__restrict__ L, int32_t *__restrict__ start,
                             int32_t *__restrict__ end) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= E) return;
  const int x = __ldg(owner + j);
  const uint32_t r = __ldg(rnk + j);
  const int a = __ldg(ptr + x), b = __ldg(ptr + x + 1);
  const uint32_t rp = j > a ? __ldg(rnk + j - 1) : 0u;
  const uint32_t rn = j + 1 < b ? __ldg(rnk + j + 1) : 0xffffffffu;
  for (int s = __ldg(slab_of + r); s < n_slabs && __ldg(L + s) <= r; ++s) {
    const int64_t cell = (int64_t)s * N1 + x;
    if (j == a || rp < __ldg(L + s)) start[cell] = (int32_t)j;   // opens x's run in slab s
    if (j + 1 == b || rn >= __ldg(S + s + 1)) end[cell] = (int32_t)(j + 1);  // closes it
  }
}

// run lengths, in place of end (cells of empty runs stay 0 - 0)
__global__ void k_slab_count(const int32_t *__restrict__ start, int32_t *__restrict__ end_cnt, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) end_cnt[i] -= start[i];
}

__global__ void k_slab_fill(const int32_t *__restrict__ owner, const uint32_t *__restrict__ rnk,
                            const int2 *__restrict__ np, int64_t E, int64_t N1, int n_slabs,
                            const uint16_t *__restrict__ slab_of, const uint32_t *__restrict__ L,
                            const int32_t *__restrict__ start, const int32_t *__restrict__ sptr,
                            int2 *__restrict__ snp, uint32_t *__restrict__ srnk) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= E) return;
  const int x = __ldg(owner + j);
  const uint32_t r = __ldg(rnk + j);
  const int2 e = __ldg(np + j);
  for (int s = __ldg(slab_of + r); s < n_slabs && __ldg(L + s) <= r; ++s) {
    const int64_t cell = (int64_t)s * N1 + x;
    const int64_t p = (int64_t)__ldg(sptr + cell) + (j - __ldg(start + cell));
    snp[p] = e;
    srnk[p] = r;
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
  for (int d = 0; d < 2; ++d) {
    if ((rc = si.start[d].ensure_pooled(sizeof(int32_t) * (size_t)cells, s, g->stream)) ||
        (rc = si.ptr[d].ensure_pooled(sizeof(int32_t) * (size_t)cells, s, g->stream)))
      return rc;
    int32_t *start = si.start[d].as<int32_t>(), *ptr = si.ptr[d].as<int32_t>();
    TM_CUDA(cudaMemsetAsync(start, 0, sizeof(int32_t) * (size_t)cells, s));
    TM_CUDA(cudaMemsetAsync(ptr, 0, sizeof(int32_t) * (size_t)cells, s));
    k_slab_edges<<<grid_for(E, kB), kB, 0, s>>>(g->owner[d].as<int32_t>(), g->rnk[d].as<uint32_t>(),
                                                g->ptr[d].as<int32_t>(), E, N1, n_slabs,
                                                si.slab_of.as<uint16_t>(), S, L, start, ptr);
    TM_LAUNCHED("k_slab_edges");
    k_slab_count<<<grid_for(cells, kB), kB, 0, s>>>(start, ptr, cells);
    TM_LAUNCHED("k_slab_count");
    if ((rc = exclusive_scan_u32(reinterpret_cast<uint32_t *>(ptr), reinterpret_cast<uint32_t *>(ptr), cells, s)))
      return rc;
    // W >= delta: an edge lands in at most two slabs, so 2 E entries bound
    // the view without reading the scan's total back (no host sync)
    si.entries[d] = 2 * E;
    if ((rc = si.np[d].ensure_pooled(sizeof(int2) * (size_t)(2 * E), s, g->stream)) ||
        (rc = si.rnk[d].ensure_pooled(sizeof(uint32_t) * (size_t)(2 * E), s, g->stream)))
      return rc;
    k_slab_fill<<<grid_for(E, kB), kB, 0, s>>>(g->owner[d].as<int32_t>(), g->rnk[d].as<uint32_t>(),
                                               g->npk[d].as<int2>(), E, N1, n_slabs, si.slab_of.as<uint16_t>(),
                                               L, start, ptr, si.np[d].as<int2>(), si.rnk[d].as<uint32_t>());
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
