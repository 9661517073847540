// tm_internal.cuh — shared declarations of the B200 mining engine.
//
// Device layout of a built graph (all arrays resident in HBM, int32 ids):
//
//   edge table       e_src/e_dst int32[E], e_rank uint32[E]
//   time ranks       uniq_time int64[R]: sorted distinct timestamps; every
//                    time is stored as its dense rank, so a window
//                    [t - delta, t] becomes the rank interval
//                    [lower_bound(uniq_time, t - delta), rank(t)] (exact,
//                    order preserving; txgraph.py:5-6 int64 ticks)
//   dual CSR         per direction d (0 = in, 1 = out): ptr int32[N+1];
//                    entries sorted by (owner, rank, eid) exactly as
//                    np.lexsort((eid, time, owner)) (txgraph.py:134-144):
//                    nbr int32[E], rnk uint32[E], eid int32[E]
//   pair index       same runs re-sorted by (owner, nbr, rank, eid):
//                    pkey uint64[E] = nbr << rank_bits | rank — answers "edge
//                    a->b inside the window?" by bisection when both windows
//                    are wide.
//   previous occurrence  prev uint32[E] per CSR slot: rank + 1 of the
//                    previous entry with the same (owner, nbr), 0 = none.
//                    Entry j is the first occurrence of its neighbour inside
//                    the window [lo, hi] (np.unique dedup, kernels.py:59)
//                    iff prev[j] <= lo: one coalesced load along the window.
//   self-loop flags  loop uint8[N] (txgraph.py:146-153 self-loop CSR)
//
// Time-slab view (tm_slab.cu, built per mining call and delta): the time
// axis is cut into slabs of width W >= delta; slab s holds, per node, the
// sub-run of edges with rank in [L_s, S_{s+1}) — its own triggers' ranks
// [S_s, S_{s+1}) plus a halo back to the earliest window start L_s.  Every
// window of a trigger in slab s lies inside that slab's run, so the mining
// kernels read short, time-local runs from a few-% slice of the edge arrays
// (L2-resident) instead of bisecting whole-horizon runs.  A DevGraph whose
// ptr / np / rnk point at a slab index is a "slab view": ptr is then the
// [n_slabs][N+1] offset table (Ctx::soff selects the slab) and gptr keeps
// the global offsets for the pair index (pkey runs).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <climits>
#include <string>

#include "../../include/tempmine_b200.h"

namespace tmb {

constexpr int kMaxPlans = 32;

struct DevGraph {
  int32_t n_nodes;
  int32_t n_edges;
  int32_t rank_bits;
  int32_t pad;
  const int32_t *e_src;
  const int32_t *e_dst;
  const uint32_t *e_rank;
  const int32_t *ptr[2];
  const int32_t *nbr[2];
  const uint32_t *rnk[2];
  const uint64_t *pkey[2];
  const uint32_t *prev[2];
  const int32_t *eid[2];   // edge id per CSR slot (members attribution)
  const int32_t *peid[2];  // edge id per pair slot (members attribution)
  const int2 *np[2];       // (nbr, prev) per CSR slot, interleaved for the walkers
  const int32_t *owner[2]; // owner node of each CSR slot (slot-parallel window sweeps)
  const uint8_t *loop;
  const int32_t *gptr[2];  // global CSR offsets: pair-index runs (== ptr in the global view)
};

constexpr int kMaxChain = 5;   // cycle_8: chain a1..a5
constexpr int kMaxCyc = 6;     // cycle_3..8 columns per group (more: another group, same delta)
constexpr int kMaxGroups = 8;  // distinct deltas per tm_mine call

// per-column launch descriptor (device side)
struct DevPlan {
  int32_t family, endpoint, direction, exclude_trigger, cycle_len, min_size;
  int32_t group;  // delta group
};

// one fused chain enumeration for every cycle_3..8 column of a delta group;
// entry e closes at chain depth depth[e] (cycle length depth + 3)
struct CycGroup {
  int32_t mask;  // bit d: some column closes at depth d
  int32_t maxd;  // deepest chain (0..5)
  int32_t n;     // entries
  int32_t k[kMaxCyc];      // min_size per entry
  int8_t depth[kMaxCyc];
  int8_t col[kMaxCyc];     // output column per entry
  int32_t deep_split;      // chain nodes with wider windows leave the warp kernel (pull tasks)
};

constexpr int kLaneCyc2 = 1 << 8;   // lane_d kind: cycle_2 (else FAN / DEGREE)
constexpr int kLaneStack = 1 << 8;  // end_d kind: stack (else cycle_3)

// the columns sharing one delta: one set of trigger windows, one
// lower-bound table, one pass over each trigger slice
struct DevGroup {
  // the graph as this group's kernels read it: the global CSR, or the time-
  // slab view of the group's delta (tm_slab.cu); slab_of[rank] selects the
  // slab (null: global view), its offset table row is slab * stride
  DevGraph view;
  const uint16_t *slab_of;
  int64_t stride;
  const uint32_t *lo_tab;  // rank -> first rank with time >= uniq_time[rank] - delta
  // per trigger row of the call (or null): (window start rank, slab) — read
  // with the trigger's own edge fields instead of two lookups behind e_rank
  const int2 *lo_slab;
  // own windows by edge id (or null): own[1][e] = window of e's source
  // out-run at e's time (u-out), own[0][e] = of e's destination in-run (v-in)
  const int2 *own[2];
  int32_t need;            // trigger windows (1 u-in, 2 u-out, 4 v-in, 8 v-out)
  int32_t udom, vdom;      // N-(u) / N+(v) item passes needed
  int32_t has_stack;
  int32_t ncols, n_sg, n_gs;
  int8_t cols[kMaxPlans];
  // the lane-owned columns in two packed lists (the trigger kernel walks
  // these instead of every column's DevPlan): FAN / DEGREE / cycle_2 right
  // after the windows, stack / cycle_3 after the items.  lane_d = column |
  // kind << 8 | endpoint << 10 | direction << 11 | exclude_trigger << 12;
  // lane_k = min_size
  int32_t n_lane, n_end;
  int32_t lane_d[kMaxPlans], lane_k[kMaxPlans];
  int32_t end_d[kMaxPlans], end_k[kMaxPlans];
  int8_t sg_col[kMaxPlans];
  int8_t gs_col[kMaxPlans];
  CycGroup cyc;
};

struct DevPlans {
  int32_t n;
  int32_t ngroups;
  DevPlan p[kMaxPlans];
  DevGroup gr[kMaxGroups];
  // columns that receive item contributions (sg, gs, cycle_4..8) are staged
  // in shared memory: slot[col] (-1: the owner lane writes it directly) and
  // its inverse slot_col[slot]
  int32_t n_stage;
  int8_t slot[kMaxPlans];
  int8_t slot_col[kMaxPlans];
};

// ----------------------------------------------------------------- errors

void set_error(const std::string &msg);
int fail(int code, const std::string &msg);
int cuda_fail(cudaError_t e, const char *what);
void count_launch(int n = 1);
// the library's stream-ordered memory pool on `device` (tm_api.cu) and an
// allocation from it on stream s (current device)
cudaMemPool_t lib_pool(int device);
cudaError_t pool_malloc(void **p, size_t n, cudaStream_t s);
// in-place exclusive scan of n uint64 on stream s (tm_export.cu)
int scan_u64_exclusive(unsigned long long *a, int64_t n, cudaStream_t s);

#define TM_CUDA(expr)                                       \
  do {                                                      \
    cudaError_t _e = (expr);                                \
    if (_e != cudaSuccess) return ::tmb::cuda_fail(_e, #expr); \
  } while (0)

#define TM_LAUNCHED(name)                                   \
  do {                                                      \
    ::tmb::count_launch();                                   \
    cudaError_t _e = cudaGetLastError();                    \
    if (_e != cudaSuccess) return ::tmb::cuda_fail(_e, name); \
  } while (0)

// ----------------------------------------------------------------- memory

struct DevBuf {
  void *p = nullptr;
  size_t bytes = 0;
  cudaStream_t pool_stream = nullptr;  // set: stream-ordered (memory pool) allocation
  bool pooled = false;
  ~DevBuf() { release(); }
  void release() {
    if (p) {
      if (pooled && pool_stream) cudaFreeAsync(p, pool_stream);
      else cudaFree(p);  // also valid for pool memory: frees synchronously, back into the pool
    }
    p = nullptr;
    bytes = 0;
    pooled = false;
  }
  int ensure(size_t n);                     // grow-only, cudaMalloc
  int ensure_on(size_t n, cudaStream_t s);  // grow-only, cudaMallocAsync on s (pool)
  // grow-only pool allocation for scratch used on arbitrary streams: a grow
  // synchronizes the device first; frees are stream-ordered on free_stream
  // (the graph's stream; teardown synchronizes the device before) — so a
  // rebuilt graph reuses pool memory instead of paying cudaMalloc again
  int ensure_pooled(size_t n, cudaStream_t s, cudaStream_t free_stream);
  template <class T> T *as() const { return static_cast<T *>(p); }
};

// ----------------------------------------------------------------- sorting

// Stable LSD radix sort of (key, value) pairs over key bits [0, nbits).
// keys/vals hold the input; ktmp/vtmp are equally sized scratch.  On return
// *kout/*vout point at whichever buffer holds the sorted result.
int radix_sort_pairs(uint64_t *keys, uint32_t *vals, uint64_t *ktmp, uint32_t *vtmp, int64_t n,
                     int nbits, cudaStream_t s, uint64_t **kout, uint32_t **vout);

// exclusive scan of uint32 counts (n <= 2^31) into out (may alias in)
int exclusive_scan_u32(const uint32_t *in, uint32_t *out, int64_t n, cudaStream_t s);

// ----------------------------------------------------------------- slabs

constexpr int kMaxSlabs = 128;  // slab offset tables are [n_slabs][N+1]
constexpr int kMinSlabs = 3;    // fewer slabs than this: the global view is used
constexpr int kSlabMinRun = 32; // mean run length E/N below this: the global view is used

// one delta's slab index (grow-only device storage, tm_slab.cu)
struct SlabIndex {
  DevBuf start[2];   // [n_slabs][N+1] global CSR slot of each slab run's first entry
  DevBuf ptr[2];     // [n_slabs][N+1] slab run offsets (exclusive scan of the run lengths)
  DevBuf np[2];      // (nbr, prev) per slab entry
  DevBuf rnk[2];     // rank per slab entry
  DevBuf slab_of;    // uint16 [R]: slab of each rank
  DevBuf bounds;     // uint32 [2][n_slabs + 1]: S_s (first trigger rank), L_s (first halo rank)
  DevBuf scratch;    // int32 [2][N+1][n_slabs]: owner-major cell tables of the build
  int n_slabs = 0;
  int s0 = 0;  // first slab built (start / ptr rows are slabs s0..)
  int64_t entries[2] = {0, 0};
};

// window-start tables and slab views prepared for a trigger range and kept
// on the graph (tm_mine_prepare): tm_mine calls on sub-ranges with these
// deltas reuse them instead of building their own
struct PreparedViews {
  bool valid = false;
  int n = 0;
  int64_t lo = 0, hi = 0;
  int64_t delta[kMaxGroups] = {};
  DevBuf lo_tabs;  // [n][R]
  SlabIndex slabs[kMaxGroups];
  DevGraph view[kMaxGroups] = {};
  const uint16_t *slab_of[kMaxGroups] = {};
  int64_t stride[kMaxGroups] = {};
};

inline int bits_for(uint64_t maxval) {  // bits to represent [0, maxval]
  int b = 0;
  while (b < 64 && (maxval >> b) != 0) ++b;
  return b;
}

inline unsigned grid_for(int64_t n, int block) {
  int64_t g = (n + block - 1) / block;
  return (unsigned)(g < 1 ? 1 : g);
}

}  // namespace tmb

// ------------------------------------------------------------- the handle

struct tm_graph {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool owns_stream = false;
  int64_t n_nodes = 0, n_edges = 0, n_ranks = 0, n_selfloops = 0;
  int64_t t_span = 0;  // max - min timestamp (ticks)
  int64_t max_deg[2] = {0, 0};
  int rank_bits = 0, node_bits = 0;
  int64_t device_bytes = 0;

  tmb::DevBuf e_src, e_dst, e_rank, uniq_time, loop, maxdeg;
  tmb::DevBuf ptr[2], nbr[2], rnk[2], eid[2], pkey[2], prev[2], peid[2], npk[2], owner[2];

  // mining scratch (grow-only)
  tmb::DevBuf lo_tabs, own_tabs, bloom_lists, heavy_q, heavy_n, out_scratch, tasks, split_scratch, lo_slab, chain_q, split_win;
  tmb::DevBuf csv_buf;  // formatted feature CSV (tm_csv_format)
  int64_t csv_bytes = 0;
  tmb::DevBuf inst_buf;  // instance records (tm_collect_instances, tm_vm_collect)
  int64_t inst_words = 0;
  // GENERIC stage programs (tm_vm.cu): edge attributes, program, arena
  tmb::DevBuf attr_amount, attr_currency, attr_cur_rank;
  int32_t n_vocab = 0;
  tmb::DevBuf vm_prog, vm_arena, vm_ovf, vm_novf;
  int64_t lo_tab_cap = 0;
  tm_mine_stats last{};
  bool prof = false, prof_pending = false;
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};  // warp start, warp end, end, call start
  // host-output pieces: D2H of piece i overlaps mining of piece i+1
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t piece_ev[8] = {};
  tmb::DevBuf split_counts;
  tmb::SlabIndex slabs[tmb::kMaxGroups];
  tmb::PreparedViews prep;  // tm_mine_prepare
  int64_t t_min = 0;   // smallest timestamp (ticks)
  tmb::DevBuf time_order;         // int32[E]: edge ids sorted by (time, id)
  bool ids_time_ordered = false;  // time_order is the identity
  // completion of the last call that enqueued work on a (possibly user)
  // stream: the next call's stream waits on it before touching the shared
  // scratch, and tm_graph_free waits on it before freeing
  cudaEvent_t done_ev = nullptr;

  cudaError_t begin(cudaStream_t s) { return done_ev ? cudaStreamWaitEvent(s, done_ev, 0) : cudaSuccess; }
  cudaError_t end(cudaStream_t s) {
    if (!done_ev) {
      cudaError_t e = cudaEventCreateWithFlags(&done_ev, cudaEventDisableTiming);
      if (e != cudaSuccess) return e;
    }
    return cudaEventRecord(done_ev, s);
  }

  tmb::DevGraph dev() const;
};

namespace tmb {
// The slab view of `delta`: builds the slab index into si on stream s and
// fills *view / *slab_of / *stride (the global view when the horizon holds
// fewer than kMinSlabs windows).  lo_tab is the rank -> window-start table.
// restrict_range: only the slabs of triggers [trig_lo, trig_hi) (edge ids in
// time order; one host sync), else every slab.
int build_slab_view(tm_graph *g, SlabIndex &si, int64_t delta, const uint32_t *lo_tab, cudaStream_t s,
                    int64_t trig_lo, int64_t trig_hi, bool restrict_range, DevGraph *view,
                    const uint16_t **slab_of, int64_t *stride);
}  // namespace tmb
