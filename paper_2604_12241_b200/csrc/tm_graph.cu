// tm_graph.cu — device graph construction (GPU radix-sort dual CSR, time
// ranks, pair index) and read-back.
//
// Reference: TemporalGraph.__init__ (txgraph.py:113-170).  The reference
// builds out/in runs with np.lexsort((eid, time, owner)) and indptr with
// bincount+cumsum; this file computes the same runs with stable radix sorts
// of packed (owner << rank_bits | rank) keys over an eid-ordered input, and
// indptr from run boundaries of the sorted keys (no atomics on hub nodes).
#include <algorithm>
#include <mutex>
#include <cstring>
#include <vector>

#include "tm_internal.cuh"

namespace tmb {
namespace {

constexpr int kB = 256;

struct ScanStats {
  long long tmin, tmax;
  unsigned long long bad;       // ids out of range
  unsigned long long selfloops;
};

__global__ void k_validate(const int64_t *__restrict__ src, const int64_t *__restrict__ dst,
                           const int64_t *__restrict__ time, int64_t n, int64_t n_nodes,
                           ScanStats *st) {
  long long tmin = LLONG_MAX, tmax = LLONG_MIN;
  unsigned long long bad = 0, loops = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t s = src[i], d = dst[i], t = time[i];
    bad += (s < 0 || s >= n_nodes || d < 0 || d >= n_nodes);
    loops += (s == d);
    tmin = min(tmin, (long long)t);
    tmax = max(tmax, (long long)t);
  }
  for (int o = 16; o > 0; o >>= 1) {
    tmin = min(tmin, __shfl_xor_sync(0xffffffffu, tmin, o));
    tmax = max(tmax, __shfl_xor_sync(0xffffffffu, tmax, o));
    bad += __shfl_xor_sync(0xffffffffu, bad, o);
    loops += __shfl_xor_sync(0xffffffffu, loops, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(&st->tmin, tmin);
    atomicMax(&st->tmax, tmax);
    if (bad) atomicAdd(&st->bad, bad);
    if (loops) atomicAdd(&st->selfloops, loops);
  }
}

__global__ void k_prepare(const int64_t *__restrict__ src, const int64_t *__restrict__ dst,
                          const int64_t *__restrict__ time, int64_t n, long long tmin,
                          int32_t *__restrict__ s32, int32_t *__restrict__ d32,
                          uint64_t *__restrict__ tkey, uint32_t *__restrict__ ids,
                          uint8_t *__restrict__ loop) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int32_t s = (int32_t)src[i], d = (int32_t)dst[i];
  s32[i] = s;
  d32[i] = d;
  tkey[i] = (uint64_t)((unsigned long long)time[i] - (unsigned long long)tmin);
  ids[i] = (uint32_t)i;
  if (s == d) loop[s] = 1;  // benign race: every writer stores 1
}

// sorted time keys -> distinct-time table and per-edge rank
__global__ void k_rank_flags(const uint64_t *__restrict__ k, int64_t n, uint32_t *__restrict__ f) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) f[i] = (i == 0 || k[i] != k[i - 1]) ? 1u : 0u;
}

__global__ void k_rank_scatter(const uint64_t *__restrict__ k, const uint32_t *__restrict__ ids,
                               const uint32_t *__restrict__ excl, int64_t n, long long tmin,
                               int64_t *__restrict__ uniq, uint32_t *__restrict__ rank) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  bool head = (i == 0 || k[i] != k[i - 1]);
  uint32_t r = excl[i] + (head ? 1u : 0u) - 1u;
  if (head) uniq[r] = (int64_t)(k[i] + (unsigned long long)tmin);
  rank[ids[i]] = r;
}

// ids sorted by time -> the time-order array; flags any id out of place
__global__ void k_time_order(const uint32_t *__restrict__ ids, int64_t n, int32_t *__restrict__ order,
                             unsigned int *__restrict__ moved) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t e = ids[i];
  order[i] = (int32_t)e;
  if (e != (uint32_t)i) *moved = 1u;  // benign race: every writer stores 1
}

__global__ void k_csr_keys(const int32_t *__restrict__ owner, const uint32_t *__restrict__ rank,
                           int64_t n, int rbits, uint64_t *__restrict__ keys,
                           uint32_t *__restrict__ ids) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  keys[i] = ((uint64_t)(uint32_t)owner[i] << rbits) | rank[i];
  ids[i] = (uint32_t)i;
}

__global__ void k_csr_fill(const uint64_t *__restrict__ keys, const uint32_t *__restrict__ ids,
                           const int32_t *__restrict__ other, int64_t n, int rbits,
                           int32_t *__restrict__ nbr, uint32_t *__restrict__ rnk,
                           int32_t *__restrict__ eid, uint64_t *__restrict__ pair_keys,
                           uint32_t *__restrict__ pair_ids, int nbits, int32_t *__restrict__ own) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  const uint64_t key = keys[p];
  const uint32_t e = ids[p];
  const int32_t o = other[e];
  const uint64_t owner = key >> rbits;
  nbr[p] = o;
  own[p] = (int32_t)owner;
  rnk[p] = (uint32_t)(key & ((1ull << rbits) - 1));
  eid[p] = (int32_t)e;
  pair_keys[p] = (owner << nbits) | (uint32_t)o;
  pair_ids[p] = (uint32_t)p;
}

// ptr[x] = first position whose owner >= x   (run boundaries, no atomics)
__global__ void k_indptr(const uint64_t *__restrict__ keys, int64_t n, int shift, int64_t n_nodes,
                         int32_t *__restrict__ ptr) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p > n) return;
  int64_t prev = p == 0 ? -1 : (int64_t)(keys[p - 1] >> shift);
  int64_t cur = p == n ? n_nodes : (int64_t)(keys[p] >> shift);
  for (int64_t x = prev + 1; x <= cur; ++x) ptr[x] = (int32_t)p;
}

// pair slot q holds CSR slot p = pids[q]; runs of equal (owner, nbr) are in
// time order, so the pair predecessor is the previous occurrence of the same
// neighbour: prev[p] = its rank + 1 (0 = none)
__global__ void k_pair_fill(const uint64_t *__restrict__ pair_sorted, const uint32_t *__restrict__ pids,
                            const int32_t *__restrict__ nbr, const uint32_t *__restrict__ rnk,
                            const int32_t *__restrict__ eid, int64_t n, int rbits,
                            uint64_t *__restrict__ pkey, uint32_t *__restrict__ prev,
                            int32_t *__restrict__ peid) {
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= n) return;
  const uint32_t p = pids[q];
  pkey[q] = ((uint64_t)(uint32_t)nbr[p] << rbits) | rnk[p];
  peid[q] = eid[p];
  prev[p] = (q > 0 && pair_sorted[q - 1] == pair_sorted[q]) ? rnk[pids[q - 1]] + 1u : 0u;
}

__global__ void k_np_fill(const int32_t *__restrict__ nbr, const uint32_t *__restrict__ prev, int64_t n,
                          int2 *__restrict__ np) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p < n) np[p] = make_int2(nbr[p], (int)prev[p]);
}

__global__ void k_max_degree(const int32_t *__restrict__ ptr, int64_t n_nodes,
                             unsigned long long *out) {
  unsigned long long m = 0;
  for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < n_nodes;
       x += (int64_t)gridDim.x * blockDim.x)
    m = max(m, (unsigned long long)(ptr[x + 1] - ptr[x]));
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0 && m) atomicMax(out, m);
}

__global__ void k_gather_time(const uint32_t *__restrict__ rnk, const int64_t *__restrict__ uniq,
                              int64_t n, int64_t *__restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = uniq[rnk[i]];
}

}  // namespace

// every device buffer has kPad spare bytes past its end: the walkers' 16-byte
// vector loads of a run's aligned block may reach past the last entry
constexpr size_t kPad = 64;

int DevBuf::ensure_on(size_t n, cudaStream_t s) {
  if (n <= bytes && p) return TM_OK;
  release();
  cudaError_t e = pool_malloc(&p, n + kPad, s);
  if (e != cudaSuccess) {
    p = nullptr;
    cudaGetLastError();
    return fail(e == cudaErrorMemoryAllocation ? TM_E_OOM : TM_E_CUDA,
                std::string("device allocation of ") + std::to_string(n) +
                    " bytes failed: " + cudaGetErrorString(e));
  }
  bytes = n ? n : 16;
  pooled = true;
  pool_stream = s;
  return TM_OK;
}

int DevBuf::ensure_pooled(size_t n, cudaStream_t s, cudaStream_t free_stream) {
  if (n <= bytes && p) return TM_OK;
  if (p) {
    // the old block may still be read by this call's earlier kernels on s
    // or (tm_graph::begin makes s wait for them) by earlier calls
    cudaStreamSynchronize(s);
    cudaStreamSynchronize(free_stream);
    release();
  }
  cudaError_t e = pool_malloc(&p, n + kPad, s);
  if (e != cudaSuccess) {
    p = nullptr;
    cudaGetLastError();
    return fail(e == cudaErrorMemoryAllocation ? TM_E_OOM : TM_E_CUDA,
                std::string("device allocation of ") + std::to_string(n) +
                    " bytes failed: " + cudaGetErrorString(e));
  }
  bytes = n ? n : 16;
  pooled = true;
  pool_stream = free_stream;  // the graph's own stream: teardown frees back into the pool
  return TM_OK;
}

int DevBuf::ensure(size_t n) {
  if (n <= bytes && p) return TM_OK;
  release();
  cudaError_t e = cudaMalloc(&p, n + kPad);
  if (e != cudaSuccess) {
    p = nullptr;
    cudaGetLastError();
    return fail(e == cudaErrorMemoryAllocation ? TM_E_OOM : TM_E_CUDA,
                std::string("device allocation of ") + std::to_string(n) +
                    " bytes failed: " + cudaGetErrorString(e));
  }
  bytes = n ? n : 16;
  return TM_OK;
}

}  // namespace tmb

tmb::DevGraph tm_graph::dev() const {
  tmb::DevGraph g{};
  g.n_nodes = (int32_t)n_nodes;
  g.n_edges = (int32_t)n_edges;
  g.rank_bits = rank_bits;
  g.e_src = e_src.as<int32_t>();
  g.e_dst = e_dst.as<int32_t>();
  g.e_rank = e_rank.as<uint32_t>();
  for (int d = 0; d < 2; ++d) {
    g.ptr[d] = ptr[d].as<int32_t>();
    g.nbr[d] = nbr[d].as<int32_t>();
    g.rnk[d] = rnk[d].as<uint32_t>();
    g.pkey[d] = pkey[d].as<uint64_t>();
    g.prev[d] = prev[d].as<uint32_t>();
    g.eid[d] = eid[d].as<int32_t>();
    g.peid[d] = peid[d].as<int32_t>();
    g.np[d] = npk[d].as<int2>();
    g.owner[d] = owner[d].as<int32_t>();
    g.gptr[d] = g.ptr[d];
  }
  g.loop = loop.as<uint8_t>();
  return g;
}

using namespace tmb;

static int build_impl(tm_graph *g, const int64_t *src, const int64_t *dst, const int64_t *time,
                      int on_device) {
  cudaStream_t s = g->stream;
  const int64_t E = g->n_edges, N = g->n_nodes;
  DevBuf in_src, in_dst, in_time;
  const int64_t *d_src = src, *d_dst = dst, *d_time = time;
  if (!on_device && E > 0) {
    int rc;
    if ((rc = in_src.ensure_on(8 * E, s)) || (rc = in_dst.ensure_on(8 * E, s)) || (rc = in_time.ensure_on(8 * E, s)))
      return rc;
    TM_CUDA(cudaMemcpyAsync(in_src.p, src, 8 * E, cudaMemcpyHostToDevice, s));
    TM_CUDA(cudaMemcpyAsync(in_dst.p, dst, 8 * E, cudaMemcpyHostToDevice, s));
    TM_CUDA(cudaMemcpyAsync(in_time.p, time, 8 * E, cudaMemcpyHostToDevice, s));
    d_src = in_src.as<int64_t>();
    d_dst = in_dst.as<int64_t>();
    d_time = in_time.as<int64_t>();
  }

  int rc;
  const int64_t Ea = E > 0 ? E : 1;
  if ((rc = g->maxdeg.ensure_on(16, s))) return rc;
  TM_CUDA(cudaMemsetAsync(g->maxdeg.p, 0, 16, s));
  if ((rc = g->e_src.ensure_on(4 * Ea, s)) || (rc = g->e_dst.ensure_on(4 * Ea, s)) ||
      (rc = g->e_rank.ensure_on(4 * Ea, s)) || (rc = g->loop.ensure_on(N > 0 ? N : 1, s)))
    return rc;
  TM_CUDA(cudaMemsetAsync(g->loop.p, 0, N > 0 ? N : 1, s));
  for (int d = 0; d < 2; ++d) {
    if ((rc = g->ptr[d].ensure_on(4 * (N + 1), s)) || (rc = g->nbr[d].ensure_on(4 * Ea, s)) ||
        (rc = g->rnk[d].ensure_on(4 * Ea, s)) || (rc = g->eid[d].ensure_on(4 * Ea, s)) ||
        (rc = g->pkey[d].ensure_on(8 * Ea, s)) || (rc = g->prev[d].ensure_on(4 * Ea, s)) ||
        (rc = g->peid[d].ensure_on(4 * Ea, s)) || (rc = g->npk[d].ensure_on(8 * Ea, s)) ||
        (rc = g->owner[d].ensure_on(4 * Ea, s)))
      return rc;
  }
  if (E == 0) {
    for (int d = 0; d < 2; ++d) TM_CUDA(cudaMemsetAsync(g->ptr[d].p, 0, 4 * (N + 1), s));
    if ((rc = g->uniq_time.ensure_on(8, s))) return rc;
    g->n_ranks = 0;
    g->rank_bits = 1;
    g->node_bits = std::max(1, bits_for((uint64_t)(N > 0 ? N - 1 : 0)));
    return cudaStreamSynchronize(s) == cudaSuccess ? TM_OK : cuda_fail(cudaGetLastError(), "sync");
  }

  // 1. validate ids, time range, self-loops
  ScanStats h0{LLONG_MAX, LLONG_MIN, 0, 0}, h1{};
  DevBuf st;
  if ((rc = st.ensure_on(sizeof(ScanStats), s))) return rc;
  TM_CUDA(cudaMemcpyAsync(st.p, &h0, sizeof(ScanStats), cudaMemcpyHostToDevice, s));
  k_validate<<<1184, kB, 0, s>>>(d_src, d_dst, d_time, E, N, st.as<ScanStats>());
  TM_LAUNCHED("k_validate");
  TM_CUDA(cudaMemcpyAsync(&h1, st.p, sizeof(ScanStats), cudaMemcpyDeviceToHost, s));
  TM_CUDA(cudaStreamSynchronize(s));
  if (h1.bad) return fail(TM_E_BAD_ARG, std::to_string(h1.bad) + " edge endpoint(s) outside [0, n_nodes)");
  g->n_selfloops = (int64_t)h1.selfloops;
  g->t_min = (int64_t)h1.tmin;
  g->t_span = (int64_t)((unsigned long long)h1.tmax - (unsigned long long)h1.tmin);

  // 2. narrow ids, time keys
  DevBuf ka, kb, va, vb;
  if ((rc = ka.ensure_on(8 * E, s)) || (rc = kb.ensure_on(8 * E, s)) || (rc = va.ensure_on(4 * E, s)) ||
      (rc = vb.ensure_on(4 * E, s)))
    return rc;
  k_prepare<<<grid_for(E, kB), kB, 0, s>>>(d_src, d_dst, d_time, E, h1.tmin, g->e_src.as<int32_t>(),
                                           g->e_dst.as<int32_t>(), ka.as<uint64_t>(),
                                           va.as<uint32_t>(), g->loop.as<uint8_t>());
  TM_LAUNCHED("k_prepare");
  in_src.release();  // stream-ordered frees (memory pool): no device sync
  in_dst.release();
  in_time.release();

  // 3. time ranks
  const int tbits = bits_for((uint64_t)((unsigned long long)h1.tmax - (unsigned long long)h1.tmin));
  uint64_t *ks;
  uint32_t *vs;
  if ((rc = radix_sort_pairs(ka.as<uint64_t>(), va.as<uint32_t>(), kb.as<uint64_t>(),
                             vb.as<uint32_t>(), E, tbits, s, &ks, &vs)))
    return rc;
  uint32_t *flags = (ks == ka.as<uint64_t>()) ? vb.as<uint32_t>() : va.as<uint32_t>();
  // flags must not alias vs: vs is one of va/vb, flags is the other
  k_rank_flags<<<grid_for(E, kB), kB, 0, s>>>(ks, E, flags);
  TM_LAUNCHED("k_rank_flags");
  // inclusive count of heads at the last element = number of ranks
  uint32_t last_flag = 0, last_excl = 0;
  if ((rc = exclusive_scan_u32(flags, flags, E, s))) return rc;
  TM_CUDA(cudaMemcpyAsync(&last_excl, flags + (E - 1), 4, cudaMemcpyDeviceToHost, s));
  {
    uint64_t k_last = 0, k_prev = 0;
    TM_CUDA(cudaMemcpyAsync(&k_last, ks + (E - 1), 8, cudaMemcpyDeviceToHost, s));
    if (E > 1) TM_CUDA(cudaMemcpyAsync(&k_prev, ks + (E - 2), 8, cudaMemcpyDeviceToHost, s));
    TM_CUDA(cudaStreamSynchronize(s));
    last_flag = (E == 1 || k_last != k_prev) ? 1u : 0u;
  }
  g->n_ranks = (int64_t)last_excl + last_flag;
  if ((rc = g->uniq_time.ensure_on(8 * g->n_ranks, s))) return rc;
  k_rank_scatter<<<grid_for(E, kB), kB, 0, s>>>(ks, vs, flags, E, h1.tmin,
                                                g->uniq_time.as<int64_t>(), g->e_rank.as<uint32_t>());
  TM_LAUNCHED("k_rank_scatter");
  {  // edge ids in time order (the stable sort keeps id order within a timestamp)
    if ((rc = g->time_order.ensure_on(4 * E, s))) return rc;
    unsigned int moved = 0;
    unsigned int *d_moved = reinterpret_cast<unsigned int *>(st.p);  // ScanStats is no longer needed
    TM_CUDA(cudaMemsetAsync(d_moved, 0, sizeof(unsigned int), s));
    k_time_order<<<grid_for(E, kB), kB, 0, s>>>(vs, E, g->time_order.as<int32_t>(), d_moved);
    TM_LAUNCHED("k_time_order");
    TM_CUDA(cudaMemcpyAsync(&moved, d_moved, sizeof(unsigned int), cudaMemcpyDeviceToHost, s));
    TM_CUDA(cudaStreamSynchronize(s));
    g->ids_time_ordered = moved == 0;
  }
  g->rank_bits = std::max(1, bits_for((uint64_t)(g->n_ranks - 1)));
  g->node_bits = std::max(1, bits_for((uint64_t)(N - 1)));
  if (g->rank_bits + g->node_bits > 63 || 2 * g->node_bits > 64)
    return fail(TM_E_OVERFLOW, "packed key does not fit 64 bits");

  // 4. dual CSR + pair index.  dir 1 = out (owner src), dir 0 = in (owner dst)
  for (int d = 1; d >= 0; --d) {
    const int32_t *owner = d ? g->e_src.as<int32_t>() : g->e_dst.as<int32_t>();
    const int32_t *other = d ? g->e_dst.as<int32_t>() : g->e_src.as<int32_t>();
    k_csr_keys<<<grid_for(E, kB), kB, 0, s>>>(owner, g->e_rank.as<uint32_t>(), E, g->rank_bits,
                                              ka.as<uint64_t>(), va.as<uint32_t>());
    TM_LAUNCHED("k_csr_keys");
    if ((rc = radix_sort_pairs(ka.as<uint64_t>(), va.as<uint32_t>(), kb.as<uint64_t>(),
                               vb.as<uint32_t>(), E, g->node_bits + g->rank_bits, s, &ks, &vs)))
      return rc;
    k_indptr<<<grid_for(E + 1, kB), kB, 0, s>>>(ks, E, g->rank_bits, N, g->ptr[d].as<int32_t>());
    TM_LAUNCHED("k_indptr");
    // pair keys go to the buffers not holding (ks, vs)
    uint64_t *pk = (ks == ka.as<uint64_t>()) ? kb.as<uint64_t>() : ka.as<uint64_t>();
    uint32_t *pv = (vs == va.as<uint32_t>()) ? vb.as<uint32_t>() : va.as<uint32_t>();
    k_csr_fill<<<grid_for(E, kB), kB, 0, s>>>(ks, vs, other, E, g->rank_bits, g->nbr[d].as<int32_t>(),
                                              g->rnk[d].as<uint32_t>(), g->eid[d].as<int32_t>(), pk,
                                              pv, g->node_bits, g->owner[d].as<int32_t>());
    TM_LAUNCHED("k_csr_fill");
    uint64_t *ps;
    uint32_t *pvs;
    uint64_t *pk2 = (pk == ka.as<uint64_t>()) ? kb.as<uint64_t>() : ka.as<uint64_t>();
    uint32_t *pv2 = (pv == va.as<uint32_t>()) ? vb.as<uint32_t>() : va.as<uint32_t>();
    if ((rc = radix_sort_pairs(pk, pv, pk2, pv2, E, 2 * g->node_bits, s, &ps, &pvs))) return rc;
    k_pair_fill<<<grid_for(E, kB), kB, 0, s>>>(ps, pvs, g->nbr[d].as<int32_t>(),
                                               g->rnk[d].as<uint32_t>(), g->eid[d].as<int32_t>(), E,
                                               g->rank_bits, g->pkey[d].as<uint64_t>(),
                                               g->prev[d].as<uint32_t>(), g->peid[d].as<int32_t>());
    TM_LAUNCHED("k_pair_fill");
    k_np_fill<<<grid_for(E, kB), kB, 0, s>>>(g->nbr[d].as<int32_t>(), g->prev[d].as<uint32_t>(), E,
                                             g->npk[d].as<int2>());
    TM_LAUNCHED("k_np_fill");
    unsigned long long *md = g->maxdeg.as<unsigned long long>() + d;  // read lazily by info
    TM_CUDA(cudaMemsetAsync(md, 0, 8, s));
    k_max_degree<<<592, kB, 0, s>>>(g->ptr[d].as<int32_t>(), N, md);
    TM_LAUNCHED("k_max_degree");
  }
  TM_CUDA(cudaStreamSynchronize(s));
  return TM_OK;
}

extern "C" int tm_graph_build(int device, int64_t n_nodes, int64_t n_edges, const int64_t *src,
                              const int64_t *dst, const int64_t *time, int inputs_on_device,
                              void *stream, tm_graph **out) {
  if (!out) return fail(TM_E_BAD_ARG, "out is NULL");
  *out = nullptr;
  if (n_nodes < 0 || n_edges < 0) return fail(TM_E_BAD_ARG, "negative size");
  if (n_edges >= (int64_t)INT32_MAX || n_nodes >= (int64_t)INT32_MAX)
    return fail(TM_E_OVERFLOW, "n_edges and n_nodes must be < 2^31");
  if (n_edges > 0 && (!src || !dst || !time)) return fail(TM_E_BAD_ARG, "NULL edge array");
  int ndev = 0;
  TM_CUDA(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) return fail(TM_E_BAD_ARG, "bad device ordinal");
  TM_CUDA(cudaSetDevice(device));
  tm_graph *g = new tm_graph();
  g->device = device;
  g->n_nodes = n_nodes;
  g->n_edges = n_edges;
  if (stream) {
    g->stream = static_cast<cudaStream_t>(stream);
  } else {
    // one persistent library stream per device: graphs rebuilt in a loop
    // allocate and free on the same stream, so the memory pool hands the
    // previous graph's blocks straight back (no new physical mappings)
    static std::mutex mu;
    static cudaStream_t lib_stream[64] = {};
    std::lock_guard<std::mutex> lock(mu);
    if (device >= 64) {
      delete g;
      return fail(TM_E_BAD_ARG, "device ordinal >= 64");
    }
    if (!lib_stream[device]) {
      cudaError_t e = cudaStreamCreateWithFlags(&lib_stream[device], cudaStreamNonBlocking);
      if (e != cudaSuccess) {
        lib_stream[device] = nullptr;
        delete g;
        return cuda_fail(e, "cudaStreamCreate");
      }
    }
    g->stream = lib_stream[device];
    g->owns_stream = false;
  }
  int rc = build_impl(g, src, dst, time, inputs_on_device);
  if (rc) {
    tm_graph_free(g);
    return rc;
  }
  int64_t bytes = 0;
  for (const DevBuf *b : {&g->e_src, &g->e_dst, &g->e_rank, &g->uniq_time, &g->loop, &g->time_order})
    bytes += (int64_t)b->bytes;
  for (int d = 0; d < 2; ++d)
    for (const DevBuf *b : {&g->ptr[d], &g->nbr[d], &g->rnk[d], &g->eid[d], &g->pkey[d], &g->prev[d], &g->peid[d],
                            &g->npk[d], &g->owner[d]})
      bytes += (int64_t)b->bytes;
  g->device_bytes = bytes;
  *out = g;
  return TM_OK;
}

extern "C" int tm_graph_info_get(const tm_graph *g, tm_graph_info *info) {
  if (!g || !info) return fail(TM_E_BAD_ARG, "NULL argument");
  std::memset(info, 0, sizeof(*info));
  info->n_nodes = g->n_nodes;
  info->n_edges = g->n_edges;
  info->n_ranks = g->n_ranks;
  if (g->maxdeg.p && g->n_edges > 0) {
    unsigned long long md[2] = {0, 0};
    TM_CUDA(cudaSetDevice(g->device));
    TM_CUDA(cudaMemcpyAsync(md, g->maxdeg.p, 16, cudaMemcpyDeviceToHost, g->stream));
    TM_CUDA(cudaStreamSynchronize(g->stream));
    info->max_out_degree = (int64_t)md[1];
    info->max_in_degree = (int64_t)md[0];
  }
  info->n_selfloops = g->n_selfloops;
  info->device_bytes = g->device_bytes;
  info->device = g->device;
  info->rank_bits = g->rank_bits;
  info->node_bits = g->node_bits;
  return TM_OK;
}

extern "C" int tm_graph_degrees(const tm_graph *g, int dir, int64_t *deg) {
  if (!g || !deg || (dir != 0 && dir != 1)) return fail(TM_E_BAD_ARG, "bad argument");
  TM_CUDA(cudaSetDevice(g->device));
  std::vector<int32_t> p(g->n_nodes + 1);
  TM_CUDA(cudaMemcpyAsync(p.data(), g->ptr[dir].p, 4 * (g->n_nodes + 1), cudaMemcpyDeviceToHost,
                          g->stream));
  TM_CUDA(cudaStreamSynchronize(g->stream));
  for (int64_t x = 0; x < g->n_nodes; ++x) deg[x] = p[x + 1] - p[x];
  return TM_OK;
}

extern "C" int tm_graph_export_csr(const tm_graph *g, int dir, int64_t *indptr, int64_t *nbr,
                                   int64_t *time, int64_t *eid) {
  if (!g || (dir != 0 && dir != 1)) return fail(TM_E_BAD_ARG, "bad argument");
  TM_CUDA(cudaSetDevice(g->device));
  const int64_t E = g->n_edges, N = g->n_nodes;
  cudaStream_t s = g->stream;
  std::vector<int32_t> tmp(std::max<int64_t>(E, N + 1));
  if (indptr) {
    TM_CUDA(cudaMemcpyAsync(tmp.data(), g->ptr[dir].p, 4 * (N + 1), cudaMemcpyDeviceToHost, s));
    TM_CUDA(cudaStreamSynchronize(s));
    for (int64_t i = 0; i <= N; ++i) indptr[i] = tmp[i];
  }
  if (E == 0) return TM_OK;
  if (nbr) {
    TM_CUDA(cudaMemcpyAsync(tmp.data(), g->nbr[dir].p, 4 * E, cudaMemcpyDeviceToHost, s));
    TM_CUDA(cudaStreamSynchronize(s));
    for (int64_t i = 0; i < E; ++i) nbr[i] = tmp[i];
  }
  if (eid) {
    TM_CUDA(cudaMemcpyAsync(tmp.data(), g->eid[dir].p, 4 * E, cudaMemcpyDeviceToHost, s));
    TM_CUDA(cudaStreamSynchronize(s));
    for (int64_t i = 0; i < E; ++i) eid[i] = tmp[i];
  }
  if (time) {
    DevBuf t;
    int rc;
    if ((rc = t.ensure(8 * E))) return rc;
    k_gather_time<<<grid_for(E, kB), kB, 0, s>>>(g->rnk[dir].as<uint32_t>(), g->uniq_time.as<int64_t>(),
                                                 E, t.as<int64_t>());
    TM_LAUNCHED("k_gather_time");
    TM_CUDA(cudaMemcpyAsync(time, t.p, 8 * E, cudaMemcpyDeviceToHost, s));
    TM_CUDA(cudaStreamSynchronize(s));
  }
  return TM_OK;
}

extern "C" void tm_graph_free(tm_graph *g) {
  if (!g) return;
  cudaSetDevice(g->device);
  // kernels enqueued on user streams may still read the graph: the last
  // call's completion event covers them (tm_graph::end)
  if (g->done_ev) {
    cudaEventSynchronize(g->done_ev);
    cudaEventDestroy(g->done_ev);
  }
  cudaStreamSynchronize(g->stream);
  bool own = g->owns_stream;
  cudaStream_t s = g->stream;
  for (int i = 0; i < 4; ++i)
    if (g->ev[i]) cudaEventDestroy(g->ev[i]);
  for (cudaEvent_t e : g->piece_ev)
    if (e) cudaEventDestroy(e);
  if (g->copy_stream) {
    cudaStreamSynchronize(g->copy_stream);
    cudaStreamDestroy(g->copy_stream);
  }

  delete g;  // DevBuf destructors free device memory
  if (own && s) cudaStreamDestroy(s);
}
