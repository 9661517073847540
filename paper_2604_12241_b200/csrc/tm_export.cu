// tm_export.cu — feature CSV formatting on the GPU.
//
// Reference: FeatureMatrix.to_csv (engine.py:73-103): one line per edge,
// "edge_id,src,dst,timestamp,label,<features>" with "%d" fields and an empty
// label cell when the label is negative.  At HI-Large that is ~3.4 G
// integers — minutes of Python formatting.  Here: one thread per row
// computes the row's byte length, a 64-bit exclusive scan turns lengths
// into offsets, one thread per row writes its digits; the text is fetched
// with one D2H copy.  The bytes equal the reference writer's (tested).
#include "tm_internal.cuh"

namespace tmb {
namespace {

constexpr int kB = 256;

__device__ __forceinline__ int ndigits(long long x) {
  unsigned long long ux = x < 0 ? 0ull - (unsigned long long)x : (unsigned long long)x;
  int n = 1;
  while (ux >= 10ull) {
    ux /= 10ull;
    ++n;
  }
  return n + (x < 0);
}

__device__ __forceinline__ char *put(char *p, long long x) {
  const int n = ndigits(x);
  unsigned long long ux = x < 0 ? 0ull - (unsigned long long)x : (unsigned long long)x;
  char *q = p + n;
  do {
    *--q = (char)('0' + ux % 10ull);
    ux /= 10ull;
  } while (ux);
  if (x < 0) *--q = '-';
  return p + n;
}

struct Row {
  long long src, dst, t;
  int label;
};

__device__ __forceinline__ Row row_of(const DevGraph &g, const int64_t *uniq, const int8_t *labels,
                                      int64_t i) {
  return Row{__ldg(g.e_src + i), __ldg(g.e_dst + i), (long long)__ldg(uniq + __ldg(g.e_rank + i)),
             labels ? (int)labels[i] : -1};
}

__global__ void k_csv_len(const __grid_constant__ DevGraph g, const int64_t *__restrict__ uniq,
                          const int8_t *__restrict__ labels, const long long *__restrict__ vals,
                          int64_t n, int C, unsigned long long *__restrict__ len) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const Row r = row_of(g, uniq, labels, i);
  unsigned long long L = ndigits(i) + ndigits(r.src) + ndigits(r.dst) + ndigits(r.t) + 4 + 1;
  if (r.label >= 0) L += ndigits(r.label);
  for (int j = 0; j < C; ++j) L += 1 + ndigits(vals[i * C + j]);
  len[i] = L;
}

__global__ void k_csv_write(const __grid_constant__ DevGraph g, const int64_t *__restrict__ uniq,
                            const int8_t *__restrict__ labels, const long long *__restrict__ vals,
                            int64_t n, int C, const unsigned long long *__restrict__ off,
                            char *__restrict__ buf) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const Row r = row_of(g, uniq, labels, i);
  char *p = buf + off[i];
  p = put(p, i);
  *p++ = ',';
  p = put(p, r.src);
  *p++ = ',';
  p = put(p, r.dst);
  *p++ = ',';
  p = put(p, r.t);
  *p++ = ',';
  if (r.label >= 0) p = put(p, r.label);
  for (int j = 0; j < C; ++j) {
    *p++ = ',';
    p = put(p, vals[i * C + j]);
  }
  *p = '\n';
}

// exclusive scan of uint64 (in place), 1024 threads x 4 items per tile
constexpr int kST = 1024, kSI = 4, kTile = kST * kSI;

__global__ void __launch_bounds__(kST) k_scan64(unsigned long long *__restrict__ a, int64_t n,
                                                unsigned long long *__restrict__ sums) {
  __shared__ unsigned long long ws[kST / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t base = (int64_t)blockIdx.x * kTile + (int64_t)threadIdx.x * kSI;
  unsigned long long x[kSI], s = 0;
#pragma unroll
  for (int k = 0; k < kSI; ++k) {
    x[k] = base + k < n ? a[base + k] : 0ull;
    s += x[k];
  }
  unsigned long long inc = s;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) ws[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    const unsigned long long w = lane < kST / 32 ? ws[lane] : 0ull;
    unsigned long long wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long y = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += y;
    }
    if (lane < kST / 32) ws[lane] = wi - w;
    if (lane == 31 && sums) sums[blockIdx.x] = wi;
  }
  __syncthreads();
  unsigned long long run = ws[warp] + inc - s;
#pragma unroll
  for (int k = 0; k < kSI; ++k) {
    if (base + k < n) a[base + k] = run;
    run += x[k];
  }
}

__global__ void k_scan64_add(unsigned long long *__restrict__ a, int64_t n,
                             const unsigned long long *__restrict__ sums) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) a[i] += sums[i / kTile];
}

int scan64(unsigned long long *a, int64_t n, cudaStream_t s) {
  if (n <= 0) return TM_OK;
  const int64_t tiles = (n + kTile - 1) / kTile;
  if (tiles == 1) {
    k_scan64<<<1, kST, 0, s>>>(a, n, nullptr);
    TM_LAUNCHED("k_scan64");
    return TM_OK;
  }
  unsigned long long *sums = nullptr;
  TM_CUDA(pool_malloc((void **)&sums, sizeof(unsigned long long) * tiles, s));
  k_scan64<<<(unsigned)tiles, kST, 0, s>>>(a, n, sums);
  TM_LAUNCHED("k_scan64");
  int rc = scan64(sums, tiles, s);
  if (rc) return rc;
  k_scan64_add<<<grid_for(n, kB), kB, 0, s>>>(a, n, sums);
  TM_LAUNCHED("k_scan64_add");
  TM_CUDA(cudaFreeAsync(sums, s));
  return TM_OK;
}

}  // namespace

int scan_u64_exclusive(unsigned long long *a, int64_t n, cudaStream_t s) { return scan64(a, n, s); }

}  // namespace tmb

using namespace tmb;

extern "C" int tm_csv_format(tm_graph *g, const int64_t *values, int values_on_device, int n_cols,
                             const int8_t *labels, int64_t *out_bytes) {
  if (!g || !out_bytes || n_cols < 0 || (n_cols > 0 && !values && g->n_edges > 0))
    return fail(TM_E_BAD_ARG, "bad argument");
  *out_bytes = 0;
  const int64_t E = g->n_edges;
  if (E == 0) return TM_OK;
  TM_CUDA(cudaSetDevice(g->device));
  cudaStream_t s = g->stream;
  int rc;
  DevBuf vals, lab, len;
  const long long *dv = reinterpret_cast<const long long *>(values);
  if (!values_on_device && n_cols > 0) {
    if ((rc = vals.ensure_on(sizeof(long long) * (size_t)E * n_cols, s))) return rc;
    TM_CUDA(cudaMemcpyAsync(vals.p, values, sizeof(long long) * (size_t)E * n_cols,
                            cudaMemcpyHostToDevice, s));
    dv = vals.as<long long>();
  }
  const int8_t *dl = nullptr;
  if (labels) {
    if ((rc = lab.ensure_on((size_t)E, s))) return rc;
    TM_CUDA(cudaMemcpyAsync(lab.p, labels, (size_t)E, cudaMemcpyHostToDevice, s));
    dl = lab.as<int8_t>();
  }
  if ((rc = len.ensure_on(sizeof(unsigned long long) * (size_t)(E + 1), s))) return rc;
  const DevGraph dg = g->dev();
  k_csv_len<<<grid_for(E, kB), kB, 0, s>>>(dg, g->uniq_time.as<int64_t>(), dl, dv, E, n_cols,
                                           len.as<unsigned long long>());
  TM_LAUNCHED("k_csv_len");
  TM_CUDA(cudaMemsetAsync(len.as<unsigned long long>() + E, 0, sizeof(unsigned long long), s));
  if ((rc = scan64(len.as<unsigned long long>(), E + 1, s))) return rc;  // [E] = total
  unsigned long long total = 0;
  TM_CUDA(cudaMemcpyAsync(&total, len.as<unsigned long long>() + E, sizeof(total),
                          cudaMemcpyDeviceToHost, s));
  TM_CUDA(cudaStreamSynchronize(s));
  if ((rc = g->csv_buf.ensure(total ? total : 1))) return rc;
  k_csv_write<<<grid_for(E, kB), kB, 0, s>>>(dg, g->uniq_time.as<int64_t>(), dl, dv, E, n_cols,
                                             len.as<unsigned long long>(), g->csv_buf.as<char>());
  TM_LAUNCHED("k_csv_write");
  TM_CUDA(cudaStreamSynchronize(s));
  g->csv_bytes = (int64_t)total;
  *out_bytes = (int64_t)total;
  return TM_OK;
}

extern "C" int tm_csv_fetch(tm_graph *g, char *dst, int64_t n_bytes) {
  if (!g || (!dst && n_bytes > 0) || n_bytes > g->csv_bytes) return fail(TM_E_BAD_ARG, "bad argument");
  if (n_bytes == 0) return TM_OK;
  TM_CUDA(cudaSetDevice(g->device));
  TM_CUDA(cudaMemcpyAsync(dst, g->csv_buf.p, (size_t)n_bytes, cudaMemcpyDeviceToHost, g->stream));
  TM_CUDA(cudaStreamSynchronize(g->stream));
  return TM_OK;
}
