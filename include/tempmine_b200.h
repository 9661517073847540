/*
 * tempmine_b200.h — C ABI of the B200 mining engine (libtempmine_b200.so).
 *
 * This is the drop-in boundary for the reference's mining stage.  Each entry
 * point replaces one reference interface (paths relative to
 * /root/reference/pkg/src/tempmine):
 *
 *   tm_graph_build       TemporalGraph.__init__          txgraph.py:113-170
 *                        (dual (node,time,eid) CSR by np.lexsort :134-144,
 *                        _indptr :200-204, self-loop index :146-153) — here a
 *                        GPU radix-sort build plus (node,nbr,time) pair index
 *   tm_graph_export_csr  TemporalGraph.out_* / in_* arrays txgraph.py:139-144
 *                        (read back for CSR parity checks)
 *   tm_graph_degrees     GraphStats inputs (np.diff(indptr)) txgraph.py:155-162
 *   tm_mine              engine._mine_range kernel branch engine.py:607-628
 *                        dispatching _kernel_fn engine.py:569-589 to
 *                        kernels.batch_fan_degree :290, batch_cycle :306,
 *                        batch_scatter_gather :348, batch_stack :379; and the
 *                        generic-interpreter families cycle_5..8 / gs_count
 *                        (engine.py:516-562 on SURVEY.md Appendix B DSL)
 *   tm_mine_members      the same dispatch with attribution = "members":
 *                        engine.py:629-640 over _EmissionState instances
 *                        engine.py:433-513
 *   tm_csv_format /      FeatureMatrix.to_csv engine.py:73-103 (GPU int->text)
 *   tm_csv_fetch
 *   tm_last_error        Python exceptions EngineInvariantError /
 *                        ValueError (engine.py:33,589,669-670)
 *
 * Conventions: C linkage, fixed-width integers, no torch types.  Every call
 * returns TM_OK (0) or a negative tm_status; tm_last_error() then holds a
 * thread-local message.  Host buffers are caller-owned; device memory is
 * owned by the tm_graph handle.  Calls on one graph must be serialized by
 * the caller (the Python wrapper does this).  There is no CPU fallback: a
 * plan the GPU path does not implement fails with TM_E_UNSUPPORTED_PLAN.
 */
#ifndef TEMPMINE_B200_H
#define TEMPMINE_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TM_ABI_VERSION 2

/* pattern families (plan.py kernel hints + the extended north-star set) */
enum tm_family {
  TM_FAN = 1,    /* hint FAN:     fan_in / fan_out            kernels.py:290 */
  TM_DEGREE = 2, /* hint DEGREE:  deg_{in,out}_{src,dst}      kernels.py:290 */
  TM_CYCLE = 3,  /* CYCLE_2/3/4 (kernels.py:306) and cycle_5..8 (generic)   */
  TM_SG = 4,     /* SCATTER_GATHER                            kernels.py:348 */
  TM_GS = 5,     /* gather-scatter (generic)          */
  TM_STACK = 6   /* STACK                                     kernels.py:379 */
};

enum tm_status {
  TM_OK = 0,
  TM_E_CUDA = -1,
  TM_E_OOM = -2,
  TM_E_BAD_ARG = -3,
  TM_E_UNSUPPORTED_PLAN = -4,
  TM_E_OVERFLOW = -5,
  TM_E_STATE = -6
};

/* One feature column.  Mirrors the fields _kernel_fn reads from an
 * ExecutionPlan (engine.py:572-588): delta, emission.min_size and, for
 * FAN/DEGREE, cells[0].src[0].base/.direction. */
typedef struct tm_plan_desc {
  int32_t family;          /* enum tm_family */
  int32_t endpoint;        /* FAN/DEGREE: 0 = N0 (trigger src), 1 = N1 (dst) */
  int32_t direction;       /* FAN/DEGREE: 0 = in_neigh, 1 = out_neigh */
  int32_t exclude_trigger; /* FAN: 1 (skip_if e1 == e0), DEGREE: 0 */
  int32_t cycle_len;       /* CYCLE: 2..8 */
  int32_t min_size;        /* emission min_size, >= 1 */
  int64_t delta;           /* window length in ticks, >= 0 */
} tm_plan_desc;

typedef struct tm_graph tm_graph;

typedef struct tm_graph_info {
  int64_t n_nodes;
  int64_t n_edges;
  int64_t n_ranks;      /* distinct timestamps */
  int64_t max_out_degree;
  int64_t max_in_degree;
  int64_t n_selfloops;
  int64_t device_bytes; /* resident graph footprint */
  int32_t device;
  int32_t rank_bits;
  int32_t node_bits;
  int32_t reserved;
} tm_graph_info;

typedef struct tm_mine_stats {
  int64_t triggers;       /* rows mined by the last tm_mine */
  int64_t heavy_triggers; /* rows deferred to the cooperative (warp) kernel,
                             -1 when not read back (device-output calls) */
  int64_t kernel_launches;/* launches issued by the last tm_mine */
  float light_ms;         /* CUDA-event time of the last call's per-thread
                             kernel (profiling on), else -1 */
  float heavy_ms;         /* same for the heavy (per-warp + task) kernels,
                             summed over pipeline chunks (they overlap the
                             next chunk's light kernel) */
  float total_ms;         /* CUDA-event time of the whole call on the device */
  int32_t reserved;
} tm_mine_stats;

int tm_abi_version(void);

/* Build the device graph from edge arrays (int64, length n_edges).
 * inputs_on_device = 0: host pointers (copied H2D inside);
 *                    1: device pointers on `device`.
 * n_nodes must exceed every src/dst id (build_graph uses max id + 1,
 * txgraph.py:353).  Requires n_edges < 2^31 and n_nodes < 2^31. */
int tm_graph_build(int device, int64_t n_nodes, int64_t n_edges, const int64_t *src,
                   const int64_t *dst, const int64_t *time, int inputs_on_device,
                   void *stream, tm_graph **out);

int tm_graph_info_get(const tm_graph *g, tm_graph_info *info);

/* dir: 0 = in-CSR, 1 = out-CSR.  Host buffers: indptr[n_nodes+1],
 * nbr/time/eid[n_edges]; any may be NULL to skip. */
int tm_graph_export_csr(const tm_graph *g, int dir, int64_t *indptr, int64_t *nbr, int64_t *time,
                        int64_t *eid);

/* Per-node degree (dir 0 = in, 1 = out) into a host int64[n_nodes]. */
int tm_graph_degrees(const tm_graph *g, int dir, int64_t *deg);

/* Mine rows [lo, hi) for n_plans columns into out[(hi-lo) * n_plans]
 * (C order, row = trigger edge id - lo, column = plan index).
 * out_on_device = 0: host buffer (D2H inside, call is synchronous);
 *                 1: device buffer, work is enqueued on `stream`
 *                    (NULL = the graph's stream) and the call returns
 *                    without synchronizing. */
int tm_mine(tm_graph *g, const tm_plan_desc *plans, int n_plans, int64_t lo, int64_t hi,
            int64_t *out, int out_on_device, void *stream);

/* Stats of the last tm_mine; with profiling on this waits for that call's
 * kernels to finish and fills the event timings. */
/* Members attribution (engine.py:629-640, pattern_grammar.md:116-122):
 * every instance found at a trigger in [lo, hi) that has the trigger as its
 * temporally last member adds 1 to the row of EVERY member edge, so `out`
 * is the full (n_edges x n_plans) block (C order).
 * out_on_device = 1: contributions are ADDED into out (enqueued on stream);
 *                 0: host out is overwritten with this range's block. */
int tm_mine_members(tm_graph *g, const tm_plan_desc *plans, int n_plans, int64_t lo, int64_t hi,
                    int64_t *out, int out_on_device, void *stream);

int tm_last_mine_stats(tm_graph *g, tm_mine_stats *stats);

/* Feature CSV rows (FeatureMatrix.to_csv, engine.py:73-103; header line not
 * included): "edge_id,src,dst,timestamp,label,<features>\n" per edge, "%d"
 * fields, empty label cell when labels is NULL or the label is negative.
 * values: n_edges x n_cols int64 (host, or device when values_on_device);
 * labels: host int8[n_edges] or NULL.  The text stays on the device;
 * *out_bytes receives its length, tm_csv_fetch copies it out. */
int tm_csv_format(tm_graph *g, const int64_t *values, int values_on_device, int n_cols,
                  const int8_t *labels, int64_t *out_bytes);
int tm_csv_fetch(tm_graph *g, char *dst, int64_t n_bytes);

/* on = 1: bracket the mining kernels of every tm_mine with CUDA events on
 * the launch stream (read back by tm_last_mine_stats). */
int tm_set_profiling(tm_graph *g, int on);

/* Total kernels this process launched through the library. */
int64_t tm_kernel_launch_count(void);

const char *tm_last_error(void);

void tm_graph_free(tm_graph *g);

#ifdef __cplusplus
}
#endif

#endif /* TEMPMINE_B200_H */
