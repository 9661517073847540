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
 *   tm_collect_instances mine(..., collect_instances=True) engine.py:629-645,
 *   tm_fetch_instances   InstanceRecord engine.py:37-52 from _EmissionState
 *                        engine.py:455-513 (records; host dedup + sort)
 *   tm_csv_format /      FeatureMatrix.to_csv engine.py:73-103 (GPU int->text)
 *   tm_csv_fetch
 *   tm_ingest_csv /      txgraph.parse_transactions txgraph.py:253-314 +
 *   tm_ingest_fetch /    build_graph :317-354 (CSV rows -> dense first-seen
 *   tm_ingest_vocab /    node ids, ticks, amounts, currency codes, labels)
 *   tm_ingest_graph
 *   tm_last_error        Python exceptions EngineInvariantError /
 *                        ValueError (engine.py:33,589,669-670)
 *
 * Conventions: C linkage, fixed-width integers, no torch types.  Every call
 * returns TM_OK (0) or a negative tm_status; tm_last_error() then holds a
 * thread-local message.  Host buffers are caller-owned; device memory is
 * owned by the tm_graph handle.  Calls on one graph must not run
 * concurrently from several host threads (they share the handle's scratch
 * and result buffers): the Python wrapper holds a per-graph lock around
 * every call sequence (DeviceGraph.lock).  Work a call enqueues on a user
 * stream is ordered before the next call on the same graph and before
 * tm_graph_free.  There is no CPU fallback: a plan the GPU path does not
 * implement fails with TM_E_UNSUPPORTED_PLAN.
 */
#ifndef TEMPMINE_B200_H
#define TEMPMINE_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TM_ABI_VERSION 7

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
  int64_t heavy_triggers; /* rows whose slices went to the task queue (split
                             rows), -1 when not read back (device-output calls) */
  int64_t kernel_launches;/* launches issued by the last tm_mine */
  float light_ms;         /* CUDA-event time (profiling on, else -1) of the
                             trigger kernel (k_mine_warp) */
  float heavy_ms;         /* from there to the end of the task rounds and
                             k_mine_finalize (task kernel time) */
  float total_ms;         /* CUDA-event time of the whole call on the device */
  float prep_ms;          /* from the call's start to the trigger kernel:
                             window-start tables, time-slab views */
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

/* Build the window-start tables and time-slab views of the plans' deltas for
 * triggers [lo, hi) once and keep them on the graph: tm_mine calls on
 * sub-ranges of [lo, hi) with those deltas reuse them instead of building
 * their own per call.  With edge ids in time order only the slabs holding
 * [lo, hi) are built (a multi-GPU rank's share; one host sync).  Replaces
 * any earlier preparation.  Replaces: the per-worker setup of the
 * reference's fork pool (engine.py:677-690), which shares one TemporalGraph. */
int tm_mine_prepare(tm_graph *g, const tm_plan_desc *plans, int n_plans, int64_t lo, int64_t hi,
                    void *stream);

/* Forget the prepared tables (their device memory stays with the graph). */
int tm_mine_release(tm_graph *g);

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

/* Instance records of triggers [lo, hi) (engine.py:629-645 with collect):
 * every instance the reference's _EmissionState appends (engine.py:455-513),
 * whatever the plan's attribution, as an int32 stream of records
 *   [plan index, trigger edge, n_edges, n_nodes, edges..., nodes...]
 * ordered by trigger, then plan.  Edge / node lists may hold duplicates
 * (the reference's frozensets dedup them) and are unsorted.  The stream
 * stays on the device; *out_words receives its length in int32 words and
 * tm_fetch_instances copies the first n_words out (synchronous). */
int tm_collect_instances(tm_graph *g, const tm_plan_desc *plans, int n_plans, int64_t lo, int64_t hi,
                         int64_t *out_words);
int tm_fetch_instances(tm_graph *g, int32_t *dst, int64_t n_words);

/* Feature CSV rows (FeatureMatrix.to_csv, engine.py:73-103; header line not
 * included): "edge_id,src,dst,timestamp,label,<features>\n" per edge, "%d"
 * fields, empty label cell when labels is NULL or the label is negative.
 * values: n_edges x n_cols int64 (host, or device when values_on_device);
 * labels: host int8[n_edges] or NULL.  The text stays on the device;
 * *out_bytes receives its length, tm_csv_fetch copies it out. */
int tm_csv_format(tm_graph *g, const int64_t *values, int values_on_device, int n_cols,
                  const int8_t *labels, int64_t *out_bytes);
int tm_csv_fetch(tm_graph *g, char *dst, int64_t n_bytes);

/* ---------------------------------------------------------------------
 * GENERIC stage programs: the reference's generic
 * interpreter (engine.py:325-562 — execute_cell, _adjacency_map,
 * _order_satisfiable, run_plan_on_trigger, _EmissionState) as a device VM.
 * A program is one compiled ExecutionPlan (plan.py:40-91) lowered by the
 * host: cells in plan order, variables numbered 0 = N0, 1 = N1, 2 + i =
 * cell i's dst_var; edge symbols 0 = e0, k = eK. */
#define TM_VM_MAX_CELLS 8
#define TM_VM_MAX_OPS 4
#define TM_VM_MAX_PREDS 8
#define TM_VM_MAX_SYMS 16
#define TM_VM_TABLE 1024

enum tm_vm_op { TM_VM_FOR_ALL = 0, TM_VM_INTERSECT = 1, TM_VM_UNION = 2, TM_VM_DIFFERENTIATE = 3 };
enum tm_vm_operand_kind { TM_VM_SCALAR = 0, TM_VM_SET = 1, TM_VM_ADJ = 2, TM_VM_MEMBER_ADJ = 3 };
enum tm_vm_mode {
  TM_VM_SET_CARDINALITY = 0, TM_VM_SOURCE_COUNT = 1, TM_VM_PAIR_PRODUCT = 2,
  TM_VM_EDGE_COUNT = 3, TM_VM_INSTANCE_LIST = 4
};
/* comparison operators (engine.py:_compare) */
enum tm_vm_cmp { TM_VM_EQ = 0, TM_VM_NE = 1, TM_VM_LE = 2, TM_VM_LT = 3, TM_VM_GE = 4, TM_VM_GT = 5 };
/* value kinds of an edge-predicate term (engine.py:_edge_pred_keeps) */
enum tm_vm_term {
  TM_VM_T_NUMBER = 0,   /* num */
  TM_VM_T_EID = 1,      /* ref 0: the trigger's id, 1: the entry's id */
  TM_VM_T_TIME = 2,     /* the entry's timestamp */
  TM_VM_T_AMOUNT = 3,   /* ref 0: trigger, 1: entry */
  TM_VM_T_CURRENCY = 4, /* ref 0: trigger, 1: entry (compared via vocab rank or table) */
  TM_VM_T_CONST = 5     /* the whole predicate folds to `num != 0` (type-mismatch ==/!=) */
};

typedef struct tm_vm_pred {
  int32_t cmp;          /* enum tm_vm_cmp */
  int32_t lk, lref;     /* lhs kind (enum tm_vm_term), ref */
  int32_t rk, rref;
  int32_t table;        /* currency vs string: offset of a holds[n_vocab] table, else -1 */
  int32_t sym;          /* edge pred: own symbol it filters; gate pred: bound symbol it tests */
  int32_t pad;
  double lnum, rnum;
} tm_vm_pred;

typedef struct tm_vm_operand {
  int32_t kind;         /* enum tm_vm_operand_kind */
  int32_t var;          /* base variable */
  int32_t slot;         /* referenced cell (set / member_adj), -1 for N0 / N1 */
  int32_t dir;          /* 0 in_neigh, 1 out_neigh (adjacency kinds) */
  int32_t sym;          /* edge symbol (adjacency kinds), -1 otherwise */
} tm_vm_operand;

typedef struct tm_vm_cell {
  int32_t op;           /* enum tm_vm_op */
  int32_t parent;       /* -1 at trigger level */
  int32_t forward;      /* window [t, t + delta] instead of [t - delta, t] */
  int32_t n_ops;
  tm_vm_operand ops[TM_VM_MAX_OPS];
  int32_t n_node, n_edge, n_gate, n_order;
  int32_t node[TM_VM_MAX_PREDS][3];   /* skip_if var == / != var: cmp, lvar, rvar */
  tm_vm_pred edge[TM_VM_MAX_PREDS];   /* per-entry skip predicates */
  tm_vm_pred gate[TM_VM_MAX_PREDS];   /* predicates over already-bound edges */
  int32_t order[TM_VM_MAX_PREDS][3];  /* cmp, lhs sym, rhs sym (-1 = trigger time t) */
} tm_vm_cell;

typedef struct tm_vm_program {
  int32_t n_cells;
  int32_t mode;         /* enum tm_vm_mode */
  int32_t min_size;
  int32_t target[2];    /* emission target cells (pair_product: both) */
  int32_t uses_attrs;   /* amount / currency terms present: tm_graph_set_attrs first */
  int64_t delta;
  tm_vm_cell cells[TM_VM_MAX_CELLS];
  int8_t table[TM_VM_TABLE];
} tm_vm_program;

/* Edge attributes for attribute predicates: amount float64[n_edges],
 * currency int32[n_edges] (vocabulary ids), cur_rank int32[n_vocab] (rank of
 * each vocabulary string in sorted order).  Host pointers. */
int tm_graph_set_attrs(tm_graph *g, const double *amount, const int32_t *currency, int32_t n_vocab,
                       const int32_t *cur_rank);

/* Counts of triggers [lo, hi) into host out[hi - lo] (trigger attribution,
 * engine.py:607-646 generic branch). */
int tm_vm_mine(tm_graph *g, const tm_vm_program *prog, int64_t lo, int64_t hi, int64_t *out);

/* Instance records of triggers [lo, hi), tm_collect_instances' format with
 * `plan_index` in the plan field; fetch with tm_fetch_instances. */
int tm_vm_collect(tm_graph *g, const tm_vm_program *prog, int32_t plan_index, int64_t lo, int64_t hi,
                  int64_t *out_words);

/* Members attribution of triggers [lo, hi): host out[n_edges] (overwritten). */
int tm_vm_members(tm_graph *g, const tm_vm_program *prog, int64_t lo, int64_t hi, int64_t *out);

/* ------------------------------------------------------------------ ingestion
 *
 * tm_ingest_csv replaces txgraph.parse_transactions (txgraph.py:253-314) +
 * build_graph (:317-354): the data rows of a delimited transaction log (the
 * bytes AFTER the header row; the host resolves the header against the
 * ColumnMapping, _resolve_columns :207-234) are split, parsed and given
 * dense first-seen node ids and currency codes on the GPU.  Row semantics
 * follow csv.reader (excel dialect, no quoted fields: a '"' anywhere is
 * TM_PARSE_UNSUPPORTED) and the reference's per-row checks, in its order.
 */
enum tm_parse_status {
  TM_PARSE_OK = 0,
  TM_PARSE_COLUMNS = 1,      /* fewer than needed + 1 fields (:289-290) */
  TM_PARSE_TIMESTAMP = 2,    /* not an int, and no / no matching strptime format (:237-247) */
  TM_PARSE_NEGATIVE = 3,     /* negative timestamp (:294-295) */
  TM_PARSE_AMOUNT = 4,       /* float() would fail (:296) */
  TM_PARSE_LABEL = 5,        /* unrecognized label value (:307-308) */
  TM_PARSE_UNSUPPORTED = 6,  /* valid for Python but outside the GPU parser */
  TM_PARSE_COLLISION = 7     /* two distinct keys share a 64-bit hash (never expected) */
};

/* strptime program ops (ColumnMapping.timestamp_format, compiled host-side) */
enum tm_fmt_op {
  TM_FMT_END = 0, TM_FMT_LIT = 1, TM_FMT_SPACE = 2, TM_FMT_Y = 3, TM_FMT_y = 4, TM_FMT_m = 5,
  TM_FMT_d = 6, TM_FMT_H = 7, TM_FMT_M = 8, TM_FMT_S = 9
};
#define TM_FMT_MAX 48

typedef struct tm_csv_mapping {
  /* field index per mapped column, -1 = not mapped (ColumnMapping fields) */
  int32_t col_timestamp, col_src_bank, col_src_account, col_dst_bank, col_dst_account;
  int32_t col_amount, col_currency, col_label;
  int32_t needed;        /* max mapped index: rows need needed + 1 fields */
  int32_t delimiter;     /* one byte */
  int64_t tick_seconds;  /* >= 1; divides parsed datetimes only */
  int32_t n_fmt;         /* 0: integer timestamps only (timestamp_format None) */
  int32_t fmt_op[TM_FMT_MAX], fmt_arg[TM_FMT_MAX];
} tm_csv_mapping;

typedef struct tm_ingest_info {
  int64_t n_rows;      /* data rows seen by csv.reader (blank rows included) */
  int64_t n_edges;     /* records */
  int64_t n_nodes;     /* distinct (bank, account) keys */
  int64_t n_currency;  /* distinct currency strings */
  int64_t err_row;     /* -1, or 0-based data row of the first failing row */
  int32_t err_status;  /* enum tm_parse_status of that row */
  int32_t pad;
  int64_t err_begin, err_end;  /* byte span of that row in the input */
} tm_ingest_info;

typedef struct tm_ingest tm_ingest;

/* Parse `len` bytes (host, or device when on_device) on `device`.  On a
 * row error the call still succeeds (returns 0) with info->err_row >= 0 so
 * the host can raise ParseError(line = err_row + 2) with the reference's
 * message; *out is then NULL. */
int tm_ingest_csv(int device, const char *buf, int64_t len, int on_device, const tm_csv_mapping *m,
                  void *stream, tm_ingest **out, tm_ingest_info *info);

/* Host copies of the edge table (any pointer may be NULL):
 * src/dst/time int64[E], amount float64[E], currency int32[E], label int8[E]
 * (-1 = no label column), like build_graph's arrays. */
int tm_ingest_fetch(tm_ingest *h, int64_t *src, int64_t *dst, int64_t *time, double *amount,
                    int32_t *currency, int8_t *label);

/* Currency vocabulary in code (first-seen) order: offsets int64[n_currency+1]
 * into bytes (capacity cap; returns the byte total needed via offsets). */
int tm_ingest_vocab(tm_ingest *h, int64_t *offsets, char *bytes, int64_t cap);

/* Build the device graph straight from the parsed device-resident edge
 * arrays (no host round trip), as tm_graph_build with inputs_on_device. */
int tm_ingest_graph(tm_ingest *h, tm_graph **out);

void tm_ingest_free(tm_ingest *h);

/* on = 1: bracket the mining kernels of every tm_mine with CUDA events on
 * the launch stream (read back by tm_last_mine_stats). */
int tm_set_profiling(tm_graph *g, int on);

/* Total kernels this process launched through the library. */
int64_t tm_kernel_launch_count(void);

/* Page-locked (pinned, portable) host memory: outputs written here get the
 * overlapped piece-wise D2H of tm_mine.  Replaces the pageable np.zeros the
 * reference's mine() allocates for FeatureMatrix.values (engine.py:693). */
int tm_host_alloc(int64_t bytes, void **out);
void tm_host_free(void *p);

const char *tm_last_error(void);

void tm_graph_free(tm_graph *g);

#ifdef __cplusplus
}
#endif

#endif /* TEMPMINE_B200_H */
