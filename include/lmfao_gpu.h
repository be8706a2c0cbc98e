/* lmfao_gpu.h — C ABI of the B200-native LMFAO hot path.
 *
 * Evaluates a batch of group-by aggregates over the natural join of an acyclic
 * schema, bottom-up over a join tree, without materialising the join
 * (§3 "Problem Statement" P:336-347, §4):
 *
 *     Q(F_1..F_f; α_1..α_ℓ) += R_1(ω_1), …, R_m(ω_m)
 *     α_i = Σ_j Π_k f_ijk,  f ∈ {constant, identity, Kronecker 1_{X op t}}
 *
 * Semantics (DESIGN.md §3 readings): bag semantics (duplicates multiply, tuples
 * with dangling keys vanish); a query with no group-by attribute returns exactly
 * one row, also over an empty join (value 0, count 0); a query with group-by
 * attributes returns exactly the groups present in the join, in ascending
 * lexicographic order of the group-key tuple (in the order the attributes were
 * listed), together with each group's join multiplicity ("count").
 *
 * Conventions
 *  - Every function returns lmfao_status.  No C++ exception, abort or CUDA error
 *    crosses this boundary; after a non-OK status lmfao_last_error(ctx) returns a
 *    message (valid until the next call on that ctx).
 *  - Call order: create -> add_relation* -> set_join_tree -> prepare ->
 *    add_query* -> plan -> run* -> (result_shape | fetch | result_device)*.
 *    A call out of order returns LMFAO_ERR_STATE.  run may be repeated.
 *  - One ctx per (process, GPU); a ctx is not thread-safe.
 *  - Inputs are copied (the caller keeps ownership).  Host output buffers are
 *    caller-owned; device views returned by lmfao_result_device are
 *    library-owned and valid until the next run/destroy.
 *  - Multi-GPU (world > 1, one process per GPU): each rank passes the whole root
 *    relation; after the global sort in lmfao_prepare the rank keeps its
 *    contiguous shard of the sorted root (domain parallelism, "partition
 *    the largest relation"), dimension relations are replicated, and lmfao_run
 *    merges the partial aggregates over NVLink / NVSwitch: scalar queries and
 *    group-by tables below LMFAO_DIST_CELLS cells (default 65536) by an NCCL
 *    all-reduce (complete on every rank); larger dense tables by a
 *    reduce-scatter, and sparse data-cube cuboids by an exchange through peer
 *    memory (CUDA IPC), after which each rank holds the groups of its own
 *    contiguous range of cells (lmfao_owner_range) — lmfao_result_shape /
 *    lmfao_fetch return that range, lmfao_gather_result assembles the whole
 *    table on one rank.  lmfao_plan_info lists each query's placement.
 *  - There is no CPU fallback: without a usable CUDA device every call that
 *    needs one returns LMFAO_ERR_CUDA.
 */
#ifndef LMFAO_GPU_H
#define LMFAO_GPU_H

#include <stdint.h>

#if defined(__GNUC__)
#define LMFAO_API __attribute__((visibility("default")))
#else
#define LMFAO_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  LMFAO_OK = 0,
  LMFAO_ERR_INVALID_ARG = 1,        /* null pointer, negative size, bad enum, duplicate name */
  LMFAO_ERR_STATE = 2,              /* call out of order */
  LMFAO_ERR_UNKNOWN_ATTR = 3,       /* attribute / relation name or id does not exist */
  LMFAO_ERR_TYPE = 4,               /* join or group-by attribute not int32; dtype mismatch */
  LMFAO_ERR_CYCLIC_TREE = 5,        /* join tree has a cycle */
  LMFAO_ERR_DISCONNECTED_TREE = 6,  /* join tree does not span all relations */
  LMFAO_ERR_RUNNING_INTERSECTION = 7, /* ω_i ∩ ω_j ⊄ ω_k for some R_k on the path */
  LMFAO_ERR_UNSUPPORTED = 8,        /* limits: join keys of more than eight attributes, group-by
                                       attributes no root can place (see lmfao_add_query) */
  LMFAO_ERR_OOM = 9,                /* device allocation failed */
  LMFAO_ERR_CUDA = 10,              /* CUDA runtime error / no device */
  LMFAO_ERR_NCCL = 11               /* NCCL error (multi-GPU) */
} lmfao_status;

typedef enum { LMFAO_INT32 = 0, LMFAO_FP64 = 1 } lmfao_dtype;

/* Per-attribute functions f of a product term: constant, identity, and
 * the Kronecker delta 1_{X op t} for op in {<, <=, >, >=, =, !=}, compared in
 * IEEE double (int32 attributes convert exactly); LMFAO_F_IN is set inclusion
 * 1_{X ∈ S} for categorical splits, S ⊆ {0..52} given as the bit mask
 * param = Σ_{v ∈ S} 2^v (an exact integer below 2^53): true iff X is an integer
 * v in [0, 52] whose bit is set. */
typedef enum {
  LMFAO_F_CONST = 0, LMFAO_F_IDENT = 1, LMFAO_F_LT = 2, LMFAO_F_LE = 3,
  LMFAO_F_GT = 4, LMFAO_F_GE = 5, LMFAO_F_EQ = 6, LMFAO_F_NE = 7, LMFAO_F_IN = 8
} lmfao_fkind;

typedef struct {
  int32_t kind;   /* lmfao_fkind */
  int32_t attr;   /* attribute id (lmfao_attr_id); -1 for LMFAO_F_CONST */
  double param;   /* CONST: the value; predicates: the threshold t */
} lmfao_factor;

typedef struct {
  double coeff;                 /* multiplies the product */
  int32_t n_factors;            /* >= 0; 0 means the product is just coeff */
  const lmfao_factor* factors;
} lmfao_product;

typedef struct {
  int32_t n_products;           /* α = Σ products; 0 means α ≡ 0 */
  const lmfao_product* products;
} lmfao_udaf;

typedef struct lmfao_ctx lmfao_ctx;

/* Size of the opaque id passed to lmfao_create for world > 1 (ncclUniqueId). */
#define LMFAO_UNIQUE_ID_BYTES 128

/* Fills `out` (LMFAO_UNIQUE_ID_BYTES bytes) with a fresh NCCL unique id; call on
 * rank 0 and broadcast it (the Python harness uses a torch.distributed
 * broadcast).  LMFAO_ERR_NCCL if NCCL cannot be loaded. */
LMFAO_API lmfao_status lmfao_unique_id(void* out);

/* Creates a context on CUDA device `device`.  world >= 1, 0 <= rank < world;
 * unique_id must be non-NULL iff world > 1 (collective call across ranks). */
LMFAO_API lmfao_status lmfao_create(int device, int rank, int world, const void* unique_id, lmfao_ctx** out);

/* Testing the multi-GPU path on one GPU: `world` contexts of ONE process on one device form
 * the in-process group named `group` (rank 0 .. world-1), each driven by its own host thread
 * (every call that is collective for NCCL ranks — prepare's sharding, plan, run,
 * gather_result — must be made by all of them).  The data path is the one of NCCL ranks —
 * sharded root, the same kernels, reduce-scatter / exchange / gather — with the collectives
 * done by device copies and the phases of a run separated by host barriers (no kernel waits
 * for another rank's kernel; no CUDA Graph).  Not for production. */
LMFAO_API lmfao_status lmfao_create_loopback(int device, int rank, int world, const char* group, lmfao_ctx** out);

/* Host-only (no device needed): the contiguous shard [lo, hi) of a root of nrows sorted rows
 * kept by `part` of `nparts` ([n·part/nparts, n·(part+1)/nparts)), and the range of cells
 * [lo, hi) of a distributed output with ncells cells owned by `rank` of `world` (equal chunks
 * of ceil(ncells / world) cells; the last ranks' may be short or empty). */
LMFAO_API lmfao_status lmfao_shard_range(int64_t nrows, int32_t part, int32_t nparts, int64_t* lo, int64_t* hi);
LMFAO_API lmfao_status lmfao_owner_range(int64_t ncells, int32_t rank, int32_t world, int64_t* lo, int64_t* hi);
LMFAO_API lmfao_status lmfao_destroy(lmfao_ctx* ctx);
LMFAO_API const char* lmfao_last_error(const lmfao_ctx* ctx);

/* Registers relation R(ω) (relations R_1..R_m over schemas ω_1..ω_m) as
 * SoA columns: cols[i] points to nrows values of dtypes[i].  cols_on_device:
 *   LMFAO_COLS_HOST   (0) host memory, copied before the call returns;
 *   LMFAO_COLS_DEVICE (1) device memory on this ctx's device, copied before return;
 *   LMFAO_COLS_HOST_DEFERRED (2) host memory (pinned for full speed) that the caller
 *       keeps valid and unchanged until lmfao_plan returns (or lmfao_prepare fails, or
 *       lmfao_destroy returns): prepare streams the columns in on a copy stream in the
 *       order it consumes them (dimension relations, then the root's foreign keys, then
 *       its other columns), so the host->device transfer overlaps the remap, the sort
 *       and the root permutation; prepare may return while the last columns are still in
 *       flight (plan's host work then overlaps them) and plan waits for them.
 * Attributes with the same name in different relations are the natural-join
 * attributes (X = ∪ω).  *rel_id receives the relation id. */
#define LMFAO_COLS_HOST 0
#define LMFAO_COLS_DEVICE 1
#define LMFAO_COLS_HOST_DEFERRED 2
LMFAO_API lmfao_status lmfao_add_relation(lmfao_ctx* ctx, const char* name, int64_t nrows, int32_t ncols,
                                const char* const* col_names, const lmfao_dtype* dtypes,
                                const void* const* cols, int cols_on_device, int32_t* rel_id);

/* Attribute id of a column name (ids are global over the schema X). */
LMFAO_API lmfao_status lmfao_attr_id(lmfao_ctx* ctx, const char* attr_name, int32_t* attr_id);

/* Registers the rooted join tree: n_edges = m-1 edges parent->child.
 * Validates: connected, acyclic, each relation has at most one parent, the
 * running-intersection property, and that every edge shares one to eight
 * attributes, of type int32 (a multi-attribute key such as Favorita's (date, store),
 * P:1408-1411, is matched as the tuple: a chain of pair dictionaries at prepare);
 * otherwise LMFAO_ERR_UNSUPPORTED / _TYPE. */
LMFAO_API lmfao_status lmfao_set_join_tree(lmfao_ctx* ctx, int32_t root_rel, int32_t n_edges,
                                 const int32_t* parent_rel, const int32_t* child_rel);

/* Simulated sharding for testing the multi-GPU partition on one device: keep
 * part `part` of `nparts` contiguous parts of the sorted root (default: rank of
 * world).  Must precede lmfao_prepare. */
LMFAO_API lmfao_status lmfao_set_root_shard(lmfao_ctx* ctx, int32_t part, int32_t nparts);

/* Load-time preprocessing, kernel (a) ("We sort S in this order";
 * P:42 "We sort the relations once"): dense remap of every join key (rank
 * among the child's distinct key values; dangling foreign keys drop the row,
 * inner-join semantics), sort of each child by its key, and one composite LSD
 * radix sort of the root by its foreign keys in increasing domain-size order
 * (the MOO attribute order). Then sharding (see above).  With deferred
 * host columns the work is stream-ordered behind their copies and may still be in
 * flight on return; lmfao_plan waits for the copies (host buffers released there). */
LMFAO_API lmfao_status lmfao_prepare(lmfao_ctx* ctx);

/* Adds Q(F; α_1..α_n) += R_1..R_m.  Multi-root ("each aggregate to its
 * own root"): a query whose group-by attributes the user's root cannot place (below a root
 * child, or mixing a child with a non-unique key with other relations) is computed at another
 * root of the same join tree — tried in the order of P:958's heuristic (the relations holding
 * the query's group-by attributes, by how many they hold, then by size) — inside this context
 * (a re-rooted copy of the relations, prepared once, run on its own stream concurrently with the
 * main root); results and query ids are the same as for any query.  Single GPU only (world 1).  groupby_attrs: int32 attributes
 * (LMFAO_ERR_TYPE otherwise) owned by the root or by children of the root; when a
 * child's join key is not unique in it (a root row joins several of its rows) all the
 * query's group-by attributes must belong to that child — the query is then finished
 * at the child ("each aggregate to its own root") — otherwise, and for
 * attributes deeper in the tree, LMFAO_ERR_UNSUPPORTED.  n_groupby may be 0.  Each
 * product's factors must name existing attributes (CONST: attr = -1).  The batch is
 * copied. */
LMFAO_API lmfao_status lmfao_add_query(lmfao_ctx* ctx, int32_t n_groupby, const int32_t* groupby_attrs,
                             int32_t n_udafs, const lmfao_udaf* udafs, int32_t* query_id);

/* Host planner (and the plans of the queries placed at other roots): pushes every product down the join tree, dedups
 * view slots across the batch (view merging), picks the kernels and
 * allocates all device buffers.  Freezes the batch. */
LMFAO_API lmfao_status lmfao_plan(lmfao_ctx* ctx);

/* Drops the batch and its plan (queries, selected kernels, results) but keeps the loaded and
 * prepared relations, so that another batch over the same data — the next node of a decision
 * tree, whose aggregates carry a different path condition — needs only
 * add_query + plan.  Valid after prepare (state PREPARED or PLANNED), returns to PREPARED;
 * query ids restart at 0.  LMFAO_ERR_STATE otherwise. */
LMFAO_API lmfao_status lmfao_reset_batch(lmfao_ctx* ctx);

/* Dynamic functions ("Dynamic Functions": a decision tree recomputes
 * the same aggregates at every node, the only difference being the node's threshold
 * functions).  Replaces the path condition of the planned batch — the Kronecker-delta factors
 * (LMFAO_F_LT .. LMFAO_F_IN) that every product of the batch carries, as planned — by
 * factors[0 .. n_factors), for the following runs, without re-planning: every result is then
 * that of the batch with the new condition in place of the old.  The attributes must belong to
 * the root or to a root child with a primary key; at most 8 factors.  Valid after lmfao_plan;
 * LMFAO_ERR_UNSUPPORTED when the planned kernels took no path condition (plan the batch with a
 * placeholder condition, e.g. y >= -inf, to make it dynamic).  Synchronises the ctx stream. */
LMFAO_API lmfao_status lmfao_set_condition(lmfao_ctx* ctx, int32_t n_factors, const lmfao_factor* factors);

/* Runs the planned batch asynchronously on `cuda_stream` (cudaStream_t; NULL =
 * the ctx's own stream): view builds (b), the fused root scan (c) with its FP64
 * Gram tiles (d) and histograms (e), dimension-side finishing, and when world > 1
 * the collectives (see "Multi-GPU").  No host synchronisation (sizes that depend on
 * the data stay on the device; compaction of dense tables happens at the first
 * result_shape / fetch); the second run of a plan is captured in a CUDA Graph
 * (NCCL collectives included) and later runs replay it.  LMFAO_ERR_NCCL if the
 * communicator reported an asynchronous error. */
LMFAO_API lmfao_status lmfao_run(lmfao_ctx* ctx, void* cuda_stream);

/* Result shape of query_id after the last run (synchronises the stream). */
LMFAO_API lmfao_status lmfao_result_shape(lmfao_ctx* ctx, int32_t query_id, int64_t* n_groups,
                                int32_t* n_groupby, int32_t* n_udafs);

/* Copies query_id's result to caller-owned HOST buffers (synchronises):
 * keys_out [n_groups x n_groupby] int32 row-major (may be NULL if n_groupby = 0),
 * vals_out [n_groups x n_udafs] double row-major, counts_out [n_groups] uint64
 * join multiplicity of each group (nullable). Groups in ascending key order. */
LMFAO_API lmfao_status lmfao_fetch(lmfao_ctx* ctx, int32_t query_id, int32_t* keys_out, double* vals_out,
                         uint64_t* counts_out);

/* Collective (every rank calls it, world > 1): assembles a distributed result (see
 * "Multi-GPU" above) on root_rank — the ranks' groups in rank order, which is the canonical
 * ascending key order since the ranges ascend with the rank; afterwards result_shape / fetch /
 * result_device on root_rank return the whole table (until the next run), the other ranks keep
 * their own range.  Synchronises.  A no-op for results complete on every rank (scalar queries,
 * all-reduced tables) and for world == 1.  LMFAO_ERR_NCCL if a transfer fails. */
LMFAO_API lmfao_status lmfao_gather_result(lmfao_ctx* ctx, int32_t query_id, int32_t root_rank);

/* Library-owned device views of query_id's result (same layout as fetch). */
LMFAO_API lmfao_status lmfao_result_device(lmfao_ctx* ctx, int32_t query_id, const int32_t** keys,
                                 const double** vals, const uint64_t** counts);

/* Diagnostics: fills `out` (up to `cap` bytes) with a JSON object describing
 * the plan (kernel path per query group, view widths, run counts per level after
 * the last run, kernel launches per run; with world > 1, after profiled runs
 * (lmfao_profile + lmfao_profile_read): "collective_ms", the mean device time of
 * a run's NCCL all-reduce of the partial results, and "collective_bytes", the
 * bytes it reduces per rank). */
LMFAO_API lmfao_status lmfao_plan_info(lmfao_ctx* ctx, char* out, int64_t cap);

/* Measurement: when enabled, lmfao_run records CUDA events on its stream around
 * the dominant root-scan kernel (kernel (c)); lmfao_profile_read synchronises
 * and returns the summed device time and the number of timed launches since
 * the last lmfao_profile call. */
LMFAO_API lmfao_status lmfao_profile(lmfao_ctx* ctx, int enable);
LMFAO_API lmfao_status lmfao_profile_read(lmfao_ctx* ctx, double* total_ms, int64_t* launches);

#ifdef __cplusplus
}
#endif
#endif /* LMFAO_GPU_H */
