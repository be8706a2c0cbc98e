// ctx.h — the context behind the opaque lmfao_ctx handle (private).
#pragma once
#include <tuple>

#include "comm.h"
#include "internal.h"
#include "paths.h"

namespace lmfao {

enum State { S_CREATED = 0, S_TREE, S_PREPARED, S_PLANNED };

struct Column {
  std::string name;
  int attr = -1;
  lmfao_dtype dt = LMFAO_INT32;
  DevBuf buf;
  const void* host_src = nullptr;  // LMFAO_COLS_HOST_DEFERRED: copied in by prepare
  cudaEvent_t ready = nullptr;     // copy-stream event the column's consumers wait on
};

struct Rel {
  std::string name;
  int64_t nrows = 0;
  std::vector<Column> cols;
  int parent = -1;
  std::vector<int> children;
  int key_attr = -1, key_col = -1;
  int key_attr2 = -1, key_col2 = -1;  // second attribute of a two-attribute join key (-1: one attribute)
  std::vector<int> fk_col;   // per child: column of this relation holding the child's key
  std::vector<int> fk_col2;  // per child: the second key column (-1: one attribute)
  // keys of more than two attributes: the third and later key columns (as a child), and per
  // child the matching foreign-key columns; the key is dictionary-encoded pairwise in a chain,
  // (a0, a1) -> c1, (c1, a2) -> c2, ..., each code the rank of its prefix tuple, so the last
  // code is the rank of the whole tuple (lexicographic)
  std::vector<int> key_cols_more;
  std::vector<std::vector<int>> fk_cols_more;
  std::vector<DevBuf> kdict;     // the chain's pair dictionaries (u64 images), first pair first
  std::vector<int64_t> kdn;
  // prepared
  int64_t nkeys = 0;
  DevBuf dict;       // sorted distinct key values [nkeys] (int32; u64 pair images for two-attribute keys)
  DevBuf dense_key;  // dense key id per row (rows sorted by it)
  bool unique_key = false;
  std::vector<DevBuf> fk_dense;  // per child: dense id of the child key per row
  // root only, sharded runs: dictionaries of every int32 column over the WHOLE root
  // (before slicing), so group-by cells mean the same on every rank
  std::map<int, DevBuf> full_dict;
  std::map<int, int64_t> full_dict_n;
  int find_attr(int a) const {
    for (size_t i = 0; i < cols.size(); i++)
      if (cols[i].attr == a) return (int)i;
    return -1;
  }
};

struct Attr {
  std::string name;
  lmfao_dtype dt;
  std::vector<std::pair<int, int>> occ;  // (relation, column)
};

struct QFactor {
  int kind, attr;
  double param;
};
struct QProduct {
  double coeff;
  std::vector<QFactor> f;
};
struct Query {
  std::vector<int> gb;
  std::vector<std::vector<QProduct>> udafs;
};

inline uint64_t dbits(double d) {
  uint64_t u;
  std::memcpy(&u, &d, 8);
  return u;
}

struct SlotKey {
  std::vector<std::tuple<int, int, uint64_t>> own;  // (kind, attr, param bits), sorted
  std::vector<int> child_slots;
  bool operator<(const SlotKey& o) const { return std::tie(own, child_slots) < std::tie(o.own, o.child_slots); }
};

struct DevProgram {
  DevBuf pi, pd, pio, pdo;
  int nout = 0;
  cudaError_t upload(const Program& p, cudaStream_t st) {
    nout = (int)p.out_ioff.size();
    CUDA_TRY(pi.alloc(std::max<size_t>(p.ip.size(), 1) * 4));
    CUDA_TRY(pd.alloc(std::max<size_t>(p.dp.size(), 1) * 8));
    CUDA_TRY(pio.alloc(std::max<size_t>(p.out_ioff.size(), 1) * 4));
    CUDA_TRY(pdo.alloc(std::max<size_t>(p.out_doff.size(), 1) * 4));
    if (!p.ip.empty()) CUDA_TRY(cudaMemcpyAsync(pi.p, p.ip.data(), p.ip.size() * 4, cudaMemcpyHostToDevice, st));
    if (!p.dp.empty()) CUDA_TRY(cudaMemcpyAsync(pd.p, p.dp.data(), p.dp.size() * 8, cudaMemcpyHostToDevice, st));
    if (nout) {
      CUDA_TRY(cudaMemcpyAsync(pio.p, p.out_ioff.data(), nout * 4, cudaMemcpyHostToDevice, st));
      CUDA_TRY(cudaMemcpyAsync(pdo.p, p.out_doff.data(), nout * 4, cudaMemcpyHostToDevice, st));
    }
    return cudaStreamSynchronize(st);
  }
};

struct NodePlan {
  std::vector<SlotKey> slots;
  std::map<SlotKey, int> index;
  DevBuf V;
  DevProgram prog;
  bool linear = false;  // leaf with identity-only slots: k_view_lin
  ViewLinArgs lin{};
};

// Dictionary (sorted distinct values) and per-row (root) or per-dense-key (child) codes of a
// group-by attribute; shared by every query that groups by the attribute.
struct CodeSet {
  DevBuf dict, codes;
  int64_t nd = 0;
};

struct GroupPlan {
  int q = -1;
  int nudaf = 0;
  int64_t ncells = 0;
  GroupArgs g{};
  DecodeArgs d{};
  std::vector<std::shared_ptr<CodeSet>> sets;
  DevBuf table, counts;
  DevProgram prog;
  bool compacted = false;
  bool direct = false;  // a fast path writes rkeys/rvals/rcnts/ngroups itself at run (no dense table)
  DevBuf rkeys, rvals, rcnts;
  DevBuf countcoef;
  int64_t ngroups = 0;
  DevBuf ngroups_dev;              // direct outputs: the group count, written on the device
  bool ngroups_on_device = false;
  // world > 1: a distributed output — dense tables reduce-scattered (each rank keeps the sums of
  // its own range of cells), sparse cuboids exchanged by cell owner — holds only [cell_lo,
  // cell_hi) on this rank until lmfao_gather_result assembles it on one rank
  bool dist = false;
  int64_t ncells_alloc = 0;        // cells of the dense table (a multiple of world when dist)
  int64_t cell_lo = 0, cell_hi = 0;
  bool gathered = false;
  DevBuf gkeys, gvals, gcnts;      // the gathered full table (gather_result's root)
  int64_t gngroups = 0;
  int rev = -1;  // index into lmfao_ctx::revs: finished at a non-unique-keyed root child
};

// A group-by query over the attributes of a root child T with a non-unique key (generic.cu
// k_rev_root / k_rev_child): per product, its root side summed per key of T, then its T side.
struct RevPlan {
  int gi = -1, j = -1, T = -1;  // group, index of T among the root's children, relation
  DevProgram rp, tp;            // one output per product + the count term
  DevBuf pu;                    // product -> UDAF
  DevBuf A;                     // [keys of T][products + 1]
  GroupDesc d{};
};

}  // namespace lmfao

using namespace lmfao;
struct lmfao_ctx {
  int device = 0, rank = 0, world = 1;
  int shard_part = 0, shard_nparts = 1;
  cudaStream_t stream = nullptr;
  cudaStream_t copy_stream = nullptr;  // deferred host->device column copies (prepare)
  bool copies_pending = false;          // ... possibly in flight until plan (copies_wait)
  std::unique_ptr<Comm> comm;  // world > 1: NCCL, or an in-process loopback group (tests)
  int64_t root_rows_global = 0;  // the root's rows before sharding
  std::string err;
  State state = S_CREATED;
  std::vector<Rel> rels;
  std::vector<Attr> attrs;
  std::map<std::string, int> attr_by_name;
  int root = -1;
  std::vector<Query> queries;
  // plan
  std::vector<int> owner;      // per attr: top-most relation holding it
  std::vector<NodePlan> nodes;  // per relation (non-root used)
  std::vector<int> postorder;   // non-root nodes, children first
  std::vector<int> levels;      // root children in increasing domain size (the sort order)
  // scalar (no group-by) queries: one fused program over all their outputs
  std::vector<int> scalar_queries;
  std::vector<int> scalar_off;  // output offset per query (index into out)
  DevProgram scalar_prog;
  DevBuf partials, cpart, scalar_out, scalar_count;
  int scalar_grid = 0;
  std::vector<GroupPlan> groups;
  std::vector<RevPlan> revs;
  int ndescs = 0;  // group-by queries of the fused generic scan
  std::map<int, std::shared_ptr<CodeSet>> code_cache;  // per group-by attribute
  DevProgram group_prog;  // all group-by UDAFs (fused scan)
  DevBuf group_descs;     // GroupDesc per group-by query
  std::vector<int> query_kind;  // 0 scalar, 1 group (index into groups)
  std::vector<int> query_slot;
  std::unique_ptr<FastPaths> fast;  // specialised kernels (gram / hist), if the batch matches
  bool ran = false;
  int64_t launches_last_run = 0;
  // optional timer around the dominant root-scan kernel (lmfao_profile)
  bool prof = false;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> prof_events;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> coll_events;  // multi-GPU all-reduce (profiled runs)
  double coll_ms = 0.0;
  int64_t coll_n = 0;
  std::string prof_kernel;
  // CUDA Graph of lmfao_run (see abi.cpp)
  cudaGraphExec_t graph_exec = nullptr;
  int64_t graph_runs = 0, graph_launches = 0;
  // Multi-root plans (§4.3 "each aggregate to its own root"): a query the
  // user's root cannot place is computed at another root — a secondary context over the same
  // relations (device copies), its join tree re-rooted, prepared for that root — and its run
  // overlaps the main one on its own stream (task parallelism).
  struct Secondary {
    lmfao_ctx* ctx = nullptr;
    int root = -1;
    cudaStream_t stream = nullptr;
    cudaEvent_t ev_in = nullptr, ev_out = nullptr;
  };
  std::vector<Secondary> secs;
  std::vector<std::pair<int, int>> qmap;  // public query id -> (secondary index or -1, its local id)
  bool is_secondary = false;
  ~lmfao_ctx();
};

namespace lmfao {
void scan_timer_begin(lmfao_ctx* c, cudaStream_t st);
void scan_timer_end(lmfao_ctx* c, cudaStream_t st);
}

