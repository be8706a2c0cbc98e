// abi.cpp — the C ABI of liblmfao_gpu (include/lmfao_gpu.h): context, schema and
// join-tree validation, load-time preprocessing (kernel (a)), the host planner
// and the run orchestration.
//
// Planner (§4): every product term of the batch is pushed down the join
// tree (aggregate pushdown: a view V_{C->S}(F_i; α_i) per child with
// α_i the part of the product over the child's subtree); identical partial
// products share one slot of the child's view (view merging cases (2)/(3),
// P:961-1000); slot 0 of every view is the count, so multiplicities carry bag
// semantics.  All queries are computed at one root (the user's), whose sorted
// scan is the single shared pass over the largest relation (MOO).
#include <cmath>
#include <cstdarg>
#include <cstdlib>
#include <cstdio>
#include <functional>
#include <set>
#include <sstream>
#include <tuple>

#include "comm.h"
#include "ctx.h"

using namespace lmfao;

namespace {

lmfao_status fail(lmfao_ctx* c, lmfao_status s, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  std::vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (c) c->err = buf;
  return s;
}

lmfao_status cuda_fail(lmfao_ctx* c, cudaError_t e, const char* where) {
  if (e == cudaErrorMemoryAllocation) return fail(c, LMFAO_ERR_OOM, "%s: out of device memory", where);
  return fail(c, LMFAO_ERR_CUDA, "%s: CUDA error %s", where, cudaGetErrorString(e));
}

#define CTX_CUDA(c, x, where)                          \
  do {                                                 \
    cudaError_t e_ = (x);                              \
    if (e_ != cudaSuccess) return cuda_fail(c, e_, where); \
  } while (0)

// gather every column of relation r (and its fk_dense / dense_key) by `perm` of length n;
// all gathers are queued, then one synchronisation releases the old buffers
// Orders stream st after the deferred host->device copy of column col (if any).
cudaError_t column_ready(Column& col, cudaStream_t st) {
  if (!col.ready) return cudaSuccess;
  CUDA_TRY(cudaStreamWaitEvent(st, col.ready, 0));
  cudaEventDestroy(col.ready);  // the wait above is already enqueued
  col.ready = nullptr;
  return cudaSuccess;
}

// Pooled buffers are freed in stream order, so replaced buffers need no synchronisation.
cudaError_t permute_rel(Rel& r, const uint32_t* perm, int64_t n, cudaStream_t st) {
  std::vector<DevBuf> old;
  bool sync = false;
  auto regather = [&](DevBuf& b, int es) -> cudaError_t {
    DevBuf nb;
    CUDA_TRY(nb.alloc(std::max<int64_t>(n, 1) * es));
    CUDA_TRY(gather_bytes(b.p, perm, nb.p, n, es, st));
    sync |= !b.pooled || !nb.pooled || b.st != st;
    old.push_back(std::move(b));
    b = std::move(nb);
    return cudaSuccess;
  };
  for (auto& c : r.cols) {
    CUDA_TRY(column_ready(c, st));
    CUDA_TRY(regather(c.buf, c.dt == LMFAO_FP64 ? 8 : 4));
  }
  for (auto& f : r.fk_dense) CUDA_TRY(regather(f, 4));
  if (r.dense_key.p) CUDA_TRY(regather(r.dense_key, 4));
  if (sync) CUDA_TRY(cudaStreamSynchronize(st));
  r.nrows = n;
  return cudaSuccess;
}

cudaError_t slice_rel(Rel& r, int64_t lo, int64_t hi, cudaStream_t st) {
  int64_t n = hi - lo;
  std::vector<DevBuf> old;
  auto cut = [&](DevBuf& b, int es) -> cudaError_t {
    DevBuf nb;
    CUDA_TRY(nb.alloc(std::max<int64_t>(n, 1) * es));
    if (n > 0) CUDA_TRY(cudaMemcpyAsync(nb.p, (char*)b.p + lo * es, n * es, cudaMemcpyDeviceToDevice, st));
    old.push_back(std::move(b));
    b = std::move(nb);
    return cudaSuccess;
  };
  for (auto& c : r.cols) {
    CUDA_TRY(column_ready(c, st));
    CUDA_TRY(cut(c.buf, c.dt == LMFAO_FP64 ? 8 : 4));
  }
  for (auto& f : r.fk_dense) CUDA_TRY(cut(f, 4));
  CUDA_TRY(cudaStreamSynchronize(st));
  r.nrows = n;
  return cudaSuccess;
}

NodeArgs node_args(const lmfao_ctx* c, int n) {
  const Rel& r = c->rels[n];
  NodeArgs a{};
  a.nrows = r.nrows;
  for (size_t i = 0; i < r.cols.size() && i < (size_t)MAX_COLS; i++) {
    a.cols[i] = r.cols[i].buf.p;
    a.col_is_int[i] = r.cols[i].dt == LMFAO_INT32;
  }
  a.nchild = (int)r.children.size();
  for (int j = 0; j < a.nchild; j++) {
    int ch = r.children[j];
    a.fk[j] = r.fk_dense[j].as<int32_t>();
    a.V[j] = c->nodes[ch].V.as<double>();
    a.W[j] = (int)c->nodes[ch].slots.size();
  }
  return a;
}

}  // namespace

namespace {
lmfao_status relay(lmfao_ctx* c, lmfao_ctx* t, lmfao_status s);
}

lmfao_ctx::~lmfao_ctx() {
  if (graph_exec) cudaGraphExecDestroy(graph_exec);
}

// =====================================================================  ABI
extern "C" {

lmfao_status lmfao_unique_id(void* out) {
  if (!out) return LMFAO_ERR_INVALID_ARG;
  if (!nccl_available()) return LMFAO_ERR_NCCL;
  return nccl_unique_id(out) == 0 ? LMFAO_OK : LMFAO_ERR_NCCL;
}

lmfao_status lmfao_destroy(lmfao_ctx* c);

lmfao_status lmfao_create(int device, int rank, int world, const void* unique_id, lmfao_ctx** out) {
  if (!out || world < 1 || rank < 0 || rank >= world) return LMFAO_ERR_INVALID_ARG;
  if ((world > 1) != (unique_id != nullptr)) return LMFAO_ERR_INVALID_ARG;
  *out = nullptr;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return LMFAO_ERR_CUDA;
  if (device < 0 || device >= ndev) return LMFAO_ERR_INVALID_ARG;
  if (cudaSetDevice(device) != cudaSuccess) return LMFAO_ERR_CUDA;
  auto* c = new lmfao_ctx();
  c->device = device;
  c->rank = rank;
  c->world = world;
  c->shard_part = rank;
  c->shard_nparts = world;
  static bool pool_ready[64] = {};
  if (device < 64 && !pool_ready[device]) {  // keep freed blocks cached in the device pool
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    pool_ready[device] = true;
  }
  if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess) {
    delete c;
    return LMFAO_ERR_CUDA;
  }
  if (world > 1) {
    int e = 0;
    c->comm.reset(make_nccl_comm(rank, world, unique_id, e));
    if (!c->comm) {
      cudaStreamDestroy(c->stream);
      delete c;
      return LMFAO_ERR_NCCL;
    }
  }
  *out = c;
  return LMFAO_OK;
}

lmfao_status lmfao_create_loopback(int device, int rank, int world, const char* group, lmfao_ctx** out) {
  if (!out || !group || world < 1 || rank < 0 || rank >= world) return LMFAO_ERR_INVALID_ARG;
  *out = nullptr;
  lmfao_status s = lmfao_create(device, 0, 1, nullptr, out);
  if (s != LMFAO_OK) return s;
  lmfao_ctx* c = *out;
  c->rank = rank;
  c->world = world;
  c->shard_part = rank;
  c->shard_nparts = world;
  if (world > 1) {
    c->comm.reset(make_loopback_comm(group, rank, world, device));
    if (!c->comm) {
      lmfao_destroy(c);
      *out = nullptr;
      return LMFAO_ERR_INVALID_ARG;
    }
  }
  return LMFAO_OK;
}

lmfao_status lmfao_shard_range(int64_t nrows, int32_t part, int32_t nparts, int64_t* lo, int64_t* hi) {
  if (nrows < 0 || nparts < 1 || part < 0 || part >= nparts || !lo || !hi) return LMFAO_ERR_INVALID_ARG;
  shard_range(nrows, part, nparts, *lo, *hi);
  return LMFAO_OK;
}

lmfao_status lmfao_owner_range(int64_t ncells, int32_t rank, int32_t world, int64_t* lo, int64_t* hi) {
  if (ncells < 0 || world < 1 || rank < 0 || rank >= world || !lo || !hi) return LMFAO_ERR_INVALID_ARG;
  owner_range(ncells, rank, world, *lo, *hi);
  return LMFAO_OK;
}

lmfao_status lmfao_destroy(lmfao_ctx* c) {
  if (!c) return LMFAO_ERR_INVALID_ARG;
  for (auto& sc : c->secs) {
    if (sc.ctx) lmfao_destroy(sc.ctx);
    cudaSetDevice(c->device);
    if (sc.ev_in) cudaEventDestroy(sc.ev_in);
    if (sc.ev_out) cudaEventDestroy(sc.ev_out);
    if (sc.stream) cudaStreamDestroy(sc.stream);
  }
  c->secs.clear();
  cudaSetDevice(c->device);
  StreamScope scope_(c->stream);
  cudaStreamSynchronize(c->stream);
  c->fast.reset();  // peer mappings before the communicator
  c->comm.reset();
  cudaStream_t st = c->stream;
  if (c->copy_stream) {
    cudaStreamSynchronize(c->copy_stream);
    cudaStreamDestroy(c->copy_stream);
  }
  for (auto& r : c->rels)
    for (auto& col : r.cols)
      if (col.ready) cudaEventDestroy(col.ready);
  delete c;
  cudaStreamDestroy(st);
  return LMFAO_OK;
}

const char* lmfao_last_error(const lmfao_ctx* c) { return c ? c->err.c_str() : "null context"; }

lmfao_status lmfao_add_relation(lmfao_ctx* c, const char* name, int64_t nrows, int32_t ncols,
                                const char* const* col_names, const lmfao_dtype* dtypes, const void* const* cols,
                                int cols_on_device, int32_t* rel_id) {
  if (!c) return LMFAO_ERR_INVALID_ARG;
  if (c->state != S_CREATED) return fail(c, LMFAO_ERR_STATE, "add_relation after set_join_tree");
  if (!name || nrows < 0 || ncols < 1 || !col_names || !dtypes || (!cols && nrows > 0) || cols_on_device < 0 ||
      cols_on_device > LMFAO_COLS_HOST_DEFERRED)
    return fail(c, LMFAO_ERR_INVALID_ARG, "add_relation: bad arguments");
  if (ncols > MAX_COLS) return fail(c, LMFAO_ERR_UNSUPPORTED, "add_relation: more than %d columns", MAX_COLS);
  for (auto& r : c->rels)
    if (r.name == name) return fail(c, LMFAO_ERR_INVALID_ARG, "duplicate relation %s", name);
  cudaSetDevice(c->device);
  StreamScope scope_(c->stream);
  Rel r;
  r.name = name;
  r.nrows = nrows;
  int rid = (int)c->rels.size();
  std::set<std::string> seen;
  for (int i = 0; i < ncols; i++) {
    if (!col_names[i] || (dtypes[i] != LMFAO_INT32 && dtypes[i] != LMFAO_FP64))
      return fail(c, LMFAO_ERR_INVALID_ARG, "add_relation: bad column %d", i);
    if (!seen.insert(col_names[i]).second)
      return fail(c, LMFAO_ERR_INVALID_ARG, "duplicate column %s in %s", col_names[i], name);
    auto it = c->attr_by_name.find(col_names[i]);
    if (it != c->attr_by_name.end() && c->attrs[it->second].dt != dtypes[i])
      return fail(c, LMFAO_ERR_TYPE, "attribute %s has conflicting dtypes", col_names[i]);
  }
  for (int i = 0; i < ncols; i++) {
    Column col;
    col.name = col_names[i];
    col.dt = dtypes[i];
    size_t es = col.dt == LMFAO_FP64 ? 8 : 4;
    CTX_CUDA(c, col.buf.alloc(std::max<int64_t>(nrows, 1) * es), "add_relation");
    if (nrows > 0) {
      if (!cols[i]) return fail(c, LMFAO_ERR_INVALID_ARG, "add_relation: null column %d", i);
      if (cols_on_device == LMFAO_COLS_HOST_DEFERRED)
        col.host_src = cols[i];
      else
        CTX_CUDA(c, cudaMemcpyAsync(col.buf.p, cols[i], nrows * es,
                                    cols_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, c->stream),
                 "add_relation copy");
    }
    auto it = c->attr_by_name.find(col.name);
    int aid;
    if (it == c->attr_by_name.end()) {
      aid = (int)c->attrs.size();
      c->attrs.push_back(Attr{col.name, col.dt, {}});
      c->attr_by_name[col.name] = aid;
    } else {
      aid = it->second;
    }
    c->attrs[aid].occ.push_back({rid, i});
    col.attr = aid;
    r.cols.push_back(std::move(col));
  }
  // the caller may release its buffers on return
  CTX_CUDA(c, cudaStreamSynchronize(c->stream), "add_relation copy");
  c->rels.push_back(std::move(r));
  if (rel_id) *rel_id = rid;
  return LMFAO_OK;
}

lmfao_status lmfao_attr_id(lmfao_ctx* c, const char* attr_name, int32_t* attr_id) {
  if (!c || !attr_name || !attr_id) return LMFAO_ERR_INVALID_ARG;
  auto it = c->attr_by_name.find(attr_name);
  if (it == c->attr_by_name.end()) return fail(c, LMFAO_ERR_UNKNOWN_ATTR, "unknown attribute %s", attr_name);
  *attr_id = it->second;
  return LMFAO_OK;
}

lmfao_status lmfao_set_join_tree(lmfao_ctx* c, int32_t root_rel, int32_t n_edges, const int32_t* parent_rel,
                                 const int32_t* child_rel) {
  if (!c) return LMFAO_ERR_INVALID_ARG;
  if (c->state != S_CREATED) return fail(c, LMFAO_ERR_STATE, "set_join_tree called twice or out of order");
  int m = (int)c->rels.size();
  if (m == 0) return fail(c, LMFAO_ERR_STATE, "no relations");
  if (root_rel < 0 || root_rel >= m) return fail(c, LMFAO_ERR_UNKNOWN_ATTR, "bad root relation id");
  if (n_edges < 0 || (n_edges > 0 && (!parent_rel || !child_rel))) return fail(c, LMFAO_ERR_INVALID_ARG, "bad edges");
  for (int e = 0; e < n_edges; e++)
    if (parent_rel[e] < 0 || parent_rel[e] >= m || child_rel[e] < 0 || child_rel[e] >= m || parent_rel[e] == child_rel[e])
      return fail(c, LMFAO_ERR_UNKNOWN_ATTR, "edge %d names an unknown relation", e);
  if (n_edges > m - 1) return fail(c, LMFAO_ERR_CYCLIC_TREE, "%d edges for %d relations: cycle", n_edges, m);
  std::vector<int> parent(m, -1);
  std::vector<std::vector<int>> children(m);
  for (int e = 0; e < n_edges; e++) {
    int p = parent_rel[e], ch = child_rel[e];
    if (parent[ch] != -1 || ch == root_rel)
      return fail(c, LMFAO_ERR_CYCLIC_TREE, "relation %s has two parents (cycle)", c->rels[ch].name.c_str());
    parent[ch] = p;
    children[p].push_back(ch);
  }
  // reachability from the root
  std::vector<int> seen(m, 0), stack{root_rel};
  int reached = 0;
  while (!stack.empty()) {
    int u = stack.back();
    stack.pop_back();
    if (seen[u]) return fail(c, LMFAO_ERR_CYCLIC_TREE, "cycle through %s", c->rels[u].name.c_str());
    seen[u] = 1;
    reached++;
    for (int v : children[u]) stack.push_back(v);
  }
  if (reached != m) {
    if (n_edges == m - 1) return fail(c, LMFAO_ERR_CYCLIC_TREE, "edges form a cycle disconnected from the root");
    return fail(c, LMFAO_ERR_DISCONNECTED_TREE, "join tree does not reach every relation");
  }
  // running intersection: for every pair sharing an attribute, every
  // relation on the path between them holds it.
  auto path = [&](int a, int b) {
    std::vector<int> pa, pb;
    for (int u = a; u != -1; u = parent[u]) pa.push_back(u);
    for (int u = b; u != -1; u = parent[u]) pb.push_back(u);
    std::set<int> sa(pa.begin(), pa.end());
    int lca = -1;
    for (int u : pb)
      if (sa.count(u)) { lca = u; break; }
    std::vector<int> p;
    for (int u = a; u != lca; u = parent[u]) p.push_back(u);
    for (int u = b; u != lca; u = parent[u]) p.push_back(u);
    p.push_back(lca);
    return p;
  };
  for (auto& at : c->attrs) {
    for (size_t i = 0; i < at.occ.size(); i++)
      for (size_t j = i + 1; j < at.occ.size(); j++) {
        for (int u : path(at.occ[i].first, at.occ[j].first)) {
          bool has = false;
          for (auto& o : at.occ) has |= o.first == u;
          if (!has)
            return fail(c, LMFAO_ERR_RUNNING_INTERSECTION,
                        "running intersection violated: %s shared by %s and %s is missing from %s", at.name.c_str(),
                        c->rels[at.occ[i].first].name.c_str(), c->rels[at.occ[j].first].name.c_str(),
                        c->rels[u].name.c_str());
        }
      }
  }
  // one or two int32 join attributes per edge (a two-attribute key — Favorita's (date, store),
  // is matched as the pair)
  for (int ch = 0; ch < m; ch++) {
    if (parent[ch] < 0) continue;
    Rel& C = c->rels[ch];
    Rel& P = c->rels[parent[ch]];
    std::vector<int> keys;
    for (auto& col : C.cols)
      if (P.find_attr(col.attr) >= 0) keys.push_back(col.attr);
    std::sort(keys.begin(), keys.end());
    if (keys.empty() || keys.size() > 8)
      return fail(c, LMFAO_ERR_UNSUPPORTED, "edge %s-%s shares %zu attributes (one to eight supported)",
                  P.name.c_str(), C.name.c_str(), keys.size());
    for (int key : keys)
      if (c->attrs[key].dt != LMFAO_INT32)
        return fail(c, LMFAO_ERR_TYPE, "join attribute %s must be int32", c->attrs[key].name.c_str());
    C.key_attr = keys[0];
    C.key_col = C.find_attr(keys[0]);
    C.key_attr2 = keys.size() > 1 ? keys[1] : -1;
    C.key_col2 = keys.size() > 1 ? C.find_attr(keys[1]) : -1;
    C.key_cols_more.clear();
    for (size_t i = 2; i < keys.size(); i++) C.key_cols_more.push_back(C.find_attr(keys[i]));
  }
  for (int u = 0; u < m; u++) {
    c->rels[u].parent = parent[u];
    c->rels[u].children = children[u];
    c->rels[u].fk_col.clear();
    c->rels[u].fk_col2.clear();
    c->rels[u].fk_cols_more.clear();
    for (int ch : children[u]) {
      c->rels[u].fk_col.push_back(c->rels[u].find_attr(c->rels[ch].key_attr));
      c->rels[u].fk_col2.push_back(c->rels[ch].key_attr2 >= 0 ? c->rels[u].find_attr(c->rels[ch].key_attr2) : -1);
      std::vector<int> more;
      for (int kc : c->rels[ch].key_cols_more) more.push_back(c->rels[u].find_attr(c->rels[ch].cols[kc].attr));
      c->rels[u].fk_cols_more.push_back(more);
    }
  }
  c->root = root_rel;
  c->state = S_TREE;
  return LMFAO_OK;
}

lmfao_status lmfao_set_root_shard(lmfao_ctx* c, int32_t part, int32_t nparts) {
  if (!c || nparts < 1 || part < 0 || part >= nparts) return LMFAO_ERR_INVALID_ARG;
  if (c->state >= S_PREPARED) return fail(c, LMFAO_ERR_STATE, "set_root_shard after prepare");
  c->shard_part = part;
  c->shard_nparts = nparts;
  return LMFAO_OK;
}

// Deferred host columns (LMFAO_COLS_HOST_DEFERRED) stay the caller's until this returns: the
// copies prepare issued may still be in flight when prepare returns (the root's non-key
// columns arrive last), so plan's host work overlaps the transfer; plan (whatever its
// outcome), a failed prepare, secondary-root creation and destroy wait for them here.
void copies_wait(lmfao_ctx* c) {
  if (c->copy_stream && c->copies_pending) cudaStreamSynchronize(c->copy_stream);
  c->copies_pending = false;
}
lmfao_status prepare_impl(lmfao_ctx* c);
lmfao_status lmfao_prepare(lmfao_ctx* c) {
  if (!c) return LMFAO_ERR_INVALID_ARG;
  const lmfao_status s = prepare_impl(c);
  if (s != LMFAO_OK) copies_wait(c);
  return s;
}
lmfao_status prepare_impl(lmfao_ctx* c) {
  if (c->state != S_TREE) return fail(c, LMFAO_ERR_STATE, "prepare needs a join tree (and runs once)");
  cudaSetDevice(c->device);
  StreamScope scope_(c->stream);
  cudaStream_t st = c->stream;
  PhaseTrace tr("prepare");
  // post-order: children before parents
  std::vector<int> post;
  std::function<void(int)> dfs = [&](int u) {
    for (int v : c->rels[u].children) dfs(v);
    post.push_back(u);
  };
  dfs(c->root);
  {  // deferred host columns: stream them in in the order they are consumed below
    std::vector<std::pair<const Rel*, Column*>> order;
    for (int u : post) {
      Rel& r = c->rels[u];
      for (int j : r.fk_col) order.push_back({&r, &r.cols[j]});
      for (int j : r.fk_col2)
        if (j >= 0) order.push_back({&r, &r.cols[j]});
      for (auto& more : r.fk_cols_more)
        for (int j : more) order.push_back({&r, &r.cols[j]});
      if (r.key_col >= 0) order.push_back({&r, &r.cols[r.key_col]});
      if (r.key_col2 >= 0) order.push_back({&r, &r.cols[r.key_col2]});
      for (int j : r.key_cols_more) order.push_back({&r, &r.cols[j]});
    }
    for (int u : post)
      for (auto& col : c->rels[u].cols) order.push_back({&c->rels[u], &col});
    bool first = true;
    for (auto& rc : order) {
      Column* col = rc.second;
      if (!col->host_src) continue;
      if (first) {  // the column buffers were allocated on the ctx stream: copy after that
        first = false;
        if (!c->copy_stream) CTX_CUDA(c, cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking), "prepare");
        cudaEvent_t alloc_done;
        CTX_CUDA(c, cudaEventCreateWithFlags(&alloc_done, cudaEventDisableTiming), "prepare");
        CTX_CUDA(c, cudaEventRecord(alloc_done, st), "prepare");
        CTX_CUDA(c, cudaStreamWaitEvent(c->copy_stream, alloc_done, 0), "prepare");
        cudaEventDestroy(alloc_done);
      }
      size_t es = col->dt == LMFAO_FP64 ? 8 : 4;
      CTX_CUDA(c, cudaMemcpyAsync(col->buf.p, col->host_src, rc.first->nrows * es, cudaMemcpyHostToDevice,
                                  c->copy_stream),
               "prepare copy");
      col->host_src = nullptr;
      CTX_CUDA(c, cudaEventCreateWithFlags(&col->ready, cudaEventDisableTiming), "prepare");
      CTX_CUDA(c, cudaEventRecord(col->ready, c->copy_stream), "prepare");
    }
  }
  for (int u : post) {
    Rel& r = c->rels[u];
    // (1) dense remap of each child key: binary search in the child's dictionary
    r.fk_dense.clear();
    for (size_t j = 0; j < r.children.size(); j++) {
      Rel& ch = c->rels[r.children[j]];
      CTX_CUDA(c, column_ready(r.cols[r.fk_col[j]], st), "prepare copy");
      DevBuf d;
      CTX_CUDA(c, d.alloc(std::max<int64_t>(r.nrows, 1) * 4), "prepare");
      if (!ch.key_cols_more.empty()) {  // a key of three or more attributes: the chain of pair lookups
        CTX_CUDA(c, column_ready(r.cols[r.fk_col2[j]], st), "prepare copy");
        DevBuf t;
        CTX_CUDA(c, t.alloc(std::max<int64_t>(r.nrows, 1) * 4), "prepare");
        CTX_CUDA(c, lookup_dense_pair(r.cols[r.fk_col[j]].buf.as<int32_t>(), r.cols[r.fk_col2[j]].buf.as<int32_t>(),
                                      r.nrows, ch.kdict[0].as<uint64_t>(), ch.kdn[0], t.as<int32_t>(), st),
                 "prepare remap");
        for (size_t i = 0; i < ch.key_cols_more.size(); i++) {  // (code of the prefix, next attribute); -1 stays dangling
          const int fc = r.fk_cols_more[j][i];
          CTX_CUDA(c, column_ready(r.cols[fc], st), "prepare copy");
          CTX_CUDA(c, lookup_dense_pair(t.as<int32_t>(), r.cols[fc].buf.as<int32_t>(), r.nrows, ch.kdict[i + 1].as<uint64_t>(),
                                        ch.kdn[i + 1], d.as<int32_t>(), st),
                   "prepare remap");
          std::swap(t, d);
        }
        std::swap(t, d);
      } else if (r.fk_col2[j] >= 0) {  // two-attribute key
        CTX_CUDA(c, column_ready(r.cols[r.fk_col2[j]], st), "prepare copy");
        CTX_CUDA(c, lookup_dense_pair(r.cols[r.fk_col[j]].buf.as<int32_t>(), r.cols[r.fk_col2[j]].buf.as<int32_t>(),
                                      r.nrows, ch.dict.as<uint64_t>(), ch.nkeys, d.as<int32_t>(), st),
                 "prepare remap");
      } else {
        CTX_CUDA(c, lookup_dense(r.cols[r.fk_col[j]].buf.as<int32_t>(), r.nrows, ch.dict.as<int32_t>(), ch.nkeys,
                                 d.as<int32_t>(), st),
                 "prepare remap");
      }
      r.fk_dense.push_back(std::move(d));
    }
    // (2) inner join: drop rows with a dangling foreign key
    std::vector<const int32_t*> fks;
    for (auto& f : r.fk_dense) fks.push_back(f.as<int32_t>());
    DevBuf keep;
    int64_t nkeep = r.nrows;
    CTX_CUDA(c, keep_rows(fks, r.nrows, keep, nkeep, st), "prepare filter");
    if (nkeep != r.nrows) CTX_CUDA(c, permute_rel(r, keep.as<uint32_t>(), nkeep, st), "prepare compact");
    if (u != c->root) {
      // (3) dictionary of the key to the parent, dense ids, sort by them
      CTX_CUDA(c, column_ready(r.cols[r.key_col], st), "prepare copy");
      DevBuf codes;
      if (!r.key_cols_more.empty()) {  // three or more attributes: the chain of pair dictionaries
        CTX_CUDA(c, column_ready(r.cols[r.key_col2], st), "prepare copy");
        r.kdict.clear();
        r.kdn.clear();
        DevBuf dct;
        int64_t nd = 0;
        CTX_CUDA(c, dict_encode_pair(r.cols[r.key_col].buf.as<int32_t>(), r.cols[r.key_col2].buf.as<int32_t>(), r.nrows,
                                     dct, nd, &codes, st),
                 "prepare dict");
        r.kdict.push_back(std::move(dct));
        r.kdn.push_back(nd);
        for (int kc : r.key_cols_more) {
          CTX_CUDA(c, column_ready(r.cols[kc], st), "prepare copy");
          DevBuf next, d2;
          CTX_CUDA(c, dict_encode_pair(codes.as<int32_t>(), r.cols[kc].buf.as<int32_t>(), r.nrows, d2, nd, &next, st),
                   "prepare dict");
          r.kdict.push_back(std::move(d2));
          r.kdn.push_back(nd);
          codes = std::move(next);
        }
        r.nkeys = nd;
      } else if (r.key_col2 >= 0) {
        CTX_CUDA(c, column_ready(r.cols[r.key_col2], st), "prepare copy");
        CTX_CUDA(c, dict_encode_pair(r.cols[r.key_col].buf.as<int32_t>(), r.cols[r.key_col2].buf.as<int32_t>(), r.nrows,
                                     r.dict, r.nkeys, &codes, st),
                 "prepare dict");
      } else {
        CTX_CUDA(c, dict_encode_i32(r.cols[r.key_col].buf.as<int32_t>(), r.nrows, r.dict, r.nkeys, &codes, st),
                 "prepare dict");
      }
      r.dense_key = std::move(codes);
      DevBuf perm;
      CTX_CUDA(c, sort_perm_by_dense(r.dense_key.as<int32_t>(), r.nrows, r.nkeys, perm, st), "prepare sort");
      CTX_CUDA(c, permute_rel(r, perm.as<uint32_t>(), r.nrows, st), "prepare permute");
      r.unique_key = r.nkeys == r.nrows;
    }
    tr.mark(r.name.c_str(), st);
  }
  // (4) composite sort of the root by its children's dense keys, increasing
  // domain size, then keep this rank's contiguous shard.
  Rel& R = c->rels[c->root];
  c->levels.clear();
  for (size_t j = 0; j < R.children.size(); j++) c->levels.push_back((int)j);
  std::stable_sort(c->levels.begin(), c->levels.end(), [&](int a, int b) {
    return c->rels[R.children[a]].nkeys < c->rels[R.children[b]].nkeys;
  });
  if (!c->levels.empty() && R.nrows > 1) {
    std::vector<const int32_t*> keys;
    std::vector<int64_t> nk;
    for (int j : c->levels) {
      keys.push_back(R.fk_dense[j].as<int32_t>());
      nk.push_back(c->rels[R.children[j]].nkeys);
    }
    DevBuf perm;
    CTX_CUDA(c, sort_perm_composite(keys, nk, R.nrows, perm, st), "prepare root sort");
    tr.mark("root sort", st);
    CTX_CUDA(c, permute_rel(R, perm.as<uint32_t>(), R.nrows, st), "prepare root permute");
    tr.mark("root permute", st);
  }
  for (auto& r : c->rels)  // columns no permutation consumed
    for (auto& col : r.cols) CTX_CUDA(c, column_ready(col, st), "prepare copy");
  if (c->copy_stream) c->copies_pending = true;  // host buffers released by plan (copies_wait)
  c->root_rows_global = R.nrows;
  if (c->shard_nparts > 1) {
    for (size_t i = 0; i < R.cols.size(); i++) {
      if (R.cols[i].dt != LMFAO_INT32) continue;
      DevBuf d;
      int64_t nd = 0;
      CTX_CUDA(c, dict_encode_i32(R.cols[i].buf.as<int32_t>(), R.nrows, d, nd, nullptr, st), "prepare dict");
      R.full_dict_n[R.cols[i].attr] = nd;
      R.full_dict[R.cols[i].attr] = std::move(d);
    }
    int64_t lo = 0, hi = 0;
    shard_range(R.nrows, c->shard_part, c->shard_nparts, lo, hi);
    CTX_CUDA(c, slice_rel(R, lo, hi, st), "prepare shard");
  }
  // owners: the top-most relation holding each attribute (unique by P:720)
  std::vector<int> depth(c->rels.size(), 0);
  for (size_t u = 0; u < c->rels.size(); u++)
    for (int v = c->rels[u].parent; v != -1; v = c->rels[v].parent) depth[u]++;
  c->owner.assign(c->attrs.size(), -1);
  for (size_t a = 0; a < c->attrs.size(); a++) {
    int best = -1;
    for (auto& o : c->attrs[a].occ)
      if (best < 0 || depth[o.first] < depth[best]) best = o.first;
    c->owner[a] = best;
  }
  c->postorder.clear();
  for (int u : post)
    if (u != c->root) c->postorder.push_back(u);
  c->state = S_PREPARED;
  return LMFAO_OK;
}

namespace {
// Can the query's group-by attributes be placed at this context's root?  The root, a
// unique-keyed child (determined by a root row), or a child with a non-unique key (the query is
// then finished at that child: all its group-by attributes must belong to it).
lmfao_status gb_placement(lmfao_ctx* c, const std::vector<int>& gb) {
  for (int a : gb) {
    const int o = c->owner[a];
    if (!(o == c->root || c->rels[o].parent == c->root))
      return fail(c, LMFAO_ERR_UNSUPPORTED, "group-by attribute %s belongs to neither the root nor a child of the root",
                  c->attrs[a].name.c_str());
  }
  int T = -1;
  bool mixed = false;
  for (int a : gb) {
    const int o = c->owner[a];
    if (o != c->root && !c->rels[o].unique_key) T = o;
  }
  if (T >= 0)
    for (int a : gb) mixed |= c->owner[a] != T;
  if (mixed)
    return fail(c, LMFAO_ERR_UNSUPPORTED, "group-by attributes of %s (a non-unique key) mixed with attributes of other relations",
                c->rels[T].name.c_str());
  return LMFAO_OK;
}

// The secondary context rooted at relation `root` (created on first use): every relation copied
// from this context's device columns, the join tree re-oriented from `root`, prepared.
int secondary_for(lmfao_ctx* c, int root) {
  for (size_t i = 0; i < c->secs.size(); i++)
    if (c->secs[i].root == root) return (int)i;
  copies_wait(c);  // the columns are copied from this context's device buffers
  if (cudaStreamSynchronize(c->stream) != cudaSuccess) return -1;
  lmfao_ctx* s = nullptr;
  if (lmfao_create(c->device, 0, 1, nullptr, &s) != LMFAO_OK) return -1;
  s->is_secondary = true;
  lmfao_ctx::Secondary sc;
  sc.ctx = s;
  sc.root = root;
  auto bad = [&]() {
    lmfao_destroy(s);
    return -1;
  };
  for (auto& r : c->rels) {
    std::vector<const char*> names;
    std::vector<lmfao_dtype> dts;
    std::vector<const void*> ptrs;
    for (auto& col : r.cols) {
      names.push_back(col.name.c_str());
      dts.push_back(col.dt);
      ptrs.push_back(col.buf.p);
    }
    int32_t rid = -1;
    if (lmfao_add_relation(s, r.name.c_str(), r.nrows, (int32_t)r.cols.size(), names.data(), dts.data(), ptrs.data(),
                           LMFAO_COLS_DEVICE, &rid) != LMFAO_OK)
      return bad();
  }
  // re-orient the tree: breadth first from `root` over the undirected edges
  const int m = (int)c->rels.size();
  std::vector<std::vector<int>> adj(m);
  for (int u = 0; u < m; u++)
    if (c->rels[u].parent >= 0) {
      adj[u].push_back(c->rels[u].parent);
      adj[c->rels[u].parent].push_back(u);
    }
  std::vector<int32_t> par, chi;
  std::vector<int> seen(m, 0), queue{root};
  seen[root] = 1;
  for (size_t i = 0; i < queue.size(); i++)
    for (int v : adj[queue[i]])
      if (!seen[v]) {
        seen[v] = 1;
        par.push_back(queue[i]);
        chi.push_back(v);
        queue.push_back(v);
      }
  if (lmfao_set_join_tree(s, root, (int32_t)par.size(), par.data(), chi.data()) != LMFAO_OK || lmfao_prepare(s) != LMFAO_OK)
    return bad();
  cudaSetDevice(c->device);
  if (cudaStreamCreateWithFlags(&sc.stream, cudaStreamNonBlocking) ||
      cudaEventCreateWithFlags(&sc.ev_in, cudaEventDisableTiming) ||
      cudaEventCreateWithFlags(&sc.ev_out, cudaEventDisableTiming))
    return bad();
  c->secs.push_back(sc);
  return (int)c->secs.size() - 1;
}
}  // namespace

lmfao_status lmfao_add_query(lmfao_ctx* c, int32_t n_groupby, const int32_t* groupby_attrs, int32_t n_udafs,
                             const lmfao_udaf* udafs, int32_t* query_id) {
  if (!c) return LMFAO_ERR_INVALID_ARG;
  if (c->state != S_PREPARED) return fail(c, LMFAO_ERR_STATE, "add_query needs prepare and must precede plan");
  if (n_groupby < 0 || n_udafs < 0 || (n_groupby > 0 && !groupby_attrs) || (n_udafs > 0 && !udafs))
    return fail(c, LMFAO_ERR_INVALID_ARG, "add_query: bad arguments");
  if (n_groupby > 8) return fail(c, LMFAO_ERR_UNSUPPORTED, "more than 8 group-by attributes");
  Query q;
  int na = (int)c->attrs.size();
  std::set<int> gbs;
  for (int i = 0; i < n_groupby; i++) {
    int a = groupby_attrs[i];
    if (a < 0 || a >= na) return fail(c, LMFAO_ERR_UNKNOWN_ATTR, "unknown group-by attribute id %d", a);
    if (c->attrs[a].dt != LMFAO_INT32)
      return fail(c, LMFAO_ERR_TYPE, "group-by attribute %s must be int32", c->attrs[a].name.c_str());
    if (!gbs.insert(a).second) return fail(c, LMFAO_ERR_INVALID_ARG, "duplicate group-by attribute");
    q.gb.push_back(a);
  }
  if (lmfao_status ps = gb_placement(c, q.gb)) {
    // each aggregate to its own root: another root of the same join tree, chosen
    // as P:958 does — the relations holding the query's group-by attributes, by the number of
    // them they hold, then by size — where the query can be placed
    if (c->is_secondary || c->world > 1) return ps;
    std::vector<std::pair<std::pair<int, int64_t>, int>> cand;  // ((held, rows), relation)
    for (size_t u = 0; u < c->rels.size(); u++) {
      int held = 0;
      for (int a : q.gb) held += c->rels[u].find_attr(a) >= 0;
      if (held > 0 && (int)u != c->root) cand.push_back({{held, c->rels[u].nrows}, (int)u});
    }
    std::sort(cand.rbegin(), cand.rend());
    const std::string why = c->err;
    for (auto& cd : cand) {
      const int si = secondary_for(c, cd.second);
      if (si < 0) continue;
      int32_t sq = -1;
      if (lmfao_add_query(c->secs[si].ctx, n_groupby, groupby_attrs, n_udafs, udafs, &sq) != LMFAO_OK) continue;
      c->qmap.push_back({si, sq});
      if (query_id) *query_id = (int)c->qmap.size() - 1;
      return LMFAO_OK;
    }
    return fail(c, ps, "%s (and no other root of the join tree places it)", why.c_str());
  }
  for (int j = 0; j < n_udafs; j++) {
    const lmfao_udaf& u = udafs[j];
    if (u.n_products < 0 || (u.n_products > 0 && !u.products))
      return fail(c, LMFAO_ERR_INVALID_ARG, "udaf %d: bad products", j);
    std::vector<QProduct> ps;
    for (int p = 0; p < u.n_products; p++) {
      const lmfao_product& pr = u.products[p];
      if (pr.n_factors < 0 || (pr.n_factors > 0 && !pr.factors))
        return fail(c, LMFAO_ERR_INVALID_ARG, "udaf %d product %d: bad factors", j, p);
      QProduct qp{pr.coeff, {}};
      for (int f = 0; f < pr.n_factors; f++) {
        const lmfao_factor& fa = pr.factors[f];
        if (fa.kind < LMFAO_F_CONST || fa.kind > LMFAO_F_IN) return fail(c, LMFAO_ERR_INVALID_ARG, "bad factor kind");
        if (fa.kind == LMFAO_F_IN && !(fa.param >= 0.0 && fa.param < 9007199254740992.0 && fa.param == std::floor(fa.param)))
          return fail(c, LMFAO_ERR_INVALID_ARG, "LMFAO_F_IN: the set mask must be an integer in [0, 2^53)");
        if (fa.kind == LMFAO_F_CONST) {
          qp.f.push_back(QFactor{fa.kind, -1, fa.param});
          continue;
        }
        if (fa.attr < 0 || fa.attr >= na) return fail(c, LMFAO_ERR_UNKNOWN_ATTR, "unknown attribute id %d", fa.attr);
        qp.f.push_back(QFactor{fa.kind, fa.attr, fa.param});
      }
      ps.push_back(qp);
    }
    q.udafs.push_back(ps);
  }
  c->queries.push_back(std::move(q));
  c->qmap.push_back({-1, (int)c->queries.size() - 1});
  if (query_id) *query_id = (int)c->qmap.size() - 1;
  return LMFAO_OK;
}

}  // extern "C"

// ===================================================================== planner
namespace {

int child_toward(const lmfao_ctx* c, int node, int target) {
  // the child of `node` whose subtree contains `target` (target != node)
  int u = target;
  while (c->rels[u].parent != node) u = c->rels[u].parent;
  return u;
}

int slot_of(lmfao_ctx* c, int node, const std::vector<QFactor>& fs) {
  const Rel& r = c->rels[node];
  SlotKey key;
  std::vector<std::vector<QFactor>> sub(r.children.size());
  for (auto& f : fs) {
    int o = c->owner[f.attr];
    if (o == node) {
      key.own.emplace_back(f.kind, f.attr, dbits(f.param));
    } else {
      int ch = child_toward(c, node, o);
      for (size_t j = 0; j < r.children.size(); j++)
        if (r.children[j] == ch) sub[j].push_back(f);
    }
  }
  std::sort(key.own.begin(), key.own.end());
  for (size_t j = 0; j < r.children.size(); j++) key.child_slots.push_back(slot_of(c, r.children[j], sub[j]));
  NodePlan& np = c->nodes[node];
  auto it = np.index.find(key);
  if (it != np.index.end()) return it->second;
  int s = (int)np.slots.size();
  np.slots.push_back(key);
  np.index[key] = s;
  return s;
}

void emit_term(Program& p, const lmfao_ctx* c, int node, double coef, const std::vector<std::tuple<int, int, uint64_t>>& own,
               const std::vector<int>& child_slots) {
  const Rel& r = c->rels[node];
  p.ip.push_back((int)own.size());
  p.dp.push_back(coef);
  for (auto& o : own) {
    int kind = std::get<0>(o), attr = std::get<1>(o);
    double prm;
    uint64_t b = std::get<2>(o);
    std::memcpy(&prm, &b, 8);
    p.ip.push_back(kind);
    p.ip.push_back(r.find_attr(attr));
    p.dp.push_back(prm);
  }
  for (int s : child_slots) p.ip.push_back(s);
}

// root term of a product: own factors at the root, one slot per root child
void root_term(lmfao_ctx* c, const QProduct& pr, double& coef, std::vector<std::tuple<int, int, uint64_t>>& own,
               std::vector<int>& slots) {
  const Rel& R = c->rels[c->root];
  coef = pr.coeff;
  std::vector<std::vector<QFactor>> sub(R.children.size());
  for (auto& f : pr.f) {
    if (f.kind == LMFAO_F_CONST) {
      coef *= f.param;
      continue;
    }
    int o = c->owner[f.attr];
    if (o == c->root) {
      own.emplace_back(f.kind, f.attr, dbits(f.param));
    } else {
      int ch = child_toward(c, c->root, o);
      for (size_t j = 0; j < R.children.size(); j++)
        if (R.children[j] == ch) sub[j].push_back(f);
    }
  }
  for (size_t j = 0; j < R.children.size(); j++) slots.push_back(slot_of(c, R.children[j], sub[j]));
}

void append_udaf_program(lmfao_ctx* c, Program& p, const std::vector<QProduct>& u) {
  p.out_ioff.push_back((int)p.ip.size());
  p.out_doff.push_back((int)p.dp.size());
  p.ip.push_back((int)u.size());
  for (auto& pr : u) {
    double coef;
    std::vector<std::tuple<int, int, uint64_t>> own;
    std::vector<int> slots;
    root_term(c, pr, coef, own, slots);
    emit_term(p, c, c->root, coef, own, slots);
  }
}

// Programs of a query finished at the non-unique-keyed root child T (see RevPlan): per
// product, the root side (root factors, the other children's view slots, T left out as
// slot -1) and the T side (T's factors, its children's view slots); a last output each for
// the multiplicities.
void build_rev(lmfao_ctx* c, const Query& Q, int T, RevPlan& rv, Program& rp, Program& tp, std::vector<int32_t>& pu) {
  const Rel& R = c->rels[c->root];
  const Rel& TR = c->rels[T];
  int jT = 0;
  while (R.children[jT] != T) jT++;
  rv.T = T;
  rv.j = jT;
  auto out = [](Program& p) {
    p.out_ioff.push_back((int)p.ip.size());
    p.out_doff.push_back((int)p.dp.size());
    p.ip.push_back(1);  // one term
  };
  for (size_t u = 0; u < Q.udafs.size(); u++)
    for (auto& pr : Q.udafs[u]) {
      double coef = pr.coeff;
      std::vector<std::tuple<int, int, uint64_t>> own, ownT;
      std::vector<std::vector<QFactor>> sub(R.children.size()), subT(TR.children.size());
      for (auto& f : pr.f) {
        if (f.kind == LMFAO_F_CONST) {
          coef *= f.param;
          continue;
        }
        const int o = c->owner[f.attr];
        if (o == c->root) {
          own.emplace_back(f.kind, f.attr, dbits(f.param));
          continue;
        }
        const int ch = child_toward(c, c->root, o);
        if (ch != T) {
          for (size_t j = 0; j < R.children.size(); j++)
            if (R.children[j] == ch) sub[j].push_back(f);
        } else if (o == T) {
          ownT.emplace_back(f.kind, f.attr, dbits(f.param));
        } else {
          const int cT = child_toward(c, T, o);
          for (size_t k = 0; k < TR.children.size(); k++)
            if (TR.children[k] == cT) subT[k].push_back(f);
        }
      }
      std::sort(own.begin(), own.end());
      std::sort(ownT.begin(), ownT.end());
      std::vector<int> slots, slotsT;
      for (size_t j = 0; j < R.children.size(); j++)
        slots.push_back((int)j == jT ? -1 : slot_of(c, R.children[j], sub[j]));
      for (size_t k = 0; k < TR.children.size(); k++) slotsT.push_back(slot_of(c, TR.children[k], subT[k]));
      out(rp);
      emit_term(rp, c, c->root, coef, own, slots);
      out(tp);
      emit_term(tp, c, T, 1.0, ownT, slotsT);
      pu.push_back((int32_t)u);
    }
  std::vector<int> cs, csT(TR.children.size(), 0);  // the count terms
  for (size_t j = 0; j < R.children.size(); j++) cs.push_back((int)j == jT ? -1 : 0);
  out(rp);
  emit_term(rp, c, c->root, 1.0, {}, cs);
  out(tp);
  emit_term(tp, c, T, 1.0, {}, csT);
}

}  // namespace

static lmfao_status plan_local(lmfao_ctx* c) {
  if (!c) return LMFAO_ERR_INVALID_ARG;
  if (c->state != S_PREPARED) return fail(c, LMFAO_ERR_STATE, "plan needs prepare (and runs once)");
  cudaSetDevice(c->device);
  StreamScope scope_(c->stream);
  // LMFAO_PLAIN_SITES (A/B): plan-time allocations from plain cudaMalloc instead of the pool,
  // bit 1 group tables, 2 code sets, 4 specialised paths, 8 views and programs
  const int plain_sites = [] {
    const char* e = std::getenv("LMFAO_PLAIN_SITES");
    return e ? std::atoi(e) : 0;
  }();
  cudaStream_t st = c->stream;
  PhaseTrace tr("plan");
  c->nodes.clear();
  c->nodes.resize(c->rels.size());
  // slot 0 = count for every view (post-order: grandchildren first)
  for (int u : c->postorder) slot_of(c, u, {});
  // root programs (this also registers every view slot)
  Program scal;
  c->scalar_queries.clear();
  c->scalar_off.clear();
  c->query_kind.assign(c->queries.size(), 0);
  c->query_slot.assign(c->queries.size(), 0);
  std::vector<Program> gprogs;
  c->groups.clear();
  c->revs.clear();
  c->code_cache.clear();
  for (size_t q = 0; q < c->queries.size(); q++) {
    const Query& Q = c->queries[q];
    if (Q.gb.empty()) {
      c->query_kind[q] = 0;
      c->query_slot[q] = (int)c->scalar_queries.size();
      c->scalar_queries.push_back((int)q);
      c->scalar_off.push_back((int)scal.out_ioff.size());
      for (auto& u : Q.udafs) append_udaf_program(c, scal, u);
    } else {
      c->query_kind[q] = 1;
      c->query_slot[q] = (int)c->groups.size();
      c->groups.emplace_back();
      Program gp;
      int T = -1;
      for (int a : Q.gb)
        if (c->owner[a] != c->root && !c->rels[c->owner[a]].unique_key) T = c->owner[a];
      if (T >= 0) {  // finished at T (k_rev_*); no fused-scan program
        c->groups.back().rev = (int)c->revs.size();
        c->revs.emplace_back();
        RevPlan& rv = c->revs.back();
        rv.gi = (int)c->groups.size() - 1;
        Program rp, tp;
        std::vector<int32_t> pu;
        build_rev(c, Q, T, rv, rp, tp, pu);
        CTX_CUDA(c, rv.rp.upload(rp, st), "plan rev");
        CTX_CUDA(c, rv.tp.upload(tp, st), "plan rev");
        CTX_CUDA(c, rv.pu.alloc(std::max<size_t>(pu.size(), 1) * 4), "plan rev");
        if (!pu.empty())
          CTX_CUDA(c, cudaMemcpyAsync(rv.pu.p, pu.data(), pu.size() * 4, cudaMemcpyHostToDevice, st), "plan rev");
        CTX_CUDA(c, rv.A.alloc((size_t)std::max<int64_t>(c->rels[T].nkeys, 1) * rv.rp.nout * 8), "plan rev");
      } else {
        for (auto& u : Q.udafs) append_udaf_program(c, gp, u);
      }
      gprogs.push_back(std::move(gp));
    }
  }
  tr.mark("root programs");
  // view programs: one output per slot
  for (int u : c->postorder) {
    NodePlan& np = c->nodes[u];
    Program p;
    for (auto& s : np.slots) {
      p.out_ioff.push_back((int)p.ip.size());
      p.out_doff.push_back((int)p.dp.size());
      p.ip.push_back(1);
      emit_term(p, c, u, 1.0, s.own, s.child_slots);
    }
    StreamScope vs(st, !(plain_sites & 8));
    CTX_CUDA(c, np.prog.upload(p, st), "plan upload view program");
    CTX_CUDA(c, np.V.alloc(std::max<int64_t>(c->rels[u].nkeys, 1) * np.slots.size() * 8), "plan alloc view");
    {  // leaf child with slots of <= 2 identity factors: the linear view kernel
      const Rel& r = c->rels[u];
      bool lin = r.children.empty() && np.slots.size() <= 64;
      for (auto& sl : np.slots) {
        if (sl.own.size() > 2) lin = false;
        for (auto& o : sl.own)
          if (std::get<0>(o) != LMFAO_F_IDENT) lin = false;
      }
      np.linear = lin;
      if (lin) {
        np.lin = ViewLinArgs{};
        np.lin.nslots = (int)np.slots.size();
        for (size_t i = 0; i < np.slots.size(); i++) {
          const auto& own = np.slots[i].own;
          for (size_t f = 0; f < own.size(); f++) {
            const Column& col = r.cols[r.find_attr(std::get<1>(own[f]))];
            (f == 0 ? np.lin.ca[i] : np.lin.cb[i]) = col.buf.p;
            (f == 0 ? np.lin.ia[i] : np.lin.ib[i]) = col.dt == LMFAO_INT32;
          }
        }
      }
    }
  }
  tr.mark("view programs", st);
  // scalar outputs
  CTX_CUDA(c, c->scalar_prog.upload(scal, st), "plan upload");
  int nout = c->scalar_prog.nout;
  c->scalar_grid = 148 * 4;
  CTX_CUDA(c, c->partials.alloc((size_t)c->scalar_grid * std::max(nout, 1) * 8), "plan");
  CTX_CUDA(c, c->cpart.alloc((size_t)c->scalar_grid * 8), "plan");
  CTX_CUDA(c, c->scalar_out.alloc((size_t)std::max(nout, 1) * 8), "plan");
  CTX_CUDA(c, c->scalar_count.alloc(8), "plan");
  // group-by queries: dictionaries, codes, dense cell tables
  const int64_t sparse_cells = [] {  // cube.cu's threshold for sparse cuboids (LMFAO_CUBE_SPARSE_CELLS)
    const char* e = std::getenv("LMFAO_CUBE_SPARSE_CELLS");
    return e ? std::atoll(e) : ((int64_t)1 << 25);
  }();
  for (size_t q = 0; q < c->queries.size(); q++) {
    if (c->query_kind[q] != 1) continue;
    GroupPlan& gp = c->groups[c->query_slot[q]];
    const Query& Q = c->queries[q];
    gp.q = (int)q;
    gp.nudaf = (int)Q.udafs.size();
    gp.g.ngb = gp.d.ngb = (int)Q.gb.size();
    std::vector<int64_t> radix;
    for (size_t i = 0; i < Q.gb.size(); i++) {
      int a = Q.gb[i], o = c->owner[a];
      const Rel& r = c->rels[o];
      std::shared_ptr<CodeSet>& cs = c->code_cache[a];
      if (!cs) {
        StreamScope cs_scope(st, !(plain_sites & 2));
        cs = std::make_shared<CodeSet>();
        DevBuf& dict = cs->dict;
        DevBuf& codes = cs->codes;
        int64_t& nd = cs->nd;
        auto fd = r.full_dict.find(a);
        if (fd != r.full_dict.end()) {  // sharded root: the global dictionary
          nd = r.full_dict_n.at(a);
          CTX_CUDA(c, dict.alloc(std::max<int64_t>(nd, 1) * 4), "plan dictionary");
          CTX_CUDA(c, cudaMemcpyAsync(dict.p, fd->second.p, nd * 4, cudaMemcpyDeviceToDevice, st), "plan dictionary");
          CTX_CUDA(c, codes.alloc(std::max<int64_t>(r.nrows, 1) * 4), "plan codes");
          CTX_CUDA(c, lookup_dense(r.cols[r.find_attr(a)].buf.as<int32_t>(), r.nrows, dict.as<int32_t>(), nd,
                                   codes.as<int32_t>(), st),
                   "plan codes");
          CTX_CUDA(c, cudaStreamSynchronize(st), "plan codes");
        } else {
          CTX_CUDA(c, dict_encode_i32(r.cols[r.find_attr(a)].buf.as<int32_t>(), r.nrows, dict, nd, &codes, st),
                   "plan dictionary");
        }
      }
      const DevBuf& dict = cs->dict;
      const DevBuf& codes = cs->codes;
      const int64_t nd = cs->nd;
      gp.g.code[i] = codes.as<int32_t>();
      gp.g.code_child[i] = -1;
      if (o != c->root) {
        const Rel& R = c->rels[c->root];
        for (size_t j = 0; j < R.children.size(); j++)
          if (R.children[j] == o) gp.g.code_child[i] = (int)j;
      }
      gp.d.dict[i] = dict.as<int32_t>();
      gp.d.radix[i] = std::max<int64_t>(nd, 1);
      radix.push_back(std::max<int64_t>(nd, 1));
      gp.sets.push_back(cs);
    }
    int64_t cells = 1;
    for (int i = (int)radix.size() - 1; i >= 0; i--) {
      gp.g.stride[i] = gp.d.stride[i] = cells;
      cells *= radix[i];
      if (cells > (int64_t)1 << 34) return fail(c, LMFAO_ERR_UNSUPPORTED, "group-by domain too large for v1");
    }
    gp.ncells = cells;
    if ((double)cells * (gp.nudaf + 1) * 8 > 40e9)
      return fail(c, LMFAO_ERR_UNSUPPORTED, "dense group-by table too large (%lld cells)", (long long)cells);
    // world > 1: tables of at least LMFAO_DIST_CELLS cells (default 2^16) are distributed —
    // reduce-scattered by cell range; smaller ones are all-reduced (complete on every rank)
    {
      const int64_t dist_min = [] {
        const char* e = std::getenv("LMFAO_DIST_CELLS");
        return e ? std::atoll(e) : ((int64_t)1 << 16);
      }();
      gp.dist = c->world > 1 && cells >= dist_min;
      gp.ncells_alloc = gp.dist ? (cells + c->world - 1) / c->world * c->world : cells;
      owner_range(cells, c->rank, c->world, gp.cell_lo, gp.cell_hi);
      if (!gp.dist) gp.cell_lo = 0, gp.cell_hi = cells;
    }
    // tables the data-cube path keeps sparse (no dense table: run records sorted by cell) are
    // allocated only if no specialised path takes them (below)
    if (cells <= sparse_cells || cells > ((int64_t)1 << 32)) {
      StreamScope ts(st, !(plain_sites & 1));
      CTX_CUDA(c, gp.table.alloc(gp.ncells_alloc * std::max(gp.nudaf, 1) * 8), "plan group table");
      CTX_CUDA(c, gp.counts.alloc(gp.ncells_alloc * 8), "plan group counts");
      CTX_CUDA(c, cudaMemsetAsync(gp.table.p, 0, gp.table.bytes, st), "plan group table");
      CTX_CUDA(c, cudaMemsetAsync(gp.counts.p, 0, gp.counts.bytes, st), "plan group counts");
    }
    CTX_CUDA(c, gp.prog.upload(gprogs[c->query_slot[q]], st), "plan upload group");
  }
  // fused group-by scan: one combined program, one descriptor per group-by query
  std::vector<GroupDesc> descs;
  std::vector<int> desc_group;  // group index of each descriptor
  {
    Program all;
    for (size_t gi = 0; gi < c->groups.size(); gi++) {
      GroupPlan& gp = c->groups[gi];
      const Query& Q = c->queries[gp.q];
      const bool rev = gp.rev >= 0;  // finished at its child: no fused-scan outputs (and no new view slots:
                                     // the views are laid out already)
      GroupDesc d{};
      d.ngb = gp.g.ngb;
      d.nudaf = gp.nudaf;
      d.prog_base = (int)all.out_ioff.size();
      for (int i = 0; i < d.ngb; i++) {
        d.code[i] = gp.g.code[i];
        d.code_child[i] = gp.g.code_child[i];
        d.stride[i] = gp.g.stride[i];
      }
      d.table = gp.table.as<double>();
      d.counts = gp.counts.as<unsigned long long>();
      if (gp.nudaf > 64) return fail(c, LMFAO_ERR_UNSUPPORTED, "more than 64 UDAFs in a group-by query");
      std::vector<double> cc(std::max(gp.nudaf, 1), std::nan(""));
      for (int j = 0; j < gp.nudaf; j++) {
        const auto& u = Q.udafs[j];
        // a UDAF whose products are all constants is c * COUNT, c = Σ_p coeff_p Π params
        bool constant = true;
        double coef = 0.0;
        for (auto& pr : u) {
          double v = pr.coeff;
          for (auto& f : pr.f) {
            if (f.kind != LMFAO_F_CONST) constant = false;
            else v *= f.param;
          }
          coef += v;
        }
        if (!constant) coef = 0.0;
        d.countlike[j] = constant;
        if (!constant) d.nsum++;
        if (constant) cc[j] = coef;
        if (rev) continue;
        all.out_ioff.push_back((int)all.ip.size());
        all.out_doff.push_back((int)all.dp.size());
        all.ip.push_back((int)u.size());
        for (auto& pr : u) {
          double coef2;
          std::vector<std::tuple<int, int, uint64_t>> own;
          std::vector<int> slots;
          root_term(c, pr, coef2, own, slots);
          emit_term(all, c, c->root, coef2, own, slots);
        }
      }
      CTX_CUDA(c, gp.countcoef.alloc(cc.size() * 8), "plan");
      CTX_CUDA(c, cudaMemcpyAsync(gp.countcoef.p, cc.data(), cc.size() * 8, cudaMemcpyHostToDevice, st), "plan");
      gp.d.countcoef = gp.countcoef.as<double>();
      if (gp.rev >= 0) {  // finished at its child, not by the fused scan
        c->revs[gp.rev].d = d;
        continue;
      }
      descs.push_back(d);
      desc_group.push_back((int)gi);
    }
    CTX_CUDA(c, c->group_prog.upload(all, st), "plan upload groups");
    c->ndescs = (int)descs.size();
    CTX_CUDA(c, c->group_descs.alloc(std::max<size_t>(descs.size(), 1) * sizeof(GroupDesc)), "plan");
    if (!descs.empty())
      CTX_CUDA(c, cudaMemcpyAsync(c->group_descs.p, descs.data(), descs.size() * sizeof(GroupDesc), cudaMemcpyHostToDevice, st),
               "plan");
  }
  tr.mark("group plans", st);
  // specialised kernels for recognised batch shapes (gram.cu / hist.cu)
  {
    StreamScope fs(st, !(plain_sites & 4));
    c->fast.reset(plan_fast_paths(c));
  }
  {  // deferred tables that no specialised path took sparse: allocate them now, re-plan
    bool late = false;
    for (auto& gp : c->groups) {
      if (gp.table.p || gp.direct) continue;
      StreamScope ts(st, !(plain_sites & 1));
      CTX_CUDA(c, gp.table.alloc(gp.ncells_alloc * std::max(gp.nudaf, 1) * 8), "plan group table");
      CTX_CUDA(c, gp.counts.alloc(gp.ncells_alloc * 8), "plan group counts");
      CTX_CUDA(c, cudaMemsetAsync(gp.table.p, 0, gp.table.bytes, st), "plan group table");
      CTX_CUDA(c, cudaMemsetAsync(gp.counts.p, 0, gp.counts.bytes, st), "plan group counts");
      late = true;
    }
    if (late) {
      for (size_t i = 0; i < descs.size(); i++) {
        descs[i].table = c->groups[desc_group[i]].table.as<double>();
        descs[i].counts = c->groups[desc_group[i]].counts.as<unsigned long long>();
      }
      for (auto& rv : c->revs) {
        rv.d.table = c->groups[rv.gi].table.as<double>();
        rv.d.counts = c->groups[rv.gi].counts.as<unsigned long long>();
      }
      if (!descs.empty())
        CTX_CUDA(c, cudaMemcpyAsync(c->group_descs.p, descs.data(), descs.size() * sizeof(GroupDesc),
                                    cudaMemcpyHostToDevice, st),
                 "plan");
      c->fast.reset();
      StreamScope fs(st, !(plain_sites & 4));
      c->fast.reset(plan_fast_paths(c));
    }
  }
  tr.mark("fast paths", st);
  c->state = S_PLANNED;
  return LMFAO_OK;
}

static lmfao_status run_body(lmfao_ctx* c, cudaStream_t st) {
  launches_counter_reset();
  // (b) views, bottom-up
  for (int u : c->postorder) {
    if (c->fast && c->fast->skip_generic_views()) break;
    NodePlan& np = c->nodes[u];
    const Rel& r = c->rels[u];
    CTX_CUDA(c, cudaMemsetAsync(np.V.p, 0, np.V.bytes, st), "run memset view");
    if (np.linear) {
      ViewLinArgs la = np.lin;
      la.nrows = r.nrows;
      CTX_CUDA(c, launch_view_lin(la, r.dense_key.as<int32_t>(), np.V.as<double>(), st), "run view build");
      continue;
    }
    NodeArgs a = node_args(c, u);
    CTX_CUDA(c, launch_view_build(a, r.dense_key.as<int32_t>(), np.prog.pi.as<int32_t>(), np.prog.pd.as<double>(),
                                  np.prog.pio.as<int32_t>(), np.prog.pdo.as<int32_t>(), (int)np.slots.size(),
                                  np.V.as<double>(), st),
             "run view build");
  }
  NodeArgs ra = node_args(c, c->root);
  bool scalar_done = false;
  if (c->fast) {
    int e = c->fast->run(c, ra, st, scalar_done);
    if (e) return fail(c, LMFAO_ERR_CUDA, "fast path: %s", cudaGetErrorString((cudaError_t)e));
  }
  // (c) root scan, generic path
  if (!c->scalar_queries.empty() && !scalar_done) {
    int nout = c->scalar_prog.nout;
    scan_timer_begin(c, st);
    CTX_CUDA(c, launch_root_scalar(ra, c->scalar_prog.pi.as<int32_t>(), c->scalar_prog.pd.as<double>(),
                                   c->scalar_prog.pio.as<int32_t>(), c->scalar_prog.pdo.as<int32_t>(), nout,
                                   c->partials.as<double>(), c->cpart.as<unsigned long long>(), c->scalar_grid, st),
             "run root scan");
    scan_timer_end(c, st);
    CTX_CUDA(c, launch_combine_partials(c->partials.as<double>(), c->cpart.as<unsigned long long>(), c->scalar_grid,
                                        nout, c->scalar_out.as<double>(), c->scalar_count.as<unsigned long long>(), st),
             "run combine");
  }
  if (!c->groups.empty() && !(c->fast && c->fast->handles_all_groups())) {
    for (auto& gp : c->groups) {
      CTX_CUDA(c, cudaMemsetAsync(gp.table.p, 0, gp.table.bytes, st), "run memset");
      CTX_CUDA(c, cudaMemsetAsync(gp.counts.p, 0, gp.counts.bytes, st), "run memset");
    }
    if (c->ndescs > 0)
      CTX_CUDA(c, launch_groups_fused(ra, c->group_descs.as<GroupDesc>(), c->ndescs, c->group_prog.pi.as<int32_t>(),
                                      c->group_prog.pd.as<double>(), c->group_prog.pio.as<int32_t>(),
                                      c->group_prog.pdo.as<int32_t>(), st),
               "run groups");
    for (auto& rv : c->revs) {  // group-bys finished at a non-unique-keyed child
      const Rel& R = c->rels[c->root];
      const Rel& T = c->rels[rv.T];
      auto pp = [](const DevProgram& p) {
        return ProgPtrs{p.pi.as<int32_t>(), p.pd.as<double>(), p.pio.as<int32_t>(), p.pdo.as<int32_t>(), p.nout};
      };
      CTX_CUDA(c, launch_rev(ra, R.fk_dense[rv.j].as<int32_t>(), pp(rv.rp), node_args(c, rv.T),
                             T.dense_key.as<int32_t>(), pp(rv.tp), rv.pu.as<int32_t>(), rv.A.as<double>(), T.nkeys,
                             rv.d, st),
               "run groups at a child");
    }
  }
  // combine across GPUs (domain parallelism): small outputs all-reduced, distributed
  // tables reduce-scattered by cell range (sparse cuboids were exchanged by their fast path)
  if (c->world > 1) {
    int e = 0;
    cudaEvent_t ca = nullptr, cb = nullptr;
    if (c->prof) {  // the collective's own time (lmfao_profile), reported by lmfao_plan_info
      cudaEventCreate(&ca);
      cudaEventCreate(&cb);
      cudaEventRecord(ca, st);
    }
    Comm& cm = *c->comm;
    if (!c->scalar_queries.empty()) {
      e = e ? e : cm.allreduce_sum(c->scalar_out.p, c->scalar_prog.nout, COMM_F64, st);
      e = e ? e : cm.allreduce_sum(c->scalar_count.p, 1, COMM_U64, st);
    }
    for (auto& gp : c->groups) {
      if (gp.direct) continue;
      if (gp.dist) {
        const size_t chunk = (size_t)(gp.ncells_alloc / c->world);
        e = e ? e : cm.reduce_scatter_sum(gp.table.p, chunk * gp.nudaf, COMM_F64, st);
        e = e ? e : cm.reduce_scatter_sum(gp.counts.p, chunk, COMM_U64, st);
      } else {
        e = e ? e : cm.allreduce_sum(gp.table.p, gp.ncells * gp.nudaf, COMM_F64, st);
        e = e ? e : cm.allreduce_sum(gp.counts.p, gp.ncells, COMM_U64, st);
      }
    }
    if (ca) {
      cudaEventRecord(cb, st);
      c->coll_events.push_back({ca, cb});
    }
    if (e) return fail(c, LMFAO_ERR_NCCL, "%s collective failed: %s", cm.backend(), cm.error_string(e).c_str());
  }
  for (auto& gp : c->groups) gp.gathered = false;
  for (auto& gp : c->groups) gp.compacted = false;
  c->ran = true;
  c->launches_last_run = launches_counter_reset();
  return LMFAO_OK;
}

// lmfao_run: the first run executes eagerly (lazy kernel attributes, validation);
// the second captures the whole sequence into a CUDA Graph on the ctx stream and
// every later run replays it on the caller's stream (one launch instead of ~a dozen).
// Profiling runs and multi-GPU runs (NCCL) stay eager.
// Drops the batch and its plan (queries, kernels selected, results) and keeps the loaded,
// prepared relations: the next batch over the same data (a tree learner's next node) needs
// add_query + plan only.
extern "C" lmfao_status lmfao_reset_batch(lmfao_ctx* c) {
  if (!c) return LMFAO_ERR_INVALID_ARG;
  if (c->state != S_PREPARED && c->state != S_PLANNED) return fail(c, LMFAO_ERR_STATE, "reset_batch needs prepare");
  cudaSetDevice(c->device);
  StreamScope scope_(c->stream);
  CTX_CUDA(c, cudaStreamSynchronize(c->stream), "reset_batch");
  if (c->graph_exec) cudaGraphExecDestroy(c->graph_exec);
  c->graph_exec = nullptr;
  c->graph_runs = c->graph_launches = 0;
  c->fast.reset();
  c->queries.clear();
  c->nodes.clear();
  c->scalar_queries.clear();
  c->scalar_off.clear();
  c->groups.clear();
  c->revs.clear();
  c->code_cache.clear();
  c->query_kind.clear();
  c->query_slot.clear();
  c->qmap.clear();
  c->ran = false;
  c->state = S_PREPARED;
  for (auto& sc : c->secs)  // keep the secondary roots prepared for the next batch
    if (lmfao_status e = lmfao_reset_batch(sc.ctx)) return fail(c, e, "secondary root: %s", sc.ctx->err.c_str());
  return LMFAO_OK;
}

// Dynamic functions: the next node of a decision tree differs from the
// planned batch only in its path condition; the planned kernels take the new one as is.
extern "C" lmfao_status lmfao_set_condition(lmfao_ctx* c, int32_t n_factors, const lmfao_factor* factors) {
  if (!c) return LMFAO_ERR_INVALID_ARG;
  if (c->state != S_PLANNED) return fail(c, LMFAO_ERR_STATE, "set_condition needs plan");
  if (n_factors < 0 || (n_factors > 0 && !factors)) return fail(c, LMFAO_ERR_INVALID_ARG, "bad condition");
  for (int i = 0; i < n_factors; i++) {
    const lmfao_factor& f = factors[i];
    if (f.kind < LMFAO_F_LT || f.kind > LMFAO_F_IN) return fail(c, LMFAO_ERR_INVALID_ARG, "condition factor %d is not a predicate", i);
    if (f.attr < 0 || f.attr >= (int)c->attrs.size()) return fail(c, LMFAO_ERR_UNKNOWN_ATTR, "condition factor %d: unknown attribute", i);
  }
  cudaSetDevice(c->device);
  StreamScope scope_(c->stream);
  CTX_CUDA(c, cudaStreamSynchronize(c->stream), "set_condition");
  if (!c->fast || c->fast->set_condition(c, n_factors, factors) != 0)
    return fail(c, LMFAO_ERR_UNSUPPORTED, "the planned batch has no path condition the kernels can rebind "
                                         "(regression-tree batches whose products all carry the same predicates)");
  if (c->graph_exec) cudaGraphExecDestroy(c->graph_exec);  // the captured kernel arguments are stale
  c->graph_exec = nullptr;
  c->graph_runs = 0;
  for (auto& sc : c->secs)
    if (lmfao_status s = lmfao_set_condition(sc.ctx, n_factors, factors)) return relay(c, sc.ctx, s);
  return LMFAO_OK;
}

static lmfao_status run_local(lmfao_ctx* c, void* cuda_stream) {
  if (!c) return LMFAO_ERR_INVALID_ARG;
  if (c->state != S_PLANNED) return fail(c, LMFAO_ERR_STATE, "run needs plan");
  cudaSetDevice(c->device);
  StreamScope scope_(c->stream);
  cudaStream_t st = cuda_stream ? (cudaStream_t)cuda_stream : c->stream;
  if (c->comm)
    if (int e = c->comm->async_error())
      return fail(c, LMFAO_ERR_NCCL, "%s asynchronous error: %s", c->comm->backend(), c->comm->error_string(e).c_str());
  const char* ng = std::getenv("LMFAO_NO_GRAPH");
  // CUDA Graph: one capture of the whole run, NCCL collectives included (a loopback group
  // synchronises the host between phases and stays eager)
  bool use_graph = !c->prof && (c->world == 1 || c->comm->capturable()) && !(ng && ng[0] == '1') &&
                   !(c->fast && !c->fast->graph_ok());
  if (!use_graph || c->graph_runs == 0) {
    c->graph_runs++;
    return run_body(c, st);
  }
  if (!c->graph_exec) {
    cudaStream_t cs = c->stream;
    if (st != cs) {  // order the capture stream after the caller's work
      cudaEvent_t ev;
      CTX_CUDA(c, cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "graph");
      CTX_CUDA(c, cudaEventRecord(ev, st), "graph");
      CTX_CUDA(c, cudaStreamWaitEvent(cs, ev, 0), "graph");
      cudaEventDestroy(ev);
    }
    CTX_CUDA(c, cudaStreamSynchronize(cs), "graph");
    CTX_CUDA(c, cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal), "graph capture");
    lmfao_status s = run_body(c, cs);
    cudaGraph_t graph = nullptr;
    cudaError_t e = cudaStreamEndCapture(cs, &graph);
    if (s != LMFAO_OK) {
      if (graph) cudaGraphDestroy(graph);
      return s;
    }
    CTX_CUDA(c, e, "graph end capture");
    e = cudaGraphInstantiate(&c->graph_exec, graph, 0);
    cudaGraphDestroy(graph);
    CTX_CUDA(c, e, "graph instantiate");
    c->graph_launches = c->launches_last_run;
  }
  CTX_CUDA(c, cudaGraphLaunch(c->graph_exec, st), "graph launch");
  for (auto& gp : c->groups) gp.compacted = gp.gathered = false;
  c->launches_last_run = c->graph_launches;
  c->graph_runs++;
  return LMFAO_OK;
}

namespace {
lmfao_status ensure_compacted(lmfao_ctx* c, GroupPlan& gp) {
  if (gp.compacted) return LMFAO_OK;
  CTX_CUDA(c, cudaStreamSynchronize(c->stream), "sync");
  CTX_CUDA(c, cudaDeviceSynchronize(), "sync");
  if (c->comm)
    if (int e = c->comm->async_error())
      return fail(c, LMFAO_ERR_NCCL, "%s asynchronous error: %s", c->comm->backend(), c->comm->error_string(e).c_str());
  if (gp.direct) {  // written by a fast path; the group count on the device
    if (gp.ngroups_on_device) {
      unsigned long long n = 0;
      CTX_CUDA(c, cudaMemcpy(&n, gp.ngroups_dev.p, 8, cudaMemcpyDeviceToHost), "group count");
      gp.ngroups = (int64_t)n;
    }
    gp.compacted = true;
    return LMFAO_OK;
  }
  DecodeArgs d = gp.d;  // this rank's range of the cells (all of them unless distributed)
  d.cell0 = gp.cell_lo;
  const int64_t n = gp.cell_hi - gp.cell_lo;
  if (n <= 0) {
    gp.ngroups = 0;
  } else {
    CTX_CUDA(c, launch_compact(gp.table.as<double>() + gp.cell_lo * gp.nudaf, gp.counts.as<unsigned long long>() + gp.cell_lo,
                               n, gp.nudaf, d, gp.rkeys, gp.rvals, gp.rcnts, gp.ngroups, c->stream),
             "compaction");
  }
  gp.compacted = true;
  return LMFAO_OK;
}
}  // namespace

static lmfao_status result_shape_local(lmfao_ctx* c, int32_t q, int64_t* n_groups, int32_t* n_groupby,
                                           int32_t* n_udafs) {
  if (!c) return LMFAO_ERR_INVALID_ARG;
  if (c->state != S_PLANNED || !c->ran) return fail(c, LMFAO_ERR_STATE, "no results: run first");
  if (q < 0 || q >= (int)c->queries.size()) return fail(c, LMFAO_ERR_INVALID_ARG, "bad query id");
  cudaSetDevice(c->device);
  StreamScope scope_(c->stream);
  const Query& Q = c->queries[q];
  if (n_groupby) *n_groupby = (int)Q.gb.size();
  if (n_udafs) *n_udafs = (int)Q.udafs.size();
  if (c->query_kind[q] == 0) {
    if (n_groups) *n_groups = 1;
    return LMFAO_OK;
  }
  GroupPlan& gp = c->groups[c->query_slot[q]];
  lmfao_status s = ensure_compacted(c, gp);
  if (s != LMFAO_OK) return s;
  if (n_groups) *n_groups = gp.gathered ? gp.gngroups : gp.ngroups;
  return LMFAO_OK;
}

static lmfao_status result_device_local(lmfao_ctx* c, int32_t q, const int32_t** keys, const double** vals,
                                            const uint64_t** counts) {
  if (!c) return LMFAO_ERR_INVALID_ARG;
  if (c->state != S_PLANNED || !c->ran) return fail(c, LMFAO_ERR_STATE, "no results: run first");
  if (q < 0 || q >= (int)c->queries.size()) return fail(c, LMFAO_ERR_INVALID_ARG, "bad query id");
  cudaSetDevice(c->device);
  StreamScope scope_(c->stream);
  if (c->query_kind[q] == 0) {
    int off = c->scalar_off[c->query_slot[q]];
    if (keys) *keys = nullptr;
    if (vals) *vals = c->scalar_out.as<double>() + off;
    if (counts) *counts = (const uint64_t*)c->scalar_count.p;
    return LMFAO_OK;
  }
  GroupPlan& gp = c->groups[c->query_slot[q]];
  lmfao_status s = ensure_compacted(c, gp);
  if (s != LMFAO_OK) return s;
  if (keys) *keys = (gp.gathered ? gp.gkeys : gp.rkeys).as<int32_t>();
  if (vals) *vals = (gp.gathered ? gp.gvals : gp.rvals).as<double>();
  if (counts) *counts = (const uint64_t*)(gp.gathered ? gp.gcnts : gp.rcnts).p;
  return LMFAO_OK;
}

static lmfao_status fetch_local(lmfao_ctx* c, int32_t q, int32_t* keys_out, double* vals_out,
                                    uint64_t* counts_out) {
  int64_t ng = 0;
  int32_t ngb = 0, nu = 0;
  lmfao_status s = result_shape_local(c, q, &ng, &ngb, &nu);
  if (s != LMFAO_OK) return s;
  const int32_t* dk = nullptr;
  const double* dv = nullptr;
  const uint64_t* dc = nullptr;
  s = result_device_local(c, q, &dk, &dv, &dc);
  if (s != LMFAO_OK) return s;
  if (ng > 0 && nu > 0 && !vals_out) return fail(c, LMFAO_ERR_INVALID_ARG, "vals_out is NULL");
  if (ng > 0 && ngb > 0 && !keys_out) return fail(c, LMFAO_ERR_INVALID_ARG, "keys_out is NULL");
  cudaStream_t st = c->stream;
  CTX_CUDA(c, cudaDeviceSynchronize(), "fetch sync");
  if (ng > 0 && ngb > 0) CTX_CUDA(c, cudaMemcpyAsync(keys_out, dk, ng * ngb * 4, cudaMemcpyDeviceToHost, st), "fetch");
  if (ng > 0 && nu > 0) CTX_CUDA(c, cudaMemcpyAsync(vals_out, dv, ng * nu * 8, cudaMemcpyDeviceToHost, st), "fetch");
  if (ng > 0 && counts_out) CTX_CUDA(c, cudaMemcpyAsync(counts_out, dc, ng * 8, cudaMemcpyDeviceToHost, st), "fetch");
  CTX_CUDA(c, cudaStreamSynchronize(st), "fetch sync");
  return LMFAO_OK;
}

// Collective (every rank calls it with the same arguments).  A distributed output holds one
// range of cells per rank, the ranges ascending with the rank, so the full table in canonical
// order is the ranks' groups concatenated in rank order: every rank sends its compacted groups to
// root_rank (counts first, all-gathered), which keeps the result next to its own range.
static lmfao_status gather_local(lmfao_ctx* c, int32_t q, int32_t root_rank) {
  if (!c) return LMFAO_ERR_INVALID_ARG;
  if (c->state != S_PLANNED || !c->ran) return fail(c, LMFAO_ERR_STATE, "no results: run first");
  if (q < 0 || q >= (int)c->queries.size()) return fail(c, LMFAO_ERR_INVALID_ARG, "bad query id");
  if (root_rank < 0 || root_rank >= c->world) return fail(c, LMFAO_ERR_INVALID_ARG, "bad root rank");
  if (c->world == 1 || c->query_kind[q] == 0) return LMFAO_OK;  // complete on every rank
  cudaSetDevice(c->device);
  StreamScope scope_(c->stream);
  GroupPlan& gp = c->groups[c->query_slot[q]];
  if (!gp.dist && !gp.direct) return LMFAO_OK;  // all-reduced: complete on every rank
  lmfao_status s = ensure_compacted(c, gp);
  if (s != LMFAO_OK) return s;
  Comm& cm = *c->comm;
  cudaStream_t st = c->stream;
  const int G = c->world, ngb = gp.d.ngb, nu = gp.nudaf;
  DevBuf cnt;
  CTX_CUDA(c, cnt.alloc(8 * (G + 1)), "gather");
  unsigned long long mine = (unsigned long long)gp.ngroups;
  CTX_CUDA(c, cudaMemcpyAsync(cnt.as<unsigned long long>() + G, &mine, 8, cudaMemcpyHostToDevice, st), "gather");
  int e = cm.allgather(cnt.as<unsigned long long>() + G, cnt.p, 8, st);
  if (e) return fail(c, LMFAO_ERR_NCCL, "gather counts: %s", cm.error_string(e).c_str());
  std::vector<unsigned long long> n(G);
  CTX_CUDA(c, cudaMemcpyAsync(n.data(), cnt.p, 8 * G, cudaMemcpyDeviceToHost, st), "gather");
  CTX_CUDA(c, cudaStreamSynchronize(st), "gather");
  std::vector<int64_t> off(G + 1, 0);
  for (int r = 0; r < G; r++) off[r + 1] = off[r] + (int64_t)n[r];
  const int64_t tot = off[G];
  const bool root = c->rank == root_rank;
  if (root) {
    CTX_CUDA(c, gp.gkeys.alloc(std::max<int64_t>(tot * ngb * 4, 16)), "gather");
    CTX_CUDA(c, gp.gvals.alloc(std::max<int64_t>(tot * nu * 8, 16)), "gather");
    CTX_CUDA(c, gp.gcnts.alloc(std::max<int64_t>(tot * 8, 16)), "gather");
    const int64_t o = off[c->rank], m = (int64_t)n[c->rank];
    if (m > 0) {
      if (ngb) CTX_CUDA(c, cudaMemcpyAsync(gp.gkeys.as<int32_t>() + o * ngb, gp.rkeys.p, m * ngb * 4, cudaMemcpyDeviceToDevice, st), "gather");
      if (nu) CTX_CUDA(c, cudaMemcpyAsync(gp.gvals.as<double>() + o * nu, gp.rvals.p, m * nu * 8, cudaMemcpyDeviceToDevice, st), "gather");
      CTX_CUDA(c, cudaMemcpyAsync(gp.gcnts.as<unsigned long long>() + o, gp.rcnts.p, m * 8, cudaMemcpyDeviceToDevice, st), "gather");
    }
  }
  e = cm.group_start();
  for (int r = 0; r < G && !e; r++) {
    if (r == root_rank) continue;
    const int64_t m = (int64_t)n[r];
    if (root) {
      e = e ? e : cm.recv(gp.gkeys.as<int32_t>() + off[r] * ngb, m * ngb * 4, r, st);
      e = e ? e : cm.recv(gp.gvals.as<double>() + off[r] * nu, m * nu * 8, r, st);
      e = e ? e : cm.recv(gp.gcnts.as<unsigned long long>() + off[r], m * 8, r, st);
    } else if (r == c->rank) {
      e = e ? e : cm.send(gp.rkeys.p, m * ngb * 4, root_rank, st);
      e = e ? e : cm.send(gp.rvals.p, m * nu * 8, root_rank, st);
      e = e ? e : cm.send(gp.rcnts.p, m * 8, root_rank, st);
    }
  }
  const int e2 = cm.group_end(st);
  e = e ? e : e2;
  if (e) return fail(c, LMFAO_ERR_NCCL, "gather: %s", cm.error_string(e).c_str());
  CTX_CUDA(c, cudaStreamSynchronize(st), "gather");
  if (root) {
    gp.gngroups = tot;
    gp.gathered = true;
  }
  return LMFAO_OK;
}

// ---- public entry points over the multi-root query map (see lmfao_ctx::secs)
namespace {
lmfao_status resolve(lmfao_ctx* c, int32_t q, lmfao_ctx*& t, int32_t& lq) {
  if (q < 0 || q >= (int32_t)c->qmap.size()) return fail(c, LMFAO_ERR_INVALID_ARG, "bad query id");
  const auto& m = c->qmap[q];
  t = m.first < 0 ? c : c->secs[m.first].ctx;
  lq = m.second;
  return LMFAO_OK;
}
lmfao_status relay(lmfao_ctx* c, lmfao_ctx* t, lmfao_status s) {  // a secondary's error, reported on c
  if (s != LMFAO_OK && t != c) return fail(c, s, "at root %s: %s", t->rels[t->root].name.c_str(), t->err.c_str());
  return s;
}
}  // namespace

extern "C" lmfao_status lmfao_plan(lmfao_ctx* c) {
  if (!c) return LMFAO_ERR_INVALID_ARG;
  const lmfao_status s0 = plan_local(c);
  copies_wait(c);
  if (s0) return s0;
  for (auto& sc : c->secs)
    if (lmfao_status s = lmfao_plan(sc.ctx)) return relay(c, sc.ctx, s);
  return LMFAO_OK;
}

// The secondary roots run on their own streams, ordered after the caller's work and joined
// back before lmfao_run's work on `cuda_stream` completes (they overlap the main root's run).
extern "C" lmfao_status lmfao_run(lmfao_ctx* c, void* cuda_stream) {
  if (!c) return LMFAO_ERR_INVALID_ARG;
  if (c->secs.empty()) return run_local(c, cuda_stream);
  if (c->state != S_PLANNED) return fail(c, LMFAO_ERR_STATE, "run needs plan");
  cudaSetDevice(c->device);
  cudaStream_t st = cuda_stream ? (cudaStream_t)cuda_stream : c->stream;
  CTX_CUDA(c, cudaEventRecord(c->secs[0].ev_in, st), "run");
  for (auto& sc : c->secs) {
    CTX_CUDA(c, cudaStreamWaitEvent(sc.stream, c->secs[0].ev_in, 0), "run");
    if (lmfao_status s = lmfao_run(sc.ctx, sc.stream)) return relay(c, sc.ctx, s);
    cudaSetDevice(c->device);
    CTX_CUDA(c, cudaEventRecord(sc.ev_out, sc.stream), "run");
  }
  if (!c->queries.empty())
    if (lmfao_status s = run_local(c, cuda_stream)) return s;
  for (auto& sc : c->secs) CTX_CUDA(c, cudaStreamWaitEvent(st, sc.ev_out, 0), "run");
  c->ran = true;
  return LMFAO_OK;
}

extern "C" lmfao_status lmfao_result_shape(lmfao_ctx* c, int32_t q, int64_t* n_groups, int32_t* n_groupby,
                                           int32_t* n_udafs) {
  if (!c) return LMFAO_ERR_INVALID_ARG;
  lmfao_ctx* t;
  int32_t lq;
  if (lmfao_status s = resolve(c, q, t, lq)) return s;
  return relay(c, t, result_shape_local(t, lq, n_groups, n_groupby, n_udafs));
}
extern "C" lmfao_status lmfao_result_device(lmfao_ctx* c, int32_t q, const int32_t** keys, const double** vals,
                                            const uint64_t** counts) {
  if (!c) return LMFAO_ERR_INVALID_ARG;
  lmfao_ctx* t;
  int32_t lq;
  if (lmfao_status s = resolve(c, q, t, lq)) return s;
  return relay(c, t, result_device_local(t, lq, keys, vals, counts));
}
extern "C" lmfao_status lmfao_fetch(lmfao_ctx* c, int32_t q, int32_t* keys_out, double* vals_out,
                                    uint64_t* counts_out) {
  if (!c) return LMFAO_ERR_INVALID_ARG;
  lmfao_ctx* t;
  int32_t lq;
  if (lmfao_status s = resolve(c, q, t, lq)) return s;
  return relay(c, t, fetch_local(t, lq, keys_out, vals_out, counts_out));
}
extern "C" lmfao_status lmfao_gather_result(lmfao_ctx* c, int32_t q, int32_t root_rank) {
  if (!c) return LMFAO_ERR_INVALID_ARG;
  lmfao_ctx* t;
  int32_t lq;
  if (lmfao_status s = resolve(c, q, t, lq)) return s;
  return relay(c, t, gather_local(t, lq, root_rank));
}

extern "C" lmfao_status lmfao_plan_info(lmfao_ctx* c, char* out, int64_t cap) {
  if (!c || !out || cap <= 0) return LMFAO_ERR_INVALID_ARG;
  if (c->state != S_PLANNED) return fail(c, LMFAO_ERR_STATE, "plan_info needs plan");
  std::ostringstream o;
  o << "{\"root\": \"" << c->rels[c->root].name << "\", \"root_rows\": " << c->rels[c->root].nrows;
  o << ", \"levels\": [";
  for (size_t i = 0; i < c->levels.size(); i++) {
    const Rel& ch = c->rels[c->rels[c->root].children[c->levels[i]]];
    o << (i ? ", " : "") << "{\"rel\": \"" << ch.name << "\", \"nkeys\": " << ch.nkeys << "}";
  }
  o << "], \"views\": [";
  bool first = true;
  for (int u : c->postorder) {
    o << (first ? "" : ", ") << "{\"rel\": \"" << c->rels[u].name << "\", \"width\": " << c->nodes[u].slots.size()
      << ", \"rows\": " << c->rels[u].nrows << ", \"nkeys\": " << c->rels[u].nkeys << "}";
    first = false;
  }
  o << "], \"scalar_outputs\": " << c->scalar_prog.nout << ", \"group_queries\": " << c->groups.size();
  o << ", \"fast_path\": " << (c->fast ? c->fast->describe() : std::string("null"));
  o << ", \"launches_last_run\": " << c->launches_last_run;
  o << ", \"world\": " << c->world << ", \"rank\": " << c->rank
    << ", \"comm\": \"" << (c->comm ? c->comm->backend() : "none") << "\", \"outputs\": [";
  for (size_t pq = 0; pq < c->qmap.size(); pq++) {  // where each query's result lives
    const lmfao_ctx* t = c->qmap[pq].first < 0 ? c : c->secs[c->qmap[pq].first].ctx;
    const int q = c->qmap[pq].second;
    const char* where = "replicated";
    int64_t lo = 0, hi = 1;
    if (t->query_kind[q] == 1) {
      const GroupPlan& gp = t->groups[t->query_slot[q]];
      hi = gp.ncells;
      if (t->world > 1 && gp.direct) where = "exchanged", lo = gp.cell_lo, hi = gp.cell_hi;
      else if (gp.dist) where = "reduce_scattered", lo = gp.cell_lo, hi = gp.cell_hi;
    }
    o << (pq ? ", " : "") << "{\"placement\": \"" << where << "\", \"cells\": [" << lo << ", " << hi
      << "], \"root\": \"" << t->rels[t->root].name << "\"}";
  }
  o << "], \"roots\": [\"" << c->rels[c->root].name << "\"";
  for (auto& sc : c->secs) o << ", \"" << c->rels[sc.root].name << "\"";
  o << "]";
  if (c->coll_n > 0) {  // profiled multi-GPU runs: the collectives of the partial results
    int64_t bytes = c->scalar_queries.empty() ? 0 : (int64_t)c->scalar_prog.nout * 8 + 8;
    for (auto& gp : c->groups)
      if (!gp.direct) bytes += gp.ncells_alloc * (gp.nudaf * 8 + 8);
    o << ", \"collective_ms\": " << c->coll_ms / c->coll_n << ", \"collective_bytes\": " << bytes;
  }
  o << "}";
  std::string s = o.str();
  if ((int64_t)s.size() + 1 > cap) return fail(c, LMFAO_ERR_INVALID_ARG, "plan_info buffer too small");
  std::memcpy(out, s.c_str(), s.size() + 1);
  return LMFAO_OK;
}

namespace lmfao {
void scan_timer_begin(lmfao_ctx* c, cudaStream_t st) {
  if (!c->prof) return;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a, st);
  c->prof_events.push_back({a, b});
}
void scan_timer_end(lmfao_ctx* c, cudaStream_t st) {
  if (!c->prof || c->prof_events.empty()) return;
  cudaEventRecord(c->prof_events.back().second, st);
}
}  // namespace lmfao

extern "C" lmfao_status lmfao_profile(lmfao_ctx* c, int enable) {
  if (!c) return LMFAO_ERR_INVALID_ARG;
  cudaSetDevice(c->device);
  StreamScope scope_(c->stream);
  for (auto& e : c->prof_events) {
    cudaEventDestroy(e.first);
    cudaEventDestroy(e.second);
  }
  c->prof_events.clear();
  for (auto& e : c->coll_events) {
    cudaEventDestroy(e.first);
    cudaEventDestroy(e.second);
  }
  c->coll_events.clear();
  if (enable) c->coll_ms = 0.0, c->coll_n = 0;
  c->prof = enable != 0;
  return LMFAO_OK;
}

extern "C" lmfao_status lmfao_profile_read(lmfao_ctx* c, double* total_ms, int64_t* launches) {
  if (!c || !total_ms || !launches) return LMFAO_ERR_INVALID_ARG;
  cudaSetDevice(c->device);
  StreamScope scope_(c->stream);
  double t = 0;
  for (auto& e : c->prof_events) {
    if (cudaEventSynchronize(e.second) != cudaSuccess) return fail(c, LMFAO_ERR_CUDA, "profile: event sync failed");
    float ms = 0;
    cudaEventElapsedTime(&ms, e.first, e.second);
    t += ms;
  }
  *total_ms = t;
  *launches = (int64_t)c->prof_events.size();
  for (auto& e : c->coll_events) {  // the collectives of the same runs
    if (cudaEventSynchronize(e.second) != cudaSuccess) return fail(c, LMFAO_ERR_CUDA, "profile: event sync failed");
    float ms = 0;
    cudaEventElapsedTime(&ms, e.first, e.second);
    c->coll_ms += ms;
    c->coll_n++;
    cudaEventDestroy(e.first);
    cudaEventDestroy(e.second);
  }
  c->coll_events.clear();
  return LMFAO_OK;
}
