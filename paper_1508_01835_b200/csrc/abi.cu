// C ABI (include/ifmm_b200.h): exception-to-status translation and handle
// plumbing.  No computation here beyond argument checks.
#include <cstdio>
#include <cstring>

#include "../../include/ifmm_b200.h"
#include "engine.h"

using namespace ifmm;

namespace ifmm {
const char* last_error_cstr();
extern double g_prof[];
}

#define ABI_TRY try {
#define ABI_CATCH                                        \
  }                                                      \
  catch (const ifmm::Error& e) {                         \
    set_last_error(e.what());                            \
    return e.code;                                       \
  }                                                      \
  catch (const std::exception& e) {                      \
    set_last_error(std::string("internal: ") + e.what()); \
    return E_ASSERT;                                     \
  }
#define ABI_CATCH_NULL                                   \
  }                                                      \
  catch (const ifmm::Error& e) {                         \
    set_last_error(e.what());                            \
    return nullptr;                                      \
  }                                                      \
  catch (const std::exception& e) {                      \
    set_last_error(std::string("internal: ") + e.what()); \
    return nullptr;                                      \
  }

extern "C" {

int ifmm_abi_version(void) { return 1; }
const char* ifmm_last_error(void) { return last_error_cstr(); }

void* ifmm_ctx_create(int device, unsigned long long arena_bytes) {
  ABI_TRY
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    throw Error(E_CUDA, "no CUDA device available (the IFMM engine has no CPU fallback)");
  CUDA_CHECK(cudaSetDevice(device));
  Ctx* c = new Ctx;
  c->device = device;
  CUDA_CHECK(cudaStreamCreateWithFlags(&c->st, cudaStreamNonBlocking));
  CUDA_CHECK(cudaStreamCreateWithFlags(&c->st2, cudaStreamNonBlocking));
  CUDA_CHECK(cudaStreamCreateWithFlags(&c->st3, cudaStreamNonBlocking));
  CUDA_CHECK(cudaEventCreateWithFlags(&c->side_ev, cudaEventDisableTiming));
  CUDA_CHECK(cudaEventCreateWithFlags(&c->side_done, cudaEventDisableTiming));
  CUDA_CHECK(cudaEventCreateWithFlags(&c->fork_ev, cudaEventDisableTiming));
  CUDA_CHECK(cudaEventCreateWithFlags(&c->join_ev, cudaEventDisableTiming));
  if (arena_bytes == 0) {
    size_t fr = 0, tot = 0;
    CUDA_CHECK(cudaMemGetInfo(&fr, &tot));
    arena_bytes = (unsigned long long)(fr * 0.85);
  }
  c->arena.init(arena_bytes);
  c->stage.init((size_t)256 << 20);
  CUDA_CHECK(cudaMalloc(&c->d_status, 16));
  CUDA_CHECK(cudaMemset(c->d_status, 0, 16));
  return c;
  ABI_CATCH_NULL
}

void ifmm_ctx_destroy(void* p) {
  if (!p) return;
  Ctx* c = (Ctx*)p;
  cudaStreamSynchronize(c->st);
  c->arena.release();
  c->stage.release();
  if (c->d_status) cudaFree(c->d_status);
  if (c->h_pinned_i) cudaFreeHost(c->h_pinned_i);
  cudaStreamDestroy(c->st2);
  cudaStreamDestroy(c->st3);
  cudaEventDestroy(c->side_ev);
  cudaEventDestroy(c->side_done);
  cudaStreamDestroy(c->st);
  delete c;
}

int ifmm_ctx_memory(void* p, unsigned long long* in_use, unsigned long long* peak) {
  Ctx* c = (Ctx*)p;
  *in_use = c->arena.in_use();
  *peak = c->arena.peak();
  return 0;
}

// ---- tree -------------------------------------------------------------------
void* ifmm_tree_create(void* ctx, int n_points, const double* points, const int* perm, int depth,
                       int n_clusters, const int* level, const int* parent, const int* start,
                       const int* stop, const long long* cell, const double* center,
                       const double* half_width, const int* child_ptr, const int* child_idx) {
  ABI_TRY
  // ctx == NULL: host-only tree (topology queries, no device upload)
  Ctx* Cp = (Ctx*)ctx;
  if (n_points <= 0) throw Error(E_VALUE, "points must be non-empty");
  Tree* t = new Tree;
  t->ctx = Cp;
  t->n_points = n_points;
  t->depth = depth;
  t->nc = n_clusters;
  t->points.assign(points, points + 3 * (size_t)n_points);
  t->perm.assign(perm, perm + n_points);
  t->level.assign(level, level + n_clusters);
  t->parent.assign(parent, parent + n_clusters);
  t->start.assign(start, start + n_clusters);
  t->stop.assign(stop, stop + n_clusters);
  t->cell.assign(cell, cell + 3 * (size_t)n_clusters);
  t->center.assign(center, center + 3 * (size_t)n_clusters);
  t->hw.assign(half_width, half_width + n_clusters);
  t->children.assign(n_clusters, {});
  for (int c = 0; c < n_clusters; ++c)
    t->children[c].assign(child_idx + child_ptr[c], child_idx + child_ptr[c + 1]);
  t->levels.assign(depth + 1, {});
  for (int c = 0; c < n_clusters; ++c) {
    if (level[c] < 0 || level[c] > depth) throw Error(E_VALUE, "cluster level out of range");
    t->levels[level[c]].push_back(c);
  }
  // ids within a level are Morton ordered by construction (tree.py:158-193)
  t->build_topology();
  if (Cp) {
    t->d_points = Cp->arena.alloc(3 * (size_t)n_points, &t->d_points_cls);
    CUDA_CHECK(cudaMemcpy(t->d_points, points, sizeof(double) * 3 * n_points, cudaMemcpyHostToDevice));
    t->d_perm = Cp->arena.alloc_int(n_points, &t->d_perm_cls);
    CUDA_CHECK(cudaMemcpy(t->d_perm, perm, sizeof(int) * n_points, cudaMemcpyHostToDevice));
  }
  return t;
  ABI_CATCH_NULL
}

void ifmm_tree_destroy(void* p) {
  if (!p) return;
  Tree* t = (Tree*)p;
  if (t->ctx) {
    t->ctx->sync_nothrow();
    t->ctx->free_raw(t->d_points, t->d_points_cls);
    t->ctx->free_raw(t->d_perm, t->d_perm_cls);
    t->ctx->flush();
  }
  delete t;
}

int ifmm_tree_topology_sizes(void* p, long long* nn, long long* ni) {
  Tree* t = (Tree*)p;
  long long a = 0, b = 0;
  for (int c = 0; c < t->nc; ++c) { a += t->nbrs[c].size(); b += t->inters[c].size(); }
  *nn = a; *ni = b;
  return 0;
}

int ifmm_tree_topology(void* p, long long* nbr_ptr, int* nbr_idx, long long* int_ptr,
                       int* int_idx) {
  Tree* t = (Tree*)p;
  long long a = 0, b = 0;
  for (int c = 0; c < t->nc; ++c) {
    nbr_ptr[c] = a; int_ptr[c] = b;
    for (int q : t->nbrs[c]) nbr_idx[a++] = q;
    for (int q : t->inters[c]) int_idx[b++] = q;
  }
  nbr_ptr[t->nc] = a; int_ptr[t->nc] = b;
  return 0;
}

// ---- H2 ---------------------------------------------------------------------
void* ifmm_h2_build(void* tree, int kernel_kind, double p0, int n_cheb, double epsilon) {
  return ifmm_h2_build_k(tree, kernel_kind, p0, 0.0, n_cheb, epsilon);
}

void* ifmm_h2_build_k(void* tree, int kernel_kind, double p0, double p1, int n_cheb,
                      double epsilon) {
  ABI_TRY
  Tree* t = (Tree*)tree;
  if (!t->ctx) throw Error(E_CUDA, "tree has no device context");
  if (n_cheb < 1) throw Error(E_VALUE, "n must be >= 1");
  if (n_cheb > MAX_CHEB) throw Error(E_VALUE, "n_cheb too large");
  if (kernel_kind < 1 || kernel_kind > KERNEL_KIND_MAX) throw Error(E_VALUE, "unknown kernel kind");
  H2* h = new H2;
  h->ctx = t->ctx;
  h->tree = t;
  h->kern.kind = kernel_kind;
  h->kern.p0 = p0;
  h->kern.p1 = p1;
  h->ncheb = n_cheb;
  h->eps = epsilon;
  try {
    h->build();
  } catch (...) {
    delete h;
    throw;
  }
  return h;
  ABI_CATCH_NULL
}

void ifmm_h2_destroy(void* p) {
  if (!p) return;
  H2* h = (H2*)p;
  h->ctx->sync_nothrow();
  delete h;
}

int ifmm_h2_ranks(void* p, int* out) {
  H2* h = (H2*)p;
  for (int c = 0; c < h->tree->nc; ++c) out[c] = h->rank[c];
  return 0;
}

int ifmm_h2_weights(void* p) {
  ABI_TRY
  if (((H2*)p)->consumed) throw Error(E_VALUE, "operators were consumed by a graph");
  ((H2*)p)->weights();
  return 0;
  ABI_CATCH
}

int ifmm_h2_weights_sampled(void* p, const long long* sample_ptr, const int* sample_idx) {
  ABI_TRY
  if (((H2*)p)->consumed) throw Error(E_VALUE, "operators were consumed by a graph");
  if (!sample_ptr || !sample_idx) throw Error(E_VALUE, "sample lists missing");
  ((H2*)p)->weights(sample_ptr, sample_idx);
  return 0;
  ABI_CATCH
}

int ifmm_h2_block(void* p, int which, int i, int j, double* out, int* rows, int* cols) {
  ABI_TRY
  H2* h = (H2*)p;
  const int nc = h->tree->nc;
  if (i < 0 || i >= nc || ((which == 4 || which == 5) && (j < 0 || j >= nc)))
    throw Error(E_VALUE, "cluster id out of range");
  const Blk* b = nullptr;
  switch (which) {
    case 0: b = &h->leaf_u[i]; break;
    case 1: b = &h->leaf_v[i]; break;
    case 2: b = &h->tu[i]; break;
    case 3: b = &h->tvt[i]; break;
    case 4: { auto it = h->coupling.find(key2(i, j)); if (it != h->coupling.end()) b = &it->second; break; }
    case 5: { auto it = h->near.find(key2(i, j)); if (it != h->near.end()) b = &it->second; break; }
    case 6: b = &h->su[i]; break;
    case 7: b = &h->sv[i]; break;
    default: throw Error(E_VALUE, "bad block selector");
  }
  if (!b || !b->p) { *rows = -1; *cols = -1; return 0; }
  *rows = b->r; *cols = b->c;
  if (out) {
    h->ctx->sync();
    CUDA_CHECK(cudaMemcpy(out, b->p, sizeof(double) * b->r * b->c, cudaMemcpyDeviceToHost));
  }
  return 0;
  ABI_CATCH
}

// gather/scatter by the tree permutation on device
namespace {
__global__ void k_gather(const double* in, const int* perm, int n, int bd, double* out) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = in[(size_t)perm[i / bd] * bd + i % bd];
}
__global__ void k_scatter(const double* in, const int* perm, int n, int bd, double* out) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[(size_t)perm[i / bd] * bd + i % bd] = in[i];
}
}  // namespace

int ifmm_h2_matvec(void* p, const double* x, double* y, int on_device) {
  ABI_TRY
  H2* h = (H2*)p;
  if (h->consumed) throw Error(E_VALUE, "operators were consumed by a graph");
  Ctx& C = *h->ctx;
  const int bd = h->kern.bd();
  const int N = bd * h->tree->n_points;
  Blk xin = C.alloc(1, N), xs = C.alloc(1, N), ys = C.alloc(1, N), yo = C.alloc(1, N);
  if (on_device) CUDA_CHECK(cudaMemcpyAsync(xin.p, x, 8 * (size_t)N, cudaMemcpyDeviceToDevice, C.st));
  else CUDA_CHECK(cudaMemcpyAsync(xin.p, x, 8 * (size_t)N, cudaMemcpyHostToDevice, C.st));
  k_gather<<<(N + 255) / 256, 256, 0, C.st>>>(xin.p, h->tree->d_perm, N, bd, xs.p);
  h->matvec(xs.p, ys.p);
  k_scatter<<<(N + 255) / 256, 256, 0, C.st>>>(ys.p, h->tree->d_perm, N, bd, yo.p);
  if (on_device) CUDA_CHECK(cudaMemcpyAsync(y, yo.p, 8 * (size_t)N, cudaMemcpyDeviceToDevice, C.st));
  else CUDA_CHECK(cudaMemcpyAsync(y, yo.p, 8 * (size_t)N, cudaMemcpyDeviceToHost, C.st));
  C.sync();
  for (Blk* b : {&xin, &xs, &ys, &yo}) C.free(*b);
  C.flush();
  return 0;
  ABI_CATCH
}

// Morton-range partitioned h2_matvec: one rank's share, device
// pointers in tree (sorted) order; see H2::matvec_part.
int ifmm_h2_multipole_size(void* p, long long* out) {
  ABI_TRY
  *out = ((H2*)p)->multipole_size();
  return 0;
  ABI_CATCH
}

int ifmm_h2_matvec_part(void* p, const double* xs, double* ys, double* yv, int phase, long long p_lo,
                        long long p_hi) {
  ABI_TRY
  H2* h = (H2*)p;
  if (h->consumed) throw Error(E_VALUE, "operators were consumed by a graph");
  if (phase != 0 && phase != 1) throw Error(E_VALUE, "phase must be 0 or 1");
  if (p_lo < 0 || p_hi > h->tree->n_points || p_lo > p_hi) throw Error(E_VALUE, "bad point range");
  h->matvec_part(xs, ys, yv, phase, p_lo, p_hi);
  h->ctx->sync();
  return 0;
  ABI_CATCH
}

// ---- graph ------------------------------------------------------------------
void* ifmm_graph_build(void* h2, int consume) {
  ABI_TRY
  H2* h = (H2*)h2;
  if (h->consumed) throw Error(E_VALUE, "operators were consumed by an earlier graph");
  if (h->tree->depth >= 2 && !h->weighted)
    throw Error(E_VALUE, "operators have no basis weights; run initialize_weights first");
  Graph* g = new Graph;
  g->ctx = h->ctx;
  try {
    g->build(h, consume != 0);
  } catch (...) {
    delete g;
    throw;
  }
  return g;
  ABI_CATCH_NULL
}

void ifmm_graph_destroy(void* p) {
  if (!p) return;
  Graph* g = (Graph*)p;
  g->ctx->sync_nothrow();
  delete g;
}

int ifmm_graph_info(void* p, long long* dim, long long* nn, long long* ne) {
  Graph* g = (Graph*)p;
  *dim = g->dim();
  *nn = (long long)g->size.size();
  *ne = (long long)g->E.size();
  return 0;
}

// ---- read-only graph view (graph.py:30-216 attributes) ------------------------
int ifmm_graph_nodes(void* p, int* size, int* kind, int* owner) {
  Graph* g = (Graph*)p;
  for (size_t i = 0; i < g->size.size(); ++i) {
    if (size) size[i] = g->size[i];
    if (kind) kind[i] = g->kind[i];
    if (owner) owner[i] = g->owner[i];
  }
  return 0;
}

int ifmm_graph_cluster_nodes(void* p, int* nx, int* nz, int* ny) {
  Graph* g = (Graph*)p;
  for (size_t c = 0; c < g->nx.size(); ++c) {
    nx[c] = g->nx[c]; nz[c] = g->nz[c]; ny[c] = g->ny[c];
  }
  return 0;
}

int ifmm_graph_edges(void* p, int* t, int* s, long long* peak_edges) {
  Graph* g = (Graph*)p;
  std::vector<uint64_t> keys;
  keys.reserve(g->E.size());
  for (auto& kv : g->E) keys.push_back(kv.first);
  std::sort(keys.begin(), keys.end());
  for (size_t i = 0; i < keys.size(); ++i) {
    t[i] = (int)(keys[i] >> 32);
    s[i] = (int)(keys[i] & 0xffffffffu);
  }
  if (peak_edges) *peak_edges = g->peak_edges;
  return 0;
}

int ifmm_graph_block(void* p, int t, int s, double* out, int* r, int* c) {
  ABI_TRY
  Graph* g = (Graph*)p;
  if (g->consumed) throw Error(E_VALUE, "graph already factorized");
  Blk* b = g->get(t, s);
  if (!b) { *r = -1; *c = -1; return 0; }
  *r = b->r; *c = b->c;
  if (out && b->r * b->c > 0) {
    CUDA_CHECK(cudaMemcpyAsync(out, b->p, 8 * (size_t)b->r * b->c, cudaMemcpyDeviceToHost,
                               g->ctx->st));
    g->ctx->sync();
  }
  return 0;
  ABI_CATCH
}

void* ifmm_graph_copy(void* p) {
  ABI_TRY
  Graph* g = (Graph*)p;
  if (g->consumed) throw Error(E_VALUE, "graph already factorized");
  return g->clone();
  ABI_CATCH_NULL
}

int ifmm_graph_apply(void* p, const double* in, double* out, int transpose, int on_device) {
  ABI_TRY
  Graph* g = (Graph*)p;
  if (g->consumed) throw Error(E_VALUE, "graph already factorized");
  Ctx& C = *g->ctx;
  const long long dim = g->dim();
  Blk I = C.alloc(1, (int)std::max<long long>(dim, 1)), O = C.alloc(1, (int)std::max<long long>(dim, 1));
  const cudaMemcpyKind kin = on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
  const cudaMemcpyKind kout = on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
  CUDA_CHECK(cudaMemcpyAsync(I.p, in, 8 * (size_t)dim, kin, C.st));
  g->apply(I.p, O.p, transpose != 0);
  CUDA_CHECK(cudaMemcpyAsync(out, O.p, 8 * (size_t)dim, kout, C.st));
  C.sync();
  C.free(I); C.free(O);
  C.flush();
  return 0;
  ABI_CATCH
}

int ifmm_graph_sigma0(void* p, const double* omega, int width, int power_iters, double* out) {
  ABI_TRY
  Graph* g = (Graph*)p;
  if (g->consumed) throw Error(E_VALUE, "graph already factorized");
  *out = g->sigma0(omega, width, power_iters);
  return 0;
  ABI_CATCH
}

// ---- factorize / solve --------------------------------------------------------
void* ifmm_factorize(void* graph, double epsilon, double sigma0, int flags) {
  ABI_TRY
  return factorize((Graph*)graph, epsilon, sigma0, flags);
  ABI_CATCH_NULL
}

void* ifmm_factorize_pcg64(void* graph, double epsilon, double sigma0, int flags,
                           const unsigned long long* pcg_state) {
  ABI_TRY
  uint64_t st[4] = {pcg_state[0], pcg_state[1], pcg_state[2], pcg_state[3]};
  return factorize_pcg64((Graph*)graph, epsilon, sigma0, flags, st);
  ABI_CATCH_NULL
}

int ifmm_pcg64_normals(const unsigned long long* pcg_state, long long n, double* out) {
  ABI_TRY
  uint64_t st[4] = {pcg_state[0], pcg_state[1], pcg_state[2], pcg_state[3]};
  return pcg64_normals(st, n, out);
  ABI_CATCH
}

void* ifmm_factorize_rng(void* graph, double epsilon, double sigma0, int flags,
                         ifmm_normal_source src, void* user) {
  ABI_TRY
  return factorize((Graph*)graph, epsilon, sigma0, flags, src, user);
  ABI_CATCH_NULL
}

void ifmm_factor_destroy(void* p) {
  if (!p) return;
  Factor* f = (Factor*)p;
  f->ctx->sync_nothrow();
  delete f;
}

int ifmm_factor_stats(void* p, long long* out, int n) {
  Factor* f = (Factor*)p;
  long long ne = 0, nr = 0, nm = 0;
  for (auto& e : f->events) { if (e.type == 0) ne++; else if (e.type == 1) nr++; else nm++; }
  long long mfr = 0, forced = 0;
  for (auto& l : f->levels) {
    for (int r : l.ranks) mfr = std::max<long long>(mfr, r);
    forced += l.forced;
  }
  long long topdim = 0;
  for (int s : f->top_sizes) topdim += s;
  long long v[11] = {f->peak_edges, f->n_clusters, f->max_basis_rank, mfr, forced,
                     (long long)f->levels.size(), ne, nr, nm, (long long)f->top_nodes.size(),
                     topdim};
  for (int i = 0; i < n && i < 11; ++i) out[i] = v[i];
  return 0;
}

int ifmm_factor_level_stats(void* p, long long* out, int n) {
  Factor* f = (Factor*)p;
  for (int i = 0; i < n && i < (int)f->levels.size(); ++i) {
    const LevelStats& l = f->levels[i];
    long long s = 0, mx = 0;
    for (int r : l.ranks) { s += r; mx = std::max<long long>(mx, r); }
    long long v[8] = {l.level, l.compressed, l.added, l.dropped, s, mx, (long long)l.ranks.size(),
                      l.forced};
    for (int j = 0; j < 8; ++j) out[8 * i + j] = v[j];
  }
  return 0;
}

int ifmm_factor_level_ranks(void* p, int li, int* out) {
  Factor* f = (Factor*)p;
  if (li < 0 || li >= (int)f->levels.size()) return E_VALUE;
  const auto& r = f->levels[li].ranks;
  for (size_t i = 0; i < r.size(); ++i) out[i] = r[i];
  return 0;
}

int ifmm_factor_timings(void* p, double* out, int n) {
  Factor* f = (Factor*)p;
  double v[9] = {f->t_lu, f->t_mm, f->t_lr, f->t_tr, f->t_total, f->gemm_flops, f->all_flops,
                 (double)f->rsvd_rounds, (double)f->rsvd_redraws};
  for (int i = 0; i < n && i < 9; ++i) out[i] = v[i];
  return 0;
}

// Event log and layout (factor.py:77-92): flat int64 records.  Returns the
// number of int64 written (or needed when out is NULL / cap too small).
// elim:   0, nx, nz, ny, size_x, size_z, n_src, n_tgt, src..., tgt...
// rebase: 1, ny
// merge:  2, px, n_parts, (child y, size)...
long long ifmm_factor_events(void* p, long long* out, long long cap) {
  Factor* f = (Factor*)p;
  std::vector<long long> v;
  for (auto& e : f->events) {
    if (e.type == 0) {
      const ElimEv& x = f->elims[e.idx];
      v.insert(v.end(), {0, x.nx, x.nz, x.ny, x.m, x.k, (long long)x.src.size(),
                         (long long)x.tgt.size()});
      v.insert(v.end(), x.src.begin(), x.src.end());
      v.insert(v.end(), x.tgt.begin(), x.tgt.end());
    } else if (e.type == 1) {
      v.insert(v.end(), {1, f->rebases[e.idx].ny});
    } else {
      const MergeEv& m = f->merges[e.idx];
      v.insert(v.end(), {2, m.px, (long long)m.parts.size()});
      for (size_t i = 0; i < m.parts.size(); ++i) v.insert(v.end(), {m.parts[i], m.psize[i]});
    }
  }
  if (out && cap >= (long long)v.size()) std::copy(v.begin(), v.end(), out);
  return (long long)v.size();
}

// top_nodes, top_sizes (n_top each), init_sizes (n_init), leaf x nodes /
// point start / stop (n_leaves each).  sizes: out[0..2] = n_top, n_init,
// n_leaves when the arrays are NULL.
int ifmm_factor_layout(void* p, int* sizes, int* top_nodes, int* top_sizes, int* init_sizes,
                       int* leaf_nodes, int* leaf_start, int* leaf_stop) {
  Factor* f = (Factor*)p;
  if (sizes) {
    sizes[0] = (int)f->top_nodes.size();
    sizes[1] = (int)f->init_sizes.size();
    sizes[2] = (int)f->leaf_nodes.size();
  }
  if (top_nodes) std::copy(f->top_nodes.begin(), f->top_nodes.end(), top_nodes);
  if (top_sizes) std::copy(f->top_sizes.begin(), f->top_sizes.end(), top_sizes);
  if (init_sizes) std::copy(f->init_sizes.begin(), f->init_sizes.end(), init_sizes);
  if (leaf_nodes) std::copy(f->leaf_nodes.begin(), f->leaf_nodes.end(), leaf_nodes);
  if (leaf_start) std::copy(f->leaf_start.begin(), f->leaf_start.end(), leaf_start);
  if (leaf_stop) std::copy(f->leaf_stop.begin(), f->leaf_stop.end(), leaf_stop);
  return 0;
}

int ifmm_factor_level_times(void* p, double* out, int n) {
  Factor* f = (Factor*)p;
  for (int i = 0; i < n && i < (int)f->levels.size(); ++i) out[i] = f->levels[i].compress_time;
  return 0;
}

int ifmm_ctx_event(void* ctx, int slot) {
  ABI_TRY
  Ctx& C = *(Ctx*)ctx;
  if (slot < 0 || slot >= 64) throw Error(E_VALUE, "event slot out of range");
  if (!C.ev[slot]) CUDA_CHECK(cudaEventCreate(&C.ev[slot]));
  CUDA_CHECK(cudaEventRecord(C.ev[slot], C.st));
  return 0;
  ABI_CATCH
}

int ifmm_ctx_elapsed(void* ctx, int a, int b, double* ms) {
  ABI_TRY
  Ctx& C = *(Ctx*)ctx;
  CUDA_CHECK(cudaEventSynchronize(C.ev[b]));
  float f = 0.f;
  CUDA_CHECK(cudaEventElapsedTime(&f, C.ev[a], C.ev[b]));
  *ms = f;
  return 0;
  ABI_CATCH
}

long long ifmm_ctx_launches(void* ctx) { return ((Ctx*)ctx)->launches; }

int ifmm_ktime(void* ctx, int enable, double* time_s, double* work, long long* count, int n) {
  Ctx& C = *(Ctx*)ctx;
  C.kt_collect();
  for (int i = 0; i < n && i < 16; ++i) {
    if (time_s) time_s[i] = C.ktime[i];
    if (work) work[i] = C.kwork[i];
    if (count) count[i] = C.kcount[i];
  }
  if (enable >= 0) {
    C.ktime_on = enable != 0;
    for (int i = 0; i < 16; ++i) { C.ktime[i] = 0; C.kwork[i] = 0; C.kcount[i] = 0; }
  }
  return 0;
}

int ifmm_dev_jacobi_bench(void* ctx, int s, const double* A, int reps, int threads,
                          unsigned long long* out) {
  ABI_TRY
  Ctx& C = *(Ctx*)ctx;
  Blk o = C.alloc(1, 2);
  ifmm::jacobi_bench(A, s, reps, threads, reinterpret_cast<unsigned long long*>(o.p), C.st);
  CUDA_CHECK(cudaGetLastError());
  CUDA_CHECK(cudaMemcpyAsync(out, o.p, 16, cudaMemcpyDeviceToHost, C.st));
  C.sync();
  C.free(o);
  C.flush();
  return 0;
  ABI_CATCH
}

int ifmm_union_profile(unsigned long long* out, int reset) {
  ifmm::union_profile(out, reset);
  return 0;
}

int ifmm_union_post_profile(unsigned long long* out, int reset) {
  ifmm::union_post_profile(out, reset);
  return 0;
}

int ifmm_profile(double* out, int n) {
  for (int i = 0; i < n && i < 12; ++i) out[i] = ifmm::g_prof[i];
  return 0;
}

int ifmm_solve(void* p, const double* b, double* x, int on_device) {
  ABI_TRY
  Factor* f = (Factor*)p;
  Ctx& C = *f->ctx;
  const int N = f->n_points;
  if (on_device) {
    f->solve(b, x);
    C.sync();
  } else {
    Blk bi = C.alloc(1, N), xo = C.alloc(1, N);
    CUDA_CHECK(cudaMemcpyAsync(bi.p, b, 8 * (size_t)N, cudaMemcpyHostToDevice, C.st));
    f->solve(bi.p, xo.p);
    CUDA_CHECK(cudaMemcpyAsync(x, xo.p, 8 * (size_t)N, cudaMemcpyDeviceToHost, C.st));
    C.sync();
    C.free(bi);
    C.free(xo);
    C.flush();
  }
  return 0;
  ABI_CATCH
}

// ---- exact dense matvec (experiments._matvec_oracle / dense.dense_matrix) -------
int ifmm_exact_matvec(void* ctx, int kernel_kind, double p0, int n, const double* points,
                      const double* x, double* y, int on_device) {
  return ifmm_exact_matvec_k(ctx, kernel_kind, p0, 0.0, n, points, x, y, on_device);
}

int ifmm_exact_matvec_k(void* ctx, int kernel_kind, double p0, double p1, int n,
                        const double* points, const double* x, double* y, int on_device) {
  ABI_TRY
  Ctx& C = *(Ctx*)ctx;
  if (kernel_kind < 1 || kernel_kind > KERNEL_KIND_MAX) throw Error(E_VALUE, "unknown kernel kind");
  KernelSpec k{kernel_kind, p0, p1};
  const int nd = n * k.bd();
  Blk P = C.alloc(n, 3), X = C.alloc(1, nd), Y = C.alloc(1, nd);
  const cudaMemcpyKind kin = on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
  const cudaMemcpyKind kout = on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
  CUDA_CHECK(cudaMemcpyAsync(P.p, points, 24 * (size_t)n, kin, C.st));
  CUDA_CHECK(cudaMemcpyAsync(X.p, x, 8 * (size_t)nd, kin, C.st));
  launch_exact_matvec(P.p, X.p, n, k, Y.p, C.st);
  CUDA_CHECK(cudaGetLastError());
  CUDA_CHECK(cudaMemcpyAsync(y, Y.p, 8 * (size_t)nd, kout, C.st));
  C.sync();
  C.free(P); C.free(X); C.free(Y);
  C.flush();
  return 0;
  ABI_CATCH
}

// ---- dense kernel matrix (dense.py:23-32) ---------------------------------------
int ifmm_kernel_matrix(void* ctx, int kernel_kind, double p0, int m, const double* P, int n,
                       const double* Q, double* out, int on_device) {
  return ifmm_kernel_matrix_k(ctx, kernel_kind, p0, 0.0, m, P, n, Q, out, on_device);
}

int ifmm_kernel_matrix_k(void* ctx, int kernel_kind, double p0, double p1, int m, const double* P,
                         int n, const double* Q, double* out, int on_device) {
  ABI_TRY
  Ctx& C = *(Ctx*)ctx;
  if (kernel_kind < 1 || kernel_kind > KERNEL_KIND_MAX) throw Error(E_VALUE, "unknown kernel kind");
  if (m < 0 || n < 0) throw Error(E_VALUE, "negative matrix size");
  if ((long long)m * n == 0) return 0;
  KernelSpec k{kernel_kind, p0, p1};
  const int bd = k.bd();
  const cudaMemcpyKind kin = on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
  Blk dP = C.alloc(m, 3), dQ = C.alloc(n, 3);
  CUDA_CHECK(cudaMemcpyAsync(dP.p, P, 24 * (size_t)m, kin, C.st));
  CUDA_CHECK(cudaMemcpyAsync(dQ.p, Q, 24 * (size_t)n, kin, C.st));
  // row panels of <= 8 rows: one CTA each, entries in row-major order
  const int rows = 8;
  const long long panel = (long long)rows * n;
  Blk O;
  double* dst = out;
  if (!on_device) { O = C.alloc(bd * m, bd * n); dst = O.p; }
  std::vector<EvalDesc> ed;
  for (int r0 = 0; r0 < m; r0 += rows) {
    EvalDesc d;
    d.P = dP.p + 3 * (size_t)r0; d.Q = dQ.p; d.m = std::min(rows, m - r0); d.n = n;
    d.out = dst + (size_t)(bd * r0) * (bd * n); d.ldo = bd * n;
    ed.push_back(d);
  }
  (void)panel;
  launch_eval(C.stage.push_vec(C, ed), (int)ed.size(), k, C.st);
  CUDA_CHECK(cudaGetLastError());
  if (!on_device)
    CUDA_CHECK(cudaMemcpyAsync(out, O.p, 8 * (size_t)m * n * bd * bd, cudaMemcpyDeviceToHost, C.st));
  C.sync();
  C.free(dP); C.free(dQ); C.free(O);
  C.flush();
  return 0;
  ABI_CATCH
}

// ---- block-diagonal preconditioner (krylov.py:172-196) ---------------------------
struct BlockDiag {
  Ctx* ctx;
  int n, bs;
  Blk lu;                 // the diagonal blocks, factored in place, back to back
  int* piv = nullptr;
  int piv_cls = -1;
  std::vector<LuDesc> lus;
  std::vector<int> off;   // block row offsets (nb + 1)
};

void* ifmm_blockdiag_create(void* ctx, const double* A, int n, int lda, int block_size,
                            int on_device) {
  ABI_TRY
  Ctx& C = *(Ctx*)ctx;
  if (block_size < 1 || block_size > n) throw Error(E_VALUE, "block_size must be in [1, n]");
  BlockDiag* B = new BlockDiag;
  B->ctx = &C; B->n = n; B->bs = block_size;
  long long tot = 0;
  for (int a = 0; a < n; a += block_size) {
    const int b = std::min(n, a + block_size);
    B->off.push_back(a);
    tot += (long long)(b - a) * (b - a);
  }
  B->off.push_back(n);
  B->lu = C.alloc(1, (int)tot);
  B->piv = C.arena.alloc_int(n, &B->piv_cls);
  const cudaMemcpyKind kin = on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
  long long o = 0;
  for (size_t i = 0; i + 1 < B->off.size(); ++i) {
    const int a = B->off[i], w = B->off[i + 1] - a;
    CUDA_CHECK(cudaMemcpy2DAsync(B->lu.p + o, 8 * (size_t)w, A + (size_t)a * lda + a, 8 * (size_t)lda,
                                 8 * (size_t)w, w, kin, C.st));
    LuDesc d;
    d.A = B->lu.p + o; d.n = w; d.lda = w; d.piv = B->piv + a; d.tag = a;
    B->lus.push_back(d);
    o += (long long)w * w;
  }
  std::vector<LuDesc> small, big;
  for (auto& d : B->lus) (d.n <= 160 ? small : big).push_back(d);
  if (!small.empty()) launch_lu(C.stage.push_vec(C, small), (int)small.size(), C.d_status, C.st);
  for (auto& d : big) lu_blocked(C, d.A, d.n, d.n, d.piv, d.tag);
  CUDA_CHECK(cudaGetLastError());
  C.sync();
  try {
    C.check_status("diagonal block at row ");
  } catch (...) {
    C.free(B->lu);
    C.free_raw(B->piv, B->piv_cls);
    C.flush();
    delete B;
    throw;
  }
  return B;
  ABI_CATCH_NULL
}

int ifmm_blockdiag_apply(void* h, const double* v, double* out, int on_device) {
  ABI_TRY
  BlockDiag& B = *(BlockDiag*)h;
  Ctx& C = *B.ctx;
  const cudaMemcpyKind kin = on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
  const cudaMemcpyKind kout = on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
  Blk X = C.alloc(1, B.n);
  CUDA_CHECK(cudaMemcpyAsync(X.p, v, 8 * (size_t)B.n, kin, C.st));
  std::vector<LuSolveDesc> sd;
  int maxn = 0;
  for (size_t i = 0; i < B.lus.size(); ++i) {
    LuSolveDesc d;
    d.LU = B.lus[i].A; d.piv = B.lus[i].piv; d.n = B.lus[i].n; d.lda = B.lus[i].n;
    d.X = X.p + B.off[i]; d.nrhs = 1; d.ldx = 1;
    sd.push_back(d);
    maxn = std::max(maxn, d.n);
  }
  launch_lusolve(C.stage.push_vec(C, sd), (int)sd.size(), 1, C.st, maxn);
  CUDA_CHECK(cudaGetLastError());
  CUDA_CHECK(cudaMemcpyAsync(out, X.p, 8 * (size_t)B.n, kout, C.st));
  C.sync();
  C.free(X);
  C.flush();
  return 0;
  ABI_CATCH
}

void ifmm_blockdiag_destroy(void* h) {
  if (!h) return;
  BlockDiag* B = (BlockDiag*)h;
  B->ctx->sync_nothrow();
  B->ctx->free(B->lu);
  B->ctx->free_raw(B->piv, B->piv_cls);
  B->ctx->flush();
  delete B;
}

// ---- micro-kernel entry points --------------------------------------------------
int ifmm_dev_gemm(void* ctx, int M, int N, int K, const double* A, int lda, int ta,
                  const double* B, int ldb, int tb, double* Cm, int ldc, double alpha,
                  double beta) {
  ABI_TRY
  Ctx& C = *(Ctx*)ctx;
  GemmBatch g;
  g.add(A, lda, ta, B, ldb, tb, Cm, ldc, M, N, K, alpha, beta);
  g.run(C);
  return 0;
  ABI_CATCH
}

int ifmm_dev_svd(void* ctx, int m, int n, const double* A, double thr, double* U, double* S,
                 double* V, int* rank) {
  ABI_TRY
  Ctx& C = *(Ctx*)ctx;
  Blk w = C.alloc(1, (int)svd_work_doubles(m, n));
  std::vector<SvdDesc> d(1);
  d[0].src = A; d[0].m = m; d[0].n = n; d[0].s_r = n; d[0].s_c = 1;
  d[0].U = U; d[0].S = S; d[0].V = V; d[0].rank = rank; d[0].work = w.p;
  launch_svd(C.stage.push_vec(C, d), 1, thr, 0, C.st, 0);
  CUDA_CHECK(cudaGetLastError());
  C.sync();
  C.free(w);
  C.flush();
  return 0;
  ABI_CATCH
}

int ifmm_dev_lu_solve(void* ctx, int n, double* A, int* piv, double* X, int nrhs) {
  ABI_TRY
  Ctx& C = *(Ctx*)ctx;
  lu_any(C, A, n, piv, 0);
  std::vector<LuSolveDesc> d(1);
  d[0].LU = A; d[0].piv = piv; d[0].n = n; d[0].lda = n; d[0].X = X; d[0].nrhs = nrhs;
  d[0].ldx = nrhs;
  if (nrhs > 0) launch_lusolve(C.stage.push_vec(C, d), 1, nrhs, C.st, n);
  CUDA_CHECK(cudaGetLastError());
  C.sync();
  C.check_status("test ");
  return 0;
  ABI_CATCH
}

int ifmm_dev_orth(void* ctx, int n, int w, const double* Y, double* Q) {
  ABI_TRY
  Ctx& C = *(Ctx*)ctx;
  Blk wk = C.alloc(1, 2 * n * w + 2 * w + 64);
  launch_tall_orth(Y, n, w, Q, wk.p, C.st);
  CUDA_CHECK(cudaGetLastError());
  C.sync();
  C.free(wk);
  C.flush();
  return 0;
  ABI_CATCH
}

int ifmm_dev_union(void* ctx, int m, int k_old, int k_f, const double* B, const double* w,
                   const double* F, const double* wf, double thr, int min_rank, double* NB,
                   double* NW, double* OM, double* FM, int* rank) {
  ABI_TRY
  Ctx& C = *(Ctx*)ctx;
  Blk wk = C.alloc(1, (int)union_work_doubles(m, k_old, k_f));
  std::vector<UnionDesc> d(1);
  d[0].B = B; d[0].w = w; d[0].F = F; d[0].wf = wf;
  d[0].m = m; d[0].k_old = k_old; d[0].k_f = k_f;
  d[0].b_r = k_old; d[0].b_c = 1; d[0].f_r = k_f; d[0].f_c = 1;  // row-major inputs
  d[0].min_rank = min_rank;
  d[0].NB = NB; d[0].nb_r = 1; d[0].nb_c = m;                    // col-major output
  d[0].NW = NW; d[0].OM = OM; d[0].FM = FM; d[0].rank = rank; d[0].work = wk.p;
  const int smax = std::min(m, k_old + k_f);
  const bool fits = union_fits_smem(m, k_old, k_f);
  d[0].giant = (!fits && smax > giant_union_threshold()) ? 1 : 0;
  int rg = 0, rer = 0, rec = 0;
  const char* ar = getenv("IFMM_ACA_REG");
  const bool reg = !d[0].giant && (!ar || atoi(ar)) && union_aca_reg_class(m, k_old + k_f, &rg, &rer, &rec);
  const char* up = getenv("IFMM_UNION_POST");
  const bool post = reg && (!up || atoi(up)) && union_post_eligible(m, k_old, k_f);
  if (reg) d[0].giant = post ? 3 : 2;
  UnionDesc* dd = C.stage.push_vec(C, d);
  Blk fl = C.alloc(1, union_giant_scratch_doubles(1));
  if (reg) launch_union_aca_reg(dd, 1, thr, rg, rer, rec, C.st);
  if (post) launch_union_post(dd, 1, thr, C.st);
  else
    launch_union(dd, 1, thr, C.st, fits ? 1 : 0, 0, d[0].giant == 1 ? dd : nullptr, d[0].giant == 1,
                 smax, fl.p, m, k_old + k_f);
  CUDA_CHECK(cudaGetLastError());
  C.sync();
  if (post) {  // declined (rank -1): the legacy path, as the engine does
    int hr = 0;
    CUDA_CHECK(cudaMemcpy(&hr, rank, sizeof(int), cudaMemcpyDeviceToHost));
    if (hr < 0) {
      d[0].giant = (!fits && smax > giant_union_threshold()) ? 1 : 0;
      dd = C.stage.push_vec(C, d);
      launch_union(dd, 1, thr, C.st, fits ? 1 : 0, 0, d[0].giant == 1 ? dd : nullptr, d[0].giant == 1,
                   smax, fl.p, m, k_old + k_f);
      CUDA_CHECK(cudaGetLastError());
      C.sync();
    }
  }
  C.free(fl);
  C.free(wk);
  C.flush();
  return 0;
  ABI_CATCH
}

int ifmm_dev_sync(void* ctx) {
  ABI_TRY
  ((Ctx*)ctx)->sync();
  return 0;
  ABI_CATCH
}

// ---- GMRES Arnoldi on the device (krylov.py:32-116) -----------------------------
int ifmm_krylov_mgs(void* ctx, const double* V, long long ldv, int k1, long long n, double* w,
                    double* h) {
  ABI_TRY
  if (!ctx || !V || !w || !h || k1 < 0 || n < 1 || ldv < n) throw Error(E_VALUE, "bad MGS arguments");
  krylov_mgs(*(Ctx*)ctx, V, ldv, k1, n, w, h);
  return 0;
  ABI_CATCH
}

int ifmm_krylov_div(void* ctx, const double* w, long long n, double hs, double* out) {
  ABI_TRY
  if (!ctx || !w || !out || n < 1) throw Error(E_VALUE, "bad normalisation arguments");
  krylov_div(*(Ctx*)ctx, w, n, hs, out);
  return 0;
  ABI_CATCH
}

int ifmm_krylov_combine(void* ctx, const double* V, long long ldv, int k, const double* y,
                        long long n, double* u) {
  ABI_TRY
  if (!ctx || !V || !u || (k > 0 && !y) || k < 0 || n < 1 || ldv < n)
    throw Error(E_VALUE, "bad combine arguments");
  krylov_combine(*(Ctx*)ctx, V, ldv, k, y, n, u);
  return 0;
  ABI_CATCH
}

}  // extern "C"
