// Extended sparse graph assembly (graph.py:30-229) and sigma0 estimation
// (graph.py:232-241 -> lowrank.py:79-119 with start_rank = max_rank = 1).
#include <algorithm>

#include "engine.h"
#include "spmv.cuh"

namespace ifmm {

Graph::~Graph() {
  if (!ctx) return;
  for (auto& kv : E) ctx->free(kv.second);
  for (auto& b : su) ctx->free(b);
  for (auto& b : sv) ctx->free(b);
  if (cudaStreamSynchronize(ctx->st) != cudaSuccess) cudaGetLastError();  // no throw in a destructor
  ctx->flush();
}

void Graph::build(H2* h, bool consume) {
  ops = h;
  tree = h->tree;
  ctx = h->ctx;
  Ctx& C = *ctx;
  Tree& T = *tree;
  if (consume) h->drop_plan();
  nx.assign(T.nc, -1); nz.assign(T.nc, -1); ny.assign(T.nc, -1);
  dead.assign(T.nc, 0);
  su.assign(T.nc, Blk()); sv.assign(T.nc, Blk());
  bd = h->kern.bd();
  for (int c : T.leaves()) nx[c] = new_node(bd * (T.stop[c] - T.start[c]), NK_X, c);
  for (int l = 2; l <= T.depth; ++l)
    for (int c : T.levels[l]) {
      nz[c] = new_node(h->rank[c], NK_Z, c);
      ny[c] = new_node(h->rank[c], NK_Y, c);
    }
  CopyBatch cb;
  // consume: move the operator blocks into the graph (no second copy; the
  // operators are unusable afterwards)
  auto dup = [&](Blk& s) {
    if (consume) {
      Blk b = s;
      s = Blk();
      return b;
    }
    Blk b = C.alloc(s.r, s.c);
    cb.add(s.p, s.c, 1, b.p, b.c, 1, s.r, s.c, 0);
    return b;
  };
  auto dupT = [&](Blk& s) {
    Blk b = C.alloc(s.c, s.r);
    cb.add(s.p, 1, s.c, b.p, b.c, 1, s.c, s.r, 0);
    if (consume) C.free(s);
    return b;
  };
  // graph.py:63-84
  for (auto& kv : h->near) {
    const int i = (int)(kv.first >> 32), j = (int)(kv.first & 0xffffffffu);
    set(nx[i], nx[j], dup(kv.second));
  }
  if (T.depth >= 2)
    for (int c : T.leaves()) {
      set(nx[c], nz[c], dup(h->leaf_u[c]));
      set(nz[c], nx[c], dupT(h->leaf_v[c]));
    }
  for (int l = 2; l <= T.depth; ++l)
    for (int c : T.levels[l]) {
      const int k = h->rank[c];
      Blk a = C.alloc(k, k), b = C.alloc(k, k);
      cb.eye(a, -1.0);
      cb.eye(b, -1.0);
      set(nz[c], ny[c], a);
      set(ny[c], nz[c], b);
      su[c] = dup(h->su[c]);
      sv[c] = dup(h->sv[c]);
    }
  for (auto& kv : h->coupling) {
    const int i = (int)(kv.first >> 32), j = (int)(kv.first & 0xffffffffu);
    set(ny[i], ny[j], dup(kv.second));
  }
  for (int c = 0; c < T.nc; ++c)
    if (h->tu[c].p) {
      const int p = T.parent[c];
      set(ny[c], nz[p], dup(h->tu[c]));
      set(nz[p], ny[c], dup(h->tvt[c]));
    }
  cb.run(C);
  if (consume) {
    h->consumed = true;
    C.flush();
  }
  CUDA_CHECK(cudaGetLastError());
}

// Deep copy (graph.py:190-216): same nodes, adjacency and weights, every
// block duplicated on the device (one batched copy).
Graph* Graph::clone() const {
  IFMM_ASSERT(!consumed, "copy of a consumed graph");
  Ctx& C = *ctx;
  Graph* g = new Graph;
  g->ctx = ctx; g->tree = tree; g->ops = ops; g->bd = bd;
  g->size = size; g->kind = kind; g->owner = owner;
  g->nx = nx; g->nz = nz; g->ny = ny;
  g->rows = rows; g->cols = cols; g->dead = dead;
  g->peak_edges = peak_edges;
  CopyBatch cb;
  auto dup = [&](const Blk& s) {
    if (!s.p) return Blk();
    Blk b = C.alloc(s.r, s.c);
    cb.add(s.p, s.c, 1, b.p, b.c, 1, s.r, s.c, 0);
    return b;
  };
  g->E.reserve(E.size());
  for (auto& kv : E) g->E.emplace(kv.first, dup(kv.second));
  g->su.resize(su.size()); g->sv.resize(sv.size());
  for (size_t i = 0; i < su.size(); ++i) { g->su[i] = dup(su[i]); g->sv[i] = dup(sv[i]); }
  cb.run(C);
  CUDA_CHECK(cudaGetLastError());
  return g;
}

// out = E in (or E^T in) for one full node vector (graph.py:157-170),
// deterministic block SpMV in sorted node order.
void Graph::apply(const double* d_in, double* d_out, bool transpose) {
  Ctx& C = *ctx;
  const int nn = (int)size.size();
  std::vector<long long> off(nn + 1, 0);
  for (int i = 0; i < nn; ++i) off[i + 1] = off[i] + size[i];
  std::vector<SpmvRow> rr;
  std::vector<SpmvTerm> tt;
  for (int a = 0; a < nn; ++a) {
    SpmvRow r{d_out + off[a], size[a], (int)tt.size(), 0, 0};
    if (!transpose) {
      for (int s : rows[a]) {
        const Blk& B = E.at(key2(a, s));
        tt.push_back({B.p, B.r, B.c, B.c, 0, d_in + off[s]});
        r.nt++;
      }
    } else {
      for (int t : cols[a]) {
        const Blk& B = E.at(key2(t, a));
        tt.push_back({B.p, B.r, B.c, B.c, 1, d_in + off[t]});
        r.nt++;
      }
    }
    rr.push_back(r);
  }
  SpmvTerm* dt = C.stage.push_vec(C, tt);
  SpmvRow* dr = C.stage.push_vec(C, rr);
  launch_spmv(dr, (int)rr.size(), dt, 1, 1, C.st);
  CUDA_CHECK(cudaGetLastError());
}

// ---------------------------------------------------------------------------
// sigma0 = leading singular value of the extended matrix by the reference's
// randomized SVD with one probe rank: Y = E omega; 2x Y = E E^T orth(Y);
// Q = orth(Y); sigma_max((E^T Q)^T).
// ---------------------------------------------------------------------------
double Graph::sigma0(const double* omega, int width, int power_iters) {
  Ctx& C = *ctx;
  const int nn = (int)size.size();
  std::vector<long long> off(nn + 1, 0);
  for (int i = 0; i < nn; ++i) off[i + 1] = off[i] + size[i];
  const long long dim = off[nn];
  IFMM_ASSERT(dim < (1LL << 31), "extended dimension too large");
  const int w = width;
  Blk Om = C.alloc((int)dim, w), Y = C.alloc((int)dim, w), Z = C.alloc((int)dim, w);
  Blk Q = C.alloc((int)dim, w);
  Blk work = C.alloc(1, (int)(2 * dim * w + 4 * w * w + 64 + tall_grid_work_doubles(w)));
  Blk out = C.alloc(1, 2);  // sigma0, then the breakdown flag
  CUDA_CHECK(cudaMemcpyAsync(Om.p, omega, sizeof(double) * dim * w, cudaMemcpyHostToDevice, C.st));
  // Row tasks for E and E^T (terms in sorted node order -> deterministic),
  // built and uploaded ONCE: E always maps Z -> Y (the sketch is copied into
  // Z first), E^T always Q -> Z.
  std::vector<SpmvRow> rE, rT;
  std::vector<SpmvTerm> tE, tT;
  for (int t = 0; t < nn; ++t) {
    SpmvRow r{Y.p + off[t] * w, size[t], (int)tE.size(), 0, 0};
    for (int s : rows[t]) {
      const Blk& B = E.at(key2(t, s));
      tE.push_back({B.p, B.r, B.c, B.c, 0, Z.p + off[s] * w});
      r.nt++;
    }
    rE.push_back(r);
  }
  for (int s = 0; s < nn; ++s) {
    SpmvRow r{Z.p + off[s] * w, size[s], (int)tT.size(), 0, 0};
    for (int t : cols[s]) {
      const Blk& B = E.at(key2(t, s));
      tT.push_back({B.p, B.r, B.c, B.c, 1, Q.p + off[t] * w});
      r.nt++;
    }
    rT.push_back(r);
  }
  static_assert(sizeof(SpmvRow) % 8 == 0 && sizeof(SpmvTerm) % 8 == 0, "descriptor alignment");
  auto upload = [&](const void* src, size_t bytes) {
    Blk d = C.alloc(1, (int)(bytes / 8 + 1));
    if (bytes) CUDA_CHECK(cudaMemcpyAsync(d.p, src, bytes, cudaMemcpyHostToDevice, C.st));
    return d;
  };
  Blk drE = upload(rE.data(), rE.size() * sizeof(SpmvRow));
  Blk dtE = upload(tE.data(), tE.size() * sizeof(SpmvTerm));
  Blk drT = upload(rT.data(), rT.size() * sizeof(SpmvRow));
  Blk dtT = upload(tT.data(), tT.size() * sizeof(SpmvTerm));
  auto applyE = [&]() {
    launch_spmv(reinterpret_cast<const SpmvRow*>(drE.p), (int)rE.size(),
                reinterpret_cast<const SpmvTerm*>(dtE.p), w, w, C.st);
  };
  auto applyET = [&]() {
    launch_spmv(reinterpret_cast<const SpmvRow*>(drT.p), (int)rT.size(),
                reinterpret_cast<const SpmvTerm*>(dtT.p), w, w, C.st);
  };
  // orth / sigma_max on the whole grid (tall.cu, CholeskyQR2) when w allows;
  // a Cholesky breakdown (flag) repeats the estimate with the one-CTA
  // Householder kernels
  int* d_flag = reinterpret_cast<int*>(out.p + 1);
  double s0 = 0.0;
  for (int attempt = 0; attempt < 2; ++attempt) {
    const bool grid = attempt == 0 && tall_grid_supported(w);
    if (attempt == 1 && tall_grid_supported(w) == false) break;
    auto orth = [&]() {
      if (grid) launch_tall_orth_grid(Y.p, (int)dim, w, Q.p, work.p, d_flag, C.st);
      else launch_tall_orth(Y.p, (int)dim, w, Q.p, work.p, C.st);
    };
    CUDA_CHECK(cudaMemsetAsync(d_flag, 0, sizeof(int), C.st));
    CUDA_CHECK(cudaMemcpyAsync(Z.p, Om.p, sizeof(double) * dim * w, cudaMemcpyDeviceToDevice, C.st));
    applyE();
    for (int it = 0; it < power_iters; ++it) {
      orth();
      applyET();
      applyE();
    }
    orth();
    applyET();
    if (grid) launch_tall_sigmax_grid(Z.p, (int)dim, w, out.p, work.p, C.st);
    else launch_tall_sigmax(Z.p, (int)dim, w, out.p, work.p, C.st);
    CUDA_CHECK(cudaGetLastError());
    int hflag = 0;
    CUDA_CHECK(cudaMemcpyAsync(&s0, out.p, sizeof(double), cudaMemcpyDeviceToHost, C.st));
    CUDA_CHECK(cudaMemcpyAsync(&hflag, d_flag, sizeof(int), cudaMemcpyDeviceToHost, C.st));
    C.sync();
    if (!grid || !hflag) break;
  }
  for (Blk* b : {&Om, &Y, &Z, &Q, &work, &out, &drE, &dtE, &drT, &dtT}) C.free(*b);
  C.flush();
  return s0;
}

}  // namespace ifmm
