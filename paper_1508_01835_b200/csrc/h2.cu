// H2 operator construction on the device (h2.py:104-290) and the fast H2
// matvec (krylov.py:119-159).
#include <algorithm>
#include <cmath>

#include "engine.h"
#include "spmv.cuh"

namespace ifmm {

H2::~H2() {
  if (!ctx) return;
  for (auto* v : {&leaf_u, &leaf_v, &tu, &tvt, &su, &sv})
    for (auto& b : *v) ctx->free(b);
  for (auto& kv : coupling) ctx->free(kv.second);
  for (auto& kv : near) ctx->free(kv.second);
  drop_plan();
  ctx->sync_nothrow();
  ctx->flush();
}

// ---------------------------------------------------------------------------
// chebyshev_operators (h2.py:104-182)
// ---------------------------------------------------------------------------
void H2::build() {
  Ctx& C = *ctx;
  Tree& T = *tree;
  const int g3 = ncheb * ncheb * ncheb;
  // block_dim > 1 (kernels.py:33, h2.py:70-74 _kron_bd): every interpolation
  // matrix is kron(., I_bd), so a cluster's grid has g3b = bd g3 coefficients
  // and a leaf of m points has bd m rows (point-major ordering)
  const int bd = kern.bd();
  const int g3b = bd * g3;
  const double rel = std::max(eps, 1e-13);
  // dst (bd r x bd c) = kron(src (r x c), I_bd): zero fill, then bd strided copies
  auto kron = [&](CopyBatch& zero, CopyBatch& cp, const Blk& src, const Blk& dst) {
    zero.add(nullptr, 0, 0, dst.p, dst.c, 1, dst.r, dst.c, 3);
    for (int a = 0; a < bd; ++a)
      cp.add(src.p, src.c, 1, dst.p + (size_t)a * dst.c + a, bd * dst.c, bd, src.r, src.c, 0);
  };
  const int nc = T.nc;
  rank.assign(nc, -1);
  leaf_u.assign(nc, Blk()); leaf_v.assign(nc, Blk());
  tu.assign(nc, Blk()); tvt.assign(nc, Blk());
  su.assign(nc, Blk()); sv.assign(nc, Blk());
  std::vector<Blk> G(nc);  // reduce maps k x g3

  // ---- leaves: interpolation matrix + SVD reduction (h2.py:129-135) ----
  {
    const auto leaves = T.leaves();
    const int nl = (int)leaves.size();
    std::vector<Blk> Pm(nl), Pk(nl), Ub(nl), Sb(nl), Vb(nl), Wk(nl);
    CopyBatch kz, kc;
    Blk ranks_b = C.alloc(1, (nl + 1) / 2 + 1);
    int* d_rank = reinterpret_cast<int*>(ranks_b.p);
    std::vector<InterpDesc> idesc;
    std::vector<SvdDesc> sdesc;
    for (int t = 0; t < nl; ++t) {
      const int c = leaves[t];
      const int mp = T.stop[c] - T.start[c];
      const int m = bd * mp;
      const int mn = std::min(m, g3b);
      Pm[t] = C.alloc(mp, g3);
      Pk[t] = bd > 1 ? C.alloc(m, g3b) : Pm[t];
      if (bd > 1) kron(kz, kc, Pm[t], Pk[t]);
      Ub[t] = C.alloc(m, mn);
      Sb[t] = C.alloc(1, mn);
      Vb[t] = C.alloc(g3b, mn);
      Wk[t] = C.alloc(1, (int)svd_work_doubles(m, g3b));
      InterpDesc d;
      d.pts = T.d_points + 3 * (size_t)T.start[c];
      d.count = mp;
      d.cx = T.center[3 * c]; d.cy = T.center[3 * c + 1]; d.cz = T.center[3 * c + 2];
      d.hw = T.hw[c];
      d.out = Pm[t].p;
      d.ldo = g3;
      idesc.push_back(d);
      SvdDesc s;
      s.src = Pk[t].p; s.m = m; s.n = g3b; s.s_r = g3b; s.s_c = 1;
      s.U = Ub[t].p; s.S = Sb[t].p; s.V = Vb[t].p; s.rank = d_rank + t; s.work = Wk[t].p;
      sdesc.push_back(s);
    }
    launch_interp(C.stage.push_vec(C, idesc), nl, ncheb, C.st);
    kz.run(C);
    kc.run(C);
    launch_svd(C.stage.push_vec(C, sdesc), nl, rel, 64, C.st, 1);
    CUDA_CHECK(cudaGetLastError());
    const int* hr = C.readback_ints(d_rank, nl);
    CopyBatch cb;
    for (int t = 0; t < nl; ++t) {
      const int c = leaves[t];
      const int m = bd * (T.stop[c] - T.start[c]);
      const int k = hr[t];
      rank[c] = k;
      leaf_u[c] = C.alloc(m, k);
      leaf_v[c] = C.alloc(m, k);
      G[c] = C.alloc(k, g3b);
      // U col-major (ld m) -> row-major m x k
      cb.add(Ub[t].p, 1, m, leaf_u[c].p, k, 1, m, k, 0);
      cb.add(Ub[t].p, 1, m, leaf_v[c].p, k, 1, m, k, 0);
      // G[a][j] = s_a * V(j, a), V col-major (ld g3)
      cb.add(Vb[t].p, g3b, 1, G[c].p, g3b, 1, k, g3b, 0, 1.0, Sb[t].p);
    }
    cb.run(C);
    for (int t = 0; t < nl; ++t) {
      if (bd > 1) C.free(Pk[t]);
      C.free(Pm[t]); C.free(Ub[t]); C.free(Sb[t]); C.free(Vb[t]); C.free(Wk[t]);
    }
    C.free(ranks_b);
    C.flush();
  }

  // ---- Chebyshev grids of every cluster at levels >= 2 ----
  std::vector<Blk> grid(nc);
  {
    std::vector<GridDesc> gd;
    for (int l = 2; l <= T.depth; ++l)
      for (int c : T.levels[l]) {
        grid[c] = C.alloc(g3, 3);
        GridDesc d;
        d.cx = T.center[3 * c]; d.cy = T.center[3 * c + 1]; d.cz = T.center[3 * c + 2];
        d.hw = T.hw[c];
        d.out = grid[c].p;
        gd.push_back(d);
      }
    if (!gd.empty()) launch_grid(C.stage.push_vec(C, gd), (int)gd.size(), ncheb, C.st);
  }

  // ---- transfers, levels L-1 .. 2 (h2.py:137-152) ----
  for (int l = T.depth - 1; l >= 2; --l) {
    const auto& ps = T.levels[l];
    const int np = (int)ps.size();
    std::vector<InterpDesc> idesc;
    std::vector<Blk> Tm;  // per child transfer interp (g3 x g3)
    std::vector<Blk> stack(np), Ub(np), Sb(np), Vb(np), Wk(np);
    std::vector<int> tot(np);
    Blk ranks_b = C.alloc(1, (np + 1) / 2 + 1);
    int* d_rank = reinterpret_cast<int*>(ranks_b.p);
    GemmBatch gb;
    CopyBatch kz, kc;
    std::vector<Blk> Tk;  // kron(T, I_bd) when bd > 1
    std::vector<SvdDesc> sdesc;
    for (int t = 0; t < np; ++t) {
      const int p = ps[t];
      int rows = 0;
      for (int c : T.children[p]) rows += rank[c];
      tot[t] = rows;
      stack[t] = C.alloc(rows, g3b);
      int r0 = 0;
      for (int c : T.children[p]) {
        Blk tm = C.alloc(g3, g3);
        Tm.push_back(tm);
        InterpDesc d;
        d.pts = grid[c].p; d.count = g3;
        d.cx = T.center[3 * p]; d.cy = T.center[3 * p + 1]; d.cz = T.center[3 * p + 2];
        d.hw = T.hw[p];
        d.out = tm.p; d.ldo = g3;
        idesc.push_back(d);
        Blk tk = tm;
        if (bd > 1) {
          tk = C.alloc(g3b, g3b);
          Tk.push_back(tk);
          kron(kz, kc, tm, tk);
        }
        gb.add(G[c].p, g3b, 0, tk.p, g3b, 0, stack[t].p + (size_t)r0 * g3b, g3b, rank[c], g3b,
               g3b, 1.0, 0.0);
        r0 += rank[c];
      }
      const int mn = std::min(rows, g3b);
      Ub[t] = C.alloc(rows, mn); Sb[t] = C.alloc(1, mn); Vb[t] = C.alloc(g3b, mn);
      Wk[t] = C.alloc(1, (int)svd_work_doubles(rows, g3b));
      SvdDesc s;
      s.src = stack[t].p; s.m = rows; s.n = g3b; s.s_r = g3b; s.s_c = 1;
      s.U = Ub[t].p; s.S = Sb[t].p; s.V = Vb[t].p; s.rank = d_rank + t; s.work = Wk[t].p;
      sdesc.push_back(s);
    }
    launch_interp(C.stage.push_vec(C, idesc), (int)idesc.size(), ncheb, C.st);
    kz.run(C);
    kc.run(C);
    gb.run(C);
    launch_svd(C.stage.push_vec(C, sdesc), np, rel, 64, C.st, 1);
    CUDA_CHECK(cudaGetLastError());
    const int* hr = C.readback_ints(d_rank, np);
    CopyBatch cb;
    for (int t = 0; t < np; ++t) {
      const int p = ps[t];
      const int k = hr[t];
      rank[p] = k;
      int r0 = 0;
      for (int c : T.children[p]) {
        tu[c] = C.alloc(rank[c], k);
        tvt[c] = C.alloc(k, rank[c]);
        // basis col-major (ld rows): rows [r0, r0+k_c) -> tu[c] (k_c x k)
        cb.add(Ub[t].p + r0, 1, tot[t], tu[c].p, k, 1, rank[c], k, 0);
        cb.add(Ub[t].p + r0, 1, tot[t], tvt[c].p, 1, rank[c], rank[c], k, 0);
        r0 += rank[c];
      }
      G[p] = C.alloc(k, g3b);
      cb.add(Vb[t].p, g3b, 1, G[p].p, g3b, 1, k, g3b, 0, 1.0, Sb[t].p);
    }
    cb.run(C);
    for (auto& b : Tm) C.free(b);
    for (auto& b : Tk) C.free(b);
    for (int t = 0; t < np; ++t) {
      C.free(stack[t]); C.free(Ub[t]); C.free(Sb[t]); C.free(Vb[t]); C.free(Wk[t]);
    }
    C.free(ranks_b);
    C.flush();
  }

  // ---- M2L couplings (h2.py:154-164): K(i,j) = G_i Kgrid(i,j) G_j^T, i<j ----
  {
    std::vector<std::pair<int, int>> pairs;
    for (int l = 2; l <= T.depth; ++l)
      for (int i : T.levels[l])
        for (int j : T.inters[i])
          if (j > i) pairs.emplace_back(i, j);
    const size_t per = (size_t)g3b * g3b;
    const size_t chunk = std::max<size_t>(1, ((size_t)256 << 20) / (per * 8));
    for (size_t a = 0; a < pairs.size(); a += chunk) {
      const size_t b = std::min(pairs.size(), a + chunk);
      const int n = (int)(b - a);
      Blk kg = C.alloc(n, (int)per);
      int kmax = 0;
      for (size_t t = a; t < b; ++t) kmax = std::max(kmax, rank[pairs[t].first]);
      Blk t1 = C.alloc(n, kmax * g3b);
      std::vector<EvalDesc> ed;
      GemmBatch g1, g2;
      CopyBatch cb;
      for (size_t t = a; t < b; ++t) {
        const int i = pairs[t].first, j = pairs[t].second;
        const size_t o = (t - a);
        EvalDesc e;
        e.P = grid[i].p; e.Q = grid[j].p; e.m = g3; e.n = g3;
        e.out = kg.p + o * per; e.ldo = g3b;
        ed.push_back(e);
        double* T1 = t1.p + o * (size_t)kmax * g3b;
        g1.add(G[i].p, g3b, 0, e.out, g3b, 0, T1, g3b, rank[i], g3b, g3b, 1.0, 0.0);
        Blk kij = C.alloc(rank[i], rank[j]);
        Blk kji = C.alloc(rank[j], rank[i]);
        g2.add(T1, g3b, 0, G[j].p, g3b, 1, kij.p, rank[j], rank[i], rank[j], g3b, 1.0, 0.0);
        cb.add(kij.p, 1, rank[j], kji.p, rank[i], 1, rank[j], rank[i], 0);
        coupling[key2(i, j)] = kij;
        coupling[key2(j, i)] = kji;
      }
      launch_eval(C.stage.push_vec(C, ed), n, kern, C.st);
      g1.run(C);
      g2.run(C);
      cb.run(C);
      C.free(kg);
      C.free(t1);
      C.flush();  // chunk workspaces are reusable once their launches are enqueued
    }
  }

  // ---- P2P near field (h2.py:166-177): both orientations evaluated ----
  {
    std::vector<EvalDesc> ed;
    for (int i : T.leaves()) {
      const int mi = T.stop[i] - T.start[i];
      for (int j : T.nbrs[i]) {
        const int mj = T.stop[j] - T.start[j];
        Blk s = C.alloc(bd * mi, bd * mj);
        EvalDesc e;
        e.P = T.d_points + 3 * (size_t)T.start[i];
        e.Q = T.d_points + 3 * (size_t)T.start[j];
        e.m = mi; e.n = mj; e.out = s.p; e.ldo = bd * mj;
        ed.push_back(e);
        near[key2(i, j)] = s;
        if (ed.size() >= 65536) {
          launch_eval(C.stage.push_vec(C, ed), (int)ed.size(), kern, C.st);
          ed.clear();
        }
      }
    }
    if (!ed.empty()) launch_eval(C.stage.push_vec(C, ed), (int)ed.size(), kern, C.st);
  }
  for (auto& b : G) C.free(b);
  for (auto& b : grid) C.free(b);
  CUDA_CHECK(cudaGetLastError());
  C.sync();
  C.flush();
}

// ---------------------------------------------------------------------------
// initialize_weights, rigorous, symmetric kernel (h2.py:185-231).  Left
// singular vectors / values of hstack_q K(j,q) are invariant under the
// right-rotations other clusters apply, so every cluster is computed in
// parallel from the unrotated couplings and rotated once.
// ---------------------------------------------------------------------------
void H2::weights(const long long* sptr, const int* sidx) {
  Ctx& C = *ctx;
  Tree& T = *tree;
  drop_plan();
  std::vector<int> ids;
  for (int l = 2; l <= T.depth; ++l)
    for (int c : T.levels[l]) ids.push_back(c);
  std::vector<Blk> P(T.nc);
  // the concatenated coupling rows H_j (k x sum k_q) are built and reduced
  // in chunks of at most ~2 GB so setup memory stays bounded
  const size_t chunk_doubles = (size_t)256 << 20;
  size_t pos = 0;
  while (pos < ids.size()) {
    std::vector<WeightDesc> wd;
    std::vector<int> wj;  // cluster of each descriptor
    std::vector<Blk> Hs, Ws;
    CopyBatch cb;
    size_t used = 0;
    for (; pos < ids.size() && used < chunk_doubles; ++pos) {
      const int j = ids[pos];
      const int k = rank[j];
      su[j] = C.alloc(1, k);
      sv[j] = C.alloc(1, k);
      P[j] = C.alloc(k, k);
      if (T.inters[j].empty()) {  // unit weights, no rotation (h2.py:206-209)
        cb.add(nullptr, 0, 0, su[j].p, 1, 1, 1, k, 4, 1.0);
        cb.eye(P[j], 1.0);
        continue;
      }
      int W = 0;
      for (int q : T.inters[j]) W += rank[q];
      Blk H = C.alloc(k, W);
      int off = 0;
      for (int q : T.inters[j]) {
        Blk& K = coupling.at(key2(j, q));
        cb.add(K.p, K.c, 1, H.p + off, W, 1, K.r, K.c, 0);
        off += K.c;
      }
      Blk w = C.alloc(1, (int)weights_work_doubles(k, W));
      WeightDesc d;
      d.H = H.p; d.k = k; d.W = W; d.P = P[j].p; d.w = su[j].p; d.work = w.p;
      wd.push_back(d);
      wj.push_back(j);
      Hs.push_back(H);
      Ws.push_back(w);
      used += (size_t)k * W + weights_work_doubles(k, W) + (sptr ? (size_t)(64 + k) * W : 0);
    }
    cb.run(C);
    std::vector<Blk> Ss;
    if (sptr) {
      // sampled mode (h2.py:250-262 _sampled_gram): H_j <- (m / s) Bs^T (Bs H_j)
      // for the caller's sorted row sample Bs of the cluster's basis B (leaf:
      // U_j; parent: the children's transfers stacked).  Left-multiplication
      // only, so the parallel evaluation stays valid.
      CopyBatch gs;
      GemmBatch ga, gb;
      for (size_t i = 0; i < wd.size(); ++i) {
        const int j = wj[i];
        const int k = rank[j], W = wd[i].W;
        const int s = (int)(sptr[j + 1] - sptr[j]);
        const int* idx = sidx + sptr[j];
        int m = 0;
        if (T.is_leaf(j)) m = leaf_u[j].r;
        else for (int c : T.children[j]) m += tu[c].r;
        IFMM_ASSERT(s >= 1 && s <= m, "sampled weights: bad sample size");
        Blk Bs = C.alloc(s, k), Tm = C.alloc(s, W), H2b = C.alloc(k, W);
        for (int r = 0; r < s; ++r) {
          int row = idx[r];
          IFMM_ASSERT(row >= 0 && row < m, "sampled weights: row index out of range");
          const double* src = nullptr;
          if (T.is_leaf(j)) src = leaf_u[j].p + (size_t)row * k;
          else
            for (int c : T.children[j]) {
              if (row < tu[c].r) { src = tu[c].p + (size_t)row * k; break; }
              row -= tu[c].r;
            }
          gs.add(src, k, 1, Bs.p + (size_t)r * k, k, 1, 1, k, 0);
        }
        ga.add(Bs.p, k, 0, wd[i].H, W, 0, Tm.p, W, s, W, k, 1.0, 0.0);
        gb.add(Bs.p, k, 1, Tm.p, W, 0, H2b.p, W, k, W, s, (double)m / (double)s, 0.0);
        wd[i].H = H2b.p;
        Ss.push_back(Bs); Ss.push_back(Tm); Ss.push_back(H2b);
      }
      gs.run(C);
      ga.run(C);
      gb.run(C);
    }
    if (!wd.empty()) launch_weights(C.stage.push_vec(C, wd), (int)wd.size(), C.st);
    CUDA_CHECK(cudaGetLastError());
    C.sync();
    for (auto& b : Hs) C.free(b);
    for (auto& b : Ws) C.free(b);
    for (auto& b : Ss) C.free(b);
    C.flush();
  }
  {
    CopyBatch cb;
    for (int j : ids) cb.add(su[j].p, 1, 1, sv[j].p, 1, 1, 1, rank[j], 0);
    cb.run(C);
  }

  std::vector<std::pair<Blk*, Blk>> repl;
  std::vector<Blk> tmp;
  GemmBatch g1, g2;
  // leaves: U <- U P, V <- V P   (h2.py:268-269, 282-283)
  for (int j : ids) {
    if (!T.is_leaf(j)) continue;
    const int k = rank[j];
    for (Blk* B : {&leaf_u[j], &leaf_v[j]}) {
      Blk nb = C.alloc(B->r, k);
      g1.add(B->p, B->c, 0, P[j].p, k, 0, nb.p, k, B->r, k, k, 1.0, 0.0);
      repl.emplace_back(B, nb);
    }
  }
  // transfers: tu[c] = P_c^T (tu[c] P_p) ; tvt[c] = (P_p^T tvt[c]) P_c
  for (int c = 0; c < T.nc; ++c) {
    if (!tu[c].p) continue;
    const int p = T.parent[c];
    const int kc = rank[c], kp = rank[p];
    Blk t_a = C.alloc(kc, kp), nu = C.alloc(kc, kp);
    Blk t_b = C.alloc(kp, kc), nv = C.alloc(kp, kc);
    g1.add(tu[c].p, kp, 0, P[p].p, kp, 0, t_a.p, kp, kc, kp, kp, 1.0, 0.0);
    g1.add(P[p].p, kp, 1, tvt[c].p, kc, 0, t_b.p, kc, kp, kc, kp, 1.0, 0.0);
    g2.add(P[c].p, kc, 1, t_a.p, kp, 0, nu.p, kp, kc, kp, kc, 1.0, 0.0);
    g2.add(t_b.p, kc, 0, P[c].p, kc, 0, nv.p, kc, kp, kc, kc, 1.0, 0.0);
    tmp.push_back(t_a); tmp.push_back(t_b);
    repl.emplace_back(&tu[c], nu);
    repl.emplace_back(&tvt[c], nv);
  }
  g1.run(C);
  g2.run(C);
  for (auto& r : repl) { C.free(*r.first); *r.first = r.second; }
  for (auto& b : tmp) C.free(b);
  repl.clear();
  tmp.clear();
  C.sync();
  C.flush();
  // couplings: K(j,q) = (P_j^T K(j,q)) P_q, in chunks (bounded temporaries)
  size_t nb = 0;
  for (auto& kv : coupling) {
    const int j = (int)(kv.first >> 32), q = (int)(kv.first & 0xffffffffu);
    Blk& K = kv.second;
    const int kj = K.r, kq = K.c;
    Blk t = C.alloc(kj, kq), nk = C.alloc(kj, kq);
    g1.add(P[j].p, kj, 1, K.p, kq, 0, t.p, kq, kj, kq, kj, 1.0, 0.0);
    g2.add(t.p, kq, 0, P[q].p, kq, 0, nk.p, kq, kj, kq, kq, 1.0, 0.0);
    tmp.push_back(t);
    repl.emplace_back(&K, nk);
    if (++nb % 200000 == 0) {
      g1.run(C);
      g2.run(C);
      for (auto& r : repl) { C.free(*r.first); *r.first = r.second; }
      for (auto& b : tmp) C.free(b);
      repl.clear();
      tmp.clear();
      C.sync();
      C.flush();
    }
  }
  g1.run(C);
  g2.run(C);
  for (auto& r : repl) { C.free(*r.first); *r.first = r.second; }
  for (auto& b : tmp) C.free(b);
  for (auto& b : P) C.free(b);
  weighted = true;
  CUDA_CHECK(cudaGetLastError());
  C.sync();
  C.flush();
}

// ---------------------------------------------------------------------------
// h2_matvec (krylov.py:119-159) over tree-sorted vectors
// ---------------------------------------------------------------------------
void H2::drop_plan() {
  if (!plan.valid) return;
  for (Blk* b : {&plan.desc, &plan.xin, &plan.yout, &plan.yv, &plan.zv}) {
    ctx->free(*b);
    *b = Blk();
  }
  plan.launches.clear();
  plan.valid = false;
}

// The block lists (one SpmvRow per output segment, its SpmvTerms in the
// reference's summation order) depend only on the operators, so they are
// built and uploaded once; a matvec is then two vector copies (x in, y out of
// the plan's staging vectors) and one launch per dependent stage: leaf P2M,
// M2M per level, M2L + L2L per level, P2P + L2P.
void H2::matvec(const double* xs, double* ys) {
  Ctx& C = *ctx;
  Tree& T = *tree;
  IFMM_ASSERT(!consumed, "matvec on operators whose blocks moved into a graph");
  if (!plan.valid) {
    std::vector<long long> off(T.nc, -1);
    long long tot = 0;
    for (int c = 0; c < T.nc; ++c)
      if (rank[c] > 0 && T.level[c] >= 2) { off[c] = tot; tot += rank[c]; }
    plan.yv = C.alloc(1, (int)std::max<long long>(tot, 1));
    plan.zv = C.alloc(1, (int)std::max<long long>(tot, 1));
    const int bd = kern.bd();
    plan.xin = C.alloc(1, std::max(bd * T.n_points, 1));
    plan.yout = C.alloc(1, std::max(bd * T.n_points, 1));
    const double* px = plan.xin.p;
    double* py = plan.yout.p;
    double* yv = plan.yv.p;
    double* zv = plan.zv.p;
    std::vector<SpmvRow> rows;
    std::vector<SpmvTerm> terms;
    size_t stage0 = 0;
    double bytes = 0.0;
    auto term = [&](const Blk& B, int trans, const double* in) {
      terms.push_back({B.p, B.r, B.c, B.c, trans, in});
      bytes += 8.0 * B.r * B.c;
    };
    auto stage = [&]() {
      if (rows.size() > stage0) plan.launches.push_back({stage0, (int)(rows.size() - stage0)});
      stage0 = rows.size();
    };
    const bool has_far = T.depth >= 2;
    if (has_far) {
      for (int c : T.leaves()) {  // upward leaf: y = V^T x
        rows.push_back({yv + off[c], rank[c], (int)terms.size(), 1, 0});
        term(leaf_v[c], 1, px + (size_t)bd * T.start[c]);
      }
      stage();
      for (int l = T.depth - 1; l >= 2; --l) {
        for (int p : T.levels[l]) {
          SpmvRow r{yv + off[p], rank[p], (int)terms.size(), 0, 0};
          for (int c : T.children[p]) {
            term(tvt[c], 0, yv + off[c]);
            r.nt++;
          }
          rows.push_back(r);
        }
        stage();
      }
      for (int l = 2; l <= T.depth; ++l) {
        for (int c : T.levels[l]) {
          SpmvRow r{zv + off[c], rank[c], (int)terms.size(), 0, 0};
          for (int q : T.inters[c]) {
            term(coupling.at(key2(c, q)), 0, yv + off[q]);
            r.nt++;
          }
          if (l > 2) {
            term(tu[c], 0, zv + off[T.parent[c]]);
            r.nt++;
          }
          rows.push_back(r);
        }
        stage();
      }
    }
    for (int c : T.leaves()) {
      SpmvRow r{py + (size_t)bd * T.start[c], bd * (T.stop[c] - T.start[c]), (int)terms.size(), 0, 0};
      for (int q : T.nbrs[c]) {
        term(near.at(key2(c, q)), 0, px + (size_t)bd * T.start[q]);
        r.nt++;
      }
      if (has_far) {
        term(leaf_u[c], 0, zv + off[c]);
        r.nt++;
      }
      rows.push_back(r);
    }
    stage();
    static_assert(sizeof(SpmvRow) % 8 == 0 && sizeof(SpmvTerm) % 8 == 0, "descriptor alignment");
    const size_t rb = rows.size() * sizeof(SpmvRow), tb = terms.size() * sizeof(SpmvTerm);
    plan.desc = C.alloc(1, (int)((rb + tb) / 8 + 1));
    CUDA_CHECK(cudaMemcpyAsync(plan.desc.p, rows.data(), rb, cudaMemcpyHostToDevice, C.st));
    CUDA_CHECK(cudaMemcpyAsync((char*)plan.desc.p + rb, terms.data(), tb, cudaMemcpyHostToDevice,
                               C.st));
    C.sync();  // the host vectors go out of scope
    plan.n_rows = rows.size();
    plan.n_terms = terms.size();
    plan.bytes = bytes;
    plan.valid = true;
  }
  const size_t nb = (size_t)kern.bd() * T.n_points * sizeof(double);
  CUDA_CHECK(cudaMemcpyAsync(plan.xin.p, xs, nb, cudaMemcpyDeviceToDevice, C.st));
  const SpmvRow* dr = reinterpret_cast<const SpmvRow*>(plan.desc.p);
  const SpmvTerm* dt = reinterpret_cast<const SpmvTerm*>((const char*)plan.desc.p +
                                                         plan.n_rows * sizeof(SpmvRow));
  cudaEvent_t ka = nullptr;
  C.kt_begin(K_SPMV, plan.bytes, &ka);
  for (auto& L : plan.launches) launch_spmv(dr + L.first, L.second, dt, 1, 1, C.st);
  C.kt_end(K_SPMV, plan.bytes, ka);
  C.launches += (long long)plan.launches.size();
  CUDA_CHECK(cudaMemcpyAsync(ys, plan.yout.p, nb, cudaMemcpyDeviceToDevice, C.st));
  CUDA_CHECK(cudaGetLastError());
}

// ---------------------------------------------------------------------------
// Morton-range partitioned h2_matvec (one rank's share).  A rank
// owns the points [p_lo, p_hi) of the tree order (whole leaves).
//   phase 0: partial multipoles y of every cluster whose point range meets
//            the rank's range (leaves: own only; parents: sum over children,
//            out-of-range children contribute their -- zero -- local y).
//            The caller sums yv over ranks (NCCL all-reduce).
//   phase 1: locals z of the clusters meeting the range from the full y
//            (M2L) and the parent's z (L2L, the parent meets the range too),
//            then the rows of the own leaves: L2P + P2P over the neighbour
//            leaves' x (xs must be the full sorted vector: the halo).  Rows
//            outside the range are left untouched.
// yv: device vector of length multipole_size(), offsets by cluster id.
long long H2::multipole_size() const {
  long long tot = 0;
  for (int c = 0; c < tree->nc; ++c)
    if (rank[c] > 0 && tree->level[c] >= 2) tot += rank[c];
  return tot;
}

void H2::matvec_part(const double* xs, double* ys, double* yvp, int phase, long long p_lo,
                     long long p_hi) {
  Ctx& C = *ctx;
  Tree& T = *tree;
  std::vector<long long> off(T.nc, -1);
  long long tot = 0;
  for (int c = 0; c < T.nc; ++c)
    if (rank[c] > 0 && T.level[c] >= 2) { off[c] = tot; tot += rank[c]; }
  auto meets = [&](int c) { return T.start[c] < p_hi && T.stop[c] > p_lo; };
  auto run = [&](std::vector<SpmvRow>& rows, std::vector<SpmvTerm>& terms) {
    if (rows.empty()) return;
    SpmvTerm* dt = C.stage.push_vec(C, terms);
    SpmvRow* dr = C.stage.push_vec(C, rows);
    launch_spmv(dr, (int)rows.size(), dt, 1, 1, C.st);
    rows.clear(); terms.clear();
  };
  std::vector<SpmvRow> rows;
  std::vector<SpmvTerm> terms;
  const bool has_far = T.depth >= 2;
  if (phase == 0) {
    if (!has_far) return;
    for (int c : T.leaves()) {
      if (!(T.start[c] >= p_lo && T.stop[c] <= p_hi) || off[c] < 0) continue;
      SpmvRow r{yvp + off[c], rank[c], (int)terms.size(), 1, 0};
      terms.push_back({leaf_v[c].p, leaf_v[c].r, leaf_v[c].c, leaf_v[c].c, 1, xs + T.start[c]});
      rows.push_back(r);
    }
    run(rows, terms);
    for (int l = T.depth - 1; l >= 2; --l) {
      for (int p : T.levels[l]) {
        if (!meets(p) || off[p] < 0) continue;
        SpmvRow r{yvp + off[p], rank[p], (int)terms.size(), 0, 0};
        for (int c : T.children[p]) {
          if (!meets(c) || off[c] < 0) continue;
          terms.push_back({tvt[c].p, tvt[c].r, tvt[c].c, tvt[c].c, 0, yvp + off[c]});
          r.nt++;
        }
        rows.push_back(r);
      }
      run(rows, terms);
    }
    CUDA_CHECK(cudaGetLastError());
    C.flush();
    return;
  }
  Blk zv = C.alloc(1, (int)std::max<long long>(tot, 1));
  if (has_far) {
    for (int l = 2; l <= T.depth; ++l) {
      for (int c : T.levels[l]) {
        if (!meets(c) || off[c] < 0) continue;
        SpmvRow r{zv.p + off[c], rank[c], (int)terms.size(), 0, 0};
        for (int q : T.inters[c]) {
          if (off[q] < 0) continue;
          const Blk& K = coupling.at(key2(c, q));
          terms.push_back({K.p, K.r, K.c, K.c, 0, yvp + off[q]});
          r.nt++;
        }
        if (l > 2) {
          const int p = T.parent[c];
          terms.push_back({tu[c].p, tu[c].r, tu[c].c, tu[c].c, 0, zv.p + off[p]});
          r.nt++;
        }
        rows.push_back(r);
      }
      run(rows, terms);
    }
  }
  for (int c : T.leaves()) {
    if (!(T.start[c] >= p_lo && T.stop[c] <= p_hi)) continue;
    const int m = T.stop[c] - T.start[c];
    SpmvRow r{ys + T.start[c], m, (int)terms.size(), 0, 0};
    for (int q : T.nbrs[c]) {
      const Blk& S = near.at(key2(c, q));
      terms.push_back({S.p, S.r, S.c, S.c, 0, xs + T.start[q]});
      r.nt++;
    }
    if (has_far && off[c] >= 0) {
      terms.push_back({leaf_u[c].p, leaf_u[c].r, leaf_u[c].c, leaf_u[c].c, 0, zv.p + off[c]});
      r.nt++;
    }
    rows.push_back(r);
  }
  run(rows, terms);
  C.free(zv);
  CUDA_CHECK(cudaGetLastError());
  C.flush();
}

}  // namespace ifmm
