// Level-by-level elimination of the extended graph (factor.py:176-578).
//
// Host C++ owns the graph structure (node sizes, edge map, sorted
// row/col adjacency) and makes every structural decision exactly as the
// reference does; all arithmetic runs on the device:
//   per cluster (Morton order, factor.py:249-256):
//     pivot assembly + LU (factor.py:268-274)        -> lu_kernel / lu_blocked
//     X = P^{-1}[E(x,b);0 | 0;-I] for all sources    -> one multi-RHS LU solve
//     Schur fill F = -[E(a,x)] X[:m] (+ own-y rows)  -> one grouped DMMA GEMM
//     neighbour fill scatter-add                     -> one batched copy/add
//     well-separated fill compression                -> one batched Jacobi SVD
//     per fill pair (sorted, factor.py:321-326):
//       basis unions (ACA + QR-QR-SVD)               -> one batched union launch
//       rebase of every y-edge                       -> one grouped GEMM
//       K-edge rewrite                               -> grouped GEMMs
//   merge_to_parent (factor.py:525-578)              -> batched tile copies
//   top-level LU (factor.py:233-246)                 -> blocked LU
#include <algorithm>
#include <chrono>
#include <cmath>
#include <map>
#include <random>
#include <cstdio>
#include <cstdlib>

#include "engine.h"

namespace ifmm {

static constexpr int TOP_TAG = 0x7fffffff - 1;

// IFMM_TRACE=<file>: per-pair decision trace (debug / parity triage)
// IFMM_PROFILE=1: stream-synchronised phase timers (diagnostics; perturbs
// overlap, never used for reported numbers)
enum { PH_LU = 0, PH_XSOLVE, PH_SCHUR, PH_ADD, PH_FILLSVD, PH_UNION, PH_REBASE, PH_NEWK, PH_MERGE,
       PH_TOP, PH_HOST, PH_N };
double g_prof[PH_N];
static bool prof_on() {
  static int on = -1;
  if (on < 0) { const char* p = getenv("IFMM_PROFILE"); on = (p && *p == '1') ? 1 : 0; }
  return on == 1;
}
struct Phase {
  Ctx& C;
  int id;
  std::chrono::steady_clock::time_point t0;
  Phase(Ctx& c, int i) : C(c), id(i) {
    if (prof_on()) { C.sync(); t0 = std::chrono::steady_clock::now(); }
  }
  ~Phase() {
    if (prof_on()) {
      C.sync();
      g_prof[id] += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    }
  }
};

static FILE* trace_file() {
  static FILE* f = nullptr;
  static bool init = false;
  if (!init) {
    init = true;
    const char* p = getenv("IFMM_TRACE");
    if (p && *p) f = fopen(p, "w");
  }
  return f;
}

// ---------------------------------------------------------------------------
// LU helpers
// ---------------------------------------------------------------------------
void lu_any(Ctx& C, double* A, int n, int* piv, int tag) {
  if (n <= 0) return;
  if (n <= 160) {
    std::vector<LuDesc> d(1);
    d[0].A = A; d[0].n = n; d[0].lda = n; d[0].piv = piv; d[0].tag = tag;
    LuDesc* dd = C.stage.push_vec(C, d);
    cudaEvent_t ka = nullptr;
    const double fl = 2.0 / 3.0 * (double)n * n * n;
    C.kt_begin(K_LU, fl, &ka);
    launch_lu(dd, 1, C.d_status, C.st);
    C.kt_end(K_LU, fl, ka);
    C.launches++;
  } else {
    lu_blocked(C, A, n, n, piv, tag);
  }
  CUDA_CHECK(cudaGetLastError());
}

static void lusolve(Ctx& C, const double* LU, const int* piv, int n, double* X, int nrhs) {
  if (n <= 0 || nrhs <= 0) return;
  std::vector<LuSolveDesc> d(1);
  d[0].LU = LU; d[0].piv = piv; d[0].n = n; d[0].lda = n; d[0].X = X; d[0].nrhs = nrhs;
  d[0].ldx = nrhs;
  LuSolveDesc* dd = C.stage.push_vec(C, d);
  cudaEvent_t ka = nullptr;
  const double fl = 2.0 * n * n * (double)nrhs;
  C.kt_begin(K_LUSOLVE, fl, &ka);
  launch_lusolve(dd, 1, nrhs, C.st, n);
  C.kt_end(K_LUSOLVE, fl, ka);
  C.launches++;
  CUDA_CHECK(cudaGetLastError());
}

// ---------------------------------------------------------------------------
// fill factors and basis updates
// ---------------------------------------------------------------------------
struct FillFac {
  const double* U = nullptr;  // m x r col-major (ld m)
  const double* S = nullptr;
  const double* V = nullptr;  // n x r col-major (ld n)
  int m = 0, n = 0, rank = 0;
};

struct BU {  // BasisUpdate (lowrank.py:22-51)
  bool identity = true;
  int m = 0, k_old = 0, k_f = 0, rank = 0, cap = 0;
  Blk NB;  // col-major m x cap (computed) -- unused when identity
  Blk NW;  // 1 x cap
  Blk OM;  // cap x k_old row-major
  Blk FM;  // cap x k_f row-major
  Blk W;   // workspace
};

struct PairCtx;

struct Eliminator {
  Ctx& C;
  Graph& g;
  Factor& F;
  double thr;
  std::mt19937_64 rng;
  Blk d_ranks;  // device int scratch
  int d_ranks_cap = 0;
  double flops_gemm = 0, flops_all = 0;

  Eliminator(Ctx& c, Graph& gg, Factor& f, double t, unsigned long long seed)
      : C(c), g(gg), F(f), thr(t), rng(seed) {}

  int* ranks_buf(int n) {
    if (n > d_ranks_cap) {
      C.free(d_ranks);
      d_ranks_cap = std::max(n, 4096);
      d_ranks = C.alloc(1, d_ranks_cap / 2 + 1);
    }
    return reinterpret_cast<int*>(d_ranks.p);
  }

  void run_gemm(GemmBatch& gb) {
    flops_gemm += gb.flops;
    flops_all += gb.flops;
    gb.run(C);
    gb.flops = 0;
  }

  // -------------------------------------------------------------------------
  // union launches (weighted_basis_union, lowrank.py:166-199)
  // -------------------------------------------------------------------------
  struct UReq {
    BU* bu;
    const double* B; int b_r, b_c;
    const Blk* w;
    const double* Fp; int f_r, f_c;
    const double* wf;
    int min_rank;
  };

  void launch_unions(std::vector<UReq>& reqs) {
    if (reqs.empty()) return;
    int* dr = ranks_buf((int)reqs.size());
    std::vector<UnionDesc> ud;
    double uflops = 0;
    for (size_t i = 0; i < reqs.size(); ++i) {
      UReq& q = reqs[i];
      BU& b = *q.bu;
      b.identity = false;
      b.cap = std::min(b.m, b.k_old + b.k_f);
      C.free(b.NB); C.free(b.NW); C.free(b.OM); C.free(b.FM); C.free(b.W);
      b.NB = C.alloc(std::max(b.cap, 1), b.m);
      b.NW = C.alloc(1, std::max(b.cap, 1));
      b.OM = C.alloc(std::max(b.cap, 1), std::max(b.k_old, 1));
      b.FM = C.alloc(std::max(b.cap, 1), std::max(b.k_f, 1));
      b.W = C.alloc(1, (int)union_work_doubles(b.m, b.k_old, b.k_f));
      UnionDesc d;
      d.B = q.B; d.w = q.w->p; d.F = q.Fp; d.wf = q.wf;
      d.m = b.m; d.k_old = b.k_old; d.k_f = b.k_f;
      d.b_r = q.b_r; d.b_c = q.b_c; d.f_r = q.f_r; d.f_c = q.f_c;
      d.min_rank = q.min_rank;
      d.NB = b.NB.p; d.nb_r = 1; d.nb_c = b.m;
      d.NW = b.NW.p; d.OM = b.OM.p; d.FM = b.FM.p;
      d.rank = dr + i;
      d.work = b.W.p;
      ud.push_back(d);
      // flop estimate: ACA 2mn per step (<= cap steps) + QR/SVD of cap
      const double mm = b.m, nn = b.k_old + b.k_f, s = b.cap;
      const double fl = 2 * mm * nn * s + 2 * mm * s * s + 2 * nn * s * s + 4 * s * s * s + 22 * s * s * s;
      flops_all += fl;
      uflops += fl;
    }
    Phase ph(C, PH_UNION);
    UnionDesc* dud = C.stage.push_vec(C, ud);
    cudaEvent_t ka = nullptr;
    C.kt_begin(K_UNION, uflops, &ka);
    launch_union(dud, (int)ud.size(), thr, C.st);
    C.kt_end(K_UNION, uflops, ka);
    C.launches++;
    CUDA_CHECK(cudaGetLastError());
    const int* hr = C.readback_ints(dr, reqs.size());
    for (size_t i = 0; i < reqs.size(); ++i) {
      reqs[i].bu->rank = hr[i];
      C.free(reqs[i].bu->W);
    }
  }

  void make_identity(BU& b, int m, int k, const Blk& w) {
    b.identity = true;
    b.m = m; b.k_old = k; b.k_f = 0; b.rank = k; b.cap = k;
    C.free(b.OM);
    b.OM = C.alloc(k, k);
    CopyBatch cb;
    cb.eye(b.OM, 1.0);
    cb.run(C);
    (void)w;
  }

  void free_bu(BU& b) {
    C.free(b.NB); C.free(b.NW); C.free(b.OM); C.free(b.FM); C.free(b.W);
  }

  // _extend_update (factor.py:340-358): pad with orthonormalised Gaussian
  // directions carrying zero maps and weight max(thr, 1e-14 max w).
  void extend(BU& b, int kt, const Blk& cur_basis_rowmajor, int basis_is_v, const Blk& cur_w);

  // -------------------------------------------------------------------------
  void cluster_unions(int c, const double* fu, int fu_r, int fu_c, int kfu, const double* wu,
                      const double* fv, int fv_r, int fv_c, int kfv, const double* wv, BU& bu,
                      BU& bv, LevelStats& st, std::vector<UReq>& pending);
  void finish_unions(int c, BU& bu, BU& bv, const double* fu, int fu_r, int fu_c, int kfu,
                     const double* wu, const double* fv, int fv_r, int fv_c, int kfv,
                     const double* wv, LevelStats& st);
  void rebase(int c, BU& bu, BU& bv, int partner);
  void redirect(int cj, int ck, const FillFac* f_kj, const FillFac* f_jk, LevelStats& st);
  void eliminate(int c, LevelStats& st);
  void merge(int level);
  void top();
};

// ---------------------------------------------------------------------------
void Eliminator::extend(BU& b, int kt, const Blk& cur_basis, int basis_is_v, const Blk& cur_w) {
  (void)cur_basis; (void)basis_is_v; (void)cur_w;
  const int m = b.m, k = b.rank;
  const int extra = std::min(kt, m) - k;
  if (extra <= 0) return;
  // Materialise the basis as a computed update (col-major m x cap) if needed
  IFMM_ASSERT(!b.identity, "extend of an identity update must be materialised first");
  // host Gaussians (deterministic stream), device orthogonalisation
  std::normal_distribution<double> nd(0.0, 1.0);
  std::vector<double> G((size_t)m * extra);
  for (auto& x : G) x = nd(rng);
  Blk Gd = C.alloc(m, extra);
  CUDA_CHECK(cudaMemcpyAsync(Gd.p, G.data(), G.size() * 8, cudaMemcpyHostToDevice, C.st));
  // grow capacity
  const int ncap = k + extra;
  Blk NB = C.alloc(ncap, m), NW = C.alloc(1, ncap), OM = C.alloc(ncap, std::max(b.k_old, 1)),
      FM = C.alloc(ncap, std::max(b.k_f, 1));
  CopyBatch cb;
  cb.add(b.NB.p, 1, 1, NB.p, 1, 1, 1, m * k, 0);
  cb.add(b.NW.p, 1, 1, NW.p, 1, 1, 1, k, 0);
  if (b.k_old) {
    cb.add(b.OM.p, b.k_old, 1, OM.p, b.k_old, 1, k, b.k_old, 0);
    cb.add(nullptr, 0, 0, OM.p + (size_t)k * b.k_old, b.k_old, 1, extra, b.k_old, 3);
  }
  if (b.k_f) {
    cb.add(b.FM.p, b.k_f, 1, FM.p, b.k_f, 1, k, b.k_f, 0);
    cb.add(nullptr, 0, 0, FM.p + (size_t)k * b.k_f, b.k_f, 1, extra, b.k_f, 3);
  }
  cb.run(C);
  Blk work = C.alloc(1, 4 * m * (k + extra) + 4 * extra + 64);
  launch_extend(NB.p, m, k, Gd.p, extra, NW.p, thr, work.p, C.st);
  CUDA_CHECK(cudaGetLastError());
  C.free(work);
  C.free(Gd);
  free_bu(b);
  b.NB = NB; b.NW = NW; b.OM = OM; b.FM = FM;
  b.cap = ncap;
  b.rank = ncap;
}

// Launch (or set identity for) the U- and V-side unions of cluster c.
void Eliminator::cluster_unions(int c, const double* fu, int fu_r, int fu_c, int kfu,
                                const double* wu, const double* fv, int fv_r, int fv_c, int kfv,
                                const double* wv, BU& bu, BU& bv, LevelStats& st,
                                std::vector<UReq>& pending) {
  (void)st;
  const int nxn = g.nx[c], nzn = g.nz[c];
  const Blk& Uc = *g.get(nxn, nzn);   // m x k row-major
  const Blk& Vt = *g.get(nzn, nxn);   // k x m row-major  (V = Vt^T)
  const int m = Uc.r, k = Uc.c;
  bu.m = bv.m = m;
  bu.k_old = bv.k_old = k;
  if (kfu > 0) {
    bu.k_f = kfu;
    pending.push_back({&bu, Uc.p, k, 1, &g.su[c], fu, fu_r, fu_c, wu, 0});
  } else {
    make_identity(bu, m, k, g.su[c]);
  }
  if (kfv > 0) {
    bv.k_f = kfv;
    pending.push_back({&bv, Vt.p, 1, m, &g.sv[c], fv, fv_r, fv_c, wv, 0});
  } else {
    make_identity(bv, m, k, g.sv[c]);
  }
}

// Rank equalisation of _cluster_unions (factor.py:378-391).
void Eliminator::finish_unions(int c, BU& bu, BU& bv, const double* fu, int fu_r, int fu_c,
                               int kfu, const double* wu, const double* fv, int fv_r, int fv_c,
                               int kfv, const double* wv, LevelStats& st) {
  if (bu.rank == bv.rank) return;
  const int nxn = g.nx[c], nzn = g.nz[c];
  const Blk& Uc = *g.get(nxn, nzn);
  const Blk& Vt = *g.get(nzn, nxn);
  const int m = Uc.r, k0 = Uc.c;
  int k = std::max(bu.rank, bv.rank);
  std::vector<UReq> re;
  if (bu.rank < k && kfu > 0) re.push_back({&bu, Uc.p, k0, 1, &g.su[c], fu, fu_r, fu_c, wu, k});
  if (bv.rank < k && kfv > 0) re.push_back({&bv, Vt.p, 1, m, &g.sv[c], fv, fv_r, fv_c, wv, k});
  launch_unions(re);
  // identity updates that must grow are materialised as computed updates
  auto materialise = [&](BU& b, const Blk& basis, int is_v, const Blk& w) {
    if (!b.identity) return;
    C.free(b.NB); C.free(b.NW); C.free(b.FM);
    b.NB = C.alloc(b.k_old, m);
    b.NW = C.alloc(1, std::max(b.k_old, 1));
    b.FM = C.alloc(std::max(b.k_old, 1), 1);
    CopyBatch cb;
    // NB col-major m x k: (i,a) at a*m+i
    if (!is_v) cb.add(basis.p, basis.c, 1, b.NB.p, 1, m, m, b.k_old, 0);
    else cb.add(basis.p, 1, basis.c, b.NB.p, 1, m, m, b.k_old, 0);
    cb.add(w.p, 1, 1, b.NW.p, 1, 1, 1, b.k_old, 0);
    cb.run(C);
    b.identity = false;
    b.cap = b.k_old;
  };
  if (bu.rank < k) { materialise(bu, Uc, 0, g.su[c]); extend(bu, k, Uc, 0, g.su[c]); }
  if (bv.rank < k) { materialise(bv, Vt, 1, g.sv[c]); extend(bv, k, Vt, 1, g.sv[c]); }
  if (bu.rank != bv.rank) {
    k = std::min(bu.rank, bv.rank);
    materialise(bu, Uc, 0, g.su[c]);
    materialise(bv, Vt, 1, g.sv[c]);
    bu.rank = bv.rank = k;  // _truncate_update: prefix rows/cols
    st.forced++;
  }
}

// _apply_rebase (factor.py:395-430)
void Eliminator::rebase(int c, BU& bu, BU& bv, int partner) {
  Phase ph(C, PH_REBASE);
  if (FILE* tf = trace_file()) fprintf(tf, "R %d %d %d %d\n", c, bu.k_old, bu.rank, bv.rank);
  const int nxn = g.nx[c], nzn = g.nz[c], nyn = g.ny[c];
  const int py = g.ny[partner];
  const int m = g.size[nxn];
  const int kn = bu.rank, ko = bu.k_old;
  IFMM_ASSERT(bu.rank == bv.rank, "unequal U/V ranks in rebase");
  CopyBatch cb;
  GemmBatch gb;
  // new U (m x kn row-major) and V^T (kn x m row-major)
  if (!bu.identity || kn != ko) {
    Blk nu = C.alloc(m, kn);
    cb.add(bu.NB.p, 1, m, nu.p, kn, 1, m, kn, 0);
    g.set(nxn, nzn, nu);
  }
  if (!bv.identity || kn != ko) {
    Blk nv = C.alloc(kn, m);
    cb.add(bv.NB.p, m, 1, nv.p, m, 1, kn, m, 0);
    g.set(nzn, nxn, nv);
  }
  if (!bu.identity || kn != ko) {
    Blk w = C.alloc(1, kn);
    cb.add(bu.NW.p, 1, 1, w.p, 1, 1, 1, kn, 0);
    C.free(g.su[c]);
    g.su[c] = w;
  }
  if (!bv.identity || kn != ko) {
    Blk w = C.alloc(1, kn);
    cb.add(bv.NW.p, 1, 1, w.p, 1, 1, 1, kn, 0);
    C.free(g.sv[c]);
    g.sv[c] = w;
  }
  IFMM_ASSERT(!g.get(nyn, nyn), "live cluster with a y-y self edge");
  const bool rid = bu.identity && kn == ko, tid = bv.identity && kn == ko;
  if (!rid) {
    std::vector<int> rs(g.rows[nyn].begin(), g.rows[nyn].end());
    for (int b : rs) {
      if (b == nzn || b == py) continue;
      const Blk E = *g.get(nyn, b);
      Blk nb = C.alloc(kn, E.c);
      gb.add(bu.OM.p, ko, 0, E.p, E.c, 0, nb.p, E.c, kn, E.c, ko, 1.0, 0.0);
      g.set(nyn, b, nb);
    }
  }
  if (!tid) {
    std::vector<int> cs(g.cols[nyn].begin(), g.cols[nyn].end());
    for (int a : cs) {
      if (a == nzn || a == py) continue;
      const Blk E = *g.get(a, nyn);
      Blk nb = C.alloc(E.r, kn);
      gb.add(E.p, E.c, 0, bv.OM.p, ko, 1, nb.p, kn, E.r, kn, ko, 1.0, 0.0);
      g.set(a, nyn, nb);
    }
  }
  cb.run(C);
  run_gemm(gb);
  Blk e1 = g.take(nzn, nyn), e2 = g.take(nyn, nzn);
  C.free(e1); C.free(e2);
  g.size[nzn] = kn;
  g.size[nyn] = kn;
  Blk a = C.alloc(kn, kn), b2 = C.alloc(kn, kn);
  CopyBatch ce;
  ce.eye(a, -1.0);
  ce.eye(b2, -1.0);
  ce.run(C);
  g.set(nzn, nyn, a);
  g.set(nyn, nzn, b2);
  if (!rid) {
    // keep r (kn x ko) for the solve replay
    Blk r = C.alloc(kn, ko);
    CopyBatch cr;
    cr.add(bu.OM.p, ko, 1, r.p, ko, 1, kn, ko, 0);
    cr.run(C);
    F.rebases.push_back({nyn, r});
    F.events.push_back({1, (int)F.rebases.size() - 1});
  }
}

// redirect_fillin (factor.py:433-522)
void Eliminator::redirect(int cj, int ck, const FillFac* f_kj, const FillFac* f_jk,
                          LevelStats& st) {
  const bool ej = g.dead[cj], ek = g.dead[ck];
  IFMM_ASSERT(!(ej && ek), "both-eliminated fills are added, not redirected");
  const int r1 = f_kj ? f_kj->rank : 0;
  const int r2 = f_jk ? f_jk->rank : 0;
  if (r1 == 0 && r2 == 0) {
    st.dropped++;
    if (FILE* tf = trace_file()) fprintf(tf, "D %d %d\n", cj, ck);
    return;
  }
  st.compressed++;
  st.ranks.push_back(std::max(r1, r2));
  if (FILE* tf = trace_file()) fprintf(tf, "P %d %d %d %d %d %d\n", cj, ck, r1, r2, (int)ej, (int)ek);
  const int yj = g.ny[cj], yk = g.ny[ck];
  Blk* pkj = g.get(yk, yj);
  Blk* pjk = g.get(yj, yk);
  Blk old_kj = pkj ? *pkj : Blk();
  Blk old_jk = pjk ? *pjk : Blk();
  const bool has_kj = pkj != nullptr, has_jk = pjk != nullptr;
  // keep old blocks alive through the rebases (set() on partner edges
  // happens only below)
  if (!ej && !ek) {
    BU uj, vj, uk, vk;
    std::vector<UReq> pend;
    // j: U-fill = U(F_jk) (m_j x r2, w s_jk); V-fill = V(F_kj) (m_j x r1, w s_kj)
    const double* Ujk = r2 ? f_jk->U : nullptr; const int ldUjk = r2 ? f_jk->m : 0;
    const double* Vkj = r1 ? f_kj->V : nullptr; const int ldVkj = r1 ? f_kj->n : 0;
    const double* Ukj = r1 ? f_kj->U : nullptr; const int ldUkj = r1 ? f_kj->m : 0;
    const double* Vjk = r2 ? f_jk->V : nullptr; const int ldVjk = r2 ? f_jk->n : 0;
    const double* sjk = r2 ? f_jk->S : nullptr;
    const double* skj = r1 ? f_kj->S : nullptr;
    cluster_unions(cj, Ujk, 1, ldUjk, r2, sjk, Vkj, 1, ldVkj, r1, skj, uj, vj, st, pend);
    cluster_unions(ck, Ukj, 1, ldUkj, r1, skj, Vjk, 1, ldVjk, r2, sjk, uk, vk, st, pend);
    launch_unions(pend);
    finish_unions(cj, uj, vj, Ujk, 1, ldUjk, r2, sjk, Vkj, 1, ldVkj, r1, skj, st);
    finish_unions(ck, uk, vk, Ukj, 1, ldUkj, r1, skj, Vjk, 1, ldVjk, r2, sjk, st);
    const int kjo = g.size[yj], kko = g.size[yk];
    rebase(cj, uj, vj, ck);
    rebase(ck, uk, vk, cj);
    const int kjn = uj.rank, kkn = uk.rank;
    // new_kj = rk old_kj tj^T + (rk' s_kj) tj'^T   (kkn x kjn)
    // new_jk = rj old_jk tk^T + (rj' s_jk) tk'^T   (kjn x kkn)
    Blk nkj = C.alloc(kkn, kjn), njk = C.alloc(kjn, kkn);
    Blk t1 = has_kj ? C.alloc(kko, kjn) : Blk(), t2 = has_jk ? C.alloc(kjo, kkn) : Blk();
    GemmBatch ga, gb2, gc;
    if (has_kj) {
      ga.add(old_kj.p, kjo, 0, vj.OM.p, kjo, 1, t1.p, kjn, kko, kjn, kjo, 1.0, 0.0);
      gb2.add(uk.OM.p, kko, 0, t1.p, kjn, 0, nkj.p, kjn, kkn, kjn, kko, 1.0, 0.0);
    }
    if (has_jk) {
      ga.add(old_jk.p, kko, 0, vk.OM.p, kko, 1, t2.p, kkn, kjo, kkn, kko, 1.0, 0.0);
      gb2.add(uj.OM.p, kjo, 0, t2.p, kkn, 0, njk.p, kkn, kjn, kkn, kjo, 1.0, 0.0);
    }
    if (r1 > 0)
      gc.add(uk.FM.p, uk.k_f, 0, vj.FM.p, vj.k_f, 1, nkj.p, kjn, kkn, kjn, r1, 1.0,
             has_kj ? 1.0 : 0.0, skj);
    if (r2 > 0)
      gc.add(uj.FM.p, uj.k_f, 0, vk.FM.p, vk.k_f, 1, njk.p, kkn, kjn, kkn, r2, 1.0,
             has_jk ? 1.0 : 0.0, sjk);
    Phase ph(C, PH_NEWK);
    CopyBatch z;
    if (!has_kj && r1 == 0) z.zero(nkj);
    if (!has_jk && r2 == 0) z.zero(njk);
    z.run(C);
    run_gemm(ga);
    run_gemm(gb2);
    run_gemm(gc);
    g.set(yk, yj, nkj);
    g.set(yj, yk, njk);
    C.free(t1); C.free(t2);
    for (BU* b : {&uj, &vj, &uk, &vk}) free_bu(*b);
  } else {
    const int live = ej ? ck : cj, deadc = ej ? cj : ck;
    const FillFac* fu = ej ? f_kj : f_jk;  // rows on x_live, cols on y_dead
    const FillFac* fv = ej ? f_jk : f_kj;  // rows on y_dead, cols on x_live
    const int ru = fu ? fu->rank : 0, rv = fv ? fv->rank : 0;
    const int nd = g.size[g.ny[deadc]];
    BU bu, bv;
    std::vector<UReq> pend;
    const double* Ul = ru ? fu->U : nullptr; const int ldUl = ru ? fu->m : 0;
    const double* sl = ru ? fu->S : nullptr;
    const double* Wl = ru ? fu->V : nullptr;  // nd x ru col-major (ld fu->n == nd)
    const double* Ud = rv ? fv->U : nullptr;  // nd x rv col-major (ld fv->m == nd)
    const double* sd = rv ? fv->S : nullptr;
    const double* Vl = rv ? fv->V : nullptr; const int ldVl = rv ? fv->n : 0;
    cluster_unions(live, Ul, 1, ldUl, ru, sl, Vl, 1, ldVl, rv, sd, bu, bv, st, pend);
    launch_unions(pend);
    finish_unions(live, bu, bv, Ul, 1, ldUl, ru, sl, Vl, 1, ldVl, rv, sd, st);
    const int klo = g.size[g.ny[live]];
    rebase(live, bu, bv, deadc);
    const int kln = bu.rank;
    const int ylive = g.ny[live], ydead = g.ny[deadc];
    const bool live_is_k = live == ck;
    const Blk old_ld = live_is_k ? old_kj : old_jk;  // (y_live, y_dead): klo x nd
    const Blk old_dl = live_is_k ? old_jk : old_kj;  // (y_dead, y_live): nd x klo
    const bool has_ld = live_is_k ? has_kj : has_jk;
    const bool has_dl = live_is_k ? has_jk : has_kj;
    Blk nld = C.alloc(kln, nd), ndl = C.alloc(nd, kln);
    GemmBatch ga, gb2;
    if (has_ld) ga.add(bu.OM.p, klo, 0, old_ld.p, nd, 0, nld.p, nd, kln, nd, klo, 1.0, 0.0);
    if (has_dl) ga.add(old_dl.p, klo, 0, bv.OM.p, klo, 1, ndl.p, kln, nd, kln, klo, 1.0, 0.0);
    if (ru > 0)
      gb2.add(bu.FM.p, bu.k_f, 0, Wl, nd, 0, nld.p, nd, kln, nd, ru, 1.0, has_ld ? 1.0 : 0.0, sl);
    if (rv > 0)
      gb2.add(Ud, nd, 1, bv.FM.p, bv.k_f, 1, ndl.p, kln, nd, kln, rv, 1.0, has_dl ? 1.0 : 0.0,
              sd);
    Phase ph(C, PH_NEWK);
    CopyBatch z;
    if (!has_ld && ru == 0) z.zero(nld);
    if (!has_dl && rv == 0) z.zero(ndl);
    z.run(C);
    run_gemm(ga);
    run_gemm(gb2);
    g.set(ylive, ydead, nld);
    g.set(ydead, ylive, ndl);
    free_bu(bu);
    free_bu(bv);
  }
}

// _eliminate_cluster (factor.py:259-326)
void Eliminator::eliminate(int c, LevelStats& st) {
  if (FILE* tf = trace_file()) fprintf(tf, "E %d %d %d\n", c, g.size[g.nx[c]], g.size[g.nz[c]]);
  const int nxn = g.nx[c], nzn = g.nz[c], nyn = g.ny[c];
  const int m = g.size[nxn], k = g.size[nzn], n = m + k;
  Blk D = g.take(nxn, nxn);
  Blk U = g.take(nxn, nzn);
  Blk Vt = g.take(nzn, nxn);
  Blk e1 = g.take(nzn, nyn), e2 = g.take(nyn, nzn);
  C.free(e1); C.free(e2);
  Blk P = C.alloc(n, n);
  Phase* ph = new Phase(C, PH_LU);
  {
    CopyBatch cb;
    cb.copy(D, P, 0, 0);
    cb.copy(U, P, 0, m);
    cb.copy(Vt, P, m, 0);
    cb.add(nullptr, 0, 0, P.p + (size_t)m * n + m, n, 1, k, k, 3);
    cb.run(C);
  }
  C.free(D); C.free(U); C.free(Vt);
  int pc;
  int* piv = C.arena.alloc_int(n, &pc);
  lu_any(C, P.p, n, piv, c);
  flops_gemm += 2.0 / 3.0 * (double)n * n * n;
  flops_all += 2.0 / 3.0 * (double)n * n * n;
  delete ph;
  ph = new Phase(C, PH_XSOLVE);

  ElimEv ev;
  ev.nx = nxn; ev.nz = nzn; ev.ny = nyn; ev.m = m; ev.k = k;
  ev.LU = P; ev.piv = piv; ev.piv_cls = pc;
  std::vector<Blk> srcB, tgtB;
  int Csrc = 0, Rtgt = 0;
  for (int b : std::vector<int>(g.rows[nxn].begin(), g.rows[nxn].end())) {
    Blk E = g.take(nxn, b);
    ev.src.push_back(b); ev.src_off.push_back(Csrc); ev.src_w.push_back(E.c);
    Csrc += E.c;
    srcB.push_back(E);
  }
  for (int a : std::vector<int>(g.cols[nxn].begin(), g.cols[nxn].end())) {
    Blk E = g.take(a, nxn);
    ev.tgt.push_back(a); ev.tgt_off.push_back(Rtgt); ev.tgt_h.push_back(E.r);
    Rtgt += E.r;
    tgtB.push_back(E);
  }
  IFMM_ASSERT(g.rows[nzn].empty() && g.cols[nzn].empty(), "z node unexpectedly has extra edges");
  ev.Scat = C.alloc(m, std::max(Csrc, 1));
  ev.Tstk = C.alloc(std::max(Rtgt, 1), m);
  const int NC = Csrc + k, NR = Rtgt + k;
  Blk X = C.alloc(n, NC);
  {
    CopyBatch cb;
    for (size_t i = 0; i < srcB.size(); ++i) {
      cb.add(srcB[i].p, srcB[i].c, 1, ev.Scat.p + ev.src_off[i], std::max(Csrc, 1), 1, m,
             srcB[i].c, 0);
      cb.add(srcB[i].p, srcB[i].c, 1, X.p + ev.src_off[i], NC, 1, m, srcB[i].c, 0);
    }
    for (size_t i = 0; i < tgtB.size(); ++i)
      cb.add(tgtB[i].p, tgtB[i].c, 1, ev.Tstk.p + (size_t)ev.tgt_off[i] * m, m, 1, tgtB[i].r, m,
             0);
    cb.add(nullptr, 0, 0, X.p + (size_t)m * NC, NC, 1, k, Csrc, 3);   // 0 below sources
    cb.add(nullptr, 0, 0, X.p + Csrc, NC, 1, m, k, 3);                // 0 above -I
    cb.add(nullptr, 0, 0, X.p + (size_t)m * NC + Csrc, NC, 1, k, k, 2, -1.0);  // -I
    cb.run(C);
  }
  for (auto& b : srcB) C.free(b);
  for (auto& b : tgtB) C.free(b);
  g.dead[c] = 1;

  lusolve(C, P.p, piv, n, X.p, NC);
  flops_gemm += 2.0 * n * n * (double)NC;
  flops_all += 2.0 * n * n * (double)NC;
  delete ph;
  ph = new Phase(C, PH_SCHUR);

  // Schur fill: F = [-Tstk X[:m] ; X[m:]]   (NR x NC)
  Blk Fm = C.alloc(NR, NC);
  {
    GemmBatch gb;
    gb.add(ev.Tstk.p, m, 0, X.p, NC, 0, Fm.p, NC, Rtgt, NC, m, -1.0, 0.0);
    run_gemm(gb);
    CopyBatch cb;
    cb.add(X.p + (size_t)m * NC, NC, 1, Fm.p + (size_t)Rtgt * NC, NC, 1, k, NC, 0);
    cb.run(C);
  }
  C.free(X);

  delete ph;
  ph = new Phase(C, PH_ADD);
  F.elims.push_back(std::move(ev));
  F.events.push_back({0, (int)F.elims.size() - 1});
  const ElimEv& E = F.elims.back();

  // classification (factor.py:301-318)
  std::vector<int> A_nodes(E.tgt), A_off(E.tgt_off), A_h(E.tgt_h);
  A_nodes.push_back(nyn); A_off.push_back(Rtgt); A_h.push_back(k);
  std::vector<int> B_nodes(E.src), B_off(E.src_off), B_w(E.src_w);
  B_nodes.push_back(nyn); B_off.push_back(Csrc); B_w.push_back(k);
  struct Stash { int ro, co, h, w; };
  std::map<std::pair<int, int>, Stash> stash;
  CopyBatch adds;
  for (size_t ai = 0; ai < A_nodes.size(); ++ai) {
    const int a = A_nodes[ai], ca = g.owner[a];
    for (size_t bi = 0; bi < B_nodes.size(); ++bi) {
      const int b = B_nodes[bi], cbc = g.owner[b];
      const double* sub = Fm.p + (size_t)A_off[ai] * NC + B_off[bi];
      if ((g.dead[ca] && g.dead[cbc]) || g.tree->adjacent(ca, cbc)) {
        Blk* ex = g.get(a, b);
        if (ex) {
          IFMM_ASSERT(ex->r == A_h[ai] && ex->c == B_w[bi], "fill shape mismatch");
          adds.add(sub, NC, 1, ex->p, ex->c, 1, A_h[ai], B_w[bi], 1);
        } else {
          Blk nb = C.alloc(A_h[ai], B_w[bi]);
          adds.add(sub, NC, 1, nb.p, nb.c, 1, A_h[ai], B_w[bi], 0);
          g.set(a, b, nb);
        }
        st.added++;
      } else {
        stash[{ca, cbc}] = {A_off[ai], B_off[bi], A_h[ai], B_w[bi]};
      }
    }
  }
  adds.run(C);
  delete ph;
  ph = nullptr;

  if (!stash.empty()) {
    Phase* ps = new Phase(C, PH_FILLSVD);
    // compress every stashed fill in one batched Jacobi SVD launch
    std::vector<std::pair<std::pair<int, int>, Stash>> items(stash.begin(), stash.end());
    const int ns = (int)items.size();
    int maxdim = 0;
    for (auto& it : items) maxdim = std::max(maxdim, std::max(it.second.h, it.second.w));
    const int smem_dim = std::min(maxdim, 110);
    const size_t smem_d = svd_smem_doubles(smem_dim);
    size_t tot = 0;
    std::vector<size_t> uo(ns), so(ns), vo(ns), wo(ns);
    for (int i = 0; i < ns; ++i) {
      const Stash& s = items[i].second;
      const int mn = std::min(s.h, s.w);
      uo[i] = tot; tot += (size_t)s.h * mn;
      so[i] = tot; tot += mn;
      vo[i] = tot; tot += (size_t)s.w * mn;
      wo[i] = tot;
      if (svd_work_doubles(s.h, s.w) > smem_d) tot += svd_work_doubles(s.h, s.w);
      const double mm = std::max(s.h, s.w), nn = std::min(s.h, s.w);
      flops_all += 4 * mm * nn * nn + 22 * nn * nn * nn;
    }
    double sflops = 0;
    for (int i = 0; i < ns; ++i) {
      const double mm = std::max(items[i].second.h, items[i].second.w);
      const double nn = std::min(items[i].second.h, items[i].second.w);
      sflops += 4 * mm * nn * nn + 22 * nn * nn * nn;
    }
    Blk ws = C.alloc(1, (int)std::max<size_t>(tot, 1));
    int* dr = ranks_buf(ns);
    std::vector<SvdDesc> sd(ns);
    for (int i = 0; i < ns; ++i) {
      const Stash& s = items[i].second;
      sd[i].src = Fm.p + (size_t)s.ro * NC + s.co;
      sd[i].m = s.h; sd[i].n = s.w; sd[i].s_r = NC; sd[i].s_c = 1;
      sd[i].U = ws.p + uo[i]; sd[i].S = ws.p + so[i]; sd[i].V = ws.p + vo[i];
      sd[i].rank = dr + i;
      sd[i].work = ws.p + wo[i];
    }
    SvdDesc* dsd = C.stage.push_vec(C, sd);
    cudaEvent_t ka = nullptr;
    C.kt_begin(K_SVD, sflops, &ka);
    launch_svd(dsd, ns, thr, smem_dim, C.st, 0);
    C.kt_end(K_SVD, sflops, ka);
    C.launches++;
    CUDA_CHECK(cudaGetLastError());
    const int* hr = C.readback_ints(dr, ns);
    std::map<std::pair<int, int>, FillFac> fac;
    for (int i = 0; i < ns; ++i) {
      FillFac f;
      f.U = sd[i].U; f.S = sd[i].S; f.V = sd[i].V;
      f.m = sd[i].m; f.n = sd[i].n; f.rank = hr[i];
      fac[items[i].first] = f;
    }
    delete ps;
    std::set<std::pair<int, int>> pairs;
    for (auto& it : items)
      pairs.insert({std::min(it.first.first, it.first.second),
                    std::max(it.first.first, it.first.second)});
    for (auto& pr : pairs) {
      const int cj = pr.first, ck = pr.second;
      auto a = fac.find({ck, cj});
      auto b = fac.find({cj, ck});
      redirect(cj, ck, a == fac.end() ? nullptr : &a->second,
               b == fac.end() ? nullptr : &b->second, st);
    }
    C.flush();
    C.free(ws);
  }
  C.free(Fm);
  C.flush();
}

// merge_to_parent (factor.py:525-578)
void Eliminator::merge(int level) {
  Phase ph(C, PH_MERGE);
  Tree& T = *g.tree;
  std::map<int, int> owner, offs;  // child y node -> parent cluster / offset
  std::map<int, int> px_of;
  for (int p : T.levels[level - 1]) {
    MergeEv mev;
    int off = 0;
    for (int c : T.children[p]) {
      const int cy = g.ny[c];
      offs[cy] = off;
      owner[cy] = p;
      mev.parts.push_back(cy);
      mev.psize.push_back(g.size[cy]);
      off += g.size[cy];
    }
    const int px = g.new_node(off, NK_X, p);
    g.nx[p] = px;
    px_of[p] = px;
    mev.px = px;
    F.merges.push_back(mev);
    F.events.push_back({2, (int)F.merges.size() - 1});
  }
  std::vector<std::pair<int, int>> moved;
  for (auto& kv : owner) {
    const int t = kv.first;
    for (int s : g.rows[t]) moved.push_back({t, s});
  }
  for (auto& kv : owner) {
    const int s = kv.first;
    for (int t : g.cols[s])
      if (!owner.count(t)) moved.push_back({t, s});
  }
  CopyBatch zero, tile;
  std::vector<Blk> to_free;
  for (auto& e : moved) {
    const int t = e.first, s = e.second;
    Blk blk = g.take(t, s);
    const bool ot = owner.count(t), os = owner.count(s);
    int tt = ot ? px_of[owner[t]] : t;
    int ss = os ? px_of[owner[s]] : s;
    Blk* tg = g.get(tt, ss);
    if (!tg) {
      Blk nb = C.alloc(g.size[tt], g.size[ss]);
      zero.zero(nb);
      g.set(tt, ss, nb);
      tg = g.get(tt, ss);
    }
    const int r0 = ot ? offs[t] : 0, c0 = os ? offs[s] : 0;
    tile.add(blk.p, blk.c, 1, tg->p + (size_t)r0 * tg->c + c0, tg->c, 1, blk.r, blk.c, 1);
    to_free.push_back(blk);  // freed after the tile copies are enqueued
  }
  zero.run(C);
  tile.run(C);
  for (auto& b : to_free) C.free(b);
  C.flush();
}

// _assemble_top (factor.py:233-246)
void Eliminator::top() {
  Phase ph(C, PH_TOP);
  Tree& T = *g.tree;
  std::vector<int> tn;
  if (T.depth >= 2)
    for (int c : T.levels[2]) tn.push_back(g.ny[c]);
  else
    for (int c : T.leaves()) tn.push_back(g.nx[c]);
  std::map<int, int> off;
  int tot = 0;
  for (int t : tn) {
    off[t] = tot;
    F.top_nodes.push_back(t);
    F.top_sizes.push_back(g.size[t]);
    tot += g.size[t];
  }
  if (tot == 0) return;
  F.top_lu = C.alloc(tot, tot);
  CopyBatch z, cb;
  z.zero(F.top_lu);
  for (int t : tn)
    for (int s : g.rows[t]) {
      auto it = off.find(s);
      if (it == off.end()) continue;
      const Blk& B = *g.get(t, s);
      cb.add(B.p, B.c, 1, F.top_lu.p + (size_t)off[t] * tot + it->second, tot, 1, B.r, B.c, 0);
    }
  z.run(C);
  cb.run(C);
  F.top_piv = C.arena.alloc_int(tot, &F.top_piv_cls);
  lu_any(C, F.top_lu.p, tot, F.top_piv, TOP_TAG);
  flops_gemm += 2.0 / 3.0 * (double)tot * tot * tot;
  flops_all += 2.0 / 3.0 * (double)tot * tot * tot;
}

Factor* factorize(Graph* gp, double eps, double sigma0, int flags) {
  (void)flags;
  if (!(eps > 0.0 && eps < 1.0)) throw Error(E_VALUE, "epsilon must be in (0, 1)");
  IFMM_ASSERT(!gp->consumed, "graph already consumed by a factorization");
  Graph& g = *gp;
  Ctx& C = *g.ctx;
  Tree& T = *g.tree;
  auto t0 = std::chrono::steady_clock::now();
  Factor* F = new Factor;
  F->ctx = &C;
  F->n_points = T.n_points;
  F->d_perm = T.d_perm;
  F->eps = eps;
  F->sigma0 = sigma0;
  F->init_sizes = g.size;
  F->n_clusters = T.nc;
  for (int c : T.leaves()) {
    F->leaf_nodes.push_back(g.nx[c]);
    F->leaf_start.push_back(T.start[c]);
    F->leaf_stop.push_back(T.stop[c]);
  }
  Eliminator el(C, g, *F, eps * sigma0, 0x1f2e3d4c5b6a7988ULL);
  for (double& v : g_prof) v = 0.0;
  try {
    for (int l = T.depth; l >= 2; --l) {
      LevelStats st;
      st.level = l;
      for (int c : T.levels[l]) el.eliminate(c, st);
      C.check_status("cluster ");
      F->levels.push_back(st);
      if (l > 2) el.merge(l);
    }
    el.top();
    C.sync();
    C.check_status("cluster ");
  } catch (...) {
    g.consumed = true;
    delete F;
    throw;
  }
  g.consumed = true;
  F->peak_edges = g.peak_edges;
  long long mb = 0;
  for (auto& w : g.su) mb = std::max<long long>(mb, w.p ? w.c : 0);
  F->max_basis_rank = mb;
  F->gemm_flops = el.flops_gemm;
  F->all_flops = el.flops_all;
  C.free(el.d_ranks);
  std::vector<int> final_size = g.size;
  F->build_program(final_size);
  C.sync();
  F->t_total = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return F;
}

}  // namespace ifmm
