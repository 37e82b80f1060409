// IFMM engine objects: tree/topology, H2 operators, extended graph,
// factorization (event log + solve program).
#pragma once
#include <algorithm>
#include <map>
#include <set>
#include <unordered_map>
#include <vector>

#include "runtime.h"

namespace ifmm {

inline uint64_t key2(int a, int b) { return ((uint64_t)(uint32_t)a << 32) | (uint32_t)b; }

// ---- tree + topology (tree.py:26-80, 205-239) ------------------------------
struct Tree {
  Ctx* ctx = nullptr;
  int n_points = 0, depth = 0, nc = 0;
  std::vector<double> points;  // N x 3, Morton-sorted
  double* d_points = nullptr;
  int d_points_cls = -1;
  std::vector<int> level, parent, start, stop;
  std::vector<int> perm;          // points[i] = original[perm[i]]
  int* d_perm = nullptr;
  int d_perm_cls = -1;
  std::vector<long long> cell;   // nc x 3
  std::vector<double> center;    // nc x 3
  std::vector<double> hw;
  std::vector<std::vector<int>> children;
  std::vector<std::vector<int>> levels;  // ids per level (Morton == id order)
  std::vector<std::vector<int>> nbrs, inters;
  bool is_leaf(int c) const { return children[c].empty(); }
  bool adjacent(int i, int j) const {
    const auto& v = nbrs[i];
    return std::binary_search(v.begin(), v.end(), j);
  }
  std::vector<int> leaves() const { return levels[depth]; }
  void build_topology();
};

// ---- H2 operators (h2.py:76-101) ----------------------------------------
struct H2 {
  Ctx* ctx = nullptr;
  Tree* tree = nullptr;
  KernelSpec kern{};
  int ncheb = 0;
  double eps = 0.0;
  bool weighted = false;
  bool consumed = false;  // blocks moved into a graph
  std::vector<int> rank;                 // -1 where absent
  std::vector<Blk> leaf_u, leaf_v;       // leaf: m x k
  std::vector<Blk> tu, tvt;              // child: k_c x k_p / k_p x k_c
  std::unordered_map<uint64_t, Blk> coupling, near;
  std::vector<Blk> su, sv;               // 1 x k
  ~H2();
  void build();
  // sptr / sidx (optional, CSR by cluster id): the sampled mode's row samples
  // of each cluster's basis (h2.py:250-262), drawn by the caller
  void weights(const long long* sptr = nullptr, const int* sidx = nullptr);
  void matvec(const double* d_x_sorted, double* d_y_sorted);
  // h2_matvec's block lists are built once per operator state and kept on
  // the device (h2.cu); weights() / graph consumption drop them
  struct MatvecPlan {
    bool valid = false;
    Blk desc;                  // SpmvRow[] then SpmvTerm[] (raw bytes)
    size_t n_rows = 0, n_terms = 0;
    std::vector<std::pair<size_t, int>> launches;  // (first row, rows) per dependent stage
    Blk xin, yout, yv, zv;     // staged x / y (tree order), multipoles, locals
    double bytes = 0.0;        // operator bytes one matvec reads
  } plan;
  void drop_plan();
  // Morton-range partitioned matvec (one rank's share), see h2.cu
  long long multipole_size() const;
  void matvec_part(const double* d_x_sorted, double* d_y_sorted, double* d_yv, int phase,
                   long long p_lo, long long p_hi);
};

// ---- extended graph (graph.py:30-216) ------------------------------------
enum NodeKind { NK_X = 0, NK_Z = 1, NK_Y = 2 };

struct Graph {
  Ctx* ctx = nullptr;
  Tree* tree = nullptr;
  H2* ops = nullptr;
  std::vector<int> size, kind, owner;
  std::vector<int> nx, nz, ny;  // per cluster, -1 if none
  std::unordered_map<uint64_t, Blk> E;
  std::vector<std::set<int>> rows, cols;  // row_sources / col_targets
  std::vector<char> dead;
  std::vector<Blk> su, sv;
  long long peak_edges = 0;
  bool consumed = false;
  int bd = 1;  // block_dim of the kernel (unknowns per point)
  ~Graph();

  int new_node(int sz, int k, int own) {
    int id = (int)size.size();
    size.push_back(sz); kind.push_back(k); owner.push_back(own);
    rows.emplace_back(); cols.emplace_back();
    return id;
  }
  Blk* get(int t, int s) {
    auto it = E.find(key2(t, s));
    return it == E.end() ? nullptr : &it->second;
  }
  // set_edge: replaces (and frees) an existing block unless it is the same
  void set(int t, int s, Blk b) {
    auto it = E.find(key2(t, s));
    if (it == E.end()) {
      rows[t].insert(s); cols[s].insert(t);
      E.emplace(key2(t, s), b);
      peak_edges = std::max<long long>(peak_edges, (long long)E.size());
    } else {
      if (it->second.p != b.p) ctx->free(it->second);
      it->second = b;
      peak_edges = std::max<long long>(peak_edges, (long long)E.size());
    }
  }
  Blk take(int t, int s) {
    auto it = E.find(key2(t, s));
    IFMM_ASSERT(it != E.end(), "pop of a missing edge");
    Blk b = it->second;
    E.erase(it);
    rows[t].erase(s); cols[s].erase(t);
    return b;
  }
  void build(H2* h, bool consume = false);
  long long dim() const {
    long long d = 0;
    for (int s : size) d += s;
    return d;
  }
  double sigma0(const double* omega, int width, int power_iters);
  Graph* clone() const;
  void apply(const double* d_in, double* d_out, bool transpose);
};

// ---- factorization ---------------------------------------------------------
struct LevelStats {
  int level = 0;
  long long compressed = 0, added = 0, dropped = 0, forced = 0;
  std::vector<int> ranks;
  double compress_time = 0.0;  // device s in lowrank_approximations (FillinStats.compress_time)
};

struct ElimEv {
  int nx, nz, ny, m, k;
  Blk LU;
  Blk Pinv;                              // P^{-1} (n x n), used by the solve
  int* piv = nullptr;
  int piv_cls = -1;
  std::vector<int> src, src_off, src_w;  // sources (node, col offset, width)
  Blk Scat;                              // m x Csrc
  std::vector<int> tgt, tgt_off, tgt_h;  // targets (node, row offset, height)
  Blk Tstk;                              // Rtgt x m
};
struct RebaseEv {
  int ny;
  Blk r;  // k_new x k_old
};
struct MergeEv {
  int px;
  std::vector<int> parts, psize;
};
struct Event {
  int type;  // 0 elim, 1 rebase, 2 merge
  int idx;
};

struct SolveOp;
struct SolveList;

struct Factor {
  Ctx* ctx = nullptr;
  int n_points = 0;
  const int* d_perm = nullptr;  // tree's device permutation of the POINTS (tree outlives factor)
  int bd = 1;                   // unknowns per point (block_dim); n_points counts unknowns
  double eps = 0, sigma0 = 0;
  std::vector<int> init_sizes;
  std::vector<int> leaf_nodes, leaf_start, leaf_stop;
  std::vector<ElimEv> elims;
  std::vector<RebaseEv> rebases;
  std::vector<MergeEv> merges;
  std::vector<Event> events;
  std::vector<int> top_nodes, top_sizes;
  Blk top_lu;
  int* top_piv = nullptr;
  int top_piv_cls = -1;
  std::vector<LevelStats> levels;
  long long peak_edges = 0, n_clusters = 0, max_basis_rank = 0;
  double t_lu = 0, t_mm = 0, t_lr = 0, t_tr = 0, t_total = 0;
  double gemm_flops = 0, all_flops = 0;
  unsigned long long rsvd_rounds = 0, rsvd_redraws = 0;
  // solve program (built once after factorization)
  struct Program;
  Program* prog = nullptr;
  ~Factor();
  void build_program(const std::vector<int>& final_size);
  void solve(const double* d_b_orig, double* d_x_orig);
  void enqueue_program(cudaStream_t s);
};

// Standard-normal source of the reference's factorize rng (see
// ifmm_normal_source in include/ifmm_b200.h): op 0 draws n deviates into
// out, op 1 saves the stream state in slot n, op 2 restores slot n.
typedef int (*NormalSource)(void* user, int op, long long n, double* out);
// flags bit0: strict pair order (one pair per wave); bit1: exact SVD for every
// fill; bit2: Morton cluster order (one cluster per wave; implied by src).
Factor* factorize(Graph* g, double eps, double sigma0, int flags, NormalSource src = nullptr,
                  void* src_user = nullptr);
// factorize with the reference stream generated natively: PCG64 state / inc
// as (hi, lo) 64-bit halves, st = {state_hi, state_lo, inc_hi, inc_lo}
Factor* factorize_pcg64(Graph* g, double eps, double sigma0, int flags, const uint64_t st[4]);
int pcg64_normals(const uint64_t st[4], long long n, double* out);

// blocked LU for large pivot blocks (host-driven panels)
void lu_blocked(Ctx& ctx, double* A, int n, int lda, int* piv, int tag);
void lu_any(Ctx& ctx, double* A, int n, int* piv, int tag);

// device Arnoldi pieces of GMRES (krylov.cu; krylov.py:32-116)
void krylov_mgs(Ctx& C, const double* V, long long ldv, int k1, long long n, double* w,
                double* h_host);
void krylov_div(Ctx& C, const double* w, long long n, double hs, double* out);
void krylov_combine(Ctx& C, const double* V, long long ldv, int k, const double* y_host,
                    long long n, double* u);

}  // namespace ifmm
