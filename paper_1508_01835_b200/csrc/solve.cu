// IFMMFactorization.solve (factor.py:99-157) as a device program.
//
// The event log (elim / rebase / merge) is compiled once, after the
// factorization, into SSA "slots" in one workspace vector:
//   * every rhs version of a node gets its own slot (a rebase writes a new
//     version instead of overwriting), so only true dependencies remain;
//   * merge events cost nothing: the final y versions of the children are
//     allocated *inside* the parent's x slot (factor.py:123-126), and the
//     final level-2 y versions inside the top-level rhs;
//   * the backward solution slots alias the same way (factor.py:147-152).
// Ops are levelled into dependency waves (read-after-write, write-after-
// write, write-after-read on slots).  A wave runs as two launches whose
// row tasks spread every op over many CTAs (forward: g = P^{-1}[:, :m] rhs_x,
// then the target rows rhs_a -= T_a g; backward: v = [rhs_x - S sol_src;
// sol_y], then [sol_x; sol_z] = P^{-1} v), so a wave streams its factor
// bytes at HBM rate instead of one SM per op.  Every output row is one warp's
// fixed-order dot product and ops of one wave write disjoint slots, so solves
// are bitwise reproducible (reference test_factor.py:95-106).  The whole
// program (waves + blocked top-level triangular solves) is captured once into
// a CUDA graph and replayed per right-hand side.
#include <algorithm>
#include <cstdlib>
#include <map>

#include "common.cuh"
#include "engine.h"

namespace ifmm {

enum OpType { OP_FWD_ELIM = 0, OP_REBASE = 1, OP_BWD_ELIM = 2 };

struct SolveOp {
  int type;
  int n, m, k;
  const double* LU;
  const int* piv;
  const double* M;  // Tstk (fwd), Scat (bwd), r (rebase)
  int ldm;
  int list0, nlist;
  long long a;      // fwd: rhs_x slot | rebase: in | bwd: rhs_x slot
  long long b;      // fwd: rhs_y slot | rebase: out | bwd: sol_y slot
  long long c;      // bwd: sol_x slot
  long long d;      // bwd: sol_z slot
  long long e;      // bwd: gather scratch
  int rows;         // rebase: k_new ; fwd: total target rows
  int cols;         // rebase: k_old ; bwd: Csrc
  long long g;      // scratch: g (fwd) / v (bwd), n doubles
};
struct ListEnt {
  long long slot;
  int off, len;  // fwd: row offset in Tstk, height | bwd: col offset in Scat, width
};

struct SolveTask {
  int op;       // index into the op array
  int list;     // forward target phase: list entry; -1 otherwise
  int r0, r1;   // output rows [r0, r1) of the phase
};

struct Factor::Program {
  Blk ops_d, list_d, work, perm_d;
  Blk task_d;
  std::vector<int> task_start;   // per launch: [task_start[i], task_start[i+1])
  std::vector<int> launch_kind;  // 0 fwd-g, 1 fwd-t, 2 bwd-v, 3 bwd-x
  long long scratch0 = 0;        // per-op scratch (g / v) region in the workspace
  Blk bin, bout;                 // graph-resident rhs / solution buffers
  cudaGraphExec_t graph = nullptr;
  double bytes = 0;              // algorithmic bytes of one solve
  std::vector<int> fwd_wave_start, bwd_wave_start;  // op index ranges per wave
  int n_fwd = 0, n_bwd = 0;
  long long top_rhs = 0, top_sol = 0;
  int top_n = 0;
  long long sol0 = 0;  // sol region of leaf x (N)
  int max_n = 0;
  int fwd_waves = 0, bwd_waves = 0;
  int smem = 0;  // doubles of dynamic shared memory per op
  int n_fwd_launch = 0;
  int max_csrc = 1;
  long long nsolves = 0;
};

Factor::~Factor() {
  if (!ctx) return;
  for (auto& e : elims) {
    ctx->free(e.LU); ctx->free(e.Pinv); ctx->free(e.Scat); ctx->free(e.Tstk);
    ctx->free_raw(e.piv, e.piv_cls);
  }
  ctx->free(top_lu);
  if (top_piv) ctx->free_raw(top_piv, top_piv_cls);
  if (prog) {
    ctx->free(prog->ops_d); ctx->free(prog->list_d); ctx->free(prog->work);
    ctx->free(prog->perm_d);
    ctx->free(prog->task_d); ctx->free(prog->bin); ctx->free(prog->bout);
    if (prog->graph) cudaGraphExecDestroy(prog->graph);
    delete prog;
  }
  // a destructor must not throw: after a device fault the sync reports the
  // (sticky) error, which the failing call has already raised
  if (cudaStreamSynchronize(ctx->st) != cudaSuccess) cudaGetLastError();
  ctx->flush();
}

// ---------------------------------------------------------------------------
// device side
// ---------------------------------------------------------------------------
namespace {

// Compensated dot products (TwoProd / TwoSum, _rn intrinsics so nothing is
// contracted): every row sum of the replay is accumulated to about twice the
// working precision and rounded once.  The replay multiplies by explicit
// pivot-block inverses, whose rows cancel heavily on ill-conditioned blocks;
// with plain FMA sums the solve's rounding error (~eps |P^-1| |b|, not
// ~eps |x|) made the preconditioner visibly nonlinear and stalled GMRES's
// true residual two orders above its recurrence residual (c5 recipe).
IFMM_DEV void dd_fma(double a, double b, double& s, double& c) {
  const double p = __dmul_rn(a, b);
  const double e = __fma_rn(a, b, -p);
  const double t = __dadd_rn(s, p);
  const double z = __dadd_rn(t, -s);
  c = __dadd_rn(c, __dadd_rn(__dadd_rn(__dadd_rn(s, -__dadd_rn(t, -z)), __dadd_rn(p, -z)), e));
  s = t;
}
IFMM_DEV double warp_sum_dd(double s, double c) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double s2 = __shfl_xor_sync(0xffffffffu, s, o);
    const double c2 = __shfl_xor_sync(0xffffffffu, c, o);
    // symmetric in (s, s2): both partners compute the same pair
    const double hi = fmax(s, s2), lo = fmin(s, s2);
    const double t = __dadd_rn(hi, lo);
    const double z = __dadd_rn(t, -hi);
    c = __dadd_rn(__dadd_rn(c, c2), __dadd_rn(__dadd_rn(hi, -__dadd_rn(t, -z)), __dadd_rn(lo, -z)));
    s = t;
  }
  return __dadd_rn(s, c);
}

// ---- row-task kernels (one launch per wave and phase) ----------------------
// Each CTA takes one task; its 8 warps take the task's rows round robin, one
// warp per row (lanes split the dot product, fixed shuffle tree).
constexpr int kGatherCap = 24576;  // doubles of gathered sources staged in shared memory
constexpr int kSolveRowsPerTask = 8;  // one row per warp: a wave's rows spread over the most CTAs

__global__ void __launch_bounds__(256)
solve_fwd_g_kernel(const SolveOp* __restrict__ ops, const SolveTask* __restrict__ tasks,
                   double* __restrict__ W) {
  const SolveTask t = tasks[blockIdx.x];
  const SolveOp& op = ops[t.op];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int m = op.m, n = op.n;
  const double* rx = W + op.a;
  for (int i = t.r0 + warp; i < t.r1; i += 8) {
    const double* row = op.LU + (size_t)i * n;  // P^{-1} row i, first m columns
    double s = 0.0, cc = 0.0;
    for (int j = lane; j < m; j += 32) dd_fma(row[j], rx[j], s, cc);
    s = warp_sum_dd(s, cc);
    if (lane == 0) {
      W[op.g + i] = s;
      if (i >= m) W[op.b + i - m] += s;  // rhs_y += g[m:]
    }
  }
}

__global__ void __launch_bounds__(256)
solve_fwd_t_kernel(const SolveOp* __restrict__ ops, const ListEnt* __restrict__ lists,
                   const SolveTask* __restrict__ tasks, double* __restrict__ W) {
  const SolveTask t = tasks[blockIdx.x];
  const SolveOp& op = ops[t.op];
  const ListEnt e = lists[t.list];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int m = op.m;
  const double* g = W + op.g;
  for (int i = t.r0 + warp; i < t.r1; i += 8) {
    const double* row = op.M + (size_t)(e.off + i) * op.ldm;
    double s = 0.0, cc = 0.0;
    for (int j = lane; j < m; j += 32) dd_fma(row[j], g[j], s, cc);
    s = warp_sum_dd(s, cc);
    if (lane == 0) W[e.slot + i] = W[e.slot + i] - s;
  }
}

__global__ void __launch_bounds__(256)
solve_bwd_v_kernel(const SolveOp* __restrict__ ops, const ListEnt* __restrict__ lists,
                   const SolveTask* __restrict__ tasks, double* __restrict__ W, int cap) {
  extern __shared__ double gsol[];  // the op's source solutions, gathered (Csrc <= cap)
  const SolveTask t = tasks[blockIdx.x];
  const SolveOp& op = ops[t.op];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int m = op.m;
  if (op.cols > cap) {  // sources too wide for shared memory: read them in place
    for (int i = t.r0 + warp; i < t.r1; i += 8) {
      if (i >= m) {
        if (lane == 0) W[op.g + i] = W[op.b + i - m];
        continue;
      }
      const double* row = op.M + (size_t)i * op.ldm;
      double s = 0.0, cc = 0.0;
      for (int l = op.list0; l < op.list0 + op.nlist; ++l) {
        const ListEnt e = lists[l];
        for (int j = lane; j < e.len; j += 32) dd_fma(row[e.off + j], W[e.slot + j], s, cc);
      }
      s = warp_sum_dd(s, cc);
      if (lane == 0) W[op.g + i] = W[op.a + i] - s;
    }
    return;
  }
  if (t.r0 < m) {
    for (int l = op.list0; l < op.list0 + op.nlist; ++l) {
      const ListEnt e = lists[l];
      for (int j = threadIdx.x; j < e.len; j += blockDim.x) gsol[e.off + j] = W[e.slot + j];
    }
    __syncthreads();
  }
  for (int i = t.r0 + warp; i < t.r1; i += 8) {
    if (i >= m) {  // v[m:] = sol_y
      if (lane == 0) W[op.g + i] = W[op.b + i - m];
      continue;
    }
    const double* row = op.M + (size_t)i * op.ldm;
    double s = 0.0, cc = 0.0;
#pragma unroll 4
    for (int j = lane; j < op.cols; j += 32) dd_fma(row[j], gsol[j], s, cc);
    s = warp_sum_dd(s, cc);
    if (lane == 0) W[op.g + i] = W[op.a + i] - s;
  }
}

__global__ void __launch_bounds__(256)
solve_bwd_x_kernel(const SolveOp* __restrict__ ops, const SolveTask* __restrict__ tasks,
                   double* __restrict__ W) {
  const SolveTask t = tasks[blockIdx.x];
  const SolveOp& op = ops[t.op];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int m = op.m, n = op.n;
  const double* v = W + op.g;
  for (int i = t.r0 + warp; i < t.r1; i += 8) {
    const double* row = op.LU + (size_t)i * n;
    double s = 0.0, cc = 0.0;
    for (int j = lane; j < n; j += 32) dd_fma(row[j], v[j], s, cc);
    s = warp_sum_dd(s, cc);
    if (lane == 0) {
      if (i < m) W[op.c + i] = s;
      else W[op.d + i - m] = s;
    }
  }
}

// In-place LU solve of v (smem) by one warp (top-level system).
__device__ void warp_lu_solve(const double* __restrict__ LU, const int* __restrict__ piv, int n,
                              double* v) {
  const int lane = threadIdx.x & 31;
  if (threadIdx.x >= 32) return;
  if (lane == 0)
    for (int j = 0; j < n; ++j) {
      const int p = piv[j];
      if (p != j) { const double t = v[j]; v[j] = v[p]; v[p] = t; }
    }
  __syncwarp();
  for (int i = 1; i < n; ++i) {
    const double* L = LU + (size_t)i * n;
    double s = 0.0;
    for (int j = lane; j < i; j += 32) s = fma(L[j], v[j], s);
    s = warp_sum(s);
    if (lane == 0) v[i] -= s;
    __syncwarp();
  }
  for (int i = n - 1; i >= 0; --i) {
    const double* U = LU + (size_t)i * n;
    double s = 0.0;
    for (int j = i + 1 + lane; j < n; j += 32) s = fma(U[j], v[j], s);
    s = warp_sum(s);
    if (lane == 0) v[i] = (v[i] - s) / U[i];
    __syncwarp();
  }
}

__global__ void __launch_bounds__(1024)
top_solve_kernel(const double* LU, const int* piv, int n, const double* rhs, double* out) {
  extern __shared__ double v[];
  for (int i = threadIdx.x; i < n; i += blockDim.x) v[i] = rhs[i];
  __syncthreads();
  warp_lu_solve(LU, piv, n, v);
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) out[i] = v[i];
}

// Blocked top-level solve for n beyond one CTA's shared memory:
// per 256-row block a one-warp triangular solve, then a multi-CTA GEMV update
// of the remaining rows (factor.py:129-135 semantics, LAPACK getrs order).
__global__ void top_perm_kernel(const int* piv, int n, double* v) {
  if (threadIdx.x == 0 && blockIdx.x == 0)
    for (int j = 0; j < n; ++j) {
      const int p = piv[j];
      if (p != j) { const double t = v[j]; v[j] = v[p]; v[p] = t; }
    }
}
// Triangular solve of one bs x bs diagonal block (bs <= 128), column
// oriented: the block sits in shared memory, x_j is final after step j and
// every later row subtracts L[i][j] x_j in parallel (one barrier per column).
__global__ void __launch_bounds__(128)
top_diag_kernel(const double* LU, int n, int b0, int bs, double* v, int upper) {
  extern __shared__ double blk[];  // bs x bs, then bs
  double* x = blk + bs * bs;
  for (int e = threadIdx.x; e < bs * bs; e += blockDim.x)
    blk[e] = LU[(size_t)(b0 + e / bs) * n + b0 + e % bs];
  for (int i = threadIdx.x; i < bs; i += blockDim.x) x[i] = v[b0 + i];
  __syncthreads();
  if (!upper) {  // unit lower
    for (int j = 0; j < bs - 1; ++j) {
      const double xj = x[j];
      for (int i = j + 1 + threadIdx.x; i < bs; i += blockDim.x) x[i] = fma(-blk[i * bs + j], xj, x[i]);
      __syncthreads();
    }
  } else {
    for (int j = bs - 1; j >= 0; --j) {
      if (threadIdx.x == 0) x[j] = x[j] / blk[j * bs + j];
      __syncthreads();
      const double xj = x[j];
      for (int i = threadIdx.x; i < j; i += blockDim.x) x[i] = fma(-blk[i * bs + j], xj, x[i]);
      __syncthreads();
    }
  }
  for (int i = threadIdx.x; i < bs; i += blockDim.x) v[b0 + i] = x[i];
}
// rows [r0, r1): v[i] -= sum_{j in [c0, c0+bs)} A[i][j] v[j]
__global__ void top_update_kernel(const double* LU, int n, int r0, int r1, int c0, int bs,
                                  double* v) {
  const int lane = threadIdx.x & 31;
  const int row = r0 + blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (row >= r1) return;
  const double* A = LU + (size_t)row * n + c0;
  double s = 0.0;
  for (int j = lane; j < bs; j += 32) s = fma(A[j], v[c0 + j], s);
  s = warp_sum(s);
  if (lane == 0) v[row] -= s;
}

// tree order <-> original order of the n = bd * points unknowns (point-major:
// unknown p * bd + a of point p, factor.py:104-105,154-157)
__global__ void gather_perm_kernel(const double* b, const int* perm, int n, int bd, double* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = b[(size_t)perm[i / bd] * bd + i % bd];
}
__global__ void scatter_perm_kernel(const double* in, const int* perm, int n, int bd, double* x) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) x[(size_t)perm[i / bd] * bd + i % bd] = in[i];
}

}  // namespace

// ---------------------------------------------------------------------------
// host side: compile the event log
// ---------------------------------------------------------------------------
void Factor::build_program(const std::vector<int>& final_size) {
  Ctx& C = *ctx;
  prog = new Program;
  Program& P = *prog;
  const int nnodes = (int)std::max(init_sizes.size(), final_size.size());
  // Slots.  Forward rhs: leaf x in [0, N) (sorted order); every merged
  // parent x gets a region holding its children's y slots (factor.py:123);
  // the level-2 y slots live in the top rhs region.  Rebases act on zero
  // rhs (see factor.cu) and need no slots of their own.
  std::vector<long long> rslot(nnodes, -1), sslot(nnodes, -1);
  long long top = n_points;
  auto alloc = [&](long long n) { long long o = top; top += n; return o; };
  for (int t = 0; t < (int)leaf_nodes.size(); ++t) rslot[leaf_nodes[t]] = leaf_start[t];
  for (auto& mv : merges) {
    long long sz = 0;
    for (int q : mv.psize) sz += q;
    const long long o = alloc(sz);
    rslot[mv.px] = o;
    long long off = 0;
    for (size_t q = 0; q < mv.parts.size(); ++q) {
      rslot[mv.parts[q]] = o + off;
      off += mv.psize[q];
    }
  }
  P.top_n = 0;
  for (int s : top_sizes) P.top_n += s;
  const bool top_is_x = !top_nodes.empty() && rslot[top_nodes[0]] >= 0;
  P.top_rhs = top_is_x ? 0 : alloc(P.top_n);
  if (!top_is_x) {
    long long off = 0;
    for (size_t q = 0; q < top_nodes.size(); ++q) {
      rslot[top_nodes[q]] = P.top_rhs + off;
      off += top_sizes[q];
    }
  }
  // backward solutions: leaf x in the sol region (sorted order), merged
  // parents' regions contain their children's y, the top solution holds the
  // level-2 y; z solutions get their own slots.
  P.sol0 = alloc(n_points);
  for (int t = 0; t < (int)leaf_nodes.size(); ++t) sslot[leaf_nodes[t]] = P.sol0 + leaf_start[t];
  P.top_sol = top_is_x ? P.sol0 : alloc(P.top_n);
  if (!top_is_x) {
    long long off = 0;
    for (size_t q = 0; q < top_nodes.size(); ++q) {
      sslot[top_nodes[q]] = P.top_sol + off;
      off += top_sizes[q];
    }
  }
  for (int mi = (int)merges.size() - 1; mi >= 0; --mi) {
    auto& mv = merges[mi];
    long long sz = 0;
    for (int q : mv.psize) sz += q;
    if (sslot[mv.px] < 0) sslot[mv.px] = alloc(sz);
    long long off = 0;
    for (size_t q = 0; q < mv.parts.size(); ++q) {
      sslot[mv.parts[q]] = sslot[mv.px] + off;
      off += mv.psize[q];
    }
  }
  for (auto& E : elims) {
    if (sslot[E.nz] < 0) sslot[E.nz] = alloc(E.k);
    IFMM_ASSERT(rslot[E.nx] >= 0 && rslot[E.ny] >= 0 && sslot[E.nx] >= 0 && sslot[E.ny] >= 0,
                "solve program: unmapped slot");
  }
  // composite resources: a merged parent x = its children's y slots
  std::map<int, std::vector<long long>> comp_r, comp_s;
  for (auto& mv : merges) {
    for (int q : mv.parts) {
      comp_r[mv.px].push_back(rslot[q]);
      comp_s[mv.px].push_back(sslot[q]);
    }
  }
  auto res = [](const std::map<int, std::vector<long long>>& comp, int node, long long slot,
                std::vector<long long>& out) {
    auto it = comp.find(node);
    if (it != comp.end()) for (long long s : it->second) out.push_back(s);
    else out.push_back(slot);
  };
  std::unordered_map<long long, int> lw, lr;
  auto wave_for = [&](const std::vector<long long>& rd, const std::vector<long long>& wr) {
    int w = 0;
    for (long long r : rd) { auto it = lw.find(r); if (it != lw.end()) w = std::max(w, it->second); }
    for (long long r : wr) {
      auto it = lw.find(r); if (it != lw.end()) w = std::max(w, it->second);
      auto jt = lr.find(r); if (jt != lr.end()) w = std::max(w, jt->second);
    }
    w += 1;
    for (long long r : rd) { int& x = lr[r]; x = std::max(x, w); }
    for (long long r : wr) lw[r] = w;
    return w;
  };
  std::vector<SolveOp> fops, bops;
  std::vector<ListEnt> lists;
  std::vector<int> fwave, bwave;
  P.max_n = 1;
  int max_smem = 1;
  for (auto& ev : events) {
    if (ev.type != 0) continue;
    const ElimEv& E = elims[ev.idx];
    SolveOp o{};
    o.type = OP_FWD_ELIM;
    o.n = E.m + E.k; o.m = E.m; o.k = E.k;
    o.LU = E.Pinv.p; o.M = E.Tstk.p; o.ldm = E.m;
    o.a = rslot[E.nx];
    o.b = rslot[E.ny];
    o.list0 = (int)lists.size(); o.nlist = (int)E.tgt.size();
    std::vector<long long> rd, wr;
    res(comp_r, E.nx, o.a, rd);
    wr.push_back(o.b);
    for (size_t t = 0; t < E.tgt.size(); ++t) {
      const int a = E.tgt[t];
      IFMM_ASSERT(rslot[a] >= 0, "solve program: unmapped target");
      lists.push_back({rslot[a], E.tgt_off[t], E.tgt_h[t]});
      res(comp_r, a, rslot[a], wr);
    }
    P.max_n = std::max(P.max_n, o.n);
    max_smem = std::max(max_smem, o.n + o.m);
    fops.push_back(o);
    fwave.push_back(wave_for(rd, wr));
  }
  lw.clear(); lr.clear();
  for (int ei = (int)events.size() - 1; ei >= 0; --ei) {
    const Event& ev = events[ei];
    if (ev.type != 0) continue;
    const ElimEv& E = elims[ev.idx];
    SolveOp o{};
    o.type = OP_BWD_ELIM;
    o.n = E.m + E.k; o.m = E.m; o.k = E.k;
    o.LU = E.Pinv.p; o.M = E.Scat.p; o.ldm = E.Scat.c;
    o.a = rslot[E.nx];
    o.b = sslot[E.ny];
    o.c = sslot[E.nx];
    o.d = sslot[E.nz];
    int csrc = 0;
    for (int w : E.src_w) csrc += w;
    o.cols = csrc;
    P.max_csrc = std::max(P.max_csrc, csrc);
    o.list0 = (int)lists.size(); o.nlist = (int)E.src.size();
    std::vector<long long> rd, wr;
    rd.push_back(o.b);
    for (size_t t = 0; t < E.src.size(); ++t) {
      const int b = E.src[t];
      lists.push_back({sslot[b], E.src_off[t], E.src_w[t]});
      res(comp_s, b, sslot[b], rd);
    }
    res(comp_s, E.nx, o.c, wr);
    wr.push_back(o.d);
    max_smem = std::max(max_smem, o.n + csrc);
    bops.push_back(o);
    bwave.push_back(wave_for(rd, wr));
  }
  // per-op scratch (g forward, v backward): one n-vector per elimination
  long long scr = top;
  for (auto& o : fops) { o.g = scr; scr += o.n; }
  for (size_t i = 0; i < bops.size(); ++i) bops[i].g = fops[fops.size() - 1 - i].g;  // same event
  const long long wtot = scr;
  auto order_by = [](const std::vector<int>& wv, std::vector<int>& starts) {
    std::vector<int> idx(wv.size());
    for (size_t i = 0; i < idx.size(); ++i) idx[i] = (int)i;
    std::stable_sort(idx.begin(), idx.end(), [&](int a, int b) { return wv[a] < wv[b]; });
    starts.clear();
    int last = -1;
    for (size_t i = 0; i < idx.size(); ++i)
      if (wv[idx[i]] != last) { starts.push_back((int)i); last = wv[idx[i]]; }
    starts.push_back((int)idx.size());
    return idx;
  };
  auto fi = order_by(fwave, P.fwd_wave_start);
  auto bi = order_by(bwave, P.bwd_wave_start);
  std::vector<SolveOp> all;
  for (int i : fi) all.push_back(fops[i]);
  for (int i : bi) all.push_back(bops[i]);
  P.n_fwd = (int)fops.size();
  P.n_bwd = (int)bops.size();
  P.fwd_waves = (int)P.fwd_wave_start.size() - 1;
  P.bwd_waves = (int)P.bwd_wave_start.size() - 1;
  P.smem = max_smem;
  // row tasks: two launches per wave (kinds 0/1 forward, 2/3 backward)
  std::vector<SolveTask> tasks;
  P.task_start.clear();
  P.launch_kind.clear();
  auto rows = [&](int op, int list, int nrows) {
    for (int r0 = 0; r0 < nrows; r0 += kSolveRowsPerTask)
      tasks.push_back({op, list, r0, std::min(nrows, r0 + kSolveRowsPerTask)});
  };
  auto launch = [&](int kind) { P.task_start.push_back((int)tasks.size()); P.launch_kind.push_back(kind); };
  P.bytes = 0;
  for (int w = 0; w < P.fwd_waves; ++w) {
    launch(0);
    for (int o = P.fwd_wave_start[w]; o < P.fwd_wave_start[w + 1]; ++o) {
      rows(o, -1, all[o].n);
      P.bytes += 8.0 * all[o].n * all[o].m;
    }
    launch(1);
    for (int o = P.fwd_wave_start[w]; o < P.fwd_wave_start[w + 1]; ++o)
      for (int l = all[o].list0; l < all[o].list0 + all[o].nlist; ++l) {
        rows(o, l, lists[l].len);
        P.bytes += 8.0 * lists[l].len * all[o].m;
      }
  }
  const int n_fwd_launch = (int)P.launch_kind.size();
  for (int w = 0; w < P.bwd_waves; ++w) {
    launch(2);
    for (int o = P.n_fwd + P.bwd_wave_start[w]; o < P.n_fwd + P.bwd_wave_start[w + 1]; ++o) {
      rows(o, -1, all[o].n);
      P.bytes += 8.0 * all[o].m * all[o].cols;
    }
    launch(3);
    for (int o = P.n_fwd + P.bwd_wave_start[w]; o < P.n_fwd + P.bwd_wave_start[w + 1]; ++o) {
      rows(o, -1, all[o].n);
      P.bytes += 8.0 * all[o].n * all[o].n;
    }
  }
  P.task_start.push_back((int)tasks.size());
  P.n_fwd_launch = n_fwd_launch;
  if (getenv("IFMM_MEMTRACE"))
    fprintf(stderr, "[ifmm] solve program: %d eliminations, forward %d waves, backward %d waves, %zu row tasks, top n %d\n",
            P.n_fwd, P.fwd_waves, P.bwd_waves, tasks.size(), P.top_n);
  P.bytes += 8.0 * (double)P.top_n * P.top_n;  // both triangles of the top LU, once
  const size_t ob = all.size() * sizeof(SolveOp), lb = lists.size() * sizeof(ListEnt);
  const size_t tb = tasks.size() * sizeof(SolveTask);
  P.ops_d = C.alloc(1, (int)(ob / 8 + 1));
  P.list_d = C.alloc(1, (int)(lb / 8 + 1));
  P.task_d = C.alloc(1, (int)(tb / 8 + 1));
  if (ob) CUDA_CHECK(cudaMemcpyAsync(P.ops_d.p, all.data(), ob, cudaMemcpyHostToDevice, C.st));
  if (lb) CUDA_CHECK(cudaMemcpyAsync(P.list_d.p, lists.data(), lb, cudaMemcpyHostToDevice, C.st));
  if (tb) CUDA_CHECK(cudaMemcpyAsync(P.task_d.p, tasks.data(), tb, cudaMemcpyHostToDevice, C.st));
  P.work = C.alloc(1, (int)std::max<long long>(wtot, 1));
  P.bin = C.alloc(1, std::max(n_points, 1));
  P.bout = C.alloc(1, std::max(n_points, 1));
  C.sync();  // host vectors die here
}

// The solve program on stream s: permute b (P.bin) into the workspace, the
// forward waves, the top-level LU solve, the backward waves, un-permute into
// P.bout.  Captured once into a CUDA graph (Factor::solve).
void Factor::enqueue_program(cudaStream_t s) {
  Program& P = *prog;
  const int N = n_points;
  double* W = P.work.p;
  const size_t wbytes = (size_t)P.work.r * P.work.c * sizeof(double);
  CUDA_CHECK(cudaMemsetAsync(W, 0, wbytes, s));
  gather_perm_kernel<<<(N + 255) / 256, 256, 0, s>>>(P.bin.p, d_perm, N, bd, W);
  const SolveOp* ops = reinterpret_cast<const SolveOp*>(P.ops_d.p);
  const ListEnt* lists = reinterpret_cast<const ListEnt*>(P.list_d.p);
  const SolveTask* tasks = reinterpret_cast<const SolveTask*>(P.task_d.p);
  auto run = [&](int li) {
    const int a = P.task_start[li], b = P.task_start[li + 1];
    if (b <= a) return;
    switch (P.launch_kind[li]) {
      case 0: solve_fwd_g_kernel<<<b - a, 256, 0, s>>>(ops, tasks + a, W); break;
      case 1: solve_fwd_t_kernel<<<b - a, 256, 0, s>>>(ops, lists, tasks + a, W); break;
      case 2:
        solve_bwd_v_kernel<<<b - a, 256, sizeof(double) * std::min(P.max_csrc, kGatherCap), s>>>(
            ops, lists, tasks + a, W, kGatherCap);
        break;
      default: solve_bwd_x_kernel<<<b - a, 256, 0, s>>>(ops, tasks + a, W); break;
    }
  };
  static const int parts = getenv("IFMM_SOLVE_PARTS") ? atoi(getenv("IFMM_SOLVE_PARTS")) : 7;
  if (parts & 1)
    for (int li = 0; li < P.n_fwd_launch; ++li) run(li);
  if (!(parts & 2)) {
  } else if (P.top_n > 0 && P.top_n <= 1024) {
    top_solve_kernel<<<1, 1024, (size_t)P.top_n * sizeof(double), s>>>(
        top_lu.p, top_piv, P.top_n, W + P.top_rhs, W + P.top_sol);
  } else if (P.top_n > 0) {
    // blocked getrs: a one-warp triangular solve per 128-row diagonal block,
    // then a many-CTA GEMV update of the rows below (above) it
    const int n = P.top_n, bs = 128;
    double* v = W + P.top_sol;
    CUDA_CHECK(cudaMemcpyAsync(v, W + P.top_rhs, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
    top_perm_kernel<<<1, 32, 0, s>>>(top_piv, n, v);
    for (int b0 = 0; b0 < n; b0 += bs) {  // L (unit) forward
      const int b = std::min(bs, n - b0);
      top_diag_kernel<<<1, 128, sizeof(double) * (b * b + b), s>>>(top_lu.p, n, b0, b, v, 0);
      if (b0 + b < n)
        top_update_kernel<<<(n - b0 - b + 7) / 8, 256, 0, s>>>(top_lu.p, n, b0 + b, n, b0, b, v);
    }
    for (int b0 = ((n - 1) / bs) * bs; b0 >= 0; b0 -= bs) {  // U backward
      const int b = std::min(bs, n - b0);
      top_diag_kernel<<<1, 128, sizeof(double) * (b * b + b), s>>>(top_lu.p, n, b0, b, v, 1);
      if (b0 > 0) top_update_kernel<<<(b0 + 7) / 8, 256, 0, s>>>(top_lu.p, n, 0, b0, b0, b, v);
    }
  }
  if (parts & 4)
    for (int li = P.n_fwd_launch; li + 1 < (int)P.task_start.size(); ++li) run(li);
  scatter_perm_kernel<<<(N + 255) / 256, 256, 0, s>>>(W + P.sol0, d_perm, N, bd, P.bout.p);
  CUDA_CHECK(cudaGetLastError());
}

void Factor::solve(const double* d_b, double* d_x) {
  Ctx& C = *ctx;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(top_solve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(top_diag_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(solve_bwd_v_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr = true;
  }
  Program& P = *prog;
  const int N = n_points;
  CUDA_CHECK(cudaMemcpyAsync(P.bin.p, d_b, sizeof(double) * N, cudaMemcpyDeviceToDevice, C.st));
  cudaEvent_t ka = nullptr;
  if (P.nsolves++ == 0) {
    // first right-hand side: launch the program directly (a one-off solve
    // does not pay for graph instantiation)
    C.kt_begin(K_SOLVE, P.bytes, &ka);
    enqueue_program(C.st);
    C.kt_end(K_SOLVE, P.bytes, ka);
    CUDA_CHECK(cudaMemcpyAsync(d_x, P.bout.p, sizeof(double) * N, cudaMemcpyDeviceToDevice, C.st));
    C.launches += (long long)P.launch_kind.size() + 3;
    return;
  }
  if (!P.graph) {
    // repeated solves (GMRES preconditioning, many rhs): capture the fixed
    // program once; replays differ only in P.bin's content
    cudaGraph_t g = nullptr;
    CUDA_CHECK(cudaStreamBeginCapture(C.st, cudaStreamCaptureModeThreadLocal));
    try {
      enqueue_program(C.st);
    } catch (...) {
      cudaStreamEndCapture(C.st, &g);
      if (g) cudaGraphDestroy(g);
      throw;
    }
    CUDA_CHECK(cudaStreamEndCapture(C.st, &g));
    CUDA_CHECK(cudaGraphInstantiate(&P.graph, g, 0));
    cudaGraphDestroy(g);
  }
  C.kt_begin(K_SOLVE, P.bytes, &ka);
  CUDA_CHECK(cudaGraphLaunch(P.graph, C.st));
  C.kt_end(K_SOLVE, P.bytes, ka);
  CUDA_CHECK(cudaMemcpyAsync(d_x, P.bout.p, sizeof(double) * N, cudaMemcpyDeviceToDevice, C.st));
  C.launches += (long long)P.launch_kind.size() + 3;
  CUDA_CHECK(cudaGetLastError());
}

}  // namespace ifmm
