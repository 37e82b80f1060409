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
// write, write-after-read on slots); each wave is one launch with one CTA
// per op.  Updates to one slot stay in event order, so solves are bitwise
// reproducible (reference test_factor.py:95-106).
#include <algorithm>
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
};
struct ListEnt {
  long long slot;
  int off, len;  // fwd: row offset in Tstk, height | bwd: col offset in Scat, width
};

struct Factor::Program {
  Blk ops_d, list_d, work, perm_d;
  std::vector<int> fwd_wave_start, bwd_wave_start;  // op index ranges per wave
  int n_fwd = 0, n_bwd = 0;
  long long top_rhs = 0, top_sol = 0;
  int top_n = 0;
  long long sol0 = 0;  // sol region of leaf x (N)
  int max_n = 0;
  int fwd_waves = 0, bwd_waves = 0;
  int smem = 0;  // doubles of dynamic shared memory per op
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

// One CTA per elimination op.  Forward (factor.py:111-119):
//   g = P^{-1}[:, :m] rhs_x ;  rhs[a] -= T_a g[:m] ;  rhs[y] += g[m:]
// Backward (factor.py:139-146):
//   v = [rhs_x - S gather(sol_b) ; sol_y] ;  [sol_x ; sol_z] = P^{-1} v
// Every product is a warp-per-row GEMV (lanes split the dot product, fixed
// shuffle tree) -> deterministic, no serial triangular solves.
__global__ void __launch_bounds__(256)
solve_wave_kernel(const SolveOp* __restrict__ ops, const ListEnt* __restrict__ lists, int first,
                  int count, double* __restrict__ W) {
  extern __shared__ double v[];  // n (+ Csrc gather for backward)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int oi = blockIdx.x; oi < count; oi += gridDim.x) {
    const SolveOp op = ops[first + oi];
    const int n = op.n, m = op.m;
    if (op.type == OP_FWD_ELIM) {
      double* rx = v + n;  // rhs_x staged in smem
      for (int i = threadIdx.x; i < m; i += blockDim.x) rx[i] = W[op.a + i];
      __syncthreads();
      for (int i = warp; i < n; i += nw) {
        const double* row = op.LU + (size_t)i * n;  // P^{-1} row i, first m columns
        double s = 0.0;
        for (int j = lane; j < m; j += 32) s = fma(row[j], rx[j], s);
        s = warp_sum(s);
        if (lane == 0) v[i] = s;
      }
      __syncthreads();
      for (int l = op.list0; l < op.list0 + op.nlist; ++l) {
        const ListEnt t = lists[l];
        for (int i = warp; i < t.len; i += nw) {
          const double* row = op.M + (size_t)(t.off + i) * op.ldm;
          double s = 0.0;
          for (int j = lane; j < m; j += 32) s = fma(row[j], v[j], s);
          s = warp_sum(s);
          if (lane == 0) W[t.slot + i] = W[t.slot + i] - s;
        }
      }
      for (int i = threadIdx.x; i < op.k; i += blockDim.x) W[op.b + i] = W[op.b + i] + v[m + i];
      __syncthreads();
      continue;
    }
    // OP_BWD_ELIM
    double* gsol = v + n;
    for (int l = op.list0; l < op.list0 + op.nlist; ++l) {
      const ListEnt s = lists[l];
      for (int j = threadIdx.x; j < s.len; j += blockDim.x) gsol[s.off + j] = W[s.slot + j];
    }
    __syncthreads();
    for (int i = warp; i < m; i += nw) {
      const double* row = op.M + (size_t)i * op.ldm;
      double s = 0.0;
      for (int j = lane; j < op.cols; j += 32) s = fma(row[j], gsol[j], s);
      s = warp_sum(s);
      if (lane == 0) v[i] = W[op.a + i] - s;
    }
    for (int i = threadIdx.x; i < op.k; i += blockDim.x) v[m + i] = W[op.b + i];
    __syncthreads();
    for (int i = warp; i < n; i += nw) {
      const double* row = op.LU + (size_t)i * n;
      double s = 0.0;
      for (int j = lane; j < n; j += 32) s = fma(row[j], v[j], s);
      s = warp_sum(s);
      if (lane == 0) {
        if (i < m) W[op.c + i] = s;
        else W[op.d + i - m] = s;
      }
    }
    __syncthreads();
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
__global__ void top_diag_kernel(const double* LU, int n, int b0, int bs, double* v, int upper) {
  const int lane = threadIdx.x;
  if (!upper) {
    for (int i = b0 + 1; i < b0 + bs; ++i) {
      const double* L = LU + (size_t)i * n;
      double s = 0.0;
      for (int j = b0 + lane; j < i; j += 32) s = fma(L[j], v[j], s);
      s = warp_sum(s);
      if (lane == 0) v[i] -= s;
      __syncwarp();
    }
  } else {
    for (int i = b0 + bs - 1; i >= b0; --i) {
      const double* U = LU + (size_t)i * n;
      double s = 0.0;
      for (int j = i + 1 + lane; j < b0 + bs; j += 32) s = fma(U[j], v[j], s);
      s = warp_sum(s);
      if (lane == 0) v[i] = (v[i] - s) / U[i];
      __syncwarp();
    }
  }
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

__global__ void gather_perm_kernel(const double* b, const int* perm, int n, double* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = b[perm[i]];
}
__global__ void scatter_perm_kernel(const double* in, const int* perm, int n, double* x) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) x[perm[i]] = in[i];
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
  const long long wtot = top;
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
  const size_t ob = all.size() * sizeof(SolveOp), lb = lists.size() * sizeof(ListEnt);
  P.ops_d = C.alloc(1, (int)(ob / 8 + 1));
  P.list_d = C.alloc(1, (int)(lb / 8 + 1));
  if (ob) CUDA_CHECK(cudaMemcpyAsync(P.ops_d.p, all.data(), ob, cudaMemcpyHostToDevice, C.st));
  if (lb) CUDA_CHECK(cudaMemcpyAsync(P.list_d.p, lists.data(), lb, cudaMemcpyHostToDevice, C.st));
  P.work = C.alloc(1, (int)std::max<long long>(wtot, 1));
  C.sync();  // host vectors die here
}

void Factor::solve(const double* d_b, double* d_x) {
  Ctx& C = *ctx;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(solve_wave_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(top_solve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr = true;
  }
  IFMM_ASSERT(prog->smem <= 25000, "solve vector exceeds shared memory");
  Program& P = *prog;
  const int N = n_points;
  double* W = P.work.p;
  // algorithmic bytes: P^{-1}[:, :m] + T (forward), S + P^{-1} (backward)
  double solve_bytes = 0;
  for (auto& e : elims) {
    const double n = e.m + e.k;
    solve_bytes += 8.0 * (n * e.m + n * n + (double)e.Tstk.r * e.m + (double)e.m * e.Scat.c);
  }
  const size_t wbytes = (size_t)P.work.r * P.work.c * sizeof(double);
  CUDA_CHECK(cudaMemsetAsync(W, 0, wbytes, C.st));
  gather_perm_kernel<<<(N + 255) / 256, 256, 0, C.st>>>(d_b, d_perm, N, W);
  const SolveOp* ops = reinterpret_cast<const SolveOp*>(P.ops_d.p);
  const ListEnt* lists = reinterpret_cast<const ListEnt*>(P.list_d.p);
  const size_t smem = (size_t)std::max(P.smem, 1) * sizeof(double);
  cudaEvent_t ka = nullptr;
  C.kt_begin(K_SOLVE, 0, &ka);
  for (int w = 0; w < P.fwd_waves; ++w) {
    const int a = P.fwd_wave_start[w], b = P.fwd_wave_start[w + 1];
    solve_wave_kernel<<<std::min(b - a, 65535), 256, smem, C.st>>>(ops, lists, a, b - a, W);
  }
  if (P.top_n > 0 && P.top_n <= 20000) {
    top_solve_kernel<<<1, 1024, (size_t)P.top_n * sizeof(double), C.st>>>(
        top_lu.p, top_piv, P.top_n, W + P.top_rhs, W + P.top_sol);
  } else if (P.top_n > 0) {
    const int n = P.top_n, bs = 256;
    double* v = W + P.top_sol;
    CUDA_CHECK(cudaMemcpyAsync(v, W + P.top_rhs, sizeof(double) * n, cudaMemcpyDeviceToDevice, C.st));
    top_perm_kernel<<<1, 32, 0, C.st>>>(top_piv, n, v);
    for (int b0 = 0; b0 < n; b0 += bs) {  // L (unit) forward
      const int b = std::min(bs, n - b0);
      top_diag_kernel<<<1, 32, 0, C.st>>>(top_lu.p, n, b0, b, v, 0);
      if (b0 + b < n)
        top_update_kernel<<<(n - b0 - b + 7) / 8, 256, 0, C.st>>>(top_lu.p, n, b0 + b, n, b0, b, v);
    }
    for (int b0 = ((n - 1) / bs) * bs; b0 >= 0; b0 -= bs) {  // U backward
      const int b = std::min(bs, n - b0);
      top_diag_kernel<<<1, 32, 0, C.st>>>(top_lu.p, n, b0, b, v, 1);
      if (b0 > 0) top_update_kernel<<<(b0 + 7) / 8, 256, 0, C.st>>>(top_lu.p, n, 0, b0, b0, b, v);
    }
  }
  for (int w = 0; w < P.bwd_waves; ++w) {
    const int a = P.n_fwd + P.bwd_wave_start[w], b = P.n_fwd + P.bwd_wave_start[w + 1];
    solve_wave_kernel<<<std::min(b - a, 65535), 256, smem, C.st>>>(ops, lists, a, b - a, W);
  }
  scatter_perm_kernel<<<(N + 255) / 256, 256, 0, C.st>>>(W + P.sol0, d_perm, N, d_x);
  C.kt_end(K_SOLVE, solve_bytes, ka);
  C.launches += 3 + P.fwd_waves + P.bwd_waves;
  CUDA_CHECK(cudaGetLastError());
}

}  // namespace ifmm
