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
#include <condition_variable>
#include <cstring>
#include <mutex>
#include <thread>
#include <cstdio>
#include <cstdlib>

#include "engine.h"

// numpy's own standard-normal sampler (the ziggurat of
// numpy/random/src/distributions, linked from numpy's static libnpyrandom)
// driven by a native PCG64 below: together, bit for bit the stream of
// np.random.Generator(np.random.PCG64(seed)).standard_normal.
extern "C" {
struct npy_bitgen {
  void* state;
  uint64_t (*next_uint64)(void* st);
  uint32_t (*next_uint32)(void* st);
  double (*next_double)(void* st);
  uint64_t (*next_raw)(void* st);
};
void random_standard_normal_fill(npy_bitgen* bitgen_state, long cnt, double* out);
}

namespace ifmm {

// PCG64 (O'Neill's pcg_setseq_128 with the XSL-RR 128/64 output), numpy's
// default bit generator: step, then output from the new state.
struct Pcg64 {
  unsigned __int128 state = 0, inc = 0;
  static uint64_t next64(void* p) {
    Pcg64& g = *static_cast<Pcg64*>(p);
    const unsigned __int128 mul =
        ((unsigned __int128)0x2360ED051FC65DA4ULL << 64) | 0x4385DF649FCCF645ULL;
    g.state = g.state * mul + g.inc;
    const uint64_t x = (uint64_t)(g.state >> 64) ^ (uint64_t)g.state;
    const unsigned rot = (unsigned)(g.state >> 122);
    return (x >> rot) | (x << ((-rot) & 63));
  }
  static uint32_t next32(void* p) { return (uint32_t)(next64(p) >> 32); }  // unused by normals
  static double next_double(void* p) { return (double)(next64(p) >> 11) * (1.0 / 9007199254740992.0); }
  void fill(double* out, long long n) {
    npy_bitgen bg{this, &Pcg64::next64, &Pcg64::next32, &Pcg64::next_double, &Pcg64::next64};
    random_standard_normal_fill(&bg, (long)n, out);
  }
};

// Native reference stream: the NormalSource protocol over the PCG64 normal
// sequence.  The sequence is fixed, so a saved state is just a position:
// a producer thread runs ahead of the consumer filling 1 M-normal chunks
// (hidden behind the device work), draws copy [pos, pos + n) out of the
// chunks, save / restore record / reset pos.  Chunks far behind pos are freed.
struct PcgSource {
  static constexpr long long kChunk = 1 << 20, kAhead = 24 * kChunk, kKeep = 32 * kChunk;
  Pcg64 g;                                   // producer-owned
  std::map<long long, std::vector<double>> chunks;  // chunk index -> normals
  long long produced = 0, pos = 0;           // normals generated / consumer position
  std::vector<long long> slots;
  std::mutex mu;
  std::condition_variable cv;
  bool stop = false;
  std::thread th;
  void start() { th = std::thread([this] { run(); }); }
  ~PcgSource() {
    { std::lock_guard<std::mutex> l(mu); stop = true; }
    cv.notify_all();
    if (th.joinable()) th.join();
  }
  void run() {
    std::vector<double> buf(kChunk);
    for (;;) {
      {
        std::unique_lock<std::mutex> l(mu);
        cv.wait(l, [&] { return stop || produced < pos + kAhead; });
        if (stop) return;
      }
      g.fill(buf.data(), kChunk);  // outside the lock
      std::lock_guard<std::mutex> l(mu);
      chunks[produced / kChunk] = buf;
      produced += kChunk;
      const long long lo = (pos - kKeep) / kChunk;  // free what no restore can reach
      while (!chunks.empty() && chunks.begin()->first < lo) chunks.erase(chunks.begin());
      cv.notify_all();
    }
  }
  void copy_out(long long p, long long n, double* out) {
    std::unique_lock<std::mutex> l(mu);
    cv.notify_all();
    cv.wait(l, [&] { return produced >= p + n; });
    while (n > 0) {
      const long long ci = p / kChunk, o = p % kChunk;
      const long long take = std::min(n, kChunk - o);
      const std::vector<double>& c = chunks.at(ci);
      std::memcpy(out, c.data() + o, sizeof(double) * take);
      out += take; p += take; n -= take;
    }
  }
  static int call(void* user, int op, long long n, double* out) {
    PcgSource& s = *static_cast<PcgSource*>(user);
    if (op == 0) {
      s.copy_out(s.pos, n, out);
      std::lock_guard<std::mutex> l(s.mu);
      s.pos += n;
      s.cv.notify_all();
      return 0;
    }
    if (n < 0) return 1;
    if (op == 1) { if ((long long)s.slots.size() <= n) s.slots.resize(n + 1); s.slots[n] = s.pos; return 0; }
    if (op == 2) {
      if (n >= (long long)s.slots.size() || s.slots[n] < s.pos - kKeep) return 1;
      std::lock_guard<std::mutex> l(s.mu);
      s.pos = s.slots[n];
      return 0;
    }
    return 1;
  }
};

int pcg64_normals(const uint64_t st[4], long long n, double* out) {
  Pcg64 g;
  g.state = ((unsigned __int128)st[0] << 64) | st[1];
  g.inc = ((unsigned __int128)st[2] << 64) | st[3];
  g.fill(out, n);
  return 0;
}

Factor* factorize_pcg64(Graph* g, double eps, double sigma0, int flags, const uint64_t st[4]) {
  PcgSource src;
  src.g.state = ((unsigned __int128)st[0] << 64) | st[1];
  src.g.inc = ((unsigned __int128)st[2] << 64) | st[3];
  src.start();
  return factorize(g, eps, sigma0, flags, &PcgSource::call, &src);
}

static constexpr int TOP_TAG = 0x7fffffff - 1;

// ---- IFMM_SYMCHECK (parity triage): asymmetry of the graph ----------------
// For a symmetric kernel the extended matrix stays symmetric through the
// elimination up to rounding; symcheck reports max ||E(a,b) - E(b,a)^T|| /
// ||E(a,b)|| over all edge pairs (one CTA per pair).
struct AsymDesc { const double* A; const double* B; int r, c; double* out; };
__global__ void asym_kernel(const AsymDesc* d, int n) {
  __shared__ double sd[2][32];
  for (int b = blockIdx.x; b < n; b += gridDim.x) {
    const AsymDesc q = d[b];
    double s1 = 0.0, s2 = 0.0;
    for (int e = threadIdx.x; e < q.r * q.c; e += blockDim.x) {
      const int i = e / q.c, j = e % q.c;
      const double a = q.A[e], bt = q.B[(size_t)j * q.r + i];
      s1 += (a - bt) * (a - bt);
      s2 += a * a;
    }
    for (int o = 16; o; o >>= 1) { s1 += __shfl_xor_sync(0xffffffffu, s1, o); s2 += __shfl_xor_sync(0xffffffffu, s2, o); }
    if ((threadIdx.x & 31) == 0) { sd[0][threadIdx.x >> 5] = s1; sd[1][threadIdx.x >> 5] = s2; }
    __syncthreads();
    if (threadIdx.x == 0) {
      double t1 = 0, t2 = 0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) { t1 += sd[0][w]; t2 += sd[1][w]; }
      q.out[0] = t1; q.out[1] = t2;
    }
    __syncthreads();
  }
}
static void symcheck(Ctx& C, Graph& g, const char* where) {
  std::vector<AsymDesc> d;
  std::vector<std::pair<int, int>> keys;
  for (auto& kv : g.E) {
    const int t = (int)(kv.first >> 32), s = (int)(kv.first & 0xffffffffu);
    if (t > s) continue;
    Blk* o = g.get(s, t);
    if (!o || o->r != kv.second.c || o->c != kv.second.r || kv.second.r * kv.second.c == 0) continue;
    d.push_back({kv.second.p, o->p, kv.second.r, kv.second.c, nullptr});
    keys.push_back({t, s});
  }
  if (d.empty()) return;
  Blk out = C.alloc(1, 2 * (int)d.size());
  for (size_t i = 0; i < d.size(); ++i) d[i].out = out.p + 2 * i;
  AsymDesc* dd = C.stage.push_vec(C, d);
  asym_kernel<<<(int)std::min<size_t>(d.size(), 65535), 256, 0, C.st>>>(dd, (int)d.size());
  std::vector<double> h(2 * d.size());
  CUDA_CHECK(cudaMemcpyAsync(h.data(), out.p, 8 * h.size(), cudaMemcpyDeviceToHost, C.st));
  C.sync();
  double worst = 0, sum = 0;
  size_t wi = 0;
  int over = 0;
  for (size_t i = 0; i < d.size(); ++i) {
    const double r = h[2 * i + 1] > 0 ? std::sqrt(h[2 * i] / h[2 * i + 1]) : 0.0;
    sum += r;
    if (r > 1e-8) ++over;
    if (r > worst) { worst = r; wi = i; }
  }
  const int t = keys[wi].first, s = keys[wi].second;
  fprintf(stderr, "[symcheck] %s: %zu pairs, mean %.2e, max %.2e (>1e-8: %d) at (%d[%c c%d], %d[%c c%d]) %dx%d\n",
          where, d.size(), sum / d.size(), worst, over, t, "xzy"[g.kind[t]], g.owner[t], s,
          "xzy"[g.kind[s]], g.owner[s], d[wi].r, d[wi].c);
  C.free(out);
  C.flush();
}
static int symcheck_every() {
  static int v = -1;
  if (v < 0) { const char* e = getenv("IFMM_SYMCHECK"); v = e ? atoi(e) : 0; }
  return v;
}

// IFMM_TRACE=<file>: per-pair decision trace (debug / parity triage)
// IFMM_PROFILE=1: stream-synchronised phase timers (diagnostics; perturbs
// overlap, never used for reported numbers)
enum { PH_LU = 0, PH_XSOLVE, PH_SCHUR, PH_ADD, PH_FILLSVD, PH_UNION, PH_REBASE, PH_NEWK, PH_MERGE,
       PH_TOP, PH_HOST, PH_RSVD, PH_N };
double g_prof[PH_N];
// IFMM_PROFILE=2: host-only phase timers (no synchronisation): host
// enqueue/bookkeeping cost per phase.
static int prof_mode() {
  static int on = -1;
  if (on < 0) { const char* p = getenv("IFMM_PROFILE"); on = (p && *p) ? (*p - '0') : 0; }
  return on;
}
static bool prof_on() { return prof_mode() != 0; }
struct Phase {
  Ctx& C;
  int id;
  std::chrono::steady_clock::time_point t0;
  static int bucket_of(int ph) {
    switch (ph) {
      case PH_LU: case PH_XSOLVE: case PH_TOP: return 0;   // lu_and_triangular_solves
      case PH_SCHUR: case PH_ADD: return 1;                // matmul_updates
      case PH_MERGE: return 3;                             // operator_transfer
      default: return 2;                                   // lowrank_approximations
    }
  }
  Phase(Ctx& c, int i) : C(c), id(i) {
    C.bucket(bucket_of(i));
    if (prof_on()) { if (prof_mode() == 1) C.sync(); t0 = std::chrono::steady_clock::now(); }
  }
  ~Phase() {
    if (prof_on()) {
      if (prof_mode() == 1) C.sync();
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
    if (f) setvbuf(f, nullptr, _IOLBF, 0);  // complete lines even if the process dies
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
std::vector<std::vector<int>> cluster_waves(const Tree& T, int level, bool exact, bool colored = false);

struct Eliminator {
  Ctx& C;
  Graph& g;
  Factor& F;
  double thr;
  std::mt19937_64 rng;
  Blk d_ranks;  // device int scratch
  int d_ranks_cap = 0;
  double flops_gemm = 0, flops_all = 0;

  // the reference's factorize rng (factor.py:188, Generator(PCG64(seed))):
  // when set, every Gaussian the reference draws -- rSVD sketches
  // (lowrank.py:108) and _extend_update padding (factor.py:350) -- comes
  // from this stream in the reference's call order
  NormalSource src = nullptr;
  void* src_user = nullptr;
  void draw(double* out, long long n) {
    if (src(src_user, 0, n, out) != 0) throw Error(E_VALUE, "normal source callback failed");
  }
  void src_op(int op, long long slot) {
    if (src(src_user, op, slot, nullptr) != 0) throw Error(E_VALUE, "normal source callback failed");
  }

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

  // IFMM_UNION_LOG=<file>: one line per union launch (diagnostics)
  static FILE* union_log() {
    static FILE* f = nullptr;
    static bool init = false;
    if (!init) {
      init = true;
      if (const char* n = getenv("IFMM_UNION_LOG")) f = fopen(n, "w");
    }
    return f;
  }
  // In-flight union launch of one pair wave (readback pending).
  struct UnionsInFlight {
    std::vector<UReq> reqs;
    int* dr = nullptr;
    Blk gflags;
    bool giants = false;
    std::chrono::steady_clock::time_point tl0, tl1;
    size_t ns = 0, ng = 0;
    bool active = false;
  };
  void launch_unions(std::vector<UReq>& reqs) {
    UnionsInFlight f;
    launch_unions_async(reqs, f);
    complete_unions(f);
  }
  void launch_unions_async(std::vector<UReq>& reqs, UnionsInFlight& fl) {
    fl.active = false;
    if (reqs.empty()) return;
    fl.reqs = reqs;
    fl.active = true;
    int* dr = ranks_buf((int)reqs.size());
    fl.dr = dr;
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
    std::vector<UnionDesc> us, ug;  // shared-memory vs global-workspace unions
    std::vector<UnionDesc> giants;  // global-workspace unions with a multi-CTA core SVD
    int jsd = 0;                    // shared memory for the large unions' core SVD
    int max_gs = 0;
    for (auto& u : ud) {
      const int sm = std::min(u.m, u.k_old + u.k_f);
      u.giant = 0;
      if (union_fits_smem(u.m, u.k_old, u.k_f)) { us.push_back(u); continue; }
      if (sm > giant_union_threshold() && (int)giants.size() < kMaxGiantsPerLaunch) {
        u.giant = 1;
        giants.push_back(u);
        max_gs = std::max(max_gs, sm);
      }
      ug.push_back(u);
      if (2 * sm * sm <= 28500) jsd = std::max(jsd, 2 * sm * sm);
    }
    // register-resident ACA (union_aca.cu) for every non-giant union whose
    // residual fits a register tile; IFMM_ACA_REG=0 keeps the legacy ACA
    static int aca_reg = -1;
    if (aca_reg < 0) {
      const char* e = getenv("IFMM_ACA_REG");
      aca_reg = e ? atoi(e) : 1;
    }
    // fused second half (union_post.cu) for the register-ACA unions it can
    // take (giant = 3); IFMM_UNION_POST=0 keeps union_kernel / union_svd_kernel
    static int use_post = -1;
    if (use_post < 0) {
      const char* e = getenv("IFMM_UNION_POST");
      use_post = e ? atoi(e) : 1;
    }
    // The fused path resolves the core's singular values to ~1e-13 of its
    // scale (first-order second CholeskyQR pass); rank decisions at
    // eps < 1e-8 need more (at c2, eps = 1e-10, it moved 4 of ~20,000
    // decisions against the reference), so those configurations keep the
    // two-pass kernels.
    const bool post_ok = use_post && F.eps >= 1e-8;
    int rs_g = 0, rs_er = 0, rs_ec = 0, rg_g = 0, rg_er = 0, rg_ec = 0;
    bool reg_s = false, reg_g = false;
    bool post_s = false, post_g = false, legacy_s = !us.empty(), legacy_g = !ug.empty();
    if (aca_reg && !legacy_only) {
      int mm = 0, mc = 0;
      for (auto& u : us) { mm = std::max(mm, u.m); mc = std::max(mc, u.k_old + u.k_f); }
      reg_s = !us.empty() && union_aca_reg_class(mm, mc, &rs_g, &rs_er, &rs_ec);
      if (reg_s) {
        legacy_s = false;
        for (auto& u : us) {
          u.giant = (post_ok && union_post_eligible(u.m, u.k_old, u.k_f)) ? 3 : 2;
          (u.giant == 3 ? post_s : legacy_s) = true;
        }
      }
      mm = 0; mc = 0;
      for (auto& u : ug)
        if (!u.giant) { mm = std::max(mm, u.m); mc = std::max(mc, u.k_old + u.k_f); }
      reg_g = mm > 0 && union_aca_reg_class(mm, mc, &rg_g, &rg_er, &rg_ec);
      if (reg_g) {
        legacy_g = false;
        for (auto& u : ug) {
          if (!u.giant) u.giant = (post_ok && union_post_eligible(u.m, u.k_old, u.k_f)) ? 3 : 2;
          (u.giant == 3 ? post_g : legacy_g) = true;
        }
      }
    }
    UnionDesc* dus = us.empty() ? nullptr : C.stage.push_vec(C, us);
    UnionDesc* dug = ug.empty() ? nullptr : C.stage.push_vec(C, ug);
    UnionDesc* dgi = giants.empty() ? nullptr : C.stage.push_vec(C, giants);
    Blk gflags;
    if (!giants.empty()) gflags = C.alloc(1, union_giant_scratch_doubles((int)giants.size()));
    double* dfl = giants.empty() ? nullptr : gflags.p;
    const int ngi = (int)giants.size();
    int max_gm = 0, max_gc = 0;
    for (auto& u : giants) { max_gm = std::max(max_gm, u.m); max_gc = std::max(max_gc, u.k_old + u.k_f); }
    cudaEvent_t ka = nullptr;
    FILE* ulog = union_log();
    auto tl0 = std::chrono::steady_clock::now();
    if (ulog) CUDA_CHECK(cudaStreamSynchronize(C.st));
    auto tl1 = std::chrono::steady_clock::now();
    C.kt_begin(K_UNION, uflops, &ka);
    auto run_s = [&](cudaStream_t s) {
      if (reg_s) launch_union_aca_reg(dus, (int)us.size(), thr, rs_g, rs_er, rs_ec, s);
      if (post_s) launch_union_post(dus, (int)us.size(), thr, s);
      if (legacy_s) launch_union(dus, (int)us.size(), thr, s, 1);
    };
    auto run_g = [&](cudaStream_t s, int reserved) {
      if (reg_g) launch_union_aca_reg(dug, (int)ug.size(), thr, rg_g, rg_er, rg_ec, s);
      if (post_g) launch_union_post(dug, (int)ug.size(), thr, s);
      if (legacy_g)
        launch_union(dug, (int)ug.size(), thr, s, 0, jsd, dgi, ngi, max_gs, dfl, max_gm, max_gc, reserved);
    };
    if (dus && dug)
      C.fork2([&](cudaStream_t s) { run_s(s); }, [&](cudaStream_t s) { run_g(s, (int)us.size()); });
    else if (dus) run_s(C.st);
    else run_g(C.st, 0);
    C.kt_end(K_UNION, uflops, ka);
    C.launches += (!us.empty()) + (!ug.empty());
    CUDA_CHECK(cudaGetLastError());
    fl.gflags = gflags;
    fl.giants = !giants.empty();
    fl.tl0 = tl0;
    fl.tl1 = tl1;
    fl.ns = us.size();
    fl.ng = ug.size();
  }
  void complete_unions(UnionsInFlight& fl) {
    if (!fl.active) return;
    fl.active = false;
    std::vector<UReq>& reqs = fl.reqs;
    FILE* ulog = union_log();
    const auto tl0 = fl.tl0, tl1 = fl.tl1;
    const size_t nus = fl.ns, nug = fl.ng;
    const int* hr0 = C.readback_ints(fl.dr, reqs.size());
    std::vector<int> hrv(hr0, hr0 + reqs.size());
    const int* hr = hrv.data();
    if (ulog) {
      auto tl2 = std::chrono::steady_clock::now();
      int mm = 0, mc = 0, mk = 0;
      for (size_t i = 0; i < reqs.size(); ++i) {
        mm = std::max(mm, reqs[i].bu->m);
        mc = std::max(mc, reqs[i].bu->k_old + reqs[i].bu->k_f);
        mk = std::max(mk, hr[i]);
      }
      static auto prev = tl0;
      fprintf(ulog, "%zu %zu %d %d %d %.3f %.3f %.3f\n", nus, nug, mm, mc, mk,
              std::chrono::duration<double, std::milli>(tl2 - tl1).count(),
              std::chrono::duration<double, std::milli>(tl1 - tl0).count(),
              std::chrono::duration<double, std::milli>(tl0 - prev).count());
      prev = tl2;
    }
    std::vector<UReq> redo;
    for (size_t i = 0; i < reqs.size(); ++i) {
      reqs[i].bu->rank = hr[i];
      C.free(reqs[i].bu->W);
      if (hr[i] < 0) redo.push_back(reqs[i]);  // union_post_kernel declined it
    }
    if (fl.giants) C.free(fl.gflags);
    if (!redo.empty()) {
      post_fallbacks += redo.size();
      const bool was = legacy_only;
      legacy_only = true;
      launch_unions(redo);
      legacy_only = was;
    }
  }
  // A wave's clusters in chunks whose Schur fill matrices (the largest
  // per-cluster temporaries: NR x NC, plus X) stay within IFMM_WAVE_GB
  // (default 6) GB, so the big colour waves of the upper levels fit the arena.
  std::vector<std::vector<int>> split_wave(const std::vector<int>& wave) {
    static double budget = -1.0;
    if (budget < 0) {
      const char* e = getenv("IFMM_WAVE_GB");
      budget = (e ? atof(e) : 6.0) * 1073741824.0;
    }
    std::vector<std::vector<int>> out(1);
    double acc = 0.0;
    for (int c : wave) {
      const int nx = g.nx[c];
      double R = g.size[g.nz[c]], Cc = R;
      for (int a : g.cols[nx]) R += g.size[a];
      for (int b : g.rows[nx]) Cc += g.size[b];
      const double need = 8.0 * (R * Cc + 2.0 * (g.size[nx] + g.size[g.nz[c]]) * (Cc + g.size[nx]));
      if (!out.back().empty() && acc + need > budget) {
        out.emplace_back();
        acc = 0.0;
      }
      out.back().push_back(c);
      acc += need;
    }
    return out;
  }
  bool legacy_only = false;  // reruns of unions the fused second half declined
  unsigned long long post_fallbacks = 0;

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
  struct RebaseReq {
    int c, partner;
    BU* bu;
    BU* bv;
  };
  void rebase_basis(std::vector<RebaseReq>& reqs);
  void rebase_edges(std::vector<RebaseReq>& reqs);
  void rebase_many(std::vector<RebaseReq>& reqs) { rebase_basis(reqs); rebase_edges(reqs); }
  struct PairJob {
    int cj, ck;
    const FillFac* f_kj;
    const FillFac* f_jk;
    bool ej = false, ek = false;
    int r1 = 0, r2 = 0;
    BU uj, vj, uk, vk;  // live-dead: (uj, vj) belong to the live cluster
    Blk old_kj, old_jk;
    bool has_kj = false, has_jk = false;
  };
  bool exact_order = false;
  void process_pairs(std::vector<PairJob>& pairs, LevelStats& st);
  void run_wave(std::vector<PairJob*>& jobs, LevelStats& st);
  void wave_launch(std::vector<PairJob*>& jobs, LevelStats& st, UnionsInFlight& fl);
  void wave_complete(std::vector<PairJob*>& jobs, LevelStats& st, UnionsInFlight& fl);
  void wave_basis(std::vector<PairJob*>& jobs, std::vector<RebaseReq>& reqs);
  void wave_rest(std::vector<PairJob*>& jobs, std::vector<RebaseReq>& reqs, LevelStats& st);
  void eliminate_wave(const std::vector<int>& cs, LevelStats& st);
  bool exact_fill = false;
  unsigned long long rsvd_calls = 0;
  template <class T>
  std::vector<unsigned long long> items_key(const T& items) {
    std::vector<unsigned long long> k;
    for (auto& it : items)
      k.push_back(((unsigned long long)(unsigned)it.first.first << 32) | (unsigned)it.first.second);
    return k;
  }
  struct RsvdAct { int i, m, n, full, k_try; };
  std::vector<int> rsvd_round(std::vector<SvdDesc>& sd, std::vector<RsvdAct>& act,
                              const std::vector<unsigned long long>* keys,
                              const std::vector<double, PinnedAlloc<double>>* h_omega);
  void rsvd_fills(std::vector<SvdDesc>& sd, const std::vector<int>& big,
                  const std::vector<unsigned long long>& keys, int* dr);
  void rsvd_fills_ref(std::vector<SvdDesc>& sd, const std::vector<int>& order);
  unsigned long long rsvd_redraws = 0;
  std::vector<double, PinnedAlloc<double>> rs_h;
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
  std::vector<double> G((size_t)m * extra);
  if (src) {
    // rng.standard_normal((m, extra)) is row-major; launch_extend wants m x extra col-major
    std::vector<double> R((size_t)m * extra);
    draw(R.data(), (long long)R.size());
    for (int i = 0; i < m; ++i)
      for (int j = 0; j < extra; ++j) G[(size_t)j * m + i] = R[(size_t)i * extra + j];
  } else {
    std::normal_distribution<double> nd(0.0, 1.0);
    for (auto& x : G) x = nd(rng);
  }
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

// _apply_rebase (factor.py:395-430) for every cluster of one pair wave.
// Row-side updates r E of all clusters run first, then column-side updates
// E t^T read the already row-updated blocks, so an edge between two clusters
// of the wave receives r_j E t_l^T (the reference applies the same two
// products in pair order; matrix products associate).
void Eliminator::rebase_basis(std::vector<RebaseReq>& reqs) {
  Phase ph(C, PH_REBASE);
  CopyBatch cb;
  for (auto& q : reqs) {
    const int c = q.c;
    BU& bu = *q.bu;
    BU& bv = *q.bv;
    const int nxn = g.nx[c], nzn = g.nz[c];
    const int m = g.size[nxn];
    const int kn = bu.rank, ko = bu.k_old;
    IFMM_ASSERT(bu.rank == bv.rank, "unequal U/V ranks in rebase");
    if (FILE* tf = trace_file()) fprintf(tf, "R %d %d %d %d\n", c, ko, bu.rank, bv.rank);
    if (!bu.identity || kn != ko) {
      Blk nu = C.alloc(m, kn);
      cb.add(bu.NB.p, 1, m, nu.p, kn, 1, m, kn, 0);
      g.set(nxn, nzn, nu);
      Blk w = C.alloc(1, kn);
      cb.add(bu.NW.p, 1, 1, w.p, 1, 1, 1, kn, 0);
      C.free(g.su[c]);
      g.su[c] = w;
    }
    if (!bv.identity || kn != ko) {
      Blk nv = C.alloc(kn, m);
      cb.add(bv.NB.p, m, 1, nv.p, m, 1, kn, m, 0);
      g.set(nzn, nxn, nv);
      Blk w = C.alloc(1, kn);
      cb.add(bv.NW.p, 1, 1, w.p, 1, 1, 1, kn, 0);
      C.free(g.sv[c]);
      g.sv[c] = w;
    }
  }
  cb.run(C);
}

// _apply_rebase (factor.py:395-430), edge part: every y-edge of the rebased
// clusters (rebase_basis already swapped the bases and weights).
void Eliminator::rebase_edges(std::vector<RebaseReq>& reqs) {
  Phase ph(C, PH_REBASE);
  GemmBatch rowg, colg;
  for (auto& q : reqs) {
    const int c = q.c;
    BU& bu = *q.bu;
    const int nzn = g.nz[c], nyn = g.ny[c];
    const int py = g.ny[q.partner];
    const int kn = bu.rank, ko = bu.k_old;
    IFMM_ASSERT(!g.get(nyn, nyn), "live cluster with a y-y self edge");
    if (!(bu.identity && kn == ko)) {
      // the edge set of y is unchanged by a block replacement: iterate it in
      // place, one map lookup per edge (the old block is freed at the next
      // flush, after the GEMM that reads it)
      for (int b : g.rows[nyn]) {
        if (b == nzn || b == py) continue;
        Blk* e = g.get(nyn, b);
        const Blk E = *e;
        Blk nb = C.alloc(kn, E.c);
        rowg.add(bu.OM.p, ko, 0, E.p, E.c, 0, nb.p, E.c, kn, E.c, ko, 1.0, 0.0);
        *e = nb;
        C.free_raw(E.p, E.cls);
      }
    }
  }
  run_gemm(rowg);
  for (auto& q : reqs) {
    const int c = q.c;
    BU& bu = *q.bu;
    BU& bv = *q.bv;
    const int nzn = g.nz[c], nyn = g.ny[c];
    const int py = g.ny[q.partner];
    const int kn = bu.rank, ko = bu.k_old;
    if (!(bv.identity && kn == ko)) {
      for (int a : g.cols[nyn]) {
        if (a == nzn || a == py) continue;
        Blk* e = g.get(a, nyn);
        const Blk E = *e;
        Blk nb = C.alloc(E.r, kn);
        colg.add(E.p, E.c, 0, bv.OM.p, ko, 1, nb.p, kn, E.r, kn, ko, 1.0, 0.0);
        *e = nb;
        C.free_raw(E.p, E.cls);
      }
    }
  }
  run_gemm(colg);
  CopyBatch ce;
  for (auto& q : reqs) {
    const int c = q.c;
    BU& bu = *q.bu;
    const int nzn = g.nz[c], nyn = g.ny[c];
    const int kn = bu.rank, ko = bu.k_old;
    Blk e1 = g.take(nzn, nyn), e2 = g.take(nyn, nzn);
    C.free(e1); C.free(e2);
    g.size[nzn] = kn;
    g.size[nyn] = kn;
    Blk a = C.alloc(kn, kn), b2 = C.alloc(kn, kn);
    ce.eye(a, -1.0);
    ce.eye(b2, -1.0);
    g.set(nzn, nyn, a);
    g.set(nyn, nzn, b2);
    if (!(bu.identity && kn == ko)) {
      // factor.py:429-430 records ("rebase", ny, r).  In the replay a rebase
      // always acts on a zero vector: a live cluster's y node has no edge to
      // any x node, so its rhs is untouched until its own elimination.  The
      // event is counted, r itself is not needed by the solve.
      F.rebases.push_back({nyn, Blk()});
      F.events.push_back({1, (int)F.rebases.size() - 1});
    }
  }
  ce.run(C);
}

// redirect_fillin (factor.py:433-522) for a list of fill pairs in sorted
// (min, max) order.  Dropped pairs only count; compressed pairs are grouped
// into waves of cluster-disjoint pairs (a pair's wave is one past the last
// wave that touched either of its clusters, so pairs sharing a cluster keep
// the reference order) and each wave is executed with batched launches.
void Eliminator::process_pairs(std::vector<PairJob>& pairs, LevelStats& st) {
  std::vector<PairJob*> live;
  for (auto& p : pairs) {
    p.ej = g.dead[p.cj];
    p.ek = g.dead[p.ck];
    IFMM_ASSERT(!(p.ej && p.ek), "both-eliminated fills are added, not redirected");
    p.r1 = p.f_kj ? p.f_kj->rank : 0;
    p.r2 = p.f_jk ? p.f_jk->rank : 0;
    if (p.r1 == 0 && p.r2 == 0) {
      st.dropped++;
      if (FILE* tf = trace_file()) fprintf(tf, "D %d %d\n", p.cj, p.ck);
      continue;
    }
    st.compressed++;
    st.ranks.push_back(std::max(p.r1, p.r2));
    if (FILE* tf = trace_file())
      fprintf(tf, "P %d %d %d %d %d %d\n", p.cj, p.ck, p.r1, p.r2, (int)p.ej, (int)p.ek);
    live.push_back(&p);
  }
  if (live.empty()) return;
  std::map<int, int> last;
  std::vector<int> wave(live.size());
  int maxw = 0;
  for (size_t i = 0; i < live.size(); ++i) {
    int w = 0;
    if (exact_order) w = (int)i + 1;
    else {
      auto a = last.find(live[i]->cj), b = last.find(live[i]->ck);
      if (a != last.end()) w = std::max(w, a->second);
      if (b != last.end()) w = std::max(w, b->second);
      w += 1;
    }
    last[live[i]->cj] = w;
    last[live[i]->ck] = w;
    wave[i] = w;
    maxw = std::max(maxw, w);
  }
  std::vector<std::vector<PairJob*>> waves(maxw + 1);
  for (size_t i = 0; i < live.size(); ++i) waves[wave[i]].push_back(live[i]);
  // Pipelined: wave w+1's unions (which read only the bases swapped by
  // rebase_basis of wave w) run on the device while the host builds wave w's
  // edge rebases and K rewrite.  Device work stays in the sequential order's
  // data dependencies (stream order); results are identical.
  //
  // Wave w's rebases and K rewrite also run on a side stream (st3), so their
  // small GEMMs overlap wave w+1's unions on the device.  st3 starts after
  // wave w's basis swap; the engine stream waits for st3 before it reads
  // wave w+1's ranks (after which wave w's freed blocks may be reused) and
  // at the end of the pairs.
  UnionsInFlight fl[2];
  wave_launch(waves[1], st, fl[1]);
  wave_complete(waves[1], st, fl[1]);
  std::vector<RebaseReq> reqs;
  for (int w = 1; w <= maxw; ++w) {
    wave_basis(waves[w], reqs);
    CUDA_CHECK(cudaEventRecord(C.side_ev, C.st));
    UnionsInFlight& nx = fl[(w + 1) & 1];
    if (w < maxw) wave_launch(waves[w + 1], st, nx);
    CUDA_CHECK(cudaStreamWaitEvent(C.st3, C.side_ev, 0));
    std::swap(C.st, C.st3);
    wave_rest(waves[w], reqs, st);
    std::swap(C.st, C.st3);
    CUDA_CHECK(cudaEventRecord(C.side_done, C.st3));
    CUDA_CHECK(cudaStreamWaitEvent(C.st, C.side_done, 0));
    if (w < maxw) wave_complete(waves[w + 1], st, nx);
  }
}

void Eliminator::run_wave(std::vector<PairJob*>& jobs, LevelStats& st) {
  UnionsInFlight fl;
  wave_launch(jobs, st, fl);
  wave_complete(jobs, st, fl);
  std::vector<RebaseReq> reqs;
  wave_basis(jobs, reqs);
  wave_rest(jobs, reqs, st);
}

void Eliminator::wave_launch(std::vector<PairJob*>& jobs, LevelStats& st, UnionsInFlight& fl) {
  // ---- unions of every cluster of the wave, one launch ----
  std::vector<UReq> pend;
  for (PairJob* pj : jobs) {
    PairJob& p = *pj;
    const int r1 = p.r1, r2 = p.r2;
    if (!p.ej && !p.ek) {
      cluster_unions(p.cj, r2 ? p.f_jk->U : nullptr, 1, r2 ? p.f_jk->m : 0, r2,
                     r2 ? p.f_jk->S : nullptr, r1 ? p.f_kj->V : nullptr, 1,
                     r1 ? p.f_kj->n : 0, r1, r1 ? p.f_kj->S : nullptr, p.uj, p.vj, st, pend);
      cluster_unions(p.ck, r1 ? p.f_kj->U : nullptr, 1, r1 ? p.f_kj->m : 0, r1,
                     r1 ? p.f_kj->S : nullptr, r2 ? p.f_jk->V : nullptr, 1,
                     r2 ? p.f_jk->n : 0, r2, r2 ? p.f_jk->S : nullptr, p.uk, p.vk, st, pend);
    } else {
      const int live = p.ej ? p.ck : p.cj;
      const FillFac* fu = p.ej ? p.f_kj : p.f_jk;  // rows on x_live, cols on y_dead
      const FillFac* fv = p.ej ? p.f_jk : p.f_kj;  // rows on y_dead, cols on x_live
      const int ru = fu ? fu->rank : 0, rv = fv ? fv->rank : 0;
      cluster_unions(live, ru ? fu->U : nullptr, 1, ru ? fu->m : 0, ru, ru ? fu->S : nullptr,
                     rv ? fv->V : nullptr, 1, rv ? fv->n : 0, rv, rv ? fv->S : nullptr, p.uj,
                     p.vj, st, pend);
    }
  }
  launch_unions_async(pend, fl);
}

void Eliminator::wave_complete(std::vector<PairJob*>& jobs, LevelStats& st, UnionsInFlight& fl) {
  complete_unions(fl);
  // ---- rank equalisation (rare relaunches) ----
  for (PairJob* pj : jobs) {
    PairJob& p = *pj;
    const int r1 = p.r1, r2 = p.r2;
    if (!p.ej && !p.ek) {
      finish_unions(p.cj, p.uj, p.vj, r2 ? p.f_jk->U : nullptr, 1, r2 ? p.f_jk->m : 0, r2,
                    r2 ? p.f_jk->S : nullptr, r1 ? p.f_kj->V : nullptr, 1, r1 ? p.f_kj->n : 0,
                    r1, r1 ? p.f_kj->S : nullptr, st);
      finish_unions(p.ck, p.uk, p.vk, r1 ? p.f_kj->U : nullptr, 1, r1 ? p.f_kj->m : 0, r1,
                    r1 ? p.f_kj->S : nullptr, r2 ? p.f_jk->V : nullptr, 1, r2 ? p.f_jk->n : 0,
                    r2, r2 ? p.f_jk->S : nullptr, st);
    } else {
      const int live = p.ej ? p.ck : p.cj;
      const FillFac* fu = p.ej ? p.f_kj : p.f_jk;
      const FillFac* fv = p.ej ? p.f_jk : p.f_kj;
      const int ru = fu ? fu->rank : 0, rv = fv ? fv->rank : 0;
      finish_unions(live, p.uj, p.vj, ru ? fu->U : nullptr, 1, ru ? fu->m : 0, ru,
                    ru ? fu->S : nullptr, rv ? fv->V : nullptr, 1, rv ? fv->n : 0, rv,
                    rv ? fv->S : nullptr, st);
    }
  }
}

void Eliminator::wave_basis(std::vector<PairJob*>& jobs, std::vector<RebaseReq>& reqs) {
  reqs.clear();
  for (size_t i = 0; i < jobs.size(); ++i) {
    PairJob& p = *jobs[i];
    if (!p.ej && !p.ek) {
      reqs.push_back({p.cj, p.ck, &p.uj, &p.vj});
      reqs.push_back({p.ck, p.cj, &p.uk, &p.vk});
    } else {
      const int live = p.ej ? p.ck : p.cj, deadc = p.ej ? p.cj : p.ck;
      reqs.push_back({live, deadc, &p.uj, &p.vj});
    }
  }
  rebase_basis(reqs);
}

void Eliminator::wave_rest(std::vector<PairJob*>& jobs, std::vector<RebaseReq>& reqs, LevelStats& st) {
  (void)st;
  // K-rewrite inputs: the current (y_k, y_j) / (y_j, y_k) blocks and y sizes,
  // taken after every earlier wave's edge rebases
  std::vector<int> kjo(jobs.size()), kko(jobs.size());
  for (size_t i = 0; i < jobs.size(); ++i) {
    PairJob& p = *jobs[i];
    const int yj = g.ny[p.cj], yk = g.ny[p.ck];
    Blk* pkj = g.get(yk, yj);
    Blk* pjk = g.get(yj, yk);
    p.has_kj = pkj != nullptr;
    p.has_jk = pjk != nullptr;
    if (p.has_kj) p.old_kj = *pkj;
    if (p.has_jk) p.old_jk = *pjk;
    kjo[i] = g.size[g.ny[p.cj]];
    kko[i] = g.size[g.ny[p.ck]];
  }
  rebase_edges(reqs);
  // ---- K-edge rewrite ----
  Phase ph(C, PH_NEWK);
  GemmBatch ga, gb2, gc;
  CopyBatch z;
  std::vector<Blk> tmp;
  struct Out { int t, s; Blk b; };
  std::vector<Out> outs;
  for (size_t i = 0; i < jobs.size(); ++i) {
    PairJob& p = *jobs[i];
    const int yj = g.ny[p.cj], yk = g.ny[p.ck];
    const int r1 = p.r1, r2 = p.r2;
    if (!p.ej && !p.ek) {
      BU &uj = p.uj, &vj = p.vj, &uk = p.uk, &vk = p.vk;
      const int kj0 = kjo[i], kk0 = kko[i];
      const int kjn = uj.rank, kkn = uk.rank;
      // new_kj = rk old_kj tj^T + (rk' s_kj) tj'^T ; new_jk = rj old_jk tk^T + (rj' s_jk) tk'^T
      Blk nkj = C.alloc(kkn, kjn), njk = C.alloc(kjn, kkn);
      if (p.has_kj) {
        Blk t1 = C.alloc(kk0, kjn);
        tmp.push_back(t1);
        ga.add(p.old_kj.p, kj0, 0, vj.OM.p, kj0, 1, t1.p, kjn, kk0, kjn, kj0, 1.0, 0.0);
        gb2.add(uk.OM.p, kk0, 0, t1.p, kjn, 0, nkj.p, kjn, kkn, kjn, kk0, 1.0, 0.0);
      }
      if (p.has_jk) {
        Blk t2 = C.alloc(kj0, kkn);
        tmp.push_back(t2);
        ga.add(p.old_jk.p, kk0, 0, vk.OM.p, kk0, 1, t2.p, kkn, kj0, kkn, kk0, 1.0, 0.0);
        gb2.add(uj.OM.p, kj0, 0, t2.p, kkn, 0, njk.p, kkn, kjn, kkn, kj0, 1.0, 0.0);
      }
      if (r1 > 0)
        gc.add(uk.FM.p, uk.k_f, 0, vj.FM.p, vj.k_f, 1, nkj.p, kjn, kkn, kjn, r1, 1.0,
               p.has_kj ? 1.0 : 0.0, p.f_kj->S);
      if (r2 > 0)
        gc.add(uj.FM.p, uj.k_f, 0, vk.FM.p, vk.k_f, 1, njk.p, kkn, kjn, kkn, r2, 1.0,
               p.has_jk ? 1.0 : 0.0, p.f_jk->S);
      if (!p.has_kj && r1 == 0) z.zero(nkj);
      if (!p.has_jk && r2 == 0) z.zero(njk);
      outs.push_back({yk, yj, nkj});
      outs.push_back({yj, yk, njk});
    } else {
      const int live = p.ej ? p.ck : p.cj, deadc = p.ej ? p.cj : p.ck;
      const FillFac* fu = p.ej ? p.f_kj : p.f_jk;
      const FillFac* fv = p.ej ? p.f_jk : p.f_kj;
      const int ru = fu ? fu->rank : 0, rv = fv ? fv->rank : 0;
      const int nd = g.size[g.ny[deadc]];
      BU &bu = p.uj, &bv = p.vj;
      const int klo = bu.k_old, kln = bu.rank;
      const bool live_is_k = live == p.ck;
      const Blk old_ld = live_is_k ? p.old_kj : p.old_jk;  // (y_live, y_dead)
      const Blk old_dl = live_is_k ? p.old_jk : p.old_kj;  // (y_dead, y_live)
      const bool has_ld = live_is_k ? p.has_kj : p.has_jk;
      const bool has_dl = live_is_k ? p.has_jk : p.has_kj;
      Blk nld = C.alloc(kln, nd), ndl = C.alloc(nd, kln);
      if (has_ld) ga.add(bu.OM.p, klo, 0, old_ld.p, nd, 0, nld.p, nd, kln, nd, klo, 1.0, 0.0);
      if (has_dl) ga.add(old_dl.p, klo, 0, bv.OM.p, klo, 1, ndl.p, kln, nd, kln, klo, 1.0, 0.0);
      if (ru > 0)
        gb2.add(bu.FM.p, bu.k_f, 0, fu->V, nd, 0, nld.p, nd, kln, nd, ru, 1.0,
                has_ld ? 1.0 : 0.0, fu->S);
      if (rv > 0)
        gb2.add(fv->U, nd, 1, bv.FM.p, bv.k_f, 1, ndl.p, kln, nd, kln, rv, 1.0,
                has_dl ? 1.0 : 0.0, fv->S);
      if (!has_ld && ru == 0) z.zero(nld);
      if (!has_dl && rv == 0) z.zero(ndl);
      outs.push_back({g.ny[live], g.ny[deadc], nld});
      outs.push_back({g.ny[deadc], g.ny[live], ndl});
    }
  }
  z.run(C);
  run_gemm(ga);
  run_gemm(gb2);
  run_gemm(gc);
  for (auto& o : outs) g.set(o.t, o.s, o.b);
  for (auto& b : tmp) C.free(b);
  for (PairJob* pj : jobs)
    for (BU* b : {&pj->uj, &pj->vj, &pj->uk, &pj->vk}) free_bu(*b);
  C.flush();
}

// _eliminate_cluster (factor.py:259-326) for a wave of clusters that are
// pairwise at Chebyshev distance >= 3 (no shared neighbour: their
// eliminations touch disjoint edges and commute).  Every stage is one
// batched launch over the wave.
void Eliminator::eliminate_wave(const std::vector<int>& cs, LevelStats& st) {
  struct W {
    int c, nx, nz, ny, m, k, n, Csrc, Rtgt, NC, NR;
    Blk P, X, Fm;
    int* piv;
    int pc;
    std::vector<Blk> srcB, tgtB;
  };
  std::vector<W> ws(cs.size());
  Phase* ph = new Phase(C, PH_LU);
  // ---- pivot blocks P = [[D, U], [V^T, 0]] and their LU ----
  {
    CopyBatch cb;
    std::vector<Blk> dead_blks;
    for (size_t i = 0; i < cs.size(); ++i) {
      W& w = ws[i];
      w.c = cs[i];
      if (FILE* tf = trace_file())
        fprintf(tf, "E %d %d %d\n", w.c, g.size[g.nx[w.c]], g.size[g.nz[w.c]]);
      w.nx = g.nx[w.c]; w.nz = g.nz[w.c]; w.ny = g.ny[w.c];
      w.m = g.size[w.nx]; w.k = g.size[w.nz]; w.n = w.m + w.k;
      Blk D = g.take(w.nx, w.nx), U = g.take(w.nx, w.nz), Vt = g.take(w.nz, w.nx);
      Blk e1 = g.take(w.nz, w.ny), e2 = g.take(w.ny, w.nz);
      w.P = C.alloc(w.n, w.n);
      cb.copy(D, w.P, 0, 0);
      cb.copy(U, w.P, 0, w.m);
      cb.copy(Vt, w.P, w.m, 0);
      cb.add(nullptr, 0, 0, w.P.p + (size_t)w.m * w.n + w.m, w.n, 1, w.k, w.k, 3);
      for (Blk b : {D, U, Vt, e1, e2}) dead_blks.push_back(b);
      w.piv = C.arena.alloc_int(w.n, &w.pc);
    }
    cb.run(C);
    for (auto& b : dead_blks) C.free(b);
    std::vector<LuDesc> small;
    double fl = 0;
    for (W& w : ws) {
      const double f3 = 2.0 / 3.0 * (double)w.n * w.n * w.n;
      flops_gemm += f3;
      flops_all += f3;
      if (w.n <= 160) {
        LuDesc d;
        d.A = w.P.p; d.n = w.n; d.lda = w.n; d.piv = w.piv; d.tag = w.c;
        small.push_back(d);
        fl += f3;
      } else {
        lu_blocked(C, w.P.p, w.n, w.n, w.piv, w.c);
      }
    }
    if (!small.empty()) {
      LuDesc* dd = C.stage.push_vec(C, small);
      cudaEvent_t ka = nullptr;
      C.kt_begin(K_LU, fl, &ka);
      launch_lu(dd, (int)small.size(), C.d_status, C.st);
      C.kt_end(K_LU, fl, ka);
      C.launches++;
      CUDA_CHECK(cudaGetLastError());
    }
  }
  delete ph;
  ph = new Phase(C, PH_XSOLVE);
  // ---- sources / targets, event records, X = P^{-1}[E(x,b);0 | 0;-I] ----
  {
    CopyBatch cb;
    std::vector<LuSolveDesc> sd;
    int max_nrhs = 0, max_n = 0;
    double fl = 0;
    for (W& w : ws) {
      ElimEv ev;
      ev.nx = w.nx; ev.nz = w.nz; ev.ny = w.ny; ev.m = w.m; ev.k = w.k;
      ev.LU = w.P; ev.piv = w.piv; ev.piv_cls = w.pc;
      w.Csrc = 0; w.Rtgt = 0;
      for (int b : std::vector<int>(g.rows[w.nx].begin(), g.rows[w.nx].end())) {
        Blk E = g.take(w.nx, b);
        ev.src.push_back(b); ev.src_off.push_back(w.Csrc); ev.src_w.push_back(E.c);
        w.Csrc += E.c;
        w.srcB.push_back(E);
      }
      for (int a : std::vector<int>(g.cols[w.nx].begin(), g.cols[w.nx].end())) {
        Blk E = g.take(a, w.nx);
        ev.tgt.push_back(a); ev.tgt_off.push_back(w.Rtgt); ev.tgt_h.push_back(E.r);
        w.Rtgt += E.r;
        w.tgtB.push_back(E);
      }
      IFMM_ASSERT(g.rows[w.nz].empty() && g.cols[w.nz].empty(),
                  "z node unexpectedly has extra edges");
      const int m = w.m, k = w.k, Csrc = w.Csrc;
      ev.Scat = C.alloc(m, std::max(Csrc, 1));
      ev.Tstk = C.alloc(std::max(w.Rtgt, 1), m);
      w.NC = Csrc + k;
      w.NR = w.Rtgt + k;
      // X = P^{-1} [[E_src, 0, I_m], [0, -I_k, 0]]: the trailing m columns and
      // the -I_k block give P^{-1} itself (kept for the solve replay)
      const int LDX = w.NC + m;
      w.X = C.alloc(w.n, LDX);
      const int NC = LDX;
      for (size_t i = 0; i < w.srcB.size(); ++i) {
        cb.add(w.srcB[i].p, w.srcB[i].c, 1, ev.Scat.p + ev.src_off[i], std::max(Csrc, 1), 1, m,
               w.srcB[i].c, 0);
        cb.add(w.srcB[i].p, w.srcB[i].c, 1, w.X.p + ev.src_off[i], NC, 1, m, w.srcB[i].c, 0);
      }
      for (size_t i = 0; i < w.tgtB.size(); ++i)
        cb.add(w.tgtB[i].p, w.tgtB[i].c, 1, ev.Tstk.p + (size_t)ev.tgt_off[i] * m, m, 1,
               w.tgtB[i].r, m, 0);
      cb.add(nullptr, 0, 0, w.X.p + (size_t)m * NC, NC, 1, k, Csrc, 3);
      cb.add(nullptr, 0, 0, w.X.p + Csrc, NC, 1, m, k, 3);
      cb.add(nullptr, 0, 0, w.X.p + (size_t)m * NC + Csrc, NC, 1, k, k, 2, -1.0);
      cb.add(nullptr, 0, 0, w.X.p + Csrc + k, NC, 1, m, m, 2, 1.0);                 // I_m
      cb.add(nullptr, 0, 0, w.X.p + (size_t)m * NC + Csrc + k, NC, 1, k, m, 3);     // 0
      g.dead[w.c] = 1;
      LuSolveDesc d;
      d.LU = w.P.p; d.piv = w.piv; d.n = w.n; d.lda = w.n; d.X = w.X.p; d.nrhs = NC; d.ldx = NC;
      sd.push_back(d);
      max_nrhs = std::max(max_nrhs, NC);
      max_n = std::max(max_n, w.n);
      const double f2 = 2.0 * w.n * w.n * (double)NC;
      flops_gemm += f2;
      flops_all += f2;
      fl += f2;
      F.elims.push_back(std::move(ev));
      F.events.push_back({0, (int)F.elims.size() - 1});
    }
    cb.run(C);
    for (W& w : ws) {
      for (auto& b : w.srcB) C.free(b);
      for (auto& b : w.tgtB) C.free(b);
    }
    LuSolveDesc* dd = C.stage.push_vec(C, sd);
    cudaEvent_t ka = nullptr;
    C.kt_begin(K_LUSOLVE, fl, &ka);
    launch_lusolve(dd, (int)sd.size(), max_nrhs, C.st, max_n);
    C.kt_end(K_LUSOLVE, fl, ka);
    C.launches++;
    CUDA_CHECK(cudaGetLastError());
  }
  delete ph;
  ph = new Phase(C, PH_SCHUR);
  // ---- Schur fill F = [-Tstk X[:m] ; X[m:]]  (NR x NC), one grouped GEMM ----
  const size_t e0 = F.elims.size() - ws.size();
  {
    GemmBatch gb;
    CopyBatch cb;
    for (size_t i = 0; i < ws.size(); ++i) {
      W& w = ws[i];
      ElimEv& ev = F.elims[e0 + i];
      const int LDX = w.NC + w.m;
      w.Fm = C.alloc(w.NR, w.NC);
      gb.add(ev.Tstk.p, w.m, 0, w.X.p, LDX, 0, w.Fm.p, w.NC, w.Rtgt, w.NC, w.m, -1.0, 0.0);
      cb.add(w.X.p + (size_t)w.m * LDX, LDX, 1, w.Fm.p + (size_t)w.Rtgt * w.NC, w.NC, 1, w.k,
             w.NC, 0);
      // P^{-1} = [X[:, NC:NC+m] | -X[:, Csrc:Csrc+k]]  (n x n)
      ev.Pinv = C.alloc(w.n, w.n);
      cb.add(w.X.p + w.NC, LDX, 1, ev.Pinv.p, w.n, 1, w.n, w.m, 0);
      cb.add(w.X.p + w.Csrc, LDX, 1, ev.Pinv.p + w.m, w.n, 1, w.n, w.k, 0, -1.0);
    }
    run_gemm(gb);
    cb.run(C);
    for (size_t i = 0; i < ws.size(); ++i) {
      W& w = ws[i];
      ElimEv& ev = F.elims[e0 + i];
      C.free(w.X);
      C.free(ev.LU);  // the solve replays with P^{-1}
      C.free_raw(ev.piv, ev.piv_cls);
      ev.piv = nullptr;
      ev.piv_cls = -1;
    }
  }
  delete ph;
  ph = new Phase(C, PH_ADD);
  // ---- classification (factor.py:301-318) ----
  struct Stash { int wi, ro, co, h, w; };
  // per eliminated cluster: (cluster pair) -> block of Fm, sorted by pair (a
  // flat vector sorted once instead of a node-based map: ~700 entries per
  // cluster, millions per level)
  std::vector<std::vector<std::pair<std::pair<int, int>, Stash>>> stash(ws.size());
  {
    CopyBatch adds;
    for (size_t wi = 0; wi < ws.size(); ++wi) {
      W& w = ws[wi];
      const ElimEv& E = F.elims[e0 + wi];
      std::vector<int> A_nodes(E.tgt), A_off(E.tgt_off), A_h(E.tgt_h);
      A_nodes.push_back(w.ny); A_off.push_back(w.Rtgt); A_h.push_back(w.k);
      std::vector<int> B_nodes(E.src), B_off(E.src_off), B_w(E.src_w);
      B_nodes.push_back(w.ny); B_off.push_back(w.Csrc); B_w.push_back(w.k);
      const int NC = w.NC;
      for (size_t ai = 0; ai < A_nodes.size(); ++ai) {
        const int a = A_nodes[ai], ca = g.owner[a];
        for (size_t bi = 0; bi < B_nodes.size(); ++bi) {
          const int b = B_nodes[bi], cbc = g.owner[b];
          const double* sub = w.Fm.p + (size_t)A_off[ai] * NC + B_off[bi];
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
            stash[wi].push_back({{ca, cbc}, {(int)wi, A_off[ai], B_off[bi], A_h[ai], B_w[bi]}});
          }
        }
      }
    }
    adds.run(C);
    for (auto& v : stash) {
      std::stable_sort(v.begin(), v.end(),
                       [](const auto& x, const auto& y) { return x.first < y.first; });
      // a cluster pair occurs once per elimination (one live node per cluster);
      // keep the map semantics (last write wins) all the same
      size_t o = 0;
      for (size_t i = 0; i < v.size(); ++i) {
        if (i + 1 < v.size() && v[i + 1].first == v[i].first) continue;
        v[o++] = v[i];
      }
      v.resize(o);
    }
  }
  delete ph;
  // IFMM_DUMP=E,cj,ck,file: raw fills (ck, cj) and (cj, ck) of one pair when
  // cluster E is eliminated (parity triage; row-major doubles after a
  // "rows cols" text line per block)
  if (const char* dp = getenv("IFMM_DUMP")) {
    int E = -1, dj = -1, dk = -1;
    char path[512] = {0};
    if (sscanf(dp, "%d,%d,%d,%511s", &E, &dj, &dk, path) == 4)
      for (size_t wi = 0; wi < ws.size(); ++wi) {
        if (ws[wi].c != E) continue;
        FILE* f = fopen(path, "wb");
        for (auto key : {std::make_pair(dk, dj), std::make_pair(dj, dk)}) {
          auto it = std::find_if(stash[wi].begin(), stash[wi].end(),
                                 [&](const auto& kv) { return kv.first == key; });
          if (it == stash[wi].end()) { fprintf(f, "0 0\n"); continue; }
          const Stash& st = it->second;
          std::vector<double> hb((size_t)st.h * st.w);
          CUDA_CHECK(cudaMemcpy2DAsync(hb.data(), 8 * (size_t)st.w, ws[wi].Fm.p + (size_t)st.ro * ws[wi].NC + st.co,
                                       8 * (size_t)ws[wi].NC, 8 * (size_t)st.w, st.h, cudaMemcpyDeviceToHost, C.st));
          C.sync();
          fprintf(f, "%d %d\n", st.h, st.w);
          fwrite(hb.data(), 8, hb.size(), f);
        }
        fclose(f);
      }
  }
  // ---- fill compression of every stashed block of the wave, one launch ----
  std::vector<std::pair<std::pair<int, int>, Stash>> items;
  std::vector<size_t> first(ws.size() + 1, 0);
  for (size_t wi = 0; wi < ws.size(); ++wi) {
    first[wi] = items.size();
    for (auto& kv : stash[wi]) items.push_back(kv);
  }
  first[ws.size()] = items.size();
  std::vector<FillFac> fac(items.size());
  Blk wsb;
  if (!items.empty()) {
    Phase ps(C, PH_FILLSVD);
    const int ns = (int)items.size();
    int maxdim = 0;
    for (auto& it : items) maxdim = std::max(maxdim, std::max(it.second.h, it.second.w));
    const int smem_dim = std::min(maxdim, 110);
    const size_t smem_d = svd_smem_doubles(smem_dim);
    size_t tot = 0;
    std::vector<size_t> uo(ns), so(ns), vo(ns), wo(ns);
    double sflops = 0;
    // Transposition-consistent exact SVDs.  For a symmetric kernel the fill
    // pair is F(b, a) = F(a, b)^T up to rounding, and the reference's LAPACK
    // SVD treats M and M^T through the same factorisation, so the singular
    // vectors of both fills agree and the U- and V-side basis unions get the
    // same input (the graph stays symmetric).  A QRCP + Jacobi SVD of M and
    // of M^T is not transposition-consistent (vectors of close singular
    // values rotate), and the full-pivot ACA of the unions is not rotation
    // invariant: so the fill whose cluster pair is (hi, lo) is factorised as
    // its transpose and U / V are swapped back.  rSVD fills keep their
    // orientation (their sketch is drawn for the fill as given, lowrank.py:108).
    std::vector<char> tr(ns, 0);
    for (int i = 0; i < ns; ++i) {
      const Stash& s = items[i].second;
      const bool rs = std::min(s.h, s.w) > 64 && !exact_fill;
      tr[i] = (!rs && items[i].first.first > items[i].first.second) ? 1 : 0;
    }
    for (int i = 0; i < ns; ++i) {
      const Stash& s = items[i].second;
      const int mn = std::min(s.h, s.w);
      uo[i] = tot; tot += (size_t)(tr[i] ? s.w : s.h) * mn;
      so[i] = tot; tot += mn;
      vo[i] = tot; tot += (size_t)(tr[i] ? s.h : s.w) * mn;
      wo[i] = tot;
      const int dm = tr[i] ? s.w : s.h, dn = tr[i] ? s.h : s.w;  // the descriptor's orientation
      if (svd_work_doubles(dm, dn) > smem_d) tot += svd_work_doubles(dm, dn);
      const double mm = std::max(s.h, s.w), nn = mn;
      sflops += 4 * mm * nn * nn + 22 * nn * nn * nn;
    }
    flops_all += sflops;
    wsb = C.alloc(1, (int)std::max<size_t>(tot, 1));
    int* dr = ranks_buf(ns);
    std::vector<SvdDesc> sd(ns);
    for (int i = 0; i < ns; ++i) {
      const Stash& s = items[i].second;
      const W& w = ws[s.wi];
      sd[i].src = w.Fm.p + (size_t)s.ro * w.NC + s.co;
      if (tr[i]) { sd[i].m = s.w; sd[i].n = s.h; sd[i].s_r = 1; sd[i].s_c = w.NC; }
      else { sd[i].m = s.h; sd[i].n = s.w; sd[i].s_r = w.NC; sd[i].s_c = 1; }
      sd[i].U = wsb.p + uo[i]; sd[i].S = wsb.p + so[i]; sd[i].V = wsb.p + vo[i];
      sd[i].rank = dr + i;
      sd[i].work = wsb.p + wo[i];
    }
    // factor.py:329-332: fills with min(shape) > 64 are compressed by the
    // randomized SVD (as the reference does); the rest exactly, through the
    // rank-revealing pivoted QR (shared- or global-memory workspace variants
    // run as two concurrent launches).
    std::vector<SvdDesc> sds, sdg;
    std::vector<int> big;
    for (int i = 0; i < ns; ++i) {
      const SvdDesc& x = sd[i];
      if (std::min(x.m, x.n) > 64 && !exact_fill) big.push_back(i);
      else (svd_work_doubles(x.m, x.n) <= smem_d ? sds : sdg).push_back(x);
    }
    SvdDesc* dss = sds.empty() ? nullptr : C.stage.push_vec(C, sds);
    SvdDesc* dsg = sdg.empty() ? nullptr : C.stage.push_vec(C, sdg);
    cudaEvent_t ka = nullptr;
    C.kt_begin(K_SVD, sflops, &ka);
    if (dss && dsg)
      C.fork2([&](cudaStream_t s) { launch_svd(dss, (int)sds.size(), thr, smem_dim, s, 0); },
              [&](cudaStream_t s) { launch_svd(dsg, (int)sdg.size(), thr, 0, s, 0); });
    else if (dss) launch_svd(dss, (int)sds.size(), thr, smem_dim, C.st, 0);
    else if (dsg) launch_svd(dsg, (int)sdg.size(), thr, 0, C.st, 0);
    C.kt_end(K_SVD, sflops, ka);
    if (!big.empty()) {
      Phase pr(C, PH_RSVD);
      if (src) {
        // reference call order: cluster (wave slot), pair (min, max), F_kj (target = max) first
        std::vector<int> order(big);
        auto rk = [&](int i) {
          const auto& k = items[i].first;
          const int lo = std::min(k.first, k.second), hi = std::max(k.first, k.second);
          return std::make_tuple(items[i].second.wi, lo, hi, k.first == hi ? 0 : 1);
        };
        std::sort(order.begin(), order.end(), [&](int a, int b) { return rk(a) < rk(b); });
        rsvd_fills_ref(sd, order);
      } else {
        rsvd_fills(sd, big, items_key(items), dr);
      }
    }
    const int* hr = C.readback_ints(dr, ns);
    for (int i = 0; i < ns; ++i) {
      if (tr[i]) {  // factors of F^T: F = (U S V^T)^T = V S U^T
        fac[i].U = sd[i].V; fac[i].S = sd[i].S; fac[i].V = sd[i].U;
        fac[i].m = sd[i].n; fac[i].n = sd[i].m;
      } else {
        fac[i].U = sd[i].U; fac[i].S = sd[i].S; fac[i].V = sd[i].V;
        fac[i].m = sd[i].m; fac[i].n = sd[i].n;
      }
      fac[i].rank = hr[i];
    }
  }
  // ---- pairs of every cluster (cluster-disjoint across the wave) ----
  std::vector<PairJob> jobs;
  for (size_t wi = 0; wi < ws.size(); ++wi) {
    // items[first[wi] .. first[wi + 1]) are sorted by (ca, cb)
    const size_t i0 = first[wi], i1 = first[wi + 1];
    auto find = [&](int ca, int cb) -> const FillFac* {
      const std::pair<int, int> key{ca, cb};
      size_t lo = i0, hi = i1;
      while (lo < hi) {
        const size_t mid = (lo + hi) / 2;
        if (items[mid].first < key) lo = mid + 1; else hi = mid;
      }
      return (lo < i1 && items[lo].first == key) ? &fac[lo] : nullptr;
    };
    std::vector<std::pair<int, int>> pairs;
    pairs.reserve(i1 - i0);
    for (size_t i = i0; i < i1; ++i)
      pairs.push_back({std::min(items[i].first.first, items[i].first.second),
                       std::max(items[i].first.first, items[i].first.second)});
    std::sort(pairs.begin(), pairs.end());
    pairs.erase(std::unique(pairs.begin(), pairs.end()), pairs.end());
    for (auto& pr : pairs) {
      PairJob pj;
      pj.cj = pr.first;
      pj.ck = pr.second;
      pj.f_kj = find(pr.second, pr.first);
      pj.f_jk = find(pr.first, pr.second);
      jobs.push_back(std::move(pj));
    }
  }
  if (!jobs.empty()) process_pairs(jobs, st);
  C.free(wsb);
  for (W& w : ws) C.free(w.Fm);
  C.flush();
}

// Randomized SVD of the large fills (lowrank.py:79-125, start_rank 16,
// oversample 10, 2 power iterations, rank doubling), batched across the
// fills: sketch, GEMMs (grouped DMMA), orthonormalisation and the final
// small SVD are one launch each per round.  rsvd_round runs one round for
// every active fill and returns the reference's "stop doubling" flags.
// h_omega (optional): the sketches, concatenated in `act` order, each
// n x w row-major exactly as rng.standard_normal((n, w)) (lowrank.py:108);
// without it a counter-based device generator draws them.
std::vector<int> Eliminator::rsvd_round(std::vector<SvdDesc>& sd, std::vector<RsvdAct>& act,
                                        const std::vector<unsigned long long>* keys,
                                        const std::vector<double, PinnedAlloc<double>>* h_omega) {
  ++rsvd_calls;
  const int na = (int)act.size();
  std::vector<Blk> Om(na), Yt(na), Zt(na), Ow(na), Fw(na);
  std::vector<RandDesc> rd;
  std::vector<OrthDesc> od;
  std::vector<RsvdFinDesc> fd;
  GemmBatch g0, g1, g2;
  Blk stopb = C.alloc(1, na / 2 + 2);
  int* d_stop = reinterpret_cast<int*>(stopb.p);
  Blk omb;
  if (h_omega) {
    omb = C.alloc(1, (int)std::max<size_t>(h_omega->size(), 1));
    CUDA_CHECK(cudaMemcpyAsync(omb.p, h_omega->data(), h_omega->size() * 8, cudaMemcpyHostToDevice,
                               C.st));  // pinned (host_buf): asynchronous
  }
  size_t ooff = 0;
  for (int t = 0; t < na; ++t) {
    RsvdAct& a = act[t];
    const SvdDesc& s = sd[a.i];
    const int w = std::min(a.k_try + 10, a.full);
    const double* M = s.src;  // row-major m x n, ld s_r
    const int ld = s.s_r;
    double* om;
    if (h_omega) {
      om = omb.p + ooff;
      ooff += (size_t)a.n * w;
    } else {
      Om[t] = C.alloc(a.n, w);
      om = Om[t].p;
      rd.push_back({om, a.n * w,
                    ((*keys)[a.i] * 0x9e3779b97f4a7c15ULL) ^ ((unsigned long long)a.k_try << 48) ^ rsvd_calls});
    }
    Yt[t] = C.alloc(w, a.m);   // Y col-major m x w
    Zt[t] = C.alloc(w, a.n);   // Z col-major n x w
    Ow[t] = C.alloc(1, a.m * w + w + 8);
    Fw[t] = C.alloc(1, w * w + 2 * w + 8);
    // Y^T = Om^T M^T ; Z^T = Q^T M ; Y^T = Z^T M^T
    g0.add(om, w, 1, M, ld, 1, Yt[t].p, a.m, w, a.m, a.n, 1.0, 0.0);
    g1.add(Yt[t].p, a.m, 0, M, ld, 0, Zt[t].p, a.n, w, a.n, a.m, 1.0, 0.0);
    g2.add(Zt[t].p, a.n, 0, M, ld, 1, Yt[t].p, a.m, w, a.m, a.n, 1.0, 0.0);
    od.push_back({Yt[t].p, a.m, w, Ow[t].p});
    RsvdFinDesc f;
    f.Bt = Zt[t].p; f.Q = Yt[t].p; f.m = a.m; f.n = a.n; f.w = w; f.k_try = a.k_try;
    f.full = a.full; f.U = s.U; f.S = s.S; f.V = s.V; f.rank = s.rank; f.stop = d_stop + t;
    f.work = Fw[t].p;
    fd.push_back(f);
  }
  if (!h_omega) launch_randn(C.stage.push_vec(C, rd), na, C.st);
  OrthDesc* dod = C.stage.push_vec(C, od);
  run_gemm(g0);
  for (int q = 0; q < 2; ++q) {  // power iterations (lowrank.py:99-100)
    launch_orth(dod, na, C.st);
    GemmBatch a1 = g1, a2 = g2;
    run_gemm(a1);
    run_gemm(a2);
  }
  launch_orth(dod, na, C.st);
  run_gemm(g1);  // B^T = M^T Q  (into Zt)
  launch_rsvd_fin(C.stage.push_vec(C, fd), na, thr, C.st);
  C.launches += 8;
  CUDA_CHECK(cudaGetLastError());
  const int* hs = C.readback_ints(d_stop, na);
  std::vector<int> stop(hs, hs + na);
  for (int t = 0; t < na; ++t) {
    C.free(Om[t]); C.free(Yt[t]); C.free(Zt[t]); C.free(Ow[t]); C.free(Fw[t]);
  }
  C.free(omb);
  C.free(stopb);
  C.flush();
  return stop;
}

// Device-generator rSVD: every fill doubles independently.
void Eliminator::rsvd_fills(std::vector<SvdDesc>& sd, const std::vector<int>& big,
                            const std::vector<unsigned long long>& keys, int* dr) {
  std::vector<RsvdAct> act;
  for (int i : big) {
    const int full = std::min(sd[i].m, sd[i].n);
    act.push_back({i, sd[i].m, sd[i].n, full, std::min(16, full)});
  }
  while (!act.empty()) {
    std::vector<int> stop = rsvd_round(sd, act, &keys, nullptr);
    std::vector<RsvdAct> next;
    for (size_t t = 0; t < act.size(); ++t)
      if (!stop[t]) {
        RsvdAct a = act[t];
        a.k_try = std::min(2 * a.k_try, a.full);
        next.push_back(a);
      }
    act.swap(next);
  }
  (void)dr;
}

// rSVD with the reference's Gaussian stream.  `order` lists the large fills
// in the reference's call order (_compress_fill of F_kj then F_jk per pair,
// pairs sorted, factor.py:321-332); call i's doubling rounds all precede call
// i+1's first round in the stream (lowrank.py:104-117).  Batched
// speculatively: every pending call runs its current round on the stream
// position it would have if no earlier pending call doubles; the calls up to
// the first one that must double are final, that one continues from the
// stream state right after its own draw, and the calls behind it are
// re-drawn from there (their sketches moved).
void Eliminator::rsvd_fills_ref(std::vector<SvdDesc>& sd, const std::vector<int>& order) {
  std::vector<RsvdAct> act;
  for (int i : order) {
    const int full = std::min(sd[i].m, sd[i].n);
    act.push_back({i, sd[i].m, sd[i].n, full, std::min(16, full)});
  }
  auto& h = rs_h;  // pinned, kept across clusters (grows, never shrinks)
  std::vector<double> skip;
  while (!act.empty()) {
    // one save + one draw per round: the sketches of every pending call,
    // back to back in call order (call t's run starts at off[t])
    std::vector<size_t> off(act.size() + 1, 0);
    for (size_t t = 0; t < act.size(); ++t) {
      const RsvdAct& a = act[t];
      off[t + 1] = off[t] + (size_t)a.n * std::min(a.k_try + 10, a.full);
    }
    src_op(1, 0);  // stream state at the start of the round
    if (h.capacity() < off.back()) h.reserve(std::max(off.back(), 2 * h.capacity()));
    h.resize(off.back());
    draw(h.data(), (long long)h.size());
    std::vector<int> stop = rsvd_round(sd, act, nullptr, &h);
    size_t t0 = 0;
    while (t0 < act.size() && stop[t0]) ++t0;
    if (t0 == act.size()) break;  // every call final; the stream sits after the last draw
    ++rsvd_redraws;
    if (t0 + 1 < act.size()) {
      // back to just after call t0's sketch: replay the round's stream up to there
      src_op(2, 0);
      skip.resize(off[t0 + 1]);
      draw(skip.data(), (long long)skip.size());
    }
    std::vector<RsvdAct> next;
    RsvdAct a = act[t0];
    a.k_try = std::min(2 * a.k_try, a.full);
    next.push_back(a);
    for (size_t t = t0 + 1; t < act.size(); ++t) next.push_back(act[t]);
    act.swap(next);
  }
}

// Waves of clusters of one level: Morton order, a cluster joins the first
// wave after every earlier cluster within Chebyshev distance 2.
//
// colored: the relaxed order of SURVEY 8e instead -- one wave per colour
// (x mod 3, y mod 3, z mod 3), colours in lexicographic order, Morton order
// inside a colour.  Same-colour clusters are at Chebyshev distance >= 3 (no
// shared neighbour), so a wave is still one batched stage, but the
// elimination order is no longer the reference's.
std::vector<std::vector<int>> cluster_waves(const Tree& T, int level, bool exact, bool colored) {
  const auto& ids = T.levels[level];
  std::vector<std::vector<int>> out;
  if (exact) {
    for (int c : ids) out.push_back({c});
    return out;
  }
  if (colored) {
    std::vector<std::vector<int>> by(27);
    for (int c : ids) {
      const long long x = T.cell[3 * c], y = T.cell[3 * c + 1], z = T.cell[3 * c + 2];
      by[(x % 3) * 9 + (y % 3) * 3 + (z % 3)].push_back(c);
    }
    for (auto& v : by)
      if (!v.empty()) out.push_back(std::move(v));
    return out;
  }
  std::unordered_map<uint64_t, int> wave_at;
  auto key = [](long long x, long long y, long long z) {
    return ((uint64_t)(x & 0x1fffff) << 42) | ((uint64_t)(y & 0x1fffff) << 21) |
           (uint64_t)(z & 0x1fffff);
  };
  for (int c : ids) {
    const long long x = T.cell[3 * c], y = T.cell[3 * c + 1], z = T.cell[3 * c + 2];
    int w = 0;
    for (int dx = -2; dx <= 2; ++dx)
      for (int dy = -2; dy <= 2; ++dy)
        for (int dz = -2; dz <= 2; ++dz) {
          if (x + dx < 0 || y + dy < 0 || z + dz < 0) continue;
          auto it = wave_at.find(key(x + dx, y + dy, z + dz));
          if (it != wave_at.end()) w = std::max(w, it->second);
        }
    wave_at[key(x, y, z)] = w + 1;
    if ((int)out.size() < w + 1) out.resize(w + 1);
    out[w].push_back(c);
  }
  return out;
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

Factor* factorize(Graph* gp, double eps, double sigma0, int flags, NormalSource src, void* src_user) {
  if (!(eps > 0.0 && eps < 1.0)) throw Error(E_VALUE, "epsilon must be in (0, 1)");
  IFMM_ASSERT(!gp->consumed, "graph already consumed by a factorization");
  Graph& g = *gp;
  Ctx& C = *g.ctx;
  Tree& T = *g.tree;
  auto t0 = std::chrono::steady_clock::now();
  Factor* F = new Factor;
  F->ctx = &C;
  F->bd = g.bd;
  F->n_points = g.bd * T.n_points;
  F->d_perm = T.d_perm;
  F->eps = eps;
  F->sigma0 = sigma0;
  F->init_sizes = g.size;
  F->n_clusters = T.nc;
  for (int c : T.leaves()) {
    F->leaf_nodes.push_back(g.nx[c]);
    F->leaf_start.push_back(g.bd * T.start[c]);
    F->leaf_stop.push_back(g.bd * T.stop[c]);
  }
  Eliminator el(C, g, *F, eps * sigma0, 0x1f2e3d4c5b6a7988ULL);
  el.exact_order = (flags & 1) != 0;
  el.exact_fill = (flags & 2) != 0 || getenv("IFMM_EXACT_FILL") != nullptr;
  el.src = src;
  el.src_user = src_user;
  // Morton cluster order (one cluster per wave): implied by the reference
  // stream, whose consumption order is the reference's cluster order
  const bool morton = el.exact_order || src != nullptr || (flags & 4) != 0;
  for (double& v : g_prof) v = 0.0;
  C.bucket_start(C.st);
  C.fail_fast = true;
  C.fail_prefix = "cluster ";
  try {
    for (int l = T.depth; l >= 2; --l) {
      LevelStats st;
      st.level = l;
      const double lr0 = C.bc.acc[2];
      int nwave = 0;
      for (auto& wave : cluster_waves(T, l, morton, !morton && (flags & 8) != 0))
      for (auto& wv : el.split_wave(wave)) {
        el.eliminate_wave(wv, st);
        if (symcheck_every() > 0 && ++nwave % symcheck_every() == 0) {
          char w[64];
          snprintf(w, sizeof w, "level %d after %d waves (cluster %d)", l, nwave, wv.back());
          symcheck(C, g, w);
        }
      }
      C.check_status("cluster ");
      C.bucket_collect();
      st.compress_time = C.bc.acc[2] - lr0;
      F->levels.push_back(st);
      if (symcheck_every() > 0) symcheck(C, g, "level end");
      if (l > 2) el.merge(l);
      if (symcheck_every() > 0 && l > 2) symcheck(C, g, "after merge");
      if (getenv("IFMM_MEMTRACE")) {
        fprintf(stderr, "[ifmm] level %d done: arena in use %.2f GB, peak %.2f GB, %.1f s\n", l,
                C.arena.in_use() / 1073741824.0, C.arena.peak() / 1073741824.0,
                std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
        if (C.ktime_on) {
          C.kt_collect();
          static const char* nm[] = {"gemm", "copy", "svd", "union", "lu", "lusolve", "spmv",
                                     "solve", "other"};
          fprintf(stderr, "[ifmm]   cumulative kernel s:");
          for (int i = 0; i < K_NCAT; ++i)
            if (C.kcount[i]) fprintf(stderr, " %s %.2f (%lld)", nm[i], C.ktime[i], C.kcount[i]);
          fprintf(stderr, "\n");
        }
      }
    }
    el.top();
    C.sync();
    C.check_status("cluster ");
  } catch (...) {
    C.fail_fast = false;
    C.bc.s = nullptr;
    g.consumed = true;
    delete F;
    throw;
  }
  C.fail_fast = false;
  C.bucket_stop();
  F->t_lu = C.bc.acc[0];
  F->t_mm = C.bc.acc[1];
  F->t_lr = C.bc.acc[2];
  F->t_tr = C.bc.acc[3];
  g.consumed = true;
  F->peak_edges = g.peak_edges;
  long long mb = 0;
  for (auto& w : g.su) mb = std::max<long long>(mb, w.p ? w.c : 0);
  F->max_basis_rank = mb;
  F->gemm_flops = el.flops_gemm;
  F->all_flops = el.flops_all;
  F->rsvd_rounds = el.rsvd_calls;
  F->rsvd_redraws = el.rsvd_redraws;
  C.free(el.d_ranks);
  std::vector<int> final_size = g.size;
  F->build_program(final_size);
  C.sync();
  F->t_total = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return F;
}

}  // namespace ifmm
