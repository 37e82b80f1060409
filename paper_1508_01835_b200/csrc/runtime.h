// Host runtime of the IFMM engine: device arena, descriptor staging,
// batched-launch helpers, error plumbing.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <map>
#include <unordered_map>
#include <set>
#include <stdexcept>
#include <string>
#include <vector>

#include "dense.h"
#include "h2_kernels.h"

namespace ifmm {

// ---- errors ------------------------------------------------------------
enum Status { OK = 0, E_VALUE = 1, E_SINGULAR = 2, E_CUDA = 3, E_OOM = 4, E_ASSERT = 5 };

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

void set_last_error(const std::string& s);

#define CUDA_CHECK(x)                                                                  \
  do {                                                                                 \
    cudaError_t _e = (x);                                                              \
    if (_e != cudaSuccess)                                                             \
      throw ::ifmm::Error(::ifmm::E_CUDA, std::string("CUDA error: ") +               \
                                              cudaGetErrorString(_e) + " at " __FILE__ ":" +      \
                                              std::to_string(__LINE__));                 \
  } while (0)

#define IFMM_ASSERT(c, msg)                                              \
  do {                                                                   \
    if (!(c)) throw ::ifmm::Error(::ifmm::E_ASSERT, std::string(msg)); \
  } while (0)

// ---- device arena: best-fit, coalescing free list over one cudaMalloc ----
// Blocks are multiples of 256 B; `cls` carries the length in 256-B units.
class Arena {
 public:
  void init(size_t bytes);
  void release();
  double* alloc(size_t ndoubles, int* cls);
  int* alloc_int(size_t n, int* cls) { return reinterpret_cast<int*>(alloc((n + 1) / 2, cls)); }
  void free(void* p, int cls);
  static constexpr int kExternCls = 0x7fffffff;
  size_t in_use() const { return in_use_; }
  size_t peak() const { return peak_; }
  size_t capacity() const { return cap_; }

 private:
  void insert_free(size_t off, size_t len);
  void backend_free(size_t off, size_t len);
  bool drain_cache();
  // exact-size cache in front of the best-fit backend: most edge blocks are
  // re-requested with the same shape, so reuse is an O(1) vector pop.  The
  // cache is drained back (with coalescing) only when the backend is full.
  std::map<size_t, std::vector<size_t>> cache_;  // ordered: a larger class can serve a miss
  size_t cached_ = 0;
  // large requests the fragmented slab cannot serve go to cudaMalloc
  std::unordered_map<void*, size_t> extern_;
  char* base_ = nullptr;
  size_t cap_ = 0, in_use_ = 0, peak_ = 0;
  std::map<size_t, size_t> by_addr_;              // offset -> length
  std::set<std::pair<size_t, size_t>> by_size_;   // (length, offset)
};

// Page-locked host allocator: host staging whose cudaMemcpyAsync is truly
// asynchronous (the buffer must outlive the copy: callers sync before reuse).
template <class T>
struct PinnedAlloc {
  using value_type = T;
  PinnedAlloc() = default;
  template <class U> PinnedAlloc(const PinnedAlloc<U>&) {}
  T* allocate(size_t n) {
    void* p = nullptr;
    if (cudaMallocHost(&p, n * sizeof(T)) != cudaSuccess) throw std::bad_alloc();
    return static_cast<T*>(p);
  }
  void deallocate(T* p, size_t) { cudaFreeHost(p); }
  template <class U> bool operator==(const PinnedAlloc<U>&) const { return true; }
  template <class U> bool operator!=(const PinnedAlloc<U>&) const { return false; }
};

// ---- dense block handle (row-major r x c, ld = c) ------------------------
struct Blk {
  double* p = nullptr;
  int r = 0, c = 0;
  int cls = -1;
  bool valid() const { return p != nullptr || (r * c == 0 && cls == -2); }
};

struct Ctx;

// ---- pinned-host -> device descriptor ring --------------------------------
class Staging {
 public:
  void init(size_t bytes);
  void release();
  // copy `bytes` from host memory into the ring; returns the device address
  void* push(Ctx& ctx, const void* src, size_t bytes);
  template <class T>
  T* push_vec(Ctx& ctx, const std::vector<T>& v) {
    return reinterpret_cast<T*>(push(ctx, v.data(), v.size() * sizeof(T)));
  }

 private:
  char* h_ = nullptr;
  char* d_ = nullptr;
  size_t cap_ = 0, off_ = 0;
};

struct Ctx {
  int device = 0;
  int n_sms = 0;       // SM count of `device` (sm_count())
  int mgs_occ = -1;    // cached occupancy of the cooperative MGS kernel on `device`
  int sm_count() {
    if (n_sms <= 0 && cudaDeviceGetAttribute(&n_sms, cudaDevAttrMultiProcessorCount, device) != cudaSuccess)
      n_sms = 148;
    return n_sms;
  }
  cudaStream_t st = nullptr;
  cudaStream_t st2 = nullptr;        // forked side stream (concurrent variants)
  cudaStream_t st3 = nullptr;        // side stream for a pair wave's rebases / K rewrite
  cudaEvent_t side_ev = nullptr, side_done = nullptr;
  cudaEvent_t fork_ev = nullptr, join_ev = nullptr;
  // run `a` on st and `b` on st2 concurrently; st waits for both afterwards
  template <class FA, class FB>
  void fork2(FA a, FB b) {
    CUDA_CHECK(cudaEventRecord(fork_ev, st));
    CUDA_CHECK(cudaStreamWaitEvent(st2, fork_ev, 0));
    a(st);
    b(st2);
    CUDA_CHECK(cudaEventRecord(join_ev, st2));
    CUDA_CHECK(cudaStreamWaitEvent(st, join_ev, 0));
  }
  Arena arena;
  Staging stage;
  int* d_status = nullptr;   // singular-pivot flag (tag+1)
  int* h_pinned_i = nullptr; // small pinned readback buffer
  size_t h_pinned_n = 0;
  long long launches = 0;
  cudaEvent_t ev[64] = {};
  // per-category kernel timing (IFMM_KTIME=1 or ktime_on): event pairs
  bool ktime_on = false;
  struct KRec { int cat; cudaEvent_t a, b; double work; };
  std::vector<KRec> krec;
  std::vector<cudaEvent_t> kpool;
  double ktime[16] = {}, kwork[16] = {};
  long long kcount[16] = {};
  void kt_begin(int cat, double work, cudaEvent_t* a) {
    if (!ktime_on) return;
    if (kpool.size() < 2) for (int i = 0; i < 256; ++i) { cudaEvent_t e; cudaEventCreate(&e); kpool.push_back(e); }
    *a = kpool.back(); kpool.pop_back();
    cudaEventRecord(*a, st);
    (void)cat; (void)work;
  }
  void kt_end(int cat, double work, cudaEvent_t a) {
    if (!ktime_on) return;
    cudaEvent_t b = kpool.back(); kpool.pop_back();
    cudaEventRecord(b, st);
    krec.push_back({cat, a, b, work});
    if (krec.size() > 4096) kt_collect();
  }
  void kt_collect() {
    if (krec.empty()) return;
    cudaStreamSynchronize(st);
    for (auto& k : krec) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, k.a, k.b);
      ktime[k.cat] += ms * 1e-3;
      kwork[k.cat] += k.work;
      kcount[k.cat]++;
      kpool.push_back(k.a);
      kpool.push_back(k.b);
    }
    krec.clear();
  }

  // Device time of the reference's timing buckets (factor.py:71-72:
  // lu_and_triangular_solves, matmul_updates, lowrank_approximations,
  // operator_transfer): one event on the engine stream per bucket switch;
  // the time between consecutive marks goes to the bucket active in between.
  struct BucketClock {
    cudaStream_t s = nullptr;
    std::vector<cudaEvent_t> pool;
    std::vector<std::pair<int, cudaEvent_t>> marks;
    double acc[4] = {};
  } bc;
  void bucket(int b) {
    if (!bc.s) return;
    if (!bc.marks.empty() && bc.marks.back().first == b) return;
    cudaEvent_t e;
    if (bc.pool.empty()) CUDA_CHECK(cudaEventCreate(&e));
    else { e = bc.pool.back(); bc.pool.pop_back(); }
    CUDA_CHECK(cudaEventRecord(e, bc.s));
    bc.marks.push_back({b, e});
  }
  void bucket_collect() {  // reaps every completed interval
    size_t i = 0;
    for (; i + 1 < bc.marks.size(); ++i) {
      if (cudaEventQuery(bc.marks[i + 1].second) != cudaSuccess) { cudaGetLastError(); break; }
      float ms = 0.f;
      if (cudaEventElapsedTime(&ms, bc.marks[i].second, bc.marks[i + 1].second) == cudaSuccess &&
          bc.marks[i].first >= 0 && bc.marks[i].first < 4)
        bc.acc[bc.marks[i].first] += ms * 1e-3;
      cudaGetLastError();
      bc.pool.push_back(bc.marks[i].second);
    }
    bc.marks.erase(bc.marks.begin(), bc.marks.begin() + i);
  }
  void bucket_start(cudaStream_t s) {
    for (auto& m : bc.marks) bc.pool.push_back(m.second);
    bc.marks.clear();
    for (double& a : bc.acc) a = 0.0;
    bc.s = s;
  }
  void bucket_stop() {  // after a sync of bc.s
    bucket(-1);
    CUDA_CHECK(cudaStreamSynchronize(bc.s));
    bucket_collect();
    for (auto& m : bc.marks) bc.pool.push_back(m.second);
    bc.marks.clear();
    bc.s = nullptr;
  }

  Blk alloc(int r, int c) {
    Blk b;
    b.r = r;
    b.c = c;
    size_t n = (size_t)r * c;
    b.p = arena.alloc(n ? n : 1, &b.cls);
    return b;
  }
  // Frees are deferred: a block released while a batch that references it
  // is still being built must not be handed out again before that batch is
  // enqueued.  flush() returns them to the arena at points where no batch
  // is under construction (stream order then protects in-flight readers).
  std::vector<std::pair<void*, int>> pending;
  void free(Blk& b) {
    if (b.p && b.cls >= 0) pending.emplace_back(b.p, b.cls);
    b.p = nullptr;
    b.cls = -1;
  }
  void free_raw(void* p, int cls) {
    if (p && cls >= 0) pending.emplace_back(p, cls);
  }
  void flush() {
    for (auto& q : pending) arena.free(q.first, q.second);
    pending.clear();
  }
  void sync() { CUDA_CHECK(cudaStreamSynchronize(st)); }
  // destructors / destroy entry points must not throw
  void sync_nothrow() { if (cudaStreamSynchronize(st) != cudaSuccess) cudaGetLastError(); }
  // while set, every readback also checks the singular-pivot flag
  bool fail_fast = false;
  const char* fail_prefix = "cluster ";
  // read back n ints from device (synchronizes)
  const int* readback_ints(const int* d, size_t n);
  void check_status(const char* what_prefix);
};

// ---- batched launch builders ---------------------------------------------
enum KCat { K_GEMM = 0, K_COPY, K_SVD, K_UNION, K_LU, K_LUSOLVE, K_SPMV, K_SOLVE, K_OTHER, K_NCAT };

struct GemmBatch {
  std::vector<GemmDesc> d;
  double flops = 0.0;
  void add(const double* A, int lda, int ta, const double* B, int ldb, int tb, double* C,
           int ldc, int M, int N, int K, double alpha, double beta,
           const double* dscale = nullptr) {
    if (M <= 0 || N <= 0) return;
    GemmDesc g;
    g.A = A; g.B = B; g.C = C; g.dscale = dscale;
    g.M = M; g.N = N; g.K = K; g.lda = lda; g.ldb = ldb; g.ldc = ldc;
    g.ta = ta; g.tb = tb; g.alpha = alpha; g.beta = beta;
    d.push_back(g);
    flops += 2.0 * M * N * (double)K;
  }
  void run(Ctx& ctx);
  bool empty() const { return d.empty(); }
};

struct CopyBatch {
  std::vector<CopyDesc> d;
  void add(const double* src, int ss_r, int ss_c, double* dst, int ds_r, int ds_c, int rows,
           int cols, int mode, double alpha = 1.0, const double* rscale = nullptr) {
    if (rows <= 0 || cols <= 0) return;
    CopyDesc c;
    c.src = src; c.dst = dst; c.rows = rows; c.cols = cols;
    c.ss_r = ss_r; c.ss_c = ss_c; c.ds_r = ds_r; c.ds_c = ds_c;
    c.mode = mode; c.alpha = alpha; c.rscale = rscale;
    d.push_back(c);
  }
  // convenience: row-major blocks
  void copy(const Blk& s, Blk& t, int r0 = 0, int c0 = 0) {
    add(s.p, s.c, 1, t.p + (size_t)r0 * t.c + c0, t.c, 1, s.r, s.c, 0);
  }
  void zero(Blk& t) { add(nullptr, 0, 0, t.p, t.c, 1, t.r, t.c, 3); }
  void eye(Blk& t, double a) { add(nullptr, 0, 0, t.p, t.c, 1, t.r, t.c, 2, a); }
  void run(Ctx& ctx);
  bool empty() const { return d.empty(); }
};

}  // namespace ifmm
