// Host runtime: arena allocator, descriptor staging ring, batched launches.
#include "runtime.h"

#include <algorithm>
#include <cstdio>

namespace ifmm {

static thread_local std::string g_last_error;
void set_last_error(const std::string& s) { g_last_error = s; }
const char* last_error_cstr() { return g_last_error.c_str(); }

// ---------------------------------------------------------------------------
// Arena: best-fit with coalescing.  Reuse is safe because every kernel runs
// on the one context stream and frees are deferred (Ctx::free/flush).
// ---------------------------------------------------------------------------
void Arena::init(size_t bytes) {
  bytes = bytes / 4096 * 4096;
  CUDA_CHECK(cudaMalloc(&base_, bytes));
  cap_ = bytes;
  in_use_ = peak_ = 0;
  by_addr_.clear();
  by_size_.clear();
  insert_free(0, bytes);
}

void Arena::release() {
  for (auto& kv : extern_) cudaFree(kv.first);
  extern_.clear();
  if (base_) cudaFree(base_);
  base_ = nullptr;
  cap_ = 0;
  by_addr_.clear();
  by_size_.clear();
}

void Arena::insert_free(size_t off, size_t len) {
  by_addr_[off] = len;
  by_size_.insert({len, off});
}

bool Arena::drain_cache() {
  if (cached_ == 0) return false;
  for (auto& kv : cache_)
    for (size_t off : kv.second) backend_free(off, kv.first);
  cache_.clear();
  cached_ = 0;
  return true;
}

// size classes: 256-B steps up to 4 KiB, then 8 classes per octave
static size_t class_round(size_t bytes) {
  if (bytes <= 4096) return (bytes + 255) / 256 * 256;
  int e = 63 - __builtin_clzll(bytes - 1);      // 2^e < bytes <= 2^(e+1)
  const size_t step = (size_t)1 << (e - 3);      // 1/8 octave
  return (bytes + step - 1) / step * step;
}

double* Arena::alloc(size_t ndoubles, int* cls) {
  size_t bytes = ndoubles * sizeof(double);
  if (bytes == 0) bytes = 256;
  bytes = class_round(bytes);
  *cls = (int)(bytes / 256);
  auto ci = cache_.find(bytes);
  if (ci != cache_.end() && !ci->second.empty()) {
    const size_t off = ci->second.back();
    ci->second.pop_back();
    cached_ -= bytes;
    in_use_ += bytes;
    peak_ = std::max(peak_, in_use_);
    return reinterpret_cast<double*>(base_ + off);
  }
  if (bytes >= ((size_t)256 << 20)) {
    // very large (top-level LU, solve workspace): dedicated cudaMalloc, so a
    // fragmented slab can never block them (bench leaves headroom for this)
    void* p = nullptr;
    if (cudaMalloc(&p, bytes) == cudaSuccess) {
      extern_[p] = bytes;
      in_use_ += bytes;
      peak_ = std::max(peak_, in_use_);
      *cls = kExternCls;
      return reinterpret_cast<double*>(p);
    }
    cudaGetLastError();
  }
  if (bytes >= ((size_t)8 << 20)) {
    // large: carved from the END of a free block near the top of the slab
    // (keeps large and small blocks apart).  The walk from the top is bounded
    // -- after a cache drain the free list can hold millions of small blocks,
    // and an unbounded first-fit scan per large request made a c4 step 1.6x
    // slower from the second factorization on -- then best fit by size.
    for (int attempt = 0; attempt < 2; ++attempt) {
      size_t boff = 0, blen = 0;
      int seen = 0;
      for (auto rit = by_addr_.rbegin(); rit != by_addr_.rend() && seen < 64; ++rit, ++seen)
        if (rit->second >= bytes) { boff = rit->first; blen = rit->second; break; }
      if (!blen) {
        auto bi = by_size_.lower_bound({bytes, 0});
        if (bi != by_size_.end()) { blen = bi->first; boff = bi->second; }
      }
      if (blen) {
        by_size_.erase({blen, boff});
        by_addr_.erase(boff);
        if (blen > bytes) insert_free(boff, blen - bytes);
        in_use_ += bytes;
        peak_ = std::max(peak_, in_use_);
        return reinterpret_cast<double*>(base_ + boff + blen - bytes);
      }
      if (!drain_cache()) break;
    }
    void* p = nullptr;
    if (cudaMalloc(&p, bytes) == cudaSuccess) {
      extern_[p] = bytes;
      in_use_ += bytes;
      peak_ = std::max(peak_, in_use_);
      *cls = kExternCls;
      return reinterpret_cast<double*>(p);
    }
    cudaGetLastError();
    char msg[200];
    snprintf(msg, sizeof msg, "device arena exhausted: need %zu B, %zu of %zu B in use", bytes,
             in_use_, cap_);
    throw Error(E_OOM, msg);
  }
  auto it = by_size_.lower_bound({bytes, 0});
  if (it == by_size_.end()) {
    // no coalesced block fits: split a cached block of the next larger class
    // before paying for a full drain (which coalesces every cached block)
    for (auto cj = cache_.upper_bound(bytes); cj != cache_.end(); ++cj) {
      if (cj->second.empty()) continue;
      const size_t len = cj->first, off = cj->second.back();
      cj->second.pop_back();
      cached_ -= len;
      insert_free(off + bytes, len - bytes);
      in_use_ += bytes;
      peak_ = std::max(peak_, in_use_);
      return reinterpret_cast<double*>(base_ + off);
    }
    if (drain_cache()) it = by_size_.lower_bound({bytes, 0});
  }
  if (it == by_size_.end()) {
    void* p = nullptr;
    if (cudaMalloc(&p, bytes) == cudaSuccess) {
      extern_[p] = bytes;
      in_use_ += bytes;
      peak_ = std::max(peak_, in_use_);
      *cls = kExternCls;
      return reinterpret_cast<double*>(p);
    }
    cudaGetLastError();
    char msg[200];
    snprintf(msg, sizeof msg, "device arena exhausted: need %zu B, %zu of %zu B in use", bytes,
             in_use_, cap_);
    throw Error(E_OOM, msg);
  }
  const size_t len = it->first, off = it->second;
  by_size_.erase(it);
  by_addr_.erase(off);
  if (len > bytes) insert_free(off + bytes, len - bytes);
  in_use_ += bytes;
  peak_ = std::max(peak_, in_use_);
  *cls = (int)(bytes / 256);
  return reinterpret_cast<double*>(base_ + off);
}

void Arena::free(void* p, int cls) {
  if (!p || cls <= 0) return;
  if (cls == kExternCls) {
    auto it = extern_.find(p);
    if (it != extern_.end()) {
      in_use_ -= it->second;
      cudaFree(p);  // implicitly synchronises: no in-flight reader remains
      extern_.erase(it);
    }
    return;
  }
  const size_t off = (size_t)(reinterpret_cast<char*>(p) - base_);
  const size_t len = (size_t)cls * 256;
  in_use_ -= len;
  if (len <= ((size_t)1 << 20)) {  // cache blocks up to 1 MiB
    cache_[len].push_back(off);
    cached_ += len;
    return;
  }
  backend_free(off, len);
}

void Arena::backend_free(size_t off, size_t len) {
  auto nx = by_addr_.lower_bound(off);
  if (nx != by_addr_.end() && nx->first == off + len) {  // merge with next
    len += nx->second;
    by_size_.erase({nx->second, nx->first});
    nx = by_addr_.erase(nx);
  }
  if (nx != by_addr_.begin()) {
    auto pv = std::prev(nx);
    if (pv->first + pv->second == off) {  // merge with previous
      off = pv->first;
      len += pv->second;
      by_size_.erase({pv->second, pv->first});
      by_addr_.erase(pv);
    }
  }
  insert_free(off, len);
}

// ---------------------------------------------------------------------------
void Staging::init(size_t bytes) {
  cap_ = bytes;
  CUDA_CHECK(cudaMallocHost(&h_, bytes));
  CUDA_CHECK(cudaMalloc(&d_, bytes));
  off_ = 0;
}

void Staging::release() {
  if (h_) cudaFreeHost(h_);
  if (d_) cudaFree(d_);
  h_ = d_ = nullptr;
}

void* Staging::push(Ctx& ctx, const void* src, size_t bytes) {
  const size_t nb = (bytes + 255) / 256 * 256;
  if (nb > cap_) throw Error(E_OOM, "descriptor batch larger than staging ring");
  if (off_ + nb > cap_) {
    // ring wrap: all earlier copies/kernels reading the ring must be done,
    // on every stream that takes descriptors (engine, forked, side)
    CUDA_CHECK(cudaDeviceSynchronize());
    off_ = 0;
  }
  std::memcpy(h_ + off_, src, bytes);
  CUDA_CHECK(cudaMemcpyAsync(d_ + off_, h_ + off_, bytes, cudaMemcpyHostToDevice, ctx.st));
  void* r = d_ + off_;
  off_ += nb;
  return r;
}

// ---------------------------------------------------------------------------
const int* Ctx::readback_ints(const int* d, size_t n) {
  if (n + 1 > h_pinned_n) {
    if (h_pinned_i) cudaFreeHost(h_pinned_i);
    h_pinned_n = std::max<size_t>(n + 1, 1 << 16);
    CUDA_CHECK(cudaMallocHost(&h_pinned_i, h_pinned_n * sizeof(int)));
  }
  if (n) CUDA_CHECK(cudaMemcpyAsync(h_pinned_i, d, n * sizeof(int), cudaMemcpyDeviceToHost, st));
  // the singular-pivot flag rides along with every readback: a failed LU
  // stops the factorization at the first sync after it (the reference raises
  // at the failing cluster, factor.py:166-173) instead of carrying NaNs on
  if (fail_fast && d != d_status)
    CUDA_CHECK(cudaMemcpyAsync(h_pinned_i + h_pinned_n - 1, d_status, sizeof(int),
                               cudaMemcpyDeviceToHost, st));
  sync();
  if (bc.s) bucket_collect();
  if (fail_fast && d != d_status && h_pinned_i[h_pinned_n - 1] != 0) check_status(fail_prefix);
  return h_pinned_i;
}

void Ctx::check_status(const char* what_prefix) {
  const int* s = readback_ints(d_status, 1);
  if (s[0] != 0) {
    const int tag = s[0] - 1;
    CUDA_CHECK(cudaMemsetAsync(d_status, 0, sizeof(int), st));
    std::string what = tag == 0x7fffffff - 1 ? std::string("top-level system")
                                              : std::string(what_prefix) + std::to_string(tag);
    throw Error(E_SINGULAR, what);
  }
}

static constexpr size_t kMaxBatch = (size_t)1 << 19;  // descriptors per launch

void GemmBatch::run(Ctx& ctx) {
  if (d.empty()) return;
  // One tile shape for every problem: the 64 x 64 cp.async kernel at 3 CTAs per
  // SM measured equal to or faster than a 128 x 128 variant at every size
  // (27.7 vs 27.4 TF/s at 4096^3, 16.7 vs 9.4 at 280 x 7000 x 280;
  // profiles/r02_gemm_ncu.md), so the large-tile path was removed.
  int bm = 64, bn = 64;
  gemm_tile_dims(&bm, &bn);
  for (size_t c0 = 0; c0 < d.size(); c0 += kMaxBatch) {
    const size_t c1 = std::min(d.size(), c0 + kMaxBatch);
    const GemmDesc* part = d.data() + c0;
    const size_t np = c1 - c0;
    std::vector<int> ts(np + 1);
    long long tot = 0;
    double fl = 0;
    for (size_t i = 0; i < np; ++i) {
      ts[i] = (int)tot;
      tot += (long long)((part[i].M + bm - 1) / bm) * ((part[i].N + bn - 1) / bn);
      fl += 2.0 * part[i].M * part[i].N * (double)part[i].K;
    }
    IFMM_ASSERT(tot < (1LL << 31), "GEMM batch tile count overflow");
    ts[np] = (int)tot;
    GemmDesc* dd = reinterpret_cast<GemmDesc*>(ctx.stage.push(ctx, part, np * sizeof(GemmDesc)));
    int* dt = ctx.stage.push_vec(ctx, ts);
    cudaEvent_t ka = nullptr;
    ctx.kt_begin(K_GEMM, fl, &ka);
    launch_gemm(dd, dt, (int)np, (int)tot, ctx.st);
    ctx.kt_end(K_GEMM, fl, ka);
    ctx.launches++;
    CUDA_CHECK(cudaGetLastError());
  }
  d.clear();
}

void CopyBatch::run(Ctx& ctx) {
  if (d.empty()) return;
  for (size_t c0 = 0; c0 < d.size(); c0 += kMaxBatch) {
    const size_t c1 = std::min(d.size(), c0 + kMaxBatch);
    std::vector<CopyDesc> part(d.begin() + c0, d.begin() + c1);
    CopyDesc* dd = ctx.stage.push_vec(ctx, part);
    double bytes = 0;
    for (auto& x : part) bytes += 16.0 * x.rows * x.cols;
    cudaEvent_t ka = nullptr;
    ctx.kt_begin(K_COPY, bytes, &ka);
    launch_copy(dd, (int)part.size(), ctx.st);
    ctx.kt_end(K_COPY, bytes, ka);
    ctx.launches++;
    CUDA_CHECK(cudaGetLastError());
  }
  d.clear();
}

}  // namespace ifmm
