// Host runtime: arena allocator, descriptor staging ring, batched launches.
#include "runtime.h"

#include <algorithm>
#include <cstdio>

namespace ifmm {

static thread_local std::string g_last_error;
void set_last_error(const std::string& s) { g_last_error = s; }
const char* last_error_cstr() { return g_last_error.c_str(); }

// ---------------------------------------------------------------------------
// Arena: classes of 256 B up to 4 KiB, then geometric with 8 steps / octave.
// Frees go to per-class free lists; reuse is safe because every kernel runs
// on the one context stream (a freed block is only handed to work enqueued
// after the last reader).
// ---------------------------------------------------------------------------
static std::vector<size_t>& class_table() {
  static std::vector<size_t> t;
  if (t.empty()) {
    size_t s = 256;
    while (s < (size_t)1 << 41) {
      t.push_back(s);
      size_t nx = s + 256;
      if (s >= 4096) {
        size_t g = s / 8;
        g = (g + 255) / 256 * 256;
        nx = s + g;
      }
      s = nx;
    }
  }
  return t;
}

int Arena::class_of(size_t bytes) {
  auto& t = class_table();
  auto it = std::lower_bound(t.begin(), t.end(), bytes);
  return (int)(it - t.begin());
}
size_t Arena::class_bytes(int cls) { return class_table()[cls]; }

void Arena::init(size_t bytes) {
  bytes = bytes / 4096 * 4096;
  CUDA_CHECK(cudaMalloc(&base_, bytes));
  cap_ = bytes;
  top_ = in_use_ = peak_ = 0;
  bins_.assign(class_table().size(), {});
}

void Arena::release() {
  if (base_) cudaFree(base_);
  base_ = nullptr;
  cap_ = top_ = 0;
  bins_.clear();
}

double* Arena::alloc(size_t ndoubles, int* cls) {
  const size_t bytes = ndoubles * sizeof(double);
  const int c = class_of(bytes);
  const size_t cb = class_bytes(c);
  char* p;
  if (!bins_[c].empty()) {
    p = bins_[c].back();
    bins_[c].pop_back();
  } else {
    if (top_ + cb > cap_) {
      char msg[160];
      snprintf(msg, sizeof msg, "device arena exhausted: need %zu B, %zu of %zu B used", cb,
               in_use_, cap_);
      throw Error(E_OOM, msg);
    }
    p = base_ + top_;
    top_ += cb;
  }
  in_use_ += cb;
  peak_ = std::max(peak_, in_use_);
  *cls = c;
  return reinterpret_cast<double*>(p);
}

void Arena::free(void* p, int cls) {
  if (!p || cls < 0) return;
  bins_[cls].push_back(reinterpret_cast<char*>(p));
  in_use_ -= class_bytes(cls);
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
    // ring wrap: all earlier copies/kernels reading the ring must be done
    ctx.sync();
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
  if (n > h_pinned_n) {
    if (h_pinned_i) cudaFreeHost(h_pinned_i);
    h_pinned_n = std::max<size_t>(n, 1 << 16);
    CUDA_CHECK(cudaMallocHost(&h_pinned_i, h_pinned_n * sizeof(int)));
  }
  if (n) CUDA_CHECK(cudaMemcpyAsync(h_pinned_i, d, n * sizeof(int), cudaMemcpyDeviceToHost, st));
  sync();
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

void GemmBatch::run(Ctx& ctx) {
  if (d.empty()) return;
  std::vector<int> ts(d.size() + 1);
  int tot = 0;
  for (size_t i = 0; i < d.size(); ++i) {
    ts[i] = tot;
    tot += ((d[i].M + 63) / 64) * ((d[i].N + 63) / 64);
  }
  ts[d.size()] = tot;
  GemmDesc* dd = ctx.stage.push_vec(ctx, d);
  int* dt = ctx.stage.push_vec(ctx, ts);
  launch_gemm(dd, dt, (int)d.size(), tot, ctx.st);
  ctx.launches++;
  CUDA_CHECK(cudaGetLastError());
  d.clear();
}

void CopyBatch::run(Ctx& ctx) {
  if (d.empty()) return;
  CopyDesc* dd = ctx.stage.push_vec(ctx, d);
  launch_copy(dd, (int)d.size(), ctx.st);
  ctx.launches++;
  CUDA_CHECK(cudaGetLastError());
  d.clear();
}

}  // namespace ifmm
