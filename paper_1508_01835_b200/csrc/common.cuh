// Shared device helpers for the IFMM B200 engine (sm_100a, fp64).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <cmath>
#include <cstdio>
#include <cstdlib>

#define IFMM_DEV __device__ __forceinline__

namespace ifmm {

// IFMM_DEBUG_SYNC=1: synchronise after every batched launch and abort with the
// launcher's name on a device fault (diagnostics only).
inline bool dbg_sync_on() {
  static int on = -1;
  if (on < 0) { const char* e = getenv("IFMM_DEBUG_SYNC"); on = e && atoi(e) ? 1 : 0; }
  return on == 1;
}
struct DbgSync {
  cudaStream_t s;
  const char* name;
  ~DbgSync() {
    if (!dbg_sync_on()) return;
    const cudaError_t e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) {
      fprintf(stderr, "[ifmm] device fault after %s: %s\n", name, cudaGetErrorString(e));
      abort();
    }
  }
};

constexpr double kEps = 2.220446049250313e-16;

// --- warp / block reductions ------------------------------------------------

IFMM_DEV double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

IFMM_DEV double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// argmax of |value| with ties -> smallest index (numpy/idamax semantics).
IFMM_DEV void warp_argmax(double& v, long long& idx) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    double ov = __shfl_xor_sync(0xffffffffu, v, o);
    long long oi = __shfl_xor_sync(0xffffffffu, idx, o);
    if (ov > v || (ov == v && oi < idx)) { v = ov; idx = oi; }
  }
}

// Block-wide sum; `red` must hold >= 32 doubles of shared scratch.
// All threads receive the result.
IFMM_DEV double block_sum(double v, double* red) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int nw = (blockDim.x + 31) >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  double t = (lane < nw) ? red[lane] : 0.0;
  t = warp_sum(t);
  return t;
}

// Block-wide argmax (value >= 0 expected, ties -> smallest idx).
IFMM_DEV void block_argmax(double& v, long long& idx, double* redv, long long* redi) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int nw = (blockDim.x + 31) >> 5;
  warp_argmax(v, idx);
  __syncthreads();
  if (lane == 0) { redv[w] = v; redi[w] = idx; }
  __syncthreads();
  double tv = (lane < nw) ? redv[lane] : -1.0;
  long long ti = (lane < nw) ? redi[lane] : (1LL << 62);
  warp_argmax(tv, ti);
  v = tv; idx = ti;
}

// --- FP64 tensor-core MMA (DMMA.8x8x4 on sm_100a) ------------------------------
// A fragment: row-major 8x4, lane holds A[lane>>2][lane&3]
// B fragment: col 4x8,        lane holds B[lane&3][lane>>2]
// C fragment: 8x8,            lane holds C[lane>>2][2*(lane&3) + {0,1}]
IFMM_DEV void dmma_8x8x4(double& c0, double& c1, double a, double b) {
  asm volatile(
      "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}

}  // namespace ifmm
