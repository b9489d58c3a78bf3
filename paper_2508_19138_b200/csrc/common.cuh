// Shared device helpers for the NEGF+GW hot path (sm_100a, complex FP64).
//
// Every matrix-valued quantity is complex128 stored interleaved (re, im) as
// double2, row-major, one dense N_BS x N_BS block per (energy, block index).
// This is the in-HBM layout of torch.complex128 tensors of shape
// (n_e, n_blocks, bs, bs), so the Python side hands raw pointers straight in.
#pragma once

#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

namespace negf {

using z_t = double2;

enum Op : int { OP_N = 0, OP_T = 1, OP_C = 2, OP_H = 3 };

__host__ __device__ inline bool op_trans(int op) { return op == OP_T || op == OP_H; }
__host__ __device__ inline bool op_conj(int op) { return op == OP_C || op == OP_H; }

__device__ __forceinline__ z_t zmake(double r, double i) { return make_double2(r, i); }
__device__ __forceinline__ z_t zadd(z_t a, z_t b) { return zmake(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ z_t zsub(z_t a, z_t b) { return zmake(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ z_t zmul(z_t a, z_t b) {
  return zmake(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ z_t zconj(z_t a) { return zmake(a.x, -a.y); }
// c + a*b and c - a*b as four FMAs (zadd(c, zmul(a, b)) compiles to six FP64 ops)
__device__ __forceinline__ z_t zfma(z_t a, z_t b, z_t c) {
  return zmake(fma(-a.y, b.y, fma(a.x, b.x, c.x)), fma(a.y, b.x, fma(a.x, b.y, c.y)));
}
__device__ __forceinline__ z_t zfms(z_t a, z_t b, z_t c) {
  return zmake(fma(a.y, b.y, fma(-a.x, b.x, c.x)), fma(-a.y, b.x, fma(-a.x, b.y, c.y)));
}
__device__ __forceinline__ z_t zscale(double s, z_t a) { return zmake(s * a.x, s * a.y); }
// 1/a = conj(a) / |a|^2 with a single division (pivots here are far from the
// overflow range where LAPACK's scaled zladiv matters).
__device__ __forceinline__ z_t zinv(z_t a) {
  const double s = 1.0 / (a.x * a.x + a.y * a.y);
  return zmake(a.x * s, -a.y * s);
}
__device__ __forceinline__ double zabs1(z_t a) { return fabs(a.x) + fabs(a.y); }

// Flip the sign bit of a double with an integer op (keeps the FP64 pipe free).
__device__ __forceinline__ double dneg_if(double x, unsigned long long mask) {
  return __longlong_as_double(__double_as_longlong(x) ^ (long long)mask);
}

__device__ __forceinline__ void dmma_m8n8k4(double& c0, double& c1, double a, double b) {
  asm(
      "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}

// Ordered variants (volatile asm keeps their program order relative to each
// other): for software-pipelined DMMA loops.
__device__ __forceinline__ void dmma_v(double& c0, double& c1, double a, double b) {
  asm volatile(
      "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool pred) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  int n = pred ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(n));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

}  // namespace negf

namespace negf {
// Process-wide count of kernels launched by this library (bench.py's
// gpu_launches evidence); relaxed atomic increment per launch.
void count_launch();
}  // namespace negf

#define NEGF_LAUNCHED()                     \
  do {                                      \
    negf::count_launch();                   \
    NEGF_CUDA_CHECK(cudaGetLastError());    \
  } while (0)

#define NEGF_CUDA_CHECK(expr)                                                        \
  do {                                                                               \
    cudaError_t _e = (expr);                                                         \
    if (_e != cudaSuccess) {                                                         \
      fprintf(stderr, "negf_b200: CUDA error %s at %s:%d\n", cudaGetErrorString(_e), \
              __FILE__, __LINE__);                                                   \
      return (int)_e;                                                                \
    }                                                                                \
  } while (0)
