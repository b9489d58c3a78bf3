// Opt-in per-launch CUDA-event profiler for the dominant kernel classes
// (bench.py's live roofline). Off by default; process-global when enabled.
#pragma once
#include "common.cuh"

namespace negf {

bool prof_enabled();
// Returns a token; call prof_end with it after the launch(es).
int prof_begin(int cls, cudaStream_t st);
void prof_end(int token, cudaStream_t st, double flops, double bytes);

enum ProfClass : int {
  PROF_ZGEMM = 0,        // DMMA GEMM launches with K > 32
  PROF_ZINV = 1,         // inversion panel / swap / rows / unpermute kernels
  PROF_EW = 2,
  PROF_OTHER = 3,
  PROF_ZGEMM_SMALLK = 4, // DMMA GEMM launches with K <= 32 (inversion sweeps)
  PROF_NCLASS = 5,
  PROF_CONV = 9,         // fused P / Sigma FFT convolution kernels (algorithmic HBM bytes recorded)
  PROF_LAYOUT = 10       // E<->nnz pack / unpack kernels (algorithmic HBM bytes recorded)
};

// RAII span recording algorithmic flops/bytes for its launches.
struct ProfSpan {
  int tok;
  cudaStream_t st;
  double flops, bytes;
  ProfSpan(int cls, cudaStream_t s, double f, double b) : tok(prof_begin(cls, s)), st(s), flops(f), bytes(b) {}
  ~ProfSpan() { prof_end(tok, st, flops, bytes); }
};



}  // namespace negf

namespace negf {
// RAII span: CUDA events around the launches made while it is alive.
struct ProfScope {
  int tok;
  cudaStream_t st;
  ProfScope(int cls, cudaStream_t s) : tok(prof_begin(cls, s)), st(s) {}
  ~ProfScope() { prof_end(tok, st, 0.0, 0.0); }
};
}  // namespace negf
