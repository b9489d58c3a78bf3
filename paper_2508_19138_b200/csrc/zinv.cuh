// Batched complex-FP64 inversion with partial pivoting (see zinv.cu).
#pragma once
#include "common.cuh"

namespace negf {

constexpr int kInvSmallMax = 64;

// Per-call error/conditioning reporting. status[b] is set (first writer wins)
// to status_code when matrix b hits an exactly-zero or non-finite pivot;
// u_spread[b * spread_stride] receives max|U_jj| / min|U_jj|.
struct InvAux {
  int* status;
  int status_code;
  double* u_spread;
  long long spread_stride;
  const int* active;  // optional per-batch mask (skip matrices with active[b]==0)
};

int zinv_panel_width(int n, int batch);
size_t zinv_workspace_bytes(int n, int batch);
// S is destroyed for n > 64. X must not alias S.
int zinv_batched(z_t* S, long long sS, int lds, z_t* X, long long sX, int ldx, int n, int batch,
                 InvAux aux, void* ws, size_t ws_bytes, cudaStream_t stream);

}  // namespace negf
