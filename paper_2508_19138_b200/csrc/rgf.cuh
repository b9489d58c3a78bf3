// Batched-over-energy RGF selected solve (host orchestration of the DMMA
// GEMM, pivoted inversion and elementwise kernels). See rgf.cu.
#pragma once
#include "common.cuh"

namespace negf {

// One batch of block-tridiagonal systems, all complex128 device pointers,
// energy-major packed: diag [n_e][n_b][bs][bs], off [n_e][n_b-1][bs][bs].
struct RgfArgs {
  int n_e, n_b, bs;
  const z_t* m_diag;
  const z_t* m_upper;
  const z_t* m_lower;
  const z_t* b_diag[2];   // lesser, greater (nullptr: kind absent)
  const z_t* b_upper[2];  // lg-compressed: B[i+1][i] = -B[i][i+1]^dag
  z_t* xr_diag;
  z_t* xr_upper;
  z_t* xr_lower;
  z_t* xl_diag[2];
  z_t* xl_upper[2];
  int symmetrize;      // bit 0: apply (X - X^dag)/2 to the lesser/greater diagonal blocks;
                       // bit 1: the B^lg diagonal blocks are anti-Hermitian (every lg source of
                       // the solver is), so anti-Hermitian forward products run on half the tiles
  int* status;         // [n_e] device: 0 ok, 1 + forward step of the first singular block
  double* u_spread;    // [n_e][n_b] device, optional
  int overlap;         // forward sweep: Keldysh products on a second stream (default 1)
  // 0: forward + backward (selected_solve). 1: forward only -- x_fwd lands in
  // xr_diag, xl_fwd in xl_diag (forward_retarded / forward_lg, rgf.py:113-149).
  // 2: backward only -- xr_diag / xl_diag hold x_fwd / xl_fwd on entry, with the
  // last block optionally pre-seeded (rgf_retarded / rgf_lesser_greater x_last).
  int mode;
  int fwd_given;       // mode 1: xr_diag already holds x_fwd; run only the Keldysh recursion
};

// Process-wide default for RgfArgs::overlap used by the C ABI.
int rgf_overlap_default();
void set_rgf_overlap_default(int on);

size_t rgf_workspace_bytes(int n_e, int n_b, int bs);
int rgf_selected_solve(const RgfArgs& a, void* ws, size_t ws_bytes, cudaStream_t stream);

}  // namespace negf
