// Open-boundary (contact) self-energies on the GPU, batched over energies
// and contact sides. See obc.cu.
#pragma once
#include "common.cuh"

namespace negf {

enum ObcStatus : int {
  OBC_OK = 0,
  OBC_SINGULAR = 1,       // SingularBlockError (obc.py:125-128 via _linalg.invert)
  OBC_NOT_CONVERGED = 2,  // ConvergenceError "did not converge in max_iter sweeps" (obc.py:179-182)
  OBC_RESIDUAL = 3,       // ConvergenceError "decimation closed but residual ..." (obc.py:171-176)
  OBC_SPECTRAL = 4,       // SpectralRadiusError (obc.py:434-437)
};

// Sancho-Rubio decimation for `batch` independent surface problems
// x = (m - n x n')^-1, contiguous [batch][bs][bs] inputs.
size_t sancho_workspace_bytes(int batch, int bs);
int sancho_batched(const z_t* m, const z_t* n, const z_t* np, int batch, int bs, double tol,
                   int max_iter, z_t* x, int* status, int* iters, double* resid, void* ws,
                   size_t ws_bytes, cudaStream_t st, const int* select = nullptr);
// (select, optional: only problems with select[b] != 0 are solved; x, status,
// iters and resid of the others are left as they are, status 0, iters 0.)

// obc_fixed_point (obc.py:108-135) for `batch` problems: x <- (m - n x n')^-1
// from x0 (NULL: zeros) until |x_new - x|_F / |x_new|_F < tol; frozen problems
// stop updating. status: OBC_OK / OBC_SINGULAR / OBC_NOT_CONVERGED.
size_t fixed_point_workspace_bytes(int batch, int bs);
int fixed_point_batched(const z_t* m, const z_t* n, const z_t* np, int batch, int bs, const z_t* x0, double tol,
                        int max_iter, z_t* x, int* status, int* iters, double* resid, void* ws, size_t ws_bytes,
                        cudaStream_t st);

// G-side closure of one batch: per side, read the contact cell from the
// assembled M (energy-major tridiagonal), solve the surface problem, and
// fold Sigma^R_obc, Sigma^<_obc, Sigma^>_obc into the corner blocks.
struct GObcArgs {
  int n_e, n_b, bs;
  z_t* m_diag;
  const z_t* m_upper;
  const z_t* m_lower;
  z_t* bl_diag;  // may be null (kind absent)
  z_t* bg_diag;
  const double* f_left;   // [n_e] fermi(E, mu_left, kT)
  const double* f_right;  // [n_e]
  double tol;
  int max_iter;
  // outputs (optional, [n_e][bs][bs]): boundary lesser/greater self-energies
  z_t* sl_left;
  z_t* sg_left;
  z_t* sl_right;
  z_t* sg_right;
  int* status;  // [2][n_e]
  int* iters;   // [2][n_e]
  double* resid;  // [2][n_e]
  // OBC memoizer (obc.py:519-608), optional (memo_cache null: direct Sancho
  // everywhere). memo_cache: side g's block e at memo_cache + (g*memo_ld+e)*bs^2;
  // memo_has / memo_used: [2][memo_ld] ints (in/out; out).
  z_t* memo_cache = nullptr;
  int* memo_has = nullptr;
  int* memo_used = nullptr;
  long long memo_ld = 0;
  int n_fpi = 20;
  double memo_tol = 0.0;
  // optional [2][n_e] surface blocks computed by the caller (replaces Sancho)
  const z_t* x_surface = nullptr;
};
size_t g_obc_workspace_bytes(int n_e, int bs);
int g_obc_apply(const GObcArgs& a, void* ws, size_t ws_bytes, cudaStream_t st);

// Carrier system assembly (scba.py:670-727): energy-independent H plus
// optional scattering self-energy blocks (energy-major) into M~ and B^<>.
struct GAssembleArgs {
  int n_e, n_b, bs;
  const z_t* h_diag;   // [n_b][bs][bs]
  const z_t* h_upper;  // [n_b-1][bs][bs]
  const z_t* h_lower;
  const double* energy;  // [n_e]
  const double* f_bath;  // [n_e] fermi(E, mu_mean, kT)
  double eta;
  const z_t* sr_diag;  // Sigma^R_scatt blocks [n_e][...] (nullable)
  const z_t* sr_upper;
  const z_t* sr_lower;
  const z_t* sl_diag;  // Sigma^<_scatt (nullable)
  const z_t* sl_upper;
  const z_t* sg_diag;
  const z_t* sg_upper;
  z_t* m_diag;
  z_t* m_upper;
  z_t* m_lower;
  z_t* bl_diag;
  z_t* bl_upper;
  z_t* bg_diag;
  z_t* bg_upper;
};
int g_assemble(const GAssembleArgs& a, cudaStream_t st);

}  // namespace negf

namespace negf {
// sigma_lg_obc (obc.py:460-486), batched: Sigma^R = n x n', Gamma = Sigma^R - Sigma^R^dag,
// Sigma^< = -f Gamma, Sigma^> = (1 - f) Gamma. Any output may be null.
int sigma_lg_obc_batched(const z_t* x, const z_t* n, const z_t* np, const double* f, int batch,
                         int bs, z_t* sr, z_t* sl, z_t* sg, void* ws, size_t ws_bytes,
                         cudaStream_t st);
size_t sigma_lg_obc_workspace_bytes(int batch, int bs);
}  // namespace negf
