// Contour-integral moments of Beyn's boundary solver (obc.py:198-296),
// batched over surface problems: for each quadrature node z_k,
//   P(z_k) = n' + z_k m + z_k^2 n           (ew kernel, complex coefficients)
//   X_k    = P(z_k)^-1                      (pivoted batched inverse)
//   S0 += w_k X_k,  S1 += w_k z_k X_k       (ew accumulation)
// and finally a0 = S0 probe, a1 = S1 probe (one grouped DMMA GEMM; the seeded
// probe is shared by every problem). The reference solves P(z) R = probe per
// node; (sum_k w_k P^-1) probe is the same moment up to roundoff. The small
// rank-revealing SVD / eigenproblem / pseudo-inverse steps run in obc.py on
// the device (cuSOLVER through torch.linalg).
#include "../../include/negf_b200.h"
#include "ew.cuh"
#include "zgemm.cuh"
#include "zinv.cuh"

namespace negf {
namespace {
inline size_t a256(size_t x) { return (x + 255) & ~size_t(255); }
#define RC(x) do { int _rc = (x); if (_rc) return _rc; } while (0)
}  // namespace
}  // namespace negf

using namespace negf;

extern "C" {

size_t negf_beyn_workspace_bytes(int batch, int bs) {
  const size_t blk = a256(sizeof(z_t) * (size_t)batch * bs * bs);
  return 4 * blk + a256(zinv_workspace_bytes(bs, batch));
}

int negf_beyn_moments(int batch, int bs, int n_quad, const void* m, const void* n, const void* np,
                      const double* z, const double* w, const void* probe, void* a0, void* a1,
                      int* status, void* workspace, size_t workspace_bytes, void* stream) {
  if (batch < 0 || bs < 1 || n_quad < 1 || !m || !n || !np || !z || !w || !probe || !a0 || !a1 || !status)
    return -1;
  if (batch == 0) return 0;
  if (workspace_bytes < negf_beyn_workspace_bytes(batch, bs)) return -4;
  cudaStream_t st = (cudaStream_t)stream;
  const long long n2 = (long long)bs * bs;
  const size_t blk = a256(sizeof(z_t) * (size_t)batch * n2);
  char* p = (char*)workspace;
  z_t* P = (z_t*)p; p += blk;
  z_t* X = (z_t*)p; p += blk;
  z_t* S0 = (z_t*)p; p += blk;
  z_t* S1 = (z_t*)p; p += blk;
  void* inv_ws = p;
  const size_t inv_bytes = zinv_workspace_bytes(bs, batch);
  InvAux aux;
  aux.status = status; aux.status_code = 1; aux.u_spread = nullptr; aux.spread_stride = 0; aux.active = nullptr;
  for (int k = 0; k < n_quad; ++k) {
    const double2 zk = make_double2(z[2 * k], z[2 * k + 1]);
    const double2 zk2 = make_double2(zk.x * zk.x - zk.y * zk.y, 2.0 * zk.x * zk.y);
    const double2 wk = make_double2(w[2 * k], w[2 * k + 1]);
    const double2 wzk = make_double2(wk.x * zk.x - wk.y * zk.y, wk.x * zk.y + wk.y * zk.x);
    {
      EwGroup g;
      g.n = 1; g.rows = bs; g.cols = bs;
      EwDesc& d = g.d[0];
      d.batch = batch; d.nterms = 3; d.out = P; d.sOut = n2;
      d.X[0] = (const z_t*)np; d.sX[0] = n2; d.opH[0] = 0; d.coef[0] = make_double2(1.0, 0.0);
      d.X[1] = (const z_t*)m; d.sX[1] = n2; d.opH[1] = 0; d.coef[1] = zk;
      d.X[2] = (const z_t*)n; d.sX[2] = n2; d.opH[2] = 0; d.coef[2] = zk2;
      RC(ew_group_launch(g, st));
    }
    aux.status_code = 1 + k;
    RC(zinv_batched(P, n2, bs, X, n2, bs, bs, batch, aux, inv_ws, inv_bytes, st));
    {
      EwGroup g;
      g.n = 2; g.rows = bs; g.cols = bs;
      for (int s = 0; s < 2; ++s) {
        EwDesc& d = g.d[s];
        z_t* S = s ? S1 : S0;
        d.batch = batch; d.out = S; d.sOut = n2;
        d.nterms = k ? 2 : 1;
        d.X[0] = X; d.sX[0] = n2; d.opH[0] = 0; d.coef[0] = s ? wzk : wk;
        d.X[1] = S; d.sX[1] = n2; d.opH[1] = 0; d.coef[1] = make_double2(1.0, 0.0);
      }
      RC(ew_group_launch(g, st));
    }
  }
  ZGemmGroup g;
  g.n = 2;
  for (int s = 0; s < 2; ++s) {
    ZGemmDesc d = zdesc_default();
    d.M = bs; d.N = bs; d.batch = batch;
    d.t[0] = zterm(s ? S1 : S0, n2, bs, OP_N, (const z_t*)probe, 0, bs, OP_N, bs);
    for (int i = 1; i < kMaxTerms; ++i) d.t[i] = d.t[0];
    d.D = (z_t*)(s ? a1 : a0); d.sD = n2; d.ldd = bs;
    g.d[s] = d;
  }
  return zgemm_group_launch(g, st);
}

}  // extern "C"
