// extern "C" entry points declared in include/negf_b200.h.
#include "../../include/negf_b200.h"
#include "memo.cuh"
#include "obc.cuh"
#include "rgf.cuh"
#include "zgemm.cuh"
#include "zinv.cuh"

using namespace negf;

extern "C" {

int negf_abi_version(void) { return 100; }

int negf_set_rgf_overlap(int on) {
  set_rgf_overlap_default(on ? 1 : 0);
  return 0;
}

int negf_set_gemm_algo(int algo) {
  if (algo != 0 && algo != 2 && algo != 3) return -1;
  set_gemm_algo(algo);
  return 0;
}

size_t negf_rgf_workspace_bytes(int n_e, int n_b, int bs) {
  return rgf_workspace_bytes(n_e, n_b, bs);
}

int negf_rgf_selected_solve_batched(int n_e, int n_b, int bs, const void* m_diag,
                                    const void* m_upper, const void* m_lower, const void* bl_diag,
                                    const void* bl_upper, const void* bg_diag,
                                    const void* bg_upper, void* xr_diag, void* xr_upper,
                                    void* xr_lower, void* xl_diag, void* xl_upper, void* xg_diag,
                                    void* xg_upper, int symmetrize, int* status, double* u_spread,
                                    void* workspace, size_t workspace_bytes, void* stream) {
  if (n_e < 0 || n_b < 1 || bs < 1 || !m_diag || !xr_diag) return -1;
  if (n_b > 1 && (!m_upper || !m_lower || !xr_upper || !xr_lower)) return -1;
  if ((bl_diag && !xl_diag) || (bg_diag && !xg_diag)) return -1;
  if (n_b > 1 && ((bl_diag && (!bl_upper || !xl_upper)) || (bg_diag && (!bg_upper || !xg_upper))))
    return -1;
  RgfArgs a;
  a.n_e = n_e; a.n_b = n_b; a.bs = bs;
  a.m_diag = (const z_t*)m_diag; a.m_upper = (const z_t*)m_upper; a.m_lower = (const z_t*)m_lower;
  a.b_diag[0] = (const z_t*)bl_diag; a.b_upper[0] = (const z_t*)bl_upper;
  a.b_diag[1] = (const z_t*)bg_diag; a.b_upper[1] = (const z_t*)bg_upper;
  a.xr_diag = (z_t*)xr_diag; a.xr_upper = (z_t*)xr_upper; a.xr_lower = (z_t*)xr_lower;
  a.xl_diag[0] = (z_t*)xl_diag; a.xl_upper[0] = (z_t*)xl_upper;
  a.xl_diag[1] = (z_t*)xg_diag; a.xl_upper[1] = (z_t*)xg_upper;
  a.symmetrize = symmetrize;
  a.status = status;
  a.u_spread = u_spread;
  a.overlap = rgf_overlap_default();
  a.mode = 0;
  a.fwd_given = 0;
  return rgf_selected_solve(a, workspace, workspace_bytes, (cudaStream_t)stream);
}

int negf_rgf_sweeps_batched(int mode, int fwd_given, int n_e, int n_b, int bs, const void* m_diag,
                            const void* m_upper, const void* m_lower, const void* bl_diag,
                            const void* bl_upper, const void* bg_diag, const void* bg_upper,
                            void* xr_diag, void* xr_upper, void* xr_lower, void* xl_diag,
                            void* xl_upper, void* xg_diag, void* xg_upper, int symmetrize,
                            int* status, double* u_spread, void* workspace,
                            size_t workspace_bytes, void* stream) {
  if (mode < 0 || mode > 2) return -1;
  if (n_e < 0 || n_b < 1 || bs < 1 || !m_diag || !xr_diag) return -1;
  if (n_b > 1 && (!m_upper || !m_lower)) return -1;
  if (mode != 1 && n_b > 1 && (!xr_upper || !xr_lower)) return -1;
  if ((bl_diag && !xl_diag) || (bg_diag && !xg_diag)) return -1;
  if (n_b > 1 && ((bl_diag && !bl_upper) || (bg_diag && !bg_upper))) return -1;
  if (mode != 1 && n_b > 1 && ((bl_diag && !xl_upper) || (bg_diag && !xg_upper))) return -1;
  RgfArgs a;
  a.n_e = n_e; a.n_b = n_b; a.bs = bs;
  a.m_diag = (const z_t*)m_diag; a.m_upper = (const z_t*)m_upper; a.m_lower = (const z_t*)m_lower;
  a.b_diag[0] = (const z_t*)bl_diag; a.b_upper[0] = (const z_t*)bl_upper;
  a.b_diag[1] = (const z_t*)bg_diag; a.b_upper[1] = (const z_t*)bg_upper;
  a.xr_diag = (z_t*)xr_diag; a.xr_upper = (z_t*)xr_upper; a.xr_lower = (z_t*)xr_lower;
  a.xl_diag[0] = (z_t*)xl_diag; a.xl_upper[0] = (z_t*)xl_upper;
  a.xl_diag[1] = (z_t*)xg_diag; a.xl_upper[1] = (z_t*)xg_upper;
  a.symmetrize = mode == 1 ? (symmetrize & 2) : symmetrize;
  a.status = status;
  a.u_spread = u_spread;
  a.overlap = rgf_overlap_default();
  a.mode = mode;
  a.fwd_given = fwd_given;
  return rgf_selected_solve(a, workspace, workspace_bytes, (cudaStream_t)stream);
}

int negf_zgemm_batched(int m, int n, int k, int batch, double alpha_re, double alpha_im,
                       const void* a, long long stride_a, int lda, int op_a, const void* b,
                       long long stride_b, int ldb, int op_b, double beta_re, double beta_im,
                       const void* c, long long stride_c, int ldc, void* d, long long stride_d,
                       int ldd, void* stream) {
  if (m < 0 || n < 0 || k < 0 || batch < 0 || !d) return -1;
  if (op_a < 0 || op_a > 3 || op_b < 0 || op_b > 3) return -1;
  ZGemmDesc g = zdesc_default();
  g.M = m; g.N = n; g.batch = batch; g.nterms = 1;
  g.t[0] = zterm((const z_t*)a, stride_a, lda, op_a, (const z_t*)b, stride_b, ldb, op_b, k);
  g.t[1] = g.t[0];
  g.alpha = make_double2(alpha_re, alpha_im);
  g.beta = make_double2(beta_re, beta_im);
  g.C = (const z_t*)c; g.sC = stride_c; g.ldc = ldc;
  g.D = (z_t*)d; g.sD = stride_d; g.ldd = ldd; g.transD = 0; g.active = nullptr;
  return zgemm_launch(g, (cudaStream_t)stream);
}

size_t negf_zinv_workspace_bytes(int n, int batch) { return zinv_workspace_bytes(n, batch); }

int negf_zinv_batched(int n, int batch, void* s, void* x, int* status, double* u_spread,
                      void* workspace, size_t workspace_bytes, void* stream) {
  if (n < 1 || batch < 0 || !s || !x) return -1;
  InvAux aux;
  aux.status = status; aux.status_code = 1; aux.u_spread = u_spread; aux.spread_stride = 1;
  aux.active = nullptr;
  long long s2 = (long long)n * n;
  return zinv_batched((z_t*)s, s2, n, (z_t*)x, s2, n, n, batch, aux, workspace, workspace_bytes,
                      (cudaStream_t)stream);
}

size_t negf_sancho_workspace_bytes(int batch, int bs) { return sancho_workspace_bytes(batch, bs); }

int negf_obc_sancho_batched(int batch, int bs, const void* m, const void* n, const void* np,
                            double tol, int max_iter, void* x, int* status, int* iters,
                            double* resid, const int* select, void* workspace,
                            size_t workspace_bytes, void* stream) {
  if (batch < 0 || bs < 1 || !m || !n || !np || !x || !status || !iters) return -1;
  if (!(tol > 0.0) || max_iter < 1) return -1;
  return sancho_batched((const z_t*)m, (const z_t*)n, (const z_t*)np, batch, bs, tol, max_iter,
                        (z_t*)x, status, iters, resid, workspace, workspace_bytes,
                        (cudaStream_t)stream, select);
}

size_t negf_fixed_point_workspace_bytes(int batch, int bs) { return fixed_point_workspace_bytes(batch, bs); }

int negf_obc_fixed_point_batched(int batch, int bs, const void* m, const void* n, const void* np, const void* x0,
                                 double tol, int max_iter, void* x, int* status, int* iters, double* resid,
                                 void* workspace, size_t workspace_bytes, void* stream) {
  if (batch < 0 || bs < 1 || !m || !n || !np || !x || !status || !iters || !(tol > 0.0) || max_iter < 1) return -1;
  return fixed_point_batched((const z_t*)m, (const z_t*)n, (const z_t*)np, batch, bs, (const z_t*)x0, tol, max_iter,
                             (z_t*)x, status, iters, resid, workspace, workspace_bytes, (cudaStream_t)stream);
}

size_t negf_memo_workspace_bytes(int map, int n_side, int n_kind, int bs) {
  return memo_workspace_bytes(map, n_side, n_kind, bs);
}

int negf_memo_refresh_batched(int map, int n_side, int n_kind, int bs, const void* m, const void* n,
                              const void* np, const void* a, const void* q, int n_fpi, double tol,
                              const void* x0, const int* has, void* out, int* need_direct, int* used,
                              void* workspace, size_t workspace_bytes, void* stream) {
  if (n_side < 0 || n_kind < 1 || bs < 1 || n_fpi < 2 || !x0 || !has || !out || !need_direct || !used) return -1;
  if (map == MEMO_SURFACE && (!m || !n || !np || n_kind != 1)) return -1;
  if (map == MEMO_STEIN && (!a || !q)) return -1;
  return memo_refresh(map, n_side, n_kind, bs, (const z_t*)m, (const z_t*)n, (const z_t*)np, (const z_t*)a,
                      (const z_t*)q, n_fpi, tol, (const z_t*)x0, has, (z_t*)out, need_direct, used, workspace,
                      workspace_bytes, (cudaStream_t)stream);
}

size_t negf_sigma_lg_obc_workspace_bytes(int batch, int bs) {
  return sigma_lg_obc_workspace_bytes(batch, bs);
}

int negf_sigma_lg_obc_batched(int batch, int bs, const void* x, const void* n, const void* np,
                              const double* f, void* sigma_r, void* sigma_lesser,
                              void* sigma_greater, void* workspace, size_t workspace_bytes,
                              void* stream) {
  if (batch < 0 || bs < 1 || !x || !n || !np || !f) return -1;
  return sigma_lg_obc_batched((const z_t*)x, (const z_t*)n, (const z_t*)np, f, batch, bs,
                              (z_t*)sigma_r, (z_t*)sigma_lesser, (z_t*)sigma_greater, workspace,
                              workspace_bytes, (cudaStream_t)stream);
}

size_t negf_g_obc_workspace_bytes(int n_e, int bs) { return g_obc_workspace_bytes(n_e, bs); }

int negf_g_obc_apply(int n_e, int n_b, int bs, void* m_diag, const void* m_upper,
                     const void* m_lower, void* bl_diag, void* bg_diag, const double* f_left,
                     const double* f_right, double tol, int max_iter, void* sl_left,
                     void* sg_left, void* sl_right, void* sg_right, int* status, int* iters,
                     double* resid, void* memo_cache, int* memo_has, int* memo_used,
                     long long memo_ld, int n_fpi, double memo_tol, const void* x_surface,
                     void* workspace, size_t workspace_bytes, void* stream) {
  if (n_e < 0 || n_b < 2 || bs < 1 || !m_diag || !m_upper || !m_lower || !f_left || !f_right)
    return -1;
  if (!status || !iters) return -1;
  if (memo_cache && (!memo_has || memo_ld < n_e || n_fpi < 2)) return -1;
  GObcArgs a;
  a.n_e = n_e; a.n_b = n_b; a.bs = bs;
  a.m_diag = (z_t*)m_diag; a.m_upper = (const z_t*)m_upper; a.m_lower = (const z_t*)m_lower;
  a.bl_diag = (z_t*)bl_diag; a.bg_diag = (z_t*)bg_diag;
  a.f_left = f_left; a.f_right = f_right; a.tol = tol; a.max_iter = max_iter;
  a.sl_left = (z_t*)sl_left; a.sg_left = (z_t*)sg_left;
  a.sl_right = (z_t*)sl_right; a.sg_right = (z_t*)sg_right;
  a.status = status; a.iters = iters; a.resid = resid;
  a.memo_cache = (z_t*)memo_cache; a.memo_has = memo_has; a.memo_used = memo_used;
  a.memo_ld = memo_ld; a.n_fpi = n_fpi; a.memo_tol = memo_tol;
  a.x_surface = (const z_t*)x_surface;
  return g_obc_apply(a, workspace, workspace_bytes, (cudaStream_t)stream);
}

int negf_g_assemble(int n_e, int n_b, int bs, const void* h_diag, const void* h_upper,
                    const void* h_lower, const double* energy, const double* f_bath, double eta,
                    const void* sr_diag, const void* sr_upper, const void* sr_lower,
                    const void* sl_diag, const void* sl_upper, const void* sg_diag,
                    const void* sg_upper, void* m_diag, void* m_upper, void* m_lower,
                    void* bl_diag, void* bl_upper, void* bg_diag, void* bg_upper, void* stream) {
  if (n_e < 0 || n_b < 1 || bs < 1 || !h_diag || !energy || !f_bath || !m_diag) return -1;
  if (n_b > 1 && (!h_upper || !h_lower || !m_upper || !m_lower)) return -1;
  GAssembleArgs a;
  a.n_e = n_e; a.n_b = n_b; a.bs = bs;
  a.h_diag = (const z_t*)h_diag; a.h_upper = (const z_t*)h_upper; a.h_lower = (const z_t*)h_lower;
  a.energy = energy; a.f_bath = f_bath; a.eta = eta;
  a.sr_diag = (const z_t*)sr_diag; a.sr_upper = (const z_t*)sr_upper;
  a.sr_lower = (const z_t*)sr_lower;
  a.sl_diag = (const z_t*)sl_diag; a.sl_upper = (const z_t*)sl_upper;
  a.sg_diag = (const z_t*)sg_diag; a.sg_upper = (const z_t*)sg_upper;
  a.m_diag = (z_t*)m_diag; a.m_upper = (z_t*)m_upper; a.m_lower = (z_t*)m_lower;
  a.bl_diag = (z_t*)bl_diag; a.bl_upper = (z_t*)bl_upper;
  a.bg_diag = (z_t*)bg_diag; a.bg_upper = (z_t*)bg_upper;
  return g_assemble(a, (cudaStream_t)stream);
}

}  // extern "C"
