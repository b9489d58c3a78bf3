// Spatial domain decomposition of the selected solve (dist.py:354-717),
// batched over energies: the partition-local pieces that run on each GPU.
//
//   negf_dd_schur_tail     _schur_tail   dist.py:365-385
//   negf_dd_middle_sweep   _middle_sweep dist.py:388-448
//   negf_dd_fold_corner    _fold_corner  dist.py:451-473
//   negf_dd_reverse_chain  reverse_blocks (blocks.py) for the bottom partition
//
// The end partitions' forward/backward sweeps are negf_rgf_sweeps_batched
// (mode 1 / mode 2 with the exact boundary block seeded into the last
// diagonal), the middles' local solve is negf_rgf_selected_solve_batched; the
// reduced boundary chain (dist.py:486-561) is assembled from the all-gathered
// contributions and solved with the same entry points (dd.py). Every block
// product is a term of a grouped DMMA GEMM; layouts are the energy-major
// packed stacks of the rest of the library.
#include <initializer_list>
#include <utility>

#include "../../include/negf_b200.h"
#include "ew.cuh"
#include "prof.cuh"
#include "zgemm.cuh"
#include "zinv.cuh"

namespace negf {
namespace {

inline size_t a256(size_t x) { return (x + 255) & ~size_t(255); }
#define RC(x) do { int _rc = (x); if (_rc) return _rc; } while (0)

// One term op(A) op(B) on batch n_e with explicit batch strides.
struct Opnd {
  const z_t* p;
  long long s;
  int op;
};

ZGemmDesc gemm_desc(int bs, int n_e, std::initializer_list<std::pair<Opnd, Opnd>> terms,
                    std::initializer_list<int> negs, z_t* D, long long sD, const z_t* C = nullptr,
                    long long sC = 0, double beta = 0.0, double alpha = 1.0) {
  ZGemmDesc d = zdesc_default();
  d.M = bs; d.N = bs; d.batch = n_e;
  int k = 0;
  auto ng = negs.begin();
  for (const auto& t : terms) {
    d.t[k] = zterm(t.first.p, t.first.s, bs, t.first.op, t.second.p, t.second.s, bs, t.second.op, bs,
                   ng != negs.end() && *ng);
    if (ng != negs.end()) ++ng;
    ++k;
  }
  d.nterms = k;
  for (int i = k; i < kMaxTerms; ++i) d.t[i] = d.t[0];
  d.alpha = make_double2(alpha, 0.0);
  d.C = C; d.sC = sC; d.ldc = bs; d.beta = make_double2(beta, 0.0);
  d.D = D; d.sD = sD; d.ldd = bs;
  return d;
}

int launch1(const ZGemmDesc& d, cudaStream_t st) { return zgemm_launch(d, st); }

int launch_group(std::initializer_list<ZGemmDesc> ds, cudaStream_t st) {
  ZGemmGroup g;
  g.n = 0;
  for (const auto& d : ds) g.d[g.n++] = d;
  return zgemm_group_launch(g, st);
}

// out = sum coef_k op_k(X_k), batch n_e, blocks bs x bs
struct EwT {
  const z_t* x;
  long long s;
  int herm;
  double coef;
};
EwDesc ew_desc(int n_e, z_t* out, long long sOut, std::initializer_list<EwT> t) {
  EwDesc d;
  d.batch = n_e; d.nterms = 0; d.out = out; d.sOut = sOut;
  for (const auto& x : t) {
    d.X[d.nterms] = x.x;
    d.sX[d.nterms] = x.s;
    d.opH[d.nterms] = x.herm;
    d.coef[d.nterms] = make_double2(x.coef, 0.0);
    ++d.nterms;
  }
  return d;
}

int ew1(int bs, const EwDesc& d, cudaStream_t st) {
  EwGroup g;
  g.n = 1; g.rows = bs; g.cols = bs;
  g.d[0] = d;
  return ew_group_launch(g, st);
}

}  // namespace
}  // namespace negf

using namespace negf;

extern "C" {

size_t negf_dd_workspace_bytes(int n_e, int bs) {
  const size_t blk = a256(sizeof(z_t) * (size_t)n_e * bs * bs);
  return 24 * blk + a256(zinv_workspace_bytes(bs, n_e));
}

int negf_dd_schur_tail(int n_e, int w, int bs, const void* m_diag, const void* m_upper,
                       const void* m_lower, const void* bl_diag, const void* bl_upper,
                       const void* bg_diag, const void* bg_upper, const void* x_fwd,
                       const void* xl_fwd, const void* xg_fwd, void* s_out, void* bl_out,
                       void* bg_out, void* workspace, size_t workspace_bytes, void* stream) {
  if (n_e < 0 || w < 2 || bs < 1 || !m_diag || !m_upper || !m_lower || !x_fwd || !s_out) return -1;
  if (n_e == 0) return 0;
  if (workspace_bytes < negf_dd_workspace_bytes(n_e, bs)) return -4;
  cudaStream_t st = (cudaStream_t)stream;
  const long long n2 = (long long)bs * bs, sd = (long long)w * n2, so = (long long)(w - 1) * n2;
  const int last = w - 1;
  auto D = [&](const void* base, int i) { return (const z_t*)base + (long long)i * n2; };
  char* p = (char*)workspace;
  const size_t blk = a256(sizeof(z_t) * (size_t)n_e * n2);
  z_t* t = (z_t*)p; p += blk;
  z_t* y = (z_t*)p; p += blk;
  z_t* q = (z_t*)p; p += blk;
  // t = a x_{last-1}, a = M[last, last-1]
  RC(launch1(gemm_desc(bs, n_e, {{{D(m_lower, last - 1), so, OP_N}, {D(x_fwd, last - 1), sd, OP_N}}}, {}, t, n2), st));
  // s = M[last,last] - t M[last-1,last]
  RC(launch1(gemm_desc(bs, n_e, {{{t, n2, OP_N}, {D(m_upper, last - 1), so, OP_N}}}, {}, (z_t*)s_out, n2,
                       D(m_diag, last), sd, 1.0, -1.0), st));
  const void* bd[2] = {bl_diag, bg_diag};
  const void* bu[2] = {bl_upper, bg_upper};
  const void* xl[2] = {xl_fwd, xg_fwd};
  void* bo[2] = {bl_out, bg_out};
  for (int k = 0; k < 2; ++k) {
    if (!bd[k] || !bu[k] || !xl[k] || !bo[k]) continue;
    // y = t B[last-1, last];  q = a xl_{last-1}
    RC(launch_group({gemm_desc(bs, n_e, {{{t, n2, OP_N}, {D(bu[k], last - 1), so, OP_N}}}, {}, y, n2),
                     gemm_desc(bs, n_e, {{{D(m_lower, last - 1), so, OP_N}, {D(xl[k], last - 1), sd, OP_N}}}, {}, q,
                               n2)},
                    st));
    // b_out = B[last,last] + q a^H - y + y^H
    RC(launch1(gemm_desc(bs, n_e, {{{q, n2, OP_N}, {D(m_lower, last - 1), so, OP_H}}}, {}, (z_t*)bo[k], n2,
                         D(bd[k], last), sd, 1.0), st));
    RC(ew1(bs, ew_desc(n_e, (z_t*)bo[k], n2, {{(const z_t*)bo[k], n2, 0, 1.0}, {y, n2, 0, -1.0}, {y, n2, 1, 1.0}}),
           st));
  }
  return 0;
}

int negf_dd_middle_sweep(int n_e, int w, int bs, const void* m_diag, const void* m_upper,
                         const void* m_lower, const void* bl_diag, const void* bl_upper,
                         const void* bg_diag, const void* bg_upper, void* s_out, void* bl_out,
                         void* bg_out, int* status, void* workspace, size_t workspace_bytes,
                         void* stream) {
  if (n_e < 0 || w < 2 || bs < 1 || !m_diag || !m_upper || !m_lower || !s_out || !status) return -1;
  if (n_e == 0) return 0;
  if (workspace_bytes < negf_dd_workspace_bytes(n_e, bs)) return -4;
  cudaStream_t st = (cudaStream_t)stream;
  const long long n2 = (long long)bs * bs, sd = (long long)w * n2, so = (long long)(w - 1) * n2;
  const size_t bytes = sizeof(z_t) * (size_t)n_e * n2;
  auto D = [&](const void* base, int i) { return (const z_t*)base + (long long)i * n2; };
  // outputs: s_out [4][n_e] = s_aa, s_ab, s_ba, s_bb;  b*_out [3][n_e] = b_aa, b_ab, b_bb
  z_t* s_aa = (z_t*)s_out;
  z_t* s_ab = s_aa + n_e * n2;
  z_t* s_ba = s_ab + n_e * n2;
  z_t* s_bb = s_ba + n_e * n2;
  const void* bd[2] = {bl_diag, bg_diag};
  const void* bu[2] = {bl_upper, bg_upper};
  z_t* bo[2] = {(z_t*)bl_out, (z_t*)bg_out};
  bool kind_on[2];
  for (int k = 0; k < 2; ++k) kind_on[k] = bd[k] && bu[k] && bo[k];
  // gather a strided block column [n_e] (stride sx) into a contiguous [n_e] array
  auto gather = [&](z_t* dst, const z_t* src, long long sx) -> int {
    NEGF_CUDA_CHECK(cudaMemcpy2DAsync(dst, n2 * sizeof(z_t), src, sx * sizeof(z_t), n2 * sizeof(z_t), n_e,
                                      cudaMemcpyDeviceToDevice, st));
    return 0;
  };
  RC(gather(s_aa, D(m_diag, 0), sd));
  RC(gather(s_ab, D(m_upper, 0), so));   // f
  RC(gather(s_ba, D(m_lower, 0), so));   // f'
  RC(gather(s_bb, D(m_diag, 1), sd));    // s_i
  for (int k = 0; k < 2; ++k)
    if (kind_on[k]) {
      RC(gather(bo[k], D(bd[k], 0), sd));              // b_a
      RC(gather(bo[k] + n_e * n2, D(bu[k], 0), so));   // b_ai
      RC(gather(bo[k] + 2 * n_e * n2, D(bd[k], 1), sd));  // b_i
    }
  if (w == 2) return 0;
  char* p = (char*)workspace;
  const size_t blk = a256(bytes);
  auto take = [&]() { z_t* r = (z_t*)p; p += blk; return r; };
  z_t *y = take(), *fy = take(), *my = take(), *tmp = take(), *f2 = take(), *fp2 = take();
  z_t *ybh[2], *t1[2], *fyb[2], *myb[2], *bai2[2], *T1[2];
  for (int k = 0; k < 2; ++k) { ybh[k] = take(); t1[k] = take(); fyb[k] = take(); myb[k] = take(); bai2[k] = take(); T1[k] = take(); }
  void* inv_ws = p;
  const size_t inv_bytes = zinv_workspace_bytes(bs, n_e);
  InvAux aux;
  aux.status = status; aux.u_spread = nullptr; aux.spread_stride = 0; aux.active = nullptr;
  z_t* f = s_ab;
  z_t* fp = s_ba;
  for (int i = 1; i < w - 1; ++i) {
    // y = s_i^-1 (s_i is consumed; status code = 1 + step)
    aux.status_code = 1 + i;
    NEGF_CUDA_CHECK(cudaMemcpyAsync(tmp, s_bb, bytes, cudaMemcpyDeviceToDevice, st));
    RC(zinv_batched(tmp, n2, bs, y, n2, bs, bs, n_e, aux, inv_ws, inv_bytes, st));
    const z_t* m_dn = D(m_lower, i);
    const z_t* m_up = D(m_upper, i);
    // fy = f y, my = m_dn y
    RC(launch_group({gemm_desc(bs, n_e, {{{f, n2, OP_N}, {y, n2, OP_N}}}, {}, fy, n2),
                     gemm_desc(bs, n_e, {{{m_dn, so, OP_N}, {y, n2, OP_N}}}, {}, my, n2)}, st));
    // s_a -= fy f'
    RC(launch1(gemm_desc(bs, n_e, {{{fy, n2, OP_N}, {fp, n2, OP_N}}}, {}, s_aa, n2, s_aa, n2, 1.0, -1.0), st));
    for (int k = 0; k < 2; ++k) {
      if (!kind_on[k]) continue;
      z_t* b_a = bo[k];
      z_t* b_ai = bo[k] + n_e * n2;
      z_t* b_i = bo[k] + 2 * n_e * n2;
      const z_t* bu_i = D(bu[k], i);
      // ybh = (y b_i) y^H
      RC(launch1(gemm_desc(bs, n_e, {{{y, n2, OP_N}, {b_i, n2, OP_N}}}, {}, T1[k], n2), st));
      RC(launch1(gemm_desc(bs, n_e, {{{T1[k], n2, OP_N}, {y, n2, OP_H}}}, {}, ybh[k], n2), st));
      // fyb = f ybh, myb = m_dn ybh, t1 = my B[i, i+1]
      RC(launch_group({gemm_desc(bs, n_e, {{{f, n2, OP_N}, {ybh[k], n2, OP_N}}}, {}, fyb[k], n2),
                       gemm_desc(bs, n_e, {{{m_dn, so, OP_N}, {ybh[k], n2, OP_N}}}, {}, myb[k], n2),
                       gemm_desc(bs, n_e, {{{my, n2, OP_N}, {bu_i, so, OP_N}}}, {}, t1[k], n2)}, st));
      // b_a += fy b_ai^H - b_ai fy^H + fyb f^H;   b_ai' = -fy B[i,i+1] - b_ai my^H + fyb m_dn^H
      RC(launch_group(
          {gemm_desc(bs, n_e, {{{fy, n2, OP_N}, {b_ai, n2, OP_H}}, {{b_ai, n2, OP_N}, {fy, n2, OP_H}},
                               {{fyb[k], n2, OP_N}, {f, n2, OP_H}}},
                     {0, 1, 0}, b_a, n2, b_a, n2, 1.0),
           gemm_desc(bs, n_e, {{{fy, n2, OP_N}, {bu_i, so, OP_N}}, {{b_ai, n2, OP_N}, {my, n2, OP_H}},
                               {{fyb[k], n2, OP_N}, {m_dn, so, OP_H}}},
                     {1, 1, 0}, bai2[k], n2)},
          st));
      NEGF_CUDA_CHECK(cudaMemcpyAsync(b_ai, bai2[k], bytes, cudaMemcpyDeviceToDevice, st));
      // b_i' = B[i+1,i+1] - t1 + t1^H + myb m_dn^H
      RC(launch1(gemm_desc(bs, n_e, {{{myb[k], n2, OP_N}, {m_dn, so, OP_H}}}, {}, b_i, n2, D(bd[k], i + 1), sd, 1.0),
                 st));
      RC(ew1(bs, ew_desc(n_e, b_i, n2, {{b_i, n2, 0, 1.0}, {t1[k], n2, 0, -1.0}, {t1[k], n2, 1, 1.0}}), st));
    }
    // f' <- -my f', f <- -fy m_up, s_i <- M[i+1,i+1] - my m_up
    RC(launch_group({gemm_desc(bs, n_e, {{{my, n2, OP_N}, {fp, n2, OP_N}}}, {}, fp2, n2, nullptr, 0, 0.0, -1.0),
                     gemm_desc(bs, n_e, {{{fy, n2, OP_N}, {m_up, so, OP_N}}}, {}, f2, n2, nullptr, 0, 0.0, -1.0),
                     gemm_desc(bs, n_e, {{{my, n2, OP_N}, {m_up, so, OP_N}}}, {}, s_bb, n2, D(m_diag, i + 1), sd,
                               1.0, -1.0)},
                    st));
    NEGF_CUDA_CHECK(cudaMemcpyAsync(fp, fp2, bytes, cudaMemcpyDeviceToDevice, st));
    NEGF_CUDA_CHECK(cudaMemcpyAsync(f, f2, bytes, cudaMemcpyDeviceToDevice, st));
  }
  return 0;
}

int negf_dd_fold_corner(int n_e, int w, int bs, int j, int side, void* m_diag, void* bl_diag,
                        void* bg_diag, const void* m_out, const void* m_in, const void* bl_couple,
                        const void* bg_couple, const void* x_env, const void* xl_env,
                        const void* xg_env, void* workspace, size_t workspace_bytes, void* stream) {
  if (n_e < 0 || w < 1 || bs < 1 || j < 0 || j >= w || !m_diag || !m_out || !m_in || !x_env) return -1;
  if (side != 0 && side != 1) return -1;
  if (n_e == 0) return 0;
  if (workspace_bytes < negf_dd_workspace_bytes(n_e, bs)) return -4;
  cudaStream_t st = (cudaStream_t)stream;
  const long long n2 = (long long)bs * bs, sd = (long long)w * n2;
  char* p = (char*)workspace;
  const size_t blk = a256(sizeof(z_t) * (size_t)n_e * n2);
  z_t* t = (z_t*)p; p += blk;
  z_t* u = (z_t*)p; p += blk;
  z_t* v = (z_t*)p; p += blk;
  z_t* mj = (z_t*)m_diag + (long long)j * n2;
  // t = m_out x_env;  M_jj -= t m_in
  RC(launch1(gemm_desc(bs, n_e, {{{(const z_t*)m_out, n2, OP_N}, {(const z_t*)x_env, n2, OP_N}}}, {}, t, n2), st));
  RC(launch1(gemm_desc(bs, n_e, {{{t, n2, OP_N}, {(const z_t*)m_in, n2, OP_N}}}, {}, mj, sd, mj, sd, 1.0, -1.0), st));
  // sources: the stored coupling block Bc is B_in = Bc, B_out = -Bc^H on the
  // left corner (side 0) and B_out = Bc, B_in = -Bc^H on the right (side 1).
  void* bd[2] = {bl_diag, bg_diag};
  const void* bc[2] = {bl_couple, bg_couple};
  const void* xe[2] = {xl_env, xg_env};
  for (int k = 0; k < 2; ++k) {
    if (!bd[k] || !bc[k] || !xe[k]) continue;
    const z_t* Bc = (const z_t*)bc[k];
    z_t* bj = (z_t*)bd[k] + (long long)j * n2;
    // u = B_out x_env^H ; v = m_out xl_env
    if (side == 0)
      RC(launch_group({gemm_desc(bs, n_e, {{{Bc, n2, OP_H}, {(const z_t*)x_env, n2, OP_H}}}, {1}, u, n2),
                       gemm_desc(bs, n_e, {{{(const z_t*)m_out, n2, OP_N}, {(const z_t*)xe[k], n2, OP_N}}}, {}, v, n2)},
                      st));
    else
      RC(launch_group({gemm_desc(bs, n_e, {{{Bc, n2, OP_N}, {(const z_t*)x_env, n2, OP_H}}}, {}, u, n2),
                       gemm_desc(bs, n_e, {{{(const z_t*)m_out, n2, OP_N}, {(const z_t*)xe[k], n2, OP_N}}}, {}, v, n2)},
                      st));
    // B_jj += -t B_in - u m_out^H + v m_out^H
    const bool left = side == 0;
    RC(launch1(gemm_desc(bs, n_e,
                         {{{t, n2, OP_N}, {Bc, n2, left ? OP_N : OP_H}},
                          {{u, n2, OP_N}, {(const z_t*)m_out, n2, OP_H}},
                          {{v, n2, OP_N}, {(const z_t*)m_out, n2, OP_H}}},
                         {left ? 1 : 0, 1, 0}, bj, sd, bj, sd, 1.0),
               st));
  }
  return 0;
}

int negf_dd_reverse_chain(int n_e, int w, int bs, const void* diag_in, const void* upper_in,
                          const void* lower_in, void* diag_out, void* upper_out, void* lower_out,
                          void* stream) {
  if (n_e < 0 || w < 1 || bs < 1 || !diag_in || !diag_out) return -1;
  if (w > 1 && (!upper_in || !upper_out)) return -1;
  if (n_e == 0) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  const long long n2 = (long long)bs * bs, sd = (long long)w * n2, so = (long long)(w - 1) * n2;
  // diagonal reversed; full storage: upper' = lower reversed, lower' = upper reversed;
  // lg-compressed (lower_in == NULL): upper'[t] = -upper[w-2-t]^H
  EwGroup g;
  g.rows = bs; g.cols = bs; g.n = 0;
  auto flush = [&]() -> int {
    if (g.n) { RC(ew_group_launch(g, st)); g.n = 0; }
    return 0;
  };
  for (int t = 0; t < w; ++t) {
    g.d[g.n++] = ew_desc(n_e, (z_t*)diag_out + t * n2, sd, {{(const z_t*)diag_in + (w - 1 - t) * n2, sd, 0, 1.0}});
    if (g.n == kEwGroup) RC(flush());
  }
  for (int t = 0; t + 1 < w; ++t) {
    const long long src = (long long)(w - 2 - t) * n2;
    if (lower_in) {
      g.d[g.n++] = ew_desc(n_e, (z_t*)upper_out + t * n2, so, {{(const z_t*)lower_in + src, so, 0, 1.0}});
      if (g.n == kEwGroup) RC(flush());
      if (lower_out) {
        g.d[g.n++] = ew_desc(n_e, (z_t*)lower_out + t * n2, so, {{(const z_t*)upper_in + src, so, 0, 1.0}});
        if (g.n == kEwGroup) RC(flush());
      }
    } else {
      g.d[g.n++] = ew_desc(n_e, (z_t*)upper_out + t * n2, so, {{(const z_t*)upper_in + src, so, 1, -1.0}});
      if (g.n == kEwGroup) RC(flush());
    }
  }
  return flush();
}

}  // extern "C"
