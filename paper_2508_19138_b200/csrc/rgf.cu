// Batched-over-energy RGF selected inversion (retarded + lesser + greater in
// one fused forward sweep and one fused backward sweep).
//
// Reference recurrences (negfgw/rgf.py):
//   forward_retarded   rgf.py:113-129   x_i = (M_ii - M_{i,i-1} x_{i-1} M_{i-1,i})^-1
//   forward_lg         rgf.py:132-149   b_i = B_ii + a xl_{i-1} a^dag - (y - y^dag),
//                                       y = (a x_{i-1}) B_{i-1,i};  xl_i = x_i b_i x_i^dag
//   rgf_retarded       rgf.py:152-183   backward: t = x_i M_{i,i+1}, u = t X_{i+1}, ...
//   rgf_lesser_greater rgf.py:186-229   backward lesser/greater
//   SelectedSolution.symmetrize rgf.py:82-88
//
// All energies of the batch advance in lock-step; every block product is one
// grouped, batched DMMA launch (zgemm.cu) and independent products of the
// same step (both kinds, retarded and lesser/greater) share a launch.
// Reuse versus the reference's 43 N_B - 39 products per energy:
//   * A_i = M_{i,i-1} x_{i-1} is shared by the retarded Schur update and y;
//   * t, u (= -X_up), mx are shared by the retarded and both Keldysh passes;
//   * with Q = p^dag + mxl (p = x_i B_{i,i+1}, mxl = M_{i+1,i} xl_i) and
//     T = X_{i+1} Q, W = XL_{i+1} t^dag, the lower block is -T - W (the
//     reference's X_{i+1} B_{i+1,i} x_i^dag equals -X_{i+1} p^dag by the lg
//     symmetry of B) and the diagonal update t W + (z - z^dag) - (y - y^dag)
//     is the anti-Hermitian part of Z = t (W + 2T): one product where the
//     direct form takes three (see the backward sweep; B^lg anti-Hermitian).
// => 27 N_B - 23 products + N_B inversions per energy (both kinds;
//    17 N_B - 15 with one Keldysh kind).
// x_fwd lives in xr_diag and xl_fwd in xl_diag: each is overwritten in place
// by the backward pass once its last reader has run.
#include <unordered_map>

#include "ew.cuh"
#include "rgf.cuh"
#include "zgemm.cuh"
#include "zinv.cuh"

#ifndef NEGF_RGF_HERM
// Anti-Hermitian products run on lower-triangle tiles only (zgemm.cuh herm),
// bit mask of sites: 1 = xl_0 = x_0 B_00 x_0^dag, 2 = b_i = M xl M^dag + E,
// 4 = xl_i = x_i b_i x_i^dag. Site 4 is off: on ill-conditioned chains it
// costs accuracy against the dense solution (34x the oracle's error on the
// unscaled random systems of test_gpu_rgf), sites 1 and 2 do not.
// C2 carrier +1.2 % (G^> by recursion +2.1 %), C3-shape iteration -1.7 %.
#define NEGF_RGF_HERM 3
#endif

namespace negf {

namespace {

constexpr int kTmpShared = 3;  // tA, tS, second tA buffer (forward pipeline)
constexpr int kTmpKind = 6;    // k0..k5
constexpr int kTmpTotal = kTmpShared + 2 * kTmpKind;

inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

struct Ctx {
  int n_e, n_b, bs;
  long long bs2, sdiag, soff;
  cudaStream_t st;
  z_t* tmp;  // [kTmpTotal][n_e][bs][bs]
  void* inv_ws;
  size_t inv_ws_bytes;

  z_t* T(int slot) const { return tmp + (long long)slot * n_e * bs2; }
  z_t* K(int kind, int j) const { return T(kTmpShared + kind * kTmpKind + j); }
  ZTerm term(const z_t* A, long long sA, int opA, const z_t* B, long long sB, int opB,
             bool neg = false) const {
    return zterm(A, sA, bs, opA, B, sB, bs, opB, bs, neg);
  }
  ZGemmDesc desc(const ZTerm& t0, z_t* D, long long sD, double alpha_re = 1.0,
                 const z_t* C = nullptr, long long sC = 0, double beta_re = 0.0,
                 int transD = 0) const {
    ZGemmDesc d = zdesc_default();
    d.M = bs; d.N = bs; d.batch = n_e; d.nterms = 1;
    d.t[0] = t0; d.t[1] = t0;
    d.alpha = make_double2(alpha_re, 0.0);
    d.beta = make_double2(beta_re, 0.0);
    d.C = C; d.sC = sC; d.ldc = bs;
    d.D = D; d.sD = sD; d.ldd = bs;
    d.transD = transD;
    d.active = nullptr;
    return d;
  }
  // anti-Hermitian output: only the lower-triangle tiles run (zgemm.cuh herm)
  int lg_ah = 0;  // B^lg diagonal blocks anti-Hermitian (RgfArgs.symmetrize bit 1)
  ZGemmDesc ah(ZGemmDesc d, int site) const {
    if (lg_ah && (NEGF_RGF_HERM & site)) d.herm = 1;
    return d;
  }
};

struct Group {
  ZGemmGroup g;
  Group() { g.n = 0; }
  void add(const ZGemmDesc& d) { g.d[g.n++] = d; }
  int run(cudaStream_t s) { int rc = zgemm_group_launch(g, s); g.n = 0; return rc; }
};

struct EGroup {
  EwGroup g;
  EGroup(int bs) { g.n = 0; g.rows = bs; g.cols = bs; }
  void add(z_t* out, long long sOut, int batch, std::initializer_list<const z_t*> X,
           std::initializer_list<long long> sX, std::initializer_list<int> opH,
           std::initializer_list<double> coef) {
    EwDesc& d = g.d[g.n++];
    d.batch = batch; d.out = out; d.sOut = sOut; d.nterms = (int)X.size();
    int i = 0;
    for (auto p : X) d.X[i++] = p;
    i = 0; for (auto s : sX) d.sX[i++] = s;
    i = 0; for (auto o : opH) d.opH[i++] = o;
    i = 0; for (auto c : coef) d.coef[i++] = make_double2(c, 0.0);
  }
  int run(cudaStream_t s) { int rc = ew_group_launch(g, s); g.n = 0; return rc; }
};

#define RC(x) do { int _rc = (x); if (_rc) return _rc; } while (0)

}  // namespace

static int g_overlap = 1;
int rgf_overlap_default() { return g_overlap; }
void set_rgf_overlap_default(int on) { g_overlap = on; }

size_t rgf_workspace_bytes(int n_e, int n_b, int bs) {
  size_t tmp = align256(sizeof(z_t) * (size_t)kTmpTotal * n_e * bs * bs);
  return tmp + align256(zinv_workspace_bytes(bs, n_e));
}

int rgf_selected_solve(const RgfArgs& a, void* ws, size_t ws_bytes, cudaStream_t st) {
  if (a.n_e <= 0) return 0;
  if (a.n_b < 1 || a.bs < 1) return -1;

  if (ws_bytes < rgf_workspace_bytes(a.n_e, a.n_b, a.bs)) return -4;
  Ctx c;
  c.n_e = a.n_e; c.n_b = a.n_b; c.bs = a.bs;
  c.lg_ah = (a.symmetrize & 2) != 0;
  c.bs2 = (long long)a.bs * a.bs;
  c.sdiag = (long long)a.n_b * c.bs2;
  c.soff = (long long)(a.n_b > 1 ? a.n_b - 1 : 0) * c.bs2;
  c.st = st;
  c.tmp = reinterpret_cast<z_t*>(ws);
  c.inv_ws = reinterpret_cast<char*>(ws) + align256(sizeof(z_t) * (size_t)kTmpTotal * a.n_e * c.bs2);
  c.inv_ws_bytes = ws_bytes - align256(sizeof(z_t) * (size_t)kTmpTotal * a.n_e * c.bs2);

  const int n = a.n_b, bs = a.bs, ne = a.n_e;
  const long long bs2 = c.bs2, sd = c.sdiag, so = c.soff;
  const long long st1 = bs2;  // temp energy stride
  int kinds[2], nk = 0;
  for (int k = 0; k < 2; ++k)
    if (a.b_diag[k]) kinds[nk++] = k;

  auto Md = [&](int i) { return a.m_diag + i * bs2; };
  auto Mu = [&](int i) { return a.m_upper + i * bs2; };
  auto Ml = [&](int i) { return a.m_lower + i * bs2; };
  auto Bd = [&](int k, int i) { return a.b_diag[k] + i * bs2; };
  auto Bu = [&](int k, int i) { return a.b_upper[k] + i * bs2; };
  auto Xd = [&](int i) { return a.xr_diag + i * bs2; };
  auto Xu = [&](int i) { return a.xr_upper + i * bs2; };
  auto Xl = [&](int i) { return a.xr_lower + i * bs2; };
  auto Ld = [&](int k, int i) { return a.xl_diag[k] + i * bs2; };
  auto Lu = [&](int k, int i) { return a.xl_upper[k] + i * bs2; };
  z_t* tA = c.T(0);
  z_t* tS = c.T(1);

  auto invert_into = [&](int i) -> int {
    InvAux aux;
    aux.status = a.status;
    aux.status_code = 1 + i;
    aux.u_spread = a.u_spread ? a.u_spread + i : nullptr;
    aux.spread_stride = n;
    aux.active = nullptr;
    return zinv_batched(tS, st1, bs, Xd(i), sd, bs, bs, ne, aux, c.inv_ws, c.inv_ws_bytes, st);
  };

  Group G;
  EGroup E(bs);

  // ---------------- forward sweep ----------------
  // Two-stream pipeline. The retarded chain (A_i, S_i, pivoted inverse) runs on
  // the caller's stream `st`; the Keldysh forward products of step i run on an
  // auxiliary stream `sk`, so the latency-bound inversion panels of step i+1
  // overlap the lesser/greater GEMMs of step i. A_i is double-buffered
  // (tA[i & 1]); events order the hand-offs:
  //   evA[p]: A_i ready (R -> K)   evX[p]: x_i ready (R -> K)
  //   evK[p]: step i's K work done, before R overwrites tA[p] at step i + 2.
  const bool pipe = a.overlap && nk > 0 && n > 1;
  // The auxiliary stream and its events are created once per (thread,
  // device, caller stream) and reused by every call (no per-call
  // create/destroy); keying on the caller's stream keeps concurrent solves
  // on different streams (carrier energy slices) and threads apart.
  struct AuxStreams {
    cudaStream_t sk = nullptr;
    cudaEvent_t evA[2], evX[2], evK[2], ev0;
  };
  thread_local std::unordered_map<unsigned long long, AuxStreams> aux_cache;
  cudaStream_t sk = st;
  cudaEvent_t *evA = nullptr, *evX = nullptr, *evK = nullptr, ev0 = nullptr;
  if (pipe) {
    int dev = 0;
    NEGF_CUDA_CHECK(cudaGetDevice(&dev));
    const unsigned long long key = (reinterpret_cast<unsigned long long>(st) << 6) ^ (unsigned long long)dev;
    AuxStreams& ax = aux_cache[key];
    if (!ax.sk) {
      for (int j = 0; j < 2; ++j) {
        NEGF_CUDA_CHECK(cudaEventCreateWithFlags(&ax.evA[j], cudaEventDisableTiming));
        NEGF_CUDA_CHECK(cudaEventCreateWithFlags(&ax.evX[j], cudaEventDisableTiming));
        NEGF_CUDA_CHECK(cudaEventCreateWithFlags(&ax.evK[j], cudaEventDisableTiming));
      }
      NEGF_CUDA_CHECK(cudaEventCreateWithFlags(&ax.ev0, cudaEventDisableTiming));
      NEGF_CUDA_CHECK(cudaStreamCreateWithFlags(&ax.sk, cudaStreamNonBlocking));
    }
    sk = ax.sk;
    evA = ax.evA; evX = ax.evX; evK = ax.evK; ev0 = ax.ev0;
    NEGF_CUDA_CHECK(cudaEventRecord(ev0, st));
    NEGF_CUDA_CHECK(cudaStreamWaitEvent(sk, ev0, 0));
  }
  // On EVERY exit (including an early error return after work was queued on
  // sk) the caller's stream waits for sk, so the caller never frees or reuses
  // workspace / outputs that sk kernels may still be writing.
  struct JoinGuard {
    cudaStream_t s, main;
    cudaEvent_t ev;
    bool on;
    ~JoinGuard() {
      if (on && cudaEventRecord(ev, s) == cudaSuccess) cudaStreamWaitEvent(main, ev, 0);
    }
  } jguard{sk, st, ev0, pipe};
  z_t* tAb[2] = {tA, c.T(2)};

  const bool do_fwd = a.mode != 2;
  const bool do_inv = !(a.mode == 1 && a.fwd_given);
  if (do_fwd) {
  // i = 0
  if (do_inv) {
    NEGF_CUDA_CHECK(cudaMemcpy2DAsync(tS, st1 * sizeof(z_t), Md(0), sd * sizeof(z_t),
                                      bs2 * sizeof(z_t), ne, cudaMemcpyDeviceToDevice, st));
    RC(invert_into(0));
  }
  if (pipe) {
    NEGF_CUDA_CHECK(cudaEventRecord(evX[0], st));
    NEGF_CUDA_CHECK(cudaStreamWaitEvent(sk, evX[0], 0));
  }
  for (int q = 0; q < nk; ++q) {  // U = x_0 B_00
    int k = kinds[q];
    G.add(c.desc(c.term(Xd(0), sd, OP_N, Bd(k, 0), sd, OP_N), c.K(k, 0), st1));
  }
  RC(G.run(sk));
  for (int q = 0; q < nk; ++q) {  // xl_0 = U x_0^dag
    int k = kinds[q];
    G.add(c.ah(c.desc(c.term(c.K(k, 0), st1, OP_N, Xd(0), sd, OP_H), Ld(k, 0), sd), 1));
  }
  RC(G.run(sk));
  if (pipe) NEGF_CUDA_CHECK(cudaEventRecord(evK[0], sk));

  for (int i = 1; i < n; ++i) {
    const int p = i & 1;
    z_t* Ai = pipe ? tAb[p] : tA;
    // --- retarded chain (stream st)
    if (pipe && i >= 2) NEGF_CUDA_CHECK(cudaStreamWaitEvent(st, evK[p], 0));  // K done with tA[p]
    G.add(c.desc(c.term(Ml(i - 1), so, OP_N, Xd(i - 1), sd, OP_N), Ai, st1));  // A = M_{i,i-1} x_{i-1}
    if (!pipe)
      for (int q = 0; q < nk; ++q) {  // T1_k = M_{i,i-1} xl_{k,i-1} (same launch when serial)
        int k = kinds[q];
        G.add(c.desc(c.term(Ml(i - 1), so, OP_N, Ld(k, i - 1), sd, OP_N), c.K(k, 0), st1));
      }
    RC(G.run(st));
    if (pipe) NEGF_CUDA_CHECK(cudaEventRecord(evA[p], st));
    if (do_inv) G.add(c.desc(c.term(Ai, st1, OP_N, Mu(i - 1), so, OP_N), tS, st1, -1.0, Md(i), sd, 1.0));
    if (!pipe)
      for (int q = 0; q < nk; ++q) {  // Y_k = A B_{k,i-1,i}
        int k = kinds[q];
        G.add(c.desc(c.term(Ai, st1, OP_N, Bu(k, i - 1), so, OP_N), c.K(k, 1), st1));
      }
    RC(G.run(st));  // S = M_ii - A M_{i-1,i}
    if (do_inv) RC(invert_into(i));
    if (pipe) NEGF_CUDA_CHECK(cudaEventRecord(evX[p], st));
    if (nk == 0) continue;
    // --- Keldysh forward products (stream sk)
    if (pipe) {
      for (int q = 0; q < nk; ++q) {  // T1_k: needs only K-stream data
        int k = kinds[q];
        G.add(c.desc(c.term(Ml(i - 1), so, OP_N, Ld(k, i - 1), sd, OP_N), c.K(k, 0), st1));
      }
      RC(G.run(sk));
      NEGF_CUDA_CHECK(cudaStreamWaitEvent(sk, evA[p], 0));
      for (int q = 0; q < nk; ++q) {  // Y_k = A B_{k,i-1,i}
        int k = kinds[q];
        G.add(c.desc(c.term(Ai, st1, OP_N, Bu(k, i - 1), so, OP_N), c.K(k, 1), st1));
      }
      RC(G.run(sk));
    }
    // E_k = B_k,ii - Y_k + Y_k^dag
    for (int q = 0; q < nk; ++q) {
      int k = kinds[q];
      E.add(c.K(k, 2), st1, ne, {Bd(k, i), c.K(k, 1), c.K(k, 1)}, {sd, st1, st1}, {0, 0, 1},
            {1.0, -1.0, 1.0});
    }
    RC(E.run(sk));
    // b_k = T1_k M_{i,i-1}^dag + E_k
    for (int q = 0; q < nk; ++q) {
      int k = kinds[q];
      G.add(c.ah(c.desc(c.term(c.K(k, 0), st1, OP_N, Ml(i - 1), so, OP_H), c.K(k, 3), st1, 1.0,
                           c.K(k, 2), st1, 1.0), 2));
    }
    RC(G.run(sk));
    if (pipe) NEGF_CUDA_CHECK(cudaStreamWaitEvent(sk, evX[p], 0));
    // U_k = x_i b_k
    for (int q = 0; q < nk; ++q) {
      int k = kinds[q];
      G.add(c.desc(c.term(Xd(i), sd, OP_N, c.K(k, 3), st1, OP_N), c.K(k, 0), st1));
    }
    RC(G.run(sk));
    // xl_k,i = U_k x_i^dag
    for (int q = 0; q < nk; ++q) {
      int k = kinds[q];
      G.add(c.ah(c.desc(c.term(c.K(k, 0), st1, OP_N, Xd(i), sd, OP_H), Ld(k, i), sd), 4));
    }
    RC(G.run(sk));
    if (pipe) NEGF_CUDA_CHECK(cudaEventRecord(evK[p], sk));
  }
  if (pipe) {  // join: the backward sweep reads everything the K stream wrote
    NEGF_CUDA_CHECK(cudaEventRecord(ev0, sk));
    NEGF_CUDA_CHECK(cudaStreamWaitEvent(st, ev0, 0));
  }
  }  // do_fwd
  if (a.mode == 1) return 0;

  // ---------------- backward sweep ----------------
  // X_{n-1,n-1} = x_{n-1} and XL_{n-1} = xl_{n-1} already sit in place.
  for (int i = n - 2; i >= 0; --i) {
    // G1: t = x_i M_{i,i+1}; mx = M_{i+1,i} x_i; p_k = x_i B_{k,i,i+1}; mxl_k = M_{i+1,i} xl_{k,i}
    G.add(c.desc(c.term(Xd(i), sd, OP_N, Mu(i), so, OP_N), tA, st1));
    G.add(c.desc(c.term(Ml(i), so, OP_N, Xd(i), sd, OP_N), tS, st1));
    for (int q = 0; q < nk; ++q) {
      int k = kinds[q];
      G.add(c.desc(c.term(Xd(i), sd, OP_N, Bu(k, i), so, OP_N), c.K(k, 0), st1));
      G.add(c.desc(c.term(Ml(i), so, OP_N, Ld(k, i), sd, OP_N), c.K(k, 1), st1));
    }
    RC(G.run(st));
    // G2: X_up = -t X_{i+1}; X_lo = -X_{i+1} mx; W_k = XL_{k,i+1} t^dag
    G.add(c.desc(c.term(tA, st1, OP_N, Xd(i + 1), sd, OP_N), Xu(i), so, -1.0));
    G.add(c.desc(c.term(Xd(i + 1), sd, OP_N, tS, st1, OP_N), Xl(i), so, -1.0));
    for (int q = 0; q < nk; ++q) {
      int k = kinds[q];
      G.add(c.desc(c.term(Ld(k, i + 1), sd, OP_N, tA, st1, OP_H), c.K(k, 3), st1));
    }
    RC(G.run(st));
    // Q_k = p_k^dag + mxl_k
    for (int q = 0; q < nk; ++q) {
      int k = kinds[q];
      E.add(c.K(k, 5), st1, ne, {c.K(k, 0), c.K(k, 1)}, {st1, st1}, {1, 0}, {1.0, 1.0});
    }
    if (nk) RC(E.run(st));
    // G3: X_ii = x_i - X_up mx (in place); T_k = X_{i+1} Q_k.
    // The Keldysh diagonal is XL_ii = xl_i + t W + (z - z^dag) - (y - y^dag):
    //   (z - z^dag) - (y - y^dag) = v - v^dag with v = -X_up mxl + p X_up^dag
    //   = -X_up Q + Q^dag X_up^dag = t T - (t T)^dag          (X_up = -t X_{i+1})
    // and t W = t XL_{i+1} t^dag is anti-Hermitian (B^lg is, so is XL), hence
    //   XL_ii = xl_i + (Z - Z^dag)/2 with Z = t (W + 2 T):
    // one product where the direct form takes three (t W, u mxl, p u^dag).
    G.add(c.desc(c.term(Xu(i), so, OP_N, tS, st1, OP_N), Xd(i), sd, -1.0, Xd(i), sd, 1.0));
    for (int q = 0; q < nk; ++q) {
      int k = kinds[q];
      G.add(c.desc(c.term(Xd(i + 1), sd, OP_N, c.K(k, 5), st1, OP_N), c.K(k, 2), st1));
    }
    RC(G.run(st));
    if (nk == 0) continue;
    // F_k = W_k + 2 T_k ; XL_k,up = T_k^dag + W_k^dag  (= (-lower)^dag, lower = -T - W)
    for (int q = 0; q < nk; ++q) {
      int k = kinds[q];
      E.add(c.K(k, 4), st1, ne, {c.K(k, 3), c.K(k, 2)}, {st1, st1}, {0, 0}, {1.0, 2.0});
      E.add(Lu(k, i), so, ne, {c.K(k, 2), c.K(k, 3)}, {st1, st1}, {1, 1}, {1.0, 1.0});
    }
    RC(E.run(st));
    // G4: Z_k = t F_k
    for (int q = 0; q < nk; ++q) {
      int k = kinds[q];
      G.add(c.desc(c.term(tA, st1, OP_N, c.K(k, 4), st1, OP_N), c.K(k, 0), st1));
    }
    RC(G.run(st));
    // XL_k,ii = xl_k,i + (Z_k - Z_k^dag)/2 (in place)
    for (int q = 0; q < nk; ++q) {
      int k = kinds[q];
      E.add(Ld(k, i), sd, ne, {Ld(k, i), c.K(k, 0), c.K(k, 0)}, {sd, st1, st1}, {0, 0, 1}, {1.0, 0.5, -0.5});
    }
    RC(E.run(st));
  }
  if (a.symmetrize & 1)
    for (int q = 0; q < nk; ++q) RC(antiherm_inplace(a.xl_diag[kinds[q]], bs2, bs, ne * n, st));
  return 0;
}

}  // namespace negf
