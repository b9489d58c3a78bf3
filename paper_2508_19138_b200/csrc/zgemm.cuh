// Batched, grouped complex-FP64 GEMM on the FP64 tensor pipe (DMMA) for sm_100a.
//
//   D[b] = alpha * sum_t s_t * op(A_t[b]) op(B_t[b]) + beta * C[b]      (t < 4)
//   optionally stored conjugate-transposed: D[b][n][m] = conj(value(m, n)).
//
// This is the kernel behind every dense block product of the RGF recursion
// (reference: negfgw/_linalg.py:19 `gemm`, called from rgf.py:113-229),
// the OBC decimation (obc.py:162-178), the Stein doubling (obc.py:427-447)
// and the W assembly products (blocks.py:277 `bt_multiply`).
//
// Design (B200): tcgen05 has no f64 kind, so FP64 runs on the warp-level DMMA
// path (mma.sync.m8n8k4.f64 -> SASS DMMA.8x8x4). Measured on this pool's
// B200: DMMA 37.0 TFLOP/s, DFMA 36.7, cuBLAS ZGEMM 36.8 (profiles/).
// Operands are staged global->smem with cp.async (LDGSTS, 16 B = one complex)
// through a multi-stage pipeline. Complex values stay interleaved in smem
// so one LDS.128 yields both the real and the imaginary fragment.
// Two smem layouts, chosen per operand from its transpose flag so the global
// read is always coalesced:
//   k-contiguous  [mn][BK+4]   (op N for A, op T/H for B)
//   mn-contiguous [BK][BMN+2]  (op T/H for A, op N for B)
// Both paddings make the DMMA fragment read (lane -> (mn=lane/4, k=lane%4))
// bank-conflict free per 8-lane LDS.128 phase.
// A complex product takes four real DMMAs: re += ar*br + (-ai)*bi,
// im += ar*bi + ai*br; conjugation and term signs are sign-bit flips done on
// the integer pipe.
#pragma once
#include "common.cuh"

namespace negf {

struct ZTerm {
  const z_t* A;
  long long sA;  // batch stride (elements)
  int lda;
  int opA;
  const z_t* B;
  long long sB;
  int ldb;
  int opB;
  int K;
  int neg;  // bit 0: subtract this term; bit 1 (kTermReal): A or B has an exactly
            // zero imaginary part, so the 3M kernel skips the ai*bi product;
            // bit 2 / 3 (kTermRealA / kTermRealB): that operand is STORED as
            // doubles (pointer reinterpreted, ld and batch stride in doubles,
            // op N, ld and K (A) or N (B) even): the real x complex kernel
};

constexpr int kTermReal = 2;
constexpr int kTermRealA = 4;
constexpr int kTermRealB = 8;

constexpr int kMaxTerms = 4;

struct ZGemmDesc {
  int M, N, batch, nterms;  // nterms <= kMaxTerms
  ZTerm t[kMaxTerms];
  double2 alpha, beta;
  const z_t* C;
  long long sC;
  int ldc;
  z_t* D;
  long long sD;
  int ldd;
  int transD;  // store conj-transposed
  // anti-Hermitian output (D = -D^H, e.g. x b x^dag with b anti-Hermitian;
  // M == N): only tiles meeting the lower triangle run, each element below
  // the diagonal is stored with its mirror -conj(v), the diagonal as i Im v
  // (keeping a computed real part lets the Hermitian rounding component of a
  // chained x b x^dag recursion grow step by step) -- about half the products
  int herm;
  const int* active;  // optional per-batch mask: problems with active[b]==0 are skipped
  // Optional per-batch row indirection (stride s_map per batch entry): logical
  // row m of op(A) (non-transposed A only), of C and of D is physical row
  // map[m]. Used by the inversion sweep to fold the panel's row interchanges
  // into the update instead of moving rows.
  const int* rowmap_a;
  const int* rowmap_c;
  const int* rowmap_d;
  long long s_map;
};

constexpr int kMaxGroup = 6;
struct ZGemmGroup {
  int n;
  ZGemmDesc d[kMaxGroup];
};

// Host-side helpers -----------------------------------------------------------
inline ZGemmDesc zdesc_default() {
  ZGemmDesc d;
  d.M = d.N = d.batch = 0; d.nterms = 1;
  d.alpha = make_double2(1.0, 0.0); d.beta = make_double2(0.0, 0.0);
  d.C = nullptr; d.sC = 0; d.ldc = 0;
  d.D = nullptr; d.sD = 0; d.ldd = 0;
  d.transD = 0; d.herm = 0; d.active = nullptr;
  d.rowmap_a = d.rowmap_c = d.rowmap_d = nullptr;
  d.s_map = 0;
  return d;
}

inline ZTerm zterm(const z_t* A, long long sA, int lda, int opA, const z_t* B, long long sB,
                   int ldb, int opB, int K, bool neg = false, bool real_operand = false) {
  ZTerm t;
  t.A = A; t.sA = sA; t.lda = lda; t.opA = opA;
  t.B = B; t.sB = sB; t.ldb = ldb; t.opB = opB;
  t.K = K; t.neg = (neg ? 1 : 0) | (real_operand ? kTermReal : 0);
  return t;
}

// Launch a group of GEMM problems (same tile config) on `stream`.
int zgemm_group_launch(const ZGemmGroup& g, cudaStream_t stream);
int gemm_algo();
void set_gemm_algo(int a);
int zgemm_launch(const ZGemmDesc& d, cudaStream_t stream);

// Streamed Gauss-Jordan sweep of the blocked inverse (zinv.cu): rows m < n - wd
// outside the pivot rows K, A_new[dst(m), :] = C - A_old[src(m), K] A_new[K, :]
// with C = A_old[src(m), :] outside the columns K and 0 on them.
struct SweepArgs {
  const z_t* cur;
  long long cs;
  z_t* nxt;
  long long ns;
  int n, k0, wd;
  const int* map_src;  // [batch][n]
  const int* map_dst;  // [batch][n]
  const int* active;   // optional per-matrix mask
  int ng;              // column groups (set by the launcher)
  // fused mode (one-CTA panels): T = Pinv R is formed here, not by the panel
  const z_t* pinv;     // [batch][wd][wd]
  const int* prow;     // [batch][32] A_old row of pivot q (nullptr: T already in A_new rows K)
};
int zinv_sweep_launch(const SweepArgs& a, int batch, cudaStream_t stream);

}  // namespace negf
