// Batched grouped complex-FP64 DMMA GEMM (see zgemm.cuh for the contract).
#include "prof.cuh"
#include "zgemm.cuh"

namespace negf {

namespace {

constexpr unsigned long long kSign = 0x8000000000000000ull;

template <int BM_, int BN_, int WM_, int WN_, int STAGES_, int MINB_, bool GAUSS_ = false, int BK_ = 8,
          bool ROWMAP_ = false, bool SWZ_ = false>
struct Cfg {
  static constexpr bool ROWMAP = ROWMAP_;  // honour ZGemmDesc row maps (inversion sweeps only)
  // SWZ: k-contiguous tiles unpadded, element (mn, k) at mn*BK + (k ^ 4*(mn&1))
  // (XOR swizzle instead of the +4 pad: same conflict-free fragment reads,
  // a third less shared memory at BK = 8, a fifth at BK = 16)
  static constexpr bool SWZ = SWZ_;
  static constexpr int BM = BM_, BN = BN_, WM = WM_, WN = WN_, STAGES = STAGES_, MINB = MINB_;
  // GAUSS: 3 real products per complex product (3M / Gauss):
  //   P1 = ar br, P2 = ai bi, P3 = (ar + ai)(br + bi);  re = P1 - P2, im = P3 - P1 - P2
  static constexpr bool GAUSS = GAUSS_;
  static constexpr int BK = BK_;
  static constexpr int NT = WM * WN * 32;
  static constexpr int WTM = BM / WM;  // warp tile rows
  static constexpr int WTN = BN / WN;
  static constexpr int TM = WTM / 8;  // 8x8 DMMA tiles per warp
  static constexpr int TN = WTN / 8;
  static constexpr int SK = SWZ ? BK : BK + 4;  // k-contiguous row stride
  static constexpr int SMA = BM + 2;  // mn-contiguous row stride (A)
  static constexpr int SMB = BN + 2;  // mn-contiguous row stride (B)
  static constexpr int A_ELEMS = (BM * SK > BK * SMA) ? BM * SK : BK * SMA;
  static constexpr int B_ELEMS = (BN * SK > BK * SMB) ? BN * SK : BK * SMB;
  static constexpr int STAGE_ELEMS = A_ELEMS + B_ELEMS;
  static constexpr size_t SMEM = (size_t)STAGES * STAGE_ELEMS * sizeof(z_t);
};

// Stage one BK-slice of both operands into shared memory with cp.async.
struct KtBounds {
  int b1, b2, b3;  // cumulative k-tile counts after terms 0, 1, 2 (clamped to the total)
  __device__ __forceinline__ int term(int kt) const {
    return (kt >= b1) + (kt >= b2) + (kt >= b3);
  }
  __device__ __forceinline__ int base(int term) const {
    return term == 0 ? 0 : term == 1 ? b1 : term == 2 ? b2 : b3;
  }
};

// k-contiguous smem index of (mn, k)
template <class CF>
__device__ __forceinline__ int kc_idx(int mn, int k) {
  if constexpr (CF::SWZ) return mn * CF::SK + (k ^ ((mn & 1) << 2));
  else return mn * CF::SK + k;
}

template <class CF>
__device__ __forceinline__ void load_stage(const ZGemmDesc& d, int kt, const KtBounds& kb, int b,
                                           int m0, int n0, z_t* sA, z_t* sB) {
  const int term = kb.term(kt);
  const ZTerm& t = d.t[term];
  const int k0 = (kt - kb.base(term)) * CF::BK;
  const z_t* A = t.A + (long long)b * t.sA;
  const z_t* B = t.B + (long long)b * t.sB;
  const int K = t.K, M = d.M, N = d.N;
  if (!op_trans(t.opA)) {  // A stored [M][K]: k contiguous
#pragma unroll
    for (int e = threadIdx.x; e < CF::BM * CF::BK; e += CF::NT) {
      int mn = e / CF::BK, k = e % CF::BK;
      int gm = m0 + mn, gk = k0 + k;
      bool p = gm < M && gk < K;
      int pm = gm;
      if constexpr (CF::ROWMAP)
        if (p && d.rowmap_a) pm = d.rowmap_a[(long long)b * d.s_map + gm];
      const z_t* src = p ? A + (long long)pm * t.lda + gk : A;
      cp_async16(sA + kc_idx<CF>(mn, k), src, p);
    }
  } else {  // A stored [K][M]: m contiguous
#pragma unroll
    for (int e = threadIdx.x; e < CF::BM * CF::BK; e += CF::NT) {
      int mn = e % CF::BM, k = e / CF::BM;
      int gm = m0 + mn, gk = k0 + k;
      bool p = gm < M && gk < K;
      const z_t* src = p ? A + (long long)gk * t.lda + gm : A;
      cp_async16(sA + k * CF::SMA + mn, src, p);
    }
  }
  if (!op_trans(t.opB)) {  // B stored [K][N]: n contiguous
#pragma unroll
    for (int e = threadIdx.x; e < CF::BN * CF::BK; e += CF::NT) {
      int mn = e % CF::BN, k = e / CF::BN;
      int gn = n0 + mn, gk = k0 + k;
      bool p = gn < N && gk < K;
      const z_t* src = p ? B + (long long)gk * t.ldb + gn : B;
      cp_async16(sB + k * CF::SMB + mn, src, p);
    }
  } else {  // B stored [N][K]: k contiguous
#pragma unroll
    for (int e = threadIdx.x; e < CF::BN * CF::BK; e += CF::NT) {
      int mn = e / CF::BK, k = e % CF::BK;
      int gn = n0 + mn, gk = k0 + k;
      bool p = gn < N && gk < K;
      const z_t* src = p ? B + (long long)gn * t.ldb + gk : B;
      cp_async16(sB + kc_idx<CF>(mn, k), src, p);
    }
  }
}

// One k4 step of the 3M product on a warp tile of TM x TN 8x8 DMMA tiles:
// acc_re += ar br, acc_im += ai bi (skipped for a real operand), acc_s +=
// (ar+ai)(br+bi). ORD (4 x 2 tiles): the 24 DMMAs issue in an order in which
// consecutive DMMAs share neither operand register (volatile: kept by the
// compiler; +1.5 % for the cp.async kernel at 256^3 / 512^3, -1.2 % for the
// bulk-copy kernel, which keeps the compiler's order).
template <int TM, int TN, bool RV, bool ORD = true>
__device__ __forceinline__ void mma3m_step(double (&acc_re)[TM][TN][2], double (&acc_im)[TM][TN][2],
                                           double (&acc_s)[TM][TN][2], const double* ar, const double* ai,
                                           const double* as, const double* br, const double* bi, const double* bs) {
  if constexpr (ORD && TM == 4 && TN == 2) {
    constexpr int oi[8] = {0, 1, 2, 3, 1, 0, 3, 2}, oj[8] = {0, 1, 0, 1, 0, 1, 0, 1};
#pragma unroll
    for (int x = 0; x < 8; ++x) dmma_v(acc_re[oi[x]][oj[x]][0], acc_re[oi[x]][oj[x]][1], ar[oi[x]], br[oj[x]]);
    if constexpr (!RV) {
#pragma unroll
      for (int x = 0; x < 8; ++x) dmma_v(acc_im[oi[x]][oj[x]][0], acc_im[oi[x]][oj[x]][1], ai[oi[x]], bi[oj[x]]);
    }
#pragma unroll
    for (int x = 0; x < 8; ++x) dmma_v(acc_s[oi[x]][oj[x]][0], acc_s[oi[x]][oj[x]][1], as[oi[x]], bs[oj[x]]);
  } else {
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
      for (int j = 0; j < TN; ++j) dmma_m8n8k4(acc_re[i][j][0], acc_re[i][j][1], ar[i], br[j]);
    if constexpr (!RV) {
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) dmma_m8n8k4(acc_im[i][j][0], acc_im[i][j][1], ai[i], bi[j]);
    }
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
      for (int j = 0; j < TN; ++j) dmma_m8n8k4(acc_s[i][j][0], acc_s[i][j][1], as[i], bs[j]);
  }
}

// One BK stage of the 3M product for fixed operand layouts (AKC: A tile
// k-contiguous, BKC: B tile k-contiguous). With XOR-swizzled k-contiguous
// tiles, step k4 of a row of parity p reads k-chunk k4 ^ p: two per-thread
// bases (even / odd k4) plus compile-time offsets.
template <class CF, bool RV, bool AKC, bool BKC>
__device__ __forceinline__ void gauss_stage(const z_t* __restrict__ sA, const z_t* __restrict__ sB,
                                            double (&acc_re)[CF::TM][CF::TN][2], double (&acc_im)[CF::TM][CF::TN][2],
                                            double (&acc_s)[CF::GAUSS ? CF::TM : 1][CF::GAUSS ? CF::TN : 1][2],
                                            unsigned long long negm, unsigned long long conjA,
                                            unsigned long long conjB, int wm, int wn, int lane) {
  const int r = lane >> 2, q = lane & 3, p = CF::SWZ ? (r & 1) : 0;
  // per-thread bases for even and odd k4 (k-contiguous) or one base (mn-contiguous)
  const z_t* a0;
  const z_t* a1;
  const z_t* b0;
  const z_t* b1;
  if constexpr (AKC) {
    const z_t* row = sA + (wm * CF::WTM + r) * CF::SK;
    a0 = row + 4 * p + q;
    a1 = row + 4 * (1 - p) + q;
  } else {
    a0 = a1 = sA + q * CF::SMA + wm * CF::WTM + r;
  }
  if constexpr (BKC) {
    const z_t* row = sB + (wn * CF::WTN + r) * CF::SK;
    b0 = row + 4 * p + q;
    b1 = row + 4 * (1 - p) + q;
  } else {
    b0 = b1 = sB + q * CF::SMB + wn * CF::WTN + r;
  }
#pragma unroll
  for (int k4 = 0; k4 < CF::BK / 4; ++k4) {
    const z_t* pa = (k4 & 1) ? a1 : a0;
    const z_t* pb = (k4 & 1) ? b1 : b0;
    double ar[CF::TM], ai[CF::TM], as[CF::TM], br[CF::TN], bi[CF::TN], bs[CF::TN];
#pragma unroll
    for (int i = 0; i < CF::TM; ++i) {
      const z_t v = AKC ? pa[i * 8 * CF::SK + (k4 >> 1) * 8] : pa[k4 * 4 * CF::SMA + i * 8];
      ar[i] = dneg_if(v.x, negm);
      ai[i] = dneg_if(v.y, negm ^ conjA);
      as[i] = ar[i] + ai[i];
    }
#pragma unroll
    for (int j = 0; j < CF::TN; ++j) {
      const z_t v = BKC ? pb[j * 8 * CF::SK + (k4 >> 1) * 8] : pb[k4 * 4 * CF::SMB + j * 8];
      br[j] = v.x;
      bi[j] = dneg_if(v.y, conjB);
      bs[j] = br[j] + bi[j];
    }
    mma3m_step<CF::TM, CF::TN, RV>(acc_re, acc_im, acc_s, ar, ai, as, br, bi, bs);
  }
}

// RV: every term of the group has a real operand (kTermReal), so the 3M
// product ai*bi vanishes and is not issued (2 DMMA products per complex one).
template <class CF, bool RV = false>
__global__ void __launch_bounds__(CF::NT, CF::MINB) zgemm_kernel(const __grid_constant__ ZGemmGroup grp) {
  extern __shared__ __align__(16) z_t smem[];
  const ZGemmDesc& d = grp.d[blockIdx.z];
  const int tiles_n = (d.N + CF::BN - 1) / CF::BN;
  const int tiles_m = (d.M + CF::BM - 1) / CF::BM;
  if ((int)blockIdx.x >= tiles_m * tiles_n || (int)blockIdx.y >= d.batch) return;
  if (d.active && !d.active[blockIdx.y]) return;
  const int b = blockIdx.y;
  const int m0 = (blockIdx.x / tiles_n) * CF::BM;
  const int n0 = (blockIdx.x % tiles_n) * CF::BN;
  if (d.herm && n0 >= m0 + CF::BM) return;  // strictly above the diagonal: mirrored by the lower tiles
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int wm = warp / CF::WN, wn = warp % CF::WN;

  KtBounds kb;
  {
    auto nk = [&](int i) { return i < d.nterms ? (d.t[i].K + CF::BK - 1) / CF::BK : 0; };
    kb.b1 = nk(0);
    kb.b2 = kb.b1 + nk(1);
    kb.b3 = kb.b2 + nk(2);
  }
  const int KT = kb.b3 + (d.nterms > 3 ? (d.t[3].K + CF::BK - 1) / CF::BK : 0);
  // terms past nterms have zero tiles, so their bounds equal KT and are never reached

  double acc_re[CF::TM][CF::TN][2], acc_im[CF::TM][CF::TN][2];
  double acc_s[CF::GAUSS ? CF::TM : 1][CF::GAUSS ? CF::TN : 1][2];
#pragma unroll
  for (int i = 0; i < CF::TM; ++i)
#pragma unroll
    for (int j = 0; j < CF::TN; ++j) {
      acc_re[i][j][0] = acc_re[i][j][1] = 0.0;
      acc_im[i][j][0] = acc_im[i][j][1] = 0.0;
      if constexpr (CF::GAUSS) acc_s[i][j][0] = acc_s[i][j][1] = 0.0;
    }

  auto stageA = [&](int s) { return smem + s * CF::STAGE_ELEMS; };
  auto stageB = [&](int s) { return smem + s * CF::STAGE_ELEMS + CF::A_ELEMS; };

#pragma unroll
  for (int s = 0; s < CF::STAGES - 1; ++s) {
    if (s < KT) load_stage<CF>(d, s, kb, b, m0, n0, stageA(s), stageB(s));
    cp_async_commit();
  }

  // Epilogue operands: this thread's C fragment (and its row maps) are loaded
  // as one batch of independent loads -- for the short-K row-mapped sweeps
  // before the main loop, so their latency hides behind it; otherwise after.
  const double2 al = d.alpha, be = d.beta;
  const bool use_c = d.C != nullptr && (be.x != 0.0 || be.y != 0.0);
  const z_t* C = use_c ? d.C + (long long)b * d.sC : nullptr;
  const int er = lane >> 2, eq = lane & 3;
  // The row maps are read before the main loop. C is read in the epilogue one
  // fragment row (2*TN independent loads) at a time -- or, for 4M row-mapped
  // configs, as a whole fragment before the main loop (measured slower for
  // the inversion sweeps: 255 registers, 2 CTAs/SM; kept for experiments).
  constexpr bool PREC = CF::ROWMAP && !CF::GAUSS;
  constexpr int CI = PREC ? CF::TM : 1;
  int crow[CF::TM], drow[CF::TM];
  z_t cfrag[CI][CF::TN][2];
  auto map_rows = [&]() {
#pragma unroll
    for (int i = 0; i < CF::TM; ++i) {
      const int gm = m0 + wm * CF::WTM + i * 8 + er;
      crow[i] = drow[i] = gm;
      if constexpr (CF::ROWMAP) {
        if (gm < d.M) {
          if (d.rowmap_c) crow[i] = d.rowmap_c[(long long)b * d.s_map + gm];
          if (d.rowmap_d) drow[i] = d.rowmap_d[(long long)b * d.s_map + gm];
        }
      }
    }
  };
  auto load_c_row = [&](int i, int slot) {
    const int gm = m0 + wm * CF::WTM + i * 8 + er;
#pragma unroll
    for (int j = 0; j < CF::TN; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int gn = n0 + wn * CF::WTN + j * 8 + 2 * eq + h;
        cfrag[slot][j][h] = (use_c && gm < d.M && gn < d.N) ? C[(long long)crow[i] * d.ldc + gn]
                                                            : make_double2(0.0, 0.0);
      }
  };
  map_rows();
  if constexpr (PREC) {
#pragma unroll
    for (int i = 0; i < CF::TM; ++i) load_c_row(i, i);
  }

  for (int kt = 0; kt < KT; ++kt) {
    cp_async_wait<CF::STAGES - 2>();
    __syncthreads();
    {
      int nk = kt + CF::STAGES - 1;
      if (nk < KT) {
        int s = nk % CF::STAGES;
        load_stage<CF>(d, nk, kb, b, m0, n0, stageA(s), stageB(s));
      }
      cp_async_commit();
    }
    const int s = kt % CF::STAGES;
    const z_t* sA = stageA(s);
    const z_t* sB = stageB(s);
    const ZTerm& t = d.t[kb.term(kt)];
    const bool a_kc = !op_trans(t.opA);
    const bool b_kc = op_trans(t.opB);
    const unsigned long long negm = (t.neg & 1) ? kSign : 0ull;
    const unsigned long long conjA = op_conj(t.opA) ? kSign : 0ull;
    const unsigned long long conjB = op_conj(t.opB) ? kSign : 0ull;
    // fragment addressing: element (mn, k) at mn*s_mn + k*s_k
    const int a_smn = a_kc ? CF::SK : 1, a_sk = a_kc ? 1 : CF::SMA;
    const int b_smn = b_kc ? CF::SK : 1, b_sk = b_kc ? 1 : CF::SMB;
    const int r = lane >> 2, q = lane & 3;
    // operand fragments of one k4 step (raw complex values from smem)
    auto fetch = [&](int k4, z_t* fa, z_t* fb) {
      const int kk = k4 * 4 + q;
      // k-contiguous reads: row parity of (.. + r) is r&1 (row bases are multiples of 8)
      const int kka = (CF::SWZ && a_kc) ? (kk ^ ((r & 1) << 2)) : kk;
      const int kkb = (CF::SWZ && b_kc) ? (kk ^ ((r & 1) << 2)) : kk;
#pragma unroll
      for (int i = 0; i < CF::TM; ++i) fa[i] = sA[(wm * CF::WTM + i * 8 + r) * a_smn + kka * a_sk];
#pragma unroll
      for (int j = 0; j < CF::TN; ++j) fb[j] = sB[(wn * CF::WTN + j * 8 + r) * b_smn + kkb * b_sk];
    };
    if constexpr (CF::GAUSS) {
      // the stage's layouts are uniform: dispatch to a copy of the 3M step
      // with compile-time fragment strides (LDS with immediate offsets instead
      // of per-fragment IMAD/LEA address arithmetic)
      const int sel = (a_kc ? 1 : 0) | (b_kc ? 2 : 0);
      if (sel == 0) gauss_stage<CF, RV, false, false>(sA, sB, acc_re, acc_im, acc_s, negm, conjA, conjB, wm, wn, lane);
      else if (sel == 1) gauss_stage<CF, RV, true, false>(sA, sB, acc_re, acc_im, acc_s, negm, conjA, conjB, wm, wn, lane);
      else if (sel == 2) gauss_stage<CF, RV, false, true>(sA, sB, acc_re, acc_im, acc_s, negm, conjA, conjB, wm, wn, lane);
      else gauss_stage<CF, RV, true, true>(sA, sB, acc_re, acc_im, acc_s, negm, conjA, conjB, wm, wn, lane);
    } else {
      // 4M (algo 0): the textbook four real products per complex one
#pragma unroll
      for (int k4 = 0; k4 < CF::BK / 4; ++k4) {
        z_t va[CF::TM], vb[CF::TN];
        fetch(k4, va, vb);
        double ar[CF::TM], ai[CF::TM], nai[CF::TM], br[CF::TN], bi[CF::TN];
#pragma unroll
        for (int i = 0; i < CF::TM; ++i) {
          ar[i] = dneg_if(va[i].x, negm);
          ai[i] = dneg_if(va[i].y, negm ^ conjA);
          nai[i] = dneg_if(ai[i], kSign);
        }
#pragma unroll
        for (int j = 0; j < CF::TN; ++j) {
          br[j] = vb[j].x;
          bi[j] = dneg_if(vb[j].y, conjB);
        }
        // Phase-major issue order: the two DMMAs feeding the same accumulator
        // are TM*TN*2 instructions apart, so the FP64 tensor pipe never waits
        // on its own accumulation dependency.
#pragma unroll
        for (int i = 0; i < CF::TM; ++i)
#pragma unroll
          for (int j = 0; j < CF::TN; ++j) {
            dmma_m8n8k4(acc_re[i][j][0], acc_re[i][j][1], ar[i], br[j]);
            dmma_m8n8k4(acc_im[i][j][0], acc_im[i][j][1], ar[i], bi[j]);
          }
#pragma unroll
        for (int i = 0; i < CF::TM; ++i)
#pragma unroll
          for (int j = 0; j < CF::TN; ++j) {
            dmma_m8n8k4(acc_re[i][j][0], acc_re[i][j][1], nai[i], bi[j]);
            dmma_m8n8k4(acc_im[i][j][0], acc_im[i][j][1], ai[i], br[j]);
          }
      }
    }
  }
  cp_async_wait<0>();

  // Epilogue: value = alpha*acc + beta*C, stored plain or conj-transposed.
  z_t* D = d.D + (long long)b * d.sD;
#pragma unroll
  for (int i = 0; i < CF::TM; ++i) {
    if constexpr (!PREC) load_c_row(i, 0);
#pragma unroll
    for (int j = 0; j < CF::TN; ++j) {
      const int gm = m0 + wm * CF::WTM + i * 8 + er;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int gn = n0 + wn * CF::WTN + j * 8 + 2 * eq + h;
        if (gm < d.M && gn < d.N) {
          double xr = acc_re[i][j][h], xi = acc_im[i][j][h];
          if constexpr (CF::GAUSS) {
            const double p1 = xr, p2 = xi;
            xr = p1 - p2;
            xi = acc_s[i][j][h] - p1 - p2;
          }
          z_t v = zmake(al.x * xr - al.y * xi, al.x * xi + al.y * xr);
          const z_t c = cfrag[PREC ? i : 0][j][h];
          v.x += be.x * c.x - be.y * c.y;
          v.y += be.x * c.y + be.y * c.x;
          if (d.herm) {  // lower triangle + mirror; the diagonal projected to i Im v
            if (gm > gn) {
              D[(long long)gm * d.ldd + gn] = v;
              D[(long long)gn * d.ldd + gm] = zmake(-v.x, v.y);
            } else if (gm == gn) {
              D[(long long)gm * d.ldd + gn] = zmake(0.0, v.y);
            }
          } else if (d.transD)
            D[(long long)gn * d.ldd + gm] = zconj(v);
          else
            D[(long long)drow[i] * d.ldd + gn] = v;
        }
      }
    }
  }
}

template <class CF, bool RV = false>
int launch_cfg(const ZGemmGroup& g, cudaStream_t stream) {
  // cudaFuncSetAttribute applies to the current device's context: once per device
  static unsigned long long attr_done = 0;
  int dev = 0;
  NEGF_CUDA_CHECK(cudaGetDevice(&dev));
  if (dev >= 64) return -1;
  if (!(__atomic_load_n(&attr_done, __ATOMIC_ACQUIRE) & (1ull << dev))) {
    NEGF_CUDA_CHECK(cudaFuncSetAttribute(zgemm_kernel<CF, RV>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)CF::SMEM));
    __atomic_fetch_or(&attr_done, 1ull << dev, __ATOMIC_RELEASE);
  }
  int max_tiles = 0, max_batch = 0;
  for (int i = 0; i < g.n; ++i) {
    int tm = (g.d[i].M + CF::BM - 1) / CF::BM, tn = (g.d[i].N + CF::BN - 1) / CF::BN;
    if (tm * tn > max_tiles) max_tiles = tm * tn;
    if (g.d[i].batch > max_batch) max_batch = g.d[i].batch;
  }
  if (max_tiles == 0 || max_batch == 0) return 0;
  dim3 grid(max_tiles, max_batch, g.n);
  int maxk = 0;
  for (int i = 0; i < g.n; ++i)
    for (int t = 0; t < g.d[i].nterms; ++t) maxk = g.d[i].t[t].K > maxk ? g.d[i].t[t].K : maxk;
  const int tok = prof_begin(maxk <= 32 ? PROF_ZGEMM_SMALLK : PROF_ZGEMM, stream);
  zgemm_kernel<CF, RV><<<grid, CF::NT, CF::SMEM, stream>>>(g);
  NEGF_LAUNCHED();
  if (tok >= 0) {
    double fl = 0.0, by = 0.0;
    for (int i = 0; i < g.n; ++i) {
      const ZGemmDesc& d = g.d[i];
      for (int t = 0; t < d.nterms; ++t) {
        fl += 8.0 * d.M * d.N * (double)d.t[t].K * d.batch;
        by += 16.0 * ((double)d.M * d.t[t].K + (double)d.t[t].K * d.N) * d.batch;
      }
      by += 16.0 * (double)d.M * d.N * d.batch * ((d.C && (d.beta.x != 0.0 || d.beta.y != 0.0)) ? 2 : 1);
    }
    prof_end(tok, stream, fl, by);
  }
  return 0;
}

// ---------------------------------------------------------------------------
// Warp-specialised variant: operand tiles move global -> smem on the TMA
// engine (cp.async.bulk, one bulk copy per contiguous tile row, completion
// counted in bytes on an mbarrier) through a STAGES-deep ring of
// full / empty mbarriers: one producer warp arms and issues the copies, the
// 4 consumer warps wait on "full", run the DMMA step, and release the slot on
// "empty" -- no __syncthreads and no per-thread LDGSTS address streams in the
// main loop. Bulk copies land rows contiguously, so the k-contiguous tiles use
// the +4 pad (conflict-free fragment reads) instead of the XOR swizzle.
// Row-mapped problems (inversion sweeps) stay on the cp.async kernel.
template <int BM_, int BN_, int BK_, int STAGES_, int MINB_, int WM_ = 2, int WN_ = 2>
struct BulkCfg {
  static constexpr int BM = BM_, BN = BN_, BK = BK_, STAGES = STAGES_, MINB = MINB_;
  static constexpr int WM = WM_, WN = WN_, NCW = WM * WN;  // consumer warps
  static constexpr int NT = (NCW + 1) * 32;            // + one producer warp
  static constexpr int WTM = BM / WM, WTN = BN / WN, TM = WTM / 8, TN = WTN / 8;
  static constexpr int SK = BK + 4, SMA = BM + 2, SMB = BN + 2;
  static constexpr int A_ELEMS = (BM * SK > BK * SMA) ? BM * SK : BK * SMA;
  static constexpr int B_ELEMS = (BN * SK > BK * SMB) ? BN * SK : BK * SMB;
  static constexpr int STAGE_ELEMS = A_ELEMS + B_ELEMS;
  static constexpr size_t SMEM = (size_t)STAGES * STAGE_ELEMS * sizeof(z_t) + 2 * STAGES * sizeof(unsigned long long);
};

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(unsigned long long* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned parity) {
  unsigned done = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
        "selp.b32 %0, 1, 0, P1;\n\t}"
        : "=r"(done)
        : "r"(smem_u32(b)), "r"(parity)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// Producer side of one stage: every tile row of A and B as a bulk copy.
template <class CF>
__device__ __forceinline__ void bulk_stage(const ZGemmDesc& d, int kt, const KtBounds& kb, int b, int m0, int n0,
                                           z_t* sA, z_t* sB, unsigned long long* full, int lane) {
  const int term = kb.term(kt);
  const ZTerm& t = d.t[term];
  const int k0 = (kt - kb.base(term)) * CF::BK;
  const z_t* A = t.A + (long long)b * t.sA;
  const z_t* B = t.B + (long long)b * t.sB;
  const int K = t.K, M = d.M, N = d.N;
  const int vk = K - k0 < CF::BK ? K - k0 : CF::BK;
  // zero tails first (generic stores), then arm the barrier, then the copies
  auto rows = [&](auto&& fn) {  // fn(dst, src, cnt, len) for every row of both operands
    if (!op_trans(t.opA)) {  // [M][K]: BM rows of BK
      for (int r = lane; r < CF::BM; r += 32) {
        const int gm = m0 + r;
        fn(sA + r * CF::SK, A + (long long)gm * t.lda + k0, gm < M ? vk : 0, CF::BK);
      }
    } else {  // [K][M]: BK rows of BM
      const int vm = M - m0 < CF::BM ? M - m0 : CF::BM;
      for (int r = lane; r < CF::BK; r += 32) {
        const int gk = k0 + r;
        fn(sA + r * CF::SMA, A + (long long)gk * t.lda + m0, gk < K ? vm : 0, CF::BM);
      }
    }
    if (!op_trans(t.opB)) {  // [K][N]: BK rows of BN
      const int vn = N - n0 < CF::BN ? N - n0 : CF::BN;
      for (int r = lane; r < CF::BK; r += 32) {
        const int gk = k0 + r;
        fn(sB + r * CF::SMB, B + (long long)gk * t.ldb + n0, gk < K ? vn : 0, CF::BN);
      }
    } else {  // [N][K]: BN rows of BK
      for (int r = lane; r < CF::BN; r += 32) {
        const int gn = n0 + r;
        fn(sB + r * CF::SK, B + (long long)gn * t.ldb + k0, gn < N ? vk : 0, CF::BK);
      }
    }
  };
  unsigned bytes = 0;
  rows([&](z_t* dst, const z_t*, int cnt, int len) {
    for (int e = cnt > 0 ? cnt : 0; e < len; ++e) dst[e] = make_double2(0.0, 0.0);
    bytes += cnt > 0 ? (unsigned)cnt * 16u : 0u;
  });
  bytes = __reduce_add_sync(0xffffffffu, bytes);
  __syncwarp();
  if (lane == 0) mbar_arrive_tx(full, bytes);
  __syncwarp();
  rows([&](z_t* dst, const z_t* src, int cnt, int) {
    if (cnt > 0) bulk_g2s(dst, src, (unsigned)cnt * 16u, full);
  });
}

template <class CF, bool RV = false>
__global__ void __launch_bounds__(CF::NT, CF::MINB) zgemm_bulk_kernel(const __grid_constant__ ZGemmGroup grp) {
  extern __shared__ __align__(16) z_t smem[];
  const ZGemmDesc& d = grp.d[blockIdx.z];
  const int tiles_n = (d.N + CF::BN - 1) / CF::BN;
  const int tiles_m = (d.M + CF::BM - 1) / CF::BM;
  if ((int)blockIdx.x >= tiles_m * tiles_n || (int)blockIdx.y >= d.batch) return;
  if (d.active && !d.active[blockIdx.y]) return;
  const int b = blockIdx.y;
  const int m0 = (blockIdx.x / tiles_n) * CF::BM;
  const int n0 = (blockIdx.x % tiles_n) * CF::BN;
  if (d.herm && n0 >= m0 + CF::BM) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned long long* full = reinterpret_cast<unsigned long long*>(smem + CF::STAGES * CF::STAGE_ELEMS);
  unsigned long long* empty = full + CF::STAGES;
  if (threadIdx.x == 0) {
    for (int s = 0; s < CF::STAGES; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, CF::NCW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  KtBounds kb;
  {
    auto nk = [&](int i) { return i < d.nterms ? (d.t[i].K + CF::BK - 1) / CF::BK : 0; };
    kb.b1 = nk(0);
    kb.b2 = kb.b1 + nk(1);
    kb.b3 = kb.b2 + nk(2);
  }
  const int KT = kb.b3 + (d.nterms > 3 ? (d.t[3].K + CF::BK - 1) / CF::BK : 0);
  auto stageA = [&](int s) { return smem + s * CF::STAGE_ELEMS; };
  auto stageB = [&](int s) { return smem + s * CF::STAGE_ELEMS + CF::A_ELEMS; };

  if (warp == CF::NCW) {  // producer warp
    for (int kt = 0; kt < KT; ++kt) {
      const int s = kt % CF::STAGES, u = kt / CF::STAGES;
      if (u > 0) mbar_wait(empty + s, (u - 1) & 1);
      bulk_stage<CF>(d, kt, kb, b, m0, n0, stageA(s), stageB(s), full + s, lane);
    }
    return;
  }

  const int wm = warp / CF::WN, wn = warp % CF::WN;
  double acc_re[CF::TM][CF::TN][2], acc_im[CF::TM][CF::TN][2], acc_s[CF::TM][CF::TN][2];
#pragma unroll
  for (int i = 0; i < CF::TM; ++i)
#pragma unroll
    for (int j = 0; j < CF::TN; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) acc_re[i][j][h] = acc_im[i][j][h] = acc_s[i][j][h] = 0.0;
  const int r = lane >> 2, q = lane & 3;
  for (int kt = 0; kt < KT; ++kt) {
    const int s = kt % CF::STAGES;
    mbar_wait(full + s, (kt / CF::STAGES) & 1);
    const z_t* sA = stageA(s);
    const z_t* sB = stageB(s);
    const ZTerm& t = d.t[kb.term(kt)];
    const bool a_kc = !op_trans(t.opA);
    const bool b_kc = op_trans(t.opB);
    const unsigned long long negm = (t.neg & 1) ? kSign : 0ull;
    const unsigned long long conjA = op_conj(t.opA) ? kSign : 0ull;
    const unsigned long long conjB = op_conj(t.opB) ? kSign : 0ull;
    const int a_smn = a_kc ? CF::SK : 1, a_sk = a_kc ? 1 : CF::SMA;
    const int b_smn = b_kc ? CF::SK : 1, b_sk = b_kc ? 1 : CF::SMB;
#pragma unroll
    for (int k4 = 0; k4 < CF::BK / 4; ++k4) {
      const int kk = k4 * 4 + q;
      double ar[CF::TM], ai[CF::TM], br[CF::TN], bi[CF::TN], as[CF::TM], bsum[CF::TN];
#pragma unroll
      for (int i = 0; i < CF::TM; ++i) {
        const z_t v = sA[(wm * CF::WTM + i * 8 + r) * a_smn + kk * a_sk];
        ar[i] = dneg_if(v.x, negm);
        ai[i] = dneg_if(v.y, negm ^ conjA);
        as[i] = ar[i] + ai[i];
      }
#pragma unroll
      for (int j = 0; j < CF::TN; ++j) {
        const z_t v = sB[(wn * CF::WTN + j * 8 + r) * b_smn + kk * b_sk];
        br[j] = v.x;
        bi[j] = dneg_if(v.y, conjB);
        bsum[j] = br[j] + bi[j];
      }
      // 3M: acc_re <- ar br, acc_im <- ai bi, acc_s <- (ar+ai)(br+bi)
      mma3m_step<CF::TM, CF::TN, RV, false>(acc_re, acc_im, acc_s, ar, ai, as, br, bi, bsum);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(empty + s);
  }

  // Epilogue: value = alpha*acc + beta*C, stored plain or conj-transposed.
  const double2 al = d.alpha, be = d.beta;
  const bool use_c = d.C != nullptr && (be.x != 0.0 || be.y != 0.0);
  const z_t* C = use_c ? d.C + (long long)b * d.sC : nullptr;
  z_t* D = d.D + (long long)b * d.sD;
  const int er = lane >> 2, eq = lane & 3;
#pragma unroll
  for (int i = 0; i < CF::TM; ++i) {
    const int gm = m0 + wm * CF::WTM + i * 8 + er;
    z_t cv[CF::TN][2];
#pragma unroll
    for (int j = 0; j < CF::TN; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int gn = n0 + wn * CF::WTN + j * 8 + 2 * eq + h;
        cv[j][h] = (use_c && gm < d.M && gn < d.N) ? C[(long long)gm * d.ldc + gn] : make_double2(0.0, 0.0);
      }
#pragma unroll
    for (int j = 0; j < CF::TN; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int gn = n0 + wn * CF::WTN + j * 8 + 2 * eq + h;
        if (gm < d.M && gn < d.N) {
          const double p1 = acc_re[i][j][h], p2 = acc_im[i][j][h];
          const double xr = p1 - p2, xi = acc_s[i][j][h] - p1 - p2;
          z_t v = zmake(al.x * xr - al.y * xi, al.x * xi + al.y * xr);
          const z_t c = cv[j][h];
          v.x += be.x * c.x - be.y * c.y;
          v.y += be.x * c.y + be.y * c.x;
          if (d.herm) {  // lower triangle + mirror; the diagonal projected to i Im v
            if (gm > gn) {
              D[(long long)gm * d.ldd + gn] = v;
              D[(long long)gn * d.ldd + gm] = zmake(-v.x, v.y);
            } else if (gm == gn) {
              D[(long long)gm * d.ldd + gn] = zmake(0.0, v.y);
            }
          } else if (d.transD)
            D[(long long)gn * d.ldd + gm] = zconj(v);
          else
            D[(long long)gm * d.ldd + gn] = v;
        }
      }
  }
}

template <class CF, bool RV = false>
int launch_bulk(const ZGemmGroup& g, cudaStream_t stream) {
  static unsigned long long attr_done = 0;
  int dev = 0;
  NEGF_CUDA_CHECK(cudaGetDevice(&dev));
  if (dev >= 64) return -1;
  if (!(__atomic_load_n(&attr_done, __ATOMIC_ACQUIRE) & (1ull << dev))) {
    NEGF_CUDA_CHECK(cudaFuncSetAttribute(zgemm_bulk_kernel<CF, RV>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)CF::SMEM));
    __atomic_fetch_or(&attr_done, 1ull << dev, __ATOMIC_RELEASE);
  }
  int max_tiles = 0, max_batch = 0;
  for (int i = 0; i < g.n; ++i) {
    int tm = (g.d[i].M + CF::BM - 1) / CF::BM, tn = (g.d[i].N + CF::BN - 1) / CF::BN;
    if (tm * tn > max_tiles) max_tiles = tm * tn;
    if (g.d[i].batch > max_batch) max_batch = g.d[i].batch;
  }
  if (max_tiles == 0 || max_batch == 0) return 0;
  dim3 grid(max_tiles, max_batch, g.n);
  int maxk = 0;
  for (int i = 0; i < g.n; ++i)
    for (int t = 0; t < g.d[i].nterms; ++t) maxk = g.d[i].t[t].K > maxk ? g.d[i].t[t].K : maxk;
  const int tok = prof_begin(maxk <= 32 ? PROF_ZGEMM_SMALLK : PROF_ZGEMM, stream);
  zgemm_bulk_kernel<CF, RV><<<grid, CF::NT, CF::SMEM, stream>>>(g);
  NEGF_LAUNCHED();
  if (tok >= 0) {
    double fl = 0.0, by = 0.0;
    for (int i = 0; i < g.n; ++i) {
      const ZGemmDesc& d = g.d[i];
      for (int t = 0; t < d.nterms; ++t) {
        fl += 8.0 * d.M * d.N * (double)d.t[t].K * d.batch;
        by += 16.0 * ((double)d.M * d.t[t].K + (double)d.t[t].K * d.N) * d.batch;
      }
      by += 16.0 * (double)d.M * d.N * d.batch * ((d.C && (d.beta.x != 0.0 || d.beta.y != 0.0)) ? 2 : 1);
    }
    prof_end(tok, stream, fl, by);
  }
  return 0;
}

// ---------------------------------------------------------------------------
// Real x complex products with the real operand STORED as doubles (the W
// assembly's Coulomb V, kTermRealA / kTermRealB): a complex product with one
// real factor is exactly two real products (re += v br, im += v bi), so the
// kernel issues 2 DMMAs per fragment pair with no 3M sums, and the real tile
// costs half the global traffic and shared memory of a complex one. The real
// operand is op N only ([M][K] for A, [K][N] for B, leading dimension and K
// or N even so every 16-byte cp.async chunk holds two whole doubles).
// Real tiles: A [BM][BK+4], B [BK][BN+4] doubles -- both conflict-free for
// the DMMA fragment reads (row strides = 4 mod 16 double-banks).
template <int BM_, int BN_, int BK_, int STAGES_, int MINB_, int WM_, int WN_, int RSIDE_>
struct DzCfg {
  static constexpr int BM = BM_, BN = BN_, BK = BK_, STAGES = STAGES_, MINB = MINB_, WM = WM_, WN = WN_;
  static constexpr int RSIDE = RSIDE_;  // 1: A real, 2: B real
  static constexpr int NT = WM * WN * 32;
  static constexpr int WTM = BM / WM, WTN = BN / WN, TM = WTM / 8, TN = WTN / 8;
  static constexpr int SKR = BK + 4, SMBR = BN + 4;        // real strides (doubles)
  static constexpr int SK = BK + 4, SMA = BM + 2, SMB = BN + 2;  // complex strides (complex)
  // sizes in doubles
  static constexpr int A_D = RSIDE == 1 ? BM * SKR : 2 * ((BM * SK > BK * SMA) ? BM * SK : BK * SMA);
  static constexpr int B_D = RSIDE == 2 ? BK * SMBR : 2 * ((BN * SK > BK * SMB) ? BN * SK : BK * SMB);
  static constexpr int STAGE_D = A_D + B_D;
  static constexpr size_t SMEM = (size_t)STAGES * STAGE_D * sizeof(double);
  static_assert(A_D % 2 == 0 && B_D % 2 == 0, "16-byte aligned tiles");
};

template <class CF>
__device__ __forceinline__ void dz_load_stage(const ZGemmDesc& d, int kt, const KtBounds& kb, int b, int m0, int n0,
                                              double* sA, double* sB) {
  const int term = kb.term(kt);
  const ZTerm& t = d.t[term];
  const int k0 = (kt - kb.base(term)) * CF::BK;
  const int K = t.K, M = d.M, N = d.N;
  if constexpr (CF::RSIDE == 1) {  // real A [M][K]
    const double* A = reinterpret_cast<const double*>(t.A) + (long long)b * t.sA;
#pragma unroll
    for (int e = threadIdx.x; e < CF::BM * CF::BK / 2; e += CF::NT) {
      const int mn = e / (CF::BK / 2), kc = 2 * (e % (CF::BK / 2));
      const int gm = m0 + mn, gk = k0 + kc;
      const bool p = gm < M && gk < K;
      cp_async16(sA + mn * CF::SKR + kc, p ? A + (long long)gm * t.lda + gk : A, p);
    }
  } else {
    const z_t* A = t.A + (long long)b * t.sA;
    z_t* zA = reinterpret_cast<z_t*>(sA);
    if (!op_trans(t.opA)) {
#pragma unroll
      for (int e = threadIdx.x; e < CF::BM * CF::BK; e += CF::NT) {
        const int mn = e / CF::BK, k = e % CF::BK, gm = m0 + mn, gk = k0 + k;
        const bool p = gm < M && gk < K;
        cp_async16(zA + mn * CF::SK + k, p ? A + (long long)gm * t.lda + gk : A, p);
      }
    } else {
#pragma unroll
      for (int e = threadIdx.x; e < CF::BM * CF::BK; e += CF::NT) {
        const int mn = e % CF::BM, k = e / CF::BM, gm = m0 + mn, gk = k0 + k;
        const bool p = gm < M && gk < K;
        cp_async16(zA + k * CF::SMA + mn, p ? A + (long long)gk * t.lda + gm : A, p);
      }
    }
  }
  if constexpr (CF::RSIDE == 2) {  // real B [K][N]
    const double* B = reinterpret_cast<const double*>(t.B) + (long long)b * t.sB;
#pragma unroll
    for (int e = threadIdx.x; e < CF::BK * CF::BN / 2; e += CF::NT) {
      const int k = e / (CF::BN / 2), nc = 2 * (e % (CF::BN / 2));
      const int gn = n0 + nc, gk = k0 + k;
      const bool p = gn < N && gk < K;
      cp_async16(sB + k * CF::SMBR + nc, p ? B + (long long)gk * t.ldb + gn : B, p);
    }
  } else {
    const z_t* B = t.B + (long long)b * t.sB;
    z_t* zB = reinterpret_cast<z_t*>(sB);
    if (!op_trans(t.opB)) {
#pragma unroll
      for (int e = threadIdx.x; e < CF::BN * CF::BK; e += CF::NT) {
        const int mn = e % CF::BN, k = e / CF::BN, gn = n0 + mn, gk = k0 + k;
        const bool p = gn < N && gk < K;
        cp_async16(zB + k * CF::SMB + mn, p ? B + (long long)gk * t.ldb + gn : B, p);
      }
    } else {
#pragma unroll
      for (int e = threadIdx.x; e < CF::BN * CF::BK; e += CF::NT) {
        const int mn = e / CF::BK, k = e % CF::BK, gn = n0 + mn, gk = k0 + k;
        const bool p = gn < N && gk < K;
        cp_async16(zB + mn * CF::SK + k, p ? B + (long long)gn * t.ldb + gk : B, p);
      }
    }
  }
}

template <class CF>
__global__ void __launch_bounds__(CF::NT, CF::MINB) zgemm_dz_kernel(const __grid_constant__ ZGemmGroup grp) {
  extern __shared__ __align__(16) double dsm[];
  const ZGemmDesc& d = grp.d[blockIdx.z];
  const int tiles_n = (d.N + CF::BN - 1) / CF::BN;
  const int tiles_m = (d.M + CF::BM - 1) / CF::BM;
  if ((int)blockIdx.x >= tiles_m * tiles_n || (int)blockIdx.y >= d.batch) return;
  if (d.active && !d.active[blockIdx.y]) return;
  const int b = blockIdx.y;
  const int m0 = (blockIdx.x / tiles_n) * CF::BM;
  const int n0 = (blockIdx.x % tiles_n) * CF::BN;
  if (d.herm && n0 >= m0 + CF::BM) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int wm = warp / CF::WN, wn = warp % CF::WN;
  KtBounds kb;
  {
    auto nk = [&](int i) { return i < d.nterms ? (d.t[i].K + CF::BK - 1) / CF::BK : 0; };
    kb.b1 = nk(0);
    kb.b2 = kb.b1 + nk(1);
    kb.b3 = kb.b2 + nk(2);
  }
  const int KT = kb.b3 + (d.nterms > 3 ? (d.t[3].K + CF::BK - 1) / CF::BK : 0);
  auto stA = [&](int s) { return dsm + s * CF::STAGE_D; };
  auto stB = [&](int s) { return dsm + s * CF::STAGE_D + CF::A_D; };
  double acc_re[CF::TM][CF::TN][2], acc_im[CF::TM][CF::TN][2];
#pragma unroll
  for (int i = 0; i < CF::TM; ++i)
#pragma unroll
    for (int j = 0; j < CF::TN; ++j) acc_re[i][j][0] = acc_re[i][j][1] = acc_im[i][j][0] = acc_im[i][j][1] = 0.0;
#pragma unroll
  for (int s = 0; s < CF::STAGES - 1; ++s) {
    if (s < KT) dz_load_stage<CF>(d, s, kb, b, m0, n0, stA(s), stB(s));
    cp_async_commit();
  }
  const int r = lane >> 2, q = lane & 3;
  for (int kt = 0; kt < KT; ++kt) {
    cp_async_wait<CF::STAGES - 2>();
    __syncthreads();
    {
      const int nk = kt + CF::STAGES - 1;
      if (nk < KT) dz_load_stage<CF>(d, nk, kb, b, m0, n0, stA(nk % CF::STAGES), stB(nk % CF::STAGES));
      cp_async_commit();
    }
    const int s = kt % CF::STAGES;
    const double* sA = stA(s);
    const double* sB = stB(s);
    const ZTerm& t = d.t[kb.term(kt)];
    const unsigned long long negm = (t.neg & 1) ? kSign : 0ull;
    const unsigned long long conjA = op_conj(t.opA) ? kSign : 0ull;
    const unsigned long long conjB = op_conj(t.opB) ? kSign : 0ull;
    const bool a_kc = !op_trans(t.opA), b_kc = op_trans(t.opB);
    const int a_smn = a_kc ? CF::SK : 1, a_sk = a_kc ? 1 : CF::SMA;
    const int b_smn = b_kc ? CF::SK : 1, b_sk = b_kc ? 1 : CF::SMB;
#pragma unroll
    for (int k4 = 0; k4 < CF::BK / 4; ++k4) {
      const int kk = k4 * 4 + q;
      if constexpr (CF::RSIDE == 1) {
        double a[CF::TM], br[CF::TN], bi[CF::TN];
#pragma unroll
        for (int i = 0; i < CF::TM; ++i) a[i] = dneg_if(sA[(wm * CF::WTM + i * 8 + r) * CF::SKR + kk], negm);
        const z_t* zB = reinterpret_cast<const z_t*>(sB);
#pragma unroll
        for (int j = 0; j < CF::TN; ++j) {
          const z_t v = zB[(wn * CF::WTN + j * 8 + r) * b_smn + kk * b_sk];
          br[j] = v.x;
          bi[j] = dneg_if(v.y, conjB);
        }
#pragma unroll
        for (int i = 0; i < CF::TM; ++i)
#pragma unroll
          for (int j = 0; j < CF::TN; ++j) dmma_m8n8k4(acc_re[i][j][0], acc_re[i][j][1], a[i], br[j]);
#pragma unroll
        for (int i = 0; i < CF::TM; ++i)
#pragma unroll
          for (int j = 0; j < CF::TN; ++j) dmma_m8n8k4(acc_im[i][j][0], acc_im[i][j][1], a[i], bi[j]);
      } else {
        double ar[CF::TM], ai[CF::TM], bv[CF::TN];
        const z_t* zA = reinterpret_cast<const z_t*>(sA);
#pragma unroll
        for (int i = 0; i < CF::TM; ++i) {
          const z_t v = zA[(wm * CF::WTM + i * 8 + r) * a_smn + kk * a_sk];
          ar[i] = v.x;
          ai[i] = dneg_if(v.y, conjA);
        }
#pragma unroll
        for (int j = 0; j < CF::TN; ++j) bv[j] = dneg_if(sB[kk * CF::SMBR + wn * CF::WTN + j * 8 + r], negm);
#pragma unroll
        for (int i = 0; i < CF::TM; ++i)
#pragma unroll
          for (int j = 0; j < CF::TN; ++j) dmma_m8n8k4(acc_re[i][j][0], acc_re[i][j][1], ar[i], bv[j]);
#pragma unroll
        for (int i = 0; i < CF::TM; ++i)
#pragma unroll
          for (int j = 0; j < CF::TN; ++j) dmma_m8n8k4(acc_im[i][j][0], acc_im[i][j][1], ai[i], bv[j]);
      }
    }
  }
  cp_async_wait<0>();
  const double2 al = d.alpha, be = d.beta;
  const bool use_c = d.C != nullptr && (be.x != 0.0 || be.y != 0.0);
  const z_t* C = use_c ? d.C + (long long)b * d.sC : nullptr;
  z_t* D = d.D + (long long)b * d.sD;
  const int er = lane >> 2, eq = lane & 3;
#pragma unroll
  for (int i = 0; i < CF::TM; ++i) {
    const int gm = m0 + wm * CF::WTM + i * 8 + er;
#pragma unroll
    for (int j = 0; j < CF::TN; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int gn = n0 + wn * CF::WTN + j * 8 + 2 * eq + h;
        if (gm < d.M && gn < d.N) {
          const double xr = acc_re[i][j][h], xi = acc_im[i][j][h];
          z_t v = zmake(al.x * xr - al.y * xi, al.x * xi + al.y * xr);
          if (use_c) {
            const z_t c = C[(long long)gm * d.ldc + gn];
            v.x += be.x * c.x - be.y * c.y;
            v.y += be.x * c.y + be.y * c.x;
          }
          if (d.herm) {  // lower triangle + mirror; the diagonal projected to i Im v
            if (gm > gn) {
              D[(long long)gm * d.ldd + gn] = v;
              D[(long long)gn * d.ldd + gm] = zmake(-v.x, v.y);
            } else if (gm == gn) {
              D[(long long)gm * d.ldd + gn] = zmake(0.0, v.y);
            }
          } else if (d.transD)
            D[(long long)gn * d.ldd + gm] = zconj(v);
          else
            D[(long long)gm * d.ldd + gn] = v;
        }
      }
  }
}

template <class CF>
int launch_dz(const ZGemmGroup& g, cudaStream_t stream) {
  static unsigned long long attr_done = 0;
  int dev = 0;
  NEGF_CUDA_CHECK(cudaGetDevice(&dev));
  if (dev >= 64) return -1;
  if (!(__atomic_load_n(&attr_done, __ATOMIC_ACQUIRE) & (1ull << dev))) {
    NEGF_CUDA_CHECK(
        cudaFuncSetAttribute(zgemm_dz_kernel<CF>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CF::SMEM));
    __atomic_fetch_or(&attr_done, 1ull << dev, __ATOMIC_RELEASE);
  }
  int max_tiles = 0, max_batch = 0;
  for (int i = 0; i < g.n; ++i) {
    const int tm = (g.d[i].M + CF::BM - 1) / CF::BM, tn = (g.d[i].N + CF::BN - 1) / CF::BN;
    max_tiles = tm * tn > max_tiles ? tm * tn : max_tiles;
    max_batch = g.d[i].batch > max_batch ? g.d[i].batch : max_batch;
  }
  if (max_tiles == 0 || max_batch == 0) return 0;
  const int tok = prof_begin(PROF_ZGEMM, stream);
  zgemm_dz_kernel<CF><<<dim3(max_tiles, max_batch, g.n), CF::NT, CF::SMEM, stream>>>(g);
  NEGF_LAUNCHED();
  if (tok >= 0) {
    double fl = 0.0, by = 0.0;  // real x complex: 4 M N K flops; the real operand 8 B per element
    for (int i = 0; i < g.n; ++i) {
      const ZGemmDesc& d = g.d[i];
      for (int t = 0; t < d.nterms; ++t) {
        fl += 4.0 * d.M * d.N * (double)d.t[t].K * d.batch;
        by += (CF::RSIDE == 1 ? 8.0 : 16.0) * d.M * d.t[t].K * d.batch +
              (CF::RSIDE == 2 ? 8.0 : 16.0) * d.t[t].K * (double)d.N * d.batch;
      }
      by += 16.0 * (double)d.M * d.N * d.batch * ((d.C && (d.beta.x != 0.0 || d.beta.y != 0.0)) ? 2 : 1);
    }
    prof_end(tok, stream, fl, by);
  }
  return 0;
}

#ifndef NEGF_DZ_BM
#define NEGF_DZ_BM 64
#endif
#ifndef NEGF_DZ_BN
#define NEGF_DZ_BN 32
#endif
#ifndef NEGF_DZ_BK
#define NEGF_DZ_BK 16
#endif
#ifndef NEGF_DZ_STAGES
#define NEGF_DZ_STAGES 2
#endif
#ifndef NEGF_DZ_MINB
#define NEGF_DZ_MINB 4
#endif
using DzA = DzCfg<NEGF_DZ_BM, NEGF_DZ_BN, NEGF_DZ_BK, NEGF_DZ_STAGES, NEGF_DZ_MINB, 2, 2, 1>;
using DzB = DzCfg<NEGF_DZ_BM, NEGF_DZ_BN, NEGF_DZ_BK, NEGF_DZ_STAGES, NEGF_DZ_MINB, 2, 2, 2>;

// BK = 32 x 2 stages x 2 CTAs/SM measured best of the bulk family (8 x 1024^3:
// 39.1 TFLOP/s algorithmic vs 36.2 for the cp.async kernel and 36.0 for cuBLAS;
// BK 16 x 3 stages 24.9, BK 8 x 4 stages 19.0, BK 16 x 2 stages x 3 CTAs 32.5)
#ifndef NEGF_BULK_BK
#define NEGF_BULK_BK 32
#endif
#ifndef NEGF_BULK_STAGES
#define NEGF_BULK_STAGES 2
#endif
#ifndef NEGF_BULK_MINB
#define NEGF_BULK_MINB 2
#endif
#ifndef NEGF_BULK_BM
#define NEGF_BULK_BM 64
#endif
#ifndef NEGF_BULK_BN
#define NEGF_BULK_BN 32
#endif
#ifndef NEGF_BULK_WM
#define NEGF_BULK_WM 2
#endif
#ifndef NEGF_BULK_WN
#define NEGF_BULK_WN 2
#endif
using BulkGauss = BulkCfg<NEGF_BULK_BM, NEGF_BULK_BN, NEGF_BULK_BK, NEGF_BULK_STAGES, NEGF_BULK_MINB, NEGF_BULK_WM,
                          NEGF_BULK_WN>;

using CfgSmall = Cfg<32, 32, 1, 1, 4, 4>;
// default (algo 2): 3M, 64x32 CTA tiles of 4 warps, 3 CTAs/SM, BK = 16 with a
// 2-stage cp.async pipeline and XOR-swizzled k-contiguous tiles (50 KB smem):
// 96 DMMAs per warp between barriers
#ifndef NEGF_G2_MINB
#define NEGF_G2_MINB 3
#endif
#ifndef NEGF_G2_STAGES
#define NEGF_G2_STAGES 2
#endif
using CfgGauss2 = Cfg<64, 32, 2, 2, NEGF_G2_STAGES, NEGF_G2_MINB, true, 16, false, true>;
using CfgGauss2S = Cfg<32, 64, 2, 2, 2, 3, true, 16, false, true>;  // short M
// algo 0: 4 real products per complex product (the textbook arithmetic)
using Cfg4M32 = Cfg<64, 32, 2, 2, 4, 3, false>;
// row-mapped inversion sweeps (K <= 32): 16x16 warp tiles, 5 CTAs/SM
using CfgMapT = Cfg<32, 32, 2, 2, 2, 5, true, 16, true, true>;
using CfgMapT4 = Cfg<32, 32, 2, 2, 2, 5, false, 16, true, true>;  // same, 4M (algo 0)
// Round-1 measurements that picked these (C2 carrier batch, energies/s, G^> by
// the identity): 64x32 BK16 2 stages swizzled 149.2 | 8 warps of 16x16 133.8 |
// 32x32 at 5 CTAs/SM 142.6 | 64x32 BK8 4 stages padded 137.9 | 32x64 BK16 140.0 |
// 64x32 BK32 2 CTAs/SM 133.5 | 64x32 BK16 4 CTAs/SM (spills) 109.4. The
// alternatives were removed from the library.

}  // namespace

// Complex-product algorithm (process-wide, negf_set_gemm_algo): 2 = 3M /
// Gauss with 64x32 tiles (default: the fastest on B200, profiles/, and its
// normwise error bound keeps every parity test at the 1e-9 bar); 0 = 4M.
static int g_algo = 2;
int gemm_algo() { return g_algo; }
void set_gemm_algo(int a) { g_algo = a; }


// ---------------------------------------------------------------------------
// Gauss-Jordan inversion sweep (zinv.cu), streamed: for the rows m < n - wd
// outside the panel's pivot rows K,
//   A_new[dst(m), :] = C(m, :) - A_old[src(m), K] * A_new[K, :],
//   C(m, j) = A_old[src(m), j] for j outside K, 0 on K
// (A_new[K, K] = Pinv gives the -C' Pinv block). One CTA keeps its 64 rows of
// C' = A_old[src(m), K] in shared memory and streams column chunks of 32:
// the next chunk's A_new[K, chunk] arrives by cp.async while this chunk's
// DMMAs run, the chunk's C fragment is loaded into registers before the wait.
// 32-row CTAs of 4 warps (16 x 16 warp tiles, 126 registers, 4 CTAs/SM): the
// 64-row CTAs (236 registers, 2/SM) were 7 % slower at 256 x 128
// (profiles/zinv_sweep_r02.txt).
// The generic row-mapped GEMM re-staged C' per 32 x 32 tile and exposed the
// C load latency in every tile's epilogue (40 % DMMA pipe at K = 32).
namespace {
#ifndef NEGF_SWEEP_BM
#define NEGF_SWEEP_BM 32
#endif
#ifndef NEGF_SWEEP_MINB
#define NEGF_SWEEP_MINB 4
#endif
struct CfgSweep {  // the tile geometry gauss_stage reads (3M, +4-padded k-contiguous A, n-contiguous B)
  static constexpr bool GAUSS = true, SWZ = false;
  static constexpr int BM = NEGF_SWEEP_BM, BN = 32, BK = 16, WM = 2, WN = 2, NT = WM * WN * 32;
  static constexpr int WTM = BM / WM, WTN = BN / WN, TM = WTM / 8, TN = WTN / 8;
  static constexpr int SK = BK + 4, SMA = BM + 2, SMB = BN + 2;
};
constexpr int kSweepSlices = 2;  // K = wd <= 32: two 16-deep slices
constexpr size_t kSweepSmem = sizeof(z_t) * ((size_t)kSweepSlices * CfgSweep::BM * CfgSweep::SK +
                                             2 * (size_t)kSweepSlices * CfgSweep::BK * CfgSweep::SMB);

__global__ void __launch_bounds__(CfgSweep::NT, NEGF_SWEEP_MINB) zinv_sweep_kernel(const __grid_constant__ SweepArgs a) {
  using CF = CfgSweep;
  extern __shared__ __align__(16) z_t smem[];
  const int b = blockIdx.z;
  if (a.active && !a.active[b]) return;
  const int rows = a.n - a.wd;
  const int m0 = blockIdx.x * CF::BM;
  const int nchunks = (a.n + CF::BN - 1) / CF::BN;
  const int cpg = (nchunks + a.ng - 1) / a.ng;
  const int c_begin = blockIdx.y * cpg;
  const int c_end = c_begin + cpg < nchunks ? c_begin + cpg : nchunks;
  if (m0 >= rows || c_begin >= c_end) return;
  const int nsl = (a.wd + CF::BK - 1) / CF::BK;
  const z_t* A = a.cur + (long long)b * a.cs;
  z_t* Nw = a.nxt + (long long)b * a.ns;
  const int* msrc = a.map_src + (long long)b * a.n;
  const int* mdst = a.map_dst + (long long)b * a.n;
  auto sA = [&](int s) { return smem + s * CF::BM * CF::SK; };
  auto sB = [&](int buf, int s) {
    return smem + kSweepSlices * CF::BM * CF::SK + (buf * kSweepSlices + s) * CF::BK * CF::SMB;
  };
  for (int s = 0; s < nsl; ++s)
    for (int e = threadIdx.x; e < CF::BM * CF::BK; e += CF::NT) {
      const int mn = e / CF::BK, k = e % CF::BK, gm = m0 + mn, gk = s * CF::BK + k;
      const bool p = gm < rows && gk < a.wd;
      cp_async16(sA(s) + mn * CF::SK + k, p ? A + (long long)msrc[gm] * a.n + a.k0 + gk : A, p);
    }
  auto load_b = [&](int c, int buf) {
    for (int s = 0; s < nsl; ++s)
      for (int e = threadIdx.x; e < CF::BK * CF::BN; e += CF::NT) {
        const int k = e / CF::BN, nn = e % CF::BN, gk = s * CF::BK + k, gn = c * CF::BN + nn;
        const bool p = gk < a.wd && gn < a.n;
        cp_async16(sB(buf, s) + k * CF::SMB + nn, p ? Nw + (long long)(a.k0 + gk) * a.n + gn : Nw, p);
      }
  };
  load_b(c_begin, 0);
  cp_async_commit();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int wm = warp / CF::WN, wn = warp % CF::WN;
  const int er = lane >> 2, eq = lane & 3;
  int srow[CF::TM], drow[CF::TM];
#pragma unroll
  for (int i = 0; i < CF::TM; ++i) {
    const int gm = m0 + wm * CF::WTM + i * 8 + er;
    srow[i] = gm < rows ? msrc[gm] : 0;
    drow[i] = gm < rows ? mdst[gm] : -1;
  }
  for (int c = c_begin; c < c_end; ++c) {
    const int buf = (c - c_begin) & 1;
    if (c + 1 < c_end) load_b(c + 1, buf ^ 1);
    cp_async_commit();
    z_t cv[CF::TM][CF::TN][2];  // C fragment, in flight during the wait and the DMMAs
#pragma unroll
    for (int i = 0; i < CF::TM; ++i)
#pragma unroll
      for (int j = 0; j < CF::TN; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int gn = c * CF::BN + wn * CF::WTN + j * 8 + 2 * eq + h;
          const bool in = drow[i] >= 0 && gn < a.n && (gn < a.k0 || gn >= a.k0 + a.wd);
          cv[i][j][h] = in ? A[(long long)srow[i] * a.n + gn] : make_double2(0.0, 0.0);
        }
    cp_async_wait<1>();
    __syncthreads();
    double acc_re[CF::TM][CF::TN][2], acc_im[CF::TM][CF::TN][2], acc_s[CF::TM][CF::TN][2];
#pragma unroll
    for (int i = 0; i < CF::TM; ++i)
#pragma unroll
      for (int j = 0; j < CF::TN; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) acc_re[i][j][h] = acc_im[i][j][h] = acc_s[i][j][h] = 0.0;
    for (int s = 0; s < nsl; ++s)
      gauss_stage<CF, false, true, false>(sA(s), sB(buf, s), acc_re, acc_im, acc_s, 0ull, 0ull, 0ull, wm, wn, lane);
#pragma unroll
    for (int i = 0; i < CF::TM; ++i) {
      if (drow[i] < 0) continue;
#pragma unroll
      for (int j = 0; j < CF::TN; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int gn = c * CF::BN + wn * CF::WTN + j * 8 + 2 * eq + h;
          if (gn < a.n) {
            const double p1 = acc_re[i][j][h], p2 = acc_im[i][j][h];
            const z_t v = cv[i][j][h];
            Nw[(long long)drow[i] * a.n + gn] = zmake(v.x - (p1 - p2), v.y - (acc_s[i][j][h] - p1 - p2));
          }
        }
    }
    __syncthreads();  // every warp is done with buf before the next iteration refills it
  }
  cp_async_wait<0>();
}

// Fused variant (SweepArgs.prow set, one-CTA panels): the panel kernel leaves
// T = Pinv R (R = the pivot rows of A_old) to this kernel. Row CTAs form
// L' = C' Pinv in shared memory (one small DMMA product), write -L' into the
// columns K and stream D = C - L' R over the other chunks; one extra CTA per
// column group (blockIdx.x == row blocks) streams T = Pinv R into the rows K
// of A_new (Pinv itself on the columns K). T leaves the single-CTA panel,
// where it was ~40 % of the panel time, for the whole GPU.
__global__ void __launch_bounds__(CfgSweep::NT, NEGF_SWEEP_MINB) zinv_sweep_fused_kernel(
    const __grid_constant__ SweepArgs a) {
  using CF = CfgSweep;
  extern __shared__ __align__(16) z_t smem[];
  const int b = blockIdx.z;
  if (a.active && !a.active[b]) return;
  const int rows = a.n - a.wd;
  const int rb = (rows + CF::BM - 1) / CF::BM;
  const bool trole = (int)blockIdx.x == rb;
  const int m0 = trole ? 0 : blockIdx.x * CF::BM;
  const int nchunks = (a.n + CF::BN - 1) / CF::BN;
  const int cpg = (nchunks + a.ng - 1) / a.ng;
  const int c_begin = blockIdx.y * cpg;
  const int c_end = c_begin + cpg < nchunks ? c_begin + cpg : nchunks;
  if (c_begin >= c_end) return;
  const int nsl = (a.wd + CF::BK - 1) / CF::BK;
  const int wd = a.wd, n = a.n, k0 = a.k0;
  const z_t* A = a.cur + (long long)b * a.cs;
  z_t* Nw = a.nxt + (long long)b * a.ns;
  const z_t* P = a.pinv + (long long)b * wd * wd;
  const int* pr = a.prow + (long long)b * 32;
  const int* msrc = a.map_src + (long long)b * n;
  const int* mdst = a.map_dst + (long long)b * n;
  auto sA = [&](int s) { return smem + s * CF::BM * CF::SK; };
  auto sB = [&](int buf, int s) {
    return smem + kSweepSlices * CF::BM * CF::SK + (buf * kSweepSlices + s) * CF::BK * CF::SMB;
  };
  // group 0: the A tile (C' rows, or Pinv for the T CTA) and, for row CTAs, Pinv as a B tile in buffer 1
  for (int s = 0; s < nsl; ++s)
    for (int e = threadIdx.x; e < CF::BM * CF::BK; e += CF::NT) {
      const int mn = e / CF::BK, k = e % CF::BK, gk = s * CF::BK + k;
      if (trole) {
        const bool p = mn < wd && gk < wd;
        cp_async16(sA(s) + mn * CF::SK + k, p ? P + (long long)mn * wd + gk : P, p);
      } else {
        const int gm = m0 + mn;
        const bool p = gm < rows && gk < wd;
        cp_async16(sA(s) + mn * CF::SK + k, p ? A + (long long)msrc[gm] * n + k0 + gk : A, p);
      }
    }
  if (!trole)
    for (int s = 0; s < nsl; ++s)
      for (int e = threadIdx.x; e < CF::BK * CF::BN; e += CF::NT) {
        const int k = e / CF::BN, nn = e % CF::BN, gk = s * CF::BK + k;
        const bool p = gk < wd && nn < wd;
        cp_async16(sB(1, s) + k * CF::SMB + nn, p ? P + (long long)gk * wd + nn : P, p);
      }
  cp_async_commit();
  auto load_r = [&](int c, int buf) {  // B chunk: R[q][chunk] = A_old[prow[q]][chunk]
    for (int s = 0; s < nsl; ++s)
      for (int e = threadIdx.x; e < CF::BK * CF::BN; e += CF::NT) {
        const int k = e / CF::BN, nn = e % CF::BN, gk = s * CF::BK + k, gn = c * CF::BN + nn;
        const bool p = gk < wd && gn < n;
        cp_async16(sB(buf, s) + k * CF::SMB + nn, p ? A + (long long)pr[gk] * n + gn : A, p);
      }
  };
  load_r(c_begin, 0);
  cp_async_commit();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int wm = warp / CF::WN, wn = warp % CF::WN;
  const int er = lane >> 2, eq = lane & 3;
  double acc_re[CF::TM][CF::TN][2], acc_im[CF::TM][CF::TN][2], acc_s[CF::TM][CF::TN][2];
  auto zero_acc = [&]() {
#pragma unroll
    for (int i = 0; i < CF::TM; ++i)
#pragma unroll
      for (int j = 0; j < CF::TN; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) acc_re[i][j][h] = acc_im[i][j][h] = acc_s[i][j][h] = 0.0;
  };
  int srow[CF::TM], drow[CF::TM];
#pragma unroll
  for (int i = 0; i < CF::TM; ++i) {
    const int gm = m0 + wm * CF::WTM + i * 8 + er;
    if (trole) {
      srow[i] = 0;
      drow[i] = gm < wd ? k0 + gm : -1;
    } else {
      srow[i] = gm < rows ? msrc[gm] : 0;
      drow[i] = gm < rows ? mdst[gm] : -1;
    }
  }
  const int cK = k0 / CF::BN;  // the chunk holding the columns K (nb divides BN)
  const bool ownK = cK >= c_begin && cK < c_end;
  cp_async_wait<1>();
  __syncthreads();
  if (!trole) {
    // L' = C' Pinv (32 x wd x wd), then -L' into the columns K and L' as the A tile
    zero_acc();
    for (int s = 0; s < nsl; ++s)
      gauss_stage<CF, false, true, false>(sA(s), sB(1, s), acc_re, acc_im, acc_s, 0ull, 0ull, 0ull, wm, wn, lane);
    __syncthreads();  // every warp has read C' before it is overwritten
#pragma unroll
    for (int i = 0; i < CF::TM; ++i)
#pragma unroll
      for (int j = 0; j < CF::TN; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int row = wm * CF::WTM + i * 8 + er, col = wn * CF::WTN + j * 8 + 2 * eq + h;
          const double p1 = acc_re[i][j][h], p2 = acc_im[i][j][h];
          const z_t l = zmake(p1 - p2, acc_s[i][j][h] - p1 - p2);
          sA(col / CF::BK)[row * CF::SK + col % CF::BK] = l;
          if (ownK && drow[i] >= 0 && col < wd) Nw[(long long)drow[i] * n + k0 + col] = zmake(-l.x, -l.y);
        }
  } else if (ownK) {  // the T CTA: Pinv on the columns K of the rows K
    for (int e = threadIdx.x; e < wd * wd; e += CF::NT)
      Nw[(long long)(k0 + e / wd) * n + k0 + e % wd] = P[e];
  }
  __syncthreads();  // L' in place, buffer 1 free
  for (int c = c_begin; c < c_end; ++c) {
    const int buf = (c - c_begin) & 1;
    if (c + 1 < c_end) load_r(c + 1, buf ^ 1);
    cp_async_commit();
    z_t cv[CF::TM][CF::TN][2];
#pragma unroll
    for (int i = 0; i < CF::TM; ++i)
#pragma unroll
      for (int j = 0; j < CF::TN; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int gn = c * CF::BN + wn * CF::WTN + j * 8 + 2 * eq + h;
          const bool in = !trole && drow[i] >= 0 && gn < n && (gn < k0 || gn >= k0 + wd);
          cv[i][j][h] = in ? A[(long long)srow[i] * n + gn] : make_double2(0.0, 0.0);
        }
    cp_async_wait<1>();
    __syncthreads();
    zero_acc();
    for (int s = 0; s < nsl; ++s)
      gauss_stage<CF, false, true, false>(sA(s), sB(buf, s), acc_re, acc_im, acc_s, 0ull, 0ull, 0ull, wm, wn, lane);
#pragma unroll
    for (int i = 0; i < CF::TM; ++i) {
      if (drow[i] < 0) continue;
#pragma unroll
      for (int j = 0; j < CF::TN; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int gn = c * CF::BN + wn * CF::WTN + j * 8 + 2 * eq + h;
          if (gn < n && (gn < k0 || gn >= k0 + wd)) {
            const double p1 = acc_re[i][j][h], p2 = acc_im[i][j][h];
            const double xr = p1 - p2, xi = acc_s[i][j][h] - p1 - p2;
            const z_t v = cv[i][j][h];
            Nw[(long long)drow[i] * n + gn] = trole ? zmake(xr, xi) : zmake(v.x - xr, v.y - xi);
          }
        }
    }
    __syncthreads();
  }
  cp_async_wait<0>();
}
}  // namespace

int zinv_sweep_launch(const SweepArgs& a, int batch, cudaStream_t stream) {
  const int rows = a.n - a.wd;
  if (rows <= 0 || batch <= 0) return 0;
  if (a.wd > kSweepSlices * CfgSweep::BK) return -1;
  static unsigned long long attr_done = 0;
  int dev = 0;
  NEGF_CUDA_CHECK(cudaGetDevice(&dev));
  if (dev >= 64) return -1;
  if (!(__atomic_load_n(&attr_done, __ATOMIC_ACQUIRE) & (1ull << dev))) {
    NEGF_CUDA_CHECK(cudaFuncSetAttribute(zinv_sweep_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)kSweepSmem));
    NEGF_CUDA_CHECK(cudaFuncSetAttribute(zinv_sweep_fused_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)kSweepSmem));
    __atomic_fetch_or(&attr_done, 1ull << dev, __ATOMIC_RELEASE);
  }
  SweepArgs g = a;
  const int rb = (rows + CfgSweep::BM - 1) / CfgSweep::BM;
  const int nchunks = (a.n + CfgSweep::BN - 1) / CfgSweep::BN;
  // column groups: enough CTAs to fill every SM (148 x resident CTAs), each streaming >= 2 chunks
  const int target = 148 * NEGF_SWEEP_MINB;
  int ng = (target + rb * batch - 1) / (rb * batch);
  ng = ng < 1 ? 1 : (ng > (nchunks + 1) / 2 ? (nchunks + 1) / 2 : ng);
  g.ng = ng < 1 ? 1 : ng;
  const int tok = prof_begin(PROF_ZGEMM_SMALLK, stream);
  if (a.prow) {
    if (a.k0 % CfgSweep::BN + a.wd > CfgSweep::BN) return -1;  // K must sit inside one column chunk
    zinv_sweep_fused_kernel<<<dim3(rb + 1, g.ng, batch), CfgSweep::NT, kSweepSmem, stream>>>(g);
  } else {
    zinv_sweep_kernel<<<dim3(rb, g.ng, batch), CfgSweep::NT, kSweepSmem, stream>>>(g);
  }
  NEGF_LAUNCHED();
  if (tok >= 0) {
    const double fl = 8.0 * rows * (double)a.n * a.wd * batch;
    const double by = 16.0 * batch * (2.0 * rows * a.n + (double)a.wd * (a.n + rows));
    prof_end(tok, stream, fl, by);
  }
  return 0;
}

int zgemm_group_launch(const ZGemmGroup& g, cudaStream_t stream) {
  if (g.n <= 0) return 0;
  int mx = 0;
  for (int i = 0; i < g.n; ++i) {
    if (g.d[i].M > mx) mx = g.d[i].M;
    if (g.d[i].N > mx) mx = g.d[i].N;
  }
  bool mapped = false;
  for (int i = 0; i < g.n; ++i) mapped |= g.d[i].rowmap_a || g.d[i].rowmap_c || g.d[i].rowmap_d;
  if (mapped)  // inversion sweeps (K <= 32): occupancy wins over tile size
    return gemm_algo() == 0 ? launch_cfg<CfgMapT4>(g, stream) : launch_cfg<CfgMapT>(g, stream);
  {  // real operand stored as doubles (every term of the group, same side)
    int ra = 0, rb = 0, nt = 0;
    for (int i = 0; i < g.n; ++i)
      for (int t = 0; t < g.d[i].nterms; ++t, ++nt) {
        ra += (g.d[i].t[t].neg & kTermRealA) != 0;
        rb += (g.d[i].t[t].neg & kTermRealB) != 0;
      }
    if (ra || rb) {
      if (ra != nt && rb != nt) return -1;  // mixed groups are a caller bug
#ifndef NEGF_DZ_OFF  // experiments: the same products through the complex kernels
      return ra ? launch_dz<DzA>(g, stream) : launch_dz<DzB>(g, stream);
#else
      return -1;
#endif
    }
  }
  if (mx <= 32) return launch_cfg<CfgSmall>(g, stream);
  if (gemm_algo() == 0) return launch_cfg<Cfg4M32>(g, stream);
  constexpr int kBulkMinM = 512;
  int mm = 0;
  bool real = true;  // every term has a real operand: 2-product Gauss kernel
  for (int i = 0; i < g.n; ++i) {
    mm = g.d[i].M > mm ? g.d[i].M : mm;
    for (int t = 0; t < g.d[i].nterms; ++t) real &= (g.d[i].t[t].neg & kTermReal) != 0;
  }
  // TMA-engine bulk copies + mbarrier ring (warp-specialised): faster than the
  // cp.async kernel for complex x complex products from 512-orbital blocks up
  // (8 x 1024^3: 39.1 vs 36.2 TFLOP/s; C4 W RGF 0.87 vs 0.81 of the FP64
  // peak), slower at 256 (C2) and for the real-V W-assembly products
  // (profiles/gemm_bulk_r02.txt). algo 3 forces it everywhere (experiments).
  if (gemm_algo() == 3 || (gemm_algo() == 2 && !real && mm >= kBulkMinM))
    return real ? launch_bulk<BulkGauss, true>(g, stream) : launch_bulk<BulkGauss>(g, stream);
  if (real)
    return mm <= 32 ? launch_cfg<CfgGauss2S, true>(g, stream) : launch_cfg<CfgGauss2, true>(g, stream);
  return mm <= 32 ? launch_cfg<CfgGauss2S>(g, stream) : launch_cfg<CfgGauss2>(g, stream);
}

int zgemm_launch(const ZGemmDesc& d, cudaStream_t stream) {
  ZGemmGroup g;
  g.n = 1;
  g.d[0] = d;
  return zgemm_group_launch(g, stream);
}

}  // namespace negf
