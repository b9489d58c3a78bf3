// Runtime OBC memoization, batched over energies and contact sides.
//
// Reference: memoized_obc / _memo_refresh / _memo_direct (obc.py:519-608),
// used for the retarded surfaces (scba.py:577-614, key (subsystem, side,
// energy, "R"), refresh map fixed_point_step obc.py:138-141) and the W-side
// lesser/greater Stein solves (scba.py:647-658, map w <- q + a w a^dag).
//
// Per problem, from the cached block x0: x1 = f(x0), delta1 = |x1-x0|/|x1|;
// x2 = f(x1), delta2; rho = delta2/delta1, tail = rho/(1-rho). Refresh only
// if delta2 rho^(n_fpi-2) tail < tol, then iterate until last*tail < tol
// within the budget; any non-finite iterate, singular update, rho >= 1 or
// exhausted budget sends the problem to the direct solver. On the device
// every problem of the batch advances together under an active mask (the
// map is two grouped DMMA GEMMs, plus a masked pivoted inverse for the
// surface map); one CTA per problem makes the reference's decision after
// each step from fused Frobenius norms and copies the accepted iterate out.
// The host only reads the count of problems still iterating.
#include "memo.cuh"
#include "prof.cuh"
#include "zgemm.cuh"
#include "zinv.cuh"

namespace negf {

namespace {

inline size_t a256(size_t x) { return (x + 255) & ~size_t(255); }

enum : int { PH_RUN = 0, PH_ACCEPT = 1, PH_DIRECT = 2 };

struct MemoState {
  int* phase;
  int* active;
  double* delta1;
  double* tail;
};

__global__ void memo_init_kernel(const int* has, MemoState s, int n, int* n_act) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  const int run = has[p] != 0;
  s.phase[p] = run ? PH_RUN : PH_DIRECT;
  s.active[p] = run;
  s.delta1[p] = 0.0;
  s.tail[p] = 0.0;
  if (run) atomicAdd(n_act, 1);
}

// One CTA per problem: |cur - prev|, |cur|, finiteness, then the decision of
// obc.py:567-600 for step t (1-based; steps >= 3 are the budgeted loop).
__global__ void memo_check_kernel(const z_t* __restrict__ prev, const z_t* __restrict__ cur, long long n2,
                                  const int* inv_st, MemoState s, int t, int n_fpi, double tol, z_t* out,
                                  int* n_act) {
  __shared__ double red[3][32];
  __shared__ int s_dec;
  const int p = blockIdx.x;
  if (s.phase[p] != PH_RUN) return;
  const z_t* P = prev + p * n2;
  const z_t* C = cur + p * n2;
  double d2 = 0.0, c2 = 0.0, bad = 0.0;
  for (long long e = threadIdx.x; e < n2; e += blockDim.x) {
    const z_t c = C[e], q = P[e];
    const double dr = c.x - q.x, di = c.y - q.y;
    d2 += dr * dr + di * di;
    c2 += c.x * c.x + c.y * c.y;
    if (!isfinite(c.x) || !isfinite(c.y)) bad += 1.0;
  }
  for (int o = 16; o > 0; o >>= 1) {
    d2 += __shfl_down_sync(0xffffffffu, d2, o);
    c2 += __shfl_down_sync(0xffffffffu, c2, o);
    bad += __shfl_down_sync(0xffffffffu, bad, o);
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) { red[0][w] = d2; red[1][w] = c2; red[2][w] = bad; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double D = 0.0, S = 0.0, B = 0.0;
    for (int i = 0; i < (int)(blockDim.x + 31) / 32; ++i) { D += red[0][i]; S += red[1][i]; B += red[2][i]; }
    const double d = sqrt(D), sc = sqrt(S);
    const bool finite = B == 0.0;
    int dec = PH_RUN;
    if (inv_st && inv_st[p]) {
      dec = PH_DIRECT;  // SingularBlockError inside fixed_point_step -> direct
    } else if (t <= 2) {
      if (!isfinite(d) || sc == 0.0 || !finite) {
        dec = PH_DIRECT;
      } else {
        const double delta = d / sc;
        if (t == 1) {
          if (delta == 0.0) dec = PH_ACCEPT;
          else s.delta1[p] = delta;
        } else if (delta <= 1e-14) {
          dec = PH_ACCEPT;
        } else {
          const double rho = delta / s.delta1[p];
          if (rho >= 1.0) {
            dec = PH_DIRECT;
          } else {
            const double tail = rho / (1.0 - rho);
            const int ex = n_fpi - 2 > 0 ? n_fpi - 2 : 0;
            if (delta * pow(rho, (double)ex) * tail >= tol) dec = PH_DIRECT;
            else if (delta * tail < tol) dec = PH_ACCEPT;  // loop breaks before its first update
            else if (ex == 0) dec = PH_DIRECT;
            s.tail[p] = tail;
          }
        }
      }
    } else {
      if (!finite) {
        dec = PH_DIRECT;
      } else {
        const double last = d / fmax(sc, 1e-300);
        if (last * s.tail[p] < tol) dec = PH_ACCEPT;
        else if (t - 2 >= n_fpi - 2) dec = PH_DIRECT;  // budget spent, tail bound still >= tol
      }
    }
    s.phase[p] = dec;
    s.active[p] = dec == PH_RUN;
    if (dec == PH_RUN) atomicAdd(n_act, 1);
    s_dec = dec;
  }
  __syncthreads();
  if (s_dec == PH_ACCEPT) {
    z_t* O = out + p * n2;
    for (long long e = threadIdx.x; e < n2; e += blockDim.x) O[e] = C[e];
  }
}

__global__ void memo_finish_kernel(const int* phase, int n, int* need_direct, int* used) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  const int acc = phase[p] == PH_ACCEPT;
  need_direct[p] = !acc;
  used[p] = acc;
}

__global__ void copy_selected_kernel(z_t* dst, const z_t* src, long long n2, const int* sel) {
  const int p = blockIdx.y;
  if (!sel[p]) return;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n2;
       e += (long long)gridDim.x * blockDim.x)
    dst[p * n2 + e] = src[p * n2 + e];
}

__global__ void memo_store_flags_kernel(const int* used_buf, int n_seg, int seg_len, int* has, int* used,
                                        long long has_ld) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_seg * seg_len) return;
  const int g = i / seg_len, e = i % seg_len;
  has[g * has_ld + e] = 1;
  if (used) used[g * has_ld + e] = used_buf ? used_buf[i] : 0;
}

#define RC(x) do { int _rc = (x); if (_rc) return _rc; } while (0)

}  // namespace

size_t memo_workspace_bytes(int map, int n_side, int n_kind, int bs) {
  const int np = n_side * n_kind;
  const size_t blk = a256(sizeof(z_t) * (size_t)np * bs * bs);
  size_t b = 4 * blk + 8 * a256(sizeof(double) * (size_t)np + 64);
  if (map == MEMO_SURFACE) b += a256(zinv_workspace_bytes(bs, np));
  return b;
}

int memo_refresh(int map, int n_side, int n_kind, int bs, const z_t* m, const z_t* n, const z_t* np_,
                 const z_t* a, const z_t* q, int n_fpi, double tol, const z_t* x0, const int* has,
                 z_t* out, int* need_direct, int* used, void* ws, size_t ws_bytes, cudaStream_t st) {
  const int P = n_side * n_kind;
  if (P <= 0) return 0;
  if (map != MEMO_SURFACE && map != MEMO_STEIN) return -1;
  if (map == MEMO_SURFACE && n_kind != 1) return -1;
  if (n_kind > kMaxGroup) return -1;
  if (ws_bytes < memo_workspace_bytes(map, n_side, n_kind, bs)) return -4;
  const long long n2 = (long long)bs * bs;
  const size_t blk = a256(sizeof(z_t) * (size_t)P * n2);
  char* w = (char*)ws;
  auto take = [&](size_t b) { char* r = w; w += a256(b); return r; };
  z_t* buf[2] = {(z_t*)take(blk), (z_t*)take(blk)};
  z_t* T = (z_t*)take(blk);
  z_t* S = (z_t*)take(blk);
  MemoState s;
  s.phase = (int*)take(sizeof(double) * P + 64);
  s.active = (int*)take(sizeof(double) * P + 64);
  s.delta1 = (double*)take(sizeof(double) * P + 64);
  s.tail = (double*)take(sizeof(double) * P + 64);
  int* inv_st = (int*)take(sizeof(double) * P + 64);
  int* n_act = (int*)take(sizeof(double) * 8 + 64);
  take(sizeof(double) * P + 64);
  take(sizeof(double) * P + 64);
  void* inv_ws = map == MEMO_SURFACE ? (void*)w : nullptr;
  const size_t inv_bytes = map == MEMO_SURFACE ? zinv_workspace_bytes(bs, P) : 0;

  NEGF_CUDA_CHECK(cudaMemsetAsync(n_act, 0, sizeof(int), st));
  {
    ProfScope ps(PROF_OTHER, st);
    memo_init_kernel<<<(P + 127) / 128, 128, 0, st>>>(has, s, P, n_act);
    NEGF_LAUNCHED();
  }
  int h_act = 0;
  NEGF_CUDA_CHECK(cudaMemcpyAsync(&h_act, n_act, sizeof(int), cudaMemcpyDeviceToHost, st));
  NEGF_CUDA_CHECK(cudaStreamSynchronize(st));
  const int t_max = n_fpi > 2 ? n_fpi : 2;
  for (int t = 1; t <= t_max && h_act > 0; ++t) {
    const z_t* prev = t == 1 ? x0 : buf[(t - 1) & 1];
    z_t* cur = buf[t & 1];
    if (map == MEMO_SURFACE) {
      ZGemmDesc d = zdesc_default();  // T = n prev
      d.M = bs; d.N = bs; d.batch = P;
      d.t[0] = zterm(n, n2, bs, OP_N, prev, n2, bs, OP_N, bs);
      for (int i = 1; i < kMaxTerms; ++i) d.t[i] = d.t[0];
      d.D = T; d.sD = n2; d.ldd = bs;
      d.active = s.active;
      RC(zgemm_launch(d, st));
      d.t[0] = zterm(T, n2, bs, OP_N, np_, n2, bs, OP_N, bs);  // S = m - T n'
      for (int i = 1; i < kMaxTerms; ++i) d.t[i] = d.t[0];
      d.alpha = make_double2(-1.0, 0.0);
      d.C = m; d.sC = n2; d.ldc = bs; d.beta = make_double2(1.0, 0.0);
      d.D = S;
      RC(zgemm_launch(d, st));
      NEGF_CUDA_CHECK(cudaMemsetAsync(inv_st, 0, sizeof(int) * P, st));
      InvAux aux;
      aux.status = inv_st; aux.status_code = 1; aux.u_spread = nullptr; aux.spread_stride = 0;
      aux.active = s.active;
      RC(zinv_batched(S, n2, bs, cur, n2, bs, bs, P, aux, inv_ws, inv_bytes, st));
    } else {
      ZGemmGroup g;
      g.n = n_kind;
      for (int k = 0; k < n_kind; ++k) {  // T_k = a prev_k
        ZGemmDesc d = zdesc_default();
        d.M = bs; d.N = bs; d.batch = n_side;
        d.t[0] = zterm(a, n2, bs, OP_N, prev + (long long)k * n_side * n2, n2, bs, OP_N, bs);
        for (int i = 1; i < kMaxTerms; ++i) d.t[i] = d.t[0];
        d.D = T + (long long)k * n_side * n2; d.sD = n2; d.ldd = bs;
        d.active = s.active + k * n_side;
        g.d[k] = d;
      }
      RC(zgemm_group_launch(g, st));
      for (int k = 0; k < n_kind; ++k) {  // cur_k = q_k + T_k a^dag
        ZGemmDesc& d = g.d[k];
        d.t[0] = zterm(T + (long long)k * n_side * n2, n2, bs, OP_N, a, n2, bs, OP_H, bs);
        for (int i = 1; i < kMaxTerms; ++i) d.t[i] = d.t[0];
        d.C = q + (long long)k * n_side * n2; d.sC = n2; d.ldc = bs; d.beta = make_double2(1.0, 0.0);
        d.D = cur + (long long)k * n_side * n2;
      }
      RC(zgemm_group_launch(g, st));
    }
    NEGF_CUDA_CHECK(cudaMemsetAsync(n_act, 0, sizeof(int), st));
    {
      ProfScope ps(PROF_OTHER, st);
      memo_check_kernel<<<P, 256, 0, st>>>(prev, cur, n2, map == MEMO_SURFACE ? inv_st : nullptr, s, t, n_fpi,
                                           tol, out, n_act);
      NEGF_LAUNCHED();
    }
    if ((t & 3) == 0 || t == t_max) {  // host check every 4 updates (decided problems are masked)
      NEGF_CUDA_CHECK(cudaMemcpyAsync(&h_act, n_act, sizeof(int), cudaMemcpyDeviceToHost, st));
      NEGF_CUDA_CHECK(cudaStreamSynchronize(st));
    }
  }
  {
    ProfScope ps(PROF_OTHER, st);
    memo_finish_kernel<<<(P + 127) / 128, 128, 0, st>>>(s.phase, P, need_direct, used);
    NEGF_LAUNCHED();
  }
  return 0;
}

int memo_gather(const z_t* cache, long long ld, const int* has, long long has_ld, int n_seg, int seg_len,
                int bs, z_t* buf, int* has_buf, cudaStream_t st) {
  if (n_seg <= 0 || seg_len <= 0) return 0;
  const size_t n2b = sizeof(z_t) * (size_t)bs * bs;
  NEGF_CUDA_CHECK(cudaMemcpy2DAsync(buf, seg_len * n2b, cache, ld * n2b, seg_len * n2b, n_seg,
                                    cudaMemcpyDeviceToDevice, st));
  NEGF_CUDA_CHECK(cudaMemcpy2DAsync(has_buf, seg_len * sizeof(int), has, has_ld * sizeof(int),
                                    seg_len * sizeof(int), n_seg, cudaMemcpyDeviceToDevice, st));
  return 0;
}

int memo_store(const z_t* buf, const int* used_buf, int n_seg, int seg_len, int bs, z_t* cache, long long ld,
               int* has, int* used, long long has_ld, cudaStream_t st) {
  if (n_seg <= 0 || seg_len <= 0) return 0;
  const size_t n2b = sizeof(z_t) * (size_t)bs * bs;
  NEGF_CUDA_CHECK(cudaMemcpy2DAsync(cache, ld * n2b, buf, seg_len * n2b, seg_len * n2b, n_seg,
                                    cudaMemcpyDeviceToDevice, st));
  const int n = n_seg * seg_len;
  {
    ProfScope ps(PROF_OTHER, st);
    memo_store_flags_kernel<<<(n + 127) / 128, 128, 0, st>>>(used_buf, n_seg, seg_len, has, used, has_ld);
    NEGF_LAUNCHED();
  }
  return 0;
}

int copy_selected(z_t* dst, const z_t* src, long long n2, const int* sel, int n, cudaStream_t st) {
  if (n <= 0) return 0;
  int bx = (int)((n2 + 255) / 256);
  if (bx > 64) bx = 64;
  dim3 grid(bx, n);
  {
    ProfScope ps(PROF_EW, st);
    copy_selected_kernel<<<grid, 256, 0, st>>>(dst, src, n2, sel);
    NEGF_LAUNCHED();
  }
  return 0;
}

}  // namespace negf
