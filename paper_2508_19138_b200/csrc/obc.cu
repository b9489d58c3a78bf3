// Contact self-energies (open boundary conditions) on the GPU.
//
// Reference: negfgw/obc.py
//   obc_sancho_rubio  obc.py:144-182   decimation, per sweep: g = b^-1,
//                     agb = a g b', bga = b' g a, s -= agb, b -= agb + bga,
//                     a <- a g a, b' <- b' g b'; stop when |a|+|b'| < tol*scale;
//                     x = s^-1; raise if the recursion residual > 10 max(tol,1e-14)
//   recursion_residual obc.py:98-104
//   sigma_lg_obc      obc.py:460-486   Sigma^R = n x n', Gamma = Sigma^R - Sigma^R^dag,
//                     Sigma^< = -f Gamma, Sigma^> = (1-f) Gamma
// and the carrier-side closure scba.py:755-774 (_lead_cell :558, corner
// updates), assembly scba.py:670-727.
//
// All surface problems of a batch (energies x sides) advance together; each
// sweep is one pivoted batched inverse + two grouped DMMA launches. A device
// mask freezes problems the moment they meet the reference's stopping test,
// so every problem stops at exactly the sweep the reference would.
#include "ew.cuh"
#include "prof.cuh"
#include "memo.cuh"
#include "obc.cuh"
#include "zgemm.cuh"
#include "zinv.cuh"

namespace negf {

namespace {

inline size_t a256(size_t x) { return (x + 255) & ~size_t(255); }

__device__ double block_sum(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0) {
    for (int i = 0; i < (int)(blockDim.x + 31) / 32; ++i) s += red[i];
    red[0] = s;
  }
  __syncthreads();
  s = red[0];
  __syncthreads();
  return s;
}

__device__ double fro(const z_t* x, long long n2, double* red) {
  double s = 0.0;
  for (long long e = threadIdx.x; e < n2; e += blockDim.x) s += x[e].x * x[e].x + x[e].y * x[e].y;
  return sqrt(block_sum(s, red));
}

__global__ void sancho_init_kernel(const z_t* n, const z_t* np, int bs, double* scale, int* active,
                                   int* status, int* iters, const int* select) {
  __shared__ double red[32];
  const int b = blockIdx.x;
  if (select && !select[b]) {
    if (threadIdx.x == 0) { active[b] = 0; scale[b] = 1.0; status[b] = OBC_OK; iters[b] = 0; }
    return;
  }
  const long long n2 = (long long)bs * bs;
  double a = fro(n + b * n2, n2, red), c = fro(np + b * n2, n2, red);
  if (threadIdx.x == 0) {
    scale[b] = fmax(fmax(a, c), 1e-300);
    active[b] = 1;
    status[b] = OBC_OK;
    iters[b] = 0;
  }
}

__global__ void sancho_check_kernel(const z_t* alpha, const z_t* beta, int bs, double tol,
                                    const double* scale, int* active, int* inv_status, int* status,
                                    int* iters, int it, int* n_active) {
  __shared__ double red[32];
  const int b = blockIdx.x;
  if (!active[b]) return;
  const long long n2 = (long long)bs * bs;
  double na = fro(alpha + b * n2, n2, red), nb = fro(beta + b * n2, n2, red);
  if (threadIdx.x == 0) {
    if (inv_status[b]) {
      status[b] = OBC_SINGULAR;
      active[b] = 0;
      iters[b] = it;
    } else if (na + nb < tol * scale[b]) {
      active[b] = 0;
      iters[b] = it;
    } else {
      atomicAdd(n_active, 1);
    }
  }
}

__global__ void sancho_finish_kernel(const z_t* x, const z_t* y, int bs, double thr, int* active,
                                     int* inv_status, int* status, double* resid, const int* select) {
  __shared__ double red[32];
  const int b = blockIdx.x;
  if (select && !select[b]) return;
  const long long n2 = (long long)bs * bs;
  const z_t* xb = x + b * n2;
  const z_t* yb = y + b * n2;
  double s = 0.0;
  for (long long e = threadIdx.x; e < n2; e += blockDim.x) {
    double dr = yb[e].x - xb[e].x, di = yb[e].y - xb[e].y;
    s += dr * dr + di * di;
  }
  double num = sqrt(block_sum(s, red));
  double den = fro(xb, n2, red);
  if (threadIdx.x == 0) {
    double r = den > 0.0 ? num / den : num;
    if (resid) resid[b] = r;
    if (status[b] == OBC_OK) {
      if (active[b]) status[b] = OBC_NOT_CONVERGED;
      else if (inv_status[b]) status[b] = OBC_SINGULAR;
      else if (!isfinite(r) || r > thr) status[b] = OBC_RESIDUAL;
    }
  }
}

// Corner fold of one side: M_cc -= S, B<_cc += -f Gamma, B>_cc += (1-f) Gamma,
// Gamma = S - S^dag, S = Sigma^R_obc. Tiles of 32x32 through smem for S^dag.
__global__ void g_corner_kernel(const z_t* __restrict__ sig, int bs, const double* f, z_t* m,
                                z_t* bl, z_t* bg, long long s_blk, z_t* sl_out, z_t* sg_out) {
  __shared__ z_t tt[32][33];
  const int e = blockIdx.y;
  const long long n2 = (long long)bs * bs;
  const z_t* S = sig + e * n2;
  const int tiles_c = (bs + 31) / 32;
  const int r0 = (blockIdx.x / tiles_c) * 32, c0 = (blockIdx.x % tiles_c) * 32;
  const int tx = threadIdx.x, ty = threadIdx.y;
  for (int k = ty; k < 32; k += 8) {
    int rr = c0 + k, cc = r0 + tx;
    if (rr < bs && cc < bs) tt[k][tx] = S[(long long)rr * bs + cc];
  }
  __syncthreads();
  const double fe = f[e];
  for (int k = ty; k < 32; k += 8) {
    int r = r0 + k, c = c0 + tx;
    if (r >= bs || c >= bs) continue;
    z_t s = S[(long long)r * bs + c];
    z_t sh = zconj(tt[tx][k]);  // S^dag[r][c] = conj(S[c][r])
    z_t gam = zsub(s, sh);
    long long off = e * s_blk + (long long)r * bs + c;
    m[off] = zsub(m[off], s);
    z_t lw = zscale(-fe, gam), gr = zscale(1.0 - fe, gam);
    if (bl) bl[off] = zadd(bl[off], lw);
    if (bg) bg[off] = zadd(bg[off], gr);
    if (sl_out) sl_out[e * n2 + (long long)r * bs + c] = lw;
    if (sg_out) sg_out[e * n2 + (long long)r * bs + c] = gr;
  }
}

__global__ void sigma_lg_kernel(const z_t* __restrict__ sig, int bs, const double* f, z_t* sl,
                                z_t* sg) {
  __shared__ z_t tt[32][33];
  const int e = blockIdx.y;
  const long long n2 = (long long)bs * bs;
  const z_t* S = sig + e * n2;
  const int tiles_c = (bs + 31) / 32;
  const int r0 = (blockIdx.x / tiles_c) * 32, c0 = (blockIdx.x % tiles_c) * 32;
  const int tx = threadIdx.x, ty = threadIdx.y;
  for (int k = ty; k < 32; k += 8) {
    int rr = c0 + k, cc = r0 + tx;
    if (rr < bs && cc < bs) tt[k][tx] = S[(long long)rr * bs + cc];
  }
  __syncthreads();
  const double fe = f[e];
  for (int k = ty; k < 32; k += 8) {
    int r = r0 + k, c = c0 + tx;
    if (r >= bs || c >= bs) continue;
    z_t gam = zsub(S[(long long)r * bs + c], zconj(tt[tx][k]));
    if (sl) sl[e * n2 + (long long)r * bs + c] = zscale(-fe, gam);
    if (sg) sg[e * n2 + (long long)r * bs + c] = zscale(1.0 - fe, gam);
  }
}

__global__ void g_assemble_kernel(GAssembleArgs a) {
  // grid: (tiles of bs*bs, n_b, n_e); block 256
  const int e = blockIdx.z, i = blockIdx.y;
  const long long n2 = (long long)a.bs * a.bs;
  const long long sd = (long long)a.n_b * n2, so = (long long)(a.n_b - 1) * n2;
  const double E = a.energy[e], f = a.f_bath[e];
  const double bl_im = 2.0 * a.eta * f, bg_im = -2.0 * a.eta * (1.0 - f);
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < n2;
       q += (long long)gridDim.x * blockDim.x) {
    const int r = (int)(q / a.bs), c = (int)(q % a.bs);
    const bool dg = r == c;
    const long long hd = i * n2 + q, od = e * sd + i * n2 + q;
    z_t h = a.h_diag[hd];
    z_t m = zmake((dg ? E : 0.0) - h.x, (dg ? a.eta : 0.0) - h.y);
    if (a.sr_diag) m = zsub(m, a.sr_diag[od]);
    a.m_diag[od] = m;
    if (a.bl_diag) {
      z_t v = zmake(0.0, dg ? bl_im : 0.0);
      if (a.sl_diag) v = zadd(v, a.sl_diag[od]);
      a.bl_diag[od] = v;
    }
    if (a.bg_diag) {
      z_t v = zmake(0.0, dg ? bg_im : 0.0);
      if (a.sg_diag) v = zadd(v, a.sg_diag[od]);
      a.bg_diag[od] = v;
    }
    if (i + 1 < a.n_b) {
      const long long ho = i * n2 + q, oo = e * so + i * n2 + q;
      z_t u = a.h_upper[ho], l = a.h_lower[ho];
      z_t mu = zmake(-u.x, -u.y), ml = zmake(-l.x, -l.y);
      if (a.sr_upper) mu = zsub(mu, a.sr_upper[oo]);
      if (a.sr_lower) ml = zsub(ml, a.sr_lower[oo]);
      a.m_upper[oo] = mu;
      a.m_lower[oo] = ml;
      if (a.bl_upper) a.bl_upper[oo] = a.sl_upper ? a.sl_upper[oo] : zmake(0.0, 0.0);
      if (a.bg_upper) a.bg_upper[oo] = a.sg_upper ? a.sg_upper[oo] : zmake(0.0, 0.0);
    }
  }
}

// obc_fixed_point convergence test (obc.py:122-133): x <- x_new on active
// problems; freeze those with |x_new - x| / |x_new| < tol.
__global__ void fp_step_kernel(z_t* x, const z_t* xn, long long n2, double tol, int* active, const int* inv_st,
                               int* status, int* iters, double* resid, int it, int* n_act) {
  __shared__ double red[2][32];
  __shared__ int s_keep;
  const int b = blockIdx.x;
  if (!active[b]) return;
  z_t* X = x + b * n2;
  const z_t* XN = xn + b * n2;
  double d2 = 0.0, c2 = 0.0;
  for (long long e = threadIdx.x; e < n2; e += blockDim.x) {
    const z_t v = XN[e], u = X[e];
    const double dr = v.x - u.x, di = v.y - u.y;
    d2 += dr * dr + di * di;
    c2 += v.x * v.x + v.y * v.y;
  }
  for (int o = 16; o > 0; o >>= 1) {
    d2 += __shfl_down_sync(0xffffffffu, d2, o);
    c2 += __shfl_down_sync(0xffffffffu, c2, o);
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) { red[0][w] = d2; red[1][w] = c2; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double D = 0.0, C = 0.0;
    for (int i = 0; i < (int)(blockDim.x + 31) / 32; ++i) { D += red[0][i]; C += red[1][i]; }
    int keep = 1;
    if (inv_st[b]) {
      status[b] = OBC_SINGULAR;
      iters[b] = it;
      active[b] = 0;
      keep = 0;
    } else {
      const double num = sqrt(D), den = sqrt(C);
      if (den > 0.0 && num / den < tol) {
        active[b] = 0;
        iters[b] = it;
        if (resid) resid[b] = num / den;
      } else {
        atomicAdd(n_act, 1);
      }
    }
    s_keep = keep;
  }
  __syncthreads();
  if (s_keep)
    for (long long e = threadIdx.x; e < n2; e += blockDim.x) X[e] = XN[e];
}

__global__ void fp_init_kernel(int* active, int* status, int* iters, int n) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= n) return;
  active[b] = 1;
  status[b] = OBC_OK;
  iters[b] = 0;
}

__global__ void fp_finish_kernel(const int* active, int* status, int* iters, int max_iter, int n) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b < n && active[b] && status[b] == OBC_OK) {
    status[b] = OBC_NOT_CONVERGED;
    iters[b] = max_iter;
  }
}

__global__ void count_active_kernel(const int* active, int n, int* n_act) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b < n && active[b]) atomicAdd(n_act, 1);
}

#define RC(x) do { int _rc = (x); if (_rc) return _rc; } while (0)

}  // namespace

size_t sancho_workspace_bytes(int batch, int bs) {
  size_t blk = a256(sizeof(z_t) * (size_t)batch * bs * bs);
  return 10 * blk + a256(zinv_workspace_bytes(bs, batch)) + 6 * a256(sizeof(double) * batch + 16);
}

int sancho_batched(const z_t* m, const z_t* n, const z_t* np, int batch, int bs, double tol,
                   int max_iter, z_t* x, int* status, int* iters, double* resid, void* ws,
                   size_t ws_bytes, cudaStream_t st, const int* select) {
  if (batch <= 0) return 0;
  if (ws_bytes < sancho_workspace_bytes(batch, bs)) return -4;
  const long long n2 = (long long)bs * bs;
  const size_t blk = a256(sizeof(z_t) * (size_t)batch * n2);
  char* w = reinterpret_cast<char*>(ws);
  auto take = [&](size_t b) { char* r = w; w += a256(b); return r; };
  z_t* s = (z_t*)take(blk);
  z_t* b = (z_t*)take(blk);
  z_t* al = (z_t*)take(blk);
  z_t* be = (z_t*)take(blk);
  z_t* al2 = (z_t*)take(blk);
  z_t* be2 = (z_t*)take(blk);
  z_t* g = (z_t*)take(blk);
  z_t* ag = (z_t*)take(blk);
  z_t* bg = (z_t*)take(blk);
  z_t* tb = (z_t*)take(blk);
  double* scale = (double*)take(sizeof(double) * batch);
  int* active = (int*)take(sizeof(int) * batch);
  int* inv_st = (int*)take(sizeof(int) * batch);
  int* n_act = (int*)take(sizeof(int) * 4);
  void* inv_ws = take(zinv_workspace_bytes(bs, batch));
  size_t inv_bytes = zinv_workspace_bytes(bs, batch);
  const size_t bytes = sizeof(z_t) * (size_t)batch * n2;
  NEGF_CUDA_CHECK(cudaMemcpyAsync(s, m, bytes, cudaMemcpyDeviceToDevice, st));
  NEGF_CUDA_CHECK(cudaMemcpyAsync(b, m, bytes, cudaMemcpyDeviceToDevice, st));
  NEGF_CUDA_CHECK(cudaMemcpyAsync(al, n, bytes, cudaMemcpyDeviceToDevice, st));
  NEGF_CUDA_CHECK(cudaMemcpyAsync(be, np, bytes, cudaMemcpyDeviceToDevice, st));
  NEGF_CUDA_CHECK(cudaMemsetAsync(inv_st, 0, sizeof(int) * batch, st));
  {
    ProfScope ps_sancho_init_kernel(PROF_OTHER, (cudaStream_t)(st));
    sancho_init_kernel<<<batch, 256, 0, st>>>(n, np, bs, scale, active, status, iters, select);
    NEGF_LAUNCHED();
  }
  InvAux aux;
  aux.status = inv_st; aux.status_code = 1; aux.u_spread = nullptr; aux.spread_stride = 0;
  aux.active = active;
  auto desc = [&](const z_t* A, const z_t* B, z_t* D, double alpha, const z_t* C, double beta) {
    ZGemmDesc d = zdesc_default();
    d.M = bs; d.N = bs; d.batch = batch;
    d.t[0] = zterm(A, n2, bs, OP_N, B, n2, bs, OP_N, bs);
    d.t[1] = d.t[0];
    d.alpha = make_double2(alpha, 0.0);
    d.beta = make_double2(beta, 0.0);
    d.C = C; d.sC = n2; d.ldc = bs;
    d.D = D; d.sD = n2; d.ldd = bs;
    d.active = active;
    return d;
  };
  int h_active = batch;
  if (select) {  // problems outside the selection never start
    NEGF_CUDA_CHECK(cudaMemsetAsync(n_act, 0, sizeof(int), st));
    {
      ProfScope ps_count(PROF_OTHER, st);
      count_active_kernel<<<(batch + 127) / 128, 128, 0, st>>>(active, batch, n_act);
      NEGF_LAUNCHED();
    }
    NEGF_CUDA_CHECK(cudaMemcpyAsync(&h_active, n_act, sizeof(int), cudaMemcpyDeviceToHost, st));
    NEGF_CUDA_CHECK(cudaStreamSynchronize(st));
  }
  for (int it = 1; h_active > 0 && it <= max_iter; ++it) {
    NEGF_CUDA_CHECK(cudaMemcpyAsync(tb, b, bytes, cudaMemcpyDeviceToDevice, st));
    RC(zinv_batched(tb, n2, bs, g, n2, bs, bs, batch, aux, inv_ws, inv_bytes, st));
    ZGemmGroup G1;
    G1.n = 2;
    G1.d[0] = desc(al, g, ag, 1.0, nullptr, 0.0);
    G1.d[1] = desc(be, g, bg, 1.0, nullptr, 0.0);
    RC(zgemm_group_launch(G1, st));
    ZGemmGroup G2;
    G2.n = 4;
    G2.d[0] = desc(ag, be, s, -1.0, s, 1.0);                 // s -= (a g) b'
    G2.d[1] = desc(ag, be, b, 1.0, b, 1.0);                  // b -= (a g) b' + (b' g) a
    G2.d[1].t[0].neg = 1;
    G2.d[1].nterms = 2;
    G2.d[1].t[1] = zterm(bg, n2, bs, OP_N, al, n2, bs, OP_N, bs, true);
    G2.d[2] = desc(ag, al, al2, 1.0, nullptr, 0.0);          // a <- (a g) a
    G2.d[3] = desc(bg, be, be2, 1.0, nullptr, 0.0);          // b' <- (b' g) b'
    RC(zgemm_group_launch(G2, st));
    std::swap(al, al2);
    std::swap(be, be2);
    NEGF_CUDA_CHECK(cudaMemsetAsync(n_act, 0, sizeof(int), st));
    {
      ProfScope ps_sancho_check_kernel(PROF_OTHER, (cudaStream_t)(st));
      sancho_check_kernel<<<batch, 256, 0, st>>>(al, be, bs, tol, scale, active, inv_st, status, iters,
                                                 it, n_act);
      NEGF_LAUNCHED();
    }
    // host check every 4 sweeps: problems that converge in between are
    // masked off on the device (their GEMM / inverse CTAs exit at once), so
    // the results are those of a per-sweep check with a quarter of the syncs
    if ((it & 3) == 0 || it == max_iter) {
      NEGF_CUDA_CHECK(cudaMemcpyAsync(&h_active, n_act, sizeof(int), cudaMemcpyDeviceToHost, st));
      NEGF_CUDA_CHECK(cudaStreamSynchronize(st));
      if (h_active == 0) break;
    }
  }
  // x = s^-1 for every problem (s is consumed)
  InvAux aux2 = aux;
  aux2.active = select;
  aux2.status = inv_st;
  RC(zinv_batched(s, n2, bs, x, n2, bs, bs, batch, aux2, inv_ws, inv_bytes, st));
  // residual: y = (m - n x n')^-1
  ZGemmGroup G3;
  G3.n = 1;
  G3.d[0] = desc(n, x, ag, 1.0, nullptr, 0.0);
  G3.d[0].active = select;
  RC(zgemm_group_launch(G3, st));
  G3.d[0] = desc(ag, np, tb, -1.0, m, 1.0);
  G3.d[0].active = select;
  RC(zgemm_group_launch(G3, st));
  RC(zinv_batched(tb, n2, bs, g, n2, bs, bs, batch, aux2, inv_ws, inv_bytes, st));
  const double thr = 10.0 * (tol > 1e-14 ? tol : 1e-14);
  {
    ProfScope ps_sancho_finish_kernel(PROF_OTHER, (cudaStream_t)(st));
    sancho_finish_kernel<<<batch, 256, 0, st>>>(x, g, bs, thr, active, inv_st, status, resid, select);
    NEGF_LAUNCHED();
  }
  return 0;
}

size_t fixed_point_workspace_bytes(int batch, int bs) {
  const size_t blk = a256(sizeof(z_t) * (size_t)batch * bs * bs);
  return 3 * blk + a256(zinv_workspace_bytes(bs, batch)) + 4 * a256(sizeof(int) * (size_t)batch + 64);
}

int fixed_point_batched(const z_t* m, const z_t* n, const z_t* np, int batch, int bs, const z_t* x0, double tol,
                        int max_iter, z_t* x, int* status, int* iters, double* resid, void* ws, size_t ws_bytes,
                        cudaStream_t st) {
  if (batch <= 0) return 0;
  if (ws_bytes < fixed_point_workspace_bytes(batch, bs)) return -4;
  const long long n2 = (long long)bs * bs;
  const size_t bytes = sizeof(z_t) * (size_t)batch * n2;
  char* w = reinterpret_cast<char*>(ws);
  auto take = [&](size_t b_) { char* r = w; w += a256(b_); return r; };
  z_t* T = (z_t*)take(bytes);
  z_t* S = (z_t*)take(bytes);
  z_t* XN = (z_t*)take(bytes);
  int* active = (int*)take(sizeof(int) * batch + 64);
  int* inv_st = (int*)take(sizeof(int) * batch + 64);
  int* n_act = (int*)take(sizeof(int) * 4 + 64);
  take(sizeof(int) * batch + 64);
  void* inv_ws = w;
  const size_t inv_bytes = zinv_workspace_bytes(bs, batch);
  if (x0) NEGF_CUDA_CHECK(cudaMemcpyAsync(x, x0, bytes, cudaMemcpyDeviceToDevice, st));
  else NEGF_CUDA_CHECK(cudaMemsetAsync(x, 0, bytes, st));
  {
    ProfScope ps(PROF_OTHER, st);
    fp_init_kernel<<<(batch + 127) / 128, 128, 0, st>>>(active, status, iters, batch);
    NEGF_LAUNCHED();
  }
  InvAux aux;
  aux.status = inv_st; aux.status_code = 1; aux.u_spread = nullptr; aux.spread_stride = 0; aux.active = active;
  int h_act = batch;
  for (int it = 1; it <= max_iter && h_act > 0; ++it) {
    ZGemmDesc d = zdesc_default();  // T = n x ; S = m - T n'
    d.M = bs; d.N = bs; d.batch = batch; d.active = active;
    d.t[0] = zterm(n, n2, bs, OP_N, x, n2, bs, OP_N, bs);
    for (int i = 1; i < kMaxTerms; ++i) d.t[i] = d.t[0];
    d.D = T; d.sD = n2; d.ldd = bs;
    RC(zgemm_launch(d, st));
    d.t[0] = zterm(T, n2, bs, OP_N, np, n2, bs, OP_N, bs);
    for (int i = 1; i < kMaxTerms; ++i) d.t[i] = d.t[0];
    d.alpha = make_double2(-1.0, 0.0);
    d.C = m; d.sC = n2; d.ldc = bs; d.beta = make_double2(1.0, 0.0);
    d.D = S;
    RC(zgemm_launch(d, st));
    NEGF_CUDA_CHECK(cudaMemsetAsync(inv_st, 0, sizeof(int) * batch, st));
    RC(zinv_batched(S, n2, bs, XN, n2, bs, bs, batch, aux, inv_ws, inv_bytes, st));
    NEGF_CUDA_CHECK(cudaMemsetAsync(n_act, 0, sizeof(int), st));
    {
      ProfScope ps(PROF_OTHER, st);
      fp_step_kernel<<<batch, 256, 0, st>>>(x, XN, n2, tol, active, inv_st, status, iters, resid, it, n_act);
      NEGF_LAUNCHED();
    }
    if ((it & 15) == 0 || it == max_iter) {  // host check every 16 updates
      NEGF_CUDA_CHECK(cudaMemcpyAsync(&h_act, n_act, sizeof(int), cudaMemcpyDeviceToHost, st));
      NEGF_CUDA_CHECK(cudaStreamSynchronize(st));
    }
  }
  {
    ProfScope ps(PROF_OTHER, st);
    fp_finish_kernel<<<(batch + 127) / 128, 128, 0, st>>>(active, status, iters, max_iter, batch);
    NEGF_LAUNCHED();
  }
  return 0;
}

size_t g_obc_workspace_bytes(int n_e, int bs) {
  size_t blk = a256(sizeof(z_t) * (size_t)2 * n_e * bs * bs);
  size_t solver = sancho_workspace_bytes(2 * n_e, bs);
  size_t memo = memo_workspace_bytes(MEMO_SURFACE, 2 * n_e, 1, bs);
  return 6 * blk + (solver > memo ? solver : memo) + 3 * a256(sizeof(int) * 2 * (size_t)n_e + 64);
}

int g_obc_apply(const GObcArgs& a, void* ws, size_t ws_bytes, cudaStream_t st) {
  if (a.n_e <= 0) return 0;
  if (a.n_b < 2) return -1;
  if (ws_bytes < g_obc_workspace_bytes(a.n_e, a.bs)) return -4;
  const int ne = a.n_e, bs = a.bs, nb = a.n_b;
  const long long n2 = (long long)bs * bs, sd = (long long)nb * n2, so = (long long)(nb - 1) * n2;
  const size_t half = sizeof(z_t) * (size_t)ne * n2;
  const size_t blk = a256(2 * half);
  char* w = reinterpret_cast<char*>(ws);
  z_t* cm = (z_t*)w; w += blk;
  z_t* cn = (z_t*)w; w += blk;
  z_t* cnp = (z_t*)w; w += blk;
  z_t* xr = (z_t*)w; w += blk;
  z_t* t1 = (z_t*)w; w += blk;
  z_t* sig = (z_t*)w; w += blk;
  int* has_buf = (int*)w; w += a256(sizeof(int) * 2 * (size_t)ne + 64);
  int* need = (int*)w; w += a256(sizeof(int) * 2 * (size_t)ne + 64);
  int* used_buf = (int*)w; w += a256(sizeof(int) * 2 * (size_t)ne + 64);
  void* sws = w;
  size_t sbytes = ws_bytes - (size_t)(w - reinterpret_cast<char*>(ws));
  // gather contact cells: side 0 = left (corner 0), side 1 = right (corner n_b-1)
  auto gather = [&](z_t* dst, const z_t* src, long long stride) -> int {
    NEGF_CUDA_CHECK(cudaMemcpy2DAsync(dst, n2 * sizeof(z_t), src, stride * sizeof(z_t), n2 * sizeof(z_t),
                                      ne, cudaMemcpyDeviceToDevice, st));
    return 0;
  };
  const long long hn = (long long)ne * n2;
  RC(gather(cm, a.m_diag, sd));                          // M_00
  RC(gather(cm + hn, a.m_diag + (nb - 1) * n2, sd));     // M_{N-1,N-1}
  RC(gather(cn, a.m_lower, so));                         // n  = M_10
  RC(gather(cn + hn, a.m_upper + (nb - 2) * n2, so));    // n  = M_{N-2,N-1}
  RC(gather(cnp, a.m_upper, so));                        // n' = M_01
  RC(gather(cnp + hn, a.m_lower + (nb - 2) * n2, so));   // n' = M_{N-1,N-2}
  if (a.x_surface) {  // surfaces supplied by the caller (Beyn / fixed point, scba.py:577-614)
    NEGF_CUDA_CHECK(cudaMemcpyAsync(xr, a.x_surface, 2 * half, cudaMemcpyDeviceToDevice, st));
    NEGF_CUDA_CHECK(cudaMemsetAsync(a.status, 0, sizeof(int) * 2 * ne, st));
    NEGF_CUDA_CHECK(cudaMemsetAsync(a.iters, 0, sizeof(int) * 2 * ne, st));
  } else if (a.memo_cache) {
    // refresh cached surfaces first (staged through t1); Sancho only where rejected
    RC(memo_gather(a.memo_cache, a.memo_ld, a.memo_has, a.memo_ld, 2, ne, bs, t1, has_buf, st));
    RC(memo_refresh(MEMO_SURFACE, 2 * ne, 1, bs, cm, cn, cnp, nullptr, nullptr, a.n_fpi, a.memo_tol, t1,
                    has_buf, xr, need, used_buf, sws, sbytes, st));
    RC(sancho_batched(cm, cn, cnp, 2 * ne, bs, a.tol, a.max_iter, xr, a.status, a.iters, a.resid, sws,
                      sbytes, st, need));
    RC(memo_store(xr, used_buf, 2, ne, bs, a.memo_cache, a.memo_ld, a.memo_has, a.memo_used, a.memo_ld, st));
  } else {
    RC(sancho_batched(cm, cn, cnp, 2 * ne, bs, a.tol, a.max_iter, xr, a.status, a.iters, a.resid, sws,
                      sbytes, st));
  }
  // Sigma^R_obc = n x n'
  ZGemmDesc d = zdesc_default();
  d.M = bs; d.N = bs; d.batch = 2 * ne;
  d.t[0] = zterm(cn, n2, bs, OP_N, xr, n2, bs, OP_N, bs);
  d.t[1] = d.t[0];
  d.D = t1; d.sD = n2; d.ldd = bs;
  RC(zgemm_launch(d, st));
  d.t[0] = zterm(t1, n2, bs, OP_N, cnp, n2, bs, OP_N, bs);
  d.t[1] = d.t[0];
  d.D = sig;
  RC(zgemm_launch(d, st));
  const int tiles = ((bs + 31) / 32) * ((bs + 31) / 32);
  dim3 grid(tiles, ne), block(32, 8);
  {
    ProfScope ps_g_corner_kernel(PROF_OTHER, (cudaStream_t)(st));
    g_corner_kernel<<<grid, block, 0, st>>>(sig, bs, a.f_left, a.m_diag, a.bl_diag, a.bg_diag, sd,
                                            a.sl_left, a.sg_left);
    NEGF_LAUNCHED();
  }
  const long long cc = (long long)(nb - 1) * n2;
  {
    ProfScope ps_g_corner_kernel(PROF_OTHER, (cudaStream_t)(st));
    g_corner_kernel<<<grid, block, 0, st>>>(sig + hn, bs, a.f_right, a.m_diag + cc,
                                            a.bl_diag ? a.bl_diag + cc : nullptr,
                                            a.bg_diag ? a.bg_diag + cc : nullptr, sd, a.sl_right,
                                            a.sg_right);
    NEGF_LAUNCHED();
  }
  return 0;
}

size_t sigma_lg_obc_workspace_bytes(int batch, int bs) {
  return 2 * a256(sizeof(z_t) * (size_t)batch * bs * bs);
}

int sigma_lg_obc_batched(const z_t* x, const z_t* n, const z_t* np, const double* f, int batch,
                         int bs, z_t* sr, z_t* sl, z_t* sg, void* ws, size_t ws_bytes,
                         cudaStream_t st) {
  if (batch <= 0) return 0;
  if (ws_bytes < sigma_lg_obc_workspace_bytes(batch, bs)) return -4;
  const long long n2 = (long long)bs * bs;
  z_t* t1 = (z_t*)ws;
  z_t* sig = sr ? sr : (z_t*)((char*)ws + a256(sizeof(z_t) * (size_t)batch * n2));
  ZGemmDesc d = zdesc_default();
  d.M = bs; d.N = bs; d.batch = batch;
  d.t[0] = zterm(n, n2, bs, OP_N, x, n2, bs, OP_N, bs);
  d.t[1] = d.t[0];
  d.D = t1; d.sD = n2; d.ldd = bs;
  RC(zgemm_launch(d, st));
  d.t[0] = zterm(t1, n2, bs, OP_N, np, n2, bs, OP_N, bs);
  d.t[1] = d.t[0];
  d.D = sig;
  RC(zgemm_launch(d, st));
  const int tiles = ((bs + 31) / 32) * ((bs + 31) / 32);
  dim3 grid(tiles, batch), block(32, 8);
  {
    ProfScope ps_sigma_lg_kernel(PROF_OTHER, (cudaStream_t)(st));
    sigma_lg_kernel<<<grid, block, 0, st>>>(sig, bs, f, sl, sg);
    NEGF_LAUNCHED();
  }
  return 0;
}

int g_assemble(const GAssembleArgs& a, cudaStream_t st) {
  if (a.n_e <= 0) return 0;
  const long long n2 = (long long)a.bs * a.bs;
  int bx = (int)((n2 + 255) / 256);
  if (bx > 64) bx = 64;
  dim3 grid(bx, a.n_b, a.n_e);
  {
    ProfScope ps_g_assemble_kernel(PROF_OTHER, (cudaStream_t)(st));
    g_assemble_kernel<<<grid, 256, 0, st>>>(a);
    NEGF_LAUNCHED();
  }
  return 0;
}

}  // namespace negf
