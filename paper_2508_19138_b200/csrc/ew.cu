// Elementwise block kernels (HBM-bound; 32x32 tiles staged through smem so
// the conjugate-transposed reads stay coalesced).
#include "ew.cuh"
#include "prof.cuh"

namespace negf {

namespace {

constexpr int TILE = 32;

__global__ void ew_kernel(const __grid_constant__ EwGroup g) {
  __shared__ z_t tile[TILE][TILE + 1];
  const EwDesc& d = g.d[blockIdx.z];
  const int b = blockIdx.y;
  if (b >= d.batch) return;
  const int tiles_c = (g.cols + TILE - 1) / TILE;
  const int r0 = (blockIdx.x / tiles_c) * TILE, c0 = (blockIdx.x % tiles_c) * TILE;
  const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
  z_t acc[TILE / 8];
#pragma unroll
  for (int k = 0; k < TILE / 8; ++k) acc[k] = make_double2(0.0, 0.0);
  for (int t = 0; t < d.nterms; ++t) {
    const z_t* X = d.X[t] + (long long)b * d.sX[t];
    const double2 cf = d.coef[t];
    if (!d.opH[t]) {
#pragma unroll
      for (int k = 0; k < TILE / 8; ++k) {
        int r = r0 + ty + 8 * k, c = c0 + tx;
        if (r < g.rows && c < g.cols) acc[k] = zadd(acc[k], zmul(cf, X[(long long)r * g.cols + c]));
      }
    } else {
      // X^dag[r][c] = conj(X[c][r]); X is cols x rows
      __syncthreads();
#pragma unroll
      for (int k = 0; k < TILE / 8; ++k) {
        int xr = c0 + ty + 8 * k, xc = r0 + tx;  // row of X = output col
        if (xr < g.cols && xc < g.rows) tile[ty + 8 * k][tx] = X[(long long)xr * g.rows + xc];
      }
      __syncthreads();
#pragma unroll
      for (int k = 0; k < TILE / 8; ++k) {
        int r = r0 + ty + 8 * k, c = c0 + tx;
        if (r < g.rows && c < g.cols)
          acc[k] = zadd(acc[k], zmul(cf, zconj(tile[tx][ty + 8 * k])));
      }
    }
  }
  z_t* out = d.out + (long long)b * d.sOut;
#pragma unroll
  for (int k = 0; k < TILE / 8; ++k) {
    int r = r0 + ty + 8 * k, c = c0 + tx;
    if (r < g.rows && c < g.cols) out[(long long)r * g.cols + c] = acc[k];
  }
}

// Tile pair (I, J), I <= J, handled by one CTA so the in-place update is race free.
__global__ void antiherm_kernel(z_t* X, long long sX, int n) {
  __shared__ z_t a[TILE][TILE + 1], bt[TILE][TILE + 1];
  const int nt = (n + TILE - 1) / TILE;
  // decode linear upper-triangular tile index
  int idx = blockIdx.x, I = 0;
  while (idx >= nt - I) { idx -= nt - I; ++I; }
  const int J = I + idx;
  z_t* x = X + (long long)blockIdx.y * sX;
  const int tx = threadIdx.x, ty = threadIdx.y;
  for (int k = ty; k < TILE; k += 8) {
    int r = I * TILE + k, c = J * TILE + tx;
    if (r < n && c < n) a[k][tx] = x[(long long)r * n + c];
    r = J * TILE + k; c = I * TILE + tx;
    if (r < n && c < n) bt[k][tx] = x[(long long)r * n + c];
  }
  __syncthreads();
  for (int k = ty; k < TILE; k += 8) {
    // block (I,J) element (k, tx): (a[k][tx] - conj(bt[tx][k]))/2
    int r = I * TILE + k, c = J * TILE + tx;
    if (r < n && c < n) {
      z_t v = a[k][tx], w = bt[tx][k];
      x[(long long)r * n + c] = make_double2(0.5 * (v.x - w.x), 0.5 * (v.y + w.y));
    }
    if (I != J) {
      r = J * TILE + k; c = I * TILE + tx;
      if (r < n && c < n) {
        z_t v = bt[k][tx], w = a[tx][k];
        x[(long long)r * n + c] = make_double2(0.5 * (v.x - w.x), 0.5 * (v.y + w.y));
      }
    }
  }
}

__global__ void add_identity_kernel(z_t* Y, long long sY, int n, double2 s) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  z_t* y = Y + (long long)blockIdx.y * sY + (long long)i * n + i;
  y->x += s.x;
  y->y += s.y;
}

}  // namespace

int ew_group_launch(const EwGroup& g, cudaStream_t stream) {
  if (g.n <= 0) return 0;
  int mb = 0;
  for (int i = 0; i < g.n; ++i) mb = g.d[i].batch > mb ? g.d[i].batch : mb;
  if (mb == 0) return 0;
  const int tiles = ((g.rows + TILE - 1) / TILE) * ((g.cols + TILE - 1) / TILE);
  dim3 grid(tiles, mb, g.n), block(TILE, 8);
  ProfScope ps_(PROF_EW, stream);
  ew_kernel<<<grid, block, 0, stream>>>(g);
  NEGF_LAUNCHED();
  return 0;
}

int antiherm_inplace(z_t* X, long long sX, int n, int batch, cudaStream_t stream) {
  if (batch <= 0) return 0;
  const int nt = (n + TILE - 1) / TILE;
  dim3 grid(nt * (nt + 1) / 2, batch), block(TILE, 8);
  ProfScope ps_(PROF_EW, stream);
  antiherm_kernel<<<grid, block, 0, stream>>>(X, sX, n);
  NEGF_LAUNCHED();
  return 0;
}

int add_identity(z_t* Y, long long sY, int n, int batch, double2 s, cudaStream_t stream) {
  if (batch <= 0) return 0;
  dim3 grid((n + 127) / 128, batch);
  ProfScope ps_(PROF_EW, stream);
  add_identity_kernel<<<grid, 128, 0, stream>>>(Y, sY, n, s);
  NEGF_LAUNCHED();
  return 0;
}

}  // namespace negf

extern "C" int negf_greater_from_identity(int n_e, int n_b, int bs, const void* xl_diag,
                                          const void* xl_upper, const void* xr_diag,
                                          const void* xr_upper, const void* xr_lower,
                                          void* xg_diag, void* xg_upper, void* stream) {
  using namespace negf;
  if (n_e < 0 || n_b < 1 || bs < 1 || !xl_diag || !xr_diag || !xg_diag) return -1;
  if (n_b > 1 && (!xl_upper || !xr_upper || !xr_lower || !xg_upper)) return -1;
  if (n_e == 0) return 0;
  const long long n2 = (long long)bs * bs;
  EwGroup g;
  g.n = 0; g.rows = bs; g.cols = bs;
  auto add = [&](z_t* out, const z_t* l, const z_t* r, const z_t* rh, int batch) {
    EwDesc& d = g.d[g.n++];
    d.batch = batch; d.nterms = 3; d.out = out; d.sOut = n2;
    d.X[0] = l; d.sX[0] = n2; d.opH[0] = 0; d.coef[0] = make_double2(1, 0);
    d.X[1] = r; d.sX[1] = n2; d.opH[1] = 0; d.coef[1] = make_double2(1, 0);
    d.X[2] = rh; d.sX[2] = n2; d.opH[2] = 1; d.coef[2] = make_double2(-1, 0);
  };
  // X^>_ii = X^<_ii + X^R_ii - X^R_ii^dag ; X^>_{i,i+1} = X^<_{i,i+1} + X^R_{i,i+1} - X^R_{i+1,i}^dag
  add((z_t*)xg_diag, (const z_t*)xl_diag, (const z_t*)xr_diag, (const z_t*)xr_diag, n_e * n_b);
  if (n_b > 1)
    add((z_t*)xg_upper, (const z_t*)xl_upper, (const z_t*)xr_upper, (const z_t*)xr_lower,
        n_e * (n_b - 1));
  return ew_group_launch(g, (cudaStream_t)stream);
}
