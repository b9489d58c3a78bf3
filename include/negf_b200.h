/* negf_b200 -- C ABI of the B200-native NEGF+GW hot path (sm_100a).
 *
 * Plain pointers and sizes only. Every matrix argument is a DEVICE pointer to
 * complex128 data stored interleaved (re, im), row-major, energy-major packed:
 *   diagonal blocks   [n_e][n_b][bs][bs]
 *   off-diagonal      [n_e][n_b-1][bs][bs]
 * which is the memory layout of a contiguous torch.complex128 tensor of that
 * shape. `stream` is a cudaStream_t (NULL = legacy default stream). All calls
 * are stream-ordered and asynchronous; they return 0 on success, a CUDA error
 * code (>0) on launch failure, or a negative code on invalid arguments.
 * Caller owns all buffers, including the workspace (query its size first).
 * No global mutable state beyond per-kernel attribute setup: calls are
 * reentrant across threads and streams.
 */
#ifndef NEGF_B200_H
#define NEGF_B200_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ABI version (major*100 + minor). */
int negf_abi_version(void);

/* Complex block-product algorithm of the DMMA GEMM (process-wide):
 * 2 = 3M/Gauss, 3 real products per complex product (default; cp.async
 *     operand staging, TMA-engine bulk copies + mbarrier ring for complex
 *     products with M >= 512),
 * 3 = 3M with the bulk-copy kernel for every product,
 * 0 = 4 real products (the textbook arithmetic). Anything else: -1.
 * 3M trades ~25% of the FP64 tensor work for a normwise error bound that is
 * still O(eps |A||B|). */
int negf_set_gemm_algo(int algo);

/* Forward-sweep pipelining of negf_rgf_selected_solve_batched (process-wide,
 * default 1): the Keldysh (lesser/greater) forward products run on an
 * internal second stream so they overlap the retarded chain's pivoted
 * inversions. 0 serialises everything on the caller's stream. */
int negf_set_rgf_overlap(int on);

/* ---- (1) selected solve -------------------------------------------------
 * Replaces negfgw.rgf.selected_solve (pkg/src/negfgw/rgf.py:232-243) and, with
 * symmetrize bit 0, the SelectedSolution.symmetrize() that scba_run applies
 * after it (scba.py:987,1087; rgf.py:82-88), for a batch of n_e energies.
 * symmetrize bit 1 declares the B^lg diagonal blocks anti-Hermitian (as every
 * lg source of the NEGF/GW solver is): the anti-Hermitian forward products
 * then run on the lower-triangle tiles only.
 *   M X^R = I,  M X^lg M^dag = B^lg  (selected blocks).
 * b_lesser / b_greater are lg-compressed (diag + upper; lower implied by
 * B[i+1][i] = -B[i][i+1]^dag, blocks.py:110-118); pass NULL for an absent
 * kind (its outputs are then not touched).
 * status[n_e] (device int): 0, or 1 + forward step of the first singular
 * Schur complement (rgf.py:121-126 SingularBlockError). u_spread[n_e][n_b]
 * (device double, may be NULL): LU pivot spread per step (rgf.py:44-49).
 * Blocks up to 4096 orbitals are inverted by the pivoted Gauss-Jordan
 * kernels (LAPACK zgetf2 pivot order over the whole column; one-CTA register
 * panel up to 512, thread-block-cluster panel above). */
size_t negf_rgf_workspace_bytes(int n_e, int n_b, int bs);
int negf_rgf_selected_solve_batched(
    int n_e, int n_b, int bs,
    const void* m_diag, const void* m_upper, const void* m_lower,
    const void* bl_diag, const void* bl_upper,
    const void* bg_diag, const void* bg_upper,
    void* xr_diag, void* xr_upper, void* xr_lower,
    void* xl_diag, void* xl_upper,
    void* xg_diag, void* xg_upper,
    int symmetrize, int* status, double* u_spread,
    void* workspace, size_t workspace_bytes, void* stream);

/* The two sweeps separately (spatial-decomposition building blocks,
 * dist.py:529-533, 647-681):
 *   mode 1: forward only. x_fwd (rgf.py:113-129) is written to xr_diag and
 *           xl_fwd / xg_fwd (rgf.py:132-149) to xl_diag / xg_diag. With
 *           fwd_given = 1, xr_diag already holds x_fwd on entry and only the
 *           lesser/greater recursion runs (forward_lg with a given RetardedPass).
 *   mode 2: backward only (rgf.py:152-229). On entry xr_diag / xl_diag / xg_diag
 *           hold x_fwd / xl_fwd / xg_fwd; a caller-written last block acts as
 *           the x_last seed of rgf_retarded / rgf_lesser_greater.
 *   mode 0: both (= negf_rgf_selected_solve_batched).
 * Same workspace as negf_rgf_selected_solve_batched. */
int negf_rgf_sweeps_batched(int mode, int fwd_given, int n_e, int n_b, int bs,
                            const void* m_diag, const void* m_upper, const void* m_lower,
                            const void* bl_diag, const void* bl_upper,
                            const void* bg_diag, const void* bg_upper,
                            void* xr_diag, void* xr_upper, void* xr_lower,
                            void* xl_diag, void* xl_upper, void* xg_diag, void* xg_upper,
                            int symmetrize, int* status, double* u_spread,
                            void* workspace, size_t workspace_bytes, void* stream);

/* Greater selected blocks from the lesser and retarded ones:
 *   X^>_ii = X^<_ii + X^R_ii - X^R_ii^dag,  X^>_{i,i+1} = X^<_{i,i+1} + X^R_{i,i+1} - X^R_{i+1,i}^dag,
 * exact for the carrier system because its sources satisfy
 * B^> - B^< = M^dag - M (bath construction, scba.py:16-19, 706-716; contact and
 * scattering self-energies obey the same identity). Opt-in replacement of the
 * greater Keldysh recursion; NOT valid for the W system. */
int negf_greater_from_identity(int n_e, int n_b, int bs, const void* xl_diag,
                               const void* xl_upper, const void* xr_diag, const void* xr_upper,
                               const void* xr_lower, void* xg_diag, void* xg_upper, void* stream);

/* ---- dense block primitives (negfgw/_linalg.py:19-64) --------------------
 * D[b] = alpha*op(A[b])op(B[b]) + beta*C[b]; op: 0=N 1=T 2=conj 3=conj-trans.
 * Replaces _linalg.gemm (_linalg.py:19-22), batched. C may be NULL. */
int negf_zgemm_batched(int m, int n, int k, int batch,
                       double alpha_re, double alpha_im,
                       const void* a, long long stride_a, int lda, int op_a,
                       const void* b, long long stride_b, int ldb, int op_b,
                       double beta_re, double beta_im,
                       const void* c, long long stride_c, int ldc,
                       void* d, long long stride_d, int ldd, void* stream);

/* Batched pivoted inverse, replaces _linalg.invert (_linalg.py:30-52):
 * partial pivoting over the whole remaining column with LAPACK zgetf2's
 * choice (max |re|+|im|, first index on ties), u_spread[b] (may be NULL) =
 * max|U_jj| / min|U_jj| like scipy's LU. n <= 64: one CTA in smem;
 * n <= 512: one CTA per matrix with the panel in registers; 512 < n <= 4096:
 * a thread-block cluster of up to 16 CTAs (256 rows each; non-portable
 * cluster size above 8) per matrix exchanging the pivot
 * candidates through distributed shared memory (also used for 256 < n <= 512
 * when batch >= 64); n > 4096 returns -5.
 * s (n x n packed, stride n*n) is destroyed for n > 64. status[b] = 1 on an
 * exactly-zero or non-finite pivot. */
size_t negf_zinv_workspace_bytes(int n, int batch);
int negf_zinv_batched(int n, int batch, void* s, void* x, int* status, double* u_spread,
                      void* workspace, size_t workspace_bytes, void* stream);


/* ---- (2) open boundary conditions (negfgw/obc.py) -------------------------
 * Sancho-Rubio decimation for `batch` surface problems x = (m - n x n')^-1,
 * replaces obc_sancho_rubio (obc.py:144-182), including its stopping rule
 * |a|_F + |b|_F < tol * max(|n|_F, |n'|_F) and the closing recursion-residual
 * check (> 10 max(tol, 1e-14) fails). m, n, np, x: [batch][bs][bs] device.
 * status[b] (device int): 0 ok, 1 singular block, 2 not converged in
 * max_iter sweeps, 3 residual check failed. iters[b]: sweeps used;
 * resid[b] (may be NULL): recursion residual. Converged problems are masked
 * on the device after every sweep; the host reads the active count (one
 * stream synchronisation) every 4 sweeps. */
size_t negf_sancho_workspace_bytes(int batch, int bs);
int negf_obc_sancho_batched(int batch, int bs, const void* m, const void* n, const void* np,
                            double tol, int max_iter, void* x, int* status, int* iters,
                            double* resid, const int* select, void* workspace,
                            size_t workspace_bytes, void* stream);
/* select[batch] (device int, may be NULL = all): solve only problems with
 * select[b] != 0; the others keep x and get status 0, iters 0 (the direct leg
 * of the memoizer below). */

/* obc_fixed_point (obc.py:108-135), batched: x <- (m - n x n')^-1 from x0
 * (NULL = zeros) until |x_new - x|_F / |x_new|_F < tol; status as Sancho's
 * (1 singular update, 2 not converged in max_iter), iters, resid (may be NULL:
 * the final relative update). Synchronises `stream` every 16 updates. */
size_t negf_fixed_point_workspace_bytes(int batch, int bs);
int negf_obc_fixed_point_batched(int batch, int bs, const void* m, const void* n, const void* np, const void* x0,
                                 double tol, int max_iter, void* x, int* status, int* iters, double* resid,
                                 void* workspace, size_t workspace_bytes, void* stream);

/* sigma_lg_obc (obc.py:460-486), batched: Sigma^R = n x n',
 * Sigma^< = -f (Sigma^R - Sigma^R^dag), Sigma^> = (1-f)(Sigma^R - Sigma^R^dag)
 * with f[b] = fermi(E_b - mu) (device double). Outputs may be NULL. */
size_t negf_sigma_lg_obc_workspace_bytes(int batch, int bs);
int negf_sigma_lg_obc_batched(int batch, int bs, const void* x, const void* n, const void* np,
                              const double* f, void* sigma_r, void* sigma_lesser,
                              void* sigma_greater, void* workspace, size_t workspace_bytes,
                              void* stream);

/* stein_geometric (obc.py:427-447) for `batch` problems w - a w a^dag = q by
 * squared doubling, stopping at |a_k w a_k^dag|_F < tol max(|w|_F, 1e-300).
 * v0[bs] (device complex128): start vector of the spectral-radius power
 * iteration (obc.py:320-342: numpy default_rng(5), normal re + i normal im,
 * normalised). status[b]: 0 ok, 2 not converged, 4 spectral radius estimate
 * >= 1 (SpectralRadiusError; the Kronecker fallback of scba.py:534-543 is not
 * ported). bs <= 6000. */
size_t negf_stein_workspace_bytes(int batch, int bs);
int negf_stein_batched(int batch, int bs, const void* a, const void* q, void* w, double tol,
                       int max_iter, const void* v0, int* status, int* iters, const int* select,
                       void* workspace, size_t workspace_bytes, void* stream);

/* Beyn contour moments (obc_beyn, obc.py:198-296, nearest-neighbour stencil
 * [n', m, n]) for `batch` surface problems: a0 = sum_k w_k P(z_k)^-1 probe,
 * a1 = sum_k w_k z_k P(z_k)^-1 probe with P(z) = n' + z m + z^2 n. z, w: HOST
 * arrays of n_quad complex numbers (interleaved re, im); probe [bs][bs]
 * device (the seeded probe, numpy default_rng(1278)). status[b] = 1 + k when
 * P(z_k) is singular (the reference's "contour node" SingularBlockError).
 * The SVD / eigen / pseudo-inverse steps follow in obc.py. */
size_t negf_beyn_workspace_bytes(int batch, int bs);
int negf_beyn_moments(int batch, int bs, int n_quad, const void* m, const void* n, const void* np,
                      const double* z, const double* w, const void* probe, void* a0, void* a1,
                      int* status, void* workspace, size_t workspace_bytes, void* stream);

/* Runtime OBC memoizer, batched: the refresh leg of memoized_obc
 * (obc.py:519-600; _memo_refresh :551-600). map 0 = surface fixed point
 * x <- (m - n x n')^-1 (fixed_point_step, obc.py:138-141; n_kind must be 1),
 * map 1 = Stein map w <- q + a w a^dag (scba.py:653-655) for n_kind kinds
 * sharing a[s] (problem p = k*n_side + s, q[p]). x0[p]: cached block, used
 * where has[p] != 0. Per problem: two trial updates give delta1, delta2,
 * rho = delta2/delta1 and tail = rho/(1-rho); refresh only if
 * delta2 rho^(n_fpi-2) tail < tol, stopping once last*tail < tol within
 * n_fpi updates. Accepted iterates go to out[p] with used[p] = 1; every
 * other problem (no cache, non-finite or singular update, rho >= 1, budget
 * spent) gets need_direct[p] = 1 for the caller's direct solve (Sancho /
 * Stein with select = need_direct). Synchronises `stream` once per update. */
size_t negf_memo_workspace_bytes(int map, int n_side, int n_kind, int bs);
int negf_memo_refresh_batched(int map, int n_side, int n_kind, int bs, const void* m, const void* n,
                              const void* np, const void* a, const void* q, int n_fpi, double tol,
                              const void* x0, const int* has, void* out, int* need_direct, int* used,
                              void* workspace, size_t workspace_bytes, void* stream);

/* Carrier-side contact closure of an assembled batch (scba.py:755-774):
 * for the left (corner 0) and right (corner n_b-1) leads, solve the surface
 * problem by Sancho-Rubio on the contact cell of M (scba.py:558-574), then
 * M_cc -= Sigma^R_obc, B^<_cc += Sigma^<_obc, B^>_cc += Sigma^>_obc in place.
 * f_left/f_right[n_e]: contact occupations. sl/sg_left/right [n_e][bs][bs]
 * (may be NULL) receive the boundary lesser/greater self-energies.
 * status/iters/resid: [2][n_e] (left block first). */
size_t negf_g_obc_workspace_bytes(int n_e, int bs);
int negf_g_obc_apply(int n_e, int n_b, int bs, void* m_diag, const void* m_upper,
                     const void* m_lower, void* bl_diag, void* bg_diag, const double* f_left,
                     const double* f_right, double tol, int max_iter, void* sl_left,
                     void* sg_left, void* sl_right, void* sg_right, int* status, int* iters,
                     double* resid, void* memo_cache, int* memo_has, int* memo_used,
                     long long memo_ld, int n_fpi, double memo_tol, const void* x_surface,
                     void* workspace, size_t workspace_bytes, void* stream);
/* Memoizer (optional; memo_cache NULL = direct Sancho for every problem, the
 * reference with MemoizerOptions(enabled=False)): memo_cache holds the cached
 * surface of side g (0 left, 1 right) and batch energy e at block
 * g*memo_ld + e (memo_ld >= n_e: the caller's energies per side, pointer
 * already offset to this batch); memo_has/memo_used [2][memo_ld] ints. Cached
 * problems are refreshed (negf_memo_refresh_batched, n_fpi, memo_tol), the
 * rest solved by Sancho; every result is written back to the cache
 * (has = 1) and used[] = 1 marks memoized calls (the reference's
 * cache.stats). x_surface (optional, [2][n_e][bs][bs]): surface blocks from
 * the caller's solver (Beyn / fixed point, scba.py:577-614); replaces the
 * Sancho and memoizer step. */

/* Carrier system assembly (scba.py:670-727) for n_e energies:
 *   M_ii = (E + i eta) I - H_ii - SR_ii,  M_{i,i+-1} = -H - SR,
 *   B^<_ii = 2 i eta f I + SL_ii, B^>_ii = -2 i eta (1-f) I + SG_ii, B_{i,i+1} = S_{i,i+1}.
 * h_*: energy-independent blocks [n_b or n_b-1][bs][bs]; energy, f_bath:
 * [n_e] device doubles; scattering self-energies s*_ (energy-major blocks)
 * may be NULL (ballistic). Lesser/greater outputs may be NULL. */
int negf_g_assemble(int n_e, int n_b, int bs, const void* h_diag, const void* h_upper,
                    const void* h_lower, const double* energy, const double* f_bath, double eta,
                    const void* sr_diag, const void* sr_upper, const void* sr_lower,
                    const void* sl_diag, const void* sl_upper, const void* sg_diag,
                    const void* sg_upper, void* m_diag, void* m_upper, void* m_lower,
                    void* bl_diag, void* bl_upper, void* bg_diag, void* bg_upper, void* stream);

/* ---- observables (scba.py:1313-1376), reduced on the device -------------
 * Per energy e and block b: tr_gr[e][b] = tr G^R_bb, tr_gl[e][b] = tr G^<_bb
 * (complex); current_spectrum[e][b] (b < n_b-1, double) as
 * scba.current_spectrum; terminal[e][0|1] = tr(S^<_c G^>_cc) - tr(S^>_c G^<_cc)
 * at the left / right corner (complex). Optional outputs may be NULL. */
int negf_observables(int n_e, int n_b, int bs, const void* gr_diag, const void* gl_diag,
                     const void* gg_diag, const void* gl_upper, const void* h_upper,
                     const void* sl_left, const void* sg_left, const void* sl_right,
                     const void* sg_right, void* tr_gr, void* tr_gl, double* current_spectrum,
                     void* terminal, void* stream);

/* ---- (3) energy convolutions (negfgw/convolve.py) -----------------------
 * Entry-major series: row r of an array is the energy series of one matrix
 * entry, x[r][0..n_e) complex128, rows contiguous (stride n_e).
 * L: power-of-two circular length >= max(8, 2 n_e - 1); L <= 4096 on one CTA
 * per row, L = 8192 (n_e <= 4096) for the fused P / Sigma kernels on a
 * cluster pair of CTAs (even / odd frequency bins, halves combined through
 * distributed shared memory); larger L returns -1 / -5.
 * tw[L] = exp(-2 pi i k/L).
 * kf/kcf[L]: spectrum (natural order) of the causal kernel
 * K = ifft_m(theta), m = scipy next_fast_len(2 n_e) made even, and of conj(K),
 * laid out circularly on L (see paper_2508_19138_b200/conv.py ConvPlan).
 * diag[r] (uint8, may be NULL): 1 for row == col entries, which are projected
 * to their imaginary part (scba.py:406-409).
 *
 * Polarization, fused (scba.py:1035-1048):
 *   P^<[k] = scale sum_m G^<[m] (-conj G^>[m-k]),  P^>[k] = scale sum_m G^>[m] (-conj G^<[m-k])
 *   (scale = C_POLARIZATION * dE), projection, P^R_up = retarded(P^<, P^>),
 *   P^R_lo = retarded(-conj P^<, -conj P^>). */
int negf_conv_polarization(long long n_rows, int n_e, int L, const void* gl, const void* gg,
                           const void* tw, const void* kf, const void* kcf,
                           const unsigned char* diag, double scale_re, double scale_im, void* pl,
                           void* pg, void* pr_up, void* pr_lo, void* stream);
/* Self-energy, fused (scba.py:1118-1132): Sigma^<>[k] = scale sum_m G^<>[k-m] W^<>[m]
 * with W rows gathered through w_rows[r] (int64, may be NULL = identity;
 * the w_to_g map of scba.py:933-937), projection, retarded upper/lower. */
int negf_conv_sigma(long long n_rows, int n_e, int L, const void* gl, const void* gg,
                    const void* wl, const void* wg, const long long* w_rows, const void* tw,
                    const void* kf, const void* kcf, const unsigned char* diag, double scale_re,
                    double scale_im, void* sl, void* sg, void* sr_up, void* sr_lo, void* stream);
/* convolve_energy (convolve.py:39-71): mode 0 convolution, 1 correlation. */
int negf_convolve_energy(long long n_rows, int n_e, int L, const void* x1, const void* x2,
                         int mode, double scale_re, double scale_im, const void* tw, void* out,
                         void* stream);
/* retarded_from_lg (convolve.py:101-129). */
int negf_retarded_from_lg(long long n_rows, int n_e, int L, const void* x_lesser,
                          const void* x_greater, const void* tw, const void* kf, void* out,
                          void* stream);

/* ---- (4) energy <-> entry layout switch (K11/K12) -------------------------
 * Compressed bandwidth-3 EntryPattern (convolve.py:135-187): per block row bi,
 * the upper triangle (row-major, r <= c) of block (bi,bi), then block
 * (bi,bi+1) row-major; n_entries = n_b bs(bs+1)/2 + (n_b-1) bs^2.
 * tri_q[bs(bs+1)/2] (device int32) = r*bs + c of the triangle entries in order.
 * Entry-major arrays are (n_entries, ld) row-major; columns e0..e0+n_e-1 are
 * read/written. Blocks are energy-major [n_e][n_b(-1)][bs][bs]. */
long long negf_pattern_entries(int n_b, int bs);
/* _gather_entries (scba.py:252-271) for n_e energies at once. */
int negf_pack_lg(int n_e, int n_b, int bs, const int* tri_q, const void* x_diag,
                 const void* x_upper, void* out, long long ld, int e0, void* stream);
/* _scatter_lg (scba.py:295-308): diagonal blocks get X[c][r] = -conj X[r][c]. */
/* negf_pack_lg fused with the E -> nnz redistribution (scba.py:342-368,
 * to_entry_major): entry row t goes to rank s with row_start[s] <= t <
 * row_start[s+1] (device array, n_ranks + 1 values), written into dest[s]
 * (device array of n_ranks device pointers -- peer memory mapped over NVLink,
 * e.g. symmetric-memory buffers) at row t - row_start[s], column col0 + e of
 * a row-major (rows, ld) complex128 array. n_ranks <= 16. The caller orders
 * the peers' reads after all writes (a cross-rank barrier). */
int negf_pack_lg_p2p(int n_e, int n_b, int bs, const int* tri_q, const void* x_diag, const void* x_upper,
                     int n_ranks, const unsigned long long* dest, const long long* row_start, long long ld,
                     int col0, void* stream);
/* nnz -> E redistribution fused with the unpack (scba.py:1053-1056 then
 * _scatter_lg / _scatter_retarded): entry row t is read from rank s
 * (row_start[s] <= t < row_start[s+1]) at row t - row_start[s], columns
 * col0 .. col0 + n_e of its (rows, ld) entry-major array src_upper[s]
 * (and src_lower[s] when retarded != 0: the retarded unpack), peer memory
 * over NVLink. Writes the n_e energies' blocks like negf_unpack_lg /
 * negf_unpack_retarded. n_ranks <= 16. */
int negf_unpack_p2p(int n_e, int n_b, int bs, const int* tri_q, int retarded, int n_ranks,
                    const unsigned long long* src_upper, const unsigned long long* src_lower,
                    const long long* row_start, long long ld, int col0, void* x_diag, void* x_upper,
                    void* x_lower, void* stream);
int negf_unpack_lg(int n_e, int n_b, int bs, const int* tri_q, const void* in, long long ld,
                   int e0, void* x_diag, void* x_upper, void* stream);
/* _scatter_retarded (scba.py:311-325): upper values at (r,c), lower values at
 * (c,r) (x_lower gets the (bi+1,bi) blocks; diagonal elements take the lower value). */
int negf_unpack_retarded(int n_e, int n_b, int bs, const int* tri_q, const void* in_upper,
                         const void* in_lower, long long ld, int e0, void* x_diag, void* x_upper,
                         void* x_lower, void* stream);

/* Table-driven layout for patterns / blockings other than the reference's
 * full compressed band on the stacks' own blocking: the paper's r_cut
 * nonzero subset of the band and the coarser W grid
 * bs_w = k bs of scba_run (scba.py:893-937: P scattered from the G pattern
 * into W blocks by _scatter_groups(pat_g, bs_w), W read back at G-pattern
 * coordinates through w_to_g). Entry t (of n_entries, any subset of the
 * compressed band in EntryPattern order) lives in block row bi = code[t] >> 1
 * of the diagonal (code & 1 == 0) or upper (== 1) stack of n_bt blocks of
 * bs_t orbitals, at flat offset q[t] = r bs_t + c; code and q are device
 * int32 arrays. Same mirror / write-order rules as negf_unpack_lg and
 * negf_unpack_retarded (retarded != 0). zero_fill != 0 clears the target
 * stacks first (entries outside the pattern are zero, like the reference's
 * zero-initialised scatter buffers). */
int negf_pack_lg_table(int n_e, long long n_entries, int n_bt, int bs_t, const int* code, const int* q,
                       const void* x_diag, const void* x_upper, void* out, long long ld, int e0, void* stream);
int negf_unpack_table(int n_e, long long n_entries, int n_bt, int bs_t, const int* code, const int* q,
                      int retarded, const void* in_upper, const void* in_lower, long long ld, int e0,
                      void* x_diag, void* x_upper, void* x_lower, int zero_fill, void* stream);

/* ---- (5) screened interaction W (scba.py:784-858) ------------------------
 * Assembly for n_e energies: M_W = I - trunc3(V P^R), B^<> = trunc3((V P^<>) V).
 * V blocks are energy independent (v_diag [n_b], v_upper/v_lower [n_b-1]);
 * P^R full (diag/upper/lower), P^<> lg-compressed (diag/upper, lower implied).
 * Only tridiagonal output blocks are formed. Workspace: 4 n_b blocks/energy. */
size_t negf_w_assemble_workspace_bytes(int n_e, int n_b, int bs);
int negf_w_assemble(int n_e, int n_b, int bs, const void* v_diag, const void* v_upper,
                    const void* v_lower, const void* pr_diag, const void* pr_upper,
                    const void* pr_lower, const void* pl_diag, const void* pl_upper,
                    const void* pg_diag, const void* pg_upper, void* m_diag, void* m_upper,
                    void* m_lower, void* bl_diag, void* bl_upper, void* bg_diag, void* bg_upper,
                    int v_real, void* workspace, size_t workspace_bytes, void* stream);
/* v_real bit 0: the caller guarantees imag(V) == 0 exactly (e.g. a real
 * Coulomb matrix); each V product then runs as a real x complex product
 * (2 real GEMMs instead of 3). Bit 1: V is Hermitian (v_diag[i] = v_diag[i]^H,
 * v_lower[i] = v_upper[i]^H) and the P^<> diagonal blocks are anti-Hermitian
 * (as every lg-compressed quantity of the solver is), so the diagonal source
 * blocks (V P V)_ii are anti-Hermitian and are formed on the lower-triangle
 * tiles only.
 * W contact closure in place (scba.py:839-858, _lead_lg_boundary :617-664):
 * Sancho surface block per side (status/iters [2][n_e], codes as
 * negf_obc_sancho_batched), geometric Stein per side and kind (stein_status/
 * stein_iters [2 kinds][2 sides][n_e]; 4 = spectral radius estimate >= 1,
 * 2 = not converged; v0 as in negf_stein_batched), corner source corrections, and
 * M_cc -= n x n'. */
size_t negf_w_obc_workspace_bytes(int n_e, int bs);
int negf_w_obc_apply(int n_e, int n_b, int bs, void* m_diag, const void* m_upper,
                     const void* m_lower, void* bl_diag, const void* bl_upper, void* bg_diag,
                     const void* bg_upper, double surface_tol, int max_sweeps, double stein_tol,
                     int stein_max_iter, const void* v0, int* status, int* iters,
                     int* stein_status, int* stein_iters, void* memo_r_cache, int* memo_r_has,
                     int* memo_r_used, void* memo_lg_cache, int* memo_lg_has, int* memo_lg_used,
                     long long memo_ld, int n_fpi_r, int n_fpi_lg, double memo_tol,
                     const void* x_surface, void* workspace, size_t workspace_bytes, void* stream);
/* Memoizer (optional, as for negf_g_obc_apply): memo_r_* cache the W
 * surfaces (key (W, side, e, R), [2 sides][memo_ld]), memo_lg_* the Stein
 * solutions (key (W, side, e, kind), [2 kinds][2 sides][memo_ld]); budgets
 * n_fpi_r / n_fpi_lg (SurfaceCache.n_fpi, obc.py:504-512).
 * x_surface (optional, [2][n_e][bs][bs]): retarded surface blocks computed by
 * the caller (the reference's Beyn solve, scba.py:844); replaces the Sancho /
 * memoized surface step. */

/* ---- (5b) spatial domain decomposition (negfgw/dist.py) ------------------
 * Partition-local pieces of dist_selected_solve (dist.py:622-717) for a
 * batch of n_e energies; the caller (paper_2508_19138_b200/dd.py) runs one
 * partition per GPU, all-gathers the boundary contributions over NCCL and
 * solves the reduced chain (dist.py:486-561) on every rank with
 * negf_rgf_sweeps_batched / negf_rgf_selected_solve_batched. Inputs are the
 * partition's own energy-major stacks (w blocks; upper/lower w-1); source
 * kinds may be NULL. Workspace: negf_dd_workspace_bytes(n_e, bs). */
size_t negf_dd_workspace_bytes(int n_e, int bs);
/* _schur_tail (dist.py:365-385): after the forward sweep of an end
 * partition (x_fwd / xl_fwd / xg_fwd = the forward diagonal stacks),
 * s = M[w-1,w-1] - M[w-1,w-2] x_{w-2} M[w-2,w-1] and the effective sources
 * b = B[w-1,w-1] + a xl_{w-2} a^H - (y - y^H), y = a x_{w-2} B[w-2,w-1];
 * outputs [n_e][bs][bs]. */
int negf_dd_schur_tail(int n_e, int w, int bs, const void* m_diag, const void* m_upper,
                       const void* m_lower, const void* bl_diag, const void* bl_upper,
                       const void* bg_diag, const void* bg_upper, const void* x_fwd,
                       const void* xl_fwd, const void* xg_fwd, void* s_out, void* bl_out,
                       void* bg_out, void* workspace, size_t workspace_bytes, void* stream);
/* _middle_sweep (dist.py:388-448): two-sided Schur elimination of blocks
 * 1..w-2. s_out [4][n_e] = s_aa, s_ab, s_ba, s_bb; bl_out/bg_out [3][n_e] =
 * b_aa, b_ab, b_bb. status[e] = 1 + i when the Schur block of step i is
 * singular (0 ok). */
int negf_dd_middle_sweep(int n_e, int w, int bs, const void* m_diag, const void* m_upper,
                         const void* m_lower, const void* bl_diag, const void* bl_upper,
                         const void* bg_diag, const void* bg_upper, void* s_out, void* bl_out,
                         void* bg_out, int* status, void* workspace, size_t workspace_bytes,
                         void* stream);
/* _fold_corner (dist.py:451-473), in place on diagonal block j of the
 * partition: M_jj -= m_out x_env m_in; B_jj += -(m_out x_env) B_in
 * - B_out x_env^H m_out^H + m_out xl_env m_out^H. The stored coupling source
 * block Bc is B_in = Bc, B_out = -Bc^H for the left corner (side 0) and
 * B_out = Bc, B_in = -Bc^H for the right corner (side 1). Blocks [n_e]. */
int negf_dd_fold_corner(int n_e, int w, int bs, int j, int side, void* m_diag, void* bl_diag,
                        void* bg_diag, const void* m_out, const void* m_in, const void* bl_couple,
                        const void* bg_couple, const void* x_env, const void* xl_env,
                        const void* xg_env, void* workspace, size_t workspace_bytes, void* stream);
/* reverse_blocks: block order reversed. Full storage (lower_in != NULL):
 * upper'[t] = lower[w-2-t], lower'[t] = upper[w-2-t]; lg-compressed
 * (lower_in == NULL): upper'[t] = -upper[w-2-t]^H. */
int negf_dd_reverse_chain(int n_e, int w, int bs, const void* diag_in, const void* upper_in,
                          const void* lower_in, void* diag_out, void* upper_out, void* lower_out,
                          void* stream);

/* Keldysh identity defects (scba.py:1223-1248), the per-iteration
 * diagnostics of ScbaResult.identity_defects. out[2] (device double, zeroed
 * by the caller) accumulates max |(X^> - X^<) - (X^R - X^R^dag)| and the scale
 * max |X^R - X^R^dag| over every stored block (upper blocks against
 * X^R_up - X^R_lo^dag); the entry form takes entry-major series. */
int negf_g_identity_defect(int n_e, int n_b, int bs, const void* xr_diag, const void* xr_upper,
                           const void* xr_lower, const void* xl_diag, const void* xl_upper, const void* xg_diag,
                           const void* xg_upper, double* out, void* stream);
int negf_entry_identity_defect(long long n, const void* lesser, const void* greater, const void* ret_upper,
                               const void* ret_lower, double* out, void* stream);

/* ---- (6) mixing and residual (scba.py:478-481, 1155-1167) ----------------
 * s_k <- (1 - alpha) s_k + alpha r_k elementwise over n complex values, for
 * each non-NULL pair. diag_traces: tr[b][e] = sum_r x[diag_rows[b*bs + r]][e]
 * (the per-block traces _diag_traces, scba.py:1251-1255). */
int negf_mix(long long n, double alpha, void* s_lesser, void* s_greater, void* s_ret_up,
             void* s_ret_lo, const void* r_lesser, const void* r_greater, const void* r_ret_up,
             const void* r_ret_lo, void* stream);
/* negf_mix with the new Sigma read from its entry owners (fused nnz -> E,
 * scba.py:1138-1141 then :478-481): state (n_rows, n_own) local arrays;
 * src = device array of 4 * n_ranks pointers [lesser | greater | ret_up |
 * ret_lo] x rank to (rows, ld) entry-major arrays; row q of the state mixes
 * with row q - row_start[s] of rank s, columns col0 .. col0 + n_own. */
int negf_mix_p2p(long long n_rows, int n_own, double alpha, void* s_lesser, void* s_greater, void* s_ret_up,
                 void* s_ret_lo, int n_ranks, const unsigned long long* src, const long long* row_start,
                 long long ld, int col0, void* stream);
int negf_diag_traces(const void* x, long long ld, int n_e, const long long* diag_rows, int n_b,
                     int bs, void* tr, void* stream);

/* ---- opt-in CUDA-event profiler (bench.py live roofline) ---------------
 * class 0 = DMMA ZGEMM launches. Process-global, off by default. query()
 * synchronises on the recorded events and returns the summed device time
 * (ms), algorithmic flops and operand bytes of the recorded launches. */
void negf_prof_enable(int on);
/* Number of kernels this library has launched since it was loaded. */
long long negf_launch_count(void);
void negf_prof_reset(void);
int negf_prof_query(int cls, double* ms, double* flops, double* bytes, long long* launches);

#ifdef __cplusplus
}
#endif
#endif /* NEGF_B200_H */
