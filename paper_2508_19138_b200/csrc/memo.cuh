// Runtime OBC memoization on the GPU (see memo.cu).
#pragma once
#include "common.cuh"

namespace negf {

enum MemoMap : int {
  MEMO_SURFACE = 0,  // x <- (m - n x n')^-1      fixed_point_step, obc.py:138-141
  MEMO_STEIN = 1,    // w <- q + a w a^dag          scba.py:653-655
};

// One batched memoized_obc refresh (obc.py:519-600) over n_kind * n_side
// problems p = k * n_side + s (surface map: n_kind = 1; Stein: a is shared
// by the kinds of one side, a[s], q[p]). x0[p] is the cached block, used
// only where has[p] != 0. Writes the accepted refresh into out[p] and sets
// need_direct[p] = 1 (refresh rejected or no cache: caller runs the direct
// solver for exactly those) or used[p] = 1 (memoized).
size_t memo_workspace_bytes(int map, int n_side, int n_kind, int bs);
int memo_refresh(int map, int n_side, int n_kind, int bs, const z_t* m, const z_t* n, const z_t* np,
                 const z_t* a, const z_t* q, int n_fpi, double tol, const z_t* x0, const int* has,
                 z_t* out, int* need_direct, int* used, void* ws, size_t ws_bytes, cudaStream_t st);

// Strided cache <-> contiguous staging: n_seg segments of seg_len blocks;
// segment g of the cache starts at cache + g * ld * n2 (ld >= seg_len
// energies), of the contiguous buffer at buf + g * seg_len * n2.
int memo_gather(const z_t* cache, long long ld, const int* has, long long has_ld, int n_seg, int seg_len,
                int bs, z_t* buf, int* has_buf, cudaStream_t st);
int memo_store(const z_t* buf, const int* used_buf, int n_seg, int seg_len, int bs, z_t* cache, long long ld,
               int* has, int* used, long long has_ld, cudaStream_t st);

// Copy src -> dst for problems with sel[p] != 0 (n problems of n2 elements).
int copy_selected(z_t* dst, const z_t* src, long long n2, const int* sel, int n, cudaStream_t st);

}  // namespace negf
