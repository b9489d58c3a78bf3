// Block-level elementwise combinations with optional conjugate-transposed
// operands (the "y - y^dag" terms of rgf.py:140-148, 209-226 and the
// anti-Hermitian projection of rgf.py:82-88).
#pragma once
#include "common.cuh"

namespace negf {

constexpr int kEwTerms = 4;
constexpr int kEwGroup = 6;

struct EwDesc {
  int batch, nterms;
  z_t* out;
  long long sOut;
  const z_t* X[kEwTerms];
  long long sX[kEwTerms];
  int opH[kEwTerms];  // 1: use X^dag
  double2 coef[kEwTerms];
};

struct EwGroup {
  int n;
  int rows, cols;  // all blocks rows x cols, row-major packed (ld = cols)
  EwDesc d[kEwGroup];
};

// out = sum_t coef_t * op_t(X_t). `out` must not alias an X_t used with opH.
int ew_group_launch(const EwGroup& g, cudaStream_t stream);

// In place X <- (X - X^dag)/2 on `batch` square n x n blocks (stride sX).
int antiherm_inplace(z_t* X, long long sX, int n, int batch, cudaStream_t stream);

// Y <- Y + s * I on `batch` square n x n blocks
int add_identity(z_t* Y, long long sY, int n, int batch, double2 s, cudaStream_t stream);

}  // namespace negf
