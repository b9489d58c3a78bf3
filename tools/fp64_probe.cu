// FP64 throughput probe for B200 (sm_100a): DMMA shapes, DFMA, cuBLAS D/ZGEMM.
// Measures the FP64 roofline denominator that MEASURED_PEAKS.json lacks.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
#include <cublas_v2.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

template <int SHAPE>
__global__ void dmma_loop(double* out, int iters) {
  double a[8], b[4], c[8][4];
  for (int i = 0; i < 8; ++i) a[i] = 1e-3 * (threadIdx.x + i);
  for (int i = 0; i < 4; ++i) b[i] = 1e-3 * (threadIdx.x - i);
  for (int j = 0; j < 8; ++j) for (int i = 0; i < 4; ++i) c[j][i] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (SHAPE == 0) {
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[j][0]), "+d"(c[j][1]) : "d"(a[0]), "d"(b[0]));
      } else if (SHAPE == 1) {
        asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
                     : "+d"(c[j][0]), "+d"(c[j][1]), "+d"(c[j][2]), "+d"(c[j][3]) : "d"(a[0]), "d"(a[1]), "d"(b[0]));
      } else if (SHAPE == 2) {
        asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                     : "+d"(c[j][0]), "+d"(c[j][1]), "+d"(c[j][2]), "+d"(c[j][3]) : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
      } else {
        asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                     : "+d"(c[j][0]), "+d"(c[j][1]), "+d"(c[j][2]), "+d"(c[j][3])
                     : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                       "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
      }
    }
  }
  double s = 0;
  for (int j = 0; j < 8; ++j) for (int i = 0; i < 4; ++i) s += c[j][i];
  if (s == 12345.678) out[threadIdx.x] = s;
}

__global__ void dfma_loop(double* out, int iters) {
  double x[8];
  double y = 1.0000001, z = 1e-9;
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fma(x[i], y, z);
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 12345.678) out[threadIdx.x] = s;
}

template <int SHAPE>
double run_dmma(int blocks, int threads, int iters) {
  double* d; CK(cudaMalloc(&d, 4096 * 8));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  dmma_loop<SHAPE><<<blocks, threads>>>(d, 10); CK(cudaDeviceSynchronize());
  cudaEventRecord(e0);
  dmma_loop<SHAPE><<<blocks, threads>>>(d, iters);
  cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  const int mnk[4] = {8 * 8 * 4, 16 * 8 * 4, 16 * 8 * 8, 16 * 8 * 16};
  double flops = 2.0 * mnk[SHAPE] * 8.0 * iters * (double)blocks * (threads / 32);
  cudaFree(d);
  return flops / (ms * 1e-3) / 1e12;
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  printf("device %s SMs %d clock %d kHz\n", p.name, p.multiProcessorCount, p.clockRate);
  int sms = p.multiProcessorCount;
  const char* names[4] = {"m8n8k4", "m16n8k4", "m16n8k8", "m16n8k16"};
  for (int w : {4, 8, 16}) {
    printf("DMMA %s warps/SM=%d : %.2f TFLOP/s\n", names[0], w, run_dmma<0>(sms * (w / 4), 128, 20000));
    printf("DMMA %s warps/SM=%d : %.2f TFLOP/s\n", names[1], w, run_dmma<1>(sms * (w / 4), 128, 10000));
    printf("DMMA %s warps/SM=%d : %.2f TFLOP/s\n", names[2], w, run_dmma<2>(sms * (w / 4), 128, 5000));
    printf("DMMA %s warps/SM=%d : %.2f TFLOP/s\n", names[3], w, run_dmma<3>(sms * (w / 4), 128, 2500));
  }
  {
    double* d; CK(cudaMalloc(&d, 4096 * 8));
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    int iters = 20000;
    for (int bps : {2, 4, 8}) {
      dfma_loop<<<sms * bps, 256>>>(d, 10); CK(cudaDeviceSynchronize());
      cudaEventRecord(e0);
      dfma_loop<<<sms * bps, 256>>>(d, iters);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double flops = 2.0 * 8 * iters * (double)sms * bps * 256;
      printf("DFMA blocks/SM=%d x256 : %.2f TFLOP/s\n", bps, flops / (ms * 1e-3) / 1e12);
    }
  }
  cublasHandle_t h; cublasCreate(&h);
  {
    int n = 8192;
    double *A, *B, *C; CK(cudaMalloc(&A, 8.0 * n * n)); CK(cudaMalloc(&B, 8.0 * n * n)); CK(cudaMalloc(&C, 8.0 * n * n));
    cudaMemset(A, 0, 8.0 * n * n); cudaMemset(B, 0, 8.0 * n * n);
    double al = 1, be = 0;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, n, n, n, &al, A, n, B, n, &be, C, n);
    CK(cudaDeviceSynchronize());
    for (int r = 0; r < 3; ++r) {
      cudaEventRecord(e0);
      for (int i = 0; i < 3; ++i) cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, n, n, n, &al, A, n, B, n, &be, C, n);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      printf("cublasDgemm %d : %.2f TFLOP/s\n", n, 3 * 2.0 * n * n * (double)n / (ms * 1e-3) / 1e12);
    }
    cudaFree(A); cudaFree(B); cudaFree(C);
  }
  for (int n : {4096}) {
    cuDoubleComplex *A, *B, *C; size_t bytes = 16.0 * n * n;
    CK(cudaMalloc(&A, bytes)); CK(cudaMalloc(&B, bytes)); CK(cudaMalloc(&C, bytes));
    cudaMemset(A, 0, bytes); cudaMemset(B, 0, bytes);
    cuDoubleComplex al = {1, 0}, be = {0, 0};
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cublasZgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, n, n, n, &al, A, n, B, n, &be, C, n);
    CK(cudaDeviceSynchronize());
    for (int r = 0; r < 3; ++r) {
      cudaEventRecord(e0);
      for (int i = 0; i < 3; ++i) cublasZgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, n, n, n, &al, A, n, B, n, &be, C, n);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      printf("cublasZgemm %d : %.2f TFLOP/s\n", n, 3 * 8.0 * n * n * (double)n / (ms * 1e-3) / 1e12);
    }
    cudaFree(A); cudaFree(B); cudaFree(C);
  }
  for (int n : {32, 64, 128, 256, 512}) {
    int batch = (int)(64.0 * 256 * 256 * 256 / ((double)n * n * n));
    if (batch > 65535) batch = 65535;
    if (batch < 8) batch = 8;
    cuDoubleComplex *A, *B, *C; size_t bytes = 16.0 * n * n * batch;
    CK(cudaMalloc(&A, bytes)); CK(cudaMalloc(&B, bytes)); CK(cudaMalloc(&C, bytes));
    cudaMemset(A, 0, bytes); cudaMemset(B, 0, bytes);
    cuDoubleComplex al = {1, 0}, be = {0, 0};
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    long long s = (long long)n * n;
    cublasZgemmStridedBatched(h, CUBLAS_OP_N, CUBLAS_OP_N, n, n, n, &al, A, n, s, B, n, s, &be, C, n, s, batch);
    CK(cudaDeviceSynchronize());
    for (int r = 0; r < 2; ++r) {
      cudaEventRecord(e0);
      for (int i = 0; i < 5; ++i)
        cublasZgemmStridedBatched(h, CUBLAS_OP_N, CUBLAS_OP_N, n, n, n, &al, A, n, s, B, n, s, &be, C, n, s, batch);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      printf("cublasZgemmStridedBatched n=%d batch=%d : %.2f TFLOP/s (%.3f ms/call)\n", n, batch,
             5 * 8.0 * n * n * (double)n * batch / (ms * 1e-3) / 1e12, ms / 5);
    }
    cudaFree(A); cudaFree(B); cudaFree(C);
  }
  return 0;
}
