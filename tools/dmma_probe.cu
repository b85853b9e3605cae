// Probe: (1) verify the mma.sync.m8n8k4 f64 fragment layout used by the LU
// trailing update, (2) measure DMMA vs SIMT DFMA throughput on this GPU.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

__global__ void layout(const double* A, const double* B, double* C) {
  int l = threadIdx.x;
  double a = A[(l >> 2) * 4 + (l & 3)];       // A[row=l/4][col=l%4]
  double b = B[(l & 3) * 8 + (l >> 2)];       // B[row=l%4][col=l/4]
  double c0 = 0, c1 = 0;
  dmma(c0, c1, a, b);
  C[(l >> 2) * 8 + (l & 3) * 2] = c0;          // C[row=l/4][col=2(l%4)]
  C[(l >> 2) * 8 + (l & 3) * 2 + 1] = c1;
}

__global__ void dmma_tput(double* out, int iters) {
  double c[8][2] = {};
  double a = threadIdx.x * 1e-3, b = 1.0 + blockIdx.x * 1e-6;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) dmma(c[j][0], c[j][1], a, b);
  }
  double s = 0;
  for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void dfma_tput(double* out, int iters) {
  double c[16];
  for (int j = 0; j < 16; ++j) c[j] = j;
  double a = threadIdx.x * 1e-3, b = 1.0 + blockIdx.x * 1e-6;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) c[j] = fma(c[j], a, b);
  }
  double s = 0;
  for (int j = 0; j < 16; ++j) s += c[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  double hA[32], hB[32], hC[64], ref[64];
  for (int i = 0; i < 32; ++i) { hA[i] = i + 1; hB[i] = 0.5 * i - 3; }
  for (int r = 0; r < 8; ++r)
    for (int c = 0; c < 8; ++c) {
      double s = 0;
      for (int k = 0; k < 4; ++k) s += hA[r * 4 + k] * hB[k * 8 + c];
      ref[r * 8 + c] = s;
    }
  double *dA, *dB, *dC, *dO;
  cudaMalloc(&dA, 256); cudaMalloc(&dB, 256); cudaMalloc(&dC, 512);
  cudaMemcpy(dA, hA, 256, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB, 256, cudaMemcpyHostToDevice);
  layout<<<1, 32>>>(dA, dB, dC);
  cudaMemcpy(hC, dC, 512, cudaMemcpyDeviceToHost);
  double err = 0;
  for (int i = 0; i < 64; ++i) err = fmax(err, fabs(hC[i] - ref[i]));
  printf("m8n8k4 layout max err = %g (%s)\n", err, err == 0 ? "OK" : "MISMATCH");
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int blocks = sms * 8, threads = 256, iters = 4096;
  cudaMalloc(&dO, sizeof(double) * blocks * threads);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    dmma_tput<<<blocks, threads>>>(dO, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 256 * 8.0 * iters * (blocks * threads / 32);
    printf("DMMA m8n8k4: %.2f TFLOP/s\n", flops / ms / 1e9);
    cudaEventRecord(e0);
    dfma_tput<<<blocks, threads>>>(dO, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    flops = 2.0 * 16 * iters * (double)blocks * threads;
    printf("SIMT DFMA:   %.2f TFLOP/s\n", flops / ms / 1e9);
  }
  return 0;
}
