// FP64 pipe peak microbenchmark for B200 (sm_100a): DMMA.8x8x4 (mma.sync f64) and DFMA.
// Every SM runs `warps` warps issuing independent MMAs / FMAs back to back; timed with CUDA
// events over a multi-second loop so that power-cap clock behaviour is included (sustained).
#include <cstdio>
#include <cuda_runtime.h>
#include <vector>
#include <algorithm>

__global__ void dmma_loop(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) { c[i][0] = 0.0; c[i][1] = 0.0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.0) out[0] = s;
}

__global__ void dfma_loop(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-12, b = 1.0 - threadIdx.x * 1e-12;
  double c[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) c[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) c[i] = fma(a, c[i], b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += c[i];
  if (s == 12345.0) out[0] = s;
}

int main() {
  double* d; cudaMalloc(&d, 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int warps : {4, 8, 16}) {
    int iters = 200000;
    dmma_loop<<<sms, warps * 32>>>(d, 100); cudaDeviceSynchronize();
    // sustained: repeat launches for ~3 s
    std::vector<float> ts;
    for (int r = 0; r < 12; ++r) {
      cudaEventRecord(e0); dmma_loop<<<sms * 2, warps * 32>>>(d, iters); cudaEventRecord(e1);
      cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); ts.push_back(ms);
    }
    double flop = 2.0 * sms * warps * 8.0 * iters * 512.0;
    float best = *std::min_element(ts.begin(), ts.end()); float last = ts.back();
    printf("{\"kernel\":\"dmma_m8n8k4\",\"warps_per_cta\":%d,\"best_tflops\":%.3f,\"last_tflops\":%.3f,\"ms\":%.2f}\n",
           warps, flop / best / 1e9, flop / last / 1e9, best);
  }
  for (int warps : {8, 16, 32}) {
    int iters = 200000;
    std::vector<float> ts;
    for (int r = 0; r < 12; ++r) {
      cudaEventRecord(e0); dfma_loop<<<sms * 2, warps * 32>>>(d, iters); cudaEventRecord(e1);
      cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); ts.push_back(ms);
    }
    double flop = 2.0 * sms * 2 * warps * 32.0 * 16.0 * iters;
    float best = *std::min_element(ts.begin(), ts.end()); float last = ts.back();
    printf("{\"kernel\":\"dfma\",\"warps_per_cta\":%d,\"best_tflops\":%.3f,\"last_tflops\":%.3f,\"ms\":%.2f}\n",
           warps, flop / best / 1e9 / 1e3 * 1e3, flop / last / 1e9, best);
  }
  cudaError_t err = cudaGetLastError();
  printf("status %s\n", cudaGetErrorString(err));
  return 0;
}
