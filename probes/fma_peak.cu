// fma_peak.cu -- measured SIMT FMA peaks of this B200 (the roofline denominators of the f64
// parity path and the fp32 FFMA fallbacks): 8 independent FMA chains per thread, 148 x 8 blocks
// of 256 threads, CUDA events.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fma_peak fma_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

template <typename T>
__global__ void fma_loop(T* out, int iters, T a, T b) {
  T x[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) x[j] = (T)(threadIdx.x + j);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = fma(x[j], a, b);
  }
  T s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += x[j];
  if (s == (T)12345.678) out[0] = s;                 // keep the chains alive
}

template <typename T>
double run(const char* name) {
  T* d;
  cudaMalloc(&d, 64);
  const int blocks = 148 * 8, threads = 256, iters = 1 << 14;
  fma_loop<T><<<blocks, threads>>>(d, 16, (T)0.999, (T)0.001);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  fma_loop<T><<<blocks, threads>>>(d, iters, (T)0.999, (T)0.001);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double flops = 2.0 * blocks * threads * (double)iters * 8;
  const double tf = flops / (ms * 1e-3) / 1e12;
  printf("{\"dtype\": \"%s\", \"tflops\": %.3f, \"ms\": %.3f}\n", name, tf, ms);
  cudaFree(d);
  return tf;
}

int main() {
  run<double>("f64");
  run<float>("f32");
  return 0;
}
