// Latency of a dependent fp64 chain on this GPU (what bounds K2's exact,
// sequentially-rounded rescoring): DFMA chain, DADD chain, and the rescoring
// inner loop shape (smem operands + F2F widening).  Prints cycles per step.
#include <cstdio>
#include <cuda_runtime.h>
#ifndef NCHAIN
#define NCHAIN 8
#endif

__global__ void chains(long long* out, double seed, const float* __restrict__ g) {
  __shared__ float rows[4096];
  __shared__ double q[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) {
    rows[i] = g[i];
    q[i] = (double)g[4095 - i];
  }
  __syncthreads();
  if (threadIdx.x >= NCHAIN) return;
  double a = seed + threadIdx.x, b = 1.0000001, c = 1e-9;
  long long t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < 4096; ++i) a = __fma_rn(a, b, c);
  long long t1 = clock64();
  double s = seed;
#pragma unroll 16
  for (int i = 0; i < 4096; ++i) s = __dadd_rn(s, c * i);
  long long t2 = clock64();
  double acc = 0.0;
#pragma unroll 16
  for (int j = 0; j < 4096; ++j) acc = __fma_rn(q[j], (double)rows[j], acc);
  long long t3 = clock64();
  // software-pipelined: operands of the next 16 steps are loaded (and widened)
  // before the current 16 dependent FMAs issue
  double acc2 = 0.0;
  double qa[16], ka[16];
#pragma unroll
  for (int u = 0; u < 16; ++u) {
    qa[u] = q[u];
    ka[u] = (double)rows[u];
  }
  for (int j = 0; j < 4096; j += 16) {
    double qb[16], kb[16];
    const int jn = j + 16 < 4096 ? j + 16 : j;
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      qb[u] = q[jn + u];
      kb[u] = (double)rows[jn + u];
    }
#pragma unroll
    for (int u = 0; u < 16; ++u) acc2 = __fma_rn(qa[u], ka[u], acc2);
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      qa[u] = qb[u];
      ka[u] = kb[u];
    }
  }
  long long t4 = clock64();
  if (threadIdx.x == 0) {
    out[0] = t1 - t0;
    out[1] = t2 - t1;
    out[2] = t3 - t2;
    out[4] = t4 - t3;
    out[3] = (long long)(a + s + acc + acc2);
  }
}

int main() {
  long long* d;
  float* g;
  cudaMalloc(&d, 64);
  cudaMalloc(&g, 4096 * 4);
  cudaMemset(g, 0, 4096 * 4);
  chains<<<1, 128>>>(d, 1.0, g);
  long long h[5];
  cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  chains<<<1, 128>>>(d, 2.0, g);
  cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  printf("cycles/step: dfma chain %.2f, dadd chain %.2f, rescoring loop %.2f, pipelined loop %.2f\n",
         h[0] / 4096.0, h[1] / 4096.0, h[2] / 4096.0, h[4] / 4096.0);
  return 0;
}
