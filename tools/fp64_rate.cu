// fp64 issue rates on this GPU — what bounds K1x (k_exact.cu), whose threads
// each run a dependent DFMA chain with operands from shared memory.
// Every CTA (one per SM) runs `warps` warps; every thread runs NC independent
// chains of `steps` DFMAs (or the K1x step shape).  Prints ns and cycles per
// step per warp for each mode.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_rate fp64_rate.cu
#include <cstdio>
#include <cuda_runtime.h>

// MODE 4: k_exact.cu's chain_sub shape (widen the next 32-column sub while
// the current sub's 32 DFMAs run, query operands one group ahead)
struct Raw8 {
  uint4 v[8];
};
__device__ __forceinline__ void chain_sub_like(const double (&kc)[32], double (&kn)[32], const Raw8& rn,
                                               const double* q64, int col0, double& acc) {
  double2 qa[2], qb[2];
  qa[0] = *reinterpret_cast<const double2*>(q64 + col0);
  qa[1] = *reinterpret_cast<const double2*>(q64 + col0 + 2);
#pragma unroll
  for (int g = 0; g < 8; ++g) {
    if (g + 1 < 8) {
      qb[0] = *reinterpret_cast<const double2*>(q64 + col0 + 4 * g + 4);
      qb[1] = *reinterpret_cast<const double2*>(q64 + col0 + 4 * g + 6);
    }
    acc = __fma_rn(qa[0].x, kc[4 * g + 0], acc);
    acc = __fma_rn(qa[0].y, kc[4 * g + 1], acc);
    acc = __fma_rn(qa[1].x, kc[4 * g + 2], acc);
    acc = __fma_rn(qa[1].y, kc[4 * g + 3], acc);
    const uint4 x = rn.v[g];
    kn[4 * g + 0] = (double)__uint_as_float(x.x);
    kn[4 * g + 1] = (double)__uint_as_float(x.y);
    kn[4 * g + 2] = (double)__uint_as_float(x.z);
    kn[4 * g + 3] = (double)__uint_as_float(x.w);
    qa[0] = qb[0];
    qa[1] = qb[1];
  }
}

template <int NC, int MODE>
__global__ void rate(double* out, int steps, double seed) {
  __shared__ __align__(16) double q[2048];
  __shared__ __align__(16) float kr[128][36];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) q[i] = 1.0 + i * 1e-9;
  for (int i = threadIdx.x; i < 128 * 36; i += blockDim.x) kr[i / 36][i % 36] = 1.0f - i * 1e-7f;
  __syncthreads();
  double a[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) a[c] = seed + threadIdx.x + c;
  const int r = threadIdx.x & 127;
  if (MODE == 0) {  // register-only chains: latency (NC = 1) / throughput (NC large)
    const double b = 1.0000001, cc = 1e-9;
    for (int i = 0; i < steps; i += 8) {
#pragma unroll
      for (int u = 0; u < 8; ++u)
#pragma unroll
        for (int c = 0; c < NC; ++c) a[c] = __fma_rn(a[c], b, cc);
    }
  } else if (MODE == 1) {  // q broadcast from smem (LDS.128 = 2 doubles), k in registers
    const double kk = 1.0000001;
    for (int i = 0; i < steps; i += 4) {
      const double2 x0 = *reinterpret_cast<const double2*>(&q[i & 2047]);
      const double2 x1 = *reinterpret_cast<const double2*>(&q[(i + 2) & 2047]);
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        a[c] = __fma_rn(x0.x, kk, a[c]);
        a[c] = __fma_rn(x0.y, kk, a[c]);
        a[c] = __fma_rn(x1.x, kk, a[c]);
        a[c] = __fma_rn(x1.y, kk, a[c]);
      }
    }
  } else if (MODE == 2) {  // K1x shape: per-lane row LDS.128 + F2F + broadcast q
    for (int i = 0; i < steps; i += 4) {
      const float4 v = *reinterpret_cast<const float4*>(&kr[r][(i & 31)]);
      const double2 x0 = *reinterpret_cast<const double2*>(&q[i & 2047]);
      const double2 x1 = *reinterpret_cast<const double2*>(&q[(i + 2) & 2047]);
      const double k0 = v.x, k1 = v.y, k2 = v.z, k3 = v.w;
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        a[c] = __fma_rn(x0.x, k0, a[c]);
        a[c] = __fma_rn(x0.y, k1, a[c]);
        a[c] = __fma_rn(x1.x, k2, a[c]);
        a[c] = __fma_rn(x1.y, k3, a[c]);
      }
    }
  } else if (MODE == 4) {
    const int swz = r & 7;
    const unsigned char* rowp = reinterpret_cast<const unsigned char*>(&kr[0][0]);
    double ka[32], kb[32];
    Raw8 raw;
#pragma unroll
    for (int g = 0; g < 32; ++g) ka[g] = 1.0 + g;
    for (int u = 0; u < steps / 32; u += 2) {
#pragma unroll
      for (int c = 0; c < 8; ++c) raw.v[c] = *reinterpret_cast<const uint4*>(rowp + ((r & 31) * 144 + (((c ^ swz) << 4) & 127)));
      chain_sub_like(ka, kb, raw, q, (u * 32) & 2047, a[0]);
#pragma unroll
      for (int c = 0; c < 8; ++c) raw.v[c] = *reinterpret_cast<const uint4*>(rowp + ((r & 31) * 144 + (((c ^ swz) << 4) & 127)));
      chain_sub_like(kb, ka, raw, q, ((u + 1) * 32) & 2047, a[0]);
    }
  } else if (MODE == 3) {  // F2F throughput alone (independent conversions)
    float f = (float)seed + threadIdx.x;
    for (int i = 0; i < steps; i += 8) {
#pragma unroll
      for (int u = 0; u < 8; ++u)
#pragma unroll
        for (int c = 0; c < NC; ++c) a[c] += (double)(f + (float)(u + c));
    }
  }
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < NC; ++c) s += a[c];
  if (s == 1.2345) out[0] = s;
}

template <int NC, int MODE>
void run(const char* name, int warps, int steps) {
  double* out;
  cudaMalloc(&out, 8);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  rate<NC, MODE><<<sms, warps * 32>>>(out, steps, 1.0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  rate<NC, MODE><<<sms, warps * 32>>>(out, steps, 1.0);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double ns_step = ms * 1e6 / steps;
  printf("%-34s warps/SM %2d chains/thread %d: %.3f ms, %.2f ns/step, %.1f cycles/step @%d MHz, %.1f warp-DFMA per SM per ns\n",
         name, warps, NC, ms, ns_step, ns_step * clk / 1e6, clk / 1000, (double)warps * NC / ns_step);
  cudaFree(out);
}

int main() {
  const int S = 1 << 16;
  run<1, 0>("dfma reg chain", 4, S);
  run<2, 0>("dfma reg chain", 4, S);
  run<4, 0>("dfma reg chain", 4, S);
  run<8, 0>("dfma reg chain", 4, S);
  run<8, 0>("dfma reg chain", 8, S);
  run<8, 0>("dfma reg chain", 16, S);
  run<1, 1>("dfma + bcast LDS.128 q", 4, S);
  run<4, 1>("dfma + bcast LDS.128 q", 4, S);
  run<1, 2>("K1x shape (row LDS + F2F + q)", 4, S);
  run<4, 2>("K1x shape (row LDS + F2F + q)", 4, S);
  run<1, 2>("K1x shape (row LDS + F2F + q)", 8, S);
  run<1, 4>("chain_sub shape (k_exact.cu)", 4, S);
  run<1, 4>("chain_sub shape (k_exact.cu)", 8, S);
  run<1, 3>("f2f.f64.f32", 4, S);
  run<8, 3>("f2f.f64.f32", 4, S);
  run<8, 3>("f2f.f64.f32", 16, S);
  return 0;
}
