// tma_bw.cu — layout experiment for the key stream of the tcgen05 kernel:
// TMA read bandwidth of 128-row x 128-B boxes taken
//   (a) from a row-major [N][dim] fp32 matrix in the kernel's (k-chunk, block)
//       order (each box = 128 rows x 128 B, rows 16 KB apart), vs
//   (b) from a blocked [N/128][dim/32][128][32] layout (each box = 16 KB
//       contiguous).
// One persistent CTA per SM, kStages-deep ring, consumer warps only release.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_bw tools/tma_bw.cu
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

constexpr int kStages = 9, kGB = 3;

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@p bra.uni D;\nbra.uni W;\nD:\n}" ::"r"(su(b)),
               "r"(ph)
               : "memory");
}

__global__ void __launch_bounds__(64, 1) stream_kernel(const __grid_constant__ CUtensorMap map, int blocked, int nblocks,
                                                       int nk, int per) {
  extern __shared__ __align__(1024) unsigned char smem[];
  unsigned char* buf = smem + ((1024 - (su(smem) & 1023)) & 1023);
  uint64_t* full = reinterpret_cast<uint64_t*>(buf + kStages * 16384);
  uint64_t* empty = full + kStages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kStages; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&full[i])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&empty[i])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const int b0 = blockIdx.x * per, b1 = min(b0 + per, nblocks);
  if (warp == 0 && lane == 0) {
    int s = 0;
    uint32_t ph = 0;
    for (int g = b0; g < b1; g += kGB)
      for (int kc = 0; kc < nk; ++kc)
        for (int m = 0; m < kGB && g + m < b1; ++m) {
          wait(&empty[s], ph ^ 1);
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 16384;" ::"r"(su(&full[s])));
          const int x = blocked ? 0 : kc * 32;
          const int y = blocked ? ((g + m) * nk + kc) * 128 : (g + m) * 128;
          asm volatile(
              "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                  su(buf + s * 16384)),
              "l"((uint64_t)&map), "r"(x), "r"(y), "r"(su(&full[s]))
              : "memory");
          if (++s == kStages) s = 0, ph ^= 1;
        }
  } else if (warp == 1) {
    int s = 0;
    uint32_t ph = 0;
    for (int g = b0; g < b1; g += kGB)
      for (int kc = 0; kc < nk; ++kc)
        for (int m = 0; m < kGB && g + m < b1; ++m) {
          wait(&full[s], ph);
          if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(&empty[s])));
          __syncwarp();
          if (++s == kStages) s = 0, ph ^= 1;
        }
  }
}

int main(int argc, char** argv) {
  const long N = argc > 1 ? atol(argv[1]) : 1000064, dim = 4096;  // N: a multiple of 128
  const int nblocks = N / 128, nk = dim / 32;
  float* d;
  cudaMalloc(&d, N * dim * 4);
  cudaMemset(d, 0, N * dim * 4);
  void* fp;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fp;
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const int per = (nblocks + nsm - 1) / nsm;
  const size_t smem = kStages * 16384 + 1024 + 2 * kStages * 8;
  cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  for (int blocked = 0; blocked < 2; ++blocked) {
    CUtensorMap m;
    cuuint64_t gd[2], gs[1];
    if (blocked) {
      gd[0] = 32;
      gd[1] = (cuuint64_t)N * nk;
      gs[0] = 128;
    } else {
      gd[0] = dim;
      gd[1] = N;
      gs[0] = dim * 4;
    }
    cuuint32_t box[2] = {32, 128}, es[2] = {1, 1};
    enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, gd, gs, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int it = 0; it < 3; ++it) stream_kernel<<<nsm, 64, smem>>>(m, blocked, nblocks, nk, per);
    cudaEventRecord(a);
    const int iters = 10;
    for (int it = 0; it < iters; ++it) stream_kernel<<<nsm, 64, smem>>>(m, blocked, nblocks, nk, per);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    ms /= iters;
    printf("%s: %.3f ms  %.1f GB/s  (%s)\n", blocked ? "blocked [N/128][dim/32][128][32]" : "row-major [N][dim]", ms,
           N * dim * 4 / (ms * 1e6), cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
