// cluster_occupancy.cu — how many clusters of 2 / 4 / 6 / 8 CTAs (one CTA per
// SM: 215 KB of shared memory, 384 threads, like sim_pair_kernel) are
// co-resident on this B200, by the occupancy API and by a launch that records
// each CTA's SM and start time.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/cluster_occupancy tools/cluster_occupancy.cu
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <vector>

__global__ void probe(unsigned long long* t0, int* sm, unsigned long long spin) {
  extern __shared__ unsigned char smem[];
  unsigned long long s;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(s));
  if (threadIdx.x == 0) {
    unsigned id;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(id));
    t0[blockIdx.x] = s;
    sm[blockIdx.x] = (int)id;
    smem[0] = (unsigned char)id;
  }
  unsigned long long now = s;
  while (now - s < spin) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
}

int main() {
  const size_t smem = 215 * 1024;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(probe, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  for (int cs : {1, 2, 4, 6, 8}) {
    cudaLaunchConfig_t cfg{};
    cfg.blockDim = dim3(384);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cfg.gridDim = dim3(cs);
    int n = 0;
    cudaOccupancyMaxActiveClusters(&n, probe, &cfg);
    // launch more clusters than the API allows and see how many start together
    const int want = nsm / cs;
    cfg.gridDim = dim3(want * cs);
    unsigned long long* t0;
    int* sm;
    cudaMalloc(&t0, sizeof(unsigned long long) * want * cs);
    cudaMalloc(&sm, sizeof(int) * want * cs);
    cudaLaunchKernelEx(&cfg, probe, t0, sm, 200000ull);  // 200 us spin
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<unsigned long long> h(want * cs);
    cudaMemcpy(h.data(), t0, sizeof(unsigned long long) * h.size(), cudaMemcpyDeviceToHost);
    const unsigned long long first = *std::min_element(h.begin(), h.end());
    int together = 0;
    for (auto v : h) together += (v - first) < 100000ull;  // started within 100 us of the first
    printf("cluster %d: occupancy API %3d clusters (%3d SMs); launched %3d clusters (%3d CTAs): %3d CTAs started "
           "together  err=%s\n",
           cs, n, n * cs, want, want * cs, together, cudaGetErrorString(e));
    cudaFree(t0);
    cudaFree(sm);
  }
  return 0;
}
