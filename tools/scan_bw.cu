// scan_bw.cu — the key stream of K1x (k_exact.cu) alone: every CTA owns one
// tile of R rows and reads its 128-B row segments column by column through an
// S-stage TMA ring (consumers only release the slots).  Compares layouts and
// start orders for a small DB (C1: 10k x 4096 fp32 = 164 MB):
//   layout 0: row-major [N][dim] (a box = R rows x 128 B, rows dim*4 B apart)
//   layout 1: blocked [N/R][dim/32][R][32] (a box = R x 128 B contiguous)
//   stagger 1: CTA b starts at column chunk b * nchunk / grid (wrapping)
// Prints GB/s per configuration (L2 flushed by a 512 MB write before each).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/scan_bw tools/scan_bw.cu -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@p bra.uni D;\nbra.uni W;\nD:\n}" ::"r"(su(b)),
               "r"(ph)
               : "memory");
}

__global__ void __launch_bounds__(160, 1) scan_stream(const __grid_constant__ CUtensorMap map, int R, int S, int nchunk,
                                                      int blocked, int stagger, int ntiles) {
  extern __shared__ __align__(1024) unsigned char smem[];
  unsigned char* buf = smem + ((1024 - (su(smem) & 1023)) & 1023);
  const int stage = R * 128;
  uint64_t* full = reinterpret_cast<uint64_t*>(buf + (size_t)S * stage);
  uint64_t* empty = full + S;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&full[i])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 4;" ::"r"(su(&empty[i])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const int t = blockIdx.x;
  if (t >= ntiles) return;
  const int c0 = stagger ? (int)((long)t * nchunk / gridDim.x) : 0;
  if (warp == 4) {
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      for (int i = 0; i < nchunk; ++i) {
        const int j = (c0 + i) % nchunk;
        if (i >= S) wait(&empty[s], ph ^ 1);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&full[s])), "r"(stage));
        const int x = blocked ? 0 : j * 32;
        const int y = blocked ? (t * nchunk + j) * R : t * R;
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                su(buf + (size_t)s * stage)),
            "l"((uint64_t)&map), "r"(x), "r"(y), "r"(su(&full[s]))
            : "memory");
        if (++s == S) s = 0, ph ^= 1;
      }
    }
  } else {
    int s = 0;
    uint32_t ph = 0;
    for (int i = 0; i < nchunk; ++i) {
      wait(&full[s], ph);
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(&empty[s])) : "memory");
      if (++s == S) s = 0, ph ^= 1;
    }
  }
}

__global__ void read_flush(const int4* p, long n, int* sink) {
  int4 acc = make_int4(0, 0, 0, 0);
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
    const int4 v = __ldcg(p + i);
    acc.x ^= v.x;
  }
  if (acc.x == 0x12345678) *sink = acc.x;
}

int main(int argc, char** argv) {
  const long N = argc > 1 ? atol(argv[1]) : 10000;
  const int flush_mode = argc > 2 ? atoi(argv[2]) : 1;  // 0 none, 1 512 MB write, 2 512 MB read
  const long dim = 4096;
  PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* keys;
  cudaMalloc(&keys, (N + 256) * dim * 4);
  cudaMemset(keys, 0, (N + 256) * dim * 4);
  char* flush;
  cudaMalloc(&flush, 512 << 20);
  cudaMemset(flush, 0, 512 << 20);
  const int nchunk = dim / 32;
  const int Rs[] = {72, 128};
  for (int R : Rs) {
    const int ntiles = (int)((N + R - 1) / R);
    for (int blocked = 0; blocked < 2; ++blocked)
      for (int stagger = 0; stagger < 2; ++stagger)
        for (int S : {8, 16}) {
          if ((size_t)S * R * 128 > 200 * 1024) continue;
          CUtensorMap m;
          const cuuint64_t gdim[2] = {32 * (blocked ? 1 : (cuuint64_t)nchunk), blocked ? (cuuint64_t)ntiles * nchunk * R
                                                                                        : (cuuint64_t)N};
          const cuuint64_t gstr[1] = {blocked ? 128 : (cuuint64_t)dim * 4};
          const cuuint32_t box[2] = {32, (cuuint32_t)R};
          const cuuint32_t es[2] = {1, 1};
          if (enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, keys, gdim, gstr, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
            printf("encode failed\n");
            continue;
          }
          const size_t smem = (size_t)S * R * 128 + 2048;
          cudaFuncSetAttribute(scan_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
          const int grid = ntiles;
          float best = 1e9, sum = 0;
          for (int rep = 0; rep < 6; ++rep) {
            if (flush_mode == 1) cudaMemsetAsync(flush, rep, 512 << 20);
            if (flush_mode == 2) read_flush<<<sms * 4, 512>>>((const int4*)flush, (512 << 20) / 16, (int*)keys);
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            cudaEventRecord(e0);
            scan_stream<<<grid, 160, smem>>>(m, R, S, nchunk, blocked, stagger, ntiles);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (rep) {
              best = ms < best ? ms : best;
              sum += ms;
            }
          }
          const double bytes = (double)ntiles * R * dim * 4;
          printf("flush %d N %ld R %3d S %2d grid %4d layout %s stagger %d: %.1f us (best %.1f) -> %.2f TB/s  err=%s\n", flush_mode, N, R, S,
                 grid, blocked ? "blocked " : "rowmajor", stagger, sum / 5 * 1e3, best * 1e3,
                 bytes / (sum / 5 * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
        }
  }
  return 0;
}
