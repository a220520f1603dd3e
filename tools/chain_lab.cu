// chain_lab.cu — K1x's consumer loop (k_exact.cu) without TMA or barriers, to
// find what makes its fp64 chain slower in the kernel (~15 cycles per step)
// than the same chain_sub code alone (9.3, tools/fp64_rate.cu).  The ring is a
// static shared-memory tile; the grid is config 1's (139 CTAs x (4 + 1) warps,
// 18 active lanes per compute warp, 4096 steps).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/chain_lab tools/chain_lab.cu
//   MODE 0  replica: ring slot rotation, swizzled 16-B row loads, ping-pong widening
//   MODE 1  fixed ring slot (no slot arithmetic)
//   MODE 2  no widening of the next sub (keys reused): the DFMA chain + q loads only
//   MODE 3  replica with every lane active (lpw = 32)
//   MODE 4  replica, query operands two groups ahead
//   MODE 5  replica, the next sub widened in the second half of the current one
//   MODE 6  replica, widening by integer bit moves (x * 2^-896 exactly; the
//           queries carry the 2^896) instead of F2F on the fp64 pipe
//   MODE 7  MODE 6 with a fixed ring slot
//   MODE 8  simple loop: per 4 steps one 16-B row load + two broadcast query
//           loads + 4 F2F + 4 DFMA, straight from the ring slot (the compiler
//           schedules; no ping-pong widening)
//   MODE 9  MODE 8 with the segment loop unrolled by 2
//   MODE 10 the next sub's 8 row loads issued one sub ahead (raw registers),
//           widened just in time per group of 4 steps
//   MODE 11 MODE 10 with the query operands loaded one group ahead
//   MODE 12 tools/fp64_rate.cu's "K1x shape" loop (padded 36-float rows, one
//           fixed row per thread, q index i & 4095) inside this harness
//   MODE 14 MODE 8 plus K1x's per-segment handshake: an mbarrier wait (on an
//           already completed phase) before each sub, __syncwarp + lane-0
//           arrive on an "empty" barrier after it
//   MODE 13 the same flat loop over steps (i += 4) reading the ring: slot
//           (i / 32) mod S (S a power of two), chunk (i / 4) mod 8, swizzled
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

constexpr int kSub = 32;
struct Raw {
  uint4 v[8];
};

__device__ __forceinline__ void widen4(const Raw& r, int g, double* out) {
  const uint4 x = r.v[g];
  out[0] = (double)__uint_as_float(x.x);
  out[1] = (double)__uint_as_float(x.y);
  out[2] = (double)__uint_as_float(x.z);
  out[3] = (double)__uint_as_float(x.w);
}

// fp32 x -> the double x * 2^-896, exactly, for every finite x (zero and
// subnormals included): the fp32 exponent / fraction fields move into the
// double's unchanged, so only the bias differs.  Integer ops, not the fp64 pipe.
__device__ __forceinline__ double widen_bits(uint32_t u) {
  const uint32_t hi = (uint32_t)((int32_t)u >> 3) & 0x8FFFFFFFu;
  return __hiloint2double((int)hi, (int)(u << 29));
}
__device__ __forceinline__ void widen4b(const Raw& r, int g, double* out) {
  const uint4 x = r.v[g];
  out[0] = widen_bits(x.x);
  out[1] = widen_bits(x.y);
  out[2] = widen_bits(x.z);
  out[3] = widen_bits(x.w);
}

template <bool kNext, int kAhead, bool kLate = false, bool kBits = false>
__device__ __forceinline__ void chain_sub(const double (&kc)[kSub], double (&kn)[kSub], const Raw& rn,
                                          const double* __restrict__ q64, int col0, double& acc) {
  double2 qa[kAhead][2];
#pragma unroll
  for (int a = 0; a < kAhead; ++a) {
    qa[a][0] = *reinterpret_cast<const double2*>(q64 + col0 + 4 * a);
    qa[a][1] = *reinterpret_cast<const double2*>(q64 + col0 + 4 * a + 2);
  }
#pragma unroll
  for (int g = 0; g < kSub / 4; ++g) {
    double2 nb0, nb1;
    if (g + kAhead < kSub / 4) {
      nb0 = *reinterpret_cast<const double2*>(q64 + col0 + 4 * (g + kAhead));
      nb1 = *reinterpret_cast<const double2*>(q64 + col0 + 4 * (g + kAhead) + 2);
    }
    acc = __fma_rn(qa[0][0].x, kc[4 * g + 0], acc);
    acc = __fma_rn(qa[0][0].y, kc[4 * g + 1], acc);
    acc = __fma_rn(qa[0][1].x, kc[4 * g + 2], acc);
    acc = __fma_rn(qa[0][1].y, kc[4 * g + 3], acc);
    if (kNext && !kLate) {
      if (kBits)
        widen4b(rn, g, &kn[4 * g]);
      else
        widen4(rn, g, &kn[4 * g]);
    }
    if (kNext && kLate && g >= 4) {  // the next sub's rows: widened in the second half (its loads have landed)
      widen4(rn, 2 * (g - 4), &kn[8 * (g - 4)]);
      widen4(rn, 2 * (g - 4) + 1, &kn[8 * (g - 4) + 4]);
    }
#pragma unroll
    for (int a = 0; a + 1 < kAhead; ++a) {
      qa[a][0] = qa[a + 1][0];
      qa[a][1] = qa[a + 1][1];
    }
    qa[kAhead - 1][0] = nb0;
    qa[kAhead - 1][1] = nb1;
  }
}

template <int MODE>
__global__ void __launch_bounds__(160, 1) lab(double* out, int U, int S, int lpw) {
  extern __shared__ __align__(1024) unsigned char smem[];
  const int R = 4 * lpw;
  const int stage_bytes = R * 128;
  double* q64 = reinterpret_cast<double*>(smem + (size_t)S * stage_bytes);
  for (int i = threadIdx.x; i < S * stage_bytes / 4; i += blockDim.x)
    reinterpret_cast<float*>(smem)[i] = 1.0f + 1e-7f * (i & 1023);
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) q64[i] = 1.0 - 1e-9 * i;
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 4) return;
  const int rr = warp * lpw + lane;
  const int swz = rr & 7;
  const unsigned char* rowbase = smem + (size_t)(lane < lpw ? rr : 0) * 128;
  int wslot = 0;
  auto load_sub = [&](int u, Raw& r) {
    const unsigned char* rowp = rowbase + (size_t)(MODE == 1 || MODE == 7 ? 0 : wslot) * stage_bytes;
#pragma unroll
    for (int c = 0; c < 8; ++c) r.v[c] = *reinterpret_cast<const uint4*>(rowp + ((c ^ swz) << 4));
    if (MODE != 1 && MODE != 7 && ++wslot == S) wslot = 0;
  };
  if constexpr (MODE == 13) {
    double a13 = 0.0;
    const int smask = S - 1;  // S rounded down to a power of two by the caller
    for (int i = 0; i < U * kSub; i += 4) {
      const unsigned char* p = rowbase + (size_t)((i >> 5) & smask) * stage_bytes + ((((i >> 2) & 7) ^ swz) << 4);
      const float4 v = *reinterpret_cast<const float4*>(p);
      const double2 x0 = *reinterpret_cast<const double2*>(q64 + (i & 4095));
      const double2 x1 = *reinterpret_cast<const double2*>(q64 + ((i + 2) & 4095));
      a13 = __fma_rn(x0.x, (double)v.x, a13);
      a13 = __fma_rn(x0.y, (double)v.y, a13);
      a13 = __fma_rn(x1.x, (double)v.z, a13);
      a13 = __fma_rn(x1.y, (double)v.w, a13);
    }
    if (a13 == 1.2345) out[0] = a13;
    return;
  }
  if constexpr (MODE == 12) {
    const float* kr = reinterpret_cast<const float*>(smem) + (size_t)(lane < lpw ? rr : 0) * 36;
    double a12 = 0.0;
    for (int i = 0; i < U * kSub; i += 4) {
      const float4 v = *reinterpret_cast<const float4*>(kr + (i & 31));
      const double2 x0 = *reinterpret_cast<const double2*>(q64 + (i & 4095));
      const double2 x1 = *reinterpret_cast<const double2*>(q64 + ((i + 2) & 4095));
      a12 = __fma_rn(x0.x, (double)v.x, a12);
      a12 = __fma_rn(x0.y, (double)v.y, a12);
      a12 = __fma_rn(x1.x, (double)v.z, a12);
      a12 = __fma_rn(x1.y, (double)v.w, a12);
    }
    if (a12 == 1.2345) out[0] = a12;
    return;
  }
  if constexpr (MODE == 10 || MODE == 11) {
    double acc10 = 0.0;
    int slot = 0;
    Raw cur, nxt;
    const uint32_t ofs0 = 0;
#pragma unroll
    for (int c = 0; c < 8; ++c) cur.v[c] = *reinterpret_cast<const uint4*>(rowbase + ofs0 + ((c ^ swz) << 4));
    for (int u = 0; u < U; ++u) {
      if (++slot == S) slot = 0;
      const unsigned char* rowp = rowbase + (size_t)slot * stage_bytes;
#pragma unroll
      for (int c = 0; c < 8; ++c) nxt.v[c] = *reinterpret_cast<const uint4*>(rowp + ((c ^ swz) << 4));
      const double* q = q64 + ((u * kSub) & 4095);
      double2 qa0 = *reinterpret_cast<const double2*>(q), qa1 = *reinterpret_cast<const double2*>(q + 2);
#pragma unroll
      for (int g = 0; g < 8; ++g) {
        double2 q0, q1, qn0, qn1;
        if constexpr (MODE == 11) {
          q0 = qa0;
          q1 = qa1;
          if (g + 1 < 8) {
            qn0 = *reinterpret_cast<const double2*>(q + 4 * g + 4);
            qn1 = *reinterpret_cast<const double2*>(q + 4 * g + 6);
          }
        } else {
          q0 = *reinterpret_cast<const double2*>(q + 4 * g);
          q1 = *reinterpret_cast<const double2*>(q + 4 * g + 2);
        }
        const uint4 x = cur.v[g];
        acc10 = __fma_rn(q0.x, (double)__uint_as_float(x.x), acc10);
        acc10 = __fma_rn(q0.y, (double)__uint_as_float(x.y), acc10);
        acc10 = __fma_rn(q1.x, (double)__uint_as_float(x.z), acc10);
        acc10 = __fma_rn(q1.y, (double)__uint_as_float(x.w), acc10);
        if constexpr (MODE == 11) {
          qa0 = qn0;
          qa1 = qn1;
        }
      }
      cur = nxt;
    }
    if (acc10 == 1.2345) out[0] = acc10;
    return;
  }
  if constexpr (MODE >= 8) {
    double acc8 = 0.0;
    int slot = 0;
    __shared__ uint64_t bars[2];
    if constexpr (MODE == 14) {
      if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bars[0])));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1000000;" ::"r"((uint32_t)__cvta_generic_to_shared(&bars[1])));
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"((uint32_t)__cvta_generic_to_shared(&bars[0])) : "memory");
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");
    }
#pragma unroll (MODE == 9 ? 2 : 1)
    for (int u = 0; u < U; ++u) {
      if constexpr (MODE == 14) {  // phase 0 of bars[0] is complete: the wait returns at once
        asm volatile(
            "{\n\t.reg .pred p;\n\tW14:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t"
            "@p bra.uni D14;\n\tbra.uni W14;\n\tD14:\n\t}" ::"r"((uint32_t)__cvta_generic_to_shared(&bars[0]))
            : "memory");
      }
      const unsigned char* rowp = rowbase + (size_t)slot * stage_bytes;
      const double* q = q64 + ((u * kSub) & 4095);
#pragma unroll
      for (int g = 0; g < 8; ++g) {
        const float4 v = *reinterpret_cast<const float4*>(rowp + ((g ^ swz) << 4));
        const double2 q0 = *reinterpret_cast<const double2*>(q + 4 * g);
        const double2 q1 = *reinterpret_cast<const double2*>(q + 4 * g + 2);
        acc8 = __fma_rn(q0.x, (double)v.x, acc8);
        acc8 = __fma_rn(q0.y, (double)v.y, acc8);
        acc8 = __fma_rn(q1.x, (double)v.z, acc8);
        acc8 = __fma_rn(q1.y, (double)v.w, acc8);
      }
      if constexpr (MODE == 14) {
        __syncwarp();
        if (lane == 0)
          asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"((uint32_t)__cvta_generic_to_shared(&bars[1]))
                       : "memory");
      }
      if (++slot == S) slot = 0;
    }
    if (acc8 == 1.2345) out[0] = acc8;
    return;
  }
  constexpr int kAhead = MODE == 4 ? 2 : 1;
  constexpr bool kLate = MODE == 5;
  constexpr bool kBits = MODE == 6 || MODE == 7;
  double acc = 0.0;
  double ka[kSub], kb[kSub];
  Raw raw;
  load_sub(0, raw);
#pragma unroll
  for (int g = 0; g < kSub / 4; ++g) widen4(raw, g, &ka[4 * g]);
  for (int u = 0; u < U; u += 2) {
    if (MODE != 2) load_sub(u + 1, raw);
    chain_sub<MODE != 2, kAhead, kLate, kBits>(ka, kb, raw, q64, (u * kSub) & 4095, acc);
    if (MODE != 2) load_sub(u + 2, raw);
    if (MODE == 2)
      chain_sub<false, kAhead>(ka, kb, raw, q64, ((u + 1) * kSub) & 4095, acc);
    else
      chain_sub<true, kAhead, kLate, kBits>(kb, ka, raw, q64, ((u + 1) * kSub) & 4095, acc);
  }
  if (acc == 1.2345) out[0] = acc;
}

template <int MODE>
void run(const char* name, int lpw) {
  double* out;
  cudaMalloc(&out, 8);
  int S = (180 * 1024) / (4 * lpw * 128) < 20 ? (180 * 1024) / (4 * lpw * 128) : 20;
  if (MODE == 13)
    while (S & (S - 1)) --S;  // a power of two: the slot is a mask
  const int U = 128;
  const size_t smem = (size_t)S * 4 * lpw * 128 + 4096 * 8;
  cudaFuncSetAttribute(lab<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  lab<MODE><<<139, 160, smem>>>(out, U, S, lpw);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  // time U = 1024 subs (32768 steps) minus U = 0 (the shared-memory setup),
  // so the per-step figure is the loop's alone
  auto best_of = [&](int u) {
    float best = 1e9;
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(e0);
      lab<MODE><<<139, 160, smem>>>(out, u, S, lpw);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      best = ms < best ? ms : best;
    }
    return best;
  };
  const int UL = 8 * U;
  const float t0 = best_of(0), t1 = best_of(UL);
  const double steps = (double)UL * kSub;
  const double ns = (t1 - t0) * 1e6 / steps;
  printf("%-50s lpw %2d: setup %.1f us, %.2f ns/step, %.1f cycles/step @1965 MHz  err=%s\n", name, lpw, t0 * 1e3, ns,
         ns * 1.965, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  run<0>("replica", 18);
  run<1>("fixed ring slot", 18);
  run<2>("no next-sub widening", 18);
  run<3>("replica, every lane", 32);
  run<4>("replica, q two groups ahead", 18);
  run<5>("replica, next sub widened in the second half", 18);
  run<6>("replica, integer widening (no F2F)", 18);
  run<7>("integer widening, fixed ring slot", 18);
  run<8>("simple loop (row LDS + q LDS + F2F + DFMA)", 18);
  run<9>("simple loop, segments unrolled by 2", 18);
  run<10>("raw one sub ahead, widened just in time", 18);
  run<11>("raw one sub ahead, JIT widening, q one group ahead", 18);
  run<12>("fp64_rate K1x-shape loop in this harness", 18);
  run<13>("flat step loop over the swizzled ring", 18);
  run<14>("simple loop + per-sub mbarrier wait / arrive", 18);
  return 0;
}
