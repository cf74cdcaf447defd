// Memory-pattern micro-benchmark for the radix-8 wave kernel (wave_coset.cuh):
// one warp item = 8 slots (elements base + k*stride) x 4 positions, each a
// 256-byte run of 8 consecutive 32-byte lanes (C5: 512 lanes, step 128), plus
// the lanes' int32 tops (32-byte runs); read from buffer A, written to B.
// Variants of the data movement, no arithmetic:
//   0: cp.async 16 B per thread into a per-warp shared tile, __stcg out
//   1: cp.async.bulk (TMA, 1D) 256-byte runs into shared, mbarrier completion,
//      cp.async.bulk shared->global out
//   2: ld.global.v4 straight into registers, st.global.v4 out (no shared)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/membench2 tools/membench2.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kWarps = 4;
constexpr uint32_t kLanes = 512, kStep = 128, kElem = 16384 + 16;

__device__ __forceinline__ void cp16(uint32_t s, const void* g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(g) : "memory");
}
__device__ __forceinline__ void cp4(uint32_t s, const void* g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(g) : "memory");
}

template <int V>
__global__ void __launch_bounds__(32 * kWarps, 4) pattern(const uint8_t* A, uint8_t* B, const int* TA, int* TB,
                                                          uint64_t nitems, uint32_t nelem) {
  extern __shared__ __align__(128) uint8_t sm[];
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* tile = sm + warp * (8 * 32 * 32 + 8 * 32 * 4 + 64 + (V == 5 ? 8 * 32 * 32 : 0));
  uint64_t* bar = reinterpret_cast<uint64_t*>(tile + 8 * 32 * 32 + 8 * 32 * 4);
  const uint32_t tile_s = (uint32_t)__cvta_generic_to_shared(tile);
  const uint32_t bar_s = (uint32_t)__cvta_generic_to_shared(bar);
  if ((V == 1 || V >= 3) && lane == 0) asm volatile("mbarrier.init.shared.b64 [%0], 1;\n" ::"r"(bar_s) : "memory");
  __syncwarp();
  uint32_t phase = 0;
  const uint64_t gw = (uint64_t)blockIdx.x * kWarps + warp, nw = (uint64_t)gridDim.x * kWarps;
  for (uint64_t it = gw; it < nitems; it += nw) {
    // item -> (leaf, group): 16 groups of 8 cosets per leaf, leaves of 8
    // elements at stride 64 (a row-pass leaf), leaf bases tiled over the buffer
    const uint64_t leaf = it / 16, g = it % 16;
    const uint64_t e0 = (leaf / 64) * 512 + (leaf % 64);
    const uint32_t c = (uint32_t)g * 8 + (lane & 7), pos = lane >> 3;
    const uint32_t L0 = c + kStep * pos;
    if (V == 0) {
#pragma unroll
      for (uint32_t k = 0; k < 8; ++k) {
        const uint64_t e = (e0 + 64ull * k) % nelem;
        const uint8_t* src = A + e * kElem + (uint64_t)L0 * 32;
        cp16(tile_s + (k * 32 + lane) * 32, src);
        cp16(tile_s + (k * 32 + lane) * 32 + 16, src + 16);
        cp4(tile_s + 8 * 32 * 32 + (k * 32 + lane) * 4, TA + e * kLanes + L0);
      }
      asm volatile("cp.async.wait_all;\n" ::: "memory");
      __syncwarp();
#pragma unroll
      for (uint32_t k = 0; k < 8; ++k) {
        const uint64_t e = (e0 + 64ull * k) % nelem;
        uint4* dst = reinterpret_cast<uint4*>(B + e * kElem + (uint64_t)L0 * 32);
        const uint4* s = reinterpret_cast<const uint4*>(tile + (k * 32 + lane) * 32);
        __stcg(dst, s[0]);
        __stcg(dst + 1, s[1]);
        __stcg(TB + e * kLanes + L0, reinterpret_cast<const int*>(tile + 8 * 32 * 32)[k * 32 + lane]);
      }
      __syncwarp();
    } else if (V == 1) {
      // lane j < 32: run (slot j >> 2, position j & 3): 256 B data, 32 B tops
      const uint32_t k = lane >> 2, p = lane & 3;
      const uint64_t e = (e0 + 64ull * k) % nelem;
      const uint32_t l0 = (uint32_t)g * 8 + kStep * p;
      const uint8_t* src = A + e * kElem + (uint64_t)l0 * 32;
      const int* tsrc = TA + e * kLanes + l0;
      if (lane == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;\n" ::"r"(bar_s), "r"(32u * (256 + 32))
                     : "memory");
      __syncwarp();
      const uint32_t dsm = tile_s + (k * 4 + p) * 256, tsm = tile_s + 8 * 32 * 32 + (k * 4 + p) * 32;
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 256, [%2];\n" ::"r"(dsm),
                   "l"(src), "r"(bar_s)
                   : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 32, [%2];\n" ::"r"(tsm),
                   "l"(tsrc), "r"(bar_s)
                   : "memory");
      asm volatile(
          "{\n.reg .pred P;\nW: mbarrier.try_wait.parity.shared.b64 P, [%0], %1;\n@!P bra W;\n}\n" ::"r"(bar_s),
          "r"(phase)
          : "memory");
      phase ^= 1;
      uint8_t* dst = B + e * kElem + (uint64_t)l0 * 32;
      int* tdst = TB + e * kLanes + l0;
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 256;\n" ::"l"(dst), "r"(dsm) : "memory");
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 32;\n" ::"l"(tdst), "r"(tsm) : "memory");
      asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
      __syncwarp();
    } else if (V == 5) {
      // cp.async 16 B/lane in (as V0), rows copied by the lanes into a
      // separate staging area, TMA bulk runs out; the staging area is only
      // waited for before its next reuse
      uint8_t* stage = tile + 8 * 32 * 32 + 8 * 32 * 4 + 64;
      const uint32_t stage_s = (uint32_t)__cvta_generic_to_shared(stage);
#pragma unroll
      for (uint32_t k = 0; k < 8; ++k) {
        const uint64_t e = (e0 + 64ull * k) % nelem;
        const uint8_t* src = A + e * kElem + (uint64_t)L0 * 32;
        cp16(tile_s + (k * 32 + lane) * 32, src);
        cp16(tile_s + (k * 32 + lane) * 32 + 16, src + 16);
        cp4(tile_s + 8 * 32 * 32 + (k * 32 + lane) * 4, TA + e * kLanes + L0);
      }
      asm volatile("cp.async.wait_all;\n" ::: "memory");
      __syncwarp();
      asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
      __syncwarp();
#pragma unroll
      for (uint32_t k = 0; k < 8; ++k) {
        const uint64_t e = (e0 + 64ull * k) % nelem;
        const uint4* s = reinterpret_cast<const uint4*>(tile + (k * 32 + lane) * 32);
        uint4* d = reinterpret_cast<uint4*>(stage + ((k * 4 + pos) * 8 + (lane & 7)) * 32);
        d[0] = s[0];
        d[1] = s[1];
        __stcg(TB + e * kLanes + L0, reinterpret_cast<const int*>(tile + 8 * 32 * 32)[k * 32 + lane]);
      }
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      __syncwarp();
      {
        const uint32_t k = lane >> 2, p = lane & 3;
        const uint64_t e = (e0 + 64ull * k) % nelem;
        const uint32_t l0 = (uint32_t)g * 8 + kStep * p;
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 256;\n" ::"l"(B + e * kElem + (uint64_t)l0 * 32),
                     "r"(stage_s + (k * 4 + p) * 256)
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
      }
    } else if (V == 3 || V == 4) {
      // data runs by TMA (lane j: slot j >> 2, position j & 3), tops by cp.async 4 B per lane
      const uint32_t k = lane >> 2, p = lane & 3;
      const uint64_t e = (e0 + 64ull * k) % nelem;
      const uint32_t l0 = (uint32_t)g * 8 + kStep * p;
      if (lane == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;\n" ::"r"(bar_s), "r"(32u * 256)
                     : "memory");
      __syncwarp();
      const uint32_t dsm = tile_s + (k * 4 + p) * 256;
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 256, [%2];\n" ::"r"(dsm),
                   "l"(A + e * kElem + (uint64_t)l0 * 32), "r"(bar_s)
                   : "memory");
#pragma unroll
      for (uint32_t kk = 0; kk < 8; ++kk) {
        const uint64_t ee = (e0 + 64ull * kk) % nelem;
        cp4(tile_s + 8 * 32 * 32 + (kk * 32 + lane) * 4, TA + ee * kLanes + L0);
      }
      asm volatile("cp.async.wait_all;\n" ::: "memory");
      asm volatile(
          "{\n.reg .pred P;\nW: mbarrier.try_wait.parity.shared.b64 P, [%0], %1;\n@!P bra W;\n}\n" ::"r"(bar_s),
          "r"(phase)
          : "memory");
      phase ^= 1;
      __syncwarp();
      if (V == 3) {
#pragma unroll
        for (uint32_t kk = 0; kk < 8; ++kk) {
          const uint64_t ee = (e0 + 64ull * kk) % nelem;
          uint4* dst = reinterpret_cast<uint4*>(B + ee * kElem + (uint64_t)L0 * 32);
          // this lane's row: slot kk, position pos, coset lane & 7 -> run row (kk*4+pos), entry lane&7
          const uint4* s = reinterpret_cast<const uint4*>(tile + ((kk * 4 + pos) * 8 + (lane & 7)) * 32);
          __stcg(dst, s[0]);
          __stcg(dst + 1, s[1]);
          __stcg(TB + ee * kLanes + L0, reinterpret_cast<const int*>(tile + 8 * 32 * 32)[kk * 32 + lane]);
        }
        __syncwarp();
      } else {
#pragma unroll
        for (uint32_t kk = 0; kk < 8; ++kk) {
          const uint64_t ee = (e0 + 64ull * kk) % nelem;
          __stcg(TB + ee * kLanes + L0, reinterpret_cast<const int*>(tile + 8 * 32 * 32)[kk * 32 + lane]);
        }
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 256;\n" ::"l"(B + e * kElem + (uint64_t)l0 * 32), "r"(dsm) : "memory");
        asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
        __syncwarp();
      }
    } else {
      uint4 r[8][2];
      int t[8];
#pragma unroll
      for (uint32_t k = 0; k < 8; ++k) {
        const uint64_t e = (e0 + 64ull * k) % nelem;
        const uint4* src = reinterpret_cast<const uint4*>(A + e * kElem + (uint64_t)L0 * 32);
        r[k][0] = __ldcg(src);
        r[k][1] = __ldcg(src + 1);
        t[k] = __ldcg(TA + e * kLanes + L0);
      }
#pragma unroll
      for (uint32_t k = 0; k < 8; ++k) {
        const uint64_t e = (e0 + 64ull * k) % nelem;
        uint4* dst = reinterpret_cast<uint4*>(B + e * kElem + (uint64_t)L0 * 32);
        __stcg(dst, r[k][0]);
        __stcg(dst + 1, r[k][1]);
        __stcg(TB + e * kLanes + L0, t[k]);
      }
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
}

int main() {
  const uint32_t nelem = 200704;  // 392 x 512
  uint8_t *A, *B;
  int *TA, *TB;
  cudaMalloc(&A, (size_t)nelem * kElem);
  cudaMalloc(&B, (size_t)nelem * kElem);
  cudaMalloc(&TA, (size_t)nelem * kLanes * 4);
  cudaMalloc(&TB, (size_t)nelem * kLanes * 4);
  const uint64_t nitems = (uint64_t)nelem / 8 * 16;  // every lane of every element once
  const size_t smem = kWarps * (8 * 32 * 32 + 8 * 32 * 4 + 64 + 8 * 32 * 32);
  const double bytes = 2.0 * nitems * 8 * 32 * 36;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  auto run = [&](auto kern, const char* name, int per) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float best = 1e9f;
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(a);
      kern<<<sms * per, 32 * kWarps, smem>>>(A, B, TA, TB, nitems, nelem);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (ms < best) best = ms;
    }
    printf("%-34s CTAs/SM %d  %7.3f ms  %7.1f GB/s (r+w, data+tops)  %s\n", name, per, best, bytes / best / 1e6,
           cudaGetErrorString(cudaGetLastError()));
  };
  for (int per : {2, 3, 4}) {
    run(pattern<0>, "cp.async 16B -> smem -> stcg", per);
    run(pattern<1>, "TMA bulk 256B runs (mbarrier)", per);
    run(pattern<2>, "ld.global.v4 -> regs -> stcg", per);
    run(pattern<3>, "TMA data + cp.async tops, stcg out", per);
    run(pattern<4>, "TMA data + cp.async tops, TMA out", per);
    run(pattern<5>, "cp.async in, staging + TMA out", per);
  }
  cudaMemcpy(B, A, (size_t)nelem * kElem, cudaMemcpyDeviceToDevice);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  cudaMemcpy(B, A, (size_t)nelem * kElem, cudaMemcpyDeviceToDevice);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  printf("cudaMemcpy D2D %.3f ms %.1f GB/s (r+w)\n", ms, 2.0 * nelem * kElem / ms / 1e6);
  return 0;
}
