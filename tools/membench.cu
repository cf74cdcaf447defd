// Memory-pattern micro-benchmark: persistent CTAs copy "leaves" of SLOTS
// elements (ELEM bytes each, element k of a leaf at base + k*stride) into
// shared memory and back out, like the leaf kernel does, with no compute.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(512, 1) leafcopy(uint8_t* data, size_t elem, size_t stride_elems, int slots,
                                                   int nleaves, int leaves_per_group, unsigned* ticket) {
  extern __shared__ __align__(16) uint8_t sm[];
  __shared__ unsigned s_t;
  for (;;) {
    if (threadIdx.x == 0) s_t = atomicAdd(ticket, 1u);
    __syncthreads();
    unsigned t = s_t;
    if (t >= (unsigned)nleaves) return;
    // leaf t: group = t / leaves_per_group, member = t % leaves_per_group
    size_t grp = t / leaves_per_group, mem = t % leaves_per_group;
    size_t base = grp * leaves_per_group * slots + mem;  // element index of slot 0 (strided layout)
    size_t pieces = elem / 16;
    for (size_t idx = threadIdx.x; idx < slots * pieces; idx += blockDim.x) {
      size_t s = idx / pieces, p = idx % pieces;
      const uint4* src = reinterpret_cast<const uint4*>(data + (base + s * stride_elems) * elem) + p;
      unsigned sa = (unsigned)__cvta_generic_to_shared(sm + idx * 16);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(src) : "memory");
    }
    asm volatile("cp.async.wait_all;\n" ::: "memory");
    __syncthreads();
    for (size_t idx = threadIdx.x; idx < slots * pieces; idx += blockDim.x) {
      size_t s = idx / pieces, p = idx % pieces;
      uint4* dst = reinterpret_cast<uint4*>(data + (base + s * stride_elems) * elem) + p;
      __stcg(dst, reinterpret_cast<uint4*>(sm)[idx]);
    }
    __syncthreads();
  }
}

int main() {
  const size_t elem = 16384 + 16;
  const size_t L = 1 << 18;
  uint8_t* d;
  cudaMalloc(&d, L * elem);
  unsigned* tk;
  cudaMalloc(&tk, 4);
  const int slots = 8;
  cudaFuncSetAttribute(leafcopy, cudaFuncAttributeMaxDynamicSharedMemorySize, 140 * 1024);
  struct Cfg { const char* name; size_t stride; int lpg; };
  Cfg cfgs[] = {{"contiguous (stride 1)", 1, 1}, {"row-like stride 1 x8", 1, 1},
                {"stride 64 (inner col)", 64, 64}, {"stride 512 (top col)", 512, 512},
                {"stride 32768 (C5 level1)", 32768, 32768}};
  for (auto& c : cfgs) {
    int nleaves = (int)(L / slots);
    for (int rep = 0; rep < 3; ++rep) {
      cudaMemset(tk, 0, 4);
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      cudaEventRecord(a);
      leafcopy<<<148, 512, slots * elem>>>(d, elem, c.stride, slots, nleaves, c.lpg, tk);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (rep == 2)
        printf("%-28s %8.3f ms  %7.1f GB/s (r+w)\n", c.name, ms, 2.0 * nleaves * slots * elem / ms / 1e6);
    }
  }
  cudaError_t e = cudaGetLastError();
  printf("err: %s\n", cudaGetErrorString(e));
  return 0;
}
