// umma_bench.cu -- microbenchmark of tcgen05.mma issue/throughput for the prefill shapes
// (dev tool; not part of libeva).  One CTA per SM, one elected thread issues NITER x K-steps
// of an MMA shape into TMEM with operands already resident; reports cycles per MMA.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../include -o umma_bench umma_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

#include "../paper_2511_00576_b200/csrc/sm100.cuh"

using namespace eva::sm100;

template <int MODE>  // 0: SS M128 N64 (S tile), 1: SS M128 N128, 2: TS M128 N128 (PV, B MN-major), 3: SS M128 N256
__global__ void __launch_bounds__(128, 1) bench(int niter, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  uint8_t* a = smem;            // 32 KB: [128 rows][128 B] x 2 sub-tiles
  uint8_t* b = smem + 32768;    // 64 KB
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < (32768 + 65536) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (warp == 0) { tmem_alloc(&tbase, 512); tmem_relinquish(); }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tbase;
  unsigned long long t0 = 0, t1 = 0;
  if (warp == 0) {
    constexpr int N = MODE == 0 ? 64 : MODE == 3 ? 256 : 128;
    const uint32_t idesc = idesc_bf16_f32(128, N, MODE == 2);
    const uint32_t sa = smem_u32(a), sb = smem_u32(b);
    __syncwarp();
    t0 = clock64();
    for (int it = 0; it < niter; ++it) {
      if (elect_one()) {
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {
          if (MODE == 2) {
            const uint64_t bd = smem_desc_sw128(sb + ks * 2048, 16384, 1024);
            mma_ts(tmem + 256, tmem + ks * 8, bd, idesc, 1);
          } else {
            const uint32_t kb = ks >> 2, off = (ks & 3) * 32;
            const uint64_t ad = smem_desc_sw128(sa + kb * 16384 + off, 16, 1024);
            const uint64_t bd = smem_desc_sw128(sb + kb * (N * 128) + off, 16, 1024);
            mma_ss(tmem + (it & 1) * 256, ad, bd, idesc, ks > 0);
          }
        }
      }
      __syncwarp();
    }
    if (elect_one()) mma_commit(&bar);
    __syncwarp();
    mbar_wait(&bar, 0);
    t1 = clock64();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 512);
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 148 * 8);
  const char* names[4] = {"SS M128 N64 K16 (S tile, BN=64)", "SS M128 N128 K16", "TS M128 N128 K16 (PV, A in TMEM)",
                          "SS M128 N256 K16"};
  const double macs[4] = {128.0 * 64 * 16, 128.0 * 128 * 16, 128.0 * 128 * 16, 128.0 * 256 * 16};
  for (int mode = 0; mode < 4; ++mode) {
    for (int grid : {1, 148}) {
      const int niter = 2000;
      const size_t sm = 32768 + 65536;
      void (*fn)(int, unsigned long long*) = mode == 0 ? bench<0> : mode == 1 ? bench<1> : mode == 2 ? bench<2> : bench<3>;
      cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      fn<<<grid, 128, sm>>>(niter, d);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
      unsigned long long h[148];
      cudaMemcpy(h, d, grid * 8, cudaMemcpyDeviceToHost);
      double cyc = 0;
      for (int i = 0; i < grid; ++i) cyc += h[i];
      cyc /= grid;
      const double per = cyc / (niter * 8.0);
      printf("%-36s grid %3d: %7.1f cycles/MMA  %6.0f MAC/clk/SM\n", names[mode], grid, per, macs[mode] / per);
    }
  }
  return 0;
}
