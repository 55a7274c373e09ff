// umma_bench.cu -- microbenchmark of tcgen05.mma issue/throughput for the prefill shapes
// (dev tool; not part of libeva).  One CTA per SM, one elected thread issues NITER x K-steps
// of an MMA shape into TMEM with operands already resident; reports cycles per MMA.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../include -o umma_bench umma_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

#include "../paper_2511_00576_b200/csrc/sm100.cuh"

using namespace eva::sm100;

// 0: SS M128 N64 (S tile), 1: SS M128 N128, 2: TS M128 N128 (PV, B MN-major), 3: SS M128 N256
// LOAD: 0 none, 1 warps 4..7 hammer TMEM with ld/st (softmax-like) on columns 384..511,
//       2 warps 4..7 run MUFU ex2 loops (no TMEM)
template <int MODE, int LOAD = 0, int COMMITS = 0>
__global__ void __launch_bounds__(256, 1) bench(int niter, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint64_t bar2[4];
  __shared__ uint32_t tbase;
  uint8_t* a = smem;            // 32 KB: [128 rows][128 B] x 2 sub-tiles
  uint8_t* b = smem + 32768;    // 64 KB
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < (32768 + 65536) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); for (int i = 0; i < 4; ++i) mbar_init(&bar2[i], 1); fence_mbar_init(); }
  if (warp == 0) { tmem_alloc(&tbase, 512); tmem_relinquish(); }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tbase;
  unsigned long long t0 = 0, t1 = 0;
  __shared__ volatile int stop;
  if (threadIdx.x == 0) stop = 0;
  __syncthreads();
  if (warp >= 4 && LOAD == 1) {
    const uint32_t ta = tmem + 384 + ((uint32_t)((warp & 3) * 32) << 16);
    float acc = 0.f;
    while (!stop) {
      uint32_t r[32];
      tmem_ld32(ta, r);
      tmem_wait_ld();
#pragma unroll
      for (int i = 0; i < 32; ++i) acc += __uint_as_float(r[i]);
      uint32_t w[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) w[i] = r[i] ^ 1u;
      tmem_st32(ta + 32, w);
      tmem_wait_st();
    }
    if (acc == 12345.f) out[1000] = 1;
  }
  if (warp >= 4 && LOAD == 2) {
    float x = threadIdx.x * 1e-3f;
    while (!stop) {
#pragma unroll
      for (int i = 0; i < 64; ++i) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x));
    }
    if (x == 12345.f) out[1000] = 1;
  }
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
#pragma unroll
        for (int c = 0; c < COMMITS; ++c) mma_commit(&bar2[c]);
      }
      __syncwarp();
    }
    if (elect_one()) mma_commit(&bar);
    __syncwarp();
    mbar_wait(&bar, 0);
    t1 = clock64();
    stop = 1;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 512);
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 1024 * 8);
  const char* names[4] = {"SS M128 N64 K16 (S tile, BN=64)", "SS M128 N128 K16", "TS M128 N128 K16 (PV, A in TMEM)",
                          "SS M128 N256 K16"};
  const double macs[4] = {128.0 * 64 * 16, 128.0 * 128 * 16, 128.0 * 128 * 16, 128.0 * 256 * 16};
  {
    void (*cf[3])(int, unsigned long long*) = {bench<0, 0, 1>, bench<0, 0, 2>, bench<0, 0, 4>};
    for (int k = 0; k < 3; ++k) {
      const size_t sm = 32768 + 65536;
      cudaFuncSetAttribute(cf[k], cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      cf[k]<<<148, 256, sm>>>(2000, d);
      cudaDeviceSynchronize();
      unsigned long long h[148];
      cudaMemcpy(h, d, 148 * 8, cudaMemcpyDeviceToHost);
      double cyc = 0;
      for (int i = 0; i < 148; ++i) cyc += h[i];
      printf("SS N64 groups of 8 + %d commit(s): %.1f cycles/MMA\n", k == 2 ? 4 : k + 1, cyc / 148 / (2000 * 8.0));
    }
  }
  for (int mode = 0; mode < 4; ++mode) {
    for (int grid : {148}) {
      const int niter = 2000;
      const size_t sm = 32768 + 65536;
      void (*fns[12])(int, unsigned long long*) = {bench<0>, bench<1>, bench<2>, bench<3>, bench<0, 1>, bench<1, 1>,
                                                    bench<2, 1>, bench<3, 1>, bench<0, 2>, bench<1, 2>, bench<2, 2>, bench<3, 2>};
      auto fn = fns[mode];
      cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      fn<<<grid, 256, sm>>>(niter, d);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
      unsigned long long h[148];
      cudaMemcpy(h, d, grid * 8, cudaMemcpyDeviceToHost);
      double cyc = 0;
      for (int i = 0; i < grid; ++i) cyc += h[i];
      cyc /= grid;
      const double per = cyc / (niter * 8.0);
      const char* load[3] = {"", " + TMEM ld/st load", " + MUFU load"};
      printf("%-36s%-20s grid %3d: %7.1f cycles/MMA  %6.0f MAC/clk/SM\n", names[mode % 4], load[mode / 4], grid, per,
             macs[mode % 4] / per);
    }
  }
  return 0;
}
