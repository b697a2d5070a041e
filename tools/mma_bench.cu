// mma_bench.cu — tcgen05.mma issue-rate microbenchmark (no TMA): one CTA per SM, operands already in
// shared memory (SW128 K-major or MN-major), one thread issues `iters` x 4 MMAs (K = 16 each)
// into one TMEM accumulator, commits, waits; reports cycles per MMA and the implied chip TFLOP/s.
//   nvcc -std=c++20 -O3 -gencode arch=compute_100a,code=sm_100a -I paper_2201_05752_b200/csrc \
//        tools/mma_bench.cu -o /tmp/mma_bench && /tmp/mma_bench
#include <cstdio>

#include "ptx.cuh"

using namespace moses;

template <int N, bool MN>
__global__ void __launch_bounds__(128, 1) mma_kernel(int iters, unsigned long long* cycles) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  constexpr int kA = 128 * 128, kB = N * 128;  // one 64-wide K block of A and B
  for (int i = threadIdx.x; i < (kA + kB) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) {
    ptx::mbar_init(&bar, 1);
    ptx::fence_barrier_init();
  }
  if (threadIdx.x < 32) ptx::tmem_alloc<256>(&slot);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = slot;
  constexpr uint32_t idesc = ptx::umma_idesc(1, MN, MN, 128, N);
  if (threadIdx.x == 0) {
    const uint32_t a = ptx::smem_u32(smem), b = a + kA;
    const unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const uint64_t ad = MN ? ptx::sw128_desc(a + kk * 2048, 64 * 128, 1024, 2) : ptx::sw128_desc(a + kk * 32, 16, 1024);
        const uint64_t bd = MN ? ptx::sw128_desc(b + kk * 2048, 64 * 128, 1024, 2) : ptx::sw128_desc(b + kk * 32, 16, 1024);
        ptx::umma_f16(tmem, ad, bd, idesc, (it | kk) ? 1u : 0u);
      }
    }
    ptx::umma_commit(&bar);
    ptx::mbar_wait(&bar, 0);
    const unsigned long long t1 = clock64();
    cycles[blockIdx.x] = t1 - t0;
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) ptx::tmem_dealloc<256>(tmem);
}

template <int N, bool MN>
void run(int iters) {
  auto k = mma_kernel<N, MN>;
  const int smem = 128 * 128 + N * 128 + 2048;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  unsigned long long* d;
  cudaMalloc(&d, 148 * 8);
  k<<<148, 128, smem>>>(iters, d);  // warm
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<<<148, 128, smem>>>(iters, d);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += double(h[i]) / 148.0;
  const double mmas = 4.0 * iters;
  const double flops = 148.0 * mmas * 2.0 * 128 * N * 16;
  printf("N=%3d %s: %7.1f cycles/MMA (floor %d), kernel %.3f ms -> %.0f TFLOP/s  err=%s\n", N, MN ? "MN-major" : "K-major ",
         avg / mmas, 128 * N / 256, ms, flops / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main1() {
  for (int iters : {64, 1024}) {
    printf("iters=%d (x4 MMAs of K=16)\n", iters);
    run<64, false>(iters);
    run<128, false>(iters);
    run<256, false>(iters);
    run<64, true>(iters);
    run<128, true>(iters);
    run<256, true>(iters);
  }
  return 0;
}

// ---------------------------------------------------------------- TMA streaming rate (no MMA)
#include <cudaTypedefs.h>
template <int STAGES>
__global__ void __launch_bounds__(64, 1) tma_kernel(const __grid_constant__ CUtensorMap map, int nkb, int box_bytes,
                                                    int boxes, int mn, unsigned long long* cycles) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full[STAGES], empty[STAGES];
  const int stage_bytes = box_bytes * boxes;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
    }
    ptx::fence_barrier_init();
  }
  __syncthreads();
  const int col0 = (blockIdx.x % 8) * 64;
  if (threadIdx.x == 0) {  // producer
    int st = 0;
    uint32_t ph = 0;
    const unsigned long long t0 = clock64();
    for (int kb = 0; kb < nkb; ++kb) {
      ptx::mbar_wait(&empty[st], ph ^ 1);
      ptx::mbar_arrive_expect_tx(&full[st], stage_bytes);
      for (int b = 0; b < boxes; ++b) {
        if (mn) ptx::tma_load_2d(smem + st * stage_bytes + b * box_bytes, &map, &full[st], col0 + b * 64, kb * 64);
        else ptx::tma_load_2d(smem + st * stage_bytes + b * box_bytes, &map, &full[st], kb * 64, b * 128);
      }
      if (++st == STAGES) { st = 0; ph ^= 1; }
    }
    cycles[blockIdx.x] = t0;
  } else if (threadIdx.x == 32) {  // consumer: release each stage as soon as it lands
    int st = 0;
    uint32_t ph = 0;
    for (int kb = 0; kb < nkb; ++kb) {
      ptx::mbar_wait(&full[st], ph);
      ptx::mbar_arrive(&empty[st]);
      if (++st == STAGES) { st = 0; ph ^= 1; }
    }
    __syncwarp(1);
  }
  __syncthreads();
  if (threadIdx.x == 0) cycles[blockIdx.x] = clock64() - cycles[blockIdx.x];
}

void tma_run(int grid, int mn, int boxes, int rows) {
  static PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  if (!enc) {
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&enc), cudaEnableDefault, &q);
  }
  void* buf;
  const long long cols = 512, ld = 520;
  cudaMalloc(&buf, rows * ld * 2);
  CUtensorMap m;
  const cuuint64_t dims_mn[2] = {cuuint64_t(cols), cuuint64_t(rows)};
  const cuuint64_t dims_k[2] = {cuuint64_t(rows), cuuint64_t(cols)};  // K-major view: inner = rows (pretend)
  const cuuint64_t strides[1] = {cuuint64_t(ld * 2)};
  const cuuint32_t box_mn[2] = {64, 64}, box_k[2] = {64, 128}, es[2] = {1, 1};
  if (mn) enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims_mn, strides, box_mn, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  else {
    const cuuint64_t d2[2] = {cuuint64_t(cols), cuuint64_t(rows)};
    enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, d2, strides, box_k, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  (void)dims_k;
  const int box_bytes = mn ? 64 * 128 : 128 * 128;
  const int nkb = mn ? rows / 64 : 8;
  constexpr int S = 6;
  const int smem = S * box_bytes * boxes + 1024;
  cudaFuncSetAttribute(tma_kernel<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  unsigned long long* d;
  cudaMalloc(&d, grid * 8);
  tma_kernel<S><<<grid, 64, smem>>>(m, nkb, box_bytes, boxes, mn, d);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  tma_kernel<S><<<grid, 64, smem>>>(m, nkb, box_bytes, boxes, mn, d);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long h[148];
  cudaMemcpy(h, d, grid * 8, cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < grid; ++i) avg += double(h[i]) / grid;
  const double bytes_cta = double(nkb) * box_bytes * boxes;
  printf("TMA %s grid=%3d boxes/stage=%d: %.0f cycles/stage, %.1f B/clk/SM, kernel %.1f us (%s)\n",
         mn ? "MN {64,64} " : "K {64,128}", grid, boxes, avg / nkb, bytes_cta / avg, ms * 1e3,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
  cudaFree(buf);
}

int main2() {
  for (int grid : {40, 148})
    for (int boxes : {1, 3}) {
      tma_run(grid, 1, boxes, 2304);
      tma_run(grid, 0, boxes, 2304);
    }
  return 0;
}

int main() {
  main1();
  main2();
  return 0;
}
