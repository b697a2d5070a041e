// tma_bench.cu — per-SM TMA ingest microbenchmark: `ctas` CTAs (one per SM) each stream `mb` MB of
// 2-D TMA boxes from a global buffer into an S-stage shared-memory ring; one consumer thread releases
// each stage as soon as it lands (no compute). Reports bytes per SM clock and the chip aggregate, for
// ring depths, box shapes and L2-resident vs HBM-resident sources — the limit every streaming GEMM in
// this library is built around.
//   nvcc -std=c++20 -O3 -gencode arch=compute_100a,code=sm_100a -I paper_2201_05752_b200/csrc \
//        tools/tma_bench.cu -o /tmp/tma_bench -lcuda && /tmp/tma_bench
#include <cuda.h>
#include <cuda_bf16.h>

#include <cstdio>
#include <vector>

#include "ptx.cuh"

using namespace moses;

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                               const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                               CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncodeFn encode() {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  return reinterpret_cast<EncodeFn>(fn);
}

// rows x cols bf16 matrix, box {box_c, box_r}, 128B swizzle
static CUtensorMap make_map(void* base, long long rows, long long cols, int box_c, int box_r) {
  CUtensorMap m;
  const cuuint64_t dims[2] = {cuuint64_t(cols), cuuint64_t(rows)};
  const cuuint64_t strides[1] = {cuuint64_t(cols) * 2};
  const cuuint32_t box[2] = {cuuint32_t(box_c), cuuint32_t(box_r)};
  const cuuint32_t es[2] = {1, 1};
  CUresult r = encode()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) printf("encode failed %d\n", int(r));
  return m;
}

// `producers` warps (each elects lane 0) issue the boxes of every stage round-robin; warp 0 also
// posts the stage's expected byte count. The consumer is the warp after the producers.
__global__ void __launch_bounds__(160, 1) tma_kernel(const __grid_constant__ CUtensorMap map, int stages, int box_bytes,
                                                     int boxes_per_stage, long long n_stages_total, int box_r,
                                                     long long rows, unsigned long long* cycles, int producers) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full[16], empty[16];
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
    }
    ptx::fence_barrier_init();
  }
  __syncthreads();
  const int stage_bytes = box_bytes * boxes_per_stage;
  const int row_blocks = int(rows / box_r);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp < producers && lane == 0) {
    const unsigned long long t0 = clock64();
    int s = 0;
    uint32_t ph = 0;
    int blk = (int(blockIdx.x) * 97) % row_blocks;
    for (long long i = 0; i < n_stages_total; ++i) {
      ptx::mbar_wait(&empty[s], ph ^ 1);
      if (warp == 0) ptx::mbar_arrive_expect_tx(&full[s], stage_bytes);
      for (int b = warp; b < boxes_per_stage; b += producers) {
        int rb = blk + b;
        if (rb >= row_blocks) rb -= row_blocks;
        ptx::tma_load_2d(smem + s * stage_bytes + b * box_bytes, &map, &full[s], 0, rb * box_r);
      }
      blk += boxes_per_stage;
      if (blk >= row_blocks) blk -= row_blocks;
      if (++s == stages) { s = 0; ph ^= 1; }
    }
    if (warp == 0) {
      ptx::mbar_wait(&empty[(s + stages - 1) % stages], (s == 0) ? (ph ^ 1) : ph);
      cycles[blockIdx.x] = clock64() - t0;
    }
  } else if (warp == producers && lane == 0) {  // consumer
    int s = 0;
    uint32_t ph = 0;
    for (long long i = 0; i < n_stages_total; ++i) {
      ptx::mbar_wait(&full[s], ph);
      ptx::mbar_arrive(&empty[s]);
      if (++s == stages) { s = 0; ph ^= 1; }
    }
  }
}

int main() {
  int dev = 0;
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, dev);
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  const long long big_rows = 1LL << 23;  // 8M rows x 64 bf16 = 1 GB (HBM-resident)
  void* buf = nullptr;
  cudaMalloc(&buf, big_rows * 128);
  cudaMemset(buf, 1, big_rows * 128);
  unsigned long long* d;
  cudaMalloc(&d, 1024 * 8);
  if (cudaFuncSetAttribute(tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024 + 1024) != cudaSuccess)
    printf("attr failed\n");
  printf("{\"sm_clock_khz\": %d, \"results\": [\n", clk);
  bool first = true;
  for (int producers : {1, 2, 4}) {
  for (int cols : {512}) {                                  // 128 B of 1 KB rows
  for (long long rows : {(1LL << 17) * 64 / cols}) {        // 16 MB (L2-resident)
    for (int box_r : {64, 128, 256}) {                     // box {64 cols, box_r rows}: 8 / 16 / 32 KB
      CUtensorMap map = make_map(buf, rows, cols, 64, box_r);
      const int box_bytes = 128 * box_r;
      for (int stage_kb : {16, 32, 64}) {
        if (stage_kb * 1024 < box_bytes) continue;
        const int bps = stage_kb * 1024 / box_bytes;
        for (int stages : {3}) {
          if (stages * stage_kb > 200) continue;
          for (int ctas : {148}) {
            const long long per_cta = 16LL << 20;  // 16 MB per CTA
            const long long nst = per_cta / (stage_kb * 1024);
            const int smem = stages * stage_kb * 1024 + 1024;
            tma_kernel<<<ctas, 160, smem>>>(map, stages, box_bytes, bps, nst / 8, box_r, rows, d, producers);  // warm
            if (cudaError_t e0 = cudaDeviceSynchronize(); e0 != cudaSuccess) {
              printf("\nwarm launch error %s (ctas %d smem %d)\n", cudaGetErrorString(e0), ctas, smem);
              return 1;
            }
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            cudaEventRecord(e0);
            tma_kernel<<<ctas, 160, smem>>>(map, stages, box_bytes, bps, nst, box_r, rows, d, producers);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            std::vector<unsigned long long> cyc(ctas);
            cudaMemcpy(cyc.data(), d, ctas * 8, cudaMemcpyDeviceToHost);
            double avg = 0;
            for (auto c : cyc) avg += double(c);
            avg /= ctas;
            const double bytes = double(nst) * stage_kb * 1024;
            printf("%s{\"producers\": %d, \"row_bytes\": %d, \"box_kb\": %d, \"stage_kb\": %d, \"stages\": %d, \"ctas\": %d, "
                   "\"B_per_clk_per_sm\": %.1f, \"chip_TBps\": %.2f}",
                   first ? "" : ",\n", producers, cols * 2, box_bytes / 1024, stage_kb, stages, ctas,
                   bytes / avg, bytes * ctas / (ms * 1e-3) / 1e12);
            first = false;
            cudaError_t e = cudaGetLastError();
            if (e != cudaSuccess) {
              printf("\nerror %s\n", cudaGetErrorString(e));
              return 1;
            }
          }
        }
      }
    }
  }
  }
  }
  printf("\n]}\n");
  return 0;
}
