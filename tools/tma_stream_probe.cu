// tma_stream_probe.cu — how fast can P CTAs stream a weight matrix with TMA box loads into an
// S-stage shared-memory ring (no math: the consumer frees a stage as soon as it is full)?
// The ceiling for the cold-expert kernels (k_ffn_cold.cu, k_ffn_tc.cu split-K): HBM GB/s as a
// function of stages, box rows, row stride (matrix width), CTAs.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tma_stream_probe tools/tma_stream_probe.cu -lcuda
//   tools/tma_stream_probe
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(64, 1) stream_kernel(const __grid_constant__ CUtensorMap tm, int rows, int cols,
                                                       int box_rows, int stages, int items_per_cta, int boxes_per_item) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  __shared__ uint64_t full[16], empty[16];
  uint8_t* ring = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int box_bytes = box_rows * 128;
  const int stage_bytes = box_bytes * boxes_per_item;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&empty[s])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // item i of this CTA = column block (i % kb) of row tile (i / kb) in the CTA's range
  const int kb = cols / 64, row_tiles = rows / box_rows;
  const long total_items = (long)row_tiles * kb / boxes_per_item;
  const long i0 = (long)blockIdx.x * items_per_cta;
  if (threadIdx.x == 0) {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    int s = 0;
    uint32_t ph = 0;
    for (int i = 0; i < items_per_cta; ++i) {
      const long it = (i0 + i) % total_items;
      if (i >= stages) {
        uint32_t ok = 0;
        while (!ok)
          asm volatile("{\n.reg .pred P1;\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\nselp.u32 %0, 1, 0, P1;\n}\n"
                       : "=r"(ok) : "r"(smem_u32(&empty[s])), "r"(ph ^ 1u) : "memory");
      }
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(&full[s])), "r"(stage_bytes) : "memory");
      for (int b = 0; b < boxes_per_item; ++b) {
        const long bi = it * boxes_per_item + b;
        const int rt = (int)(bi / kb), c = (int)(bi % kb);
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
            " [%0], [%1, {%2, %3}], [%4], %5;"
            :: "r"(smem_u32(ring + s * stage_bytes + b * box_bytes)), "l"(&tm), "r"(c * 64), "r"(rt * box_rows),
               "r"(smem_u32(&full[s])), "l"(pol) : "memory");
      }
      if (++s == stages) { s = 0; ph ^= 1u; }
    }
  } else if (threadIdx.x == 32) {
    int s = 0;
    uint32_t ph = 0;
    for (int i = 0; i < items_per_cta; ++i) {
      uint32_t ok = 0;
      while (!ok)
        asm volatile("{\n.reg .pred P1;\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\nselp.u32 %0, 1, 0, P1;\n}\n"
                     : "=r"(ok) : "r"(smem_u32(&full[s])), "r"(ph) : "memory");
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(smem_u32(&empty[s])) : "memory");
      if (++s == stages) { s = 0; ph ^= 1u; }
    }
  }
}


// Cold-kernel gate/up pattern: each stage = one 3-D K-block box from matrix A and one from
// matrix B (W1 / W3 at the same rows and K blocks), box {64, 128, depth}.
__global__ void __launch_bounds__(64, 1) stream2_kernel(const __grid_constant__ CUtensorMap ta,
                                                        const __grid_constant__ CUtensorMap tb, int rows, int cols,
                                                        int depth, int stages, int items_per_cta) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  __shared__ uint64_t full[16], empty[16];
  uint8_t* ring = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int box_bytes = 128 * 128 * depth;
  const int stage_bytes = 2 * box_bytes;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&empty[s])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int kb = cols / 64 / depth, row_tiles = rows / 128;
  const long total_items = (long)row_tiles * kb;
  const long i0 = (long)blockIdx.x * items_per_cta;
  if (threadIdx.x == 0) {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    int s = 0;
    uint32_t ph = 0;
    for (int i = 0; i < items_per_cta; ++i) {
      const long it = (i0 + i) % total_items;
      const int rt = (int)(it / kb), c = (int)(it % kb);
      if (i >= stages) {
        uint32_t ok = 0;
        while (!ok)
          asm volatile("{\n.reg .pred P1;\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\nselp.u32 %0, 1, 0, P1;\n}\n"
                       : "=r"(ok) : "r"(smem_u32(&empty[s])), "r"(ph ^ 1u) : "memory");
      }
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(&full[s])), "r"(stage_bytes) : "memory");
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
          " [%0], [%1, {%2, %3, %4}], [%5], %6;"
          :: "r"(smem_u32(ring + s * stage_bytes)), "l"(&ta), "r"(0), "r"(rt * 128), "r"(c * depth),
             "r"(smem_u32(&full[s])), "l"(pol) : "memory");
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
          " [%0], [%1, {%2, %3, %4}], [%5], %6;"
          :: "r"(smem_u32(ring + s * stage_bytes + box_bytes)), "l"(&tb), "r"(0), "r"(rt * 128), "r"(c * depth),
             "r"(smem_u32(&full[s])), "l"(pol) : "memory");
      if (++s == stages) { s = 0; ph ^= 1u; }
    }
  } else if (threadIdx.x == 32) {
    int s = 0;
    uint32_t ph = 0;
    for (int i = 0; i < items_per_cta; ++i) {
      uint32_t ok = 0;
      while (!ok)
        asm volatile("{\n.reg .pred P1;\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\nselp.u32 %0, 1, 0, P1;\n}\n"
                     : "=r"(ok) : "r"(smem_u32(&full[s])), "r"(ph) : "memory");
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(smem_u32(&empty[s])) : "memory");
      if (++s == stages) { s = 0; ph ^= 1u; }
    }
  }
}

typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                        const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  Enc enc = (Enc)fn;
  const size_t bytes = (size_t)4 << 30;   // 4 GiB >> L2
  void* buf;
  cudaMalloc(&buf, bytes);
  cudaMemset(buf, 1, bytes);
  cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  printf("{\"sms\": %d}\n", sms);
  const int widths[] = {4096, 14336, 2048, 1408};
  for (int w : widths) {
    if (getenv("PROBE_SKIP_2D")) break;
    const int rows = (int)(bytes / 2 / w) / 256 * 256;
    for (int box_rows : {64, 128, 256}) {
      CUtensorMap tm;
      cuuint64_t dims[2] = {(cuuint64_t)w, (cuuint64_t)rows};
      cuuint64_t strides[1] = {(cuuint64_t)w * 2};
      cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
      cuuint32_t es[2] = {1, 1};
      enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      for (int boxes : {1, 2}) {
        const int stage_bytes = box_rows * 128 * boxes;
        for (int stages = 2; stages <= 12; stages += 2) {
          if (stages * stage_bytes > 212 * 1024) continue;
          for (int P : {sms, sms / 2}) {
            const int items = (int)(((size_t)1 << 30) / stage_bytes / P);   // 1 GiB per launch
            for (int rep = 0; rep < 3; ++rep) {
              cudaEventRecord(a);
              stream_kernel<<<P, 64, stages * stage_bytes + 1024>>>(tm, rows, w, box_rows, stages, items, boxes);
              cudaEventRecord(b);
              cudaEventSynchronize(b);
            }
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            const double gbs = (double)items * P * stage_bytes / (ms * 1e-3) / 1e9;
            printf("{\"width\": %d, \"box_rows\": %d, \"boxes_per_stage\": %d, \"stages\": %d, \"ctas\": %d, "
                   "\"inflight_kb_per_sm\": %d, \"gbs\": %.0f, \"err\": \"%s\"}\n",
                   w, box_rows, boxes, stages, P, stages * stage_bytes / 1024, gbs, cudaGetErrorString(cudaGetLastError()));
            fflush(stdout);
          }
        }
      }
    }
  }
  // W1/W3 pattern: two matrices of [rows, w], 3-D K-block boxes {64, 128, depth}
  cudaFuncSetAttribute(stream2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  for (int w : {2048, 4096}) {
    const size_t half = bytes / 2;
    const int rows = (int)(half / 2 / w) / 128 * 128;
    CUtensorMap ta, tb;
    for (int depth : {1, 2, 4}) {
      for (int m = 0; m < 2; ++m) {
        cuuint64_t dims[3] = {64, (cuuint64_t)rows, (cuuint64_t)(w / 64)};
        cuuint64_t strides[2] = {(cuuint64_t)w * 2, 128};
        cuuint32_t box[3] = {64, 128, (cuuint32_t)depth};
        cuuint32_t es[3] = {1, 1, 1};
        enc(m ? &tb : &ta, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, (char*)buf + m * half, dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      }
      const int stage_bytes = 2 * 128 * 128 * depth;
      for (int stages = 2; stages <= 6; ++stages) {
        if (stages * stage_bytes > 212 * 1024) continue;
        for (int P : {sms}) {
          const int items = (int)(((size_t)1 << 30) / stage_bytes / P);
          float ms = 0;
          for (int rep = 0; rep < 3; ++rep) {
            cudaEventRecord(a);
            stream2_kernel<<<P, 64, stages * stage_bytes + 1024>>>(ta, tb, rows, w, depth, stages, items);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
          }
          cudaEventElapsedTime(&ms, a, b);
          printf("{\"mode\": \"w1w3_3d\", \"width\": %d, \"depth\": %d, \"stages\": %d, \"ctas\": %d, "
                 "\"inflight_kb_per_sm\": %d, \"gbs\": %.0f, \"err\": \"%s\"}\n", w, depth, stages, P,
                 stages * stage_bytes / 1024, (double)items * P * stage_bytes / (ms * 1e-3) / 1e9,
                 cudaGetErrorString(cudaGetLastError()));
          fflush(stdout);
        }
      }
    }
  }
  return 0;
}
