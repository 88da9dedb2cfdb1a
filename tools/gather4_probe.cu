// Probe of TMA tile::gather4 semantics on sm_100a (not part of libamoe):
// which tensor-map box shapes are accepted and where 4 gathered rows land in a 128-byte-swizzled
// shared-memory tile. Build: nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/g4 tools/gather4_probe.cu
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdint.h>

typedef CUresult (*PFN_encode)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                               const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                               CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

__global__ void probe(const __grid_constant__ CUtensorMap tm, int r0, int r1, int r2, int r3, int nrows_out,
                      uint16_t* out) {
  extern __shared__ __align__(1024) uint8_t raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar;
  uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar);
  uint32_t d = (uint32_t)__cvta_generic_to_shared(sm);
  for (int i = threadIdx.x; i < 8 * 128 / 2; i += blockDim.x) ((uint16_t*)sm)[i] = 0xFFFF;
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(b));
    asm volatile("fence.mbarrier_init.release.cluster;");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(b), "r"(4 * 128));
    // place the 4 rows at rows 4..7 of the 8-row swizzle atom (offset 512 B)
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
        :: "r"(d + 512), "l"(&tm), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(b) : "memory");
    asm volatile(
        "{\n.reg .pred P;\nW: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n@!P bra W;\n}" :: "r"(b));
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nrows_out * 64; i += blockDim.x) out[i] = ((uint16_t*)sm)[i];
}

int main() {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  PFN_encode enc = (PFN_encode)p;
  const int R = 256, Cc = 64;
  uint16_t* h = (uint16_t*)malloc(R * Cc * 2);
  for (int r = 0; r < R; ++r)
    for (int c = 0; c < Cc; ++c) h[r * Cc + c] = (uint16_t)(r * 64 + c);   // value encodes (row, col)
  uint16_t* dsrc;
  cudaMalloc(&dsrc, R * Cc * 2);
  cudaMemcpy(dsrc, h, R * Cc * 2, cudaMemcpyHostToDevice);
  uint16_t* dout;
  cudaMalloc(&dout, 8 * 64 * 2);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 8192);
  for (int boxr = 1; boxr <= 4; boxr *= 4) {
    CUtensorMap tm;
    cuuint64_t dims[2] = {(cuuint64_t)Cc, (cuuint64_t)R};
    cuuint64_t str[1] = {(cuuint64_t)Cc * 2};
    cuuint32_t box[2] = {64, (cuuint32_t)boxr};
    cuuint32_t es[2] = {1, 1};
    CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dsrc, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("box {64,%d}: encode %d\n", boxr, (int)r);
    if (r != CUDA_SUCCESS) continue;
    cudaMemset(dout, 0, 8 * 64 * 2);
    probe<<<1, 128, 8192>>>(tm, 5, 17, 3, 200, 8, dout);
    cudaError_t e = cudaDeviceSynchronize();
    printf("  kernel: %s\n", cudaGetErrorString(e));
    if (e != cudaSuccess) return 1;
    uint16_t o[8 * 64];
    cudaMemcpy(o, dout, sizeof(o), cudaMemcpyDeviceToHost);
    // for each smem row 4..7 and 16-byte chunk j, print which (row, chunk) of the source is there
    for (int sr = 4; sr < 8; ++sr) {
      printf("  smem row %d:", sr);
      for (int j = 0; j < 8; ++j) {
        uint16_t v = o[sr * 64 + j * 8];
        printf(" (%d,%d)", v / 64, (v % 64) / 8);
      }
      printf("\n");
    }
  }
  return 0;
}
