// tma3d_probe.cu — checks the 3-D "K-block" view of a row-major matrix used by the cold kernel:
// dims {64, rows, cols/64}, strides {cols*2, 128 B}, box {64, box_rows, depth}, 128-B swizzle.
// One load must land as `depth` consecutive K-major SW128 tiles [kb][row][64] (each box_rows*128 B).
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
__global__ void k(const __grid_constant__ CUtensorMap tm, uint16_t* out, int c0, int r0, int kb0, int bytes) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  uint8_t* s = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar), d = (uint32_t)__cvta_generic_to_shared(s);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(b));
    asm volatile("fence.mbarrier_init.release.cluster;");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(b), "r"(bytes));
    asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                 :: "r"(d), "l"(&tm), "r"(c0), "r"(r0), "r"(kb0), "r"(b) : "memory");
    uint32_t ok = 0;
    while (!ok) asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\nselp.u32 %0,1,0,p;\n}" : "=r"(ok) : "r"(b));
  }
  __syncthreads();
  for (int i = threadIdx.x; i < bytes / 2; i += blockDim.x) out[i] = ((uint16_t*)s)[i];
}
typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                        const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int main() {
  const int rows = 512, cols = 1408, box_rows = 128;
  uint16_t* h = new uint16_t[rows * cols];
  for (int r = 0; r < rows; ++r) for (int c = 0; c < cols; ++c) h[r * cols + c] = (uint16_t)((r * 7 + c * 13) & 0xffff);
  uint16_t *dm, *dout;
  cudaMalloc(&dm, rows * cols * 2); cudaMemcpy(dm, h, rows * cols * 2, cudaMemcpyHostToDevice);
  cudaMalloc(&dout, 1 << 20);
  void* fn; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  int bad_total = 0;
  for (int depth : {2, 4}) {
    CUtensorMap tm;
    cuuint64_t dims[3] = {64, (cuuint64_t)rows, (cuuint64_t)(cols / 64)};
    cuuint64_t strides[2] = {(cuuint64_t)cols * 2, 128};
    cuuint32_t box[3] = {64, (cuuint32_t)box_rows, (cuuint32_t)depth};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = ((Enc)fn)(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT16, 3, dm, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("depth %d encode %d\n", depth, (int)r);
    if (r) { bad_total++; continue; }
    const int bytes = 128 * box_rows * depth, r0 = 128, kb0 = 3;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes + 1024);
    k<<<1, 256, bytes + 1024>>>(tm, dout, 0, r0, kb0, bytes);
    uint16_t* o = new uint16_t[bytes / 2];
    cudaError_t e = cudaMemcpy(o, dout, bytes, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int kb = 0; kb < depth; ++kb) for (int rr = 0; rr < box_rows; ++rr) for (int c = 0; c < 64; ++c) {
      const int off = kb * box_rows * 128 + rr * 128 + (((c / 8) ^ (rr % 8)) * 16) + (c % 8) * 2;
      const int gr = r0 + rr, gc = (kb0 + kb) * 64 + c;
      if (gc >= cols) continue;
      if (o[off / 2] != h[gr * cols + gc]) bad++;
    }
    printf("depth %d launch %s mismatches %d\n", depth, cudaGetErrorString(e), bad);
    bad_total += bad;
  }
  printf(bad_total ? "FAIL\n" : "OK\n");
  return 0;
}
