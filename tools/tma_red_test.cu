// Probe: cp.reduce.async.bulk.tensor.3d (add, f32) from a 1024-byte aligned staging tile, swizzle none / 128B.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>
__global__ void k(const __grid_constant__ CUtensorMap tm, int swz, int r0, int c0) {
  extern __shared__ __align__(1024) float sm[];
  unsigned base = (unsigned)__cvta_generic_to_shared(sm);
  unsigned st = (base + 1023u) & ~1023u;
  int lane = threadIdx.x;  // one warp: lane = rs + 2*col
  int rs = lane & 1, col = lane >> 1;
  for (int j = 0; j < 4; ++j) {
    unsigned chunk = swz ? ((4 * rs + j) ^ (col & 7)) : (4 * rs + j);
    unsigned a = st + 128u * col + 16u * chunk;
    float v0 = 1000 * col + 16 * rs + 4 * j;
    asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(a), "f"(v0), "f"(v0 + 1), "f"(v0 + 2), "f"(v0 + 3) : "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncwarp();
  if (lane == 0) {
    asm volatile("cp.reduce.async.bulk.tensor.3d.global.shared::cta.add.tile.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(&tm),
                 "r"(r0), "r"(c0), "r"(0), "r"(st) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}
using Enc = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                         const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                         CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int main() {
  void* fp; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  Enc enc = (Enc)fp;
  const int X = 32;
  float* d; cudaMalloc(&d, 4 * 64 * X);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 8192);
  int cases[4][3] = {{64, 4, 2}, {32, 0, 0}, {32, 8, 20}, {32, 30, 31}};
  for (int cs = 0; cs < 4; ++cs)
  for (int swz = 0; swz < 2; ++swz) {
    const int G = cases[cs][0], r0 = cases[cs][1], c0 = cases[cs][2];
    cudaMemset(d, 0, 4 * G * X);
    CUtensorMap tm;
    cuuint64_t dims[3] = {(cuuint64_t)G, (cuuint64_t)X, 1}, str[2] = {(cuuint64_t)(4 * G), (cuuint64_t)(4 * G * X)};
    cuuint32_t box[3] = {32, 16, 1}, es[3] = {1, 1, 1};
    CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     swz ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    k<<<1, 32, 8192>>>(tm, swz, r0, c0);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<float> h(G * X);
    cudaMemcpy(h.data(), d, 4 * G * X, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int c = 0; c < 16; ++c) for (int rr = 0; rr < 32; ++rr) {
      const int R = r0 + rr, C = c0 + c;
      if (R >= 0 && R < G && C >= 0 && C < X && h[R + G * C] != 1000 * c + rr) ++bad;
    }
    printf("G=%d r0=%d c0=%d swz=%d enc=%d err=%s bad=%d\n", G, r0, c0, swz, (int)r, cudaGetErrorString(e), bad);
    if (e != cudaSuccess) return 1;
  }
}
