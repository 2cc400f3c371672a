// Probe: cp.async.bulk.tensor 2-D LOAD with a box origin that is not a multiple of 4 floats in the inner
// dimension (odd row start), and negative origins (zero fill).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>
__global__ void k(const __grid_constant__ CUtensorMap tm, int r0, int c0, float* out) {
  __shared__ __align__(128) float sm[48 * 16];
  __shared__ __align__(8) unsigned long long bar;
  unsigned b = (unsigned)__cvta_generic_to_shared(&bar), s = (unsigned)__cvta_generic_to_shared(sm);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
    asm volatile("fence.mbarrier_init.release.cluster;");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(48 * 16 * 4));
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                 ::"r"(s), "l"(&tm), "r"(r0), "r"(c0), "r"(b) : "memory");
  }
  __syncthreads();
  asm volatile("{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(b));
  for (int i = threadIdx.x; i < 48 * 16; i += blockDim.x) out[i] = sm[i];
}
using Enc = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                         const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                         CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int main() {
  void* fp; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  Enc enc = (Enc)fp;
  const int G = 128, X = 64;
  std::vector<float> h(G * X);
  for (int i = 0; i < G * X; ++i) h[i] = (float)i;
  float *d, *o; cudaMalloc(&d, 4 * G * X); cudaMalloc(&o, 4 * 48 * 16);
  cudaMemcpy(d, h.data(), 4 * G * X, cudaMemcpyHostToDevice);
  CUtensorMap tm;
  cuuint64_t dims[2] = {G, X}, str[1] = {4 * G};
  cuuint32_t box[2] = {48, 16}, es[2] = {1, 1};
  enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  int cases[5][2] = {{4, 2}, {5, 3}, {7, 1}, {-3, -1}, {101, 50}};
  for (auto& c : cases) {
    cudaMemset(o, 0xff, 4 * 48 * 16);
    k<<<1, 128>>>(tm, c[0], c[1], o);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<float> r(48 * 16);
    cudaMemcpy(r.data(), o, 4 * 48 * 16, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int j = 0; j < 16; ++j) for (int i = 0; i < 48; ++i) {
      const int R = c[0] + i, C = c[1] + j;
      const float want = (R >= 0 && R < G && C >= 0 && C < X) ? (float)(R + G * C) : 0.f;
      if (r[i + 48 * j] != want) ++bad;
    }
    printf("r0=%d c0=%d err=%s bad=%d\n", c[0], c[1], cudaGetErrorString(e), bad);
    if (e != cudaSuccess) return 1;
  }
}
