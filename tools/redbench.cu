// redbench.cu — flush cost of the forward kernel's accumulators: per-thread red.global.add.f32
// versus STS into a shared-memory staging box + one TMA bulk reduce-add (cp.reduce.async.bulk.tensor)
// per mode.  Each CTA "item" flushes NM modes x (32 x 16) floats to box positions scattered over a
// 2048 x 2048 fp32 image (L2-resident, as g_hat is inside the MLEM graph).  Reports elements/s.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>
#include <vector>

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e_ = (x);                                                       \
    if (e_ != cudaSuccess) {                                                    \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      return 1;                                                                 \
    }                                                                           \
  } while (0)

constexpr int G = 2048, TR = 32, TC = 16, NM = 26;

__device__ __forceinline__ unsigned hash(unsigned x) {
  x ^= x >> 16;
  x *= 0x7feb352dU;
  x ^= x >> 15;
  x *= 0x846ca68bU;
  x ^= x >> 16;
  return x;
}

// positions: item it, mode c -> box origin (r, c) with r, c in [0, G - 32)
__device__ __forceinline__ void origin(int it, int c, int& r0, int& c0) {
  const unsigned h = hash(it * 131u + c * 7919u);
  r0 = (h % (G - TR)) & ~3;
  c0 = (h / 4096u) % (G - TC);
}

__global__ void __launch_bounds__(256, 2) red_kernel(float* g, int items) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int it = blockIdx.x; it < items; it += gridDim.x) {
#pragma unroll
    for (int c = 0; c < NM; ++c) {
      int r0, c0;
      origin(it, c, r0, c0);
      float* p = g + (r0 + lane) + (long long)G * (c0 + warp);
      const float v = 1.0f + c;
      asm volatile("red.global.add.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
      asm volatile("red.global.add.f32 [%0], %1;" ::"l"(p + 8LL * G), "f"(v) : "memory");
    }
  }
}

__global__ void __launch_bounds__(256, 2) tma_kernel(const __grid_constant__ CUtensorMap tm, int items) {
  extern __shared__ __align__(128) float st[];  // NM boxes of 32 x 16
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned sb = (unsigned)__cvta_generic_to_shared(st);
  for (int it = blockIdx.x; it < items; it += gridDim.x) {
    if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    __syncthreads();
#pragma unroll
    for (int c = 0; c < NM; ++c) {
      st[c * TR * TC + lane + TR * warp] = 1.0f + c;
      st[c * TR * TC + lane + TR * (warp + 8)] = 1.0f + c;
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int c = 0; c < NM; ++c) {
        int r0, c0;
        origin(it, c, r0, c0);
        asm volatile(
            "cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.tile.bulk_group [%0, {%1, %2}], [%3];" ::"l"(&tm),
            "r"(r0), "r"(c0), "r"(sb + 4u * c * TR * TC)
            : "memory");
      }
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
  }
  if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  float* g;
  CK(cudaMalloc(&g, sizeof(float) * G * G));
  CK(cudaMemset(g, 0, sizeof(float) * G * G));
  void* fp = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q));
  auto enc = reinterpret_cast<EncodeTiledFn>(fp);
  CUtensorMap tm;
  const cuuint64_t dims[2] = {G, G}, strides[1] = {4ull * G};
  const cuuint32_t box[2] = {TR, TC}, es[2] = {1, 1};
  if (enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, g, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
      CUDA_SUCCESS) {
    printf("encode failed\n");
    return 1;
  }
  const int smem = NM * TR * TC * 4;
  CK(cudaFuncSetAttribute(tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int items = 296 * 40;
  for (int v = 0; v < 2; ++v) {
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(a);
      if (v == 0)
        red_kernel<<<296, 256>>>(g, items);
      else
        tma_kernel<<<296, 256, smem>>>(tm, items);
      cudaEventRecord(b);
      CK(cudaEventSynchronize(b));
      CK(cudaGetLastError());
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      const double elems = (double)items * NM * TR * TC;
      printf("%s: %.3f ms, %.1f G elem/s\n", v == 0 ? "red.global.add.f32" : "tma reduce-add box", ms,
             elems / ms / 1e6);
    }
  }
  // correctness: sum of g equals items * sum_c (1 + c) * 512 for both variants (x 3 reps each)
  std::vector<float> h(G * G);
  CK(cudaMemcpy(h.data(), g, sizeof(float) * G * G, cudaMemcpyDeviceToHost));
  double s = 0;
  for (float x : h) s += x;
  double want = 0;
  for (int c = 0; c < NM; ++c) want += (1.0 + c) * TR * TC;
  want *= (double)items * 6;
  printf("sum check: %.6e vs %.6e\n", s, want);
  return 0;
}
