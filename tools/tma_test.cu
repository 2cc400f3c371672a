// Standalone TMA sanity test: 3-D/4-D box loads through cp.async.bulk.tensor with an mbarrier.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>
#include <cstring>
#include <cstdlib>

__device__ __forceinline__ void mbar_init(unsigned bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned parity) {
  asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(bar), "r"(parity) : "memory");
}
template <int MODE>
__global__ void k(const __grid_constant__ CUtensorMap tm, const CUtensorMap* gtm, float* out, int c0, int c1, int c2, int c3, int nbytes) {
  extern __shared__ __align__(128) float smem[];
  __shared__ __align__(8) unsigned long long bar;
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  const unsigned b = (unsigned)__cvta_generic_to_shared(&bar);
  const CUtensorMap* p = MODE == 1 ? gtm : &tm;
  if (threadIdx.x == 0) {
    mbar_init(b, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (MODE == 4) {  // mbarrier only
    if (threadIdx.x == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(b) : "memory");
    mbar_wait(b, 0);
    if (threadIdx.x == 0) out[0] = 1.f;
    return;
  }
  if (MODE == 5) {  // non-tensor bulk copy
    if (threadIdx.x == 0) {
      mbar_expect_tx(b, 1024);
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   :: "r"(s), "l"(out + 4096), "r"(1024), "r"(b) : "memory");
    }
    mbar_wait(b, 0);
    for (int i = threadIdx.x; i < 256; i += blockDim.x) out[i] = smem[i];
    return;
  }
  if (threadIdx.x == 0) {
    mbar_expect_tx(b, nbytes);
    if (MODE == 2)
      asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
                   :: "r"(s), "l"(p), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(b) : "memory");
    else if (MODE == 3)
      asm volatile("cp.async.bulk.tensor.4d.shared::cta.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
                   :: "r"(s), "l"(p), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(b) : "memory");
    else
      asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
                   :: "r"(s), "l"(p), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(b) : "memory");
  }
  mbar_wait(b, 0);
  for (int i = threadIdx.x; i < nbytes / 4; i += blockDim.x) out[i] = smem[i];
}

int main(int argc, char** argv) {
  const int only = argc > 1 ? atoi(argv[1]) : -1;
  const int A = 64, AL = 48, W = 5, F = 2;
  std::vector<float> h((size_t)A * AL * W * F);
  for (size_t i = 0; i < h.size(); ++i) h[i] = (float)i;
  float* d; cudaMalloc(&d, h.size() * 4); cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  void* fnp = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fnp, cudaEnableDefault, &q);
  auto fn = (CUresult(*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill))fnp;
  alignas(64) CUtensorMap tm;
  const cuuint64_t dims[4] = {A, AL, W, F};
  const cuuint64_t strides[3] = {4ull * A, 4ull * A * AL, 4ull * A * AL * W};
  const int BR = getenv("BR") ? atoi(getenv("BR")) : 56, BC = getenv("BC") ? atoi(getenv("BC")) : 40;
  const cuuint32_t box[4] = {BR, BC, 1, 1}, es[4] = {1, 1, 1, 1};
  const int promo = getenv("PROMO") ? atoi(getenv("PROMO")) : 2;
  CUresult r = fn(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_NONE, (CUtensorMapL2promotion)promo, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d\n", (int)r);
  CUtensorMap* gtm; cudaMalloc(&gtm, sizeof(CUtensorMap));
  float* big; cudaMalloc(&big, 1 << 20); cudaMemcpy(gtm, &tm, sizeof(tm), cudaMemcpyHostToDevice);
  float* out = big;
  { int dev; cudaGetDevice(&dev); cudaDeviceProp pr; cudaGetDeviceProperties(&pr, dev); printf("cc %d.%d %s\n", pr.major, pr.minor, pr.name); }
  for (int mode = 0; mode < 6; ++mode) {
    if (only >= 0 && mode != only) continue;
    int c0 = getenv("C0") ? atoi(getenv("C0")) : -3, c1 = 5, c2 = 2, c3 = 1;
    if (mode == 0) k<0><<<1, 128, BR * BC * 4>>>(tm, gtm, out, c0, c1, c2, c3, BR * BC * 4);
    else if (mode == 1) k<1><<<1, 128, BR * BC * 4>>>(tm, gtm, out, c0, c1, c2, c3, BR * BC * 4);
    else if (mode == 2) k<2><<<1, 128, BR * BC * 4>>>(tm, gtm, out, c0, c1, c2, c3, BR * BC * 4);
    else if (mode == 3) k<3><<<1, 128, BR * BC * 4>>>(tm, gtm, out, c0, c1, c2, c3, BR * BC * 4);
    else if (mode == 4) k<4><<<1, 128, BR * BC * 4>>>(tm, gtm, out, c0, c1, c2, c3, BR * BC * 4);
    else k<5><<<1, 128, BR * BC * 4>>>(tm, gtm, out, c0, c1, c2, c3, BR * BC * 4);
    cudaError_t e = cudaDeviceSynchronize();
    printf("mode %d: %s\n", mode, cudaGetErrorString(e));
    if (e != cudaSuccess) return 1;
    if (mode >= 4) continue;
    std::vector<float> o(BR * BC);
    cudaMemcpy(o.data(), out, o.size() * 4, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int j = 0; j < BC; ++j) for (int i = 0; i < BR; ++i) {
      int rr = c0 + i, cc = c1 + j;
      float want = (rr >= 0 && rr < A && cc >= 0 && cc < AL) ? h[rr + (size_t)A * (cc + (size_t)AL * (c2 + (size_t)W * c3))] : 0.f;
      if (o[i + BR * j] != want) ++bad;
    }
    printf("mode %d mismatches %d\n", mode, bad);
  }
  return 0;
}
