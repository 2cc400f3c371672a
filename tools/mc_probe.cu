// mc_probe.cu — can this box run the f-1 exchange (NVLS multicast: multimem.ld_reduce / multimem.st)?
// Creates a multicast object over the visible GPUs (1 in a gpurun call), binds one physical buffer per
// GPU, maps the multicast address and runs multimem.ld_reduce.add.f32 + multimem.st.f32 on it.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

#define DR(x)                                                                    \
  do {                                                                           \
    CUresult r_ = (x);                                                           \
    if (r_ != CUDA_SUCCESS) {                                                    \
      const char* s_ = nullptr;                                                  \
      cuGetErrorString(r_, &s_);                                                 \
      printf("{\"step\": \"%s\", \"error\": \"%s\"}\n", #x, s_ ? s_ : "?");      \
      return 1;                                                                  \
    }                                                                            \
  } while (0)

__global__ void mc_kernel(float* mc, const float* g, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    float v;
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.f32 %0, [%1];" : "=f"(v) : "l"(mc + i) : "memory");
    const float r = v > 0.f ? __fdiv_rn(g[i], v) : 0.f;
    asm volatile("multimem.st.relaxed.sys.global.f32 [%0], %1;" ::"l"(mc + i), "f"(r) : "memory");
  }
}

int main() {
  DR(cuInit(0));
  CUdevice dev;
  DR(cuDeviceGet(&dev, 0));
  int mcs = 0, ndev = 0;
  DR(cuDeviceGetAttribute(&mcs, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev));
  cudaGetDeviceCount(&ndev);
  printf("{\"multicast_supported\": %d, \"devices\": %d}\n", mcs, ndev);
  if (!mcs) return 0;
  CUcontext ctx;
  DR(cuDevicePrimaryCtxRetain(&ctx, dev));
  DR(cuCtxSetCurrent(ctx));
  const int n = 1 << 20;
  const size_t bytes = n * sizeof(float);
  CUmulticastObjectProp mp = {};
  mp.numDevices = 1;
  mp.size = bytes;
  size_t gran = 0;
  CUmemGenericAllocationHandle mch;
  CUresult cr = CUDA_ERROR_UNKNOWN;
  for (unsigned long long ht : {0ull, (unsigned long long)CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR,
                                (unsigned long long)CU_MEM_HANDLE_TYPE_FABRIC}) {
    mp.handleTypes = ht;
    mp.size = bytes;
    if (cuMulticastGetGranularity(&gran, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED) != CUDA_SUCCESS) continue;
    mp.size = (bytes + gran - 1) / gran * gran;
    cr = cuMulticastCreate(&mch, &mp);
    const char* es = nullptr;
    cuGetErrorString(cr, &es);
    printf("{\"handleTypes\": %llu, \"gran\": %zu, \"create\": \"%s\"}\n", ht, gran, es ? es : "?");
    if (cr == CUDA_SUCCESS) break;
  }
  DR(cr);
  DR(cuMulticastAddDevice(mch, dev));
  CUmemAllocationProp ap = {};
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = 0;
  ap.requestedHandleTypes = (CUmemAllocationHandleType)mp.handleTypes;
  size_t ugran = 0;
  DR(cuMemGetAllocationGranularity(&ugran, &ap, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
  const size_t asz = (mp.size + ugran - 1) / ugran * ugran;
  CUmemGenericAllocationHandle ph;
  DR(cuMemCreate(&ph, asz, &ap, 0));
  DR(cuMulticastBindMem(mch, 0, ph, 0, mp.size, 0));
  CUdeviceptr uc = 0, mc = 0;
  DR(cuMemAddressReserve(&uc, asz, 0, 0, 0));
  DR(cuMemMap(uc, asz, 0, ph, 0));
  DR(cuMemAddressReserve(&mc, mp.size, 0, 0, 0));
  DR(cuMemMap(mc, mp.size, 0, mch, 0));
  CUmemAccessDesc ad = {};
  ad.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ad.location.id = 0;
  ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  DR(cuMemSetAccess(uc, asz, &ad, 1));
  DR(cuMemSetAccess(mc, mp.size, &ad, 1));
  std::vector<float> h(n), gh(n);
  for (int i = 0; i < n; ++i) {
    h[i] = 1.0f + (i % 7);
    gh[i] = 2.0f * (i % 5);
  }
  float* g;
  cudaMalloc(&g, bytes);
  cudaMemcpy(g, gh.data(), bytes, cudaMemcpyHostToDevice);
  cudaMemcpy((void*)uc, h.data(), bytes, cudaMemcpyHostToDevice);
  mc_kernel<<<148 * 4, 256>>>((float*)mc, g, n);
  cudaError_t e = cudaDeviceSynchronize();
  std::vector<float> out(n);
  cudaMemcpy(out.data(), (void*)uc, bytes, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int i = 0; i < n; ++i)
    if (out[i] != gh[i] / h[i]) ++bad;
  printf("{\"kernel\": \"%s\", \"mismatches\": %d, \"granularity\": %zu}\n", cudaGetErrorString(e), bad, gran);
  return 0;
}
