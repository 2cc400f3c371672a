// microbench.cu — B200 (sm_100a) microbenchmarks that bound the CTIS hot path:
//   HBM stream, L2-resident read (coalesced and misaligned warp gathers), shared-memory LDS.32
//   operand delivery, FFMA issue rate, red.global.add(.v4).f32 into an L2-resident buffer.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/microbench tools/microbench.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cstring>
static unsigned __float_as_uint_host(float f) { unsigned u; memcpy(&u, &f, 4); return u; }

#define CK(x)                                                                  \
  do {                                                                         \
    cudaError_t e = (x);                                                       \
    if (e != cudaSuccess) {                                                    \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      exit(1);                                                                 \
    }                                                                          \
  } while (0)

__global__ void copy_kernel(const float4* __restrict__ a, float4* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) b[i] = a[i];
}

// L2-resident read: each warp reads 32 consecutive floats starting at a (possibly misaligned) offset.
__global__ void l2_gather_kernel(const float* __restrict__ a, int nfloats, int iters, int misalign, float* out) {
  const int lane = threadIdx.x & 31;
  unsigned warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  float acc = 0.f;
  unsigned x = warp * 2654435761u;
  for (int it = 0; it < iters; ++it) {
    x = x * 1664525u + 1013904223u;
    int base = (int)((x >> 4) % (unsigned)(nfloats - 64)) & ~31;
    base += misalign ? (int)(x & 31) : 0;
    acc += __ldg(a + base + lane);
  }
  if (acc == 123.f) out[0] = acc;
}

// SMEM operand delivery: LDS.32 with consecutive lanes, pseudo-random warp-uniform base.
__global__ void smem_kernel(int iters, float* out) {
  __shared__ float s[8192];
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) s[i] = (float)i;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
  int b = (threadIdx.x >> 5) * 37;
#pragma unroll 1
  for (int it = 0; it < iters; ++it) {
    b = (b + 97) & 4095;
    a0 = fmaf(1.0001f, s[b + lane], a0);
    a1 = fmaf(1.0001f, s[b + lane + 129], a1);
    a2 = fmaf(1.0001f, s[b + lane + 517], a2);
    a3 = fmaf(1.0001f, s[b + lane + 1031], a3);
  }
  if (a0 + a1 + a2 + a3 == 1.f) out[0] = a0;
}

// FFMA issue with a uniform (constant-bank style) operand and 8 independent chains.
__global__ void ffma_kernel(int iters, float w, float* out) {
  float a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x + i;
#pragma unroll 1
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 16; ++k)
#pragma unroll
      for (int i = 0; i < 8; ++i) a[i] = fmaf(w, a[i], 0.5f);
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 1.f) out[0] = s;
}

// red.global.add.f32: warp-contiguous (coalesced) reductions into an L2-resident buffer.
__global__ void red_kernel(float* buf, int nfloats, int iters) {
  const int lane = threadIdx.x & 31;
  unsigned warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  unsigned x = warp * 2654435761u;
  for (int it = 0; it < iters; ++it) {
    x = x * 1664525u + 1013904223u;
    int base = (int)((x >> 4) % (unsigned)(nfloats - 64)) & ~31;
    atomicAdd(buf + base + lane, 1.0f);
  }
}

__global__ void red_v4_kernel(float* buf, int nfloats, int iters) {
  const int lane = threadIdx.x & 31;
  unsigned warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  unsigned x = warp * 2654435761u;
  for (int it = 0; it < iters; ++it) {
    x = x * 1664525u + 1013904223u;
    int base = (int)((x >> 4) % (unsigned)(nfloats - 256)) & ~127;
    float* p = buf + base + 4 * lane;
    asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(1.f), "f"(1.f), "f"(1.f), "f"(1.f)
                 : "memory");
  }
}

__global__ void clock_kernel(long long* out, int spin) {
  long long t0 = clock64();
  unsigned long long g0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
  float x = threadIdx.x;
  for (int i = 0; i < spin; ++i) x = fmaf(x, 1.0001f, 0.5f);
  long long t1 = clock64();
  unsigned long long g1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    out[0] = t1 - t0;
    out[1] = (long long)(g1 - g0);
    out[2] = (long long)x;
  }
}


__constant__ uint2 c_taps[4096];
__device__ __forceinline__ float lds_u(unsigned a) { float v; asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a)); return v; }

// JIT-style tap loop: LDS [R + imm] and FFMA with an immediate weight.
__global__ void __launch_bounds__(512, 4) taps_imm_kernel(int iters, float* out) {
  extern __shared__ float s[];
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) s[i] = (float)i;
  __syncthreads();
  const unsigned sb = (unsigned)__cvta_generic_to_shared(s) + 4u * threadIdx.x;
  float a[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = 0.f;
#pragma unroll 1
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
#pragma unroll
      for (int i = 0; i < 16; ++i) a[i] = fmaf(0.37f + 0.01f * i + 0.1f * k, lds_u(sb + 4u * (37u * i + 301u * k)), a[i]);
    }
  }
  float t = 0.f;
#pragma unroll
  for (int i = 0; i < 16; ++i) t += a[i];
  if (t == 1.f) out[0] = t;
}

// Table-style tap loop: (offset, weight) from __constant__ via the uniform datapath.
__global__ void __launch_bounds__(512, 4) taps_ldcu_kernel(int iters, float* out) {
  extern __shared__ float s[];
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) s[i] = (float)i;
  __syncthreads();
  const unsigned sb = (unsigned)__cvta_generic_to_shared(s) + 4u * threadIdx.x;
  float a[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = 0.f;
#pragma unroll 1
  for (int it = 0; it < iters; ++it) {
    const uint2* e = c_taps + (it & 63) * 64;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const uint2 t = e[16 * k + i];
        a[i] = fmaf(__uint_as_float(t.y), lds_u(sb + t.x), a[i]);
      }
    }
  }
  float t = 0.f;
#pragma unroll
  for (int i = 0; i < 16; ++i) t += a[i];
  if (t == 1.f) out[0] = t;
}

// L2-resident streaming read with 8 independent float4 loads in flight per thread.
__global__ void l2_stream_kernel(const float4* __restrict__ a, int n4, int iters, float* out) {
  float acc = 0.f;
  const int stride = gridDim.x * blockDim.x;
  for (int it = 0; it < iters; ++it) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i + 7 * stride < n4; i += 8 * stride) {
      float4 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = __ldcg(a + i + u * stride);
#pragma unroll
      for (int u = 0; u < 8; ++u) acc += v[u].x + v[u].y + v[u].z + v[u].w;
    }
  }
  if (acc == 123.f) out[0] = acc;
}

template <typename F>
float time_ms(F&& f, int reps = 5) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  f();
  CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    cudaEventRecord(a);
    f();
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    best = ms < best ? ms : best;
  }
  return best;
}

int main() {
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, 0));
  const int sms = prop.multiProcessorCount;
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"l2_bytes\": %d, \"smem_per_sm\": %zu\n", prop.name, sms, prop.l2CacheSize,
         prop.sharedMemPerMultiprocessor);
  // clock
  long long* dclk;
  CK(cudaMalloc(&dclk, 64));
  clock_kernel<<<sms, 128>>>(dclk, 1 << 22);
  CK(cudaDeviceSynchronize());
  long long hclk[3];
  CK(cudaMemcpy(hclk, dclk, 24, cudaMemcpyDeviceToHost));
  const double mhz = (double)hclk[0] / (double)hclk[1] * 1e3;
  printf(", \"sm_clock_mhz_under_ffma\": %.0f\n", mhz);

  // HBM copy
  const size_t nbig = (size_t)1 << 28;  // 1 GiB floats? 2^28 floats = 1 GiB
  float *A, *B;
  CK(cudaMalloc(&A, nbig * 4));
  CK(cudaMalloc(&B, nbig * 4));
  CK(cudaMemset(A, 0, nbig * 4));
  float ms = time_ms([&] { copy_kernel<<<sms * 8, 256>>>((const float4*)A, (float4*)B, nbig / 4); });
  printf(", \"hbm_copy_gbs\": %.1f\n", 2.0 * nbig * 4 / ms / 1e6);

  // L2-resident gathers (32 MB buffer)
  const int nl2 = 8 << 20;
  float* out;
  CK(cudaMalloc(&out, 64));
  const int iters = 2048;
  for (int mis = 0; mis < 2; ++mis) {
    const int blocks = sms * 8, threads = 256;
    ms = time_ms([&] { l2_gather_kernel<<<blocks, threads>>>(A, nl2, iters, mis, out); });
    const double bytes = (double)blocks * threads * iters * 4;
    printf(", \"l2_gather_%s_gbs\": %.1f\n", mis ? "misaligned" : "aligned", bytes / ms / 1e6);
  }
  // SMEM
  {
    const int blocks = sms * 4, threads = 512, it = 1 << 14;
    ms = time_ms([&] { smem_kernel<<<blocks, threads>>>(it, out); });
    const double words = (double)blocks * threads * it * 4;
    printf(", \"smem_lds32_words_per_clk_per_sm\": %.2f, \"smem_gbs\": %.1f\n", words / (ms * 1e-3) / sms / (mhz * 1e6),
           words * 4 / ms / 1e6);
  }
  // FFMA
  {
    const int blocks = sms * 4, threads = 512, it = 1 << 12;
    ms = time_ms([&] { ffma_kernel<<<blocks, threads>>>(it, 0.999f, out); });
    const double fmas = (double)blocks * threads * it * 16 * 8;
    printf(", \"ffma_per_clk_per_sm\": %.1f, \"fp32_tflops\": %.1f\n", fmas / (ms * 1e-3) / sms / (mhz * 1e6),
           2 * fmas / ms / 1e9);
  }

  // tap loops (operand delivery with and without table metadata)
  {
    std::vector<uint2> h(4096);
    for (int i = 0; i < 4096; ++i) h[i] = make_uint2(4u * ((i * 37u) % 4096u), __float_as_uint_host(0.5f));
    CK(cudaMemcpyToSymbol(c_taps, h.data(), sizeof(uint2) * 4096));
    const int blocks = sms * 2, threads = 512, it = 1 << 12;
    CK(cudaFuncSetAttribute(taps_imm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 48 * 1024));
    ms = time_ms([&] { taps_imm_kernel<<<blocks, threads, 40 * 1024>>>(it, out); });
    double fmas = (double)blocks * threads * it * 64;
    printf(", \"taps_imm_fma_per_clk_per_sm\": %.2f\n", fmas / (ms * 1e-3) / sms / (mhz * 1e6));
    ms = time_ms([&] { taps_ldcu_kernel<<<blocks, threads, 40 * 1024>>>(it, out); });
    printf(", \"taps_ldcu_fma_per_clk_per_sm\": %.2f\n", fmas / (ms * 1e-3) / sms / (mhz * 1e6));
    // occupancy sweep: 1..4 CTAs of 512 threads per SM (smaller shared allocation)
    for (int occ = 1; occ <= 4; ++occ) {
      const int b2 = sms * occ;
      const double f2 = (double)b2 * threads * it * 64;
      ms = time_ms([&] { taps_imm_kernel<<<b2, threads, 33 * 1024>>>(it, out); });
      printf(", \"taps_imm_occ%d\": %.2f\n", occ, f2 / (ms * 1e-3) / sms / (mhz * 1e6));
      ms = time_ms([&] { taps_ldcu_kernel<<<b2, threads, 33 * 1024>>>(it, out); });
      printf(", \"taps_ldcu_occ%d\": %.2f\n", occ, f2 / (ms * 1e-3) / sms / (mhz * 1e6));
    }
  }
  // L2 streaming read (64 MB buffer, resident)
  {
    const int n4 = (64 << 20) / 16;
    ms = time_ms([&] { l2_stream_kernel<<<sms * 4, 512>>>((const float4*)A, n4, 8, out); });
    printf(", \"l2_stream_read_gbs\": %.1f\n", 8.0 * n4 * 16 / ms / 1e6);
  }
  // reductions into a 16 MB L2-resident buffer
  {
    const int nred = 4 << 20;
    CK(cudaMemset(B, 0, nred * 4));
    const int blocks = sms * 8, threads = 256, it = 256;
    ms = time_ms([&] { red_kernel<<<blocks, threads>>>(B, nred, it); });
    const double elems = (double)blocks * threads * it;
    printf(", \"red_f32_coalesced_gelem_s\": %.1f\n", elems / ms / 1e6);
    ms = time_ms([&] { red_v4_kernel<<<blocks, threads>>>(B, nred, it); });
    printf(", \"red_v4_f32_coalesced_gelem_s\": %.1f}\n", 4 * elems / ms / 1e6);
  }
  return 0;
}
