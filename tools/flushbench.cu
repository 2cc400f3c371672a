// flushbench.cu — cost of the forward kernel's accumulator flush with scalar versus vector L2 reductions.
// Each CTA "item" flushes NM modes x (32 x 16) floats (two positions per thread: columns warp, warp + 8)
// to box origins scattered over a 2048 x 2048 fp32 image (L2-resident, as g_hat is inside the MLEM
// graph).  Variants:
//   scalar  red.global.add.f32 per value (the round-1 flush)
//   v2      lanes pair up (shfl.xor 1): red.global.add.v2.f32 of 2 consecutive rows, 2 modes per pair
//   v4      4x4 transpose inside lane quads (shfl.xor 1, 2): red.global.add.v4.f32 of 4 consecutive rows
// Box row origins are multiples of 4 (16-byte aligned vectors).  Reports elements/s and checks the sum.
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

#define CK(x)                                                                           \
  do {                                                                                  \
    cudaError_t e_ = (x);                                                               \
    if (e_ != cudaSuccess) {                                                            \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__);   \
      return 1;                                                                         \
    }                                                                                   \
  } while (0)

constexpr int G = 2048, TR = 32, TC = 16, NM = 24;

__device__ __forceinline__ unsigned hash(unsigned x) {
  x ^= x >> 16;
  x *= 0x7feb352dU;
  x ^= x >> 15;
  x *= 0x846ca68bU;
  x ^= x >> 16;
  return x;
}

__device__ __forceinline__ long long origin(int it, int c) {
  const unsigned h = hash(it * 131u + c * 7919u);
  const int r0 = (h % (G - TR)) & ~3;
  const int c0 = (h / 4096u) % (G - TC);
  return r0 + (long long)G * c0;
}

__device__ __forceinline__ void red1(float* p, float v) {
  asm volatile("red.global.add.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
}
__device__ __forceinline__ void red2(float* p, float a, float b) {
  asm volatile("red.global.add.v2.f32 [%0], {%1, %2};" ::"l"(p), "f"(a), "f"(b) : "memory");
}
__device__ __forceinline__ void red4(float* p, float a, float b, float c, float d) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(a), "f"(b), "f"(c), "f"(d) : "memory");
}

template <int V>
__global__ void __launch_bounds__(256, 2) flush_kernel(float* g, int items, float salt) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int it = blockIdx.x; it < items; it += gridDim.x) {
    float a0[NM], a1[NM];
#pragma unroll
    for (int c = 0; c < NM; ++c) {
      a0[c] = 1.0f + c + salt * lane;
      a1[c] = 1.0f + c + salt * warp;
    }
    const long long e0 = lane + (long long)G * warp, e1 = e0 + 8LL * G;
    if (V == 1) {
#pragma unroll
      for (int c = 0; c < NM; ++c) {
        const long long o = origin(it, c);
        red1(g + o + e0, a0[c]);
        red1(g + o + e1, a1[c]);
      }
    } else if (V == 2) {
      // pair (lane even, lane odd) = rows 2k, 2k+1; modes (c, c+1): even lane takes mode c of both rows,
      // odd lane mode c + 1
      const int odd = lane & 1;
#pragma unroll
      for (int c = 0; c < NM; c += 2) {
#pragma unroll
        for (int pos = 0; pos < 2; ++pos) {
          const float* a = pos ? a1 : a0;
          const float send = odd ? a[c] : a[c + 1];
          const float recv = __shfl_xor_sync(0xffffffffu, send, 1);
          const float lo = odd ? recv : a[c];       // row 2k of my mode
          const float hi = odd ? a[c + 1] : recv;   // row 2k + 1 of my mode
          const int cm = c + odd;
          const long long o = origin(it, cm);
          red2(g + o + (pos ? e1 : e0) - odd, lo, hi);
        }
      }
    } else {
      // quad q = lane / 4, r = lane % 4: lane r of the quad ends with mode c + r at rows 4q .. 4q + 3
      const int r = lane & 3;
#pragma unroll
      for (int c = 0; c < NM; c += 4) {
#pragma unroll
        for (int pos = 0; pos < 2; ++pos) {
          const float* a = pos ? a1 : a0;
          // v[k] = value of mode c + k at my row; want w[k] = value of mode c + r at row 4q + k
          float v0 = a[c], v1 = a[c + 1], v2 = a[c + 2], v3 = a[c + 3];
          // step 1 (xor 1): exchange within pairs
          {
            const bool b = r & 1;
            float s0 = b ? v0 : v1, s1 = b ? v2 : v3;
            s0 = __shfl_xor_sync(0xffffffffu, s0, 1);
            s1 = __shfl_xor_sync(0xffffffffu, s1, 1);
            if (b) { v0 = s0; v2 = s1; } else { v1 = s0; v3 = s1; }
          }
          // step 2 (xor 2)
          {
            const bool b = r & 2;
            float s0 = b ? v0 : v2, s1 = b ? v1 : v3;
            s0 = __shfl_xor_sync(0xffffffffu, s0, 2);
            s1 = __shfl_xor_sync(0xffffffffu, s1, 2);
            if (b) { v0 = s0; v1 = s1; } else { v2 = s0; v3 = s1; }
          }
          const long long o = origin(it, c + r);
          red4(g + o + (pos ? e1 : e0) - r, v0, v1, v2, v3);
        }
      }
    }
  }
}

int main() {
  float* g;
  CK(cudaMalloc(&g, sizeof(float) * G * G));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int items = 296 * 40;
  std::vector<float> h(G * G);
  for (int v : {1, 2, 4}) {
    CK(cudaMemset(g, 0, sizeof(float) * G * G));
    float best = 1e9;
    for (int rep = 0; rep < 4; ++rep) {
      cudaEventRecord(a);
      if (v == 1) flush_kernel<1><<<296, 256>>>(g, items, 0.0f);
      if (v == 2) flush_kernel<2><<<296, 256>>>(g, items, 0.0f);
      if (v == 4) flush_kernel<4><<<296, 256>>>(g, items, 0.0f);
      cudaEventRecord(b);
      CK(cudaEventSynchronize(b));
      CK(cudaGetLastError());
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (rep > 0 && ms < best) best = ms;
    }
    const double elems = (double)items * NM * TR * TC;
    CK(cudaMemcpy(h.data(), g, sizeof(float) * G * G, cudaMemcpyDeviceToHost));
    double s = 0;
    for (float x : h) s += x;
    double want = 0;
    for (int c = 0; c < NM; ++c) want += (1.0 + c) * TR * TC;
    want *= (double)items * 4;
    printf("{\"variant\": \"v%d\", \"ms\": %.4f, \"Gelem_s\": %.1f, \"sum\": %.6e, \"want\": %.6e}\n", v, best,
           elems / best / 1e6, s, want);
  }
  return 0;
}
