// ctis_nvls.cu — SURVEY.md §8(f) f-1: the latency mode's exchange and ratio fused into ONE kernel over
// NVLink peer memory (Eq. 3: g_hat is the sum of the per-band-shard partials; Alg. 1
// line 8: r = g (/) g_hat).
//
// Every rank's exchange buffer X is one NCCL symmetric-memory window (ncclMemAlloc +
// ncclCommWindowRegister): after the partial forward projections, rank k owns the pixel slice
// [base + k*S, base + (k+1)*S) of the exchange range and, per pixel of its slice,
//   NVLS (multimem, NVSwitch in-fabric reduction):   v = multimem.ld_reduce.add(X_*[i]);
//                                                    multimem.st(X_*[i], g_i / v)
//   LSA (plain NVLink peer loads / stores):           v = sum_j X_j[i];  X_j[i] = g_i / v  for every j
// so that every rank holds r on the whole range when the kernel ends — the reduce-scatter, the ratio
// pass and the all-gather of the NCCL schedule in one launch, with no intermediate HBM round trip.
// Per-CTA LSA barriers (NCCL device API) order the partial sums before the reads and the r stores
// before every rank's back projection.  The summation order over ranks is fixed (j = 0 .. P-1 for LSA;
// the switch's order for NVLS).
#include <cuda_runtime.h>
#include <nccl.h>
#include <nccl_device.h>

#include "ctis_nvls.h"

namespace ctis {

__device__ __forceinline__ float nv_ratio(float g, float h) { return h > 0.f ? __fdiv_rn(g, h) : 0.f; }

__global__ void __launch_bounds__(256) exchange_ratio_kernel(ncclDevComm dc, ncclWindow_t win, long long base,
                                                             long long slice, const float* __restrict__ g,
                                                             long long n, int multimem) {
  ncclLsaBarrierSession<ncclCoopCta> bar(ncclCoopCta(), dc, ncclTeamTagLsa(), blockIdx.x, multimem != 0);
  // every rank's partial forward projection (the kernels before this one on each rank) is complete
  bar.sync(ncclCoopCta(), cuda::memory_order_acq_rel);
  const int P = dc.lsaSize, me = dc.lsaRank;
  const long long s0 = base + (long long)me * slice;                    // first pixel of my slice
  const long long cnt = s0 >= n ? 0 : (s0 + slice <= n ? slice : n - s0);  // pixels with a measurement
  const long long stride = (long long)gridDim.x * blockDim.x;
  const long long t0 = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const size_t off = sizeof(float) * (size_t)s0;                        // byte offset of the slice in X
  if (multimem) {
    float* mc = static_cast<float*>(ncclGetLsaMultimemPointer(win, off, dc));
    const long long n4 = cnt >> 2;  // s0 is a multiple of 4: 16-byte vectors
    for (long long i = t0; i < n4; i += stride) {
      float4 v;
      asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0, %1, %2, %3}, [%4];"
                   : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                   : "l"(mc + 4 * i)
                   : "memory");
      const float4 gv = __ldg(reinterpret_cast<const float4*>(g + s0) + i);
      asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(mc + 4 * i),
                   "f"(nv_ratio(gv.x, v.x)), "f"(nv_ratio(gv.y, v.y)), "f"(nv_ratio(gv.z, v.z)),
                   "f"(nv_ratio(gv.w, v.w))
                   : "memory");
    }
    for (long long i = 4 * n4 + t0; i < cnt; i += stride) {
      float v;
      asm volatile("multimem.ld_reduce.relaxed.sys.global.add.f32 %0, [%1];" : "=f"(v) : "l"(mc + i) : "memory");
      asm volatile("multimem.st.relaxed.sys.global.f32 [%0], %1;" ::"l"(mc + i), "f"(nv_ratio(__ldg(g + s0 + i), v))
                   : "memory");
    }
  } else {
    for (long long i = t0; i < cnt; i += stride) {
      float v = 0.f;
      for (int j = 0; j < P; ++j) v += static_cast<const volatile float*>(ncclGetLsaPointer(win, off, j))[i];
      const float r = nv_ratio(__ldg(g + s0 + i), v);
      for (int j = 0; j < P; ++j) static_cast<volatile float*>(ncclGetLsaPointer(win, off, j))[i] = r;
    }
  }
  // every rank's r stores have landed before any rank's back projection reads its X
  bar.sync(ncclCoopCta(), cuda::memory_order_acq_rel);
}

cudaError_t launch_exchange_ratio(const NvlsComm& c, long long base, long long slice, const float* g, long long n,
                                  cudaStream_t s) {
  const ncclDevComm* dc = static_cast<const ncclDevComm*>(c.devcomm);
  exchange_ratio_kernel<<<c.blocks, 256, 0, s>>>(*dc, static_cast<ncclWindow_t>(c.window), base, slice, g, n,
                                                  c.multimem);
  return cudaGetLastError();
}

size_t devcomm_bytes() { return sizeof(ncclDevComm); }

void devcomm_requirements(void* reqs, int barriers, bool multimem) {
  ncclDevCommRequirements* r = static_cast<ncclDevCommRequirements*>(reqs);
  *r = ncclDevCommRequirements{};
  r->lsaBarrierCount = barriers;
  r->lsaMultimem = multimem;
}
size_t devcomm_requirements_bytes() { return sizeof(ncclDevCommRequirements); }
int devcomm_lsa_size(const void* devcomm) { return static_cast<const ncclDevComm*>(devcomm)->lsaSize; }
bool devcomm_has_multimem(const void* devcomm) {
  const ncclDevComm* d = static_cast<const ncclDevComm*>(devcomm);
  return d->lsaMultimem.mcBasePtr != nullptr;
}

}  // namespace ctis
