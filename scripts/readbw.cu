// readbw.cu — read-only HBM bandwidth ceiling on this B200 (context for the roofline):
// (a) plain 16-byte vector loads, grid-stride, several loads in flight per thread;
// (b) the same TMA bulk ring as k_rows_tma with trivial consumers (XOR of one word).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o readbw readbw.cu && ./readbw
#include <cstdio>
#include <type_traits>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(512) k_ldg(const uint4* __restrict__ p, size_t n, unsigned* out) {
  unsigned acc = 0;
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (; i + 7 * stride < n; i += 8 * stride) {
    uint4 v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = __ldg(p + i + j * stride);
#pragma unroll
    for (int j = 0; j < 8; ++j) acc ^= v[j].x ^ v[j].y ^ v[j].z ^ v[j].w;
  }
  for (; i < n; i += stride) { uint4 v = __ldg(p + i); acc ^= v.x ^ v.w; }
  if (acc == 0x12345678u) out[0] = acc;
}

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int NS, int CH>
__global__ void __launch_bounds__(544, 1) k_tma(const char* __restrict__ p, size_t bytes, unsigned* out) {
  extern __shared__ __align__(128) uint8_t sm[];
  uint64_t* full = (uint64_t*)sm;
  uint64_t* empty = full + NS;
  uint8_t* buf = sm + 1024;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < NS; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(full + s)));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 16;" ::"r"(sa(empty + s)));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const size_t nch = bytes / CH;
  if (warp == 16) {
    if (lane == 0) {
      int st = 0; uint32_t ph = 0;
      for (size_t c = blockIdx.x; c < nch; c += gridDim.x) {
        asm volatile("{.reg .pred q; W%=: mbarrier.try_wait.parity.shared::cta.b64 q, [%0], %1; @!q bra W%=;}" ::"r"(sa(empty + st)), "r"(ph ^ 1));
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(full + st)), "r"(CH));
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sa(buf + st * CH)), "l"(p + c * CH), "r"(CH), "r"(sa(full + st)) : "memory");
        if (++st == NS) { st = 0; ph ^= 1; }
      }
    }
    return;
  }
  unsigned acc = 0;
  int st = 0; uint32_t ph = 0;
  for (size_t c = blockIdx.x; c < nch; c += gridDim.x) {
    asm volatile("{.reg .pred q; W%=: mbarrier.try_wait.parity.shared::cta.b64 q, [%0], %1; @!q bra W%=;}" ::"r"(sa(full + st)), "r"(ph) : "memory");
    acc ^= *(volatile unsigned*)(buf + st * CH + tid * 16);
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(empty + st)) : "memory");
    if (++st == NS) { st = 0; ph ^= 1; }
  }
  if (acc == 0x12345678u) out[0] = acc;
}

int main() {
  const size_t bytes = (size_t)32 << 30;
  char* p;
  unsigned* out;
  cudaMalloc(&p, bytes);
  cudaMalloc(&out, 4);
  cudaMemset(p, 1, bytes);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float ms;
  for (int blocks_per_sm : {2, 4, 8}) {
    for (int it = 0; it < 2; ++it) {
      cudaEventRecord(a);
      k_ldg<<<sms * blocks_per_sm, 512>>>((const uint4*)p, bytes / 16, out);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
    }
    printf("ldg  %d CTA/SM x 512 thr, 8x16B in flight/thread: %.1f GB/s\n", blocks_per_sm, bytes / (ms * 1e-3) / 1e9);
  }
  auto run_tma = [&](auto ns_tag, auto ch_tag, size_t nbytes, int reps) {
    constexpr int NS_ = decltype(ns_tag)::value, CH_ = decltype(ch_tag)::value;
    const int smem = 1024 + NS_ * CH_;
    cudaFuncSetAttribute(k_tma<NS_, CH_>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    float best = 1e30f;
    for (int it = 0; it < reps; ++it) {
      cudaEventRecord(a);
      k_tma<NS_, CH_><<<sms, 544, smem>>>(p + (size_t)(it % 8) * (1ull << 30), nbytes, out);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
      best = ms < best ? ms : best;
    }
    printf("tma  bulk ring %2d x %2d KB (%3d KB in flight/SM), %7.1f MB: %7.1f GB/s  %8.2f us (%s)\n", NS_, CH_ / 1024,
           NS_ * CH_ / 1024, nbytes / 1e6, nbytes / (best * 1e-3) / 1e9, best * 1e3, cudaGetErrorString(cudaGetLastError()));
  };
  using std::integral_constant;
  for (size_t nb : {(size_t)4 << 30, (size_t)33554432, (size_t)8388608}) {
    const int reps = nb > (1u << 30) ? 3 : 20;
    run_tma(integral_constant<int, 2>{}, integral_constant<int, 16384>{}, nb, reps);
    run_tma(integral_constant<int, 6>{}, integral_constant<int, 16384>{}, nb, reps);
    run_tma(integral_constant<int, 12>{}, integral_constant<int, 16384>{}, nb, reps);
    run_tma(integral_constant<int, 3>{}, integral_constant<int, 32768>{}, nb, reps);
    run_tma(integral_constant<int, 6>{}, integral_constant<int, 32768>{}, nb, reps);
    run_tma(integral_constant<int, 24>{}, integral_constant<int, 8192>{}, nb, reps);
  }
  return 0;
}
