// sb_hrad.cu — sb_hrad_predict: H-RAD length predictor inference.
//
//   h1 = relu(W1 z + b1)     z [B][Dz] bf16, W1 [256][Dz] bf16      (Eq. 4-5 P190-191,
//   h2 = relu(W2 h1 + b2)    W2 [64][256] fp32                       architecture P745:
//   l  = W3 h2 + b3          W3 [3][64]  fp32                        256-64-3, ReLU)
//   s_t = argmax l (ties -> smaller class), then H_t (P194-201, P669; DESIGN reading 35):
//   (gamma_b, s_b) = (0,0) | (stop_b, stop_b) | (G,G) for s_t = 0 | 1 | 2.
//
// Layer 1 is the only dense contraction (2*B*Dz*256 flops over B*Dz + 256*Dz bf16
// inputs).  k_hrad: grid = 128-row tiles of z x S K-splits, S chosen so the grid fills
// the SMs (one CTA per SM):
//   warp 0    TMA producer : per k-block (64 columns = one 128-byte swizzle atom) the two
//                            128-row z tiles and the W1 tile into a 3-stage ring of
//                            2 x 16 + 32 KB (SWIZZLE_128B tensor maps);
//   warp 1    MMA issuer   : allocates 512 TMEM columns; one elected thread issues
//                            tcgen05.mma.kind::f16 (M=128, N=256, K=16, fp32 accumulate
//                            in TMEM; one accumulator per row tile, both fed by the same
//                            W1 slot: half the W1 bytes per flop); tcgen05.commit frees
//                            each stage;
//   warps 2-5 epilogue     : tcgen05.ld of each 128 x 256 fp32 partial, staged through
//                            shared memory and stored coalesced to partial[s] (L2-sized).
// k_hrad_tail (programmatic dependent launch): sums the S partials of a row in split
// order (deterministic), + b1, ReLU, layers 2-3 (each thread holds a 32-column slice of
// one W2 row in registers), argmax, H_t.
#include <cuda.h>

#include <algorithm>
#include <cstdlib>

#include "sb_host.h"
#include "sb_ring.cuh"

namespace sb {

constexpr int kHM = 128;     // rows of z per UMMA tile (M)
constexpr int kTP = 2;       // row tiles per CTA: each W1 k-block feeds two MMAs (two
                             // TMEM accumulators, 512 columns) -> half the W1 bytes per flop
constexpr int kHN = 256;     // hidden-1 width (UMMA N)
constexpr int kHK = 64;      // k-block: 64 bf16 = 128 bytes = one swizzle atom row
constexpr int kHS = 3;       // ring stages
constexpr int kH2 = 64;      // hidden-2 width
constexpr int kCls = 3;      // classes
constexpr int kHThreads = 192;
constexpr int kAccStride = 260;  // floats per staged partial row (16-byte rows, spread banks)
constexpr uint32_t kStageA = kHM * kHK * 2;  // 16 KB per row tile
constexpr uint32_t kStageB = kHN * kHK * 2;  // 32 KB
constexpr uint32_t kStage = kTP * kStageA + kStageB;
constexpr uint32_t kRingBytes = kHS * kStage;
constexpr uint32_t kAccBytes = kHM * kAccStride * 4;
constexpr size_t kHradSmem = kRingBytes + 1024;  // + alignment slack (SWIZZLE_128B: 1 KB)
static_assert(kAccBytes <= kRingBytes, "the staged partial reuses the ring");
constexpr int kTailRowsMax = 16;  // rows per k_hrad_tail CTA (<=)
constexpr int kTailThreads = 512;  // two split-sums and two layer-2 outputs per thread at 16 rows

// Instruction descriptor of tcgen05.mma.kind::f16: fp32 accumulator (bits 4-5 = 1),
// A and B bf16 (bits 7-9, 10-12 = 1), both K-major (bits 15, 16 = 0), N>>3 at 17-22,
// M>>4 at 24-28.
constexpr uint32_t kIdesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(kHN >> 3) << 17) |
                            ((uint32_t)(kHM >> 4) << 24);

struct HradParams {
  int B, Dz, G, nkb, S, tail_rows;
  float* partial;  // [S][B][256]
  const float *b1, *w2, *b2, *w3, *b3;
  const int* stop;
  float* logits;
  int *s_t, *gamma, *bpos;
};

// Shared-memory matrix descriptor, K-major SWIZZLE_128B canonical layout: rows of 128 B,
// 8-row groups 1024 B apart (SBO), LBO unused (1), version 1 (sm_100), layout 2.
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr) {
  return (uint64_t)((saddr & 0x3FFFFu) >> 4) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}

__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int x, int y,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::
          "r"(dst),
      "l"(map), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(kIdesc), "r"(accumulate));
}


__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// 32 consecutive fp32 accumulator columns of this warp's 32 TMEM lanes.
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float* v) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
        "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
        "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
        "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
}

// Layer 1 partial of one (256-row block, K split): grid (S, ceil(B / 256)).
__global__ void __launch_bounds__(kHThreads, 1)
    k_hrad(const __grid_constant__ CUtensorMap tmZ, const __grid_constant__ CUtensorMap tmW1, HradParams p) {
  extern __shared__ uint8_t hsm_raw[];
  __shared__ __align__(8) uint64_t full[kHS], empty[kHS], done;
  __shared__ uint32_t tmem_slot;
  // SWIZZLE_128B tiles need 1024-byte aligned shared addresses
  const uint32_t raw = smem_u32(hsm_raw);
  uint8_t* sm = hsm_raw + ((1024u - (raw & 1023u)) & 1023u);
  const uint32_t sbase = smem_u32(sm);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int split = blockIdx.x, S = gridDim.x;
  const int m0 = blockIdx.y * (kTP * kHM);
  const int kb0 = (int)((int64_t)p.nkb * split / S), kb1 = (int)((int64_t)p.nkb * (split + 1) / S);

  if (tid == 0) {
    for (int s = 0; s < kHS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(&done, 1);
    fence_mbar_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_slot)),
                 "r"(kTP * kHN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;

  if (warp == 0) {  // ------------------------------------------------ TMA producer
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(&tmZ) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(&tmW1) : "memory");
      int stage = 0;
      uint32_t phase = 0;
      for (int kb = kb0; kb < kb1; ++kb) {
        mbar_wait(&empty[stage], phase ^ 1u);
        mbar_expect_tx(&full[stage], kStage);
        const uint32_t a = sbase + stage * kStage;
#pragma unroll
        for (int t = 0; t < kTP; ++t) tma_load_2d(a + t * kStageA, &tmZ, kb * kHK, m0 + t * kHM, &full[stage]);
        const uint32_t bb = a + kTP * kStageA;
        tma_load_2d(bb, &tmW1, kb * kHK, 0, &full[stage]);
        if (++stage == kHS) { stage = 0; phase ^= 1u; }
      }
    }
  } else if (warp == 1) {  // --------------------------------------------- MMA issuer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int kb = kb0; kb < kb1; ++kb) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        const uint32_t a = sbase + stage * kStage, bb = a + kTP * kStageA;
#pragma unroll
        for (int k = 0; k < kHK / 16; ++k)  // K = 16 per MMA: +32 bytes inside the swizzle atom
#pragma unroll
          for (int t = 0; t < kTP; ++t)
            umma_bf16(tmem + t * kHN, umma_desc_sw128(a + t * kStageA + k * 32), umma_desc_sw128(bb + k * 32),
                      (kb > kb0 || k > 0) ? 1u : 0u);
        umma_commit(&empty[stage]);
        if (++stage == kHS) { stage = 0; phase ^= 1u; }
      }
      umma_commit(&done);  // all MMAs of this CTA complete -> accumulator final
    }
  }
  // ---- epilogue: per row tile, TMEM -> shared (warps 2-5) -> coalesced global store
  const int wl = (warp & 3) * 32;  // TMEM lanes warp w may access: 32 * (w % 4) ...
  if (warp >= 2) {
    mbar_wait(&done, 0);
    tc_fence_after();
  }
  for (int t = 0; t < kTP; ++t) {
    if (warp >= 2) {
      float* acc = reinterpret_cast<float*>(sm) + (wl + lane) * kAccStride;
      for (int c = 0; c < kHN; c += 32) {
        float v[32];
        if (kb1 > kb0) {
          tmem_ld32(tmem + ((uint32_t)wl << 16) + (uint32_t)(t * kHN + c), v);
        } else {
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = 0.f;
        }
#pragma unroll
        for (int j = 0; j < 32; j += 4)
          *reinterpret_cast<float4*>(acc + c + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
      }
    }
    __syncthreads();
    const int mt = m0 + t * kHM;  // rows past B are dropped
    float* dst = p.partial + ((int64_t)split * p.B + mt) * kHN;
    const int rows = max(0, min(kHM, p.B - mt));
    for (int e = tid; e < rows * (kHN / 4); e += kHThreads) {
      const int r = e / (kHN / 4), c4 = (e % (kHN / 4)) * 4;
      *reinterpret_cast<float4*>(dst + (int64_t)r * kHN + c4) =
          *reinterpret_cast<const float4*>(reinterpret_cast<const float*>(sm) + r * kAccStride + c4);
    }
    __syncthreads();
  }
  tc_fence_before();
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTP * kHN));
}

// Split-K sum (in split order) + b1, ReLU, layers 2-3, argmax, H_t for p.tail_rows
// rows per CTA.  A programmatic dependent of k_hrad: each thread loads its slice of W2
// (output j = tid % 64, hidden-1 columns [32 sl, 32 sl + 32), sl = tid / 64) into
// registers before griddepcontrol.wait, so it overlaps k_hrad's tail.  Layer 2 then
// costs one broadcast LDS.128 per four FMAs (h1 rows in shared memory); the 8 slice
// partials of each output are summed in slice order (deterministic).
constexpr int kSl = kTailThreads / kH2;  // 8 slices of hidden-1
constexpr int kSw = kHN / kSl;           // 32 columns per slice
static_assert(kSl * kH2 == kTailThreads && kSw % 4 == 0, "tail geometry");
constexpr size_t kTailSmem = (size_t)(kTailRowsMax * kHN + kTailRowsMax * kSl * kH2 + kTailRowsMax * kH2) * 4;
__global__ void __launch_bounds__(kTailThreads, 1) k_hrad_tail(HradParams p) {
  extern __shared__ float tsm[];
  float* h1s = tsm;                              // [R][256]
  float* part = h1s + kTailRowsMax * kHN;        // [R][8][64]
  float* h2s = part + kTailRowsMax * kSl * kH2;  // [R][64]
  const int tid = threadIdx.x, j = tid % kH2, sl = tid / kH2;
  const int R = p.tail_rows;
  const int r0 = blockIdx.x * R;
  const int rows = min(R, p.B - r0);
  float4 w[kSw / 4];
  const float4* wsrc = reinterpret_cast<const float4*>(p.w2 + j * kHN + sl * kSw);
#pragma unroll
  for (int i = 0; i < kSw / 4; ++i) w[i] = __ldg(wsrc + i);
  asm volatile("griddepcontrol.wait;" ::: "memory");  // k_hrad's partials are complete
  // split sum: float4 element e = rr * 64 + c/4 of the CTA's rows (contiguous in each
  // split's partial), at most two per thread (R <= 16), 2 x 6 split loads in flight
  static_assert(kTailRowsMax * kHN / 4 <= 2 * kTailThreads, "two split-sum elements per thread");
  {
    const int nel = rows * (kHN / 4);
    const int64_t qs = (int64_t)p.B * kHN / 4;
    const float4* base = reinterpret_cast<const float4*>(p.partial) + (int64_t)r0 * (kHN / 4);
    const int e0 = tid, e1 = tid + kTailThreads;
    const bool has0 = e0 < nel, has1 = e1 < nel;
    const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
    float4 s0 = has0 ? __ldcg(base + e0) : z4, s1 = has1 ? __ldcg(base + e1) : z4;
    for (int q0 = 1; q0 < p.S; q0 += 6) {
      float4 v0[6], v1[6];
#pragma unroll
      for (int jj = 0; jj < 6; ++jj) {
        const bool in = q0 + jj < p.S;
        v0[jj] = (in && has0) ? __ldcg(base + (q0 + jj) * qs + e0) : z4;
        v1[jj] = (in && has1) ? __ldcg(base + (q0 + jj) * qs + e1) : z4;
      }
#pragma unroll
      for (int jj = 0; jj < 6; ++jj)
        if (q0 + jj < p.S) {
          s0.x += v0[jj].x; s0.y += v0[jj].y; s0.z += v0[jj].z; s0.w += v0[jj].w;
          s1.x += v1[jj].x; s1.y += v1[jj].y; s1.z += v1[jj].z; s1.w += v1[jj].w;
        }
    }
    if (has0) {
      const float4 bb = __ldg(reinterpret_cast<const float4*>(p.b1) + e0 % (kHN / 4));
      reinterpret_cast<float4*>(h1s)[e0] = make_float4(fmaxf(s0.x + bb.x, 0.f), fmaxf(s0.y + bb.y, 0.f),
                                                       fmaxf(s0.z + bb.z, 0.f), fmaxf(s0.w + bb.w, 0.f));
    }
    if (has1) {
      const float4 bb = __ldg(reinterpret_cast<const float4*>(p.b1) + e1 % (kHN / 4));
      reinterpret_cast<float4*>(h1s)[e1] = make_float4(fmaxf(s1.x + bb.x, 0.f), fmaxf(s1.y + bb.y, 0.f),
                                                       fmaxf(s1.z + bb.z, 0.f), fmaxf(s1.w + bb.w, 0.f));
    }
  }
  __syncthreads();
  for (int rr = 0; rr < rows; ++rr) {
    const float4* h = reinterpret_cast<const float4*>(h1s + rr * kHN + sl * kSw);
    float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
#pragma unroll
    for (int i = 0; i < kSw / 4; ++i) {
      const float4 x = h[i];
      a0 = fmaf(w[i].x, x.x, a0);
      a1 = fmaf(w[i].y, x.y, a1);
      a2 = fmaf(w[i].z, x.z, a2);
      a3 = fmaf(w[i].w, x.w, a3);
    }
    part[(rr * kSl + sl) * kH2 + j] = (a0 + a1) + (a2 + a3);
  }
  __syncthreads();
  for (int e = tid; e < rows * kH2; e += kTailThreads) {
    const int rr = e / kH2, jj = e % kH2;
    float a = 0.f;
#pragma unroll
    for (int q = 0; q < kSl; ++q) a += part[(rr * kSl + q) * kH2 + jj];
    h2s[rr * kH2 + jj] = fmaxf(a + __ldg(p.b2 + jj), 0.f);
  }
  __syncthreads();
  if (tid < rows) {
    const int rr = tid, b = r0 + rr;
    float l[kCls];
#pragma unroll
    for (int k = 0; k < kCls; ++k) {
      float a = 0.f;
      for (int j = 0; j < kH2; ++j) a = fmaf(__ldg(p.w3 + k * kH2 + j), h2s[rr * kH2 + j], a);
      l[k] = a + __ldg(p.b3 + k);
      if (p.logits) p.logits[(int64_t)b * kCls + k] = l[k];
    }
    int best = 0;
#pragma unroll
    for (int k = 1; k < kCls; ++k)
      if (l[k] > l[best]) best = k;  // ties -> smaller class
    p.s_t[b] = best;
    if (p.gamma || p.bpos) {
      int st = p.stop ? __ldg(p.stop + b) : p.G;
      st = min(max(st, 0), p.G);
      const int g = best == 0 ? 0 : (best == 1 ? st : p.G);
      if (p.gamma) p.gamma[b] = g;
      if (p.bpos) p.bpos[b] = g;
    }
  }
}

// ---------------------------------------------------------------- host side
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(f);
  }
  return fn;
}

// 2-D bf16 map of a row-major [rows][cols] matrix, box = [box_rows][64 columns].
static bool make_map(CUtensorMap* m, const void* base, int rows, int cols, int box_rows) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  const cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
  const cuuint32_t box[2] = {(cuuint32_t)kHK, (cuuint32_t)box_rows};
  const cuuint32_t estr[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Cluster width along the row tiles (W1 multicast) and K splits per tile: as many
// splits as fill the SMs (one CTA each), <= k-blocks, <= 16 (the tail sums them).
static int hrad_splits(int mtiles, int nkb) {
  const char* e = getenv("SB_HRAD_SPLITS");  // experiment override
  const int force = e ? std::max(1, atoi(e)) : 0;
  if (force > 0) return std::min(nkb, force);
  // fill the SMs, but no more than 18 splits (32 for a single 256-row block): the tail
  // reads S x B x 1 KB of partials (measured with the register-sliced tail: B = 2048
  // 12 / 18 / 24 splits 47.3 / 44.7 / 61.0 us; B = 256 16 / 32 / 64 splits 33.0 / 31.3 / 32.8 us)
  const int cap = mtiles == 1 ? 32 : 18;
  return std::max(1, std::min(std::min(nkb, cap), num_sms() / mtiles));
}

}  // namespace sb

using namespace sb;

extern "C" size_t sb_hrad_workspace_bytes(int32_t B, int32_t Dz) {
  if (B < 1 || Dz < kHK) return 0;
  const int mtiles = (B + kTP * kHM - 1) / (kTP * kHM);
  return (size_t)hrad_splits(mtiles, Dz / kHK) * B * kHN * sizeof(float);
}

extern "C" sb_status sb_hrad_predict(int32_t B, int32_t Dz, int32_t G, const void* z, const void* w1,
                                     const float* b1, const float* w2, const float* b2, const float* w3,
                                     const float* b3, const int32_t* stop, float* logits, int32_t* s_t,
                                     int32_t* gamma, int32_t* branch_pos, void* workspace,
                                     size_t workspace_bytes, sb_stream_t stream) {
  SB_NVTX("sb_hrad_predict");
  if (B < 1 || Dz < 1 || G < 0 || G > kMaxG || !z || !w1 || !b1 || !w2 || !b2 || !w3 || !b3 || !s_t ||
      !workspace)
    return SB_ERR_INVALID_ARG;
  if (Dz % kHK != 0 || (uintptr_t)z % 16 || (uintptr_t)w1 % 16 || (uintptr_t)b1 % 16 || (uintptr_t)w2 % 16)
    return SB_ERR_UNSUPPORTED;
  if ((uintptr_t)workspace % 16) return SB_ERR_INVALID_ARG;
  if (workspace_bytes < sb_hrad_workspace_bytes(B, Dz)) return SB_ERR_WORKSPACE;
  if (ensure_smem<k_hrad>((int)kHradSmem) != cudaSuccess || ensure_smem<k_hrad_tail>((int)kTailSmem) != cudaSuccess)
    return SB_ERR_CUDA;
  const int mtiles = (B + kTP * kHM - 1) / (kTP * kHM);
  CUtensorMap tmZ, tmW1;
  if (!make_map(&tmZ, z, B, Dz, kHM) || !make_map(&tmW1, w1, kHN, Dz, kHN)) return SB_ERR_CUDA;
  HradParams p;
  p.B = B; p.Dz = Dz; p.G = G; p.nkb = Dz / kHK; p.S = hrad_splits(mtiles, p.nkb);
  p.tail_rows = std::max(1, std::min(kTailRowsMax, (B + 127) / 128));
  p.partial = static_cast<float*>(workspace);
  p.b1 = b1; p.w2 = w2; p.b2 = b2; p.w3 = w3; p.b3 = b3; p.stop = stop;
  p.logits = logits; p.s_t = s_t; p.gamma = gamma; p.bpos = branch_pos;
  cudaStream_t s = (cudaStream_t)stream;
  k_hrad<<<dim3(p.S, mtiles), kHThreads, kHradSmem, s>>>(tmZ, tmW1, p);
  if (cudaGetLastError() != cudaSuccess) return SB_ERR_CUDA;
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at;
  at.id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at.val.programmaticStreamSerializationAllowed = 1;
  cfg.gridDim = dim3((B + p.tail_rows - 1) / p.tail_rows, 1, 1);
  cfg.blockDim = dim3(kTailThreads, 1, 1);
  cfg.dynamicSmemBytes = kTailSmem;
  cfg.stream = s;
  cfg.attrs = &at;
  cfg.numAttrs = 1;
  if (cudaLaunchKernelEx(&cfg, k_hrad_tail, p) != cudaSuccess) return SB_ERR_CUDA;
  return cuda_status(cudaGetLastError());
}
