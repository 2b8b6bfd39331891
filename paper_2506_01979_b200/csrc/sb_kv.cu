// sb_kv.cu — sb_kv_rollback: keep the surviving branch's draft KV rows and drop the
// rest (PAPER P241 "discarding all non-selected branches and their
// associated KV-Cache", shared-prefix KV P220).  A pure HBM gather driven by the keep
// mask of sb_select_branch (bit i of keep_mask[b][k] set iff the draft token at slot k,
// position i is committed — at most one slot per position, already reflecting the
// clamped gamma_b / s_b layout): the kept row of position i is copied to out[b][i]
// (out-of-place), or into slot 0 in place (out = NULL; rows already in slot 0 stay).
// 16-byte vectors, 4 in flight per thread.
#include <algorithm>

#include "sb_host.h"

namespace sb {

constexpr int kKvU = 4;  // 16-byte vectors in flight per thread

struct KvParams {
  int B, K, R1;
  int64_t row_bytes, stride;  // bytes per position, bytes between positions
  const char* kv;
  char* out;
  const uint32_t* keep;       // [B][K] keep mask of sb_select_branch
};

// one CTA per (sequence, position), sized so every thread has its U vectors of the row
// in flight at once (many small CTAs per SM hide the decision loads' latency)
template <int U>
__global__ void __launch_bounds__(256) k_kv_rollback(KvParams p) {
  const int b = blockIdx.x / p.R1, i = blockIdx.x % p.R1;
  int slot = -1;
  for (int k = 0; k < p.K; ++k)
    if ((__ldg(p.keep + (int64_t)b * p.K + k) >> i) & 1u) slot = k;
  if (slot < 0) return;  // not committed: a rolled-back position
  const char* src = p.kv + (((int64_t)b * p.K + slot) * p.R1 + i) * p.stride;
  char* dst;
  if (p.out) {
    dst = p.out + ((int64_t)b * p.R1 + i) * p.stride;
  } else {
    if (slot == 0) return;  // already in place
    dst = const_cast<char*>(p.kv) + (((int64_t)b * p.K + 0) * p.R1 + i) * p.stride;
  }
  const int64_t nv = p.row_bytes / 16;
  const uint4* s4 = reinterpret_cast<const uint4*>(src);
  uint4* d4 = reinterpret_cast<uint4*>(dst);
  for (int64_t v = threadIdx.x; v < nv; v += U * blockDim.x) {
    uint4 x[U];
#pragma unroll
    for (int j = 0; j < U; ++j)
      if (v + j * blockDim.x < nv) x[j] = ldg_stream(s4 + v + j * blockDim.x);
#pragma unroll
    for (int j = 0; j < U; ++j)
      if (v + j * blockDim.x < nv) d4[v + j * blockDim.x] = x[j];
  }
}

}  // namespace sb

using namespace sb;

extern "C" sb_status sb_kv_rollback(int32_t B, int32_t K, int32_t G, const void* kv, int64_t row_bytes,
                                    int64_t row_stride_bytes, const uint32_t* keep_mask, void* out_kv,
                                    sb_stream_t stream) {
  SB_NVTX("sb_kv_rollback");
  if (B < 1 || K < 1 || K > kMaxK || G < 0 || G > kMaxG || !kv || !keep_mask) return SB_ERR_INVALID_ARG;
  if (row_bytes <= 0 || row_bytes % 16 || row_stride_bytes < row_bytes || row_stride_bytes % 16) return SB_ERR_INVALID_ARG;
  if ((uintptr_t)kv % 16 || (uintptr_t)out_kv % 16) return SB_ERR_INVALID_ARG;
  KvParams p;
  p.B = B; p.K = K; p.R1 = G + 1; p.row_bytes = row_bytes; p.stride = row_stride_bytes;
  p.kv = static_cast<const char*>(kv); p.out = static_cast<char*>(out_kv); p.keep = keep_mask;
  // 4 vectors in flight per thread (8 KB rows: 128-thread CTAs).  Measured on the
  // C4-shaped rollback: 2 / 4 / 8 / 16 vectors per thread 35.1 / 26.2 / 29.0 / 29.0 us
  constexpr int U = kKvU;
  const int nt = (int)std::min<int64_t>(256, std::max<int64_t>(32, (row_bytes / 16 + U - 1) / U + 31) / 32 * 32);
  k_kv_rollback<U><<<B * (G + 1), nt, 0, (cudaStream_t)stream>>>(p);
  return cuda_status(cudaGetLastError());
}
