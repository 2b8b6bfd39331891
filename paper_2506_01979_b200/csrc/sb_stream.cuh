// sb_stream.cuh — pieces shared by the TMA-ring streaming kernels (k_rows_tma,
// k_step_tma, k_conf_tma): the ring geometry and the deferred exact first-argmax of a
// q row (consumer warps record candidates, an epilogue warp resolves the index).
#pragma once
#include "sb_common.cuh"

namespace sb {

template <int CW_, int NS_, int VPT_, int NP_, int NE_ = 2>
struct RC {
  static constexpr int CW = CW_, NS = NS_, VPT = VPT_, NP = NP_;
  static constexpr int CT = CW * 32;
  static constexpr int CHUNK = CT * VPT * 16;
  static constexpr int NE = NE_;  // epilogue warps (k_rows_tma), alternating units
  static constexpr int THREADS = CT + 64;
  static constexpr int ROWS_THREADS = CT + 32 * (1 + NE);
  static_assert(NP % NE == 0, "each epilogue warp owns NP / NE partial slots");
};

// Consumer side of a q row without the argmax lookup: the warp's reduced state (idx
// unresolved) and its argmax candidates: the smallest chunk tag among the lanes holding
// the warp maximum and the mask of those lanes with that tag.  The epilogue warp
// resolves the index (resolve_argmax) off the consumers' critical path.
template <bool kQ>
__device__ __forceinline__ RowStat warp_part_deferred(const LazyAcc<kQ, 4>& a, uint2& cand) {
  RowStat s = fold_lazy(a);
  float mw = s.m;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mw = fmaxf(mw, __shfl_xor_sync(0xffffffffu, mw, o));
  const bool hold = (a.m == mw) && (mw > -CUDART_INF_F) && (a.tag >= 0);
  const unsigned t = hold ? (unsigned)a.tag : 0xffffffffu;
  const unsigned tmin = __reduce_min_sync(0xffffffffu, t);
  cand = make_uint2(tmin, __ballot_sync(0xffffffffu, hold && t == tmin));
  s = warp_reduce_offsets(s);
  s.m = mw;
  s.idx = 0x7fffffff;
  return s;
}

// Epilogue side: lane w < CW holds warp w's part (mw = its maximum) and candidates;
// M = the row maximum.  The first index of M lies in the smallest candidate chunk of
// the warps holding M; the candidate lanes re-read their vectors of that chunk (one
// load round, normally one lane).  Returns the index in every lane.
template <class C, typename T>
__device__ __forceinline__ int resolve_argmax(float mw, uint2 cand, float M, const T* row, int nvec_last,
                                              int nchunks) {
  constexpr int E = Vec<T>::E;
  const int lane = threadIdx.x & 31;
  const unsigned t = (lane < C::CW && mw == M && M > -CUDART_INF_F) ? cand.x : 0xffffffffu;
  const unsigned tmin = __reduce_min_sync(0xffffffffu, t);
  int best = 0x7fffffff;
  if (t == tmin && tmin != 0xffffffffu) {
    const int c = (int)tmin;
    const int nvec = (c == nchunks - 1) ? nvec_last : C::CHUNK / 16;
    const uint4* cv =
        reinterpret_cast<const uint4*>(reinterpret_cast<const char*>(row) + (size_t)c * C::CHUNK);
    for (uint32_t m = cand.y; m; m &= m - 1) {
      const int tid = lane * 32 + __ffs(m) - 1;
#pragma unroll
      for (int j = 0; j < C::VPT; ++j) {
        const int v = tid + j * C::CT;
        if (v >= nvec) continue;
        float f[E];
        Vec<T>::unpack(__ldg(cv + v), f);
#pragma unroll
        for (int e = E - 1; e >= 0; --e)
          if (f[e] == M) best = min(best, c * (C::CHUNK / (int)sizeof(T)) + v * E + e);
      }
    }
  }
  return (int)__reduce_min_sync(0xffffffffu, (unsigned)best);
}

}  // namespace sb
