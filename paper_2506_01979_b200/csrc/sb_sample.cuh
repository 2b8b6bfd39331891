// sb_sample.cuh — inverse-CDF sampling helpers shared by k_select_tma and k_step
// (residual / bonus sample, SURVEY §8.0 "Inverse CDF"; P94, P547, P554).
#pragma once
#include "sb_common.cuh"

namespace sb {

// Sampling works in the p row's unnormalised scale: e_p = 2^(l_p c - MS_p),
// e_q = 2^(l_q c - MS_q), r' = max(0, e_p - (Z_p/Z_q) e_q) = Z_p max(0, P - Q) (bonus:
// r' = e_p = Z_p P).  The inverse CDF is scale-invariant (t' = us * sum r'), so neither
// normaliser multiply is needed per element.  Explicit rounding intrinsics keep the
// arithmetic identical wherever it is inlined (consumers and epilogue must agree).
// A segment is 1 KB of a row: lane l owns its two adjacent 16-byte vectors.
constexpr int kSegBytes = 1024;

template <typename T>
__device__ __forceinline__ void r_scaled(const uint4& vp, const uint4& vq, bool resid, float MSp, float MSq,
                                         float kq, float* r) {
  constexpr int E = Vec<T>::E;
  static_assert(E % 2 == 0, "element pairs");
  float lp[E], lq[E];
  Vec<T>::unpack(vp, lp);
  if (resid) Vec<T>::unpack(vq, lq);
  // element pairs through FFMA2 (fma.rn.f32x2: the same IEEE operation per element as
  // the scalar fmaf, so the consumers' and the epilogue's values stay bit-identical)
  const float2 c2 = make_float2(kC, kC), np = make_float2(-MSp, -MSp), nq = make_float2(-MSq, -MSq),
               nk = make_float2(-kq, -kq);
#pragma unroll
  for (int e = 0; e < E; e += 2) {
    const float2 ap = __ffma2_rn(make_float2(lp[e], lp[e + 1]), c2, np);
    const float2 ep = make_float2(ex2(ap.x), ex2(ap.y));
    if (resid) {
      const float2 aq = __ffma2_rn(make_float2(lq[e], lq[e + 1]), c2, nq);
      const float2 eq = make_float2(ex2(aq.x), ex2(aq.y));
      const float2 d = __ffma2_rn(nk, eq, ep);
      r[e] = fmaxf(d.x, 0.f);
      r[e + 1] = fmaxf(d.y, 0.f);
    } else {
      r[e] = ep.x;
      r[e + 1] = ep.y;
    }
  }
}
template <int E>
__device__ __forceinline__ float seq_sum(const float* r, float s) {
#pragma unroll
  for (int e = 0; e < E; ++e) s = __fadd_rn(s, r[e]);
  return s;
}
__device__ __forceinline__ float warp_sum_rn(float x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x = __fadd_rn(x, __shfl_xor_sync(0xffffffffu, x, o));
  return x;
}
__device__ __forceinline__ float warp_scan_rn(float x) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const float y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x = __fadd_rn(x, y);
  }
  return x;
}
template <typename T>
__device__ __forceinline__ uint4 seg_vec(const T* row, uint32_t row_bytes, uint32_t off) {
  if (off < row_bytes) return __ldg(reinterpret_cast<const uint4*>(reinterpret_cast<const char*>(row) + off));
  return sizeof(T) == 2 ? make_uint4(0xff80ff80u, 0xff80ff80u, 0xff80ff80u, 0xff80ff80u)
                        : make_uint4(0xff800000u, 0xff800000u, 0xff800000u, 0xff800000u);
}

// The epilogue warp's own pass over a whole row (rare: zero residual mass fallback).
template <typename T>
__device__ void warp_segments(const T* prow, const T* qrow, uint32_t row_bytes, int nseg, bool resid,
                              float MSp, float MSq, float kq, float* seg) {
  constexpr int E = Vec<T>::E;
  const int lane = threadIdx.x & 31;
  for (int sI = 0; sI < nseg; ++sI) {
    float own = 0.f;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const uint32_t off = (uint32_t)sI * kSegBytes + lane * 32 + j * 16;
      float r[E];
      r_scaled<T>(seg_vec(prow, row_bytes, off), resid ? seg_vec(qrow, row_bytes, off) : uint4{}, resid, MSp,
                  MSq, kq, r);
      own = seq_sum<E>(r, own);
    }
    const float tot = warp_sum_rn(own);
    if (lane == 0) seg[sI] = tot;
  }
  __syncwarp();
}


// Locate t = us * R over per-segment sums (fp64 prefix in segment order, lanes own
// contiguous ranges), re-read that one segment and return the first id whose running
// mass exceeds t (fallback: the last id with mass).  seg: nseg sums (shared memory).
// Returns the id (or -1) in every lane; *R_out = total mass (scaled).
template <typename T>
__device__ __forceinline__ int sample_segments(const T* prow, const T* qrow, uint32_t row_bytes, int V, float* seg,
                                               int nseg, bool& resid, float MSp, float MSq, float kq, float us,
                                               int& st, double* R_out) {
  constexpr int E = Vec<T>::E;
  const int lane = threadIdx.x & 31;
  const int per = (nseg + 31) / 32;
  double R = 0.0, excl = 0.0, incl = 0.0;
  for (int attempt = 0; attempt < 2; ++attempt) {
    double local = 0.0;
    for (int j = 0; j < per; ++j) {
      const int sI = lane * per + j;
      if (sI < nseg) local += (double)seg[sI];
    }
    incl = local;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double yv = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += yv;
    }
    excl = __shfl_up_sync(0xffffffffu, incl, 1);  // lane ranges [excl, incl) tile [0, R)
    if (lane == 0) excl = 0.0;
    R = __shfl_sync(0xffffffffu, incl, 31);
    if (R > 0.0 || !resid) break;
    resid = false;  // "no residual mass" (S134-140): sample from P
    st |= SB_ST_ZERO_RESID;
    warp_segments<T>(prow, qrow, row_bytes, nseg, false, MSp, MSq, kq, seg);
  }
  *R_out = R;
  const double t = (double)us * R;
  int found = -1, lastpos = -1;
  double Fprev = 0.0;
  const bool mine = (excl <= t && incl > t);
  {
    double F = excl;
    for (int j = 0; j < per; ++j) {
      const int sI = lane * per + j;
      if (sI >= nseg) break;
      if (seg[sI] > 0.f) lastpos = sI;
      if (mine && found < 0 && F + (double)seg[sI] > t) { found = sI; Fprev = F; }
      F += (double)seg[sI];
    }
  }
  const unsigned who = __ballot_sync(0xffffffffu, found >= 0);
  int sStar;
  double trem;
  if (who) {
    const int src = __ffs(who) - 1;
    sStar = __shfl_sync(0xffffffffu, found, src);
    trem = t - __shfl_sync(0xffffffffu, Fprev, src);
  } else {  // rounding: the last segment with mass, and the in-segment fallback
    const unsigned mw = __ballot_sync(0xffffffffu, mine);
    const int src = mw ? __ffs(mw) - 1 : -1;
    const int cand = src >= 0 ? __shfl_sync(0xffffffffu, lastpos, src) : -1;
    sStar = cand >= 0 ? cand : (int)__reduce_max_sync(0xffffffffu, (unsigned)(lastpos + 1)) - 1;
    trem = CUDART_INF;
  }
  int y = -1;
  if (sStar >= 0) {
    float r[2][E], own = 0.f;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const uint32_t off = (uint32_t)sStar * kSegBytes + lane * 32 + j * 16;
      r_scaled<T>(seg_vec(prow, row_bytes, off), resid ? seg_vec(qrow, row_bytes, off) : uint4{}, resid, MSp,
                  MSq, kq, r[j]);
      own = seq_sum<E>(r[j], own);
    }
    const float incl2 = warp_scan_rn(own);
    float F = __shfl_up_sync(0xffffffffu, incl2, 1);
    if (lane == 0) F = 0.f;
    int cand = 0x7fffffff, lastv = -1;
    const int vbase = (int)(((uint32_t)sStar * kSegBytes + lane * 32) / sizeof(T));
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int e = 0; e < E; ++e) {
        F = __fadd_rn(F, r[j][e]);
        const int v = vbase + j * E + e;
        if (cand == 0x7fffffff && (double)F > trem && r[j][e] > 0.f) cand = v;
        if (r[j][e] > 0.f) lastv = v;
      }
    const int pick = (int)__reduce_min_sync(0xffffffffu, (unsigned)cand);
    y = (pick != 0x7fffffff) ? pick : (int)__reduce_max_sync(0xffffffffu, (unsigned)(lastv + 1)) - 1;
    if (y >= V) y = -1;
  }
  return y;
}

// Offsets (exclusive scan of commit_len) and the packed commit stream, by one warp
// (the epilogue that completes the last sequence).
// Block-wide version (NT threads): exclusive scan of commit_len into offsets[0..B] and
// the packed token stream; each thread owns a contiguous run of sequences, all its
// loads are independent (one round trip per phase instead of one per sequence).
template <int NT>
__device__ __forceinline__ void block_offsets(int B, int G, const int* commit_len, const int* out_tok, int* offsets,
                                              int* packed_tok, int* scan /* smem, >= NT/32 ints */) {
  constexpr int NW = (NT + 31) / 32;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int per = (B + NT - 1) / NT;
  const int b0 = min(B, tid * per), b1 = min(B, b0 + per);
  int loc = 0;
  for (int qq = b0; qq < b1; ++qq) loc += __ldcg(commit_len + qq);
  int incl = loc;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int yv = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += yv;
  }
  if (lane == 31) scan[w] = incl;
  __syncthreads();
  if (w == 0) {
    int x = lane < NW ? scan[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int yv = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += yv;
    }
    if (lane < NW) scan[lane] = x;  // inclusive over warps
  }
  __syncthreads();
  int run = incl - loc + (w > 0 ? scan[w - 1] : 0);
  for (int qq = b0; qq < b1; ++qq) {
    offsets[qq] = run;
    const int cl = __ldcg(commit_len + qq);
    if (packed_tok) {
      const int* src = out_tok + (int64_t)qq * (G + 2);
#pragma unroll 4
      for (int c = 0; c < cl; ++c) packed_tok[run + c] = __ldcg(src + c);
    }
    run += cl;
  }
  if (tid == NT - 1) offsets[B] = scan[NW - 1];
}

__device__ __forceinline__ void warp_offsets(int B, int G, const int* commit_len, const int* out_tok, int* offsets,
                                             int* packed_tok) {
  const int lane = threadIdx.x & 31;
  const int per = (B + 31) / 32;
  const int b0 = min(B, lane * per), b1 = min(B, b0 + per);
  int loc = 0;
  for (int qq = b0; qq < b1; ++qq) loc += __ldcg(commit_len + qq);
  int incl = loc;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int yv = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += yv;
  }
  int run = incl - loc;
  for (int qq = b0; qq < b1; ++qq) {
    offsets[qq] = run;
    const int cl = __ldcg(commit_len + qq);
    if (packed_tok)
      for (int c = 0; c < cl; ++c) packed_tok[run + c] = __ldcg(out_tok + (int64_t)qq * (G + 2) + c);
    run += cl;
  }
  if (lane == 31) offsets[B] = incl;
}

}  // namespace sb
