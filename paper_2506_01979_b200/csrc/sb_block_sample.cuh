// sb_block_sample.cuh — whole-block inverse-CDF sampler over one row (pair): the
// residual norm(max(0, p - q)) or the bonus p (P94, P547, P554; SURVEY §8.0 "Inverse
// CDF").  Used by the fallback select kernel and by the tree verify (f3).
//   pass A  r(v) tile by tile, each thread owning E consecutive ids of a tile, per-thread
//           sequential sum, warp Kogge-Stone scan, warp totals kept in shared memory;
//           tile sums = fixed-order sums of warp totals; R = fp64 sum of tile sums.
//   locate  t = us * R, first tile whose fp64 running sum exceeds t.
//   pass B  the same arithmetic on that one tile (hits L2), prefix inside the tile,
//           first id whose running mass exceeds t (block min).
#pragma once
#include "sb_common.cuh"
#include "sb_host.h"

namespace sb {

constexpr int kMaxTiles = 512;

template <typename T, int NT>
struct Sampler {
  static constexpr int E = Vec<T>::E;
  static constexpr int TE = NT * E;  // ids per tile
  static constexpr int NW = NT / 32;

  const T* prow;
  const T* qrow;
  int V;
  bool vec_ok;
  bool resid;  // residual max(0,P-Q) (else P)
  float MSp, iZp, MSq, iZq;

  // raw logits of the E ids this thread owns in tile t (-inf past V)
  __device__ __forceinline__ void load(int t, float* lp, float* lq) const {
    const int v0 = t * TE + threadIdx.x * E;
    if (vec_ok && v0 + E <= V) {
      Vec<T>::unpack(ldg_stream(prow + v0), lp);
      if (resid) Vec<T>::unpack(ldg_stream(qrow + v0), lq);
    } else {
#pragma unroll
      for (int j = 0; j < E; ++j) {
        const bool in = v0 + j < V;
        lp[j] = in ? ld_scalar(prow + v0 + j) : -CUDART_INF_F;
        lq[j] = (in && resid) ? ld_scalar(qrow + v0 + j) : -CUDART_INF_F;
      }
    }
  }
  // r = max(0, P - Q) (or P) from the raw logits
  __device__ __forceinline__ void compute(const float* lp, const float* lq, float* r) const {
#pragma unroll
    for (int j = 0; j < E; ++j) {
      const float P = ex2(fmaf(lp[j], kC, -MSp)) * iZp;
      if (resid) {
        const float Q = ex2(fmaf(lq[j], kC, -MSq)) * iZq;
        r[j] = fmaxf(P - Q, 0.f);
      } else {
        r[j] = P;
      }
    }
  }
  __device__ __forceinline__ void values(int t, float* r) const {
    float lp[E], lq[E];
    load(t, lp, lq);
    compute(lp, lq, r);
  }
};

// Row softmax state of one row by the whole block (used for the bonus row).
template <typename T, int NT>
__device__ RowOut block_row_stats(const T* row, int V, bool vec_ok, RowStat* red, float* m_out) {
  RowAcc<false, 4> a;
  a.init();
  stream_row<T, false, 4, NT, 4>(row, V, vec_ok, a);
  const RowStat s = block_reduce<NT>(fold(a), red);
  *m_out = s.m;
  return finish(s);
}

template <int NW>
struct SampleSmem {
  float wtot[kMaxTiles][NW];
  float tsum[kMaxTiles];
  RowStat red[NW];
  int tile, pick, fb;
  double trem, R;
};

// Every thread of the block calls this (block-uniform control flow).  smp.resid may be
// cleared (zero residual mass -> sample from p, SB_ST_ZERO_RESID in st).  Returns the
// sampled id in every thread (-1 if no id has mass); mass = R.
template <typename T, int NT>
__device__ int block_sample(Sampler<T, NT>& smp, float us, SampleSmem<NT / 32>& sm, int& st, double& mass) {
  using S = Sampler<T, NT>;
  constexpr int NW = S::NW;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int ntiles = (smp.V + S::TE - 1) / S::TE;
  if (tid == 0) {
    sm.pick = 0x7fffffff;
    sm.fb = -1;
  }
  for (int attempt = 0; attempt < 2; ++attempt) {
    // pass A: per-tile warp totals
    constexpr int UT = 4;  // tiles in flight per thread
    for (int t0 = 0; t0 < ntiles; t0 += UT) {
      float lp[UT][S::E], lq[UT][S::E];
#pragma unroll
      for (int q = 0; q < UT; ++q)
        if (t0 + q < ntiles) smp.load(t0 + q, lp[q], lq[q]);
#pragma unroll
      for (int q = 0; q < UT; ++q) {
        if (t0 + q >= ntiles) break;
        float r[S::E];
        smp.compute(lp[q], lq[q], r);
        float own = 0.f;
#pragma unroll
        for (int j = 0; j < S::E; ++j) own += r[j];
        const float incl = warp_incl_scan(own);
        if (lane == 31) sm.wtot[t0 + q][w] = incl;
      }
    }
    __syncthreads();
    for (int t = tid; t < ntiles; t += NT) {
      float s = 0.f;
#pragma unroll
      for (int q = 0; q < NW; ++q) s += sm.wtot[t][q];
      sm.tsum[t] = s;
    }
    __syncthreads();
    if (tid == 0) {
      double R = 0.0;
      for (int t = 0; t < ntiles; ++t) R += (double)sm.tsum[t];
      sm.R = R;
    }
    __syncthreads();
    if (sm.R > 0.0 || !smp.resid) break;
    smp.resid = false;  // "no residual mass" (S134-140): sample from P instead
    st |= SB_ST_ZERO_RESID;
    __syncthreads();
  }
  if (tid == 0) {
    const double R = sm.R, t = (double)us * R;
    double F = 0.0;
    int tile = -1;
    for (int q = 0; q < ntiles; ++q) {
      if (F + (double)sm.tsum[q] > t) { tile = q; break; }
      F += (double)sm.tsum[q];
    }
    if (tile < 0) {  // rounding: fall back to the last tile holding mass
      for (int q = ntiles - 1; q >= 0; --q)
        if (sm.tsum[q] > 0.f) { tile = q; break; }
      F = -1e300;  // no id qualifies -> the in-tile fallback (last id with mass)
    }
    sm.tile = tile;
    sm.trem = t - F;
  }
  __syncthreads();
  const int tile = sm.tile;
  int y = -1;
  if (tile >= 0) {
    // pass B on the located tile: identical arithmetic -> same warp totals
    float r[S::E];
    smp.values(tile, r);
    float own = 0.f;
#pragma unroll
    for (int j = 0; j < S::E; ++j) own += r[j];
    const float incl = warp_incl_scan(own);
    float excl = __shfl_up_sync(0xffffffffu, incl, 1);
    if (lane == 0) excl = 0.f;
    float base = 0.f;
    for (int q = 0; q < w; ++q) base += sm.wtot[tile][q];
    float F = base + excl;
    const double trem = sm.trem;
    int mine = 0x7fffffff, last_pos = -1;
#pragma unroll
    for (int j = 0; j < S::E; ++j) {
      F += r[j];
      const int v = tile * S::TE + tid * S::E + j;
      if (mine == 0x7fffffff && (double)F > trem && r[j] > 0.f) mine = v;
      if (r[j] > 0.f) last_pos = v;
    }
    if (mine != 0x7fffffff) atomicMin(&sm.pick, mine);
    if (last_pos >= 0) atomicMax(&sm.fb, last_pos);
    __syncthreads();
    y = (sm.pick != 0x7fffffff) ? sm.pick : sm.fb;
  }
  mass = sm.R;
  return y;
}

}  // namespace sb
