// sb_select.cu — sb_select_branch: branch-point verification (Eq. 9 P236-241 /
// Alg. 1 P540), the correction or bonus sample (P94, P547, P554) and the commit /
// rollback compaction (P541, P555, P655; RB counters P317, P734).
// SURVEY §8.1 rows a3 + a4 + a5.
//
// One CTA per sequence.  Thread 0 takes the discrete decisions (exact compares of
// input values).  The sample re-streams at most one row pair:
//   pass A  r(v) = max(0, P(v) - Q(v)) (or P(v)) tile by tile, each thread owning E
//           consecutive ids of a tile, per-thread sequential sum, warp Kogge-Stone
//           inclusive scan, warp totals kept in shared memory; tile sums = fixed-order
//           sums of warp totals; R = fp64 sequential sum of tile sums.
//   locate  t = us * R, first tile whose fp64 running sum exceeds t.
//   pass B  the same arithmetic on that one tile (hits L2), prefix inside the tile,
//           first id whose running mass exceeds t (block min).
// A bonus row (not read by sb_verify_branches) first gets its own softmax pass.
// The last CTA to finish scans commit_len into offsets and writes the packed stream.
#include <algorithm>

#include "sb_host.h"

namespace sb {

struct SelParams {
  Dims d;
  const void* PL;
  const void* QL;
  const int* tok;
  const float* u;
  const float* us;
  const int* n_acc;
  int rule;
  const SeqInfo* info;
  const float4* rowstat;
  int* sel_cnt;
  int *sel_k, *commit_len, *out_tok, *y_tok, *y_kind, *offsets, *packed_tok, *path_rolled,
      *branch_discarded, *status;
  uint32_t* keep_mask;
  float* resid_mass;
};

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

template <typename T, int NT>
__global__ void __launch_bounds__(NT) k_select(SelParams p, bool vec_ok) {
  using S = Sampler<T, NT>;
  constexpr int NW = S::NW;
  __shared__ float wtot[kMaxTiles][NW];
  __shared__ float tsum[kMaxTiles];
  __shared__ RowStat red[NW];
  __shared__ int sh_ksel, sh_npath, sh_kind, sh_row, sh_slot, sh_st, sh_tile, sh_pick, sh_last,
      sh_fb;
  __shared__ double sh_trem, sh_R;
  const Dims& d = p.d;
  const int b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const SeqInfo in = p.info[b];
  const T* PL = static_cast<const T*>(p.PL);
  const T* QL = static_cast<const T*>(p.QL);

  if (tid == 0) {
    // A = {k : n_k > s_b}; Eq. 9: argmax raw target logit at the branch row (ties ->
    // smaller token id, then smaller k); Alg. 1: argmax r_b (ties -> smaller k)
    int ksel = -1, besttok = 0;
    float bestkey = 0.f;
    for (int k = 0; k < d.K; ++k) {
      if (__ldg(p.n_acc + (int64_t)b * d.K + k) <= in.s) continue;
      const int xk = __ldg(p.tok + ent(d, b, k, in.s));
      const float key = (p.rule == SB_SELECT_ALG1) ? __ldg(p.u + ent(d, b, k, in.s))
                                                   : ld_scalar(PL + row_off(d, b, 0, in.s) + xk);
      bool better;
      if (ksel < 0) better = true;
      else if (p.rule == SB_SELECT_ALG1) better = key > bestkey;
      else better = key > bestkey || (key == bestkey && xk < besttok);
      if (better) { ksel = k; bestkey = key; besttok = xk; }
    }
    int npath, kind, row = 0, slot = 0;
    if (ksel < 0) {
      const int n0 = __ldg(p.n_acc + (int64_t)b * d.K);
      npath = min(n0, in.s);  // rejection in the shared prefix or at the branch row (P655)
      kind = 1; row = npath; slot = 0;
    } else {
      npath = __ldg(p.n_acc + (int64_t)b * d.K + ksel);
      if (npath < in.L) { kind = 1; row = npath; slot = (npath <= in.s) ? 0 : ksel; }
      else if (in.s < in.g) { kind = 2; row = in.g; slot = ksel; }  // bonus from p_{gamma+1}
      else kind = 0;  // branch token accepted; continuation carried by the caller (P237)
    }
    sh_ksel = ksel; sh_npath = npath; sh_kind = kind; sh_row = row; sh_slot = slot;
    sh_st = 0;
    sh_pick = 0x7fffffff;
    sh_fb = -1;
  }
  __syncthreads();
  const int ksel = sh_ksel, npath = sh_npath;
  int kind = sh_kind;
  const int kpath = ksel < 0 ? 0 : ksel;

  int y = -1;
  double mass = 0.0;
  if (kind != 0) {
    S smp;
    smp.prow = PL + row_off(d, b, sh_slot, sh_row);
    smp.qrow = QL + row_off(d, b, sh_slot, sh_row);
    smp.V = d.V;
    smp.vec_ok = vec_ok;
    bool finite;
    float MSp, Zp, MSq = 0.f, Zq = 1.f;
    if (kind == 2) {
      float m;
      const RowOut o = block_row_stats<T, NT>(smp.prow, d.V, vec_ok, red, &m);
      MSp = o.MS; Zp = o.Z; finite = o.finite;
    } else {
      const float4 rs = p.rowstat[ent(d, b, sh_slot, sh_row)];
      MSp = rs.x; Zp = rs.y; MSq = rs.z; Zq = rs.w;
      finite = (Zp == Zp) && (Zq == Zq);
    }
    if (!finite) {
      kind = 0;
      if (tid == 0) sh_st |= SB_ST_NONFINITE;
    } else {
      smp.MSp = MSp; smp.iZp = 1.f / Zp; smp.MSq = MSq; smp.iZq = 1.f / Zq;
      smp.resid = (kind == 1);
      const int ntiles = (d.V + S::TE - 1) / S::TE;
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
            if (lane == 31) wtot[t0 + q][w] = incl;
          }
        }
        __syncthreads();
        for (int t = tid; t < ntiles; t += NT) {
          float s = 0.f;
#pragma unroll
          for (int q = 0; q < NW; ++q) s += wtot[t][q];
          tsum[t] = s;
        }
        __syncthreads();
        if (tid == 0) {
          double R = 0.0;
          for (int t = 0; t < ntiles; ++t) R += (double)tsum[t];
          sh_R = R;
        }
        __syncthreads();
        if (sh_R > 0.0 || !smp.resid) break;
        smp.resid = false;  // "no residual mass" (S134-140): sample from P instead
        if (tid == 0) sh_st |= SB_ST_ZERO_RESID;
        __syncthreads();
      }
      if (tid == 0) {
        const double R = sh_R, t = (double)__ldg(p.us + b) * R;
        double F = 0.0;
        int tile = -1;
        for (int q = 0; q < ntiles; ++q) {
          if (F + (double)tsum[q] > t) { tile = q; break; }
          F += (double)tsum[q];
        }
        if (tile < 0) {  // rounding: fall back to the last tile holding mass
          for (int q = ntiles - 1; q >= 0; --q)
            if (tsum[q] > 0.f) { tile = q; break; }
          F = -1e300;  // no id qualifies -> the in-tile fallback (last id with mass)
        }
        sh_tile = tile;
        sh_trem = t - F;
      }
      __syncthreads();
      const int tile = sh_tile;
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
        for (int q = 0; q < w; ++q) base += wtot[tile][q];
        float F = base + excl;
        const double trem = sh_trem;
        int mine = 0x7fffffff, last_pos = -1;
#pragma unroll
        for (int j = 0; j < S::E; ++j) {
          F += r[j];
          const int v = tile * S::TE + tid * S::E + j;
          if (mine == 0x7fffffff && (double)F > trem && r[j] > 0.f) mine = v;
          if (r[j] > 0.f) last_pos = v;
        }
        if (mine != 0x7fffffff) atomicMin(&sh_pick, mine);
        if (last_pos >= 0) atomicMax(&sh_fb, last_pos);
        __syncthreads();
        y = (sh_pick != 0x7fffffff) ? sh_pick : sh_fb;
      }
      mass = sh_R;
    }
  }

  // commit: path tokens, y, counters, keep mask (SURVEY §8.0 "Commit")
  const int R1 = d.G + 1;
  int* out = p.out_tok + (int64_t)b * (d.G + 2);
  for (int q = tid; q < d.G + 2; q += NT) {
    int v = -1;
    if (q < npath) v = __ldg(p.tok + ent(d, b, (q < in.s) ? 0 : kpath, q));
    else if (q == npath && kind != 0) v = y;
    out[q] = v;
  }
  if (tid < d.K) {
    uint32_t km = 0;
    for (int q = 0; q < npath; ++q)
      if (((q < in.s) ? 0 : kpath) == tid) km |= 1u << q;
    p.keep_mask[(int64_t)b * d.K + tid] = km;
  }
  (void)R1;
  if (tid == 0) {
    p.sel_k[b] = ksel;
    p.commit_len[b] = npath + (kind != 0);
    p.y_tok[b] = (kind != 0) ? y : -1;
    p.y_kind[b] = kind;
    p.path_rolled[b] = in.L - npath;
    p.branch_discarded[b] = (d.K - 1) * (in.L - in.s);
    if (p.resid_mass) p.resid_mass[b] = (kind != 0) ? (float)mass : 0.f;
    if (sh_st) atomicOr(p.status + b, sh_st);
  }

  // last CTA: offsets (exclusive scan of commit_len) and the packed commit stream
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    sh_last = (atomicAdd(p.sel_cnt, 1) == d.B - 1);
  }
  __syncthreads();
  if (!sh_last) return;
  __threadfence();
  __shared__ int wsum[NW];
  const int per = (d.B + NT - 1) / NT;
  const int b0 = min(d.B, tid * per), b1 = min(d.B, b0 + per);
  int local = 0;
  for (int q = b0; q < b1; ++q) local += __ldcg(p.commit_len + q);
  int incl = local;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int yv = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += yv;
  }
  if (lane == 31) wsum[w] = incl;
  __syncthreads();
  int run = incl - local;
  for (int q = 0; q < w; ++q) run += wsum[q];
  for (int q = b0; q < b1; ++q) {
    p.offsets[q] = run;
    const int cl = __ldcg(p.commit_len + q);
    if (p.packed_tok)
      for (int c = 0; c < cl; ++c) p.packed_tok[run + c] = __ldcg(p.out_tok + (int64_t)q * (d.G + 2) + c);
    run += cl;
  }
  if (b1 == d.B && b0 < b1) p.offsets[d.B] = run;
  if (tid == 0) {
    if (d.B <= 0) p.offsets[0] = 0;
    *p.sel_cnt = 0;
  }
}

template <typename T, int NT>
static sb_status launch_select(const SelParams& p, bool vok, cudaStream_t s) {
  k_select<T, NT><<<p.d.B, NT, 0, s>>>(p, vok);
  return cuda_status(cudaGetLastError());
}

}  // namespace sb

using namespace sb;

extern "C" sb_status sb_select_branch(const sb_dims* dd, const void* p_logits, const void* q_logits,
                                      const int32_t* tok, const float* u, const float* us,
                                      const int32_t* gamma, const int32_t* branch_pos,
                                      const int32_t* n_acc, sb_select_rule rule, int32_t* sel_k,
                                      int32_t* commit_len, int32_t* out_tok, int32_t* y_tok,
                                      int32_t* y_kind, int32_t* offsets, int32_t* packed_tok,
                                      int32_t* path_rolled, int32_t* branch_discarded,
                                      uint32_t* keep_mask, float* resid_mass, int32_t* status,
                                      void* comm, void* workspace, size_t workspace_bytes,
                                      sb_stream_t stream) {
  (void)gamma;
  (void)branch_pos;  // the clamped layout comes from the workspace (sb_verify_branches)
  if (!dims_valid(dd)) return SB_ERR_INVALID_ARG;
  if (!p_logits || !q_logits || !tok || !u || !us || !n_acc || !sel_k || !commit_len || !out_tok ||
      !y_tok || !y_kind || !offsets || !path_rolled || !branch_discarded || !keep_mask || !status ||
      !workspace)
    return SB_ERR_INVALID_ARG;
  if (rule != SB_SELECT_EQ9 && rule != SB_SELECT_ALG1) return SB_ERR_INVALID_ARG;
  if (comm) return SB_ERR_UNSUPPORTED;
  if ((uintptr_t)workspace % 256) return SB_ERR_INVALID_ARG;
  const Workspace w = carve(*dd, workspace);
  if (workspace_bytes < w.bytes) return SB_ERR_WORKSPACE;
  SelParams p;
  p.d = to_dims(dd); p.PL = p_logits; p.QL = q_logits; p.tok = tok; p.u = u; p.us = us;
  p.n_acc = n_acc; p.rule = rule; p.info = w.info; p.rowstat = w.rowstat; p.sel_cnt = w.sel_cnt;
  p.sel_k = sel_k; p.commit_len = commit_len; p.out_tok = out_tok; p.y_tok = y_tok;
  p.y_kind = y_kind; p.offsets = offsets; p.packed_tok = packed_tok; p.path_rolled = path_rolled;
  p.branch_discarded = branch_discarded; p.status = status; p.keep_mask = keep_mask;
  p.resid_mass = resid_mass;
  const bool vok = vec_ok(dd, p_logits) && vec_ok(dd, q_logits);
  cudaStream_t s = (cudaStream_t)stream;
  if (dd->dtype == SB_BF16) {
    if ((dd->V + 256 * 8 - 1) / (256 * 8) > kMaxTiles) return SB_ERR_UNSUPPORTED;
    return launch_select<__nv_bfloat16, 256>(p, vok, s);
  }
  if ((dd->V + 256 * 4 - 1) / (256 * 4) > kMaxTiles) return SB_ERR_UNSUPPORTED;
  return launch_select<float, 256>(p, vok, s);
}
