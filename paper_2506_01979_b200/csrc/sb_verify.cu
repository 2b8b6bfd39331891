// sb_verify.cu — sb_verify_branches: one streaming pass over every tested (p,q) row
// pair, fused with the acceptance test and, in the last CTA of each sequence, the
// first-rejection scan (SURVEY §8.1 rows a1 + a2; PAPER §3 P94, Alg. 1 P523-538).
//
// Kernels
//   k_plan  (1 CTA)       clamp gamma_b / s_b, L_b, tested row pairs per sequence,
//                         exclusive scan -> unit offsets.
//   k_rows  (persistent)  one unit = one physical row pair (p row, q row) of V logits,
//                         streamed once with 16-byte loads, 2 x U loads in flight per
//                         thread; online max / sum / entropy / top-1 in registers, one
//                         block reduction, then the row's path tokens: P[x], Q[x] in
//                         fp64 and acc = u*Q[x] <= P[x].  The CTA that completes a
//                         sequence (per-sequence counter) builds acc_mask, n_acc,
//                         status and the sentinels of untested entries.
#include <algorithm>
#include <cstdio>

#include "sb_host.h"

namespace sb {

struct RowsParams {
  Dims d;
  const void* PL;
  const void* QL;
  const int* tok;
  const float* u;
  const SeqInfo* info;
  const int* unit_off;
  int* cnt;
  float4* rowstat;
  uint8_t* pflag;
  float *lse_p, *lse_q, *p_tok, *q_tok, *top1_q, *entropy_q;
  int* top1_id_q;
  uint32_t* acc_mask;
  int* n_acc;
  int* status;
};

// ---------------------------------------------------------------- plan
__global__ void __launch_bounds__(1024) k_plan(Dims d, const int* __restrict__ gamma,
                                               const int* __restrict__ bpos, SeqInfo* info,
                                               int* unit_off) {
  __shared__ int wsum[32];
  const int tid = threadIdx.x, NT = blockDim.x;
  const int per = (d.B + NT - 1) / NT;
  const int b0 = min(d.B, tid * per), b1 = min(d.B, b0 + per);
  int local = 0;
  for (int b = b0; b < b1; ++b) {
    int st = 0;
    int g = gamma ? gamma[b] : d.G;
    if (g > d.G) { g = d.G; st |= SB_ST_GAMMA_CLAMPED; }
    if (g < 0) { g = 0; st |= SB_ST_GAMMA_CLAMPED; }
    int s = bpos ? bpos[b] : 0;
    if (s > g) { s = g; st |= SB_ST_BRANCH_CLAMPED; }
    if (s < 0) { s = 0; st |= SB_ST_BRANCH_CLAMPED; }
    const int L = (s < g) ? g : g + 1;
    info[b] = SeqInfo{g, s, L, st};
    local += L + (d.K - 1) * (L - 1 - s);  // slot 0: rows 0..L-1; slots k>0: s+1..L-1
  }
  // block exclusive scan of the per-thread sums
  const int lane = tid & 31, w = tid >> 5;
  int incl = local;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) wsum[w] = incl;
  __syncthreads();
  if (w == 0) {
    int x = (lane < NT / 32) ? wsum[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    wsum[lane] = x;  // inclusive over warps
  }
  __syncthreads();
  int run = incl - local + (w > 0 ? wsum[w - 1] : 0);
  for (int b = b0; b < b1; ++b) {
    unit_off[b] = run;
    const SeqInfo in = info[b];
    run += in.L + (d.K - 1) * (in.L - 1 - in.s);
  }
  if (tid == NT - 1) unit_off[d.B] = run;
}

// ---------------------------------------------------------------- rows
template <typename T, int NT, int U>
__global__ void __launch_bounds__(NT) k_rows(RowsParams p, bool vec_ok) {
  constexpr int NA = 4;
  __shared__ RowStat red[NT / 32];
  __shared__ int s_last;
  __shared__ int s_st;
  const Dims& d = p.d;
  const int tid = threadIdx.x;
  const int total = __ldg(p.unit_off + d.B);
  const T* PL = static_cast<const T*>(p.PL);
  const T* QL = static_cast<const T*>(p.QL);

  for (int unit = blockIdx.x; unit < total; unit += gridDim.x) {
    // unit -> sequence (upper bound search over the offsets), then (slot, row)
    int lo = 0, hi = d.B;  // find largest b with unit_off[b] <= unit
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (__ldg(p.unit_off + mid) <= unit) lo = mid; else hi = mid;
    }
    const int b = lo;
    const SeqInfo in = p.info[b];
    const int j = unit - __ldg(p.unit_off + b);
    int slot, i;
    if (j < in.L) {
      slot = 0; i = j;
    } else {
      const int per = in.L - 1 - in.s, jj = j - in.L;
      slot = 1 + jj / per;
      i = in.s + 1 + jj % per;
    }
    const T* prow = PL + row_off(d, b, slot, i);
    const T* qrow = QL + row_off(d, b, slot, i);

    RowAcc<false, NA> pa;
    RowAcc<true, NA> qa;
    pa.init();
    qa.init();
    stream_pair<T, NA, NT, U>(prow, qrow, d.V, vec_ok, pa, qa);
    const RowStat ps = block_reduce<NT>(fold(pa), red);
    const RowStat qs = block_reduce<NT>(fold(qa), red);
    const RowOut po = finish(ps), qo = finish(qs);

    // path tokens through this row: K branch tokens at the branch row, else one
    const bool branch_row = (slot == 0 && i == in.s);
    const int ntok = branch_row ? d.K : 1;
    if (tid < ntok) {
      const int ts = branch_row ? tid : slot;
      const int64_t e = ent(d, b, ts, i);
      const int x = __ldg(p.tok + e);
      uint8_t fl = 0;
      float pt = CUDART_NAN_F, qt = CUDART_NAN_F;
      if (!(po.finite && qo.finite)) {
        fl |= 4;
      } else if (x < 0 || x >= d.V) {
        fl |= 2;
      } else {
        const double Px = tok_prob(ld_scalar(prow + x), po.MS, po.Z);
        const double Qx = tok_prob(ld_scalar(qrow + x), qo.MS, qo.Z);
        pt = (float)Px;
        qt = (float)Qx;
        // accept iff r <= p/q (P534, P538), as u*Q[x] <= P[x]; Q[x] = 0 accepts (S127)
        if ((double)__ldg(p.u + e) * Qx <= Px) fl |= 1;
      }
      p.p_tok[e] = pt;
      p.q_tok[e] = qt;
      p.pflag[e] = fl;
    }
    if (tid == 0) {
      const int64_t e = ent(d, b, slot, i);
      const double LN2 = 0.69314718055994530942;
      p.lse_p[e] = po.finite ? (float)(((double)po.MS + log2((double)po.Z)) * LN2) : CUDART_NAN_F;
      p.lse_q[e] = qo.finite ? (float)(((double)qo.MS + log2((double)qo.Z)) * LN2) : CUDART_NAN_F;
      const bool conf_ok = po.finite && qo.finite;  // as the oracle: q stats iff both rows finite
      if (p.top1_q)
        p.top1_q[e] = conf_ok ? (float)tok_prob(qs.m, qo.MS, qo.Z) : CUDART_NAN_F;
      if (p.top1_id_q) p.top1_id_q[e] = conf_ok ? qs.idx : -1;
      if (p.entropy_q) {
        const double Z = qo.Z;
        p.entropy_q[e] = conf_ok ? (float)(LN2 * (log2(Z) - (double)qs.s1 / Z)) : CUDART_NAN_F;
      }
      p.rowstat[e] = make_float4(po.MS, po.finite ? po.Z : CUDART_NAN_F, qo.MS,
                                 qo.finite ? qo.Z : CUDART_NAN_F);
    }

    // completion: the CTA finishing the sequence decides n_k (ballot/ffs over rows)
    __syncthreads();
    if (tid == 0) {
      __threadfence();
      const int units_b = __ldg(p.unit_off + b + 1) - __ldg(p.unit_off + b);
      const int prev = atomicAdd(p.cnt + b, 1);
      s_last = (prev == units_b - 1);
      s_st = in.st;
    }
    __syncthreads();
    if (s_last) {
      __threadfence();
      const int R1 = d.G + 1;
      if (tid < d.K) {
        const int k = tid;
        uint32_t mask = 0;
        int st = 0;
        for (int r = 0; r < in.L; ++r) {
          const int ts = (r < in.s) ? 0 : k;
          const uint8_t fl = __ldcg(p.pflag + ent(d, b, ts, r));
          if (fl & 1) mask |= 1u << r;
          if (fl & 2) st |= SB_ST_BAD_TOKEN;
          if (fl & 4) st |= SB_ST_NONFINITE;
        }
        const uint32_t rej = ~mask & (in.L >= 32 ? 0xffffffffu : ((1u << in.L) - 1));
        p.acc_mask[(int64_t)b * d.K + k] = mask;
        p.n_acc[(int64_t)b * d.K + k] = rej ? (__ffs(rej) - 1) : in.L;
        if (st) atomicOr(&s_st, st);
      }
      // sentinels for entries no tested path touches
      for (int q = tid; q < d.K * R1; q += NT) {
        const int k = q / R1, r = q % R1;
        const int64_t e = ent(d, b, k, r);
        const bool phys = (k == 0) ? (r < in.L) : (r > in.s && r < in.L);
        const bool path = (k == 0) ? (r < in.L) : (r >= in.s && r < in.L);
        if (!phys) {
          p.lse_p[e] = CUDART_NAN_F;
          p.lse_q[e] = CUDART_NAN_F;
          if (p.top1_q) p.top1_q[e] = CUDART_NAN_F;
          if (p.top1_id_q) p.top1_id_q[e] = -1;
          if (p.entropy_q) p.entropy_q[e] = CUDART_NAN_F;
        }
        if (!path) {
          p.p_tok[e] = CUDART_NAN_F;
          p.q_tok[e] = CUDART_NAN_F;
        }
      }
      __syncthreads();
      if (tid == 0) {
        p.status[b] = s_st;
        p.cnt[b] = 0;  // leave the workspace re-usable
      }
    }
  }
}

template <typename T, int NT, int U>
static sb_status launch_rows(const RowsParams& p, bool vok, cudaStream_t s) {
  static int grid_cache[2] = {0, 0};
  int& g = grid_cache[std::is_same<T, float>::value ? 1 : 0];
  if (g == 0) {
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_rows<T, NT, U>, NT, 0);
    g = std::max(1, occ) * num_sms();
  }
  const int64_t max_units = (int64_t)p.d.B * p.d.K * (p.d.G + 1);
  const int grid = (int)std::min<int64_t>(g, max_units);
  k_rows<T, NT, U><<<grid, NT, 0, s>>>(p, vok);
  return cuda_status(cudaGetLastError());
}

}  // namespace sb

using namespace sb;

extern "C" sb_status sb_verify_branches(const sb_dims* dd, const void* p_logits,
                                        const void* q_logits, const int32_t* tok, const float* u,
                                        const int32_t* gamma, const int32_t* branch_pos,
                                        float* lse_p, float* lse_q, float* p_tok, float* q_tok,
                                        uint32_t* acc_mask, int32_t* n_acc, float* top1_q,
                                        int32_t* top1_id_q, float* entropy_q, int32_t* status,
                                        void* comm, void* workspace, size_t workspace_bytes,
                                        sb_stream_t stream) {
  if (!dims_valid(dd)) return SB_ERR_INVALID_ARG;
  if (!p_logits || !q_logits || !tok || !u || !lse_p || !lse_q || !p_tok || !q_tok || !acc_mask ||
      !n_acc || !status || !workspace)
    return SB_ERR_INVALID_ARG;
  if (comm) return SB_ERR_UNSUPPORTED;
  if ((uintptr_t)workspace % 256) return SB_ERR_INVALID_ARG;
  const Workspace w = carve(*dd, workspace);
  if (workspace_bytes < w.bytes) return SB_ERR_WORKSPACE;
  const Dims d = to_dims(dd);
  cudaStream_t s = (cudaStream_t)stream;

  k_plan<<<1, 1024, 0, s>>>(d, gamma, branch_pos, w.info, w.unit_off);
  if (cudaGetLastError() != cudaSuccess) return SB_ERR_CUDA;

  RowsParams p;
  p.d = d; p.PL = p_logits; p.QL = q_logits; p.tok = tok; p.u = u;
  p.info = w.info; p.unit_off = w.unit_off; p.cnt = w.cnt; p.rowstat = w.rowstat; p.pflag = w.pflag;
  p.lse_p = lse_p; p.lse_q = lse_q; p.p_tok = p_tok; p.q_tok = q_tok;
  p.top1_q = top1_q; p.entropy_q = entropy_q; p.top1_id_q = top1_id_q;
  p.acc_mask = acc_mask; p.n_acc = n_acc; p.status = status;
  const bool vok = vec_ok(dd, p_logits) && vec_ok(dd, q_logits);
  const size_t row_bytes = (size_t)dd->V * elem_size(dd);
  if (dd->dtype == SB_BF16) {
    return row_bytes <= 131072 ? launch_rows<__nv_bfloat16, 128, 4>(p, vok, s)
                               : launch_rows<__nv_bfloat16, 256, 4>(p, vok, s);
  }
  return row_bytes <= 131072 ? launch_rows<float, 128, 4>(p, vok, s)
                             : launch_rows<float, 256, 4>(p, vok, s);
}
