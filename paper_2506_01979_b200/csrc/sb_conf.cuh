// sb_conf.cuh — the per-row draft-confidence statistic and the (b,k) group completion
// (Eq. 6 stop, Eq. 7 k, gamma_next), shared by k_conf / k_conf_tma (sb_confidence.cu)
// and the single-launch adaptive step (k_astep, sb_verify.cu).  §4.2 P170, Eq. 6 P198,
// Eq. 7 P218; SURVEY §8.1 row a6.
#pragma once
#include "sb_common.cuh"

namespace sb {

struct ConfParams {
  Dims d;
  const void* QL;
  const int* tok;
  int mode;
  float eps, lambda;
  int k_max;
  float *top1_prob, *entropy, *tok_prob, *stat;
  int* top1_id;
  int *stop, *k_next, *gamma_next;
  int* cnt;
  float* ws_stat;
  float* ws_c;
  RowStat* qrs;  // [B][K][G] this row's reduced state (reuse by sb_verify_branches_reuse)
};

// Per-row statistic and the group-completion logic shared by both kernels.
template <typename T, typename Sync>
__device__ __forceinline__ void conf_epilogue(const ConfParams& p, int grp, int i, const T* row,
                                              const RowStat& s, int tid, int* s_last, Sync sync) {
  const Dims& d = p.d;
  const int G = d.G;
  const int b = grp / d.K, k = grp % d.K;
  const RowOut o = finish(s);
  if (tid == 0) {
    p.qrs[(int64_t)grp * G + i] = s;
    const int64_t e = (int64_t)grp * G + i;
    double top1 = CUDART_NAN, H = CUDART_NAN, tp = CUDART_NAN, st = CUDART_NAN;
    int id = -1;
    if (o.finite) {
      const double LN2 = 0.69314718055994530942;
      top1 = tok_prob(s.m, o.MS, o.Z);
      id = s.idx;
      H = LN2 * (log2((double)o.Z) - (double)s.s1 / (double)o.Z);
      if (p.tok) {
        const int x = __ldg(p.tok + ent(d, b, k, i));
        if (x >= 0 && x < d.V) tp = tok_prob(ld_scalar(row + x), o.MS, o.Z);
      }
      if (p.mode == SB_CONF_TOP1) st = top1;                  // max_x q(x)
      else if (p.mode == SB_CONF_TOKEN) st = tp;              // q(x_i)
      else st = 1.0 - sqrt((double)p.lambda * fmax(H, 0.0));  // 1 - sqrt(lambda H)
    }
    if (p.top1_prob) p.top1_prob[e] = (float)top1;
    if (p.top1_id) p.top1_id[e] = id;
    if (p.entropy) p.entropy[e] = (float)H;
    if (p.tok_prob) p.tok_prob[e] = (float)tp;
    if (p.stat) p.stat[e] = (float)st;
    p.ws_stat[e] = (float)st;
    p.ws_c[e] = (float)(p.mode == SB_CONF_TOKEN ? tp : top1);
    __threadfence();
    *s_last = (atomicAdd(p.cnt + grp, 1) == G - 1);
  }
  sync();
  if (*s_last && tid < 32) {  // the first warp: row r's statistic in lane r (G <= 31), one ballot
    __threadfence();
    float sv = 0.f, cv = 0.f;
    if (tid < G) {
      sv = __ldcg(p.ws_stat + (int64_t)grp * G + tid);
      cv = __ldcg(p.ws_c + (int64_t)grp * G + tid);
    }
    const unsigned low = __ballot_sync(0xffffffffu, tid < G && (double)sv <= (double)p.eps);  // Eq. 6: keep q(x) > eps
    const int stop = low ? __ffs(low) - 1 : G;
    const float cs = __shfl_sync(0xffffffffu, cv, stop < G ? stop : 0);
    if (tid == 0) {
      int kn = -1;
      if (stop < G) {
        const double kk = floor((double)p.k_max * (1.0 - (double)cs));  // Eq. 7
        kn = kk < 1.0 ? 1 : (int)kk;
      }
      p.stop[grp] = stop;
      if (p.k_next) p.k_next[grp] = kn;
      if (p.gamma_next) p.gamma_next[grp] = stop > 1 ? stop : 1;
      p.cnt[grp] = 0;
    }
  }
  sync();
}

}  // namespace sb
