// sb_rows.cuh — the row-pair epilogue shared by every verify kernel (k_rows_tma, k_astep,
// k_rows_warp): row outputs, the fp64 acceptance test u*Q[x] <= P[x] (P94, Alg. 1
// P534/P538), and in the warp completing a sequence its first rejection per branch
// n_k; plus the cross-CTA record loads of the persistent kernels.
#pragma once
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
  const int* seqpk;       // [B] packed layout (k_plan), read by the warp-cooperative decode
  const RowStat* qreuse;  // [B][G] slot-0 q-row states from sb_draft_confidence, or NULL
  int* cnt;
  float4* rowstat;
  uint8_t* pflag;
  float *lse_p, *lse_q, *p_tok, *q_tok, *top1_q, *entropy_q;
  int* top1_id_q;
  uint32_t* acc_mask;
  int* n_acc;
  int* status;
  int* ready;  // fused step: per-sequence "n_k known" flags (NULL otherwise)
  // adaptive single-launch step (k_astep): the sequence whose n_k is known is appended to
  // the sample queue (sq[atomicAdd(sq_ctr)] = b, then sq_pub[slot] released); NULL otherwise
  int *sq_ctr, *sq, *sq_pub;
  // vocabulary-shard partial mode (a7): write the shard's row states / token logits
  int partial, v_offset;
  ShardRow* rowpart;  // [B][K][G+1] physical rows
  float2* tokpart;    // [B][K][G+1] token slots: (p logit, q logit) if the token is in this shard
};

struct Unit {
  int b, slot, i;
  SeqInfo in;
};

// Records written by other CTAs during this launch are read through L2 (ld.global.cg):
// a line of neighbouring records may sit in this SM's L1 from before they were written.
__device__ __forceinline__ SeqInfo ldcg_seqinfo(const SeqInfo* src) {
  static_assert(sizeof(SeqInfo) == 32, "two 16-byte loads");
  const int4 a = __ldcg(reinterpret_cast<const int4*>(src)), b = __ldcg(reinterpret_cast<const int4*>(src) + 1);
  SeqInfo r;
  r.g = a.x; r.s = a.y; r.L = a.z; r.st = a.w; r.Lr = b.x;
  r.pad_[0] = b.y; r.pad_[1] = b.z; r.pad_[2] = b.w;
  return r;
}
__device__ __forceinline__ RowStat ldcg_rowstat(const RowStat* src) {
  static_assert(sizeof(RowStat) == 32, "two 16-byte loads");
  const int4 a = __ldcg(reinterpret_cast<const int4*>(src)), b = __ldcg(reinterpret_cast<const int4*>(src) + 1);
  RowStat r;
  int4 w[2] = {a, b};
  memcpy(&r, w, sizeof(r));
  return r;
}
__device__ __forceinline__ int ld_acq(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_rel(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Geometry of sequence b once gamma_b is known (k_plan's clamps, unsharded): its SeqInfo.
__device__ __forceinline__ SeqInfo astep_seqinfo(int g, int s, int G) {
  int st = 0;
  if (g > G) { g = G; st |= SB_ST_GAMMA_CLAMPED; }
  if (g < 0) { g = 0; st |= SB_ST_GAMMA_CLAMPED; }
  if (s > g) { s = g; st |= SB_ST_BRANCH_CLAMPED; }
  if (s < 0) { s = 0; st |= SB_ST_BRANCH_CLAMPED; }
  const int L = (s < g) ? g : g + 1;
  return SeqInfo{g, s, L, st, L, {0, 0, 0}};
}

// Epilogue of one unit by one warp, with the token data already prefetched.
template <typename T>
__device__ __forceinline__ void warp_epilogue(const RowsParams& p, const Unit& un, const RowStat& ps,
                                              const RowStat& qs, const T* qrow, int x, float lpx, float lqx,
                                              float uu, int64_t et) {
  const Dims& d = p.d;
  const int lane = threadIdx.x & 31;
  const int b = un.b, slot = un.slot, i = un.i;
  const SeqInfo& in = un.in;
  const RowOut po = finish(ps), qo = finish_q<T>(qs, qrow, d.V);
  const bool branch_row = (slot == 0 && i == in.s);
  const int ntok = branch_row ? d.K : 1;
  if (lane < ntok) {
    uint8_t fl = 0;
    float pt = CUDART_NAN_F, qt = CUDART_NAN_F;
    if (!(po.finite && qo.finite)) {
      fl |= st_flags(po.st | qo.st);
    } else if (x < 0 || x >= d.V) {
      fl |= 2;
    } else {
      const double Px = tok_prob(lpx, po.MS, po.Z);
      const double Qx = tok_prob(lqx, qo.MS, qo.Z);
      pt = (float)Px;
      qt = (float)Qx;
      // accept iff r <= p/q (P534, P538), as u*Q[x] <= P[x]; Q[x] = 0 accepts (S127)
      if ((double)uu * Qx <= Px) fl |= 1;
    }
    p.p_tok[et] = pt;
    p.q_tok[et] = qt;
    p.pflag[et] = fl;
  }
  if (lane == 0) {
    const int64_t e = ent(d, b, slot, i);
    const double LN2 = 0.69314718055994530942;
    p.lse_p[e] = po.finite ? (float)(((double)po.MS + log2((double)po.Z)) * LN2) : CUDART_NAN_F;
    p.lse_q[e] = qo.finite ? (float)(((double)qo.MS + log2((double)qo.Z)) * LN2) : CUDART_NAN_F;
    const bool conf_ok = po.finite && qo.finite;  // as the oracle: q stats iff both rows finite
    if (p.top1_q) p.top1_q[e] = conf_ok ? (float)tok_prob(qs.m, qo.MS, qo.Z) : CUDART_NAN_F;
    if (p.top1_id_q) p.top1_id_q[e] = conf_ok ? qs.idx : -1;
    if (p.entropy_q) {
      const double Z = qo.Z;
      p.entropy_q[e] = conf_ok ? (float)(LN2 * (log2(Z) - (double)qs.s1 / Z)) : CUDART_NAN_F;
    }
    p.rowstat[e] = make_float4(po.MS, z_store(po), qo.MS, z_store(qo));
  }
  __syncwarp();
  int last = 0;
  if (lane == 0) {
    __threadfence();
    // phase-1 row pairs of b (the fused unit list also interleaves sample units)
    const int units_b = in.Lr + (d.K - 1) * (in.Lr - 1 - in.s);
    last = (atomicAdd(p.cnt + b, 1) == units_b - 1);
  }
  last = __shfl_sync(0xffffffffu, last, 0);
  if (!last) return;
  __threadfence();
  // first rejection per branch: lane r holds row r's flags for every branch (loads
  // issued back to back), then one ballot per branch
  uint32_t fw[4] = {0u, 0u, 0u, 0u};  // 4 flag bits per branch, 8 branches per word
  if (lane < in.L) {
#pragma unroll 8
    for (int k = 0; k < d.K; ++k) {
      const uint32_t f = __ldcg(p.pflag + ent(d, b, (lane < in.s) ? 0 : k, lane));
      fw[k / 8] |= (f & 15u) << (4 * (k % 8));
    }
  }
  const uint32_t rowmask = in.L >= 32 ? 0xffffffffu : ((1u << in.L) - 1u);
  uint32_t anyf = 0;
  for (int k = 0; k < d.K; ++k) {
    const uint32_t f = (fw[k / 8] >> (4 * (k % 8))) & 15u;
    const uint32_t mask = __ballot_sync(0xffffffffu, f & 1u) & rowmask;
    anyf |= f;
    if (lane == 0) {
      const uint32_t rej = ~mask & rowmask;
      p.acc_mask[(int64_t)b * d.K + k] = mask;
      p.n_acc[(int64_t)b * d.K + k] = rej ? (__ffs(rej) - 1) : in.L;
    }
  }
  anyf = __reduce_or_sync(0xffffffffu, anyf);
  // sentinels for entries no tested path touches
  const int R1 = d.G + 1;
  for (int q = lane; q < d.K * R1; q += 32) {
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
  if (lane == 0) {
    p.status[b] = in.st | flags_st(anyf);
    p.cnt[b] = 0;  // leave the workspace re-usable
    if (p.ready) {  // fused step: the sequence's sample unit may start
      __threadfence();
      asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p.ready + b), "r"(1) : "memory");
    }
    if (p.sq) {  // adaptive single-launch step: queue the sequence's sample item
      const int slot = atomicAdd(p.sq_ctr, 1);
      p.sq[slot] = b;
      __threadfence();
      asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p.sq_pub + slot), "r"(1) : "memory");
    }
  }
}

// Outputs of sb_select_branch (include/specbranch.h).
struct CommitOut {
  int *sel_k, *commit_len, *out_tok, *y_tok, *y_kind, *offsets, *packed_tok, *path_rolled, *branch_discarded;
  uint32_t* keep_mask;
  float* resid_mass;
};

// Commit of sequence b (SURVEY §8.0 "Commit"; P94, P237, P541-555, rollback P655): the
// kept path k*'s tokens for rows 0..npath-1 (slot 0 before the branch row), then y if
// kind != 0; keep mask per slot, rollback counters (P317 / P734).  One warp.
__device__ __forceinline__ void commit_seq(const Dims& d, const int* tok, int* status, const CommitOut& co, int b,
                                           const SeqInfo& in, int ksel, int npath, int kind, int y, double mass,
                                           int st) {
  const int lane = threadIdx.x & 31, G = d.G;
  const int kpath = ksel < 0 ? 0 : ksel;
  int* out = co.out_tok + (int64_t)b * (G + 2);
  for (int qq = lane; qq < G + 2; qq += 32) {
    int v = -1;
    if (qq < npath) v = __ldg(tok + ent(d, b, (qq < in.s) ? 0 : kpath, qq));
    else if (qq == npath && kind != 0) v = y;
    out[qq] = v;
  }
  if (lane < d.K) {
    uint32_t km = 0;
    for (int qq = 0; qq < npath; ++qq)
      if (((qq < in.s) ? 0 : kpath) == lane) km |= 1u << qq;
    co.keep_mask[(int64_t)b * d.K + lane] = km;
  }
  if (lane == 0) {
    co.sel_k[b] = ksel;
    co.commit_len[b] = npath + (kind != 0);
    co.y_tok[b] = (kind != 0) ? y : -1;
    co.y_kind[b] = kind;
    co.path_rolled[b] = in.L - npath;
    co.branch_discarded[b] = (d.K - 1) * (in.L - in.s);
    if (co.resid_mass) co.resid_mass[b] = (kind != 0) ? (float)mass : 0.f;
    if (st) atomicOr(status + b, st);
  }
}

}  // namespace sb
