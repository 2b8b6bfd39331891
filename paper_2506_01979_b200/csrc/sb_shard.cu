// sb_shard.cu — vocabulary-sharded verify-and-branch.
//
// Rank g holds the contiguous vocabulary slice [v_offset, v_offset + V) of v_total,
// slices in rank order, so the global inverse-CDF order (ascending id) is rank order.
// Every rank sees the same tokens, uniforms, gamma and branch rows.  Split phases:
//
//   verify  : sb_shard_verify_local   k_plan (+ bonus rows) + k_rows_tma in partial mode:
//                                     per physical row the shard's (m, ms, Z) of p and
//                                     (m, ms, Z, S1, first argmax) of q, and per path
//                                     token its two logits if the token is in the shard;
//             [exchange 1: all-gather of the partials, 40 B per row entry per rank]
//             sb_shard_verify_combine k_shard_combine: rank-order combine -> the same row
//                                     states, token probabilities, accept bits, n_k and
//                                     status on every rank (decisions replicated).
//   select  : sb_shard_select_local   k_shard_select_local: Eq. 9 / Alg. 1 decision
//                                     (replicated), this shard's residual (and p) mass
//                                     and 512-byte segment sums of the sampled row;
//             [exchange 2: all-gather of (R_g, P_g), 16 B per sequence per rank]
//             sb_shard_select_sample  k_shard_sample: R = sum_g R_g in rank order,
//                                     t = us R, the owner shard locates t in its segments,
//                                     re-reads one segment -> global id; others -1;
//             [exchange 3: all-reduce MAX of the candidate token, 4 B per sequence]
//             sb_shard_select_commit  k_shard_commit: commit / rollback outputs.
//
// With a library communicator (sb_comm_create, NCCL) sb_verify_branches and
// sb_select_branch run these phases with ncclAllGather / ncclAllReduce in between.
#include <nccl.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "sb_host.h"

namespace sb {

struct ShardCombineParams {
  Dims d;
  int nranks, v_total;
  const char* gathered;    // nranks rank blocks of sb_shard_partial_bytes, rank order
  size_t rank_bytes;       // bytes of one rank block
  size_t tok_off;          // offset of the token part inside a rank block
  const int* tok;
  const float* u;
  const SeqInfo* info;
  float4* rowstat;
  uint8_t* pflag;
  float* tok_lp;
  float *lse_p, *lse_q, *p_tok, *q_tok, *top1_q, *entropy_q;
  int* top1_id_q;
  uint32_t* acc_mask;
  int* n_acc;
  int* status;
};

// one warp per sequence
__global__ void __launch_bounds__(128) k_shard_combine(ShardCombineParams p) {
  const Dims& d = p.d;
  const int lane = threadIdx.x & 31;
  const int b = blockIdx.x * 4 + (threadIdx.x >> 5);
  if (b >= d.B) return;
  const SeqInfo in = p.info[b];
  const int R1 = d.G + 1;
  const double LN2 = 0.69314718055994530942;
  // ---- physical rows: combine the shard states in rank order
  for (int q = lane; q < d.K * R1; q += 32) {
    const int k = q / R1, r = q % R1;
    const int64_t e = ent(d, b, k, r);
    const bool read = (k == 0) ? (r < in.Lr) : (r > in.s && r < in.Lr);
    const bool tested = (k == 0) ? (r < in.L) : (r > in.s && r < in.L);
    if (read) {
      RowStat P = rowstat_empty(), Q = rowstat_empty();
      int qfin = 0;
      for (int g = 0; g < p.nranks; ++g) {
        const ShardRow sr = reinterpret_cast<const ShardRow*>(p.gathered + g * p.rank_bytes)[e];
        RowStat a, c;
        a.m = sr.pm; a.ms = sr.pms; a.z = sr.pz; a.s1 = 0.0; a.idx = 0;
        c.m = sr.qm; c.ms = sr.qms; c.z = sr.qz; c.s1 = sr.qs1; c.idx = sr.qidx;
        qfin |= sr.qfin;
        P = combine(P, a);
        Q = combine(Q, c);
      }
      const RowOut po = finish(P);
      RowOut qo = finish(Q);
      if (d.dtype == SB_BF16 && Q.m == kMaskedLogit && !qfin) qo.st = SB_ST_NONFINITE;  // all -inf (finish_q)
      p.rowstat[e] = make_float4(po.MS, z_store(po), qo.MS, z_store(qo));
      if (tested) {
        p.lse_p[e] = po.finite ? (float)(((double)po.MS + log2((double)po.Z)) * LN2) : CUDART_NAN_F;
        p.lse_q[e] = qo.finite ? (float)(((double)qo.MS + log2((double)qo.Z)) * LN2) : CUDART_NAN_F;
        const bool ok = po.finite && qo.finite;
        if (p.top1_q) p.top1_q[e] = ok ? (float)tok_prob(Q.m, qo.MS, qo.Z) : CUDART_NAN_F;
        if (p.top1_id_q) p.top1_id_q[e] = ok ? Q.idx : -1;
        if (p.entropy_q) {
          const double Z = qo.Z;
          p.entropy_q[e] = ok ? (float)(LN2 * (log2(Z) - (double)Q.s1 / Z)) : CUDART_NAN_F;
        }
      }
    }
    if (!tested) {
      p.lse_p[e] = CUDART_NAN_F;
      p.lse_q[e] = CUDART_NAN_F;
      if (p.top1_q) p.top1_q[e] = CUDART_NAN_F;
      if (p.top1_id_q) p.top1_id_q[e] = -1;
      if (p.entropy_q) p.entropy_q[e] = CUDART_NAN_F;
    }
  }
  __syncwarp();
  __threadfence_block();
  // ---- path tokens: the owner shard's logits, fp64 probabilities, accept bits
  for (int q = lane; q < d.K * R1; q += 32) {
    const int k = q / R1, r = q % R1;
    const int64_t e = ent(d, b, k, r);
    const bool path = (k == 0) ? (r < in.L) : (r >= in.s && r < in.L);
    if (!path) {
      p.p_tok[e] = CUDART_NAN_F;
      p.q_tok[e] = CUDART_NAN_F;
      p.tok_lp[e] = CUDART_NAN_F;
      continue;
    }
    const int x = __ldg(p.tok + e);
    uint8_t fl = 0;
    float pt = CUDART_NAN_F, qt = CUDART_NAN_F, key = CUDART_NAN_F;
    const float4 rs = p.rowstat[ent(d, b, (r <= in.s) ? 0 : k, r)];
    const int cls = z_class(rs.y) | z_class(rs.w);
    if (cls) {
      fl |= st_flags(cls);
    } else if (x < 0 || x >= p.v_total) {
      fl |= 2;
    } else {
      float lpx = -CUDART_INF_F, lqx = -CUDART_INF_F;
      for (int g = 0; g < p.nranks; ++g) {  // exactly one shard owns x
        const float2 t = reinterpret_cast<const float2*>(p.gathered + g * p.rank_bytes + p.tok_off)[e];
        lpx = fmaxf(lpx, t.x);
        lqx = fmaxf(lqx, t.y);
      }
      const double Px = tok_prob(lpx, rs.x, rs.y), Qx = tok_prob(lqx, rs.z, rs.w);
      pt = (float)Px;
      qt = (float)Qx;
      key = lpx;
      // accept iff r <= p/q (P534, P538), as u*Q[x] <= P[x]; Q[x] = 0 accepts (S127)
      if ((double)__ldg(p.u + e) * Qx <= Px) fl |= 1;
    }
    p.p_tok[e] = pt;
    p.q_tok[e] = qt;
    p.tok_lp[e] = key;
    p.pflag[e] = fl;
  }
  __syncwarp();
  __threadfence_block();
  // ---- first rejection per branch
  uint32_t anyf = 0;
  const uint32_t rowmask = in.L >= 32 ? 0xffffffffu : ((1u << in.L) - 1u);
  for (int k = 0; k < d.K; ++k) {
    const uint32_t f = (lane < in.L) ? p.pflag[ent(d, b, (lane < in.s) ? 0 : k, lane)] : 0u;
    const uint32_t mask = __ballot_sync(0xffffffffu, f & 1u) & rowmask;
    anyf |= f;
    if (lane == 0) {
      const uint32_t rej = ~mask & rowmask;
      p.acc_mask[(int64_t)b * d.K + k] = mask;
      p.n_acc[(int64_t)b * d.K + k] = rej ? (__ffs(rej) - 1) : in.L;
    }
  }
  anyf = __reduce_or_sync(0xffffffffu, anyf);
  if (lane == 0) p.status[b] = in.st | flags_st(anyf);
}

// ---------------------------------------------------------------- select, local
struct ShardSelParams {
  Dims d;
  int v_offset, v_total, rule, nseg;
  bool vec;  // 16-byte aligned rows: vector loads (else scalar)
  const void* PL;
  const void* QL;
  const int* tok;
  const float* u;
  const float* us;
  const int* n_acc;
  const SeqInfo* info;
  const float4* rowstat;
  const float* tok_lp;
  int4* dec;     // [B] (ksel, npath, kind, row | slot << 16), [B + b] (mass bits, status, 0, 0)
  float* segs;   // [B][2][nseg]
  double2* mass; // [B] this shard's (R_g, P_g)
  const double2* gmass;  // [nranks][B]
  int nranks, rank;
  int* ycand;
};

template <typename T>
__device__ __forceinline__ void seg_values(const T* prow, const T* qrow, uint32_t row_bytes, int sI,
                                           bool resid, float MSp, float iZp, float MSq, float iZq, float* r,
                                           bool vec) {
  constexpr int E = Vec<T>::E;
  const int lane = threadIdx.x & 31;
  const uint32_t off = (uint32_t)sI * 512 + lane * 16;
  uint4 vp = sizeof(T) == 2 ? make_uint4(0xff80ff80u, 0xff80ff80u, 0xff80ff80u, 0xff80ff80u)
                            : make_uint4(0xff800000u, 0xff800000u, 0xff800000u, 0xff800000u);
  uint4 vq = vp;
  float lp[E], lq[E];
  if (vec && off + 16 <= row_bytes) {
    vp = __ldg(reinterpret_cast<const uint4*>(reinterpret_cast<const char*>(prow) + off));
    if (resid) vq = __ldg(reinterpret_cast<const uint4*>(reinterpret_cast<const char*>(qrow) + off));
    Vec<T>::unpack(vp, lp);
    Vec<T>::unpack(vq, lq);
  } else {  // unaligned rows, or the ragged end of a shard row: scalar, -inf past V
    const int v0 = (int)(off / sizeof(T)), V = (int)(row_bytes / sizeof(T));
#pragma unroll
    for (int e = 0; e < E; ++e) {
      lp[e] = v0 + e < V ? ld_scalar(prow + v0 + e) : -CUDART_INF_F;
      lq[e] = (resid && v0 + e < V) ? ld_scalar(qrow + v0 + e) : -CUDART_INF_F;
    }
  }
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const float P = __fmul_rn(ex2(__fmaf_rn(lp[e], kC, -MSp)), iZp);
    if (resid) {
      const float Q = __fmul_rn(ex2(__fmaf_rn(lq[e], kC, -MSq)), iZq);
      r[e] = fmaxf(__fsub_rn(P, Q), 0.f);
    } else {
      r[e] = P;
    }
  }
}

__device__ __forceinline__ float warp_scan_rn2(float x) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const float y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x = __fadd_rn(x, y);
  }
  return x;
}

template <int E>
__device__ __forceinline__ float seq_sum_rn(const float* r) {
  float s = 0.f;
#pragma unroll
  for (int e = 0; e < E; ++e) s = __fadd_rn(s, r[e]);
  return s;
}

// one CTA (8 warps) per sequence
template <typename T>
__global__ void __launch_bounds__(256) k_shard_select_local(ShardSelParams p) {
  constexpr int E = Vec<T>::E;
  __shared__ int4 sdec;
  __shared__ float4 srs;
  const Dims& d = p.d;
  const int b = blockIdx.x, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const SeqInfo in = p.info[b];
  if (tid == 0) {
    int ksel = -1, besttok = 0;
    float bestkey = 0.f;
    for (int k = 0; k < d.K; ++k) {
      if (__ldg(p.n_acc + (int64_t)b * d.K + k) <= in.s) continue;  // A = {k : n_k > s_b}
      const int64_t e = ent(d, b, k, in.s);
      const int xk = __ldg(p.tok + e);
      const float key = (p.rule == SB_SELECT_ALG1) ? __ldg(p.u + e) : p.tok_lp[e];  // raw target logit
      bool better;
      if (ksel < 0) better = true;
      else if (p.rule == SB_SELECT_ALG1) better = key > bestkey;
      else better = key > bestkey || (key == bestkey && xk < besttok);
      if (better) { ksel = k; bestkey = key; besttok = xk; }
    }
    int npath, kind, row = 0, slot = 0;
    if (ksel < 0) {
      npath = min(__ldg(p.n_acc + (int64_t)b * d.K), in.s);
      kind = 1; row = npath; slot = 0;
    } else {
      npath = __ldg(p.n_acc + (int64_t)b * d.K + ksel);
      if (npath < in.L) { kind = 1; row = npath; slot = (npath <= in.s) ? 0 : ksel; }
      else if (in.s < in.g) { kind = 2; row = in.g; slot = ksel; }
      else kind = 0;
    }
    sdec = make_int4(ksel, npath, kind, row | (slot << 16));
    p.dec[b] = sdec;
    srs = kind ? p.rowstat[ent(d, b, slot, row)] : make_float4(0.f, 1.f, 0.f, 1.f);
  }
  __syncthreads();
  const int4 D = sdec;
  const int kind = D.z;
  const float4 rs = srs;
  const bool ok = (z_class(rs.y) | (kind == 1 ? z_class(rs.w) : 0)) == 0;  // a bonus reads p only
  if (kind == 0 || !ok) {
    if (tid == 0) p.mass[b] = make_double2(0.0, 0.0);
    return;
  }
  const int row = D.w & 0xffff, slot = D.w >> 16;
  const T* prow = static_cast<const T*>(p.PL) + row_off(d, b, slot, row);
  const T* qrow = static_cast<const T*>(p.QL) + row_off(d, b, slot, row);
  const uint32_t row_bytes = (uint32_t)d.V * sizeof(T);
  const float iZp = 1.f / rs.y, iZq = 1.f / rs.w;
  float* segR = p.segs + (int64_t)b * 2 * p.nseg;
  float* segP = segR + p.nseg;
  for (int sI = warp; sI < p.nseg; sI += 8) {
    float r[E];
    if (kind == 1) {
      seg_values<T>(prow, qrow, row_bytes, sI, true, rs.x, iZp, rs.z, iZq, r, p.vec);
      const float incl = warp_scan_rn2(seq_sum_rn<E>(r));
      if (lane == 31) segR[sI] = incl;
    } else if (lane == 31) {
      segR[sI] = 0.f;
    }
    seg_values<T>(prow, qrow, row_bytes, sI, false, rs.x, iZp, rs.z, iZq, r, p.vec);
    const float inclp = warp_scan_rn2(seq_sum_rn<E>(r));
    if (lane == 31) segP[sI] = inclp;
  }
  __syncthreads();
  if (tid == 0) {
    double R = 0.0, Pm = 0.0;
    for (int sI = 0; sI < p.nseg; ++sI) {
      R += (double)segR[sI];
      Pm += (double)segP[sI];
    }
    p.mass[b] = make_double2(R, Pm);
  }
}

// one warp per sequence: owner shard locates t = us * R and picks the token
template <typename T>
__global__ void __launch_bounds__(128) k_shard_sample(ShardSelParams p) {
  constexpr int E = Vec<T>::E;
  const Dims& d = p.d;
  const int lane = threadIdx.x & 31;
  const int b = blockIdx.x * 4 + (threadIdx.x >> 5);
  if (b >= d.B) return;
  const int4 D = p.dec[b];
  int kind = D.z, st = 0;
  int y = -1;
  double mass = 0.0;
  const float4 rs = kind ? p.rowstat[ent(d, b, D.w >> 16, D.w & 0xffff)] : make_float4(0.f, 1.f, 0.f, 1.f);
  const int cls = kind ? (z_class(rs.y) | (kind == 1 ? z_class(rs.w) : 0)) : 0;  // a bonus reads p only
  if (cls) {
    kind = 0;
    st |= cls;
  }
  if (kind != 0) {
    bool resid = (kind == 1);
    double Rt = 0.0;
    for (int g = 0; g < p.nranks; ++g) Rt += resid ? p.gmass[g * d.B + b].x : p.gmass[g * d.B + b].y;
    if (resid && Rt == 0.0) {  // "no residual mass" (S134-140): sample from p
      resid = false;
      st |= SB_ST_ZERO_RESID;
      for (int g = 0; g < p.nranks; ++g) Rt += p.gmass[g * d.B + b].y;
    }
    mass = Rt;
    const double t = (double)__ldg(p.us + b) * Rt;
    int owner = -1, lastpos = -1;
    double F = 0.0, Fprev = 0.0;
    for (int g = 0; g < p.nranks; ++g) {
      const double m = resid ? p.gmass[g * d.B + b].x : p.gmass[g * d.B + b].y;
      if (m > 0.0) lastpos = g;
      if (owner < 0 && F + m > t) { owner = g; Fprev = F; }
      F += m;
    }
    double trem = t - Fprev;
    if (owner < 0) { owner = lastpos; trem = CUDART_INF; }
    if (owner == p.rank) {
      const float* seg = p.segs + (int64_t)b * 2 * p.nseg + (resid ? 0 : p.nseg);
      const int per = (p.nseg + 31) / 32;
      double local = 0.0;
      for (int j = 0; j < per; ++j) {
        const int sI = lane * per + j;
        if (sI < p.nseg) local += (double)seg[sI];
      }
      double incl = local;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const double yv = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += yv;
      }
      double excl = __shfl_up_sync(0xffffffffu, incl, 1);
      if (lane == 0) excl = 0.0;
      int found = -1, lastseg = -1;
      double Fp = 0.0;
      const bool mine = (excl <= trem && incl > trem);
      {
        double Fs = excl;
        for (int j = 0; j < per; ++j) {
          const int sI = lane * per + j;
          if (sI >= p.nseg) break;
          if (seg[sI] > 0.f) lastseg = sI;
          if (mine && found < 0 && Fs + (double)seg[sI] > trem) { found = sI; Fp = Fs; }
          Fs += (double)seg[sI];
        }
      }
      const unsigned who = __ballot_sync(0xffffffffu, found >= 0);
      int sStar;
      double tr;
      if (who) {
        const int src = __ffs(who) - 1;
        sStar = __shfl_sync(0xffffffffu, found, src);
        tr = trem - __shfl_sync(0xffffffffu, Fp, src);
      } else {
        sStar = (int)__reduce_max_sync(0xffffffffu, (unsigned)(lastseg + 1)) - 1;
        tr = CUDART_INF;
      }
      if (sStar >= 0) {
        const int row = D.w & 0xffff, slot = D.w >> 16;
        const T* prow = static_cast<const T*>(p.PL) + row_off(d, b, slot, row);
        const T* qrow = static_cast<const T*>(p.QL) + row_off(d, b, slot, row);
        float r[E];
        seg_values<T>(prow, qrow, (uint32_t)d.V * sizeof(T), sStar, resid, rs.x, 1.f / rs.y, rs.z,
                      1.f / rs.w, r, p.vec);
        const float inc = warp_scan_rn2(seq_sum_rn<E>(r));
        float Fv = __shfl_up_sync(0xffffffffu, inc, 1);
        if (lane == 0) Fv = 0.f;
        int cand = 0x7fffffff, lastv = -1;
        const int vbase = sStar * (512 / (int)sizeof(T)) + lane * E;
#pragma unroll
        for (int e = 0; e < E; ++e) {
          Fv = __fadd_rn(Fv, r[e]);
          if (cand == 0x7fffffff && (double)Fv > tr && r[e] > 0.f) cand = vbase + e;
          if (r[e] > 0.f) lastv = vbase + e;
        }
        const int pick = (int)__reduce_min_sync(0xffffffffu, (unsigned)cand);
        const int loc = (pick != 0x7fffffff) ? pick : (int)__reduce_max_sync(0xffffffffu, (unsigned)(lastv + 1)) - 1;
        if (loc >= 0) y = p.v_offset + loc;
      }
    }
  }
  if (lane == 0) {
    p.ycand[b] = y;
    p.dec[d.B + b] = make_int4(__float_as_int((float)mass), st, kind, 0);
  }
}

struct ShardCommitParams {
  Dims d;
  const int* y;
  const int* tok;
  const SeqInfo* info;
  const int4* dec;
  int* cnt;
  int *sel_k, *commit_len, *out_tok, *y_tok, *y_kind, *offsets, *packed_tok, *path_rolled,
      *branch_discarded, *status;
  uint32_t* keep_mask;
  float* resid_mass;
};

// one warp per sequence; the last warp to finish scans the offsets
__global__ void __launch_bounds__(128) k_shard_commit(ShardCommitParams p) {
  const Dims& d = p.d;
  const int lane = threadIdx.x & 31;
  const int b = blockIdx.x * 4 + (threadIdx.x >> 5);
  if (b >= d.B) return;
  const SeqInfo in = p.info[b];
  const int4 D = p.dec[b], D2 = p.dec[d.B + b];
  const int ksel = D.x, npath = D.y, kind = D2.z, kpath = ksel < 0 ? 0 : ksel;
  const int y = (kind != 0) ? p.y[b] : -1;
  int* out = p.out_tok + (int64_t)b * (d.G + 2);
  for (int qq = lane; qq < d.G + 2; qq += 32) {
    int v = -1;
    if (qq < npath) v = __ldg(p.tok + ent(d, b, (qq < in.s) ? 0 : kpath, qq));
    else if (qq == npath && kind != 0) v = y;
    out[qq] = v;
  }
  if (lane < d.K) {
    uint32_t km = 0;
    for (int qq = 0; qq < npath; ++qq)
      if (((qq < in.s) ? 0 : kpath) == lane) km |= 1u << qq;
    p.keep_mask[(int64_t)b * d.K + lane] = km;
  }
  if (lane == 0) {
    p.sel_k[b] = ksel;
    p.commit_len[b] = npath + (kind != 0);
    p.y_tok[b] = y;
    p.y_kind[b] = kind;
    p.path_rolled[b] = in.L - npath;
    p.branch_discarded[b] = (d.K - 1) * (in.L - in.s);
    if (p.resid_mass) p.resid_mass[b] = (kind != 0) ? __int_as_float(D2.x) : 0.f;
    if (D2.y) p.status[b] |= D2.y;
  }
  __syncwarp();
  int last = 0;
  if (lane == 0) {
    __threadfence();
    last = (atomicAdd(p.cnt, 1) == d.B - 1);
  }
  last = __shfl_sync(0xffffffffu, last, 0);
  if (!last) return;
  __threadfence();
  const int per = (d.B + 31) / 32;
  const int b0 = min(d.B, lane * per), b1 = min(d.B, b0 + per);
  int loc = 0;
  for (int qq = b0; qq < b1; ++qq) loc += __ldcg(p.commit_len + qq);
  int incl = loc;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int yv = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += yv;
  }
  int run = incl - loc;
  for (int qq = b0; qq < b1; ++qq) {
    p.offsets[qq] = run;
    const int cl = __ldcg(p.commit_len + qq);
    if (p.packed_tok)
      for (int c = 0; c < cl; ++c) p.packed_tok[run + c] = __ldcg(p.out_tok + (int64_t)qq * (d.G + 2) + c);
    run += cl;
  }
  if (lane == 31) p.offsets[d.B] = incl;
  if (lane == 0) *p.cnt = 0;
}

}  // namespace sb

// ---------------------------------------------------------------- C ABI
using namespace sb;

// defined in sb_verify.cu
sb_status sb_rows_partial(const sb_dims* dd, const void* p_logits, const void* q_logits, const int32_t* tok,
                          const float* u, const int32_t* gamma, const int32_t* branch_pos, void* partial,
                          void* workspace, size_t workspace_bytes, cudaStream_t s);

static int nseg_of(const sb_dims* d) { return (int)(((size_t)d->V * elem_size(d) + 511) / 512); }

extern "C" size_t sb_shard_partial_bytes(const sb_dims* d) {
  if (!dims_valid(d)) return 0;
  return (size_t)d->B * d->K * (d->G + 1) * (sizeof(ShardRow) + sizeof(float2));
}

extern "C" sb_status sb_shard_verify_local(const sb_dims* d, const void* p_logits, const void* q_logits,
                                           const int32_t* tok, const float* u, const int32_t* gamma,
                                           const int32_t* branch_pos, void* partial, void* workspace,
                                           size_t workspace_bytes, sb_stream_t stream) {
  SB_NVTX("sb_shard_verify_local");
  if (!dims_valid(d)) return SB_ERR_INVALID_ARG;
  if (!p_logits || !q_logits || !tok || !u || !partial || !workspace) return SB_ERR_INVALID_ARG;
  return sb_rows_partial(d, p_logits, q_logits, tok, u, gamma, branch_pos, partial, workspace,
                         workspace_bytes, (cudaStream_t)stream);
}

extern "C" sb_status sb_shard_verify_combine(const sb_dims* dd, const void* gathered, int32_t nranks,
                                             const int32_t* tok, const float* u, float* lse_p, float* lse_q,
                                             float* p_tok, float* q_tok, uint32_t* acc_mask, int32_t* n_acc,
                                             float* top1_q, int32_t* top1_id_q, float* entropy_q,
                                             int32_t* status, void* workspace, size_t workspace_bytes,
                                             sb_stream_t stream) {
  SB_NVTX("sb_shard_verify_combine");
  if (!dims_valid(dd) || nranks < 1) return SB_ERR_INVALID_ARG;
  if (!gathered || !tok || !u || !lse_p || !lse_q || !p_tok || !q_tok || !acc_mask || !n_acc || !status ||
      !workspace)
    return SB_ERR_INVALID_ARG;
  const Workspace w = carve(*dd, workspace);
  if (workspace_bytes < w.bytes) return SB_ERR_WORKSPACE;
  ShardCombineParams p;
  p.d = to_dims(dd);
  p.nranks = nranks;
  p.v_total = dd->v_total;
  const size_t per = (size_t)dd->B * dd->K * (dd->G + 1);
  p.gathered = reinterpret_cast<const char*>(gathered);
  p.rank_bytes = sb_shard_partial_bytes(dd);
  p.tok_off = per * sizeof(ShardRow);
  p.tok = tok; p.u = u; p.info = w.info; p.rowstat = w.rowstat; p.pflag = w.pflag; p.tok_lp = w.tok_lp;
  p.lse_p = lse_p; p.lse_q = lse_q; p.p_tok = p_tok; p.q_tok = q_tok; p.top1_q = top1_q;
  p.entropy_q = entropy_q; p.top1_id_q = top1_id_q; p.acc_mask = acc_mask; p.n_acc = n_acc; p.status = status;
  k_shard_combine<<<(dd->B + 3) / 4, 128, 0, (cudaStream_t)stream>>>(p);
  return cuda_status(cudaGetLastError());
}

extern "C" sb_status sb_shard_select_local(const sb_dims* dd, const void* p_logits, const void* q_logits,
                                           const int32_t* tok, const float* u, const int32_t* n_acc,
                                           sb_select_rule rule, double* mass, void* workspace,
                                           size_t workspace_bytes, sb_stream_t stream) {
  SB_NVTX("sb_shard_select_local");
  if (!dims_valid(dd)) return SB_ERR_INVALID_ARG;
  if (!p_logits || !q_logits || !tok || !u || !n_acc || !mass || !workspace) return SB_ERR_INVALID_ARG;
  if (rule != SB_SELECT_EQ9 && rule != SB_SELECT_ALG1) return SB_ERR_INVALID_ARG;
  const Workspace w = carve(*dd, workspace);
  if (workspace_bytes < w.bytes) return SB_ERR_WORKSPACE;
  ShardSelParams p{};
  p.vec = vec_ok(dd, p_logits) && vec_ok(dd, q_logits);  // else scalar loads (any alignment / length)
  p.d = to_dims(dd); p.v_offset = dd->v_offset; p.v_total = dd->v_total; p.rule = rule; p.nseg = nseg_of(dd);
  p.PL = p_logits; p.QL = q_logits; p.tok = tok; p.u = u; p.n_acc = n_acc; p.info = w.info;
  p.rowstat = w.rowstat; p.tok_lp = w.tok_lp; p.dec = w.dec; p.segs = w.segs;
  p.mass = reinterpret_cast<double2*>(mass);
  if (dd->dtype == SB_BF16) k_shard_select_local<__nv_bfloat16><<<dd->B, 256, 0, (cudaStream_t)stream>>>(p);
  else k_shard_select_local<float><<<dd->B, 256, 0, (cudaStream_t)stream>>>(p);
  return cuda_status(cudaGetLastError());
}

extern "C" sb_status sb_shard_select_sample(const sb_dims* dd, const double* gathered_mass, int32_t nranks,
                                            int32_t rank, const void* p_logits, const void* q_logits,
                                            const float* us, int32_t* ycand, void* workspace,
                                            size_t workspace_bytes, sb_stream_t stream) {
  SB_NVTX("sb_shard_select_sample");
  if (!dims_valid(dd) || nranks < 1 || rank < 0 || rank >= nranks) return SB_ERR_INVALID_ARG;
  if (!gathered_mass || !p_logits || !q_logits || !us || !ycand || !workspace) return SB_ERR_INVALID_ARG;
  const Workspace w = carve(*dd, workspace);
  if (workspace_bytes < w.bytes) return SB_ERR_WORKSPACE;
  ShardSelParams p{};
  p.vec = vec_ok(dd, p_logits) && vec_ok(dd, q_logits);
  p.d = to_dims(dd); p.v_offset = dd->v_offset; p.v_total = dd->v_total; p.nseg = nseg_of(dd);
  p.PL = p_logits; p.QL = q_logits; p.us = us; p.info = w.info; p.rowstat = w.rowstat; p.dec = w.dec;
  p.segs = w.segs; p.gmass = reinterpret_cast<const double2*>(gathered_mass); p.nranks = nranks; p.rank = rank;
  p.ycand = ycand;
  if (dd->dtype == SB_BF16) k_shard_sample<__nv_bfloat16><<<(dd->B + 3) / 4, 128, 0, (cudaStream_t)stream>>>(p);
  else k_shard_sample<float><<<(dd->B + 3) / 4, 128, 0, (cudaStream_t)stream>>>(p);
  return cuda_status(cudaGetLastError());
}

extern "C" sb_status sb_shard_select_commit(const sb_dims* dd, const int32_t* y, const int32_t* tok,
                                            int32_t* sel_k, int32_t* commit_len, int32_t* out_tok, int32_t* y_tok,
                                            int32_t* y_kind, int32_t* offsets, int32_t* packed_tok,
                                            int32_t* path_rolled, int32_t* branch_discarded, uint32_t* keep_mask,
                                            float* resid_mass, int32_t* status, void* workspace,
                                            size_t workspace_bytes, sb_stream_t stream) {
  SB_NVTX("sb_shard_select_commit");
  if (!dims_valid(dd)) return SB_ERR_INVALID_ARG;
  if (!y || !tok || !sel_k || !commit_len || !out_tok || !y_tok || !y_kind || !offsets || !path_rolled ||
      !branch_discarded || !keep_mask || !status || !workspace)
    return SB_ERR_INVALID_ARG;
  const Workspace w = carve(*dd, workspace);
  if (workspace_bytes < w.bytes) return SB_ERR_WORKSPACE;
  ShardCommitParams p;
  p.d = to_dims(dd); p.y = y; p.tok = tok; p.info = w.info; p.dec = w.dec; p.cnt = w.sel_cnt;
  p.sel_k = sel_k; p.commit_len = commit_len; p.out_tok = out_tok; p.y_tok = y_tok; p.y_kind = y_kind;
  p.offsets = offsets; p.packed_tok = packed_tok; p.path_rolled = path_rolled;
  p.branch_discarded = branch_discarded; p.status = status; p.keep_mask = keep_mask; p.resid_mass = resid_mass;
  k_shard_commit<<<(dd->B + 3) / 4, 128, 0, (cudaStream_t)stream>>>(p);
  return cuda_status(cudaGetLastError());
}

// ---------------------------------------------------------------- NCCL communicator
struct sb_comm {
  ncclComm_t nccl;
  int nranks, rank;
  void* gather;    // nranks x partial bytes
  void* mine;      // one partial
  double* gmass;   // nranks x B x 2
  double* mass;    // B x 2
  int* y;          // B
  size_t cap_partial;
  int cap_B;
};

extern "C" size_t sb_comm_unique_id_bytes(void) { return sizeof(ncclUniqueId); }

extern "C" sb_status sb_comm_unique_id(void* out) {
  SB_NVTX("sb_comm_unique_id");
  if (!out) return SB_ERR_INVALID_ARG;
  return ncclGetUniqueId(reinterpret_cast<ncclUniqueId*>(out)) == ncclSuccess ? SB_OK : SB_ERR_NCCL;
}

extern "C" sb_status sb_comm_create(const void* unique_id, int32_t nranks, int32_t rank, const sb_dims* max_dims,
                                    sb_comm** out) {
  SB_NVTX("sb_comm_create");
  if (!unique_id || !out || nranks < 1 || rank < 0 || rank >= nranks || !dims_valid(max_dims))
    return SB_ERR_INVALID_ARG;
  sb_comm* c = new sb_comm();
  c->nranks = nranks;
  c->rank = rank;
  ncclUniqueId id;
  memcpy(&id, unique_id, sizeof(id));
  if (ncclCommInitRank(&c->nccl, nranks, id, rank) != ncclSuccess) {
    delete c;
    return SB_ERR_NCCL;
  }
  c->cap_partial = sb_shard_partial_bytes(max_dims);
  c->cap_B = max_dims->B;
  bool ok = cudaMalloc(&c->gather, c->cap_partial * nranks) == cudaSuccess &&
            cudaMalloc(&c->mine, c->cap_partial) == cudaSuccess &&
            cudaMalloc(&c->gmass, sizeof(double) * 2 * c->cap_B * nranks) == cudaSuccess &&
            cudaMalloc(&c->mass, sizeof(double) * 2 * c->cap_B) == cudaSuccess &&
            cudaMalloc(&c->y, sizeof(int) * c->cap_B) == cudaSuccess;
  if (!ok) {
    ncclCommDestroy(c->nccl);
    delete c;
    return SB_ERR_CUDA;
  }
  *out = c;
  return SB_OK;
}

// Asynchronous NCCL errors (a peer died, a network error inside a collective) surface
// through ncclCommGetAsyncError only; every sharded call checks it before enqueueing
// more work on the communicator (SURVEY §5 failure detection).
static sb_status comm_health(sb_comm* c) {
  ncclResult_t e = ncclSuccess;
  if (ncclCommGetAsyncError(c->nccl, &e) != ncclSuccess) return SB_ERR_NCCL;
  return (e == ncclSuccess || e == ncclInProgress) ? SB_OK : SB_ERR_NCCL;
}

extern "C" sb_status sb_comm_check(sb_comm* c) {
  if (!c) return SB_ERR_INVALID_ARG;
  return comm_health(c);
}

extern "C" sb_status sb_comm_abort(sb_comm* c) {
  SB_NVTX("sb_comm_abort");
  if (!c) return SB_ERR_INVALID_ARG;
  const bool ok = ncclCommAbort(c->nccl) == ncclSuccess;
  cudaFree(c->gather);
  cudaFree(c->mine);
  cudaFree(c->gmass);
  cudaFree(c->mass);
  cudaFree(c->y);
  delete c;
  return ok ? SB_OK : SB_ERR_NCCL;
}

extern "C" sb_status sb_comm_destroy(sb_comm* c) {
  SB_NVTX("sb_comm_destroy");
  if (!c) return SB_ERR_INVALID_ARG;
  cudaFree(c->gather);
  cudaFree(c->mine);
  cudaFree(c->gmass);
  cudaFree(c->mass);
  cudaFree(c->y);
  const bool ok = ncclCommDestroy(c->nccl) == ncclSuccess;
  delete c;
  return ok ? SB_OK : SB_ERR_NCCL;
}

// The sharded verify / select with the exchanges inside (called from sb_verify_branches
// and sb_select_branch when comm != NULL).
sb_status sb_shard_verify_nccl(const sb_dims* d, const void* p_logits, const void* q_logits, const int32_t* tok,
                               const float* u, const int32_t* gamma, const int32_t* branch_pos, float* lse_p,
                               float* lse_q, float* p_tok, float* q_tok, uint32_t* acc_mask, int32_t* n_acc,
                               float* top1_q, int32_t* top1_id_q, float* entropy_q, int32_t* status, sb_comm* c,
                               void* workspace, size_t workspace_bytes, cudaStream_t s) {
  const size_t pb = sb_shard_partial_bytes(d);
  if (pb > c->cap_partial) return SB_ERR_INVALID_ARG;
  if (comm_health(c) != SB_OK) return SB_ERR_NCCL;
  sb_status st = sb_shard_verify_local(d, p_logits, q_logits, tok, u, gamma, branch_pos, c->mine, workspace,
                                       workspace_bytes, (sb_stream_t)s);
  if (st != SB_OK) return st;
  if (ncclAllGather(c->mine, c->gather, pb, ncclUint8, c->nccl, s) != ncclSuccess) return SB_ERR_NCCL;
  return sb_shard_verify_combine(d, c->gather, c->nranks, tok, u, lse_p, lse_q, p_tok, q_tok, acc_mask, n_acc,
                                 top1_q, top1_id_q, entropy_q, status, workspace, workspace_bytes, (sb_stream_t)s);
}

sb_status sb_shard_select_nccl(const sb_dims* d, const void* p_logits, const void* q_logits, const int32_t* tok,
                               const float* u, const float* us, const int32_t* n_acc, sb_select_rule rule,
                               int32_t* sel_k, int32_t* commit_len, int32_t* out_tok, int32_t* y_tok,
                               int32_t* y_kind, int32_t* offsets, int32_t* packed_tok, int32_t* path_rolled,
                               int32_t* branch_discarded, uint32_t* keep_mask, float* resid_mass, int32_t* status,
                               sb_comm* c, void* workspace, size_t workspace_bytes, cudaStream_t s) {
  if (d->B > c->cap_B) return SB_ERR_INVALID_ARG;
  if (comm_health(c) != SB_OK) return SB_ERR_NCCL;
  sb_status st = sb_shard_select_local(d, p_logits, q_logits, tok, u, n_acc, rule, c->mass, workspace,
                                       workspace_bytes, (sb_stream_t)s);
  if (st != SB_OK) return st;
  if (ncclAllGather(c->mass, c->gmass, (size_t)2 * d->B, ncclFloat64, c->nccl, s) != ncclSuccess)
    return SB_ERR_NCCL;
  st = sb_shard_select_sample(d, c->gmass, c->nranks, c->rank, p_logits, q_logits, us, c->y, workspace,
                              workspace_bytes, (sb_stream_t)s);
  if (st != SB_OK) return st;
  if (ncclAllReduce(c->y, c->y, d->B, ncclInt32, ncclMax, c->nccl, s) != ncclSuccess) return SB_ERR_NCCL;
  return sb_shard_select_commit(d, c->y, tok, sel_k, commit_len, out_tok, y_tok, y_kind, offsets, packed_tok,
                                path_rolled, branch_discarded, keep_mask, resid_mass, status, workspace,
                                workspace_bytes, (sb_stream_t)s);
}
