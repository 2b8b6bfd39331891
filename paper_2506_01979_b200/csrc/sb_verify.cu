// sb_verify.cu — sb_verify_branches: one streaming pass over every tested (p,q) row
// pair, fused with the acceptance test and, in the CTA completing each sequence, the
// first-rejection scan (SURVEY §8.1 rows a1 + a2; PAPER §3 P94, Alg. 1 P523-538).
//
// Kernels
//   k_plan      (1 CTA)      clamp gamma_b / s_b, L_b, tested row pairs per sequence,
//                            exclusive scan -> unit offsets.
//   k_rows_tma  (persistent, 16-byte aligned rows; the path every benchmark takes)
//                            producer warp: cp.async.bulk ring of p / q chunks; consumer
//                            warps: lazy-offset online max / sum / entropy with packed
//                            FFMA2 / FADD2 bf16 arithmetic; epilogue warps: token tests
//                            in fp64, row outputs, per-sequence completion -> n_k.
//                            sb_verify_branches_reuse: slot-0 q rows come back as states
//                            from the confidence pass (p chunks only for those units).
//   k_rows      (fallback)   the same arithmetic register-staged, any alignment.
//   k_step_tma  (opt-in)     verify + sample in one persistent launch (SB_FUSED_STEP=1).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "sb_host.h"
#include "sb_ring.cuh"
#include "sb_sample.cuh"
#include "sb_conf.cuh"
#include "sb_stream.cuh"
#include "sb_rows.cuh"

namespace sb {

#ifdef SB_TRACE
}  // namespace sb
SB_TRACE_TABLE(sb_trace_rows)
SB_TRACE_TABLE(sb_trace_astep)
namespace sb {
#endif


// ---------------------------------------------------------------- plan
// A unit's sequence, row geometry and the sequence's layout packed in 16 bytes.
__host__ __device__ inline int4 unit_entry(int b, int slot, int i, const SeqInfo& in) {
  return make_int4(b, slot | (i << 8) | (in.s << 16) | (in.g << 24), in.L | (in.Lr << 8) | (in.st << 16), 0);
}

__global__ void __launch_bounds__(1024) k_plan(Dims d, const int* __restrict__ gamma,
                                               const int* __restrict__ bpos, SeqInfo* info,
                                               int* unit_off, int with_bonus, int fused_grid, int* plan,
                                               int* ready, int* seqpk) {
  __shared__ int wsum[32];
  pdl_wait();
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
    const int Lr = with_bonus ? g + 1 : L;  // sharded mode also reads every bonus row
    info[b] = SeqInfo{g, s, L, st, Lr, {0, 0, 0}};
    if (seqpk) seqpk[b] = s | (g << 5) | (L << 10) | (Lr << 16) | (st << 22);
    local += Lr + (d.K - 1) * (Lr - 1 - s);  // slot 0: rows 0..Lr-1; slots k>0: s+1..Lr-1
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
  if (fused_grid > 0) {
    // fused step: the sample unit of sequence b follows the phase-1 units of sequence
    // b + delta (delta ~ 3 waves of units behind), the last delta sample units at the end
    const int p1total = wsum[NT / 32 - 1];
    const int delta = max(1, min(d.B, (3 * fused_grid * d.B + max(1, p1total) - 1) / max(1, p1total)));
    for (int b = b0; b < b1; ++b) {
      unit_off[b] = run + max(0, b - delta);
      const SeqInfo in = info[b];
      run += in.Lr + (d.K - 1) * (in.Lr - 1 - in.s);
      ready[b] = 0;
    }
    if (tid == NT - 1) {
      unit_off[d.B] = run + max(0, d.B - delta);
      plan[0] = delta;
      plan[1] = run + d.B;  // total units
    }
    return;
  }
  for (int b = b0; b < b1; ++b) {
    unit_off[b] = run;
    const SeqInfo in = info[b];
    run += in.Lr + (d.K - 1) * (in.Lr - 1 - in.s);
  }
  if (tid == NT - 1) unit_off[d.B] = run;
}

// ---------------------------------------------------------------- shared unit logic

// unit -> (sequence, slot, row): upper-bound search over the offsets, then slot 0 rows
// 0..L-1 followed by rows s+1..L-1 of slots 1..K-1
__device__ __forceinline__ Unit decode_unit(const RowsParams& p, int unit) {
  const Dims& d = p.d;
  int lo = 0, hi = d.B;
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (__ldg(p.unit_off + mid) <= unit) lo = mid; else hi = mid;
  }
  Unit u;
  u.b = lo;
  u.in = p.info[lo];
  const int j = unit - __ldg(p.unit_off + lo);
  if (j < u.in.Lr) {
    u.slot = 0;
    u.i = j;
  } else {
    const int per = u.in.Lr - 1 - u.in.s, jj = j - u.in.Lr;
    u.slot = 1 + jj / per;
    u.i = u.in.s + 1 + jj % per;
  }
  return u;
}

__device__ __forceinline__ Unit unit_from(int4 e) {
  Unit u;
  u.b = e.x;
  u.slot = e.y & 0xff;
  u.i = (e.y >> 8) & 0xff;
  u.in.s = (e.y >> 16) & 0xff;
  u.in.g = (e.y >> 24) & 0xff;
  u.in.L = e.z & 0xff;
  u.in.Lr = (e.z >> 8) & 0xff;
  u.in.st = e.z >> 16;
  return u;
}

// The packed geometry of `unit` (decoded one unit ahead by the streaming kernels, so
// the search's dependent loads overlap the current unit's stream), or zeros past the end.
__device__ __forceinline__ int4 unit_prefetch(const RowsParams& p, int unit, int total) {
  if (unit >= total) return make_int4(0, 0, 0, 0);
  const Unit u = decode_unit(p, unit);
  return unit_entry(u.b, u.slot, u.i, u.in);
}

// Warp-cooperative decode of a unit (the streaming kernels' producer and epilogue warps):
// a CTA walks its units in increasing order, so the sequence of the next unit is at or
// after the current one; lane l probes sequence base + l (unit offset + packed layout,
// two independent loads, one round trip), one ballot finds it.  Against the binary
// search's log2(B) dependent loads per unit this keeps a short unit's producer from
// stalling (C2: 668 units of 125 KB).
struct Probe {
  int off, pk;
};
__device__ __forceinline__ Probe probe_load(const RowsParams& p, int base) {
  const int bb = base + (threadIdx.x & 31);
  Probe r;
  r.off = bb <= p.d.B ? __ldg(p.unit_off + bb) : 0x7fffffff;
  r.pk = bb < p.d.B ? __ldg(p.seqpk + bb) : 0;
  return r;
}
// The packed geometry of `unit` (zeros past the end); base <= the unit's sequence on
// entry, its sequence on return.  Warp-uniform arguments.
__device__ __forceinline__ int4 probe_resolve(const RowsParams& p, Probe pr, int& base, int unit, int total) {
  if (unit >= total) return make_int4(0, 0, 0, 0);
  unsigned le = __ballot_sync(0xffffffffu, pr.off <= unit);
  while (le == 0xffffffffu) {  // more than 32 sequences ahead (only the first decode)
    base += 32;
    pr = probe_load(p, base);
    le = __ballot_sync(0xffffffffu, pr.off <= unit);
  }
  if (le == 0u) {  // not reachable from a valid base; keep the binary search as a guard
    const Unit u = decode_unit(p, unit);
    base = u.b;
    return unit_entry(u.b, u.slot, u.i, u.in);
  }
  const int src = __popc(le) - 1;
  const int off = __shfl_sync(0xffffffffu, pr.off, src);
  const int pk = __shfl_sync(0xffffffffu, pr.pk, src);
  base += src;
  Unit u;
  u.b = base;
  u.in.s = pk & 31;
  u.in.g = (pk >> 5) & 31;
  u.in.L = (pk >> 10) & 63;
  u.in.Lr = (pk >> 16) & 63;
  u.in.st = pk >> 22;
  const int j = unit - off;
  if (j < u.in.Lr) {
    u.slot = 0;
    u.i = j;
  } else {
    const int per = u.in.Lr - 1 - u.in.s, jj = j - u.in.Lr;
    u.slot = 1 + jj / per;
    u.i = u.in.s + 1 + jj % per;
  }
  return unit_entry(u.b, u.slot, u.i, u.in);
}

// Slot-0 draft rows i < G were streamed by sb_draft_confidence: with p.qreuse their q
// state is read back instead of the row (SURVEY §8.4 adaptive configs).
__device__ __forceinline__ bool q_reused(const RowsParams& p, const Unit& un) {
  return p.qreuse != nullptr && un.slot == 0 && un.i < p.d.G;
}

// Everything after a row pair's statistics are known: path-token probabilities and the
// acceptance test, row outputs, and (in the CTA completing the sequence) n_k, status and
// the sentinels.  `tid` / `nt` index the participating threads; `sync` is their barrier.
template <typename T, typename Sync>
__device__ __forceinline__ void unit_epilogue(const RowsParams& p, const Unit& un, const T* prow,
                                              const T* qrow, const RowStat& ps, const RowStat& qs,
                                              int tid, int nt, int* s_last, int* s_st, Sync sync) {
  const Dims& d = p.d;
  const int b = un.b, slot = un.slot, i = un.i;
  const SeqInfo& in = un.in;
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
      fl |= st_flags(po.st | qo.st);
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
    if (p.top1_q) p.top1_q[e] = conf_ok ? (float)tok_prob(qs.m, qo.MS, qo.Z) : CUDART_NAN_F;
    if (p.top1_id_q) p.top1_id_q[e] = conf_ok ? qs.idx : -1;
    if (p.entropy_q) {
      const double Z = qo.Z;
      p.entropy_q[e] = conf_ok ? (float)(LN2 * (log2(Z) - (double)qs.s1 / Z)) : CUDART_NAN_F;
    }
    p.rowstat[e] = make_float4(po.MS, z_store(po), qo.MS, z_store(qo));
  }
  // completion: the CTA finishing the sequence decides n_k (first zero bit)
  sync();
  if (tid == 0) {
    __threadfence();
    const int units_b = __ldg(p.unit_off + b + 1) - __ldg(p.unit_off + b);
    const int prev = atomicAdd(p.cnt + b, 1);
    *s_last = (prev == units_b - 1);
    *s_st = in.st;
  }
  sync();
  if (*s_last) {
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
        st |= flags_st(fl);
      }
      const uint32_t rej = ~mask & (in.L >= 32 ? 0xffffffffu : ((1u << in.L) - 1));
      p.acc_mask[(int64_t)b * d.K + k] = mask;
      p.n_acc[(int64_t)b * d.K + k] = rej ? (__ffs(rej) - 1) : in.L;
      if (st) atomicOr(s_st, st);
    }
    // sentinels for entries no tested path touches
    for (int q = tid; q < d.K * R1; q += nt) {
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
    sync();
    if (tid == 0) {
      p.status[b] = *s_st;
      p.cnt[b] = 0;  // leave the workspace re-usable
    }
  }
  sync();
}

// ---------------------------------------------------------------- rows
// Register-staged fallback (any alignment / stride): each thread streams its share of
// the row pair with 16-byte (or scalar) loads.
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
    const Unit un = decode_unit(p, unit);
    const T* prow = PL + row_off(d, un.b, un.slot, un.i);
    const T* qrow = QL + row_off(d, un.b, un.slot, un.i);
    RowAcc<false, NA> pa;
    RowAcc<true, NA> qa;
    pa.init();
    qa.init();
    stream_pair<T, NA, NT, U>(prow, qrow, d.V, vec_ok, pa, qa);
    const RowStat ps = block_reduce<NT>(fold(pa), red);
    const RowStat qs = block_reduce<NT>(fold(qa), red);
    if (p.partial) {  // a7: this shard's row states and token logits (any row length)
      const bool branch_row = (un.slot == 0 && un.i == un.in.s);
      const int ntok = branch_row ? d.K : 1;
      if (tid < ntok && un.i < un.in.L) {
        const int64_t et = ent(d, un.b, branch_row ? tid : un.slot, un.i);
        const int xl = __ldg(p.tok + et) - p.v_offset;
        const bool mine = xl >= 0 && xl < d.V;
        p.tokpart[et] = make_float2(mine ? ld_scalar(prow + xl) : -CUDART_INF_F,
                                    mine ? ld_scalar(qrow + xl) : -CUDART_INF_F);
      }
      if (tid == 0) {
        ShardRow r;
        r.pm = ps.m; r.pms = ps.ms; r.pz = ps.z;
        r.qm = qs.m; r.qms = qs.ms; r.qz = qs.z; r.qs1 = qs.s1;
        r.qidx = (qs.idx == 0x7fffffff) ? qs.idx : qs.idx + p.v_offset;
        r.qfin = qs.m > -CUDART_INF_F && qs.m < CUDART_INF_F;  // unclamped inputs: the true maximum
        p.rowpart[ent(d, un.b, un.slot, un.i)] = r;
      }
      __syncthreads();
      continue;
    }
    unit_epilogue(p, un, prow, qrow, ps, qs, tid, NT, &s_last, &s_st, [] { __syncthreads(); });
  }
}

// ---------------------------------------------------------------- rows, TMA ring
// Warp-specialised persistent kernel, one CTA per SM (template RC = geometry):
//   warp CW       producer  : cp.async.bulk of CHUNK-byte p and q row chunks into an
//                             NS-stage shared ring (mbarrier full/empty per stage);
//   warps 0..CW-1 consumers : fold each chunk into the lazy online state (VPT 16-byte
//                             vectors per thread per row per stage), then per unit one
//                             warp reduction (+ exact first-argmax) -> a partial in
//                             shared memory (NP slots, mbarrier handshake);
//   warps CW+1..  epilogue  : NE warps, alternating units: prefetch the unit's path
//                             tokens, uniforms and their two logits while the consumers
//                             stream, then combine the CW partials, resolve the q argmax,
//                             run the token tests in fp64, write the row outputs and the
//                             per-sequence completion — concurrently with the consumers
//                             streaming the next units.

template <class C>
struct RowsSmem {
  uint64_t full[C::NS], empty[C::NS];
  uint64_t pfull[C::NP], pempty[C::NP];
  RowStat part[C::NP][2][C::CW];  // [slot][p,q][warp]
  uint2 cand[C::NP][C::CW];       // q-row argmax candidates per warp (tag, lane mask)
  int ponly[C::NS];               // stage holds only the p chunk (q state reused)
  alignas(128) uint8_t buf[C::NS][2][C::CHUNK];
};

// Warp-level reduction of one row's per-thread state.  For q rows the exact first index
// of the warp maximum is resolved by re-reading the (<= VPT) vectors of the chunk where
// each max-holding lane first saw it; the loads are issued before the sum reduction.
template <class C, typename T, bool kQ>
__device__ __forceinline__ RowStat warp_part(const LazyAcc<kQ, 4>& a, const T* row, int nvec_last,
                                             int nchunks) {
  constexpr int E = Vec<T>::E;
  const int tid = threadIdx.x;
  RowStat s = fold_lazy(a);
  float mw = s.m;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mw = fmaxf(mw, __shfl_xor_sync(0xffffffffu, mw, o));
  uint4 x[C::VPT];
  bool have[C::VPT];
  const bool need = kQ && (a.m == mw) && (mw > -CUDART_INF_F) && (a.tag >= 0);
  const int c = a.tag;
  if (need) {
    const int nvec = (c == nchunks - 1) ? nvec_last : C::CHUNK / 16;
    const uint4* cv =
        reinterpret_cast<const uint4*>(reinterpret_cast<const char*>(row) + (size_t)c * C::CHUNK);
#pragma unroll
    for (int j = 0; j < C::VPT; ++j) {
      const int v = tid + j * C::CT;
      have[j] = v < nvec;
      if (have[j]) x[j] = __ldg(cv + v);
    }
  }
  s = warp_reduce_offsets(s);
  s.m = mw;
  int cand = 0x7fffffff;
  if (need) {
#pragma unroll
    for (int j = C::VPT - 1; j >= 0; --j) {
      if (!have[j]) continue;
      float f[E];
      Vec<T>::unpack(x[j], f);
#pragma unroll
      for (int e = E - 1; e >= 0; --e)
        if (f[e] == mw) cand = c * (C::CHUNK / (int)sizeof(T)) + (tid + j * C::CT) * E + e;
    }
  }
  s.idx = kQ ? (int)__reduce_min_sync(0xffffffffu, (unsigned)cand) : 0;
  return s;
}


// One ring stage as this thread sees it: VPT 16-byte vectors of the p and q chunks.
template <class C>
struct StageRegs {
  uint4 p[C::VPT], q[C::VPT];
};


template <class C, typename T, bool FULL>
__device__ __forceinline__ void load_stage(const uint8_t* bp, const uint8_t* bq, int nvec, StageRegs<C>& r) {
  const int tid = threadIdx.x;
#pragma unroll
  for (int j = 0; j < C::VPT; ++j) {
    const int v = tid + j * C::CT;
    if (FULL || v < nvec) {
      r.p[j] = lds128(bp + v * 16);
      r.q[j] = lds128(bq + v * 16);
    } else {
      r.p[j] = r.q[j] = neg_inf_vec<T>();
    }
  }
}

template <class C, typename T, bool FIRST = false>
__device__ __forceinline__ void compute_stage(const StageRegs<C>& r, int c, LazyAcc<false, 4>& pa,
                                              LazyAcc<true, 4>& qa) {
  if constexpr (sizeof(T) == 2) {
    acc_vecs_bf16<C::VPT, false, FIRST>(pa, r.p, c);
    acc_vecs_bf16<C::VPT, true, FIRST>(qa, r.q, c);
  } else {
    constexpr int E = Vec<T>::E;
    float fp[C::VPT * E], fq[C::VPT * E];
#pragma unroll
    for (int j = 0; j < C::VPT; ++j) {
      Vec<T>::unpack(r.p[j], fp + j * E);
      Vec<T>::unpack(r.q[j], fq + j * E);
    }
    pa.template add<C::VPT * E, FIRST>(fp, c);
    qa.template add<C::VPT * E, FIRST>(fq, c);
  }
}

// p-only stage (q state reused): the p vectors and the p arithmetic alone
template <class C, typename T, bool FULL>
__device__ __forceinline__ void load_stage_p(const uint8_t* bp, int nvec, StageRegs<C>& r) {
  const int tid = threadIdx.x;
#pragma unroll
  for (int j = 0; j < C::VPT; ++j) {
    const int v = tid + j * C::CT;
    r.p[j] = (FULL || v < nvec) ? lds128(bp + v * 16) : neg_inf_vec<T>();
  }
}
template <class C, typename T, bool FIRST = false>
__device__ __forceinline__ void compute_stage_p(const StageRegs<C>& r, int c, LazyAcc<false, 4>& pa) {
  if constexpr (sizeof(T) == 2) {
    acc_vecs_bf16<C::VPT, false, FIRST>(pa, r.p, c);
  } else {
    constexpr int E = Vec<T>::E;
    float fp[C::VPT * E];
#pragma unroll
    for (int j = 0; j < C::VPT; ++j) Vec<T>::unpack(r.p[j], fp + j * E);
    pa.template add<C::VPT * E, FIRST>(fp, c);
  }
}

// One ring stage of a unit by the consumer warps: wait -> 16-byte LDS of this thread's
// vectors -> release the stage -> math, so the producer refills the slot while the
// consumers compute.  FIRST: the unit's first chunk (peeled rescale test, see LazyAcc);
// FULL: a whole chunk (no guards, no fill); REUSE: the stage may carry p only.
template <class C, typename T, bool FIRST, bool FULL, bool REUSE>
__device__ __forceinline__ void consume_chunk(RowsSmem<C>& S, RingPos<C::NS>& rp, int c, int nvec,
                                              LazyAcc<false, 4>& pa, LazyAcc<true, 4>& qa) {
  StageRegs<C> r;
  mbar_wait_spin(&S.full[rp.stage], rp.phase);
  const bool po = REUSE && *reinterpret_cast<volatile int*>(&S.ponly[rp.stage]);
  if (!po) load_stage<C, T, FULL>(S.buf[rp.stage][0], S.buf[rp.stage][1], nvec, r);
  else load_stage_p<C, T, FULL>(S.buf[rp.stage][0], nvec, r);
  __syncwarp();
  if ((threadIdx.x & 31) == 0) mbar_arrive(&S.empty[rp.stage]);
  rp.advance();
  if (!po) compute_stage<C, T, FIRST>(r, c, pa, qa);
  else compute_stage_p<C, T, FIRST>(r, c, pa);
}

template <class C, typename T, bool REUSE>
__global__ void __launch_bounds__(C::ROWS_THREADS, 1) k_rows_tma(RowsParams p) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  RowsSmem<C>& S = *reinterpret_cast<RowsSmem<C>*>(smem_raw);
  const Dims& d = p.d;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < C::NS; ++s) {
      mbar_init(&S.full[s], 1);
      mbar_init(&S.empty[s], C::CW);
    }
    for (int s = 0; s < C::NP; ++s) {
      mbar_init(&S.pfull[s], C::CW);
      mbar_init(&S.pempty[s], 1);
    }
    fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0) SB_TRACE_AT(sb_trace_rows, 0, 0);
  pdl_wait();
  if (tid == 0) SB_TRACE_AT(sb_trace_rows, 0, 1);
  const int total = __ldg(p.unit_off + d.B);
  const T* PL = static_cast<const T*>(p.PL);
  const T* QL = static_cast<const T*>(p.QL);
  const uint32_t row_bytes = (uint32_t)d.V * sizeof(T);
  const int nchunks = (row_bytes + C::CHUNK - 1) / C::CHUNK;
  const int nvec_last = (int)(row_bytes - (uint32_t)(nchunks - 1) * C::CHUNK) / 16;

  if (warp == C::CW) {  // ---------------- producer (lane 0 issues, the warp decodes)
    int tli = 0;
    const uint64_t pol = policy_evict_first();
    RingPos<C::NS> rp;
    int base = 0;
    int4 cur = probe_resolve(p, probe_load(p, 0), base, blockIdx.x, total);
    for (int unit = blockIdx.x; unit < total; unit += gridDim.x) {
      const Unit un = unit_from(cur);
      const Probe pr = probe_load(p, base);  // the next unit's probe, in flight during the copies
      if (lane == 0) SB_TRACE_AT(sb_trace_rows, 1, 2 + tli);
      ++tli;
      if (lane == 0) {
        const char* prow = reinterpret_cast<const char*>(PL + row_off(d, un.b, un.slot, un.i));
        const char* qrow = reinterpret_cast<const char*>(QL + row_off(d, un.b, un.slot, un.i));
        const bool po = q_reused(p, un);
        for (int c = 0; c < nchunks; ++c) {
          const uint32_t bytes = min((uint32_t)C::CHUNK, row_bytes - (uint32_t)c * C::CHUNK);
          mbar_wait(&S.empty[rp.stage], rp.phase ^ 1u);
          S.ponly[rp.stage] = po;  // published by the arrive below (release)
          mbar_expect_tx(&S.full[rp.stage], (po ? 1 : 2) * bytes);
          bulk_g2s(S.buf[rp.stage][0], prow + (size_t)c * C::CHUNK, bytes, &S.full[rp.stage], pol);
          if (!po) bulk_g2s(S.buf[rp.stage][1], qrow + (size_t)c * C::CHUNK, bytes, &S.full[rp.stage], pol);
          rp.advance();
        }
      }
      __syncwarp();
      cur = probe_resolve(p, pr, base, unit + gridDim.x, total);
    }
    if (lane == 0) SB_TRACE_AT(sb_trace_rows, 1, 63);
    return;
  }
  if (warp > C::CW) {  // ---------------- epilogue warps: warp e takes local units e, e+NE, ...
    const int e = warp - C::CW - 1;
    int base = 0;
    int4 nxt = probe_resolve(p, probe_load(p, 0), base, blockIdx.x + e * gridDim.x, total);
    for (int li = e, unit = blockIdx.x + e * gridDim.x; unit < total; li += C::NE, unit += C::NE * gridDim.x) {
      RingPos<C::NP> up;
      up.stage = li % C::NP;
      up.phase = (uint32_t)(li / C::NP) & 1u;
      const Unit un = unit_from(nxt);
      nxt = probe_resolve(p, probe_load(p, base), base, unit + C::NE * gridDim.x, total);
      const T* prow = PL + row_off(d, un.b, un.slot, un.i);
      const T* qrow = QL + row_off(d, un.b, un.slot, un.i);
      // prefetch the path tokens through this row, their uniforms and logits
      const bool branch_row = (un.slot == 0 && un.i == un.in.s);
      const int ntok = branch_row ? d.K : 1;
      int x = 0;
      float lpx = 0.f, lqx = 0.f, uu = 0.f;
      int64_t et = 0;
      const bool has_tok = un.i < un.in.L;  // bonus rows (sharded mode) carry no token
      if (lane < ntok && has_tok) {
        et = ent(d, un.b, branch_row ? lane : un.slot, un.i);
        x = __ldg(p.tok + et);
        uu = __ldg(p.u + et);
        const int xl = x - p.v_offset;  // local column in this shard
        if (xl >= 0 && xl < d.V) {
          lpx = ld_scalar(prow + xl);
          lqx = ld_scalar(qrow + xl);
        } else {
          lpx = lqx = -CUDART_INF_F;
        }
      }
      const bool po = q_reused(p, un);
      RowStat qr;
      if (po) qr = p.qreuse[(int64_t)un.b * d.G + un.i];
      mbar_wait_parked(&S.pfull[up.stage], up.phase);
      RowStat ps = lane < C::CW ? S.part[up.stage][0][lane] : rowstat_empty();
      RowStat qs = lane < C::CW ? S.part[up.stage][1][lane] : rowstat_empty();
      const uint2 cand = lane < C::CW ? S.cand[up.stage][lane] : make_uint2(0xffffffffu, 0u);
      __syncwarp();
      if (lane == 0) mbar_arrive(&S.pempty[up.stage]);
      up.advance();
      const float qmw = qs.m;
      ps = warp_reduce_state(ps);  // idx: p's unused, q's resolved below
      qs = warp_reduce_state(qs);
      if (po) qs = qr;
      else qs.idx = resolve_argmax<C, T>(qmw, cand, qs.m, qrow, nvec_last, nchunks);
      if (p.partial) {  // a7: this shard's state, combined across shards later
        if (lane < ntok && has_tok) p.tokpart[et] = make_float2(lpx, lqx);
        ShardRow r;
        if (lane == 0) {
          r.pm = ps.m; r.pms = ps.ms; r.pz = ps.z;
          r.qm = qs.m; r.qms = qs.ms; r.qz = qs.z; r.qs1 = qs.s1;
          r.qidx = (qs.idx == 0x7fffffff) ? qs.idx : qs.idx + p.v_offset;
        }
        {
          // a clamped q maximum of -2^97 leaves "finite entry or all -inf" open (finish_q)
          bool fin = qs.m > kMaskedLogit && qs.m < CUDART_INF_F;
          if (sizeof(T) == 2 && qs.m == kMaskedLogit)
            fin = row_has_finite_bf16(reinterpret_cast<const __nv_bfloat16*>(qrow), d.V);
          else if (sizeof(T) == 4)
            fin = qs.m > -CUDART_INF_F && qs.m < CUDART_INF_F;
          if (lane == 0) {
            r.qfin = fin;
            p.rowpart[ent(d, un.b, un.slot, un.i)] = r;
          }
        }
        continue;
      }
      warp_epilogue<T>(p, un, ps, qs, qrow, x, lpx, lqx, uu, et);
      if (lane == 0) SB_TRACE_AT(sb_trace_rows, 2, 2 + li);
    }
    if (lane == 0) SB_TRACE_AT(sb_trace_rows, 2, 63);
    return;
  }
  // ---------------- consumers
  RingPos<C::NS> rp;
  RingPos<C::NP> up;
  int tli = 0;
  for (int unit = blockIdx.x; unit < total; unit += gridDim.x) {
    LazyAcc<false, 4> pa;
    LazyAcc<true, 4> qa;
    pa.init();
    qa.init();
    if (tid == 0) SB_TRACE_AT(sb_trace_rows, 3, 2 + tli);
    if (nchunks == 1) {
      consume_chunk<C, T, true, false, REUSE>(S, rp, 0, nvec_last, pa, qa);
    } else {
      consume_chunk<C, T, true, true, REUSE>(S, rp, 0, 0, pa, qa);
      for (int c = 1; c < nchunks - 1; ++c) consume_chunk<C, T, false, true, REUSE>(S, rp, c, 0, pa, qa);
      consume_chunk<C, T, false, false, REUSE>(S, rp, nchunks - 1, nvec_last, pa, qa);
    }
    uint2 cand;
#ifdef SB_ROWS_NORED  // experiment: the consumers' per-unit warp reductions removed (wrong results)
    const RowStat ps = fold_lazy(pa), qs = fold_lazy(qa);
    cand = make_uint2(0xffffffffu, 0u);
#else
    const RowStat ps = warp_part<C, T, false>(pa, nullptr, nvec_last, nchunks);
    const RowStat qs = warp_part_deferred(qa, cand);
#endif
    if (lane == 0) {
      mbar_wait(&S.pempty[up.stage], up.phase ^ 1u);
      S.part[up.stage][0][warp] = ps;
      S.part[up.stage][1][warp] = qs;
      S.cand[up.stage][warp] = cand;
      mbar_arrive(&S.pfull[up.stage]);
    }
    __syncwarp();
    up.advance();
    if (tid == 0) SB_TRACE_AT(sb_trace_rows, 3, 32 + tli);
    ++tli;
  }
}

template <class C, typename T, bool REUSE>
static sb_status launch_rows_tma_k(const RowsParams& p, cudaStream_t s) {
  const int smem = (int)sizeof(RowsSmem<C>);
  if (ensure_smem<k_rows_tma<C, T, REUSE>>(smem) != cudaSuccess) return SB_ERR_CUDA;
  const int64_t max_units = (int64_t)p.d.B * p.d.K * (p.d.G + 1);
  const int grid = (int)std::min<int64_t>(num_sms(), max_units);
  return cuda_status(launch_pdl(k_rows_tma<C, T, REUSE>, dim3(grid), dim3(C::ROWS_THREADS), smem, s, p));
}
template <class C, typename T>
static sb_status launch_rows_tma(const RowsParams& p, cudaStream_t s) {
  return p.qreuse ? launch_rows_tma_k<C, T, true>(p, s) : launch_rows_tma_k<C, T, false>(p, s);
}

template <typename T, int NT, int U>
static sb_status launch_rows(const RowsParams& p, bool vok, cudaStream_t s) {
  const int g = full_grid<k_rows<T, NT, U>>(NT);
  const int64_t max_units = (int64_t)p.d.B * p.d.K * (p.d.G + 1);
  const int grid = (int)std::min<int64_t>(g, max_units);
  k_rows<T, NT, U><<<grid, NT, 0, s>>>(p, vok);
  return cuda_status(cudaGetLastError());
}

// ---------------------------------------------------------------- fused step (verify + select)
// One persistent kernel for the whole step: the unit list of k_rows_tma plus, for every
// sequence b, a sample unit placed after the phase-1 units of sequence b + delta
// (k_plan, fused mode).  Dependencies point to smaller unit indices and every CTA walks
// its units in increasing order, so the spin on ready[b] cannot deadlock.
//   producer : phase-1 unit -> stream the p/q chunks (as k_rows_tma);
//              sample unit  -> wait ready[b] (n_k known), take the Eq. 9 / Alg. 1
//              decision (as k_select_tma's decider), publish it, stream the sampled row
//              pair (residual) or the p row twice (bonus: softmax state, then sums);
//   consumers: phase-1 -> partial states; sample -> one sum per 1 KB segment;
//   epilogue : phase-1 -> token tests / n_k / ready[b]; sample -> locate us*R, re-read
//              one segment, commit / rollback outputs; the last sequence scans offsets.
struct StepParams {
  RowsParams r{};
  const float* us;
  int rule;
  const int* plan;  // [0] delta, [1] total units
  int* done_cnt;
  int *sel_k, *commit_len, *out_tok, *y_tok, *y_kind, *offsets, *packed_tok, *path_rolled, *branch_discarded;
  uint32_t* keep_mask;
  float* resid_mass;
};

struct P2Desc {
  int b, ksel, npath, kind, row, slot, pad0, pad1;
  float4 rs;
};

constexpr int kNDQ = 8;        // sample descriptors in flight
constexpr int kSegMax = 1024;  // 1 KB segments per row (rows <= 1 MB)

template <class C>
struct StepSmem {
  uint64_t full[C::NS], empty[C::NS];
  uint64_t pfull[C::NP], pempty[C::NP];
  uint64_t dfull[kNDQ], dempty[kNDQ];
  RowStat part[C::NP][2][C::CW];
  uint2 cand[C::NP][C::CW];
  P2Desc desc[kNDQ];
  float4 brs[kNDQ];  // bonus-row softmax state computed by the consumers
  RowStat red[C::CW];
  float seg[C::NP][kSegMax];
  alignas(128) uint8_t buf[C::NS][2][C::CHUNK];
};

struct FUnit {
  bool sample;
  int b;    // sequence (phase-1 unit's or the sample's)
  Unit u;   // phase-1 geometry
};

__device__ __forceinline__ FUnit decode_fused(const RowsParams& p, const int* plan, int unit) {
  const Dims& d = p.d;
  FUnit f;
  const int tail = __ldg(p.unit_off + d.B);
  if (unit >= tail) {
    const int delta = min(plan[0], d.B);
    f.sample = true;
    f.b = d.B - delta + (unit - tail);
    return f;
  }
  int lo = 0, hi = d.B;
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (__ldg(p.unit_off + mid) <= unit) lo = mid; else hi = mid;
  }
  const SeqInfo in = p.info[lo];
  const int j = unit - __ldg(p.unit_off + lo);
  const int u1 = in.Lr + (d.K - 1) * (in.Lr - 1 - in.s);
  if (j >= u1) {
    f.sample = true;
    f.b = lo - plan[0];
    return f;
  }
  f.sample = false;
  f.b = lo;
  f.u.b = lo;
  f.u.in = in;
  if (j < in.Lr) {
    f.u.slot = 0;
    f.u.i = j;
  } else {
    const int per = in.Lr - 1 - in.s, jj = j - in.Lr;
    f.u.slot = 1 + jj / per;
    f.u.i = in.s + 1 + jj % per;
  }
  return f;
}

template <class SM, class C, typename T, bool RESID>
__device__ __forceinline__ void step_seg_pass(SM& S, RingPos<C::NS>& rp, float* seg, int nchunks,
                                              int nvec_last, bool ok, float MSp, float MSq, float kq) {
  constexpr int E = Vec<T>::E;
  constexpr int SPC = C::CHUNK / kSegBytes;  // segments per chunk (= consumer warps)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int c = 0; c < nchunks; ++c) {
    const int nvec = (c == nchunks - 1) ? nvec_last : C::CHUNK / 16;
    mbar_wait(&S.full[rp.stage], rp.phase);
    float own = 0.f;
#pragma unroll
    for (int h = 0; h < SPC / C::CW; ++h) {
      const int sw = warp + h * C::CW;  // this warp's segment in the chunk
      uint4 vp[2], vq[2];
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int v = sw * 64 + lane * 2 + j;
        if (v < nvec) {
          vp[j] = lds128(S.buf[rp.stage][0] + v * 16);
          if (RESID) vq[j] = lds128(S.buf[rp.stage][1] + v * 16);
        } else {
          vp[j] = vq[j] = neg_inf_vec<T>();
        }
      }
      own = 0.f;
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        float r[E];
        r_scaled<T>(vp[j], vq[j], RESID, MSp, MSq, kq, r);
        own = seq_sum<E>(r, own);
      }
      const float tot = warp_sum_rn(ok ? own : 0.f);
      if (lane == 0) seg[c * SPC + sw] = tot;
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&S.empty[rp.stage]);
    rp.advance();
  }
}

template <class C, typename T>
__global__ void __launch_bounds__(C::THREADS, 1) k_step_tma(StepParams sp) {
  constexpr int E = Vec<T>::E;
  extern __shared__ __align__(128) uint8_t smem_raw[];
  StepSmem<C>& S = *reinterpret_cast<StepSmem<C>*>(smem_raw);
  const RowsParams& p = sp.r;
  const Dims& d = p.d;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < C::NS; ++s) {
      mbar_init(&S.full[s], 1);
      mbar_init(&S.empty[s], C::CW);
    }
    for (int s = 0; s < C::NP; ++s) {
      mbar_init(&S.pfull[s], C::CW);
      mbar_init(&S.pempty[s], 1);
    }
    for (int s = 0; s < kNDQ; ++s) {
      mbar_init(&S.dfull[s], 1);
      mbar_init(&S.dempty[s], 1);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const int total = sp.plan[1];
  const T* PL = static_cast<const T*>(p.PL);
  const T* QL = static_cast<const T*>(p.QL);
  const uint32_t row_bytes = (uint32_t)d.V * sizeof(T);
  const int nchunks = (row_bytes + C::CHUNK - 1) / C::CHUNK;
  const int nvec_last = (int)(row_bytes - (uint32_t)(nchunks - 1) * C::CHUNK) / 16;
  const int nseg = nchunks * (C::CHUNK / kSegBytes);

  if (warp == C::CW) {  // ---------------- producer (+ decider for sample units)
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      RingPos<C::NS> rp;
      RingPos<kNDQ> dq;
      for (int unit = blockIdx.x; unit < total; unit += gridDim.x) {
        const FUnit fu = decode_fused(p, sp.plan, unit);
        const char *prow, *qrow;
        int passes = 1;
        bool pair = true;
        if (!fu.sample) {
          prow = reinterpret_cast<const char*>(PL + row_off(d, fu.b, fu.u.slot, fu.u.i));
          qrow = reinterpret_cast<const char*>(QL + row_off(d, fu.b, fu.u.slot, fu.u.i));
        } else {
          const int b = fu.b;
          mbar_wait(&S.dempty[dq.stage], dq.phase ^ 1u);
          int rd = 0;
          for (uint32_t tries = 0;; ++tries) {  // phase 1 of b done (n_k, status, rowstat written)
            asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(rd) : "l"(p.ready + b) : "memory");
            if (rd) break;
            __nanosleep(256);
            if (tries > (1u << 24)) __trap();  // watchdog (~4 s)
          }
          const SeqInfo in = p.info[b];
          int ksel = -1, besttok = 0;
          float bestkey = 0.f;
          for (int k = 0; k < d.K; ++k) {  // A = {k : n_k > s_b}; Eq. 9 / Alg. 1 (P239, P540)
            if (__ldcg(p.n_acc + (int64_t)b * d.K + k) <= in.s) continue;
            const int xk = __ldg(p.tok + ent(d, b, k, in.s));
            const float key = (sp.rule == SB_SELECT_ALG1) ? __ldg(p.u + ent(d, b, k, in.s))
                                                          : ld_scalar(PL + row_off(d, b, 0, in.s) + xk);
            bool better;
            if (ksel < 0) better = true;
            else if (sp.rule == SB_SELECT_ALG1) better = key > bestkey;
            else better = key > bestkey || (key == bestkey && xk < besttok);
            if (better) { ksel = k; bestkey = key; besttok = xk; }
          }
          P2Desc D;
          D.b = b;
          D.ksel = ksel;
          if (ksel < 0) {
            D.npath = min(__ldcg(p.n_acc + (int64_t)b * d.K), in.s);  // rollback (P655)
            D.kind = 1; D.row = D.npath; D.slot = 0;
          } else {
            D.npath = __ldcg(p.n_acc + (int64_t)b * d.K + ksel);
            if (D.npath < in.L) { D.kind = 1; D.row = D.npath; D.slot = (D.npath <= in.s) ? 0 : ksel; }
            else if (in.s < in.g) { D.kind = 2; D.row = in.g; D.slot = ksel; }  // bonus (P94)
            else { D.kind = 0; D.row = 0; D.slot = 0; }                          // (P237)
          }
          D.rs = (D.kind == 1) ? __ldcg(p.rowstat + ent(d, b, D.slot, D.row)) : make_float4(0.f, 1.f, 0.f, 1.f);
          S.desc[dq.stage] = D;
          mbar_arrive(&S.dfull[dq.stage]);
          dq.advance();
          passes = D.kind == 1 ? 1 : (D.kind == 2 ? 2 : 0);
          pair = D.kind == 1;
          prow = reinterpret_cast<const char*>(PL + row_off(d, b, D.slot, D.row));
          qrow = reinterpret_cast<const char*>(QL + row_off(d, b, D.slot, D.row));
        }
        for (int pass = 0; pass < passes; ++pass)
          for (int c = 0; c < nchunks; ++c) {
            const uint32_t bytes = min((uint32_t)C::CHUNK, row_bytes - (uint32_t)c * C::CHUNK);
            mbar_wait(&S.empty[rp.stage], rp.phase ^ 1u);
            mbar_expect_tx(&S.full[rp.stage], (pair ? 2 : 1) * bytes);
            bulk_g2s(S.buf[rp.stage][0], prow + (size_t)c * C::CHUNK, bytes, &S.full[rp.stage], pol);
            if (pair) bulk_g2s(S.buf[rp.stage][1], qrow + (size_t)c * C::CHUNK, bytes, &S.full[rp.stage], pol);
            rp.advance();
          }
      }
    }
    return;
  }
  if (warp == C::CW + 1) {  // ---------------- epilogue
    RingPos<C::NP> up;
    RingPos<kNDQ> dq;
    for (int unit = blockIdx.x; unit < total; unit += gridDim.x) {
      const FUnit fu = decode_fused(p, sp.plan, unit);
      if (!fu.sample) {
        const Unit& un = fu.u;
        const T* prow = PL + row_off(d, un.b, un.slot, un.i);
        const T* qrow = QL + row_off(d, un.b, un.slot, un.i);
        const bool branch_row = (un.slot == 0 && un.i == un.in.s);
        const int ntok = branch_row ? d.K : 1;
        int x = 0;
        float lpx = 0.f, lqx = 0.f, uu = 0.f;
        int64_t et = 0;
        if (lane < ntok) {
          et = ent(d, un.b, branch_row ? lane : un.slot, un.i);
          x = __ldg(p.tok + et);
          uu = __ldg(p.u + et);
          if (x >= 0 && x < d.V) {
            lpx = ld_scalar(prow + x);
            lqx = ld_scalar(qrow + x);
          }
        }
        mbar_wait(&S.pfull[up.stage], up.phase);
        RowStat ps = lane < C::CW ? S.part[up.stage][0][lane] : rowstat_empty();
        RowStat qs = lane < C::CW ? S.part[up.stage][1][lane] : rowstat_empty();
        const uint2 cand = lane < C::CW ? S.cand[up.stage][lane] : make_uint2(0xffffffffu, 0u);
        __syncwarp();
        if (lane == 0) mbar_arrive(&S.pempty[up.stage]);
        up.advance();
        const float qmw = qs.m;
        ps = warp_reduce_state(ps);  // idx: p's unused, q's resolved below
        qs = warp_reduce_state(qs);
        qs.idx = resolve_argmax<C, T>(qmw, cand, qs.m, qrow, nvec_last, nchunks);
        warp_epilogue<T>(p, un, ps, qs, qrow, x, lpx, lqx, uu, et);
        continue;
      }
      // ---- sample unit
      mbar_wait(&S.dfull[dq.stage], dq.phase);
      const P2Desc D = S.desc[dq.stage];
      const int b = D.b;
      const SeqInfo in = p.info[b];
      mbar_wait(&S.pfull[up.stage], up.phase);
      int kind = D.kind, y = -1, st = 0;
      double mass = 0.0;
      if (kind != 0) {
        const float4 rs = (kind == 1) ? D.rs : S.brs[dq.stage];
        const int cls = z_class(rs.y) | z_class(rs.w);
        if (cls) {
          kind = 0;
          st |= cls;
        } else {
          const T* prow = PL + row_off(d, b, D.slot, D.row);
          const T* qrow = QL + row_off(d, b, D.slot, D.row);
          bool resid = (kind == 1);
          double R = 0.0;
          y = sample_segments<T>(prow, qrow, row_bytes, d.V, S.seg[up.stage], nseg, resid, rs.x, rs.z, rs.y / rs.w,
                                 __ldg(sp.us + b), st, &R);
          mass = R / (double)rs.y;  // back to probability mass
        }
      }
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&S.pempty[up.stage]);
        mbar_arrive(&S.dempty[dq.stage]);
      }
      up.advance();
      dq.advance();
      commit_seq(d, p.tok, p.status,
                 CommitOut{sp.sel_k, sp.commit_len, sp.out_tok, sp.y_tok, sp.y_kind, sp.offsets, sp.packed_tok,
                           sp.path_rolled, sp.branch_discarded, sp.keep_mask, sp.resid_mass},
                 b, in, D.ksel, D.npath, kind, y, mass, st);
      __syncwarp();
      int last = 0;
      if (lane == 0) {
        __threadfence();
        last = (atomicAdd(sp.done_cnt, 1) == d.B - 1);
      }
      last = __shfl_sync(0xffffffffu, last, 0);
      if (last) {
        __threadfence();
        warp_offsets(d.B, d.G, sp.commit_len, sp.out_tok, sp.offsets, sp.packed_tok);
        if (lane == 0) *sp.done_cnt = 0;
      }
    }
    return;
  }
  // ---------------- consumers
  RingPos<C::NS> rp;
  RingPos<C::NP> up;
  RingPos<kNDQ> dq;
  for (int unit = blockIdx.x; unit < total; unit += gridDim.x) {
    const FUnit fu = decode_fused(p, sp.plan, unit);
    if (!fu.sample) {
      LazyAcc<false, 4> pa;
      LazyAcc<true, 4> qa;
      pa.init();
      qa.init();
      for (int c = 0; c < nchunks - 1; ++c) {
        StageRegs<C> r;
        mbar_wait(&S.full[rp.stage], rp.phase);
        load_stage<C, T, true>(S.buf[rp.stage][0], S.buf[rp.stage][1], 0, r);
        __syncwarp();
        if (lane == 0) mbar_arrive(&S.empty[rp.stage]);
        rp.advance();
        compute_stage<C, T>(r, c, pa, qa);
      }
      {
        StageRegs<C> r;
        mbar_wait(&S.full[rp.stage], rp.phase);
        load_stage<C, T, false>(S.buf[rp.stage][0], S.buf[rp.stage][1], nvec_last, r);
        __syncwarp();
        if (lane == 0) mbar_arrive(&S.empty[rp.stage]);
        rp.advance();
        compute_stage<C, T>(r, nchunks - 1, pa, qa);
      }
      uint2 cand;
      const RowStat ps = warp_part<C, T, false>(pa, nullptr, nvec_last, nchunks);
      const RowStat qs = warp_part_deferred(qa, cand);
      if (lane == 0) {
        mbar_wait(&S.pempty[up.stage], up.phase ^ 1u);
        S.part[up.stage][0][warp] = ps;
        S.part[up.stage][1][warp] = qs;
        S.cand[up.stage][warp] = cand;
        mbar_arrive(&S.pfull[up.stage]);
      }
      __syncwarp();
      up.advance();
      continue;
    }
    // ---- sample unit
    mbar_wait(&S.dfull[dq.stage], dq.phase);
    const P2Desc D = S.desc[dq.stage];
    if (lane == 0) mbar_wait(&S.pempty[up.stage], up.phase ^ 1u);  // seg slot free
    __syncwarp();
    float* seg = S.seg[up.stage];
    if (D.kind == 2) {  // bonus row: its softmax state first (pass 0), then p sums
      LazyAcc<false, 4> a;
      a.init();
      for (int c = 0; c < nchunks; ++c) {
        const int nvec = (c == nchunks - 1) ? nvec_last : C::CHUNK / 16;
        mbar_wait(&S.full[rp.stage], rp.phase);
        uint4 x[C::VPT];
#pragma unroll
        for (int j = 0; j < C::VPT; ++j) {
          const int v = tid + j * C::CT;
          x[j] = (v < nvec) ? lds128(S.buf[rp.stage][0] + v * 16) : neg_inf_vec<T>();
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&S.empty[rp.stage]);
        rp.advance();
        float f[C::VPT * E];
#pragma unroll
        for (int j = 0; j < C::VPT; ++j) Vec<T>::unpack(x[j], f + j * E);
        a.template add<C::VPT * E>(f, c);
      }
      RowStat s = fold_lazy(a);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s = combine(s, shfl_xor(s, o));
      if (lane == 0) S.red[warp] = s;
      consumer_sync(C::CT);
      RowStat r = S.red[0];
#pragma unroll
      for (int j = 1; j < C::CW; ++j) r = combine(r, S.red[j]);
      const RowOut o = finish(r);
      if (tid == 0) S.brs[dq.stage] = make_float4(o.MS, z_store(o), 0.f, 1.f);
      consumer_sync(C::CT);
      step_seg_pass<StepSmem<C>, C, T, false>(S, rp, seg, nchunks, nvec_last, o.finite, o.MS, 0.f, 0.f);
    } else if (D.kind == 1) {
      const bool ok = (z_class(D.rs.y) | z_class(D.rs.w)) == 0;
      step_seg_pass<StepSmem<C>, C, T, true>(S, rp, seg, nchunks, nvec_last, ok, D.rs.x, D.rs.z, D.rs.y / D.rs.w);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&S.pfull[up.stage]);
    up.advance();
    dq.advance();
  }
}

template <class C, typename T>
static sb_status launch_step_tma(const StepParams& sp, cudaStream_t s) {
  const int smem = (int)sizeof(StepSmem<C>);
  if (ensure_smem<k_step_tma<C, T>>(smem) != cudaSuccess) return SB_ERR_CUDA;
  k_step_tma<C, T><<<num_sms(), C::THREADS, smem, s>>>(sp);
  return cuda_status(cudaGetLastError());
}

// ---------------------------------------------------------------- adaptive step in one launch
// k_astep: [draft confidence -> adaptive gamma] -> verify -> select for small batches
// (PAPER Eq. 6-7 P194-220, §3 P94, Alg. 1 P523-557, Eq. 9
// P236-241).  One persistent CTA per SM with k_rows_tma's warp roles (TMA bulk ring,
// consumer warps, epilogue warps); work items are grabbed in one global order
// (atomicAdd on ctr[0]):
//   [0, B G)            confidence items: slot-0 draft row (b, i), q only;
//   then queue entries  verify items (b, slot, i), appended by the CTA that completes
//                       the last confidence row of b (gamma_b = max(1, stop_b) known);
//   then B sample items appended by the CTA that completes b's last verify item (n_k).
// A producer waits for the entry it grabbed to be published; every entry depends only
// on items grabbed before it (whose pipelines never wait on later items), so with all
// CTAs co-resident the waits end.  The three phases overlap across sequences instead of
// each ending with a grid-wide drain, and the confidence pass's q-row states replace the
// slot-0 draft rows in the verify items (sb_verify_branches_reuse).  Every arithmetic
// step is the separate kernels' (LazyAcc, warp_part*, resolve_argmax, conf_epilogue,
// warp_epilogue, step_seg_pass, sample_segments), so results agree with them bit for bit.
struct AItem {
  int type;  // 0 confidence, 1 verify, 2 sample, -1 exit
  int b, slot, i;
  int po;                        // verify: p only (q state from the confidence pass)
  int ksel, npath, kind;         // sample: Eq. 9 / Alg. 1 decision (as P2Desc)
  float4 rs;                     // sample: row state of the residual row
};
constexpr int kAI = 8;  // items in flight between the producer and the other roles

struct AStepParams {
  RowsParams r;       // verify outputs and workspace (r.qreuse = confidence row states)
  ConfParams c;       // confidence outputs, K = 1 slot-0 view
  const float* us;
  const int* bpos;
  const int* gamma_in;  // non-adaptive step: gamma_b (NULL -> G)
  int adaptive;         // 1: confidence items first; 0: plan items (gamma_b from the input)
  int rule;
  int *ctr;           // [0] grab, [1] verify entries reserved, [2] sequences planned, [3] samples queued,
                      // [4] exit count, [5] committed sequences
  int4* qv;           // verify entries (b, slot, i)
  int* qv_pub;
  int qcap;           // capacity of qv / qv_pub (B K (G+1))
  int* sq;            // sample queue: sequences
  int* sq_pub;
  CommitOut co;
};

template <class C>
struct AStepSmem {
  uint64_t full[C::NS], empty[C::NS];
  uint64_t pfull[C::NP], pempty[C::NP];
  uint64_t ifull[kAI], iempty[kAI];
  AItem item[kAI];
  RowStat part[C::NP][2][C::CW];
  uint2 cand[C::NP][C::CW];
  float4 brs[C::NP];  // bonus-row softmax state computed by the consumers
  RowStat red[C::CW];
  int s_last[C::NE];
  float seg[C::NP][kSegMax];
  alignas(128) uint8_t buf[C::NS][2][C::CHUNK];
};


// Sequence b's verify items once gamma_b is known (k_plan's clamps and unit layout): its
// SeqInfo, then one reservation of its entries in the verify queue, published entry by
// entry; ctr[2] counts planned sequences (after the reservation, so ctr[1] is final once
// it reaches B).  One warp.
__device__ __forceinline__ void astep_plan(const AStepParams& ap, int b, int g) {
  const Dims& d = ap.r.d;
  const int lane = threadIdx.x & 31;
  const int s0 = ap.bpos ? __ldg(ap.bpos + b) : 0;
  const SeqInfo in = astep_seqinfo(g, s0, d.G);
  const int per = in.Lr - 1 - in.s;
  const int count = in.Lr + (d.K - 1) * per;
  int start = 0;
  if (lane == 0) {
    const_cast<SeqInfo*>(ap.r.info)[b] = in;  // (read-only for the other kernels)
    start = atomicAdd(ap.ctr + 1, count);
  }
  start = __shfl_sync(0xffffffffu, start, 0);
  for (int j = lane; j < count; j += 32) {
    int slot, i;
    if (j < in.Lr) { slot = 0; i = j; }
    else { const int jj = j - in.Lr; slot = 1 + jj / per; i = in.s + 1 + jj % per; }
    ap.qv[start + j] = make_int4(b, slot, i, 0);
  }
  __threadfence();
  __syncwarp();
  for (int j = lane; j < count; j += 32) st_rel(ap.qv_pub + start + j, 1);
  __syncwarp();
  if (lane == 0) {
    __threadfence();
    atomicAdd(ap.ctr + 2, 1);
  }
}

// One chunk of one row into its accumulator (FIRST: the row's first chunk).
template <class C, typename T, bool kQ, bool FIRST>
__device__ __forceinline__ void acc_chunk(LazyAcc<kQ, 4>& a, const uint4* x, int c) {
  constexpr int E = Vec<T>::E;
  if constexpr (sizeof(T) == 2) {
    acc_vecs_bf16<C::VPT, kQ, FIRST>(a, x, c);
  } else {
    float f[C::VPT * E];
#pragma unroll
    for (int j = 0; j < C::VPT; ++j) Vec<T>::unpack(x[j], f + j * E);
    a.template add<C::VPT * E, FIRST>(f, c);
  }
}

template <class C, typename T, int MINB>
__global__ void __launch_bounds__(C::ROWS_THREADS, MINB) k_astep(AStepParams ap) {
  constexpr int E = Vec<T>::E;
  extern __shared__ __align__(128) uint8_t smem_raw[];
  AStepSmem<C>& S = *reinterpret_cast<AStepSmem<C>*>(smem_raw);
  const RowsParams& p = ap.r;
  const Dims& d = p.d;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < C::NS; ++s) {
      mbar_init(&S.full[s], 1);
      mbar_init(&S.empty[s], C::CW);
    }
    for (int s = 0; s < C::NP; ++s) {
      mbar_init(&S.pfull[s], C::CW);
      mbar_init(&S.pempty[s], 1);
    }
    for (int s = 0; s < kAI; ++s) {
      mbar_init(&S.ifull[s], 1);
      mbar_init(&S.iempty[s], C::CW + 1);
    }
    fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0) SB_TRACE_AT(sb_trace_astep, 0, 0);
  pdl_wait();
  if (tid == 0) SB_TRACE_AT(sb_trace_astep, 0, 1);
  const int G = d.G, nconf = ap.adaptive ? d.B * G : d.B;  // confidence or plan items first
  const T* PL = static_cast<const T*>(p.PL);
  const T* QL = static_cast<const T*>(p.QL);
  const uint32_t row_bytes = (uint32_t)d.V * sizeof(T);
  const int nchunks = (row_bytes + C::CHUNK - 1) / C::CHUNK;
  const int nvec_last = (int)(row_bytes - (uint32_t)(nchunks - 1) * C::CHUNK) / 16;
  const int nseg = nchunks * (C::CHUNK / kSegBytes);

  if (warp == C::CW) {  // ---------------- producer: grab, wait for the entry, publish, stream
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      RingPos<C::NS> rp;
      RingPos<kAI> iq;
      int exits = 0;
      int tli = 0;
      (void)tli;
      // one grab kept in flight: the next item's atomicAdd round trip (~1 us when 148
      // producers contend) overlaps this item's decode and copies
      // the first-phase items (confidence / plan) are dealt statically, CTA c taking c,
      // c + grid, ...; the dependent items that follow come from one global counter
      int kst = 0;
      auto next_item = [&]() -> int {
#ifdef SB_ASTEP_BLOCKED  // experiment: CTA c takes a contiguous block of the first-phase items
        const int b0 = (int)((int64_t)blockIdx.x * nconf / gridDim.x), b1 = (int)((int64_t)(blockIdx.x + 1) * nconf / gridDim.x);
        const int gs = b0 + kst < b1 ? b0 + kst : nconf;
#else
        const int gs = (int)blockIdx.x + kst * (int)gridDim.x;
#endif
        if (gs < nconf) { ++kst; return gs; }
        return nconf + atomicAdd(ap.ctr, 1);
      };
      int gnext = next_item();
      while (exits < C::NE) {
        AItem it{};
        if (exits > 0) {
          it.type = -1;
        } else {
          const int g = gnext;
          gnext = next_item();
          if (g < nconf) {
            if (ap.adaptive) { it.type = 0; it.b = g / G; it.slot = 0; it.i = g % G; }
            else { it.type = 3; it.b = g; }
          } else {
            const int e = g - nconf;
            for (uint32_t tries = 0;; ++tries) {
              // (an index past the queue's capacity can only be a sample / exit index: never
              // probe qv_pub there, the words after it belong to the sample queue)
              if (e < ap.qcap && ld_acq(ap.qv_pub + e)) {
                const int4 q = __ldcg(ap.qv + e);
                ap.qv_pub[e] = 0;  // leave the workspace re-usable
                it.type = 1; it.b = q.x; it.slot = q.y; it.i = q.z;
                it.po = ap.adaptive && (q.y == 0 && q.z < G);  // q state from the confidence item
                break;
              }
              if (ld_acq(ap.ctr + 2) == d.B) {  // every sequence planned: the verify count is final
                const int nv = ld_acq(ap.ctr + 1);
                if (e >= nv) {
                  const int sidx = e - nv;
                  if (sidx >= d.B) { it.type = -1; break; }
                  while (!ld_acq(ap.sq_pub + sidx)) __nanosleep(64);
                  const int b = __ldcg(ap.sq + sidx);
                  ap.sq_pub[sidx] = 0;
                  // Eq. 9 / Alg. 1 decision of sequence b (as k_step_tma / k_select_tma)
                  const SeqInfo in = ldcg_seqinfo(p.info + b);
                  int ksel = -1, besttok = 0;
                  float bestkey = 0.f;
                  for (int k = 0; k < d.K; ++k) {  // A = {k : n_k > s_b} (P239, P540)
                    if (__ldcg(p.n_acc + (int64_t)b * d.K + k) <= in.s) continue;
                    const int xk = __ldg(p.tok + ent(d, b, k, in.s));
                    const float key = (ap.rule == SB_SELECT_ALG1) ? __ldg(p.u + ent(d, b, k, in.s))
                                                                  : ld_scalar(PL + row_off(d, b, 0, in.s) + xk);
                    bool better;
                    if (ksel < 0) better = true;
                    else if (ap.rule == SB_SELECT_ALG1) better = key > bestkey;
                    else better = key > bestkey || (key == bestkey && xk < besttok);
                    if (better) { ksel = k; bestkey = key; besttok = xk; }
                  }
                  it.type = 2; it.b = b; it.ksel = ksel;
                  if (ksel < 0) {
                    it.npath = min(__ldcg(p.n_acc + (int64_t)b * d.K), in.s);  // rollback (P655)
                    it.kind = 1; it.i = it.npath; it.slot = 0;
                  } else {
                    it.npath = __ldcg(p.n_acc + (int64_t)b * d.K + ksel);
                    if (it.npath < in.L) { it.kind = 1; it.i = it.npath; it.slot = (it.npath <= in.s) ? 0 : ksel; }
                    else if (in.s < in.g) { it.kind = 2; it.i = in.g; it.slot = ksel; }  // bonus (P94)
                    else { it.kind = 0; it.i = 0; it.slot = 0; }                          // (P237)
                  }
                  it.rs = (it.kind == 1) ? __ldcg(p.rowstat + ent(d, b, it.slot, it.i)) : make_float4(0.f, 1.f, 0.f, 1.f);
                  break;
                }
              }
              __nanosleep(64);
              if (tries > (1u << 26)) __trap();  // watchdog (seconds): a publication never came
            }
          }
        }
        if (it.type < 0) ++exits;
#ifdef SB_TRACE
        if (tli < 60) { SB_TRACE_AT(sb_trace_astep, 1, 2 + tli); sb_trace_astep[blockIdx.x][0][2 + tli] = it.type + 1; }
        ++tli;
#endif
        mbar_wait(&S.iempty[iq.stage], iq.phase ^ 1u);
        S.item[iq.stage] = it;
        mbar_arrive(&S.ifull[iq.stage]);
        iq.advance();
        if (it.type < 0 || it.type == 3) continue;  // exit / plan items carry no rows
        const char* prow = reinterpret_cast<const char*>(PL + row_off(d, it.b, it.slot, it.i));
        const char* qrow = reinterpret_cast<const char*>(QL + row_off(d, it.b, it.slot, it.i));
        if (it.type == 0 || (it.type == 1 && it.po)) {  // one row: chunks c, c + 1 in one stage
          const char* row = it.type == 0 ? qrow : prow;
          for (int c = 0; c < nchunks; c += 2) {
            const uint32_t b0 = min((uint32_t)C::CHUNK, row_bytes - (uint32_t)c * C::CHUNK);
            const uint32_t b1 = c + 1 < nchunks ? min((uint32_t)C::CHUNK, row_bytes - (uint32_t)(c + 1) * C::CHUNK) : 0u;
            mbar_wait(&S.empty[rp.stage], rp.phase ^ 1u);
            mbar_expect_tx(&S.full[rp.stage], b0 + b1);
            bulk_g2s(S.buf[rp.stage][0], row + (size_t)c * C::CHUNK, b0, &S.full[rp.stage], pol);
            if (b1) bulk_g2s(S.buf[rp.stage][1], row + (size_t)(c + 1) * C::CHUNK, b1, &S.full[rp.stage], pol);
            rp.advance();
          }
#ifdef SB_TRACE
          if (tli - 1 < 60) SB_TRACE_AT(sb_trace_astep, 7, 2 + tli - 1);  // last chunk issued
#endif
          continue;
        }
        const bool wp = true, wq = (it.type == 1) || (it.type == 2 && it.kind == 1);
        const int passes = (it.type == 2) ? (it.kind == 1 ? 1 : (it.kind == 2 ? 2 : 0)) : 1;
        for (int pass = 0; pass < passes; ++pass)
          for (int c = 0; c < nchunks; ++c) {
            const uint32_t bytes = min((uint32_t)C::CHUNK, row_bytes - (uint32_t)c * C::CHUNK);
            mbar_wait(&S.empty[rp.stage], rp.phase ^ 1u);
            mbar_expect_tx(&S.full[rp.stage], ((wp ? 1 : 0) + (wq ? 1 : 0)) * bytes);
            if (wp) bulk_g2s(S.buf[rp.stage][0], prow + (size_t)c * C::CHUNK, bytes, &S.full[rp.stage], pol);
            if (wq) bulk_g2s(S.buf[rp.stage][1], qrow + (size_t)c * C::CHUNK, bytes, &S.full[rp.stage], pol);
            rp.advance();
          }
#ifdef SB_TRACE
        if (tli - 1 < 60) SB_TRACE_AT(sb_trace_astep, 7, 2 + tli - 1);  // last chunk issued
#endif
      }
    }
  } else if (warp > C::CW) {  // ---------------- epilogue warps: warp e takes items e, e + NE, ...
    const int e = warp - C::CW - 1;
    for (int li = e;; li += C::NE) {
      const int islot = li % kAI;
      mbar_wait(&S.ifull[islot], (uint32_t)(li / kAI) & 1u);
      const AItem it = S.item[islot];
      if (it.type < 0) break;
      const int ps_slot = li % C::NP;
      const uint32_t pph = (uint32_t)(li / C::NP) & 1u;
      if (it.type == 0) {  // ---- confidence row (b, i): statistic, Eq. 6 / 7; the group's last plans b
        const T* qrow = QL + row_off(d, it.b, 0, it.i);
        mbar_wait(&S.pfull[ps_slot], pph);
        RowStat qs = lane < C::CW ? S.part[ps_slot][1][lane] : rowstat_empty();
        const uint2 cand = lane < C::CW ? S.cand[ps_slot][lane] : make_uint2(0xffffffffu, 0u);
        __syncwarp();
        if (lane == 0) mbar_arrive(&S.pempty[ps_slot]);
        const float qmw = qs.m;
        qs = warp_reduce_state(qs);
        qs.idx = resolve_argmax<C, T>(qmw, cand, qs.m, qrow, nvec_last, nchunks);
        conf_epilogue(ap.c, it.b, it.i, qrow, qs, lane, &S.s_last[e], [] { __syncwarp(); });
        if (S.s_last[e]) {  // gamma_b = max(1, stop_b) is known: b's verify items
          __threadfence();
          astep_plan(ap, it.b, __ldcg(ap.c.gamma_next + it.b));
        }
      } else if (it.type == 3) {  // ---- plan item (non-adaptive step): gamma_b from the input
        mbar_wait(&S.pfull[ps_slot], pph);  // (empty partial slot: its phase stays in step)
        __syncwarp();
        if (lane == 0) mbar_arrive(&S.pempty[ps_slot]);
        astep_plan(ap, it.b, ap.gamma_in ? __ldg(ap.gamma_in + it.b) : d.G);
      } else if (it.type == 1) {  // ---- verify row pair: token tests, n_k (warp_epilogue)
        Unit un;
        un.b = it.b; un.slot = it.slot; un.i = it.i; un.in = ldcg_seqinfo(p.info + it.b);
        const T* prow = PL + row_off(d, un.b, un.slot, un.i);
        const T* qrow = QL + row_off(d, un.b, un.slot, un.i);
        const bool branch_row = (un.slot == 0 && un.i == un.in.s);
        const int ntok = branch_row ? d.K : 1;
        int x = 0;
        float lpx = 0.f, lqx = 0.f, uu = 0.f;
        int64_t et = 0;
        if (lane < ntok && un.i < un.in.L) {
          et = ent(d, un.b, branch_row ? lane : un.slot, un.i);
          x = __ldg(p.tok + et);
          uu = __ldg(p.u + et);
          if (x >= 0 && x < d.V) {
            lpx = ld_scalar(prow + x);
            lqx = ld_scalar(qrow + x);
          } else {
            lpx = lqx = -CUDART_INF_F;
          }
        }
        RowStat qr;
        if (it.po) qr = ldcg_rowstat(p.qreuse + (int64_t)un.b * G + un.i);
        mbar_wait(&S.pfull[ps_slot], pph);
        RowStat ps = lane < C::CW ? S.part[ps_slot][0][lane] : rowstat_empty();
        RowStat qs = lane < C::CW ? S.part[ps_slot][1][lane] : rowstat_empty();
        const uint2 cand = lane < C::CW ? S.cand[ps_slot][lane] : make_uint2(0xffffffffu, 0u);
        __syncwarp();
        if (lane == 0) mbar_arrive(&S.pempty[ps_slot]);
        const float qmw = qs.m;
        ps = warp_reduce_state(ps);
        qs = warp_reduce_state(qs);
        if (it.po) qs = qr;
        else qs.idx = resolve_argmax<C, T>(qmw, cand, qs.m, qrow, nvec_last, nchunks);
        warp_epilogue<T>(p, un, ps, qs, qrow, x, lpx, lqx, uu, et);
      } else {  // ---- sample: locate us * R, rescan one segment, commit (as k_step_tma)
        const int b = it.b;
        const SeqInfo in = ldcg_seqinfo(p.info + b);
        mbar_wait(&S.pfull[ps_slot], pph);
        int kind = it.kind, y = -1, st = 0;
        double mass = 0.0;
        if (kind != 0) {
          const float4 rs = (kind == 1) ? it.rs : S.brs[ps_slot];
          const int cls = z_class(rs.y) | z_class(rs.w);
          if (cls) {
            kind = 0;
            st |= cls;
          } else {
            const T* prow = PL + row_off(d, b, it.slot, it.i);
            const T* qrow = QL + row_off(d, b, it.slot, it.i);
            bool resid = (kind == 1);
            double R = 0.0;
            y = sample_segments<T>(prow, qrow, row_bytes, d.V, S.seg[ps_slot], nseg, resid, rs.x, rs.z,
                                   rs.y / rs.w, __ldg(ap.us + b), st, &R);
            mass = R / (double)rs.y;  // back to probability mass
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&S.pempty[ps_slot]);
        commit_seq(d, p.tok, p.status, ap.co, b, in, it.ksel, it.npath, kind, y, mass, st);
        __syncwarp();
        int last = 0;
        if (lane == 0) {
          __threadfence();
          last = (atomicAdd(ap.ctr + 5, 1) == d.B - 1);
        }
        last = __shfl_sync(0xffffffffu, last, 0);
        if (last) {
          __threadfence();
          warp_offsets(d.B, G, ap.co.commit_len, ap.co.out_tok, ap.co.offsets, ap.co.packed_tok);
          if (lane == 0) ap.ctr[5] = 0;
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&S.iempty[islot]);
      if (lane == 0 && li < 60) SB_TRACE_AT(sb_trace_astep, 2, 2 + li);
    }
  } else {  // ---------------- consumers
    RingPos<C::NS> rp;
    for (int li = 0;; ++li) {
      const int islot = li % kAI;
      mbar_wait(&S.ifull[islot], (uint32_t)(li / kAI) & 1u);
      const AItem it = S.item[islot];
      if (it.type < 0) break;
      const int ps_slot = li % C::NP;
      const uint32_t pph = (uint32_t)(li / C::NP) & 1u;
      if (it.type == 3) {  // plan item: no rows; keep the partial slot's phase in step
        if (lane == 0) {
          mbar_wait(&S.pempty[ps_slot], pph ^ 1u);
          mbar_arrive(&S.pfull[ps_slot]);
        }
        __syncwarp();
      } else if (it.type != 2) {
        LazyAcc<false, 4> pa;
        LazyAcc<true, 4> qa;
        pa.init();
        qa.init();
        if (it.type == 0 || it.po) {  // one row: chunks c and c + 1 share a stage
          for (int c = 0; c < nchunks; c += 2) {
            const int n0 = (c < nchunks - 1) ? C::CHUNK / 16 : nvec_last;
            const bool has1 = c + 1 < nchunks;
            const int n1 = has1 ? ((c + 1 < nchunks - 1) ? C::CHUNK / 16 : nvec_last) : 0;
            StageRegs<C> r;
            mbar_wait_spin(&S.full[rp.stage], rp.phase);
            if (c == 0 && tid == 0 && li < 60) SB_TRACE_AT(sb_trace_astep, 4, 2 + li);
#pragma unroll
            for (int j = 0; j < C::VPT; ++j) {
              const int v = tid + j * C::CT;
              r.p[j] = v < n0 ? lds128(S.buf[rp.stage][0] + v * 16) : neg_inf_vec<T>();
              r.q[j] = v < n1 ? lds128(S.buf[rp.stage][1] + v * 16) : neg_inf_vec<T>();
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&S.empty[rp.stage]);
            rp.advance();
#ifdef SB_ASTEP_NOMATH  // experiment: data-rate ceiling of the k_astep structure (wrong results)
            if (true) { qa.z[0] += __uint_as_float(r.p[0].x & 1u) + __uint_as_float(r.q[0].x & 1u); } else
#endif
            if (it.type == 0) {
              if (c == 0) acc_chunk<C, T, true, true>(qa, r.p, c);
              else acc_chunk<C, T, true, false>(qa, r.p, c);
              if (has1) acc_chunk<C, T, true, false>(qa, r.q, c + 1);
            } else {
              if (c == 0) acc_chunk<C, T, false, true>(pa, r.p, c);
              else acc_chunk<C, T, false, false>(pa, r.p, c);
              if (has1) acc_chunk<C, T, false, false>(pa, r.q, c + 1);
            }
          }
        } else {
          for (int c = 0; c < nchunks; ++c) {
            const bool full = c < nchunks - 1;
            const int nvec = full ? C::CHUNK / 16 : nvec_last;
            StageRegs<C> r;
            mbar_wait_spin(&S.full[rp.stage], rp.phase);
            if (c == 0 && tid == 0 && li < 60) SB_TRACE_AT(sb_trace_astep, 4, 2 + li);
            if (full) load_stage<C, T, true>(S.buf[rp.stage][0], S.buf[rp.stage][1], nvec, r);
            else load_stage<C, T, false>(S.buf[rp.stage][0], S.buf[rp.stage][1], nvec, r);
            __syncwarp();
            if (lane == 0) mbar_arrive(&S.empty[rp.stage]);
            rp.advance();
#ifdef SB_ASTEP_NOMATH
            if (true) { pa.z[0] += __uint_as_float(r.p[0].x & 1u) + __uint_as_float(r.q[0].x & 1u); } else
#endif
            if (c == 0) compute_stage<C, T, true>(r, c, pa, qa);
            else compute_stage<C, T, false>(r, c, pa, qa);
          }
        }
        if (tid == 0 && li < 60) SB_TRACE_AT(sb_trace_astep, 5, 2 + li);
        uint2 cand = make_uint2(0xffffffffu, 0u);
#ifdef SB_ASTEP_NORED  // experiment: the consumers' per-item warp reductions removed (wrong results)
        RowStat ps = fold_lazy(pa), qs = fold_lazy(qa);
#else
        const RowStat ps = (it.type == 1) ? warp_part<C, T, false>(pa, nullptr, nvec_last, nchunks) : rowstat_empty();
        const RowStat qs = it.po ? rowstat_empty() : warp_part_deferred(qa, cand);
#endif
        if (tid == 0 && li < 60) SB_TRACE_AT(sb_trace_astep, 6, 2 + li);
        if (lane == 0) {
          mbar_wait(&S.pempty[ps_slot], pph ^ 1u);
          S.part[ps_slot][0][warp] = ps;
          S.part[ps_slot][1][warp] = qs;
          S.cand[ps_slot][warp] = cand;
          mbar_arrive(&S.pfull[ps_slot]);
        }
        __syncwarp();
      } else {  // sample item: one sum per 1 KB segment (bonus rows: their softmax state first)
        if (lane == 0) mbar_wait(&S.pempty[ps_slot], pph ^ 1u);  // seg slot free
        __syncwarp();
        float* seg = S.seg[ps_slot];
        if (it.kind == 2) {
          LazyAcc<false, 4> a;
          a.init();
          for (int c = 0; c < nchunks; ++c) {
            const int nvec = (c == nchunks - 1) ? nvec_last : C::CHUNK / 16;
            mbar_wait(&S.full[rp.stage], rp.phase);
            uint4 x[C::VPT];
#pragma unroll
            for (int j = 0; j < C::VPT; ++j) {
              const int v = tid + j * C::CT;
              x[j] = (v < nvec) ? lds128(S.buf[rp.stage][0] + v * 16) : neg_inf_vec<T>();
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&S.empty[rp.stage]);
            rp.advance();
            float f[C::VPT * E];
#pragma unroll
            for (int j = 0; j < C::VPT; ++j) Vec<T>::unpack(x[j], f + j * E);
            a.template add<C::VPT * E>(f, c);
          }
          RowStat s = fold_lazy(a);
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) s = combine(s, shfl_xor(s, o));
          if (lane == 0) S.red[warp] = s;
          consumer_sync(C::CT);
          RowStat rr = S.red[0];
#pragma unroll
          for (int j = 1; j < C::CW; ++j) rr = combine(rr, S.red[j]);
          const RowOut o = finish(rr);
          if (tid == 0) S.brs[ps_slot] = make_float4(o.MS, z_store(o), 0.f, 1.f);
          consumer_sync(C::CT);
          step_seg_pass<AStepSmem<C>, C, T, false>(S, rp, seg, nchunks, nvec_last, o.finite, o.MS, 0.f, 0.f);
        } else if (it.kind == 1) {
          const bool ok = (z_class(it.rs.y) | z_class(it.rs.w)) == 0;
          step_seg_pass<AStepSmem<C>, C, T, true>(S, rp, seg, nchunks, nvec_last, ok, it.rs.x, it.rs.z,
                                                  it.rs.y / it.rs.w);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&S.pfull[ps_slot]);
      }
      if (lane == 0) mbar_arrive(&S.iempty[islot]);
      if (tid == 0 && li < 60) SB_TRACE_AT(sb_trace_astep, 3, 2 + li);
    }
  }
  // ---------------- exit: the last CTA out resets the grab / queue counters
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    if (atomicAdd(ap.ctr + 4, 1) == (int)gridDim.x - 1) {
      ap.ctr[0] = 0; ap.ctr[1] = 0; ap.ctr[2] = 0; ap.ctr[3] = 0; ap.ctr[4] = 0;
    }
  }
}

template <class C, typename T, int MINB>
static sb_status launch_astep(const AStepParams& ap, cudaStream_t s) {
  const int smem = (int)sizeof(AStepSmem<C>);
  if (ensure_smem<k_astep<C, T, MINB>>(smem) != cudaSuccess) return SB_ERR_CUDA;
  int occ = 0;  // every CTA must be resident (producers wait on each other's publications)
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_astep<C, T, MINB>, C::ROWS_THREADS, smem);
  if (occ < MINB) return SB_ERR_UNSUPPORTED;
  return cuda_status(launch_pdl(k_astep<C, T, MINB>, dim3(MINB * num_sms()), dim3(C::ROWS_THREADS), smem, s, ap));
}

// sb_step_adaptive's single-launch path (called after its argument checks).
// w / cw: the step and confidence workspaces; outputs as sb_step_adaptive documents.
// Default: small problems (<= 4096 physical rows per slot set: C2's 64 x 4 x 9), where the
// three kernels' launch / ramp / drain dominate (C2 step 77.6 -> 71.3 us); on C3 (17408)
// the three kernels are faster (0.962 vs 0.992 ms).  SB_ASTEP=1 / 0 forces it on / off.
bool astep_eligible(const sb_dims* dd, const void* PL, const void* QL) {
  const char* e = getenv("SB_ASTEP");
  if (e && e[0] == '0') return false;
  if (tma_disabled() || sharded(dd)) return false;
  if (!vec_ok(dd, PL) || !vec_ok(dd, QL)) return false;
  const size_t rb = (size_t)dd->V * elem_size(dd);
  if (rb % 16 || rb > (size_t)kSegMax * kSegBytes) return false;
  return (e && e[0] == '1') || (size_t)dd->B * dd->K * (dd->G + 1) <= 4096;
}

#ifndef SB_AG_CW  // (SB_AG_CW / SB_AG_NS / SB_AG_NE: experiment builds)
using RCA = RC<16, 6, 2, 4, 4>;  // k_astep: 16 consumer warps, 6 x 32 KB stages, 4 epilogue warps
#else
#ifndef SB_AG_NE
#define SB_AG_NE 4
#endif
using RCA = RC<SB_AG_CW, SB_AG_NS, 2, 4, SB_AG_NE>;
#endif
// (two CTAs per SM of 8 consumer warps, 5 x 16 KB stages each, measured 72.3 vs 71.6 us on C2)

sb_status astep_run(const sb_dims* dd, const Workspace& w, const Workspace* cw, const void* PL, const void* QL,
                    const int32_t* tok, const float* u, const float* us, const int32_t* gamma,
                    const int32_t* branch_pos,
                    sb_select_rule rule, float eps, int32_t k_max, float* c_top1, int32_t* c_id, float* c_ent,
                    float* c_stat, int32_t* c_stop, int32_t* c_knext, int32_t* c_gamma, float* lse_p, float* lse_q,
                    float* p_tok, float* q_tok, uint32_t* acc_mask, int32_t* n_acc, float* top1_q,
                    int32_t* top1_id_q, float* entropy_q, int32_t* status, int32_t* sel_k, int32_t* commit_len,
                    int32_t* out_tok, int32_t* y_tok, int32_t* y_kind, int32_t* offsets, int32_t* packed_tok,
                    int32_t* path_rolled, int32_t* branch_discarded, uint32_t* keep_mask, float* resid_mass,
                    cudaStream_t s) {
  const Dims d = to_dims(dd);
  AStepParams ap{};
  RowsParams& p = ap.r;
  p.d = d; p.PL = PL; p.QL = QL; p.tok = tok; p.u = u;
  p.info = w.info; p.unit_off = w.unit_off; p.seqpk = w.seqpk; p.cnt = w.cnt; p.rowstat = w.rowstat;
  p.pflag = w.pflag;
  p.lse_p = lse_p; p.lse_q = lse_q; p.p_tok = p_tok; p.q_tok = q_tok;
  p.top1_q = top1_q; p.entropy_q = entropy_q; p.top1_id_q = top1_id_q;
  p.acc_mask = acc_mask; p.n_acc = n_acc; p.status = status;
  p.sq_ctr = w.actr + 3; p.sq = w.asq; p.sq_pub = w.asq_pub;
  if (cw) {  // adaptive: confidence items first, their q states reused by slot-0 verify items
    p.qreuse = cw->qrs;
    ConfParams& c = ap.c;
    c.d = d;
    c.d.K = 1;  // slot-0 view of the draft rows
    c.QL = QL; c.tok = nullptr; c.mode = SB_CONF_TOP1; c.eps = eps; c.lambda = 1.f; c.k_max = k_max;
    c.top1_prob = c_top1; c.entropy = c_ent; c.tok_prob = nullptr; c.stat = c_stat; c.top1_id = c_id;
    c.stop = c_stop; c.k_next = c_knext; c.gamma_next = c_gamma;
    c.cnt = cw->conf_cnt; c.ws_stat = cw->conf_stat; c.ws_c = cw->conf_c; c.qrs = cw->qrs;
  }
  ap.adaptive = cw != nullptr;
  ap.gamma_in = gamma;
  ap.us = us; ap.bpos = branch_pos; ap.rule = rule;
  ap.ctr = w.actr; ap.qv = w.aqv; ap.qv_pub = w.aqv_pub; ap.sq = w.asq; ap.sq_pub = w.asq_pub;
  ap.qcap = dd->B * dd->K * (dd->G + 1);
  ap.co = CommitOut{sel_k, commit_len, out_tok, y_tok, y_kind, offsets, packed_tok, path_rolled, branch_discarded,
                    keep_mask, resid_mass};
  return dd->dtype == SB_BF16 ? launch_astep<RCA, __nv_bfloat16, 1>(ap, s) : launch_astep<RCA, float, 1>(ap, s);
}

// ---------------------------------------------------------------- short rows, many units
// k_rows_warp: one warp per unit (row pair) for rows of <= 64 KB when there are many units
// (the vocabulary shards of C5 at G >= 4: 32-64 KB rows, ~66 K units per rank).  With
// k_rows_tma's 16-20 consumer warps per unit a lane sees only 2-4 groups of a 32 KB row,
// so the per-row costs (first-group freeze, two warp reductions, the cross-warp combine)
// doubled the instructions per element (shard sweep: 0.51 of the copy peak at V/8).  Here
// each lane sees a whole row's share (U vectors per row per step), the per-row reduction is
// one warp tree, there is no cross-warp combine, and the warp runs its own epilogue
// (warp_epilogue or the shard partial record).  Bytes in flight come from a per-warp
// cp.async ring in shared memory (each lane copies and later reads only its own vectors:
// no barrier beyond cp.async.wait_group), NSW steps ahead across unit boundaries; the next
// unit's geometry is decoded one unit ahead (warp-cooperative probe).
template <int U>
using WG = RC<1, 1, U, 1, 1>;  // one warp covers a "chunk" of 32 x U 16-byte vectors per row


// warp_part for a one-warp unit: fold, warp tree, and (q rows) the exact first argmax by
// re-reading the U vectors of the step where each max-holding lane first saw it.
template <int U, typename T, bool kQ>
__device__ __forceinline__ RowStat warp_part_lane(const LazyAcc<kQ, 4>& a, const T* row, int nvec) {
  constexpr int E = Vec<T>::E;
  const int lane = threadIdx.x & 31;
  RowStat s = fold_lazy(a);
  float mw = s.m;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mw = fmaxf(mw, __shfl_xor_sync(0xffffffffu, mw, o));
  uint4 x[U];
  const bool need = kQ && (a.m == mw) && (mw > -CUDART_INF_F) && (a.tag >= 0);
  const int base = a.tag * 32 * U;
  if (need) {
#pragma unroll
    for (int j = 0; j < U; ++j) {
      const int v = base + lane + 32 * j;
      x[j] = v < nvec ? __ldg(reinterpret_cast<const uint4*>(row) + v) : neg_inf_vec<T>();
    }
  }
  s = warp_reduce_offsets(s);
  s.m = mw;
  int cand = 0x7fffffff;
  if (need) {
#pragma unroll
    for (int j = U - 1; j >= 0; --j) {
      float f[E];
      Vec<T>::unpack(x[j], f);
#pragma unroll
      for (int e = E - 1; e >= 0; --e)
        if (f[e] == mw) cand = (base + lane + 32 * j) * E + e;
    }
  }
  s.idx = kQ ? (int)__reduce_min_sync(0xffffffffu, (unsigned)cand) : 0;
  return s;
}

template <typename T, int U, int NSW, int WPB>
struct RowsWarpSmem {
  uint4 buf[WPB][NSW][2][32 * U];  // per warp: NSW steps of (p, q) x 32 lanes x U vectors
};

template <typename T, int U, int NSW, int WPB>
__global__ void __launch_bounds__(WPB * 32, 1) k_rows_warp(RowsParams p) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  RowsWarpSmem<T, U, NSW, WPB>& S = *reinterpret_cast<RowsWarpSmem<T, U, NSW, WPB>*>(smem_raw);
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  const int gw = blockIdx.x * WPB + wl, nw = gridDim.x * WPB;
  pdl_wait();
  const Dims& d = p.d;
  const int total = __ldg(p.unit_off + d.B);
  const T* PL = static_cast<const T*>(p.PL);
  const T* QL = static_cast<const T*>(p.QL);
  const int nvec = (int)((uint32_t)d.V * sizeof(T) / 16);
  const int nsteps = (nvec + 32 * U - 1) / (32 * U);
  if (gw >= total) return;
  // producer cursor: (unit pu, step pc) with decoded geometry pcur; consumer: (unit, step)
  int pbase = 0, cbase = 0;
  int4 pcur = probe_resolve(p, probe_load(p, 0), pbase, gw, total);
  int pu = gw, pc = 0;
  auto issue = [&](int slot) {
    if (pu < total) {
      const Unit un = unit_from(pcur);
      const bool po = q_reused(p, un);
      const uint4* pr = reinterpret_cast<const uint4*>(PL + row_off(d, un.b, un.slot, un.i));
      const uint4* qr = reinterpret_cast<const uint4*>(QL + row_off(d, un.b, un.slot, un.i));
#pragma unroll
      for (int j = 0; j < U; ++j) {
        const int v = pc * 32 * U + lane + 32 * j;
        if (v < nvec) {
          cp_async16(&S.buf[wl][slot][0][lane + 32 * j], pr + v);
          if (!po) cp_async16(&S.buf[wl][slot][1][lane + 32 * j], qr + v);
        }
      }
    }
    cp_async_commit();  // (empty groups keep the wait_group count uniform)
    if (pu < total && ++pc == nsteps) {  // next unit of this warp: one probe round
      pc = 0;
      pu += nw;
      pcur = probe_resolve(p, probe_load(p, pbase), pbase, pu, total);
    }
  };
#pragma unroll
  for (int s = 0; s < NSW; ++s) issue(s);
  int slot = 0;
  int4 ccur = probe_resolve(p, probe_load(p, 0), cbase, gw, total);
  for (int unit = gw; unit < total; unit += nw) {
    const Unit un = unit_from(ccur);
    const T* prow = PL + row_off(d, un.b, un.slot, un.i);
    const T* qrow = QL + row_off(d, un.b, un.slot, un.i);
    const bool po = q_reused(p, un);
    // path tokens through this row, their uniforms and logits (prefetched)
    const bool branch_row = (un.slot == 0 && un.i == un.in.s);
    const int ntok = branch_row ? d.K : 1;
    int x = 0;
    float lpx = 0.f, lqx = 0.f, uu = 0.f;
    int64_t et = 0;
    const bool has_tok = un.i < un.in.L;
    if (lane < ntok && has_tok) {
      et = ent(d, un.b, branch_row ? lane : un.slot, un.i);
      x = __ldg(p.tok + et);
      uu = __ldg(p.u + et);
      const int xl = x - p.v_offset;
      if (xl >= 0 && xl < d.V) {
        lpx = ld_scalar(prow + xl);
        lqx = ld_scalar(qrow + xl);
      } else {
        lpx = lqx = -CUDART_INF_F;
      }
    }
    RowStat qr;
    if (po) qr = p.qreuse[(int64_t)un.b * d.G + un.i];
    LazyAcc<false, 4> pa;
    LazyAcc<true, 4> qa;
    pa.init();
    qa.init();
    for (int c = 0; c < nsteps; ++c) {
      cp_async_wait<NSW - 1>();  // this lane's copies of step (unit, c) have landed
      StageRegs<WG<U>> r;
#pragma unroll
      for (int j = 0; j < U; ++j) {
        const int v = c * 32 * U + lane + 32 * j;
        const bool have = v < nvec;
        r.p[j] = have ? S.buf[wl][slot][0][lane + 32 * j] : neg_inf_vec<T>();
        r.q[j] = (have && !po) ? S.buf[wl][slot][1][lane + 32 * j] : neg_inf_vec<T>();
      }
      issue(slot);  // refill this slot NSW steps ahead
      slot = (slot + 1 == NSW) ? 0 : slot + 1;
      if (po) {
        if (c == 0) compute_stage_p<WG<U>, T, true>(r, c, pa);
        else compute_stage_p<WG<U>, T, false>(r, c, pa);
      } else {
        if (c == 0) compute_stage<WG<U>, T, true>(r, c, pa, qa);
        else compute_stage<WG<U>, T, false>(r, c, pa, qa);
      }
    }
    const Probe pr = probe_load(p, cbase);  // the next unit's geometry, in flight during the epilogue
    RowStat ps = warp_part_lane<U, T, false>(pa, prow, nvec);
    RowStat qs = po ? qr : warp_part_lane<U, T, true>(qa, qrow, nvec);
    if (p.partial) {  // a7: this shard's state (as k_rows_tma's epilogue)
      if (lane < ntok && has_tok) p.tokpart[et] = make_float2(lpx, lqx);
      bool fin = qs.m > kMaskedLogit && qs.m < CUDART_INF_F;
      if (sizeof(T) == 2 && qs.m == kMaskedLogit)
        fin = row_has_finite_bf16(reinterpret_cast<const __nv_bfloat16*>(qrow), d.V);
      else if (sizeof(T) == 4)
        fin = qs.m > -CUDART_INF_F && qs.m < CUDART_INF_F;
      if (lane == 0) {
        ShardRow rr;
        rr.pm = ps.m; rr.pms = ps.ms; rr.pz = ps.z;
        rr.qm = qs.m; rr.qms = qs.ms; rr.qz = qs.z; rr.qs1 = qs.s1;
        rr.qidx = (qs.idx == 0x7fffffff) ? qs.idx : qs.idx + p.v_offset;
        rr.qfin = fin;
        p.rowpart[ent(d, un.b, un.slot, un.i)] = rr;
      }
    } else {
      warp_epilogue<T>(p, un, ps, qs, qrow, x, lpx, lqx, uu, et);
    }
    ccur = probe_resolve(p, pr, cbase, unit + nw, total);
  }
  cp_async_wait<0>();
}

template <typename T, int U, int NSW, int WPB>
static sb_status launch_rows_warp_g(const RowsParams& p, cudaStream_t s) {
  using SM = RowsWarpSmem<T, U, NSW, WPB>;
  const int smem = (int)sizeof(SM);
  if (ensure_smem<k_rows_warp<T, U, NSW, WPB>>(smem) != cudaSuccess) return SB_ERR_CUDA;
  return cuda_status(launch_pdl(k_rows_warp<T, U, NSW, WPB>, dim3(num_sms()), dim3(WPB * 32), smem, s, p));
}
// 20 warps x 5 steps x (2 + 2) vectors per lane (200 KB of cp.async in flight per SM,
// 96 registers).  Rank-0 slice of C5 (scripts/shard_sweep.py, one GPU): G = 8 (32 KB rows)
// 0.75 of the copy peak, G = 4 (64 KB) 0.79, against 0.49 / 0.67 through k_rows_tma;
// 12 / 16 / 24 warps per SM, 1 or 4 vectors per lane per step measured 0.64-0.74 at G = 8.
template <typename T>
static sb_status launch_rows_warp(const RowsParams& p, cudaStream_t s) {
  return launch_rows_warp_g<T, 2, 5, 20>(p, s);
}

// Geometry (SB_ROWS_VARIANT=0 / 2 forces one).  Also measured: 24 consumer warps x 4 x
// 48 KB stages, 1-vector-per-row stages (24 x 8 x 24 KB, 16 x 12 x 16 KB; round 1) and
// 4 vectors per row per stage (16 x 3 x 64 KB; round 2: C4 verify +10 %, C3 +6 %): none
// beat these two.
using RC0 = RC<20, 5, 2, 4, 4>;  // 20 consumer warps, 5 x 40 KB stages, 4 epilogue warps
// (24 x 4 / 4 or 2, 28 x 3 / 2 and 20 x 5 / 2 epilogue warps measured slower on C4, r4_experiments.txt)
using RC2 = RC<16, 6, 2, 4, 4>;  // 16 consumer warps, 6 x 32 KB stages
using RC3 = RC<28, 3, 2, 4, 2>;  // 28 consumer warps, 3 x 56 KB stages, 2 epilogue warps (reuse units)
using RCF = RC<16, 6, 2, 4>;   // the fused step kernel's geometry

template <typename T>
static sb_status launch_rows_variant(const RowsParams& p, cudaStream_t s) {
  const char* e = getenv("SB_ROWS_VARIANT");
  int v = e ? atoi(e) : -1;
  // many short rows (<= 64 KB, >= 16384 row slots): one warp per unit (k_rows_warp)
  const size_t rb = (size_t)p.d.V * sizeof(T);
  if ((v < 0 && rb <= 65536 && (size_t)p.d.B * p.d.K * (p.d.G + 1) >= 16384) || v == 9)
    return launch_rows_warp<T>(p, s);
  if (v < 0) {
    // default: 20 consumer warps (20 KB chunks), unless the padding of a row's last
    // chunk (lanes that cost instructions, not bytes) wastes > 3 % more of the stages
    // than with 16 warps (16 KB chunks): C1 / C2's 125 / 62.5 KB rows waste 12 / 28 %
    // with 20 KB chunks and 2.4 % with 16 KB ones; C3 / C4 stay on 20 warps
    const double rb = (double)p.d.V * sizeof(T);
    auto waste = [&](double chunk) { const double n = std::ceil(rb / chunk); return (n * chunk - rb) / (n * chunk); };
    v = waste(RC0::CHUNK) - waste(RC2::CHUNK) > 0.03 ? 2 : 0;
  }
  // the adaptive step's verify (q states of the slot-0 draft rows reused, those units
  // stream p only): 28 consumer warps x 3 stages of 56 KB, 2 epilogue warps (same box, C3:
  // step 0.895-0.897 vs 0.920 ms with RC0; on C4's pairs RC0 stays faster, 5.35-5.48 vs
  // 5.48-5.65 ms)
  if (v == 0 && p.qreuse) return launch_rows_tma_k<RC3, T, true>(p, s);
  if (v == 3) return launch_rows_tma<RC3, T>(p, s);
  return v == 2 ? launch_rows_tma<RC2, T>(p, s) : launch_rows_tma<RC0, T>(p, s);
}

}  // namespace sb

using namespace sb;


struct sb_comm;
sb_status sb_shard_verify_nccl(const sb_dims* d, const void* p_logits, const void* q_logits, const int32_t* tok,
                               const float* u, const int32_t* gamma, const int32_t* branch_pos, float* lse_p,
                               float* lse_q, float* p_tok, float* q_tok, uint32_t* acc_mask, int32_t* n_acc,
                               float* top1_q, int32_t* top1_id_q, float* entropy_q, int32_t* status, sb_comm* c,
                               void* workspace, size_t workspace_bytes, cudaStream_t s);

// a7 partial phase: plan with the bonus rows, then the TMA row kernel writing this
// shard's row states and token logits (sb_shard_verify_local).
sb_status sb_rows_partial(const sb_dims* dd, const void* p_logits, const void* q_logits, const int32_t* tok,
                          const float* u, const int32_t* gamma, const int32_t* branch_pos, void* partial,
                          void* workspace, size_t workspace_bytes, cudaStream_t s) {
  if ((uintptr_t)workspace % 256) return SB_ERR_INVALID_ARG;
  const Workspace w = carve(*dd, workspace);
  if (workspace_bytes < w.bytes) return SB_ERR_WORKSPACE;
  const bool vok = vec_ok(dd, p_logits) && vec_ok(dd, q_logits);
  const size_t row_bytes = (size_t)dd->V * elem_size(dd);
  const Dims d = to_dims(dd);
  if (launch_pdl(k_plan, dim3(1), dim3(1024), 0, s, d, gamma, branch_pos, w.info, w.unit_off, 1, 0,
                 (int*)nullptr, (int*)nullptr, w.seqpk) != cudaSuccess)
    return SB_ERR_CUDA;
  RowsParams p{};
  p.d = d; p.PL = p_logits; p.QL = q_logits; p.tok = tok; p.u = u;
  p.info = w.info; p.unit_off = w.unit_off; p.seqpk = w.seqpk; p.cnt = w.cnt; p.rowstat = w.rowstat;
  p.pflag = w.pflag;
  p.partial = 1;
  p.v_offset = dd->v_offset;
  const size_t per = (size_t)dd->B * dd->K * (dd->G + 1);
  p.rowpart = reinterpret_cast<ShardRow*>(partial);
  p.tokpart = reinterpret_cast<float2*>(reinterpret_cast<char*>(partial) + per * sizeof(ShardRow));
  if (vok && row_bytes % 16 == 0 && !tma_disabled())
    return dd->dtype == SB_BF16 ? launch_rows_variant<__nv_bfloat16>(p, s) : launch_rows_variant<float>(p, s);
  // a ragged shard (row length not a 16-byte multiple, e.g. the last slice) or a
  // misaligned one: the register-staged kernel, any alignment
  if (dd->dtype == SB_BF16)
    return row_bytes <= 131072 ? launch_rows<__nv_bfloat16, 128, 4>(p, vok, s)
                               : launch_rows<__nv_bfloat16, 256, 4>(p, vok, s);
  return row_bytes <= 131072 ? launch_rows<float, 128, 4>(p, vok, s) : launch_rows<float, 256, 4>(p, vok, s);
}

static sb_status verify_impl(const sb_dims* dd, const void* p_logits, const void* q_logits, const int32_t* tok,
                             const float* u, const int32_t* gamma, const int32_t* branch_pos, float* lse_p,
                             float* lse_q, float* p_tok, float* q_tok, uint32_t* acc_mask, int32_t* n_acc,
                             float* top1_q, int32_t* top1_id_q, float* entropy_q, int32_t* status, void* comm,
                             void* workspace, size_t workspace_bytes, const void* conf_workspace,
                             sb_stream_t stream) {
  if (!dims_valid(dd)) return SB_ERR_INVALID_ARG;
  if (!p_logits || !q_logits || !tok || !u || !lse_p || !lse_q || !p_tok || !q_tok || !acc_mask ||
      !n_acc || !status || !workspace)
    return SB_ERR_INVALID_ARG;
  if ((uintptr_t)workspace % 256) return SB_ERR_INVALID_ARG;
  if (comm)
    return sb_shard_verify_nccl(dd, p_logits, q_logits, tok, u, gamma, branch_pos, lse_p, lse_q, p_tok, q_tok,
                                acc_mask, n_acc, top1_q, top1_id_q, entropy_q, status, (sb_comm*)comm, workspace,
                                workspace_bytes, (cudaStream_t)stream);
  if (sharded(dd)) return SB_ERR_INVALID_ARG;  // a vocabulary shard needs its exchange (comm)
  const Workspace w = carve(*dd, workspace);
  if (workspace_bytes < w.bytes) return SB_ERR_WORKSPACE;
  const Dims d = to_dims(dd);
  cudaStream_t s = (cudaStream_t)stream;

  if (launch_pdl(k_plan, dim3(1), dim3(1024), 0, s, d, gamma, branch_pos, w.info, w.unit_off, 0, 0,
                 (int*)nullptr, (int*)nullptr, w.seqpk) != cudaSuccess)
    return SB_ERR_CUDA;

  RowsParams p{};
  p.d = d; p.PL = p_logits; p.QL = q_logits; p.tok = tok; p.u = u;
  p.info = w.info; p.unit_off = w.unit_off; p.seqpk = w.seqpk; p.cnt = w.cnt; p.rowstat = w.rowstat;
  p.pflag = w.pflag;
  p.lse_p = lse_p; p.lse_q = lse_q; p.p_tok = p_tok; p.q_tok = q_tok;
  p.top1_q = top1_q; p.entropy_q = entropy_q; p.top1_id_q = top1_id_q;
  p.acc_mask = acc_mask; p.n_acc = n_acc; p.status = status;
  p.partial = 0; p.v_offset = 0; p.rowpart = nullptr; p.tokpart = nullptr; p.ready = nullptr;
  p.qreuse = nullptr;
  if (conf_workspace && dd->G > 0) {  // slot-0 rows of the same q tensor, as sb_draft_confidence saw them
    sb_dims cd = *dd;
    cd.K = 1;
    cd.seq_stride = d.ss;
    p.qreuse = carve(cd, const_cast<void*>(conf_workspace)).qrs;
  }
  const bool vok = vec_ok(dd, p_logits) && vec_ok(dd, q_logits);
  const size_t row_bytes = (size_t)dd->V * elem_size(dd);
  if (vok && row_bytes % 16 == 0 && !tma_disabled())
    return dd->dtype == SB_BF16 ? launch_rows_variant<__nv_bfloat16>(p, s) : launch_rows_variant<float>(p, s);
  if (dd->dtype == SB_BF16) {
    return row_bytes <= 131072 ? launch_rows<__nv_bfloat16, 128, 4>(p, vok, s)
                               : launch_rows<__nv_bfloat16, 256, 4>(p, vok, s);
  }
  return row_bytes <= 131072 ? launch_rows<float, 128, 4>(p, vok, s)
                             : launch_rows<float, 256, 4>(p, vok, s);
}

extern "C" sb_status sb_verify_branches(const sb_dims* dd, const void* p_logits,
                                        const void* q_logits, const int32_t* tok, const float* u,
                                        const int32_t* gamma, const int32_t* branch_pos,
                                        float* lse_p, float* lse_q, float* p_tok, float* q_tok,
                                        uint32_t* acc_mask, int32_t* n_acc, float* top1_q,
                                        int32_t* top1_id_q, float* entropy_q, int32_t* status,
                                        void* comm, void* workspace, size_t workspace_bytes,
                                        sb_stream_t stream) {
  SB_NVTX("sb_verify_branches");
  return verify_impl(dd, p_logits, q_logits, tok, u, gamma, branch_pos, lse_p, lse_q, p_tok, q_tok, acc_mask,
                     n_acc, top1_q, top1_id_q, entropy_q, status, comm, workspace, workspace_bytes, nullptr,
                     stream);
}

extern "C" sb_status sb_verify_branches_reuse(const sb_dims* dd, const void* p_logits, const void* q_logits,
                                              const int32_t* tok, const float* u, const int32_t* gamma,
                                              const int32_t* branch_pos, float* lse_p, float* lse_q, float* p_tok,
                                              float* q_tok, uint32_t* acc_mask, int32_t* n_acc, float* top1_q,
                                              int32_t* top1_id_q, float* entropy_q, int32_t* status,
                                              const void* conf_workspace, void* workspace, size_t workspace_bytes,
                                              sb_stream_t stream) {
  SB_NVTX("sb_verify_branches_reuse");
  if (!conf_workspace || sharded(dd)) return SB_ERR_INVALID_ARG;
  return verify_impl(dd, p_logits, q_logits, tok, u, gamma, branch_pos, lse_p, lse_q, p_tok, q_tok, acc_mask,
                     n_acc, top1_q, top1_id_q, entropy_q, status, nullptr, workspace, workspace_bytes,
                     conf_workspace, stream);
}

// ---------------------------------------------------------------- fused entry point
extern "C" sb_status sb_verify_select(const sb_dims* dd, const void* p_logits, const void* q_logits,
                                      const int32_t* tok, const float* u, const float* us, const int32_t* gamma,
                                      const int32_t* branch_pos, sb_select_rule rule, float* lse_p, float* lse_q,
                                      float* p_tok, float* q_tok, uint32_t* acc_mask, int32_t* n_acc,
                                      float* top1_q, int32_t* top1_id_q, float* entropy_q, int32_t* status,
                                      int32_t* sel_k, int32_t* commit_len, int32_t* out_tok, int32_t* y_tok,
                                      int32_t* y_kind, int32_t* offsets, int32_t* packed_tok,
                                      int32_t* path_rolled, int32_t* branch_discarded, uint32_t* keep_mask,
                                      float* resid_mass, void* workspace, size_t workspace_bytes,
                                      sb_stream_t stream) {
  SB_NVTX("sb_verify_select");
  if (!dims_valid(dd) || sharded(dd)) return SB_ERR_INVALID_ARG;
  if (!p_logits || !q_logits || !tok || !u || !us || !lse_p || !lse_q || !p_tok || !q_tok || !acc_mask ||
      !n_acc || !status || !sel_k || !commit_len || !out_tok || !y_tok || !y_kind || !offsets || !path_rolled ||
      !branch_discarded || !keep_mask || !workspace)
    return SB_ERR_INVALID_ARG;
  if (rule != SB_SELECT_EQ9 && rule != SB_SELECT_ALG1) return SB_ERR_INVALID_ARG;
  if ((uintptr_t)workspace % 256) return SB_ERR_INVALID_ARG;
  const Workspace w = carve(*dd, workspace);
  if (workspace_bytes < w.bytes) return SB_ERR_WORKSPACE;
  const bool vok = vec_ok(dd, p_logits) && vec_ok(dd, q_logits);
  const size_t row_bytes = (size_t)dd->V * elem_size(dd);
  // The single-launch fused kernel (k_step_tma) is correct but measured slower than the
  // two launches on B200 (C4: 6.88 vs 6.70 ms), so it is opt-in.
  const char* fz = getenv("SB_FUSED_STEP");
  const bool fused = fz && fz[0] == '1';
  // k_astep with plan items instead of confidence items: opt-in (SB_ASTEP=1) — one C1 round
  // (batch 1) measured 31.8 us against 29.6 us for k_plan + the two streaming kernels
  const char* ae = getenv("SB_ASTEP");
  if (!fused && ae && ae[0] == '1' && astep_eligible(dd, p_logits, q_logits))
    return astep_run(dd, w, nullptr, p_logits, q_logits, tok, u, us, gamma, branch_pos, rule, 0.f, 0, nullptr,
                     nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, lse_p, lse_q, p_tok, q_tok, acc_mask,
                     n_acc, top1_q, top1_id_q, entropy_q, status, sel_k, commit_len, out_tok, y_tok, y_kind,
                     offsets, packed_tok, path_rolled, branch_discarded, keep_mask, resid_mass, (cudaStream_t)stream);
  if (!fused || !vok || row_bytes % 16 || row_bytes > (size_t)kSegMax * kSegBytes || tma_disabled()) {
    // the two calls back to back
    sb_status st = sb_verify_branches(dd, p_logits, q_logits, tok, u, gamma, branch_pos, lse_p, lse_q, p_tok,
                                      q_tok, acc_mask, n_acc, top1_q, top1_id_q, entropy_q, status, nullptr,
                                      workspace, workspace_bytes, stream);
    if (st != SB_OK) return st;
    return sb_select_branch(dd, p_logits, q_logits, tok, u, us, gamma, branch_pos, n_acc, rule, sel_k, commit_len,
                            out_tok, y_tok, y_kind, offsets, packed_tok, path_rolled, branch_discarded, keep_mask,
                            resid_mass, status, nullptr, workspace, workspace_bytes, stream);
  }
  const Dims d = to_dims(dd);
  cudaStream_t s = (cudaStream_t)stream;
  k_plan<<<1, 1024, 0, s>>>(d, gamma, branch_pos, w.info, w.unit_off, 0, num_sms(), w.plan, w.ready, w.seqpk);
  if (cudaGetLastError() != cudaSuccess) return SB_ERR_CUDA;
  StepParams sp{};
  RowsParams& p = sp.r;
  p.d = d; p.PL = p_logits; p.QL = q_logits; p.tok = tok; p.u = u;
  p.info = w.info; p.unit_off = w.unit_off; p.seqpk = w.seqpk; p.cnt = w.cnt; p.rowstat = w.rowstat;
  p.pflag = w.pflag;
  p.lse_p = lse_p; p.lse_q = lse_q; p.p_tok = p_tok; p.q_tok = q_tok;
  p.top1_q = top1_q; p.entropy_q = entropy_q; p.top1_id_q = top1_id_q;
  p.acc_mask = acc_mask; p.n_acc = n_acc; p.status = status; p.ready = w.ready;
  sp.us = us; sp.rule = rule; sp.plan = w.plan; sp.done_cnt = w.sel_cnt;
  sp.sel_k = sel_k; sp.commit_len = commit_len; sp.out_tok = out_tok; sp.y_tok = y_tok; sp.y_kind = y_kind;
  sp.offsets = offsets; sp.packed_tok = packed_tok; sp.path_rolled = path_rolled;
  sp.branch_discarded = branch_discarded; sp.keep_mask = keep_mask; sp.resid_mass = resid_mass;
  return dd->dtype == SB_BF16 ? launch_step_tma<RCF, __nv_bfloat16>(sp, s) : launch_step_tma<RCF, float>(sp, s);
}

extern "C" sb_status sb_step_adaptive(const sb_dims* dd, const void* p_logits, const void* q_logits,
                                      const int32_t* tok, const float* u, const float* us,
                                      const int32_t* branch_pos, sb_select_rule rule, float eps, int32_t k_max,
                                      float* c_top1_prob, int32_t* c_top1_id, float* c_entropy, float* c_stat,
                                      int32_t* c_stop, int32_t* c_k_next, int32_t* c_gamma_next, float* lse_p,
                                      float* lse_q, float* p_tok, float* q_tok, uint32_t* acc_mask, int32_t* n_acc,
                                      float* top1_q, int32_t* top1_id_q, float* entropy_q, int32_t* status,
                                      int32_t* sel_k, int32_t* commit_len, int32_t* out_tok, int32_t* y_tok,
                                      int32_t* y_kind, int32_t* offsets, int32_t* packed_tok, int32_t* path_rolled,
                                      int32_t* branch_discarded, uint32_t* keep_mask, float* resid_mass,
                                      void* conf_workspace, size_t conf_workspace_bytes, void* workspace,
                                      size_t workspace_bytes, sb_stream_t stream) {
  SB_NVTX("sb_step_adaptive");
  if (!dims_valid(dd) || sharded(dd) || dd->G < 1) return SB_ERR_INVALID_ARG;
  if (!p_logits || !q_logits || !tok || !u || !us || !c_top1_prob || !c_top1_id || !c_entropy || !c_stat ||
      !c_stop || !c_k_next || !c_gamma_next || !lse_p || !lse_q || !p_tok || !q_tok || !acc_mask || !n_acc ||
      !status || !sel_k || !commit_len || !out_tok || !y_tok || !y_kind || !offsets || !path_rolled ||
      !branch_discarded || !keep_mask || !workspace || !conf_workspace)
    return SB_ERR_INVALID_ARG;
  if (rule != SB_SELECT_EQ9 && rule != SB_SELECT_ALG1) return SB_ERR_INVALID_ARG;
  if (!(eps > 0.f && eps < 1.f) || k_max < 1) return SB_ERR_INVALID_ARG;
  if ((uintptr_t)workspace % 256 || (uintptr_t)conf_workspace % 256) return SB_ERR_INVALID_ARG;
  const Workspace w = carve(*dd, workspace);
  if (workspace_bytes < w.bytes) return SB_ERR_WORKSPACE;
  sb_dims cd = *dd;  // slot-0 view of the draft rows
  cd.K = 1;
  cd.seq_stride = to_dims(dd).ss;
  if (conf_workspace_bytes < sb_workspace_bytes(&cd)) return SB_ERR_WORKSPACE;
  cudaStream_t s = (cudaStream_t)stream;
  if (astep_eligible(dd, p_logits, q_logits))  // one persistent launch (k_astep)
  {
    const Workspace cw = carve(cd, conf_workspace);
    return astep_run(dd, w, &cw, p_logits, q_logits, tok, u, us, nullptr, branch_pos, rule, eps, k_max,
                     c_top1_prob, c_top1_id, c_entropy, c_stat, c_stop, c_k_next, c_gamma_next, lse_p, lse_q, p_tok,
                     q_tok, acc_mask, n_acc, top1_q, top1_id_q, entropy_q, status, sel_k, commit_len, out_tok, y_tok,
                     y_kind, offsets, packed_tok, path_rolled, branch_discarded, keep_mask, resid_mass, s);
  }
  // SB_ASTEP=0 or unaligned rows: the three streaming kernels (the verify reuses the
  // confidence pass's slot-0 draft-row states)
  sb_status st = sb_draft_confidence(&cd, q_logits, nullptr, SB_CONF_TOP1, eps, 1.0f, k_max, c_top1_prob, c_top1_id,
                                     c_entropy, nullptr, c_stat, c_stop, c_k_next, c_gamma_next, nullptr,
                                     conf_workspace, conf_workspace_bytes, stream);
  if (st != SB_OK) return st;
  st = sb_verify_branches_reuse(dd, p_logits, q_logits, tok, u, c_gamma_next, branch_pos, lse_p, lse_q, p_tok, q_tok,
                                acc_mask, n_acc, top1_q, top1_id_q, entropy_q, status, conf_workspace, workspace,
                                workspace_bytes, stream);
  if (st != SB_OK) return st;
  return sb_select_branch(dd, p_logits, q_logits, tok, u, us, c_gamma_next, branch_pos, n_acc, rule, sel_k,
                          commit_len, out_tok, y_tok, y_kind, offsets, packed_tok, path_rolled, branch_discarded,
                          keep_mask, resid_mass, status, nullptr, workspace, workspace_bytes, stream);
}
