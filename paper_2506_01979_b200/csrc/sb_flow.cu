// sb_flow.cu — the small-batch step in ONE launch: [draft confidence ->] verify ->
// select (the same contract as sb_draft_confidence (TOP1, slot
// 0) + sb_verify_branches(_reuse) + sb_select_branch).  PAPER §3 P94, Alg. 1 P523-557,
// Eq. 6-7 P194-220, Eq. 9 P236-241.
//
// Why: on small batches (C1 one round: 15 row pairs; C2: 64 sequences) the separate
// kernels are each bounded by their own launch, ramp and dependent tail (C2: 22 + 38 +
// 20 us for 127 MB) and a single row pair is bounded by one SM's bandwidth.
// Here one persistent grid (several CTAs per SM, register-staged 16-byte loads) walks
// three phases of work items, every row split into V-segments so that even one
// sequence fills the GPU:
//   C  (adaptive only)  (draft row, segment) of slot 0 rows 0..G-1: partial softmax
//                       state; the last segment of a row combines (fp64, segment order)
//                       and writes the TOP1 statistics; the last row of a sequence takes
//                       the Eq. 6 stop, Eq. 7 k and gamma_b = max(1, stop).  Grid barrier.
//   R                   (row pair, segment) of every tested row pair (plan recomputed by
//                       every CTA in shared memory); the last segment combines and runs
//                       the token tests (fp64); the last row pair of a sequence takes
//                       n_k, the Eq. 9 / Alg. 1 decision and releases the sequence.
//   S                   (sequence, segment): waits for its sequence, streams its segment
//                       of the sampled row (pair): r = max(0, P - Q) (or P) sums per 1 KB
//                       sub-segment; the last segment locates us*R (fp64 prefix), re-reads
//                       one sub-segment and commits; the last sequence scans the offsets.
// Phases never wait on later phases and R items never wait at all, so the spins of S
// items cannot deadlock (all CTAs co-resident: grid = occupancy x SMs).  Every
// arithmetic step is the one of the separate kernels (LazyAcc, fp64 combine, r_scaled /
// seq_sum / warp_scan_rn sampling), so results agree with them within the same bands.
#include <algorithm>
#include <cstdlib>

#include "sb_host.h"
#include "sb_ring.cuh"
#include "sb_sample.cuh"

namespace sb {

constexpr int kFT = 256;  // threads per CTA
constexpr int kFW = kFT / 32;
constexpr int kSW = 6;          // stream warps (0..5): load, accumulate, warp-reduce
constexpr int kST = kSW * 32;
constexpr int kEW = kFW - kSW;  // finalizer warps (6, 7): combine, global partials, epilogues
constexpr int kNSlot = 4;       // items in flight between the two roles
constexpr int kFU = 4;  // 16-byte vectors per thread per row in flight
constexpr int kFlowMaxB = 1024;
constexpr int kMinSegBytes = 8192;
constexpr int kFlowMaxScale = 132;  // sample segments per row (rows <= 1 MB: nsub / 8 + 1)

enum { FC_CONF_DONE = 0, FC_SEQ_DONE = 1, FC_EXIT = 2 };

// Debug timeline (SB_FLOW_TRACE builds only): per CTA, per warp-0 / warp-6 event, the
// global timer.  Read back with sb_flow_trace_read().
#ifdef SB_FLOW_TRACE
constexpr int kTrCta = 1024, kTrEv = 64;
__device__ unsigned long long g_trace[kTrCta][2][kTrEv];
__device__ __forceinline__ void trace(int role, int ev) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  if (blockIdx.x < kTrCta && ev < kTrEv && (threadIdx.x & 31) == 0) g_trace[blockIdx.x][role][ev] = t;
}
#else
__device__ __forceinline__ void trace(int, int) {}
#endif

struct FlowParams {
  Dims d;
  const void* PL;
  const void* QL;
  const int* tok;
  const float* u;
  const float* us;
  const int* gamma_in;
  const int* bpos_in;
  int rule, adaptive;
  float eps;
  int k_max;
  float *c_top1, *c_ent, *c_stat;
  int *c_id, *c_stop, *c_knext, *c_gamma;
  float *lse_p, *lse_q, *p_tok, *q_tok, *top1_q, *entropy_q;
  int* top1_id_q;
  uint32_t* acc_mask;
  int *n_acc, *status;
  int *sel_k, *commit_len, *out_tok, *y_tok, *y_kind, *offsets, *packed_tok, *path_rolled, *branch_discarded;
  uint32_t* keep_mask;
  float* resid_mass;
  // workspace
  int *ctr, *rcnt, *ccnt, *cgrp, *seqcnt, *scnt, *gam, *ready;
  RowStat *rpart, *cpart, *qstate;
  float *cstat, *cc;
  float4* rowstat;
  uint8_t* pflag;
  int4* dec;
  float* subs;  // [B][2][sub_stride]: residual and p sums per 1 KB sub-segment
  int sub_stride;
  float* segmax;  // [B][segmax_stride]
  int segmax_stride;
  int Sc, Ss, nsub;
};

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// ---------------------------------------------------------------- segment streaming
// One row segment [v0, v1) of 16-byte vectors by the whole CTA into lazy accumulators.
// q rows also keep the exact first index of each thread's running maximum.
template <typename T, bool HASP, bool HASQ>
__device__ __forceinline__ void seg_stream(const T* prow, const T* qrow, int v0, int v1, LazyAcc<false, 4>& pa,
                                           LazyAcc<true, 4>& qa, int& qidx) {
  constexpr int E = Vec<T>::E;
  const uint4* pv = reinterpret_cast<const uint4*>(prow);
  const uint4* qv = reinterpret_cast<const uint4*>(qrow);
  for (int base = v0 + (int)threadIdx.x; base - (int)threadIdx.x < v1; base += kST * kFU) {
    uint4 xp[kFU], xq[kFU];
#pragma unroll
    for (int j = 0; j < kFU; ++j) {
      const int v = base + j * kST;
      if (HASP) xp[j] = v < v1 ? ldg_stream(pv + v) : neg_inf_vec<T>();
      if (HASQ) xq[j] = v < v1 ? ldg_stream(qv + v) : neg_inf_vec<T>();
    }
#pragma unroll
    for (int j = 0; j < kFU; ++j) {
      const int v = base + j * kST;
      if constexpr (sizeof(T) == 2) {
        if (HASP) acc_vecs_bf16<1>(pa, &xp[j], v);
        if (HASQ) {
          const float mb = qa.m;
          const float cm = acc_vecs_bf16<1>(qa, &xq[j], v);
          if (cm > mb && v < v1) {  // a new running maximum: its first index in the vector
            const uint32_t w[4] = {xq[j].x, xq[j].y, xq[j].z, xq[j].w};
            int first = 8;
#pragma unroll
            for (int e = 7; e >= 0; --e) {
              const uint32_t c = bf16x2_max_nan(w[e >> 1], kMaskedBf16x2);
              const float f = (e & 1) ? bf16_hi(c) : bf16_lo(c);
              if (f == cm) first = e;
            }
            qidx = v * 8 + first;
          }
        }
      } else {
        if (HASP) {
          float f[E];
          Vec<T>::unpack(xp[j], f);
          pa.template add<E>(f, v);
        }
        if (HASQ) {
          float f[E];
          Vec<T>::unpack(xq[j], f);
          const float cm = Vec<T>::vmax(f);
          if (cm > qa.m && v < v1) {
            int first = E;
#pragma unroll
            for (int e = E - 1; e >= 0; --e)
              if (f[e] == cm) first = e;
            qidx = v * E + first;
          }
          qa.template add_cm<E>(f, cm, v);
        }
      }
    }
  }
}

// A stream warp's state (fp64 sums, exact max / first index) reduced over its 32 lanes
// (fixed tree order).
__device__ __forceinline__ RowStat warp_state(RowStat s) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s = combine(s, shfl_xor(s, o));
  return s;
}

__device__ __forceinline__ RowStat ldcg_rowstat(const RowStat* src) {
  RowStat x;
  x.m = __ldcg(&src->m); x.ms = __ldcg(&src->ms); x.z = __ldcg(&src->z); x.s1 = __ldcg(&src->s1);
  x.idx = __ldcg(&src->idx);
  return x;
}

// Finalizer warp: publish this CTA's segment state(s) st[0..nst) of item `base` (segment
// base % S of a row) and, on the last arriving CTA, return true with the states of all S
// segments combined (lanes load the partials in parallel, fixed tree order) in st.
__device__ __forceinline__ bool warp_last_segment(RowStat* part, int base, int S, int nst, int* cnt, RowStat* st) {
  if (S == 1) return true;
  const int lane = threadIdx.x & 31;
  int last = 0;
  if (lane == 0) {
    for (int k = 0; k < nst; ++k) part[(int64_t)base * nst + k] = st[k];
    __threadfence();
    last = (atomicAdd(cnt, 1) == S - 1);
  }
  last = __shfl_sync(0xffffffffu, last, 0);
  if (!last) return false;
  __threadfence();
  const int first = base - base % S;
  for (int k = 0; k < nst; ++k) {
    RowStat r = rowstat_empty();
    for (int j = lane; j < S; j += 32) r = combine(r, ldcg_rowstat(part + (int64_t)(first + j) * nst + k));
    st[k] = warp_state(r);
  }
  if (lane == 0) *cnt = 0;  // leave the workspace re-usable
  return true;
}

// Stream-warp -> finalizer-warp handoff of one item (the shared-memory slot ring).
struct FSlot {
  RowStat part[kSW][2];
};
struct FlowSmem {
  uint64_t full[kNSlot], empty[kNSlot];
  FSlot slot[kNSlot];
  int off[kFlowMaxB + 1];
  int pk[kFlowMaxB];
  int w[kFW];
  float fred[kSW];
  double scale[kEW][kFlowMaxScale];
};

// ---------------------------------------------------------------- phase C epilogue
template <typename T>
__device__ void conf_row_final(const FlowParams& p, int b, int i, const RowStat& qs) {
  const Dims& d = p.d;
  const int G = d.G;
  const int64_t e = (int64_t)b * G + i;
  const RowOut o = finish(qs);
  double top1 = CUDART_NAN, H = CUDART_NAN;
  int id = -1;
  if (o.finite) {
    const double LN2 = 0.69314718055994530942;
    top1 = tok_prob(qs.m, o.MS, o.Z);
    id = qs.idx;
    H = LN2 * (log2(o.Z) - qs.s1 / o.Z);
  }
  p.qstate[e] = qs;
  p.c_top1[e] = (float)top1;
  p.c_id[e] = id;
  p.c_ent[e] = (float)H;
  p.c_stat[e] = (float)top1;  // TOP1 statistic (P170, P954)
  p.cstat[e] = (float)top1;
  __threadfence();
  if (atomicAdd(p.cgrp + b, 1) == G - 1) {
    __threadfence();
    int stop = G;
    for (int r = 0; r < G; ++r) {
      const float sv = __ldcg(p.cstat + (int64_t)b * G + r);
      if ((double)sv <= (double)p.eps) { stop = r; break; }  // Eq. 6: keep q(x) > eps
    }
    int kn = -1;
    if (stop < G) {
      const double c = (double)__ldcg(p.cstat + (int64_t)b * G + stop);
      const double kk = floor((double)p.k_max * (1.0 - c));  // Eq. 7
      kn = kk < 1.0 ? 1 : (int)kk;
    }
    const int g = stop > 1 ? stop : 1;
    p.c_stop[b] = stop;
    p.c_knext[b] = kn;
    p.c_gamma[b] = g;
    p.gam[b] = g;
    p.cgrp[b] = 0;
    __threadfence();
    atomicAdd(p.ctr + FC_CONF_DONE, 1);
  }
}

// ---------------------------------------------------------------- phase R epilogue
// One row pair's statistics known: token tests, row outputs; the last row pair of the
// sequence takes n_k, status, sentinels and the selection decision (Eq. 9 / Alg. 1,
// as the separate select kernel's decider), then releases the sequence.  One warp.
struct FUnit {
  int b, slot, i, g, s, L, st;
};

template <typename T>
__device__ void unit_final(const FlowParams& p, const FUnit& un, const RowStat& ps, const RowStat& qs, const T* prow,
                           const T* qrow, int units_b) {
  const Dims& d = p.d;
  const int lane = threadIdx.x & 31;
  const int b = un.b, slot = un.slot, i = un.i;
  const RowOut po = finish(ps), qo = finish_q<T>(qs, qrow, d.V);
  const bool branch_row = (slot == 0 && i == un.s);
  const int ntok = branch_row ? d.K : 1;
  if (lane < ntok) {
    const int64_t et = ent(d, b, branch_row ? lane : slot, i);
    const int x = __ldg(p.tok + et);
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
      if ((double)__ldg(p.u + et) * Qx <= Px) fl |= 1;
    }
    p.p_tok[et] = pt;
    p.q_tok[et] = qt;
    p.pflag[et] = fl;
  }
  if (lane == 0) {
    const int64_t e = ent(d, b, slot, i);
    const double LN2 = 0.69314718055994530942;
    p.lse_p[e] = po.finite ? (float)(((double)po.MS + log2(po.Z)) * LN2) : CUDART_NAN_F;
    p.lse_q[e] = qo.finite ? (float)(((double)qo.MS + log2(qo.Z)) * LN2) : CUDART_NAN_F;
    const bool conf_ok = po.finite && qo.finite;
    if (p.top1_q) p.top1_q[e] = conf_ok ? (float)tok_prob(qs.m, qo.MS, qo.Z) : CUDART_NAN_F;
    if (p.top1_id_q) p.top1_id_q[e] = conf_ok ? qs.idx : -1;
    if (p.entropy_q) p.entropy_q[e] = conf_ok ? (float)(LN2 * (log2(qo.Z) - qs.s1 / qo.Z)) : CUDART_NAN_F;
    p.rowstat[e] = make_float4(po.MS, z_store(po), qo.MS, z_store(qo));
  }
  __syncwarp();
  int last = 0;
  if (lane == 0) {
    __threadfence();
    last = (atomicAdd(p.seqcnt + b, 1) == units_b - 1);
  }
  last = __shfl_sync(0xffffffffu, last, 0);
  if (!last) return;
  __threadfence();
  const int L = un.L, s = un.s, g = un.g;
  uint32_t fw[4] = {0u, 0u, 0u, 0u};  // 4 flag bits per branch, 8 branches per word
  if (lane < L) {
    for (int k = 0; k < d.K; ++k) {
      const uint32_t f = __ldcg(p.pflag + ent(d, b, (lane < s) ? 0 : k, lane));
      fw[k / 8] |= (f & 15u) << (4 * (k % 8));
    }
  }
  const uint32_t rowmask = L >= 32 ? 0xffffffffu : ((1u << L) - 1u);
  uint32_t anyf = 0;
  int nk_lane = 0;
  for (int k = 0; k < d.K; ++k) {
    const uint32_t f = (fw[k / 8] >> (4 * (k % 8))) & 15u;
    const uint32_t mask = __ballot_sync(0xffffffffu, f & 1u) & rowmask;
    anyf |= f;
    const uint32_t rej = ~mask & rowmask;
    const int nk = rej ? (__ffs(rej) - 1) : L;
    if (lane == k) nk_lane = nk;
    if (lane == 0) {
      p.acc_mask[(int64_t)b * d.K + k] = mask;
      p.n_acc[(int64_t)b * d.K + k] = nk;
    }
  }
  anyf = __reduce_or_sync(0xffffffffu, anyf);
  const int R1 = d.G + 1;
  for (int q = lane; q < d.K * R1; q += 32) {  // sentinels for entries no tested path touches
    const int k = q / R1, r = q % R1;
    const int64_t e = ent(d, b, k, r);
    const bool phys = (k == 0) ? (r < L) : (r > s && r < L);
    const bool path = (k == 0) ? (r < L) : (r >= s && r < L);
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
  // the decision (the separate select kernel's decider): A = {k : n_k > s_b}; Eq. 9:
  // argmax raw target logit at the branch row (ties: smaller token, then smaller k);
  // Alg. 1: argmax u (ties: smaller k)
  const T* PL = static_cast<const T*>(p.PL);
  const int k = lane;
  const bool inA = k < d.K && nk_lane > s;
  int xk = 0x7fffffff;
  float key = -CUDART_INF_F;
  if (inA) {
    xk = __ldg(p.tok + ent(d, b, k, s));
    key = (p.rule == SB_SELECT_ALG1) ? __ldg(p.u + ent(d, b, k, s)) : ld_scalar(PL + row_off(d, b, 0, s) + xk);
  }
  int bk = inA ? k : 0x7fffffff, btok = inA ? (p.rule == SB_SELECT_ALG1 ? 0 : xk) : 0x7fffffff;
  float bkey = key;
  bool bin = inA;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float okey = __shfl_xor_sync(0xffffffffu, bkey, o);
    const int otok = __shfl_xor_sync(0xffffffffu, btok, o);
    const int ok_ = __shfl_xor_sync(0xffffffffu, bk, o);
    const bool oin = __shfl_xor_sync(0xffffffffu, (int)bin, o);
    bool take;
    if (!oin) take = false;
    else if (!bin) take = true;
    else take = okey > bkey || (okey == bkey && (otok < btok || (otok == btok && ok_ < bk)));
    if (take) { bkey = okey; btok = otok; bk = ok_; bin = true; }
  }
  const int ksel = bin ? bk : -1;
  const int n0 = __shfl_sync(0xffffffffu, nk_lane, 0);
  const int nsel = __shfl_sync(0xffffffffu, nk_lane, ksel < 0 ? 0 : ksel);
  if (lane == 0) {
    int npath, kind, row = 0, sl = 0;
    if (ksel < 0) {
      npath = min(n0, s);  // rejection in the shared prefix or at the branch row (P655)
      kind = 1; row = npath; sl = 0;
    } else {
      npath = nsel;
      if (nsel < L) { kind = 1; row = nsel; sl = (nsel <= s) ? 0 : ksel; }
      else if (s < g) { kind = 2; row = g; sl = ksel; }  // bonus from p_{gamma+1} (P94)
      else { kind = 0; }  // branch token accepted; continuation carried by the caller (P237)
    }
    p.dec[b] = make_int4(ksel, npath, kind, row | (sl << 8));
    p.status[b] = un.st | flags_st(anyf);
    p.seqcnt[b] = 0;
    __threadfence();
    st_release(p.ready + b, 1);
  }
}

// ---------------------------------------------------------------- phase S
// r = max(0, P - Q) (p scale) and P for the two 16-byte vectors a lane owns in a 1 KB
// sub-segment, with the sampling kernels' arithmetic (r_scaled), summed in order.
template <typename T>
__device__ __forceinline__ void sub_sums(const T* prow, const T* qrow, uint32_t rb, int sI, bool resid, float MSp,
                                         float MSq, float kq, float& sr, float& sp) {
  constexpr int E = Vec<T>::E;
  const int lane = threadIdx.x & 31;
  float orr = 0.f, op = 0.f;
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const uint32_t off = (uint32_t)sI * kSegBytes + lane * 32 + j * 16;
    const uint4 vp = seg_vec(prow, rb, off);
    float r[E];
    if (resid) {
      r_scaled<T>(vp, seg_vec(qrow, rb, off), true, MSp, MSq, kq, r);
      orr = seq_sum<E>(r, orr);
    }
    r_scaled<T>(vp, uint4{}, false, MSp, MSq, kq, r);
    op = seq_sum<E>(r, op);
  }
  sr = warp_sum_rn(orr);
  sp = warp_sum_rn(op);
}

// Segment j of a row split into S parts covers sub-segments [nsub j / S, nsub (j+1) / S);
// the segment holding sub-segment sI.
__device__ __forceinline__ int seg_of(int sI, int nsub, int S) {
  return min(S - 1, max(0, (int)((((int64_t)sI + 1) * S - 1) / nsub)));
}

// The last segment of sequence b: locate t = us R over the sub-segment sums (fp64
// prefix; a bonus row's per-segment offsets folded in as exact fp64 scales), re-read one
// sub-segment in its segment's own scale, commit.  One warp; sh_scale: Ss doubles.
template <typename T>
__device__ void sample_final(const FlowParams& p, int b, int4 D, int s, int L, double* sh_scale) {
  constexpr int E = Vec<T>::E;
  const Dims& d = p.d;
  const int lane = threadIdx.x & 31;
  const T* PL = static_cast<const T*>(p.PL);
  const T* QL = static_cast<const T*>(p.QL);
  const uint32_t rb = (uint32_t)d.V * sizeof(T);
  const int nsub = p.nsub, Ss = p.Ss;
  const int ksel = D.x, npath = D.y, row = D.w & 0xff, sl = D.w >> 8;
  int kind = D.z, st = 0, y = -1;
  double mass = 0.0;
  const T* prow = PL + row_off(d, b, sl, row);
  const T* qrow = QL + row_off(d, b, sl, row);
  const float* subR = p.subs + (int64_t)b * 2 * p.sub_stride;
  const float* subP = subR + p.sub_stride;
  const float* smax = p.segmax + (int64_t)b * p.segmax_stride;
  float MSp = 0.f, MSq = 0.f, kq = 0.f, Zp = 1.f, M = 0.f;
  if (kind == 1) {
    const float4 rs = p.rowstat[ent(d, b, sl, row)];
    const int cls = z_class(rs.y) | z_class(rs.w);
    if (cls) { kind = 0; st |= cls; }
    MSp = rs.x; Zp = rs.y; MSq = rs.z; kq = rs.y / rs.w;
  } else if (kind == 2) {  // the bonus row: per-segment offsets -> exact fp64 scales
    M = -CUDART_INF_F;
    for (int j = 0; j < Ss; ++j) M = fmaxf(M, __ldcg(smax + j));
    const double MS = (double)offset_of(M);
    for (int j = lane; j < Ss; j += 32) sh_scale[j] = exp2((double)offset_of(__ldcg(smax + j)) - MS);
    __syncwarp();
  }
  if (kind != 0) {
    bool resid = (kind == 1);
    const float* A = resid ? subR : subP;
    const int per = (nsub + 31) / 32;
    auto scale_of = [&](int sI) -> double { return kind == 2 ? sh_scale[seg_of(sI, nsub, Ss)] : 1.0; };
    double R = 0.0, excl = 0.0, incl = 0.0;
    for (int attempt = 0; attempt < 2; ++attempt) {
      double local = 0.0;
      for (int j = 0; j < per; ++j) {
        const int sI = lane * per + j;
        if (sI < nsub) local += (double)__ldcg(A + sI) * scale_of(sI);
      }
      incl = local;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const double yv = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += yv;
      }
      excl = __shfl_up_sync(0xffffffffu, incl, 1);
      if (lane == 0) excl = 0.0;
      R = __shfl_sync(0xffffffffu, incl, 31);
      if (R > 0.0 || !resid) break;
      resid = false;  // "no residual mass" (S134-140): sample from P
      st |= SB_ST_ZERO_RESID;
      A = subP;
    }
    if (kind == 2) {  // the bonus row's class (it was never read before this phase)
      const int cls = row_class(M, R);
      if (cls) { kind = 0; st |= cls; }
    }
    if (kind != 0) {
      const double t = (double)__ldg(p.us + b) * R;
      int found = -1, lastpos = -1;
      double Fprev = 0.0;
      const bool mine = (excl <= t && incl > t);
      {
        double F = excl;
        for (int j = 0; j < per; ++j) {
          const int sI = lane * per + j;
          if (sI >= nsub) break;
          const double a = (double)__ldcg(A + sI) * scale_of(sI);
          if (a > 0.0) lastpos = sI;
          if (mine && found < 0 && F + a > t) { found = sI; Fprev = F; }
          F += a;
        }
      }
      const unsigned who = __ballot_sync(0xffffffffu, found >= 0);
      int sStar;
      double trem;
      if (who) {
        const int src = __ffs(who) - 1;
        sStar = __shfl_sync(0xffffffffu, found, src);
        trem = t - __shfl_sync(0xffffffffu, Fprev, src);
      } else {  // rounding: the last sub-segment with mass, and the in-segment fallback
        const unsigned mw = __ballot_sync(0xffffffffu, mine);
        const int src = mw ? __ffs(mw) - 1 : -1;
        const int cand = src >= 0 ? __shfl_sync(0xffffffffu, lastpos, src) : -1;
        sStar = cand >= 0 ? cand : (int)__reduce_max_sync(0xffffffffu, (unsigned)(lastpos + 1)) - 1;
        trem = CUDART_INF;
      }
      if (sStar >= 0) {
        const double sc = scale_of(sStar);
        const float mseg = (kind == 2) ? offset_of(__ldcg(smax + seg_of(sStar, nsub, Ss))) : MSp;
        const double tl = trem / sc;  // the threshold in the segment's own scale
        float r[2][E], own = 0.f;
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const uint32_t off = (uint32_t)sStar * kSegBytes + lane * 32 + j * 16;
          r_scaled<T>(seg_vec(prow, rb, off), resid ? seg_vec(qrow, rb, off) : uint4{}, resid, mseg, MSq, kq, r[j]);
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
            if (cand == 0x7fffffff && (double)F > tl && r[j][e] > 0.f) cand = v;
            if (r[j][e] > 0.f) lastv = v;
          }
        const int pick = (int)__reduce_min_sync(0xffffffffu, (unsigned)cand);
        y = (pick != 0x7fffffff) ? pick : (int)__reduce_max_sync(0xffffffffu, (unsigned)(lastv + 1)) - 1;
        if (y >= d.V) y = -1;
      }
      mass = (kind == 1) ? R / (double)Zp : 1.0;  // back to probability mass (a bonus row: sum p)
    }
  }
  // commit (SURVEY §8.0 "Commit")
  const int kpath = ksel < 0 ? 0 : ksel;
  int* out = p.out_tok + (int64_t)b * (d.G + 2);
  for (int qq = lane; qq < d.G + 2; qq += 32) {
    int v = -1;
    if (qq < npath) v = __ldg(p.tok + ent(d, b, (qq < s) ? 0 : kpath, qq));
    else if (qq == npath && kind != 0) v = y;
    out[qq] = v;
  }
  if (lane < d.K) {
    uint32_t km = 0;
    for (int qq = 0; qq < npath; ++qq)
      if (((qq < s) ? 0 : kpath) == lane) km |= 1u << qq;
    p.keep_mask[(int64_t)b * d.K + lane] = km;
  }
  if (lane == 0) {
    p.sel_k[b] = ksel;
    p.commit_len[b] = npath + (kind != 0);
    p.y_tok[b] = (kind != 0) ? y : -1;
    p.y_kind[b] = kind;
    p.path_rolled[b] = L - npath;
    p.branch_discarded[b] = (d.K - 1) * (L - s);
    if (p.resid_mass) p.resid_mass[b] = (kind != 0) ? (float)mass : 0.f;
    if (st) atomicOr(p.status + b, st);
  }
}

// ---------------------------------------------------------------- the kernel
// Warp roles: warps 0..kSW-1 stream item segments (register-staged 16-byte loads, kFU
// vectors per row per thread in flight) and hand each warp's reduced state to a
// finalizer warp through a shared-memory slot (mbarrier full / empty); the kEW finalizer
// warps (items alternate between them) combine the states, publish segment partials,
// and run the epilogues (token tests, n_k, the decision, the sample, the commit) while
// the stream warps already load the next items.
template <typename T>
__device__ __forceinline__ void flow_handoff(FlowSmem& S, int li, const RowStat& a, const RowStat& b) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int sl = li % kNSlot;
  const uint32_t ph = (uint32_t)(li / kNSlot) & 1u;
  if (lane == 0) {
    mbar_wait(&S.empty[sl], ph ^ 1u);
    S.slot[sl].part[warp][0] = a;
    S.slot[sl].part[warp][1] = b;
    mbar_arrive(&S.full[sl]);
  }
  __syncwarp();
}
// Finalizer side: the kSW warp states of item li combined (lane-parallel, fixed order).
__device__ __forceinline__ void flow_take(FlowSmem& S, int li, RowStat& a, RowStat& b) {
  const int lane = threadIdx.x & 31;
  const int sl = li % kNSlot;
  const uint32_t ph = (uint32_t)(li / kNSlot) & 1u;
  mbar_wait_parked(&S.full[sl], ph);
  RowStat x = lane < kSW ? S.slot[sl].part[lane][0] : rowstat_empty();
  RowStat y = lane < kSW ? S.slot[sl].part[lane][1] : rowstat_empty();
  __syncwarp();
  if (lane == 0) mbar_arrive(&S.empty[sl]);
  a = warp_state(x);
  b = warp_state(y);
}

template <typename T>
__global__ void __launch_bounds__(kFT, 3) k_flow(FlowParams p) {
  extern __shared__ __align__(16) uint8_t flow_smem[];
  FlowSmem& S = *reinterpret_cast<FlowSmem*>(flow_smem);
  const Dims& d = p.d;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bool streamer = warp < kSW;
  const int fe = warp - kSW;  // finalizer index (streamers: < 0)
  const T* PL = static_cast<const T*>(p.PL);
  const T* QL = static_cast<const T*>(p.QL);
  const uint32_t rb = (uint32_t)d.V * sizeof(T);
  const int nv = (int)(rb / 16);
  if (tid == 0) {
    for (int k = 0; k < kNSlot; ++k) {
      mbar_init(&S.full[k], kSW);
      mbar_init(&S.empty[k], 1);
    }
    fence_mbar_init();
  }
  __syncthreads();
  pdl_wait();
  int li = 0;  // this CTA's running item count (the slot ring position)
  int tev = 0;
  const int trole = warp == 0 ? 0 : (warp == kSW ? 1 : -1);
  if (trole >= 0) trace(trole, tev);
  ++tev;

  // ---- phase C: confidence rows (slot 0, rows 0..G-1), adaptive only
  if (p.adaptive) {
    const int items = d.B * d.G * p.Sc;
    for (int it = blockIdx.x; it < items; it += gridDim.x, ++li) {
      const int r = it / p.Sc, sg = it % p.Sc, b = r / d.G, i = r % d.G;
      const T* qrow = QL + row_off(d, b, 0, i);
      if (streamer) {
        const int v0 = (int)((int64_t)nv * sg / p.Sc), v1 = (int)((int64_t)nv * (sg + 1) / p.Sc);
        LazyAcc<false, 4> pa;
        LazyAcc<true, 4> qa;
        qa.init();
        int qidx = 0x7fffffff;
        seg_stream<T, false, true>(nullptr, qrow, v0, v1, pa, qa, qidx);
        RowStat qs = fold_lazy(qa);
        qs.idx = qidx;
        flow_handoff<T>(S, li, warp_state(qs), rowstat_empty());
      } else if (li % kEW == fe) {
        RowStat st[2];
        flow_take(S, li, st[0], st[1]);
        if (warp_last_segment(p.cpart, it, p.Sc, 1, p.ccnt + r, st) && lane == 0) conf_row_final<T>(p, b, i, st[0]);
        __syncwarp();
      }
    }
    if (trole >= 0) trace(trole, tev);
    ++tev;
    if (lane == 0)  // grid barrier: every gamma_b known
      while (ld_acquire(p.ctr + FC_CONF_DONE) < d.B) __nanosleep(128);
    __syncwarp();
    if (trole >= 0) trace(trole, tev);
    ++tev;
  }

  // ---- plan (every CTA, shared memory): clamped layout, units per sequence, scan
  __syncthreads();
  {
    int carry = 0;
    for (int b0 = 0; b0 < d.B; b0 += kFT) {
      const int b = b0 + tid;
      int nu = 0;
      if (b < d.B) {
        int st = 0;
        int g = p.adaptive ? __ldcg(p.gam + b) : (p.gamma_in ? __ldg(p.gamma_in + b) : d.G);
        if (g > d.G) { g = d.G; st |= SB_ST_GAMMA_CLAMPED; }
        if (g < 0) { g = 0; st |= SB_ST_GAMMA_CLAMPED; }
        int s = p.bpos_in ? __ldg(p.bpos_in + b) : 0;
        if (s > g) { s = g; st |= SB_ST_BRANCH_CLAMPED; }
        if (s < 0) { s = 0; st |= SB_ST_BRANCH_CLAMPED; }
        const int L = (s < g) ? g : g + 1;
        S.pk[b] = s | (g << 5) | (L << 10) | (st << 16);
        nu = L + (d.K - 1) * (L - 1 - s);
      }
      int incl = nu;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int yv = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += yv;
      }
      if (lane == 31) S.w[warp] = incl;
      __syncthreads();
      int wo = 0, tot = 0;
      for (int w = 0; w < kFW; ++w) {
        if (w < warp) wo += S.w[w];
        tot += S.w[w];
      }
      if (b < d.B) S.off[b] = carry + wo + incl - nu;
      carry += tot;
      __syncthreads();
    }
    if (tid == 0) S.off[d.B] = carry;
    __syncthreads();
  }
  const int U = S.off[d.B];
  const int Smax = max(1, (int)(rb / kMinSegBytes));
  const int Sr = min(Smax, max(1, (kFlowTarget + U - 1) / max(U, 1)));

  // ---- phase R: (row pair, segment)
  for (int it = blockIdx.x; it < U * Sr; it += gridDim.x, ++li) {
    if (!streamer && li % kEW != fe) continue;
    const int u = it / Sr, sg = it % Sr;
    int lo = 0, hi = d.B;  // sequence of unit u (binary search in shared memory)
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (S.off[mid] <= u) lo = mid; else hi = mid;
    }
    const int b = lo, pk = S.pk[b];
    FUnit un;
    un.b = b; un.s = pk & 31; un.g = (pk >> 5) & 31; un.L = (pk >> 10) & 63; un.st = pk >> 16;
    const int j = u - S.off[b];
    if (j < un.L) { un.slot = 0; un.i = j; }
    else {
      const int per = un.L - 1 - un.s, jj = j - un.L;
      un.slot = 1 + jj / per;
      un.i = un.s + 1 + jj % per;
    }
    const T* prow = PL + row_off(d, b, un.slot, un.i);
    const T* qrow = QL + row_off(d, b, un.slot, un.i);
    const bool reuse = p.adaptive && un.slot == 0 && un.i < d.G;  // q state from phase C
    if (streamer) {
      const int v0 = (int)((int64_t)nv * sg / Sr), v1 = (int)((int64_t)nv * (sg + 1) / Sr);
      LazyAcc<false, 4> pa;
      LazyAcc<true, 4> qa;
      pa.init();
      qa.init();
      int qidx = 0x7fffffff;
      if (reuse) seg_stream<T, true, false>(prow, nullptr, v0, v1, pa, qa, qidx);
      else seg_stream<T, true, true>(prow, qrow, v0, v1, pa, qa, qidx);
      RowStat qs = fold_lazy(qa);
      qs.idx = qidx;
      flow_handoff<T>(S, li, warp_state(fold_lazy(pa)), reuse ? rowstat_empty() : warp_state(qs));
      if (trole == 0) trace(0, 4 + (li & 31));
    } else {
      RowStat st[2];
      flow_take(S, li, st[0], st[1]);
      if (warp_last_segment(p.rpart, it, Sr, 2, p.rcnt + ent(d, b, un.slot, un.i), st)) {
        const RowStat qf = reuse ? ldcg_rowstat(p.qstate + (int64_t)b * d.G + un.i) : st[1];
        unit_final<T>(p, un, st[0], qf, prow, qrow, un.L + (d.K - 1) * (un.L - 1 - un.s));
      }
      __syncwarp();
      if (trole == 1) trace(1, 4 + (li & 31));
    }
  }
  if (trole >= 0) trace(trole, 40);

  // ---- phase S: (sequence, segment) of the sampled row (pair)
  const int Ss = p.Ss, nsub = p.nsub;
  for (int it = blockIdx.x; it < d.B * Ss; it += gridDim.x, ++li) {
    if (!streamer && li % kEW != fe) continue;
    const int b = it / Ss, sg = it % Ss;
    if (streamer) {
      if (trole == 0) trace(0, 41);
      if (lane == 0)
        while (ld_acquire(p.ready + b) == 0) __nanosleep(64);
      __syncwarp();
      if (trole == 0) trace(0, 42);
      const int4 D = __ldcg(p.dec + b);
      const int kind = D.z, row = D.w & 0xff, sl = D.w >> 8;
      const int s0 = (int)((int64_t)nsub * sg / Ss), s1 = (int)((int64_t)nsub * (sg + 1) / Ss);
      float* subR = p.subs + (int64_t)b * 2 * p.sub_stride;
      float* subP = subR + p.sub_stride;
      if (kind != 0) {
        const T* prow = PL + row_off(d, b, sl, row);
        const T* qrow = QL + row_off(d, b, sl, row);
        float MSp, MSq = 0.f, kq = 0.f;
        if (kind == 1) {
          const float4 rs = __ldcg(p.rowstat + ent(d, b, sl, row));
          MSp = rs.x; MSq = rs.z; kq = rs.y / rs.w;
        } else {  // bonus row: this segment's exact maximum sets its own offset
          float m = -CUDART_INF_F;
          const int e0 = s0 * (kSegBytes / 16), e1 = min(s1 * (kSegBytes / 16), nv);
          for (int v = e0 + tid; v < e1; v += kST) {
            float f[Vec<T>::E];
            Vec<T>::unpack(ldg_stream(reinterpret_cast<const uint4*>(prow) + v), f);
            m = fmaxf(m, Vec<T>::vmax(f));
          }
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
          if (lane == 0) S.fred[warp] = m;
          consumer_sync(kST);
          m = S.fred[0];
          for (int w = 1; w < kSW; ++w) m = fmaxf(m, S.fred[w]);
          consumer_sync(kST);  // fred reusable
          if (tid == 0) p.segmax[(int64_t)b * p.segmax_stride + sg] = m;
          MSp = offset_of(m);
        }
        for (int sI = s0 + warp; sI < s1; sI += kSW) {
          float sr, sp;
          sub_sums<T>(prow, qrow, rb, sI, kind == 1, MSp, MSq, kq, sr, sp);
          if (lane == 0) {
            subR[sI] = sr;
            subP[sI] = sp;
          }
        }
        __threadfence();  // the sums (and segment max) before the handoff: read by another CTA
      }
      flow_handoff<T>(S, li, rowstat_empty(), rowstat_empty());
      if (trole == 0) trace(0, 43);
    } else {
      RowStat st0, st1;
      flow_take(S, li, st0, st1);  // every stream warp's sums are written
      int last = 0;
      if (lane == 0) {
        __threadfence();
        last = (atomicAdd(p.scnt + b, 1) == Ss - 1);
      }
      last = __shfl_sync(0xffffffffu, last, 0);
      if (last) {
        __threadfence();
        const int4 D = __ldcg(p.dec + b);
        const int pk = S.pk[b];
        sample_final<T>(p, b, D, pk & 31, (pk >> 10) & 63, S.scale[fe]);
        int lastseq = 0;
        if (lane == 0) {
          p.scnt[b] = 0;
          p.ready[b] = 0;  // every segment of b has passed its wait
          __threadfence();
          lastseq = (atomicAdd(p.ctr + FC_SEQ_DONE, 1) == d.B - 1);
        }
        lastseq = __shfl_sync(0xffffffffu, lastseq, 0);
        if (lastseq) {  // the last sequence: offsets and the packed stream
          __threadfence();
          warp_offsets(d.B, d.G, p.commit_len, p.out_tok, p.offsets, p.packed_tok);
        }
      }
      __syncwarp();
    }
  }
  // ---- the last CTA to leave resets the grid counters
  if (trole >= 0) trace(trole, 63);
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    if (atomicAdd(p.ctr + FC_EXIT, 1) == (int)gridDim.x - 1) {
      p.ctr[FC_CONF_DONE] = 0;
      p.ctr[FC_SEQ_DONE] = 0;
      p.ctr[FC_EXIT] = 0;
    }
  }
}

}  // namespace sb

namespace sb {
// The fused step covers unsharded, 16-byte aligned rows of 16-byte multiples and
// B <= 1024 (plan in shared memory).  It is OPT-IN (SB_FLOW=1): measured on B200 it is
// slower than the warp-specialised TMA kernels even on the small configurations it was
// built for (C2 verify + select 82 vs 56 us; C1 one round 34 vs 30 us; DESIGN.md §13 has
// the globaltimer timeline): its register-staged items execute ~2x the instructions per
// byte of k_rows_tma and every V-segment adds a chain of dependent global round trips
// (partial -> fence -> atomic -> combine -> epilogue -> release) of ~1 us each.
bool flow_eligible(const sb_dims* dd, const void* PL, const void* QL) {
  const char* e = getenv("SB_FLOW");
  if (!(e && e[0] == '1') || tma_disabled() || sharded(dd)) return false;
  if (!vec_ok(dd, PL) || !vec_ok(dd, QL)) return false;
  const size_t rb = (size_t)dd->V * elem_size(dd);
  return rb % 16 == 0 && dd->B <= kFlowMaxB && rb <= ((size_t)kFlowMaxScale - 1) * 8 * kSegBytes;
}

FlowParams flow_params(const sb_dims* dd, const Workspace& w) {
  FlowParams p{};
  p.d = to_dims(dd);
  const size_t rb = (size_t)dd->V * elem_size(dd);
  const int nsub = (int)((rb + kSegBytes - 1) / kSegBytes);
  const int smax = std::max(1, (int)(rb / kMinSegBytes));
  p.nsub = nsub;
  p.Sc = std::min(smax, std::max(1, (kFlowTarget + dd->B * std::max(1, dd->G) - 1) / (dd->B * std::max(1, dd->G))));
  p.Ss = std::min(std::max(1, nsub / 8), std::max(1, (kFlowTarget + dd->B - 1) / dd->B));
  p.ctr = w.fctr; p.rcnt = w.frcnt; p.ccnt = w.fccnt; p.cgrp = w.fcgrp; p.seqcnt = w.cnt; p.scnt = w.fscnt;
  p.gam = w.fgam; p.ready = w.ready; p.rpart = w.frpart; p.cpart = w.fcpart; p.qstate = w.qrs;
  p.cstat = w.conf_stat; p.cc = w.conf_c; p.rowstat = w.rowstat; p.pflag = w.pflag; p.dec = w.dec;
  p.subs = w.segs;
  p.sub_stride = (int)((rb + 511) / 512);  // carve() sizes segs as [B][2][512-byte segments]
  p.segmax = w.fsegmax;
  p.segmax_stride = nsub / 8 + 1;
  return p;
}

template <typename T>
static sb_status launch_flow(const FlowParams& p, cudaStream_t s) {
  const int smem = (int)sizeof(FlowSmem);
  if (ensure_smem<k_flow<T>>(smem) != cudaSuccess) return SB_ERR_CUDA;
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_flow<T>, kFT, smem);
  const int grid = std::max(1, occ) * num_sms();  // all co-resident (the S phase spins)
  return cuda_status(launch_pdl(k_flow<T>, dim3(grid), dim3(kFT), smem, s, p));
}

sb_status flow_run(const FlowParams& p, int dtype, cudaStream_t s) {
  return dtype == SB_BF16 ? launch_flow<__nv_bfloat16>(p, s) : launch_flow<float>(p, s);
}
}  // namespace sb

using namespace sb;

// Fill the verify + select outputs of a FlowParams (shared by both entry points).
static void flow_outputs(FlowParams& p, const void* p_logits, const void* q_logits, const int32_t* tok,
                         const float* u, const float* us, const int32_t* gamma, const int32_t* branch_pos,
                         sb_select_rule rule, float* lse_p, float* lse_q, float* p_tok, float* q_tok,
                         uint32_t* acc_mask, int32_t* n_acc, float* top1_q, int32_t* top1_id_q, float* entropy_q,
                         int32_t* status, int32_t* sel_k, int32_t* commit_len, int32_t* out_tok, int32_t* y_tok,
                         int32_t* y_kind, int32_t* offsets, int32_t* packed_tok, int32_t* path_rolled,
                         int32_t* branch_discarded, uint32_t* keep_mask, float* resid_mass) {
  p.PL = p_logits; p.QL = q_logits; p.tok = tok; p.u = u; p.us = us; p.gamma_in = gamma; p.bpos_in = branch_pos;
  p.rule = rule;
  p.lse_p = lse_p; p.lse_q = lse_q; p.p_tok = p_tok; p.q_tok = q_tok; p.acc_mask = acc_mask; p.n_acc = n_acc;
  p.top1_q = top1_q; p.top1_id_q = top1_id_q; p.entropy_q = entropy_q; p.status = status;
  p.sel_k = sel_k; p.commit_len = commit_len; p.out_tok = out_tok; p.y_tok = y_tok; p.y_kind = y_kind;
  p.offsets = offsets; p.packed_tok = packed_tok; p.path_rolled = path_rolled; p.branch_discarded = branch_discarded;
  p.keep_mask = keep_mask; p.resid_mass = resid_mass;
}

// sb_verify_select's small-batch path (called from sb_verify.cu after its argument checks).
sb_status sb_flow_verify_select(const sb_dims* dd, const void* p_logits, const void* q_logits, const int32_t* tok,
                                const float* u, const float* us, const int32_t* gamma, const int32_t* branch_pos,
                                sb_select_rule rule, float* lse_p, float* lse_q, float* p_tok, float* q_tok,
                                uint32_t* acc_mask, int32_t* n_acc, float* top1_q, int32_t* top1_id_q,
                                float* entropy_q, int32_t* status, int32_t* sel_k, int32_t* commit_len,
                                int32_t* out_tok, int32_t* y_tok, int32_t* y_kind, int32_t* offsets,
                                int32_t* packed_tok, int32_t* path_rolled, int32_t* branch_discarded,
                                uint32_t* keep_mask, float* resid_mass, void* workspace, cudaStream_t s) {
  FlowParams p = flow_params(dd, carve(*dd, workspace));
  flow_outputs(p, p_logits, q_logits, tok, u, us, gamma, branch_pos, rule, lse_p, lse_q, p_tok, q_tok, acc_mask,
               n_acc, top1_q, top1_id_q, entropy_q, status, sel_k, commit_len, out_tok, y_tok, y_kind, offsets,
               packed_tok, path_rolled, branch_discarded, keep_mask, resid_mass);
  p.adaptive = 0;
  return flow_run(p, dd->dtype, s);
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
  if (flow_eligible(dd, p_logits, q_logits)) {
    FlowParams p = flow_params(dd, w);
    flow_outputs(p, p_logits, q_logits, tok, u, us, c_gamma_next, branch_pos, rule, lse_p, lse_q, p_tok, q_tok,
                 acc_mask, n_acc, top1_q, top1_id_q, entropy_q, status, sel_k, commit_len, out_tok, y_tok, y_kind,
                 offsets, packed_tok, path_rolled, branch_discarded, keep_mask, resid_mass);
    p.adaptive = 1;
    p.eps = eps;
    p.k_max = k_max;
    p.c_top1 = c_top1_prob; p.c_id = c_top1_id; p.c_ent = c_entropy; p.c_stat = c_stat; p.c_stop = c_stop;
    p.c_knext = c_k_next; p.c_gamma = c_gamma_next;
    return flow_run(p, dd->dtype, s);
  }
  // large problems: the three streaming kernels (the verify reuses the confidence pass's
  // slot-0 draft-row states)
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

#ifdef SB_FLOW_TRACE
extern "C" int sb_flow_trace_read(void* host, size_t bytes) {
  return (int)cudaMemcpyFromSymbol(host, sb::g_trace, bytes < sizeof(sb::g_trace) ? bytes : sizeof(sb::g_trace));
}
#endif
