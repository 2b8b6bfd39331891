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
#include "sb_ring.cuh"
#include "sb_block_sample.cuh"
#include "sb_sample.cuh"
#include "sb_rows.cuh"

#ifdef SB_TRACE
SB_TRACE_TABLE(sb_trace_select)
#endif

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
  int* sel_cnt;   // [0] completion, [1] dynamic sequence, [2] stopped-decider counters
  int *sel_k, *commit_len, *out_tok, *y_tok, *y_kind, *offsets, *packed_tok, *path_rolled,
      *branch_discarded, *status;
  uint32_t* keep_mask;
  float* resid_mass;
};

template <typename T, int NT>
__global__ void __launch_bounds__(NT) k_select(SelParams p, bool vec_ok) {
  using S = Sampler<T, NT>;
  constexpr int NW = S::NW;
  __shared__ SampleSmem<NW> sm;
  RowStat* red = sm.red;
  __shared__ int sh_ksel, sh_npath, sh_kind, sh_row, sh_slot, sh_st, sh_last;
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
  }
  __syncthreads();
  const int ksel = sh_ksel, npath = sh_npath;
  int kind = sh_kind;
  int y = -1;
  double mass = 0.0;
  if (kind != 0) {
    S smp;
    smp.prow = PL + row_off(d, b, sh_slot, sh_row);
    smp.qrow = QL + row_off(d, b, sh_slot, sh_row);
    smp.V = d.V;
    smp.vec_ok = vec_ok;
    int cls;
    float MSp, Zp, MSq = 0.f, Zq = 1.f;
    if (kind == 2) {
      float m;
      const RowOut o = block_row_stats<T, NT>(smp.prow, d.V, vec_ok, red, &m);
      MSp = o.MS; Zp = (float)o.Z; cls = o.st;
    } else {
      const float4 rs = p.rowstat[ent(d, b, sh_slot, sh_row)];
      MSp = rs.x; Zp = rs.y; MSq = rs.z; Zq = rs.w;
      cls = z_class(Zp) | z_class(Zq);
    }
    if (cls) {
      kind = 0;
      if (tid == 0) sh_st |= cls;
    } else {
      smp.MSp = MSp; smp.iZp = 1.f / Zp; smp.MSq = MSq; smp.iZq = 1.f / Zq;
      smp.resid = (kind == 1);
      int st = 0;
      y = block_sample<T, NT>(smp, __ldg(p.us + b), sm, st, mass);
      if (tid == 0) sh_st |= st;
    }
  }

  // commit: path tokens, y, counters, keep mask (SURVEY §8.0 "Commit"), by the first warp
  if (tid < 32)
    commit_seq(d, p.tok, p.status,
               CommitOut{p.sel_k, p.commit_len, p.out_tok, p.y_tok, p.y_kind, p.offsets, p.packed_tok, p.path_rolled,
                         p.branch_discarded, p.keep_mask, p.resid_mass},
               b, in, ksel, npath, kind, y, mass, sh_st);

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

// ---------------------------------------------------------------- TMA select
// Persistent, one CTA per SM, sequences b = blockIdx.x + k*gridDim.x, four warp roles:
//   decider   (warp 18): Eq. 9 / Alg. 1 selection and the sampling row, one sequence
//                        ahead per queue slot (lanes = branches, shuffle argmax);
//   producer  (warp 16): cp.async.bulk of the sampled row (pair) in 16 KB chunks;
//   consumers (0..15)  : r(v) = max(0, P - Q) (or P) for 16 ids per thread per chunk,
//                        per-lane sums + warp Kogge-Stone scan -> one sum per
//                        512-byte segment (32 lanes x 16 B, ascending ids);
//                        a bonus row first gets a softmax-state pass;
//   epilogue  (warp 17): fp64 prefix over segment sums, locate us*R, re-read that one
//                        segment (L2), same arithmetic -> first id past us*R; commit.
// 20 consumer warps x 5 stages of 20 KB (same box, C4: select 0.236-0.237 ms against
// 0.246 ms for 16 x 6 x 16 KB; 12 x 8: 0.28, 24 x 4: 0.240-0.243; SB_SEL_NS / SB_SEL_CW:
// experiment builds)
#ifndef SB_SEL_NS
#define SB_SEL_NS 5
#endif
#ifndef SB_SEL_CW
#define SB_SEL_CW 20
#endif
constexpr int sNS = SB_SEL_NS;
constexpr int sCW = SB_SEL_CW;
constexpr int sCT = sCW * 32;
constexpr int sVPT = 2;
constexpr int sChunk = sCT * sVPT * 16;  // sCW KB per row per stage
constexpr int sNQ = 4;                   // sequences in flight
constexpr int sSegMax = 1024;            // 1 KB segments per row (one per consumer warp per chunk)
constexpr int sThreads = sCT + 96;

struct Dec {
  int b;  // sequence (-1: no more work)
  int ksel, npath, kind, row, slot;
  float4 rs;  // softmax state of the sampled row pair (kind 1; from sb_verify_branches)
};

struct SelSmem {
  uint64_t full[sNS], empty[sNS];
  uint64_t dfull[sNQ], dempty[sNQ], sfull[sNQ];
  Dec dec[sNQ];
  float rs[sNQ][4];
  int ok[sNQ];  // row class of the sampled row(s): 0, SB_ST_NONFINITE, SB_ST_RANGE
  RowStat red[sCW];
  float seg[sNQ][sSegMax];
  int s_last;
  int scan[32];
  alignas(128) uint8_t buf[sNS][2][sChunk];
};

// Consumer pass A over one sampled row (pair): one sum per 1 KB segment.  RESID is a
// template parameter so neither path is predicated into the other.
template <typename T, bool RESID>
__device__ __forceinline__ void seg_pass(SelSmem& S, RingPos<sNS>& rp, int q, int nchunks, int nvec_last,
                                         bool ok, float MSp, float MSq, float kq) {
  constexpr int E = Vec<T>::E;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int c = 0; c < nchunks; ++c) {
    const int nvec = (c == nchunks - 1) ? nvec_last : sChunk / 16;
    mbar_wait(&S.full[rp.stage], rp.phase);
    uint4 vp[2], vq[2];
#pragma unroll
    for (int j = 0; j < 2; ++j) {  // lane owns 2 adjacent vectors of its warp's 1 KB segment
      const int v = warp * 64 + lane * 2 + j;
      if (v < nvec) {
        vp[j] = lds128(S.buf[rp.stage][0] + v * 16);
        if (RESID) vq[j] = lds128(S.buf[rp.stage][1] + v * 16);
      } else {
        vp[j] = vq[j] = (sizeof(T) == 2) ? make_uint4(0xff80ff80u, 0xff80ff80u, 0xff80ff80u, 0xff80ff80u)
                                         : make_uint4(0xff800000u, 0xff800000u, 0xff800000u, 0xff800000u);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&S.empty[rp.stage]);
    rp.advance();
    float own = 0.f;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      float r[E];
      r_scaled<T>(vp[j], vq[j], RESID, MSp, MSq, kq, r);
      own = seq_sum<E>(r, own);
    }
    const float tot = warp_sum_rn(ok ? own : 0.f);
    if (lane == 0) S.seg[q][c * (sChunk / kSegBytes) + warp] = tot;
  }
}

template <typename T>
__global__ void __launch_bounds__(sThreads, 1) k_select_tma(SelParams p) {
  constexpr int E = Vec<T>::E;
  extern __shared__ __align__(128) uint8_t smem_raw[];
  SelSmem& S = *reinterpret_cast<SelSmem*>(smem_raw);
  const Dims& d = p.d;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < sNS; ++s) {
      mbar_init(&S.full[s], 1);
      mbar_init(&S.empty[s], sCW);
    }
    for (int s = 0; s < sNQ; ++s) {
      mbar_init(&S.dfull[s], 1);
      mbar_init(&S.dempty[s], 1);
      mbar_init(&S.sfull[s], sCW);
    }
    S.s_last = 0;
    fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0) SB_TRACE_AT(sb_trace_select, 0, 0);
  pdl_wait();
  if (tid == 0) SB_TRACE_AT(sb_trace_select, 0, 1);
  const T* PL = static_cast<const T*>(p.PL);
  const T* QL = static_cast<const T*>(p.QL);
  const uint32_t row_bytes = (uint32_t)d.V * sizeof(T);
  const int nchunks = (row_bytes + sChunk - 1) / sChunk;
  const int nvec_last = (int)(row_bytes - (uint32_t)(nchunks - 1) * sChunk) / 16;
  const int nseg = nchunks * (sChunk / kSegBytes);

  if (warp == sCW + 2) {  // ---------------- decider
    RingPos<sNQ> dq;
    for (;;) {
      if (lane == 0) mbar_wait(&S.dempty[dq.stage], dq.phase ^ 1u);
      __syncwarp();
      int b = 0;
      if (lane == 0) b = atomicAdd(p.sel_cnt + 1, 1);  // dynamic: sequences differ in cost
      b = __shfl_sync(0xffffffffu, b, 0);
      if (b >= d.B) {
        if (lane == 0) {
          S.dec[dq.stage].b = -1;
          mbar_arrive(&S.dfull[dq.stage]);
          // the last decider to stop resets the work counter (all increments are done)
          if (atomicAdd(p.sel_cnt + 2, 1) == (int)gridDim.x - 1) {
            p.sel_cnt[1] = 0;
            p.sel_cnt[2] = 0;
          }
        }
        break;
      }
      const SeqInfo in = p.info[b];
      // lane k: is branch k in A = {k : n_k > s_b}, and its key
      const int k = lane;
      int nk = 0, xk = 0x7fffffff;
      float key = -CUDART_INF_F;
      bool inA = false;
      if (k < d.K) {
        nk = __ldg(p.n_acc + (int64_t)b * d.K + k);
        inA = nk > in.s;
        if (inA) {
          xk = __ldg(p.tok + ent(d, b, k, in.s));
          key = (p.rule == SB_SELECT_ALG1) ? __ldg(p.u + ent(d, b, k, in.s))
                                           : ld_scalar(PL + row_off(d, b, 0, in.s) + xk);
        }
      }
      // argmax over A: larger key; Eq. 9 ties -> smaller token then smaller k; Alg. 1 ties -> smaller k
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
      const int n0 = __shfl_sync(0xffffffffu, nk, 0);
      const int nsel = __shfl_sync(0xffffffffu, nk, ksel < 0 ? 0 : ksel);
      if (lane == 0) {
        Dec D;
        D.b = b;
        D.ksel = ksel;
        if (ksel < 0) {
          D.npath = min(n0, in.s);  // rejection in the shared prefix or at the branch row (P655)
          D.kind = 1; D.row = D.npath; D.slot = 0;
        } else {
          D.npath = nsel;
          if (nsel < in.L) { D.kind = 1; D.row = nsel; D.slot = (nsel <= in.s) ? 0 : ksel; }
          else if (in.s < in.g) { D.kind = 2; D.row = in.g; D.slot = ksel; }  // bonus, p_{gamma+1}
          else { D.kind = 0; D.row = 0; D.slot = 0; }  // branch token accepted (P237)
        }
        D.rs = (D.kind == 1) ? p.rowstat[ent(d, b, D.slot, D.row)] : make_float4(0.f, 1.f, 0.f, 1.f);
        S.dec[dq.stage] = D;
        mbar_arrive(&S.dfull[dq.stage]);
      }
      dq.advance();
    }
  } else if (warp == sCW) {  // ---------------- producer
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      RingPos<sNQ> dq;
      RingPos<sNS> rp;
      for (;;) {
        mbar_wait(&S.dfull[dq.stage], dq.phase);
        const Dec D = S.dec[dq.stage];
        dq.advance();
        if (D.b < 0) break;
        const int b = D.b;
        const int npass = D.kind == 1 ? 1 : (D.kind == 2 ? 2 : 0);
        const char* prow = reinterpret_cast<const char*>(PL + row_off(d, b, D.slot, D.row));
        const char* qrow = reinterpret_cast<const char*>(QL + row_off(d, b, D.slot, D.row));
        for (int pass = 0; pass < npass; ++pass)
          for (int c = 0; c < nchunks; ++c) {
            const uint32_t bytes = min((uint32_t)sChunk, row_bytes - (uint32_t)c * sChunk);
            mbar_wait(&S.empty[rp.stage], rp.phase ^ 1u);
            mbar_expect_tx(&S.full[rp.stage], (D.kind == 1 ? 2 : 1) * bytes);
            bulk_g2s(S.buf[rp.stage][0], prow + (size_t)c * sChunk, bytes, &S.full[rp.stage], pol);
            if (D.kind == 1)
              bulk_g2s(S.buf[rp.stage][1], qrow + (size_t)c * sChunk, bytes, &S.full[rp.stage], pol);
            rp.advance();
          }
      }
    }
  } else if (warp == sCW + 1) {  // ---------------- epilogue
    RingPos<sNQ> dq;
    for (;;) {
      mbar_wait(&S.dfull[dq.stage], dq.phase);
      const Dec D = S.dec[dq.stage];
      if (D.b < 0) break;
      const int b = D.b;
      mbar_wait(&S.sfull[dq.stage], dq.phase);
      const SeqInfo in = p.info[b];
      const int q = dq.stage;
      int kind = D.kind, y = -1, st = 0;
      double mass = 0.0;
      if (kind != 0) {
        const float MSp = S.rs[q][0], Zp = S.rs[q][1], MSq = S.rs[q][2], Zq = S.rs[q][3];
        if (S.ok[q]) {
          kind = 0;
          st |= S.ok[q];
        } else {
          const T* prow = PL + row_off(d, b, D.slot, D.row);
          const T* qrow = QL + row_off(d, b, D.slot, D.row);
          bool resid = (kind == 1);
          double R = 0.0;
          y = sample_segments<T>(prow, qrow, row_bytes, d.V, S.seg[q], nseg, resid, MSp, MSq, Zp / Zq,
                                 __ldg(p.us + b), st, &R);
          mass = R / (double)Zp;  // back to probability mass
        }
      }
      commit_seq(d, p.tok, p.status,
                 CommitOut{p.sel_k, p.commit_len, p.out_tok, p.y_tok, p.y_kind, p.offsets, p.packed_tok,
                           p.path_rolled, p.branch_discarded, p.keep_mask, p.resid_mass},
                 b, in, D.ksel, D.npath, kind, y, mass, st);
      __syncwarp();
      if (lane == 0) mbar_arrive(&S.dempty[dq.stage]);
      if (lane == 0) SB_TRACE_AT(sb_trace_select, 2, 2 + (b / gridDim.x));
      dq.advance();
      // global completion -> the last sequence's epilogue scans the offsets
      int last = 0;
      if (lane == 0) {
        __threadfence();
        last = (atomicAdd(p.sel_cnt, 1) == d.B - 1);
      }
      last = __shfl_sync(0xffffffffu, last, 0);
      if (last && lane == 0) S.s_last = 1;  // the whole CTA compacts once every role is done
    }
  } else {  // ---------------- consumers
  RingPos<sNQ> dq;
  RingPos<sNS> rp;
  for (;;) {
    mbar_wait(&S.dfull[dq.stage], dq.phase);
    const Dec D = S.dec[dq.stage];
    if (D.b < 0) break;
    const int q = dq.stage;
    if (D.kind == 2) {  // bonus row: its softmax state first
      LazyAcc<false, 4> a;
      a.init();
      for (int c = 0; c < nchunks; ++c) {
        const int nvec = (c == nchunks - 1) ? nvec_last : sChunk / 16;
        mbar_wait(&S.full[rp.stage], rp.phase);
        uint4 x[sVPT];
#pragma unroll
        for (int j = 0; j < sVPT; ++j) {
          const int v = tid + j * sCT;
          x[j] = (v < nvec) ? lds128(S.buf[rp.stage][0] + v * 16) : neg_inf_vec<T>();
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&S.empty[rp.stage]);
        rp.advance();
        if constexpr (sizeof(T) == 2) {  // packed FFMA2 / FADD2 (the same operations as add())
          if (c == 0) acc_vecs_bf16<sVPT, false, true>(a, x, c);
          else acc_vecs_bf16<sVPT, false, false>(a, x, c);
        } else {
          float f[sVPT * E];
#pragma unroll
          for (int j = 0; j < sVPT; ++j) Vec<T>::unpack(x[j], f + j * E);
          if (c == 0) a.template add<sVPT * E, true>(f, c);
          else a.template add<sVPT * E, false>(f, c);
        }
      }
      RowStat s = fold_lazy(a);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s = combine(s, shfl_xor(s, o));
      if (lane == 0) S.red[warp] = s;
      consumer_sync(sCT);
      if (tid == 0) {
        RowStat r = S.red[0];
        for (int j = 1; j < sCW; ++j) r = combine(r, S.red[j]);
        const RowOut o = finish(r);
        S.rs[q][0] = o.MS; S.rs[q][1] = o.Z; S.rs[q][2] = 0.f; S.rs[q][3] = 1.f;
        S.ok[q] = o.st;
      }
      consumer_sync(sCT);
    } else if (D.kind == 1 && tid == 0) {  // the epilogue reads the same state from S.rs
      S.rs[q][0] = D.rs.x; S.rs[q][1] = D.rs.y; S.rs[q][2] = D.rs.z; S.rs[q][3] = D.rs.w;
      S.ok[q] = z_class(D.rs.y) | z_class(D.rs.w);
    }
    if (D.kind != 0) {
      const bool resid = (D.kind == 1);
      const float4 rsv = resid ? D.rs : make_float4(S.rs[q][0], S.rs[q][1], S.rs[q][2], S.rs[q][3]);
      const bool ok = resid ? (z_class(rsv.y) | z_class(rsv.w)) == 0 : (S.ok[q] == 0);
      const float MSp = rsv.x, MSq = rsv.z, kq = rsv.y / rsv.w;
      if (resid)
        seg_pass<T, true>(S, rp, q, nchunks, nvec_last, ok, MSp, MSq, kq);
      else
        seg_pass<T, false>(S, rp, q, nchunks, nvec_last, ok, MSp, MSq, kq);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&S.sfull[q]);
    dq.advance();
  }
  }
  // ---------------- the CTA that finished the last sequence: offsets + packed stream
  __syncthreads();
  if (tid == 0) SB_TRACE_AT(sb_trace_select, 2, 62);
  if (S.s_last) {
    __threadfence();
    block_offsets<sThreads>(d.B, d.G, p.commit_len, p.out_tok, p.offsets, p.packed_tok, S.scan);
    if (tid == 0) p.sel_cnt[0] = 0;  // leave the workspace re-usable
  }
}

template <typename T>
static sb_status launch_select_tma(const SelParams& p, cudaStream_t s) {
  const int smem = (int)sizeof(SelSmem);
  if (ensure_smem<k_select_tma<T>>(smem) != cudaSuccess) return SB_ERR_CUDA;
  const int grid = std::min(num_sms(), p.d.B);
  return cuda_status(launch_pdl(k_select_tma<T>, dim3(grid), dim3(sThreads), smem, s, p));
}

template <typename T, int NT>
static sb_status launch_select(const SelParams& p, bool vok, cudaStream_t s) {
  k_select<T, NT><<<p.d.B, NT, 0, s>>>(p, vok);
  return cuda_status(cudaGetLastError());
}

}  // namespace sb

using namespace sb;

struct sb_comm;
sb_status sb_shard_select_nccl(const sb_dims* d, const void* p_logits, const void* q_logits, const int32_t* tok,
                               const float* u, const float* us, const int32_t* n_acc, sb_select_rule rule,
                               int32_t* sel_k, int32_t* commit_len, int32_t* out_tok, int32_t* y_tok,
                               int32_t* y_kind, int32_t* offsets, int32_t* packed_tok, int32_t* path_rolled,
                               int32_t* branch_discarded, uint32_t* keep_mask, float* resid_mass, int32_t* status,
                               sb_comm* c, void* workspace, size_t workspace_bytes, cudaStream_t s);

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
  SB_NVTX("sb_select_branch");
  (void)gamma;
  (void)branch_pos;  // the clamped layout comes from the workspace (sb_verify_branches)
  if (!dims_valid(dd)) return SB_ERR_INVALID_ARG;
  if (!p_logits || !q_logits || !tok || !u || !us || !n_acc || !sel_k || !commit_len || !out_tok ||
      !y_tok || !y_kind || !offsets || !path_rolled || !branch_discarded || !keep_mask || !status ||
      !workspace)
    return SB_ERR_INVALID_ARG;
  if (rule != SB_SELECT_EQ9 && rule != SB_SELECT_ALG1) return SB_ERR_INVALID_ARG;
  if ((uintptr_t)workspace % 256) return SB_ERR_INVALID_ARG;
  if (comm)
    return sb_shard_select_nccl(dd, p_logits, q_logits, tok, u, us, n_acc, rule, sel_k, commit_len, out_tok,
                                y_tok, y_kind, offsets, packed_tok, path_rolled, branch_discarded, keep_mask,
                                resid_mass, status, (sb_comm*)comm, workspace, workspace_bytes,
                                (cudaStream_t)stream);
  if (sharded(dd)) return SB_ERR_INVALID_ARG;  // a vocabulary shard needs its exchange (comm)
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
  const size_t row_bytes = (size_t)dd->V * elem_size(dd);
  // every chunk holds sCW segments: rows up to (sSegMax / sCW) whole chunks (1020 KB)
  if (vok && row_bytes % 16 == 0 && (row_bytes + sChunk - 1) / sChunk * sCW <= (size_t)sSegMax && !tma_disabled())
    return dd->dtype == SB_BF16 ? launch_select_tma<__nv_bfloat16>(p, s) : launch_select_tma<float>(p, s);
  if (dd->dtype == SB_BF16) {
    if ((dd->V + 256 * 8 - 1) / (256 * 8) > kMaxTiles) return SB_ERR_UNSUPPORTED;
    return launch_select<__nv_bfloat16, 256>(p, vok, s);
  }
  if ((dd->V + 256 * 4 - 1) / (256 * 4) > kMaxTiles) return SB_ERR_UNSUPPORTED;
  return launch_select<float, 256>(p, vok, s);
}
