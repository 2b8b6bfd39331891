// sb_sv.cu — the small-batch step as ONE bulk-synchronous split-vocabulary launch (k_sv):
// sb_step_adaptive (confidence -> verify -> select) and
// sb_verify_select (verify -> select) when the batch is too small to fill the GPU with
// whole rows (C2: 64 sequences, 64 KB rows; one C1 round: 17 row pairs).
//
// Every CTA (one per SM, all co-resident) owns a slice of EVERY row, so each phase
// streams its rows with all SMs at once and no per-row item chain sits on the critical
// path.  Phases, separated by grid barriers (a counter in the workspace):
//   C  confidence rows (slot-0 draft rows 0..G-1): per (row, slice) partial softmax state
//   .  combine C: one warp per row folds its slices' partials (fixed order, fp64 sums),
//      the statistic and, in the warp completing a sequence, Eq. 6 stop / Eq. 7 k /
//      gamma_b = max(1, stop) (conf_epilogue, §4.2 P170, P198, P218)
//   V  every tested row pair of every sequence, from gamma_b (k_plan's layout): slot-0
//      draft rows the confidence pass already reduced stream their p slice only
//   .  combine V: warp_epilogue (fp64 u*Q[x] <= P[x], P94 / Alg. 1 P534, P538); the warp
//      completing a sequence takes the Eq. 9 / Alg. 1 decision (P239, P540) and writes
//      the sequence's sample descriptor (residual row P94/P554, bonus row P94, none P237)
//   S  1 KB segment sums of every sampled row (one warp per segment, the arithmetic of
//      k_select_tma's consumers, so the same sums bit for bit); bonus rows: segment-local
//      offsets, rescaled at the locate step
//   .  locate: one warp per sequence, fp64 prefix over its segments, one segment
//      re-read (sample_segments), commit (commit_seq), offsets by the last committer
//
// Streaming: a unit is one (row, slice) and belongs to ONE lane; a warp takes 32 units
// at a time.  Each warp owns a cp.async ring in shared memory: per stage it copies 4
// consecutive 16-byte vectors of each of its 32 units' rows (8 units x 64 B contiguous
// per warp instruction, coalesced), then every lane reads its own unit's vectors
// (odd pitch: conflict-free LDS.128) into the same lazy-offset accumulators as the other
// kernels (LazyAcc, sb_common.cuh).  No warp reduction per unit: a lane's unit state IS
// the partial record.  Slices are sized so that every lane gets one unit per phase.
#include <cmath>
#include <cstdlib>

#include "sb_host.h"
#include "sb_ring.cuh"
#include "sb_sample.cuh"
#include "sb_conf.cuh"
#include "sb_rows.cuh"

namespace sb {

#ifdef SB_TRACE
}  // namespace sb
SB_TRACE_TABLE(sb_trace_sv)
namespace sb {
#endif

constexpr int kSvCV = 4;              // vectors per row per lane per stage
// stage layout: vector j of unit u at 16-byte slot u*4 + (j ^ ((u >> 1) & 3)): a quarter
// warp's LDS.128 of one j touches 8 distinct 16-byte bank groups (no padding)
__host__ __device__ constexpr int sv_slot(int u, int j) { return u * kSvCV + (j ^ ((u >> 1) & 3)); }
constexpr int kSvMinV = 16;           // minimum slice length (vectors)
constexpr int kSvMaxSl = 256;         // slices per row (sv_fold: <= 8 records per lane)
constexpr int kSvMaxB = 512;          // sequences (per-CTA layout tables in shared memory)

// Sample descriptor of one sequence, written by the warp that completes its verify.
struct SvDesc {
  int kind, slot, i, ksel;
  int npath, pad_[3];
  float4 rs;  // row state (MS_p, Z_p, MS_q, Z_q) of a residual row
};
static_assert(sizeof(SvDesc) == 48, "three 16-byte loads");

struct SvParams {
  RowsParams r;  // verify outputs + workspace (r.qreuse = the confidence pass's row states)
  ConfParams c;  // confidence outputs (K = 1 slot-0 view); unused when !adaptive
  CommitOut co;
  const float* us;
  const int* bpos;
  const int* gamma_in;  // non-adaptive: gamma_b (NULL -> G)
  int adaptive, rule;
  RowStat* part_p;  // [units] per-(row, slice) partial states
  RowStat* part_q;
  SvDesc* desc;     // [B]
  float* seg;       // [B][nseg] segment sums
  float* segm;      // [B][nseg] segment maxima (bonus rows)
  int* ctr;         // [0] barrier, [1] exit count, [2] committed sequences
  int nsl_c;        // slices per confidence row
};

// One streaming sub-phase: rows of one kind, each cut into nsl slices.
struct SvSub {
  int rows, nsl, units;  // units = rows * nsl rounded up to a multiple of 32 (warp-uniform kind)
  int kind;              // 0 confidence (q), 1 verify p only (q state reused), 2 verify p + q
  int pbase;             // partial record index of (row 0, slice 0)
  int S;                 // stages per unit
};

template <int W, int NSTG>
struct SvSmem {
  uint4 ring[W][NSTG][2][32 * kSvCV];
  int pk[kSvMaxB];                    // packed SeqInfo: s | g<<5 | L<<10 | Lr<<16 | st<<22
  int offA[kSvMaxB + 1], offB[kSvMaxB + 1];
  int s_last[W];
  int geo[4];                         // nA, nB, nsl_a, nsl_b
};

__device__ __forceinline__ SeqInfo sv_unpack(int pk) {
  SeqInfo in;
  in.s = pk & 31; in.g = (pk >> 5) & 31; in.L = (pk >> 10) & 63; in.Lr = (pk >> 16) & 63; in.st = pk >> 22;
  in.pad_[0] = in.pad_[1] = in.pad_[2] = 0;
  return in;
}
__device__ __forceinline__ int sv_pack(const SeqInfo& in) {
  return in.s | (in.g << 5) | (in.L << 10) | (in.Lr << 16) | (in.st << 22);
}

// Largest b with off[b] <= r (off: B+1 ascending entries in shared memory).
__device__ __forceinline__ int sv_find(const int* off, int B, int r) {
  int lo = 0, hi = B;
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (off[mid] <= r) lo = mid; else hi = mid;
  }
  return lo;
}

// Row of a sub-phase -> (b, slot, i).
template <int W, int NSTG>
__device__ __forceinline__ void sv_row(const SvSmem<W, NSTG>& S, const Dims& d, int kind, int r, int& b, int& slot,
                                       int& i) {
  if (kind == 0) {
    b = r / d.G; slot = 0; i = r % d.G;
    return;
  }
  if (kind == 1) {
    b = sv_find(S.offA, d.B, r); slot = 0; i = r - S.offA[b];
    return;
  }
  b = sv_find(S.offB, d.B, r);
  const SeqInfo in = sv_unpack(S.pk[b]);
  const int jj = r - S.offB[b] + (S.offA[b + 1] - S.offA[b]);  // position in k_plan's order
  if (jj < in.Lr) { slot = 0; i = jj; return; }
  const int per = in.Lr - 1 - in.s, t = jj - in.Lr;
  slot = 1 + t / per;
  i = in.s + 1 + t % per;
}

__device__ __forceinline__ void st_rowstat(RowStat* dst, const RowStat& s) {
  int4 w[2];
  memcpy(w, &s, sizeof(s));
  int4* o = reinterpret_cast<int4*>(dst);
  o[0] = w[0];
  o[1] = w[1];
}

// Grid barrier n (1, 2, ...) of this launch: every CTA arrives once, then waits for all.
__device__ __forceinline__ void sv_grid_sync(int* bar, int n) {
  __syncthreads();
  if (threadIdx.x == 0) {
    SB_TRACE_AT(sb_trace_sv, 0, 2 * n);
    __threadfence();
    atomicAdd(bar, 1);
    const int target = n * (int)gridDim.x;
    for (uint32_t tries = 0; ld_acq(bar) < target; ++tries)
      if (tries > (1u << 28)) __trap();  // watchdog: a CTA never arrived
    __threadfence();
    SB_TRACE_AT(sb_trace_sv, 0, 2 * n + 1);
  }
  __syncthreads();
}

// One stage of a unit (kSvCV vectors of one row) into its accumulator.
template <typename T, bool kQ, bool FIRST>
__device__ __forceinline__ void sv_acc(LazyAcc<kQ, 4>& a, const uint4* x, int t) {
  if constexpr (sizeof(T) == 2) {
    acc_vecs_bf16<kSvCV, kQ, FIRST>(a, x, t);
  } else {
    float f[kSvCV * 4];
#pragma unroll
    for (int j = 0; j < kSvCV; ++j) Vec<float>::unpack(x[j], f + 4 * j);
    a.template add<kSvCV * 4, FIRST>(f, t);
  }
}

// Exact first index of a q unit's maximum: re-read the kSvCV vectors of the stage where
// the lane first saw it (tag) and take the first element equal to m.
template <typename T>
__device__ __forceinline__ int sv_argmax(const char* base, int v0, int nv, int tag, float m) {
  constexpr int E = Vec<T>::E;
  if (tag < 0 || !(m > -CUDART_INF_F)) return 0x7fffffff;
  int cand = 0x7fffffff;
#pragma unroll
  for (int j = kSvCV - 1; j >= 0; --j) {
    const int v = tag * kSvCV + j;
    if (v >= nv) continue;
    float f[E];
    Vec<T>::unpack(__ldg(reinterpret_cast<const uint4*>(base) + v), f);
#pragma unroll
    for (int e = E - 1; e >= 0; --e)
      if (f[e] == m) cand = (v0 + v) * E + e;
  }
  return cand;
}

// The streaming phase: this warp's units of the sub-phases, in order.  A stage holds 4
// vectors of each unit's p and q rows (pairs) or 8 vectors of its one row (the two halves
// of the stage), so every stage moves 4 KB per warp whatever the kind.
template <typename T, int W, int NSTG>
__device__ void sv_stream(const SvParams& sp, SvSmem<W, NSTG>& S, const SvSub* sub, int nsub, int nvec) {
  const Dims& d = sp.r.d;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int NC = gridDim.x;
  const char* PL = static_cast<const char*>(sp.r.PL);
  const char* QL = static_cast<const char*>(sp.r.QL);
  int total_chunks = 0;
  for (int j = 0; j < nsub; ++j) total_chunks += sub[j].units / 32;
  const int first = blockIdx.x + NC * w, step = NC * W;
  if (first >= total_chunks) return;

  struct Cur {
    int chunk;  // chunk index (global); >= total_chunks: done
    int sp;     // sub-phase
    int stage;  // stage within the unit
    int row, slice, v0, nv;   // this lane's unit
    const char *pb, *qb;      // its slice bases (p, q)
  };
  auto locate = [&](Cur& c) {
    int ch = c.chunk, j = 0;
    while (j + 1 < nsub && ch >= sub[j].units / 32) { ch -= sub[j].units / 32; ++j; }
    c.sp = j;
    c.stage = 0;
    const SvSub& su = sub[j];
    const int u = ch * 32 + lane;
    c.row = u / su.nsl;
    c.slice = u % su.nsl;
    c.nv = 0; c.v0 = 0; c.pb = c.qb = nullptr;
    if (c.row < su.rows) {
      c.v0 = (int)((int64_t)c.slice * nvec / su.nsl);
      c.nv = (int)((int64_t)(c.slice + 1) * nvec / su.nsl) - c.v0;
      int b, slot, i;
      sv_row(S, d, su.kind, c.row, b, slot, i);
      const int64_t off = (row_off(d, b, slot, i) * (int64_t)sizeof(T)) + (int64_t)c.v0 * 16;
      c.pb = PL + off;
      c.qb = QL + off;
    }
  };

  // copy side: this lane copies vector (lane & 3) of units u = k*8 + lane/4, k = 0..3
  Cur cc{first, 0, 0, 0, 0, 0, 0, nullptr, nullptr};
  locate(cc);
  const char* cpb[4];
  const char* cqb[4];
  int cnv[4];
  auto gather = [&]() {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int u = k * 8 + (lane >> 2);
      cpb[k] = reinterpret_cast<const char*>(__shfl_sync(0xffffffffu, (unsigned long long)cc.pb, u));
      cqb[k] = reinterpret_cast<const char*>(__shfl_sync(0xffffffffu, (unsigned long long)cc.qb, u));
      cnv[k] = __shfl_sync(0xffffffffu, cc.nv, u);
    }
  };
  gather();
  int issued = 0;
  auto issue = [&]() {
    if (cc.chunk < total_chunks) {
      const SvSub& su = sub[cc.sp];
      const int slot = issued % NSTG;
      const int j = lane & 3;
      if (su.kind == 2) {  // pairs: p -> half 0, q -> half 1
        const int vv = cc.stage * kSvCV + j;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int u = k * 8 + (lane >> 2);
          if (vv < cnv[k]) {
            cp_async16(&S.ring[w][slot][0][sv_slot(u, j)], cpb[k] + (size_t)vv * 16);
            cp_async16(&S.ring[w][slot][1][sv_slot(u, j)], cqb[k] + (size_t)vv * 16);
          }
        }
      } else {  // one row: vectors 8s..8s+3 -> half 0, 8s+4..8s+7 -> half 1
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int vv = cc.stage * 2 * kSvCV + h * kSvCV + j;
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const int u = k * 8 + (lane >> 2);
            const char* base = su.kind == 0 ? cqb[k] : cpb[k];
            if (vv < cnv[k]) cp_async16(&S.ring[w][slot][h][sv_slot(u, j)], base + (size_t)vv * 16);
          }
        }
      }
      if (++cc.stage == su.S) {  // this warp's next chunk
        cc.chunk += step;
        if (cc.chunk < total_chunks) {
          locate(cc);
          gather();
        }
      }
    }
    cp_async_commit();
    ++issued;
  };
#pragma unroll
  for (int t = 0; t < NSTG - 1; ++t) issue();

  Cur xc{first, 0, 0, 0, 0, 0, 0, nullptr, nullptr};  // compute side
  locate(xc);
  LazyAcc<false, 4> pa;
  LazyAcc<true, 4> qa;
  pa.init();
  qa.init();
  for (int t = 0;; ++t) {
    cp_async_wait<NSTG - 2>();
    __syncwarp();
    issue();
    const SvSub& su = sub[xc.sp];
    const int slot = t % NSTG;
    uint4 x0[kSvCV], x1[kSvCV];
    const int vb = su.kind == 2 ? xc.stage * kSvCV : xc.stage * 2 * kSvCV;
    const int vb1 = su.kind == 2 ? vb : vb + kSvCV;
#pragma unroll
    for (int j = 0; j < kSvCV; ++j) {
      x0[j] = vb + j < xc.nv ? S.ring[w][slot][0][sv_slot(lane, j)] : neg_inf_vec<T>();
      x1[j] = vb1 + j < xc.nv ? S.ring[w][slot][1][sv_slot(lane, j)] : neg_inf_vec<T>();
    }
    const int g0 = xc.stage * 2;  // 4-vector group tags: 2s, 2s + 1 (single rows)
    if (su.kind == 0) {
      if (xc.stage == 0) sv_acc<T, true, true>(qa, x0, 0);
      else sv_acc<T, true, false>(qa, x0, g0);
      sv_acc<T, true, false>(qa, x1, g0 + 1);
    } else if (su.kind == 1) {
      if (xc.stage == 0) sv_acc<T, false, true>(pa, x0, 0);
      else sv_acc<T, false, false>(pa, x0, g0);
      sv_acc<T, false, false>(pa, x1, g0 + 1);
    } else {
      if (xc.stage == 0) {
        sv_acc<T, false, true>(pa, x0, 0);
        sv_acc<T, true, true>(qa, x1, 0);
      } else {
        sv_acc<T, false, false>(pa, x0, xc.stage);
        sv_acc<T, true, false>(qa, x1, xc.stage);
      }
    }
    if (++xc.stage < su.S) continue;
    // unit complete: its partial records
    if (xc.row < su.rows) {
      const int64_t rec = su.pbase + (int64_t)xc.row * su.nsl + xc.slice;
      if (su.kind != 0) st_rowstat(sp.part_p + rec, fold_lazy(pa));
      if (su.kind != 1) {
        RowStat qs = fold_lazy(qa);
        qs.idx = sv_argmax<T>(xc.qb, xc.v0, xc.nv, qa.tag, qa.m);
        st_rowstat(sp.part_q + rec, qs);
      }
    }
    pa.init();
    qa.init();
    xc.chunk += step;
    if (xc.chunk >= total_chunks) break;
    locate(xc);
  }
  cp_async_wait<0>();
  __syncwarp();
}

// One warp: the row state of `n` partial records.  Each lane folds its records (slice
// order, two loads in flight), then the warp moves to its largest offset and sums in fp64
// (warp_reduce_offsets); the max and its first index reduce separately.  Fixed order.
// Not inlined and not unrolled: the combine phases run this once per row on cold SMs,
// where instruction fetch, not arithmetic, sets the time (profiles/r4_sv_*.txt).
__device__ __noinline__ RowStat sv_fold(const RowStat* part, int n) {
  const int lane = threadIdx.x & 31;
  RowStat s = rowstat_empty();
#pragma unroll 1
  for (int j = lane; j < n; j += 64) {
    const RowStat a = ldcg_rowstat(part + j);
    const RowStat b = j + 32 < n ? ldcg_rowstat(part + j + 32) : rowstat_empty();
    s = combine(combine(s, a), b);
  }
  float m = s.m;
#pragma unroll 1
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  const int idx = (int)__reduce_min_sync(0xffffffffu, (unsigned)(s.m == m ? s.idx : 0x7fffffff));
  float MS = s.ms;
#pragma unroll 1
  for (int o = 16; o > 0; o >>= 1) MS = fmaxf(MS, __shfl_xor_sync(0xffffffffu, MS, o));
  shift_to(s, MS);
  double z = s.z, s1 = s.s1;
#pragma unroll 1
  for (int o = 16; o > 0; o >>= 1) {
    z += __shfl_xor_sync(0xffffffffu, z, o);
    s1 += __shfl_xor_sync(0xffffffffu, s1, o);
  }
  s.z = z;
  s.s1 = s1;
  s.m = m;
  s.idx = idx;
  return s;
}

// Offsets (exclusive scan of commit_len) and the packed commit stream, by one warp with
// every load of a phase in flight at once (warp_offsets walks its sequences' tokens one
// dependent load at a time).  scratch: shared memory for 2 (B + 1) ints.
__device__ __forceinline__ void sv_offsets(int B, int G, const int* commit_len, const int* out_tok, int* offsets,
                                           int* packed_tok, int* scratch) {
  const int lane = threadIdx.x & 31;
  int* cl = scratch;
  int* off = scratch + B + 1;
  for (int b = lane; b < B; b += 32) cl[b] = __ldcg(commit_len + b);
  __syncwarp();
  const int per = (B + 31) / 32;
  const int b0 = min(B, lane * per), b1 = min(B, b0 + per);
  int loc = 0;
  for (int b = b0; b < b1; ++b) loc += cl[b];
  int incl = loc;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  int run = incl - loc;
  for (int b = b0; b < b1; ++b) {
    off[b] = run;
    offsets[b] = run;
    run += cl[b];
  }
  const int total = __shfl_sync(0xffffffffu, incl, 31);
  if (lane == 0) {
    off[B] = total;
    offsets[B] = total;
  }
  __syncwarp();
  if (!packed_tok) return;
  for (int f0 = 0; f0 < total; f0 += 128) {
    int v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int f = f0 + 32 * k + lane;
      v[k] = 0;
      if (f < total) {
        const int b = sv_find(off, B, f);
        v[k] = __ldcg(out_tok + (int64_t)b * (G + 2) + (f - off[b]));
      }
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int f = f0 + 32 * k + lane;
      if (f < total) packed_tok[f] = v[k];
    }
  }
}

// Eq. 9 / Alg. 1 decision of sequence b in the warp that completed it (lane k < K holds
// n_k): the kept branch k*, the committed path length and the row to sample from.
template <typename T>
__device__ __forceinline__ SvDesc sv_decide(const SvParams& sp, int b, const SeqInfo& in, int nk) {
  const RowsParams& p = sp.r;
  const Dims& d = p.d;
  const int lane = threadIdx.x & 31;
  float key = 0.f;
  int xk = 0;
  const bool surv = lane < d.K && nk > in.s;  // A = {k : n_k > s_b} (P239, P540)
  if (surv) {
    xk = __ldg(p.tok + ent(d, b, lane, in.s));
    key = (sp.rule == SB_SELECT_ALG1) ? __ldg(p.u + ent(d, b, lane, in.s))
                                      : ld_scalar(static_cast<const T*>(p.PL) + row_off(d, b, 0, in.s) + xk);
  }
  int ksel = -1, besttok = 0;
  float bestkey = 0.f;
  for (int k = 0; k < d.K; ++k) {  // in branch order, as the oracle: ties -> smaller token, then smaller k
    const int sk = __shfl_sync(0xffffffffu, (int)surv, k);
    const float kk = __shfl_sync(0xffffffffu, key, k);
    const int xx = __shfl_sync(0xffffffffu, xk, k);
    if (!sk) continue;
    bool better;
    if (ksel < 0) better = true;
    else if (sp.rule == SB_SELECT_ALG1) better = kk > bestkey;
    else better = kk > bestkey || (kk == bestkey && xx < besttok);
    if (better) { ksel = k; bestkey = kk; besttok = xx; }
  }
  SvDesc o{};
  o.ksel = ksel;
  if (ksel < 0) {
    o.npath = min(__shfl_sync(0xffffffffu, nk, 0), in.s);  // rollback on the shared rows (P655)
    o.kind = 1; o.i = o.npath; o.slot = 0;
  } else {
    o.npath = __shfl_sync(0xffffffffu, nk, ksel);
    if (o.npath < in.L) { o.kind = 1; o.i = o.npath; o.slot = (o.npath <= in.s) ? 0 : ksel; }  // residual (P94, P554)
    else if (in.s < in.g) { o.kind = 2; o.i = in.g; o.slot = ksel; }                            // bonus (P94)
    else { o.kind = 0; o.i = 0; o.slot = 0; }                                                   // (P237)
  }
  o.rs = (o.kind == 1) ? __ldcg(p.rowstat + ent(d, b, o.slot, o.i)) : make_float4(0.f, 1.f, 0.f, 1.f);
  return o;
}

template <typename T, int W, int NSTG>
__global__ void __launch_bounds__(W * 32, 1) k_sv(SvParams sp) {
  constexpr int E = Vec<T>::E;
  extern __shared__ __align__(128) uint8_t smem_raw[];
  SvSmem<W, NSTG>& S = *reinterpret_cast<SvSmem<W, NSTG>*>(smem_raw);
  const RowsParams& p = sp.r;
  const Dims& d = p.d;
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  const int NC = gridDim.x, NWT = NC * W;  // warps in the grid
  const int gw = blockIdx.x + NC * w;      // this warp's rank (CTA-major spread)
  const T* PLt = static_cast<const T*>(p.PL);
  const T* QLt = static_cast<const T*>(p.QL);
  const uint32_t row_bytes = (uint32_t)d.V * sizeof(T);
  const int nvec = (int)(row_bytes / 16);
  const int nseg = (int)((row_bytes + kSegBytes - 1) / kSegBytes);
  const int G = d.G;
  int bar = 0;
  if (tid == 0) SB_TRACE_AT(sb_trace_sv, 0, 0);
  pdl_wait();
  if (tid == 0) SB_TRACE_AT(sb_trace_sv, 0, 1);

  if (sp.adaptive) {
    // ---------------- C: confidence rows
    SvSub sc;
    sc.rows = d.B * G; sc.nsl = sp.nsl_c; sc.units = (sc.rows * sc.nsl + 31) / 32 * 32;
    sc.kind = 0; sc.pbase = 0; sc.S = ((nvec + sc.nsl - 1) / sc.nsl + 2 * kSvCV - 1) / (2 * kSvCV);
    sv_stream<T, W, NSTG>(sp, S, &sc, 1, nvec);
    if (lane == 0) SB_TRACE_AT(sb_trace_sv, 1, w);
    sv_grid_sync(sp.ctr, ++bar);
    // ---------------- combine C: statistic, Eq. 6 / 7 per (b, i); gamma_b by the last row of b
    for (int r = gw; r < sc.rows; r += NWT) {
      const int b = r / G, i = r % G;
      RowStat qs = sv_fold(sp.part_q + (int64_t)r * sc.nsl, sc.nsl);
      conf_epilogue(sp.c, b, i, QLt + row_off(d, b, 0, i), qs, lane, &S.s_last[w], [] { __syncwarp(); });
    }
    sv_grid_sync(sp.ctr, ++bar);
  }

  // ---------------- plan: every CTA lays out every sequence (k_plan's clamps and order)
  if (w == 0) {
    int runA = 0, runB = 0;
    for (int b0 = 0; b0 < d.B; b0 += 32) {
      const int b = b0 + lane;
      int nA = 0, nB = 0;
      if (b < d.B) {
        const int g = sp.adaptive ? __ldcg(sp.c.gamma_next + b) : (sp.gamma_in ? __ldg(sp.gamma_in + b) : G);
        const SeqInfo in = astep_seqinfo(g, sp.bpos ? __ldg(sp.bpos + b) : 0, G);
        S.pk[b] = sv_pack(in);
        if (blockIdx.x == 0) const_cast<SeqInfo*>(p.info)[b] = in;
        const int count = in.Lr + (d.K - 1) * (in.Lr - 1 - in.s);
        nA = sp.adaptive ? min(in.Lr, G) : 0;  // slot-0 rows whose q state the confidence pass left
        nB = count - nA;
      }
      int ia = nA, ib = nB;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int ya = __shfl_up_sync(0xffffffffu, ia, o), yb = __shfl_up_sync(0xffffffffu, ib, o);
        if (lane >= o) { ia += ya; ib += yb; }
      }
      if (b < d.B) { S.offA[b] = runA + ia - nA; S.offB[b] = runB + ib - nB; }
      runA += __shfl_sync(0xffffffffu, ia, 31);
      runB += __shfl_sync(0xffffffffu, ib, 31);
    }
    if (lane == 0) {
      S.offA[d.B] = runA;
      S.offB[d.B] = runB;
      // slices: a p-only row's slice twice as long as a pair's (equal bytes per lane),
      // every lane one unit (padding to whole warps included)
      const int lanes = NWT * 32 - 64;
      const int maxs = max(1, min(kSvMaxSl, nvec / kSvMinV));
      int nb = max(1, min(maxs, (int)((int64_t)lanes * 2 / max(1, runA + 2 * runB))));
      int na = max(1, min(maxs, nb / 2));
      while (nb > 1 && (int64_t)runA * na + (int64_t)runB * nb > lanes) {
        --nb;
        na = max(1, min(maxs, nb / 2));
      }
      S.geo[0] = runA; S.geo[1] = runB; S.geo[2] = na; S.geo[3] = nb;
    }
  }
  __syncthreads();

  // ---------------- V: every tested row pair
  SvSub sv[2];
  sv[0].rows = S.geo[0]; sv[0].nsl = S.geo[2]; sv[0].units = (sv[0].rows * sv[0].nsl + 31) / 32 * 32;
  sv[0].kind = 1; sv[0].pbase = 0; sv[0].S = ((nvec + sv[0].nsl - 1) / sv[0].nsl + 2 * kSvCV - 1) / (2 * kSvCV);
  sv[1].rows = S.geo[1]; sv[1].nsl = S.geo[3]; sv[1].units = (sv[1].rows * sv[1].nsl + 31) / 32 * 32;
  sv[1].kind = 2; sv[1].pbase = sv[0].units; sv[1].S = ((nvec + sv[1].nsl - 1) / sv[1].nsl + kSvCV - 1) / kSvCV;
  sv_stream<T, W, NSTG>(sp, S, sv, 2, nvec);
  if (lane == 0) SB_TRACE_AT(sb_trace_sv, 2, w);
  sv_grid_sync(sp.ctr, ++bar);

  // ---------------- combine V: row outputs, token tests, n_k, the sample decision
  {
    const int nrows = sv[0].rows + sv[1].rows;
    for (int t = gw; t < nrows; t += NWT) {
      const int kind = t < sv[0].rows ? 1 : 2;
      const int r = kind == 1 ? t : t - sv[0].rows;
      const SvSub& su = sv[kind - 1];
      Unit un;
      sv_row(S, d, kind, r, un.b, un.slot, un.i);
      un.in = sv_unpack(S.pk[un.b]);
      const T* prow = PLt + row_off(d, un.b, un.slot, un.i);
      const T* qrow = QLt + row_off(d, un.b, un.slot, un.i);
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
      const bool tr = (t == gw) && lane == 0;
      if (tr) SB_TRACE_AT(sb_trace_sv, 3, 4 * w);
      const int64_t rec = su.pbase + (int64_t)r * su.nsl;
      const RowStat ps = sv_fold(sp.part_p + rec, su.nsl);
      const RowStat qs = (kind == 1) ? ldcg_rowstat(p.qreuse + (int64_t)un.b * G + un.i) : sv_fold(sp.part_q + rec, su.nsl);
      if (tr) SB_TRACE_AT(sb_trace_sv, 3, 4 * w + 1);
      int nk = 0;
      if (warp_epilogue<T>(p, un, ps, qs, qrow, x, lpx, lqx, uu, et, &nk)) {
        if (tr) SB_TRACE_AT(sb_trace_sv, 3, 4 * w + 2);
        __threadfence();
        const SvDesc ds = sv_decide<T>(sp, un.b, un.in, nk);
        if (lane == 0) sp.desc[un.b] = ds;
        if (tr) SB_TRACE_AT(sb_trace_sv, 3, 4 * w + 3);
      } else if (tr) {
        SB_TRACE_AT(sb_trace_sv, 3, 4 * w + 2);
      }
    }
  }
  sv_grid_sync(sp.ctr, ++bar);

  // ---------------- S: segment sums of every sampled row: wps warps per sequence, each a
  // contiguous range of segments, 4 segments' loads in flight per lane
  {
    const int wps = max(1, min(nseg, NWT / d.B));
    for (int t = gw; t < d.B * wps; t += NWT) {
      const int b = t / wps, part = t % wps;
      const int s0 = (int)((int64_t)part * nseg / wps), s1 = (int)((int64_t)(part + 1) * nseg / wps);
      const int4 h = __ldcg(reinterpret_cast<const int4*>(sp.desc + b));  // kind, slot, i, ksel
      if (h.x == 0) continue;
      const float4 rs = __ldcg(&sp.desc[b].rs);
      const T* prow = PLt + row_off(d, b, h.y, h.z);
      const T* qrow = QLt + row_off(d, b, h.y, h.z);
      const bool resid = h.x == 1;
      const bool ok = !resid || (z_class(rs.y) | z_class(rs.w)) == 0;
      for (int sb0 = s0; sb0 < s1; sb0 += 4) {
        uint4 vp[4][2], vq[4][2];
#pragma unroll
        for (int k = 0; k < 4; ++k)
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            const uint32_t off = (uint32_t)(sb0 + k) * kSegBytes + lane * 32 + j * 16;
            const bool in = sb0 + k < s1;
            vp[k][j] = in ? seg_vec(prow, row_bytes, off) : neg_inf_vec<T>();
            vq[k][j] = (in && resid) ? seg_vec(qrow, row_bytes, off) : neg_inf_vec<T>();
          }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          if (sb0 + k >= s1) break;
          const int sI = sb0 + k;
          float own = 0.f;
          if (resid) {  // the k_select_tma consumers' arithmetic
#pragma unroll
            for (int j = 0; j < 2; ++j) {
              float r[E];
              r_scaled<T>(vp[k][j], vq[k][j], true, rs.x, rs.z, rs.y / rs.w, r);
              own = seq_sum<E>(r, own);
            }
            const float tot = warp_sum_rn(ok ? own : 0.f);
            if (lane == 0) sp.seg[(int64_t)b * nseg + sI] = tot;
          } else {  // bonus: the segment's own offset (its maximum), rescaled when located
            float m = -CUDART_INF_F;
#pragma unroll
            for (int j = 0; j < 2; ++j) {
              float f[E];
              Vec<T>::unpack(vp[k][j], f);
              m = fmaxf(m, Vec<T>::vmax(f));
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
            const float ms = offset_of(m);
#pragma unroll
            for (int j = 0; j < 2; ++j) {
              float r[E];
              r_scaled<T>(vp[k][j], vp[k][j], false, ms, 0.f, 0.f, r);
              own = seq_sum<E>(r, own);
            }
            const float tot = warp_sum_rn(own);
            if (lane == 0) {
              sp.seg[(int64_t)b * nseg + sI] = tot;
              sp.segm[(int64_t)b * nseg + sI] = m;
            }
          }
        }
      }
    }
  }
  sv_grid_sync(sp.ctr, ++bar);

  // ---------------- locate, commit; offsets by the last committer
  {
    float* scratch = reinterpret_cast<float*>(&S.ring[w][0][0][0]);  // the ring is idle now
    static_assert(sizeof(S.ring[0]) >= 1024 * sizeof(float), "segment scratch (nseg <= 1024)");
    for (int b = gw; b < d.B; b += NWT) {
      if (b == gw && lane == 0) SB_TRACE_AT(sb_trace_sv, 4, 4 * w);
#ifdef SB_TRACE
      if (b == 0 && lane == 0) {  // latency probes: 16 dependent L2 loads, 16 dependent HBM loads, clock rate
        unsigned long long c0 = clock64();
        SB_TRACE_AT(sb_trace_sv, 5, 0);
        int v = 0;
        for (int k = 0; k < 16; ++k) v = __ldcg(sp.ctr + 3 + (v == 123456789));
        SB_TRACE_AT(sb_trace_sv, 5, 1);
        const int* pr = reinterpret_cast<const int*>(p.PL);
        for (int k = 0; k < 16; ++k) v += __ldcg(pr + (int64_t)k * 32768 + 7 + (v == 123456789));
        SB_TRACE_AT(sb_trace_sv, 5, 2);
        unsigned long long c1 = clock64();
        sb_trace_sv[0][5][3] = c1 - c0;
        sb_trace_sv[0][5][4] = (unsigned long long)v;
      }
#endif
      SvDesc ds;  // written by other CTAs: through L2
      {
        const int4* src = reinterpret_cast<const int4*>(sp.desc + b);
        int4 v[3] = {__ldcg(src), __ldcg(src + 1), __ldcg(src + 2)};
        memcpy(&ds, v, sizeof(ds));
      }
      const SeqInfo in = sv_unpack(S.pk[b]);
      int kind = ds.kind, y = -1, st = 0;
      double mass = 0.0;
      if (kind == 1) {
        const int cls = z_class(ds.rs.y) | z_class(ds.rs.w);
        if (cls) {
          kind = 0;
          st |= cls;
        } else {
          for (int j = lane; j < nseg; j += 32) scratch[j] = __ldcg(sp.seg + (int64_t)b * nseg + j);
          __syncwarp();
          bool resid = true;
          double R = 0.0;
          const T* prow = PLt + row_off(d, b, ds.slot, ds.i);
          const T* qrow = QLt + row_off(d, b, ds.slot, ds.i);
          y = sample_segments<T>(prow, qrow, row_bytes, d.V, scratch, nseg, resid, ds.rs.x, ds.rs.z,
                                 ds.rs.y / ds.rs.w, __ldg(sp.us + b), st, &R);
          mass = R / (double)ds.rs.y;
        }
      } else if (kind == 2) {
        float mrow = -CUDART_INF_F;
        for (int j = lane; j < nseg; j += 32) mrow = fmaxf(mrow, __ldcg(sp.segm + (int64_t)b * nseg + j));
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) mrow = fmaxf(mrow, __shfl_xor_sync(0xffffffffu, mrow, o));
        const float MS = offset_of(mrow);
        double z = 0.0;
        for (int j = lane; j < nseg; j += 32) {
          const float mj = __ldcg(sp.segm + (int64_t)b * nseg + j);
          const double sc = exp2((double)offset_of(mj) - (double)MS);
          const float v = (float)((double)__ldcg(sp.seg + (int64_t)b * nseg + j) * sc);
          scratch[j] = v;
          z += (double)v;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) z += __shfl_xor_sync(0xffffffffu, z, o);
        __syncwarp();
        const int cls = row_class(mrow, z);
        if (cls) {
          kind = 0;
          st |= cls;
        } else {
          bool resid = false;
          double R = 0.0;
          const T* prow = PLt + row_off(d, b, ds.slot, ds.i);
          y = sample_segments<T>(prow, prow, row_bytes, d.V, scratch, nseg, resid, MS, 0.f, 0.f,
                                 __ldg(sp.us + b), st, &R);
          mass = R / z;
        }
      }
      if (b == gw && lane == 0) SB_TRACE_AT(sb_trace_sv, 4, 4 * w + 1);
      commit_seq(p, sp.co, b, in, ds.ksel, ds.npath, kind, y, mass, st);
      if (b == gw && lane == 0) SB_TRACE_AT(sb_trace_sv, 4, 4 * w + 2);
      __syncwarp();
      int last = 0;
      if (lane == 0) {
        __threadfence();
        last = (atomicAdd(sp.ctr + 2, 1) == d.B - 1);
      }
      last = __shfl_sync(0xffffffffu, last, 0);
      if (last) {
        __threadfence();
        sv_offsets(d.B, G, sp.co.commit_len, sp.co.out_tok, sp.co.offsets, sp.co.packed_tok,
                   reinterpret_cast<int*>(scratch));
        if (lane == 0) sp.ctr[2] = 0;
        if (lane == 0) SB_TRACE_AT(sb_trace_sv, 4, 4 * w + 3);
      }
      __syncwarp();
    }
  }
  // ---------------- exit: the last CTA out resets the barrier
  __syncthreads();
  if (tid == 0) SB_TRACE_AT(sb_trace_sv, 0, 40);
  if (tid == 0) {
    __threadfence();
    if (atomicAdd(sp.ctr + 1, 1) == NC - 1) {
      sp.ctr[0] = 0;
      sp.ctr[1] = 0;
    }
  }
}

#ifndef SB_SV_W
#define SB_SV_W 16
#endif
#ifndef SB_SV_NSTG
#define SB_SV_NSTG 3
#endif
constexpr int kSvW = SB_SV_W, kSvNS = SB_SV_NSTG;

template <typename T>
static sb_status launch_sv(const SvParams& sp, cudaStream_t s) {
  const int smem = (int)sizeof(SvSmem<kSvW, kSvNS>);
  if (ensure_smem<k_sv<T, kSvW, kSvNS>>(smem) != cudaSuccess) return SB_ERR_CUDA;
  int occ = 0;  // every CTA must be resident (grid barriers)
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_sv<T, kSvW, kSvNS>, kSvW * 32, smem);
  if (occ < 1) return SB_ERR_UNSUPPORTED;
  return cuda_status(launch_pdl(k_sv<T, kSvW, kSvNS>, dim3(num_sms()), dim3(kSvW * 32), smem, s, sp));
}

// The small-batch path applies: 16-byte aligned unsharded rows of 16-byte multiples up to
// 1 MB, B <= 512, B K (G+1) <= 4096 (the problems where whole-row items leave the GPU
// latency-bound: C2, one C1 round).  SB_SV=0 turns it off.
bool sv_eligible(const sb_dims* dd, const void* PL, const void* QL) {
  const char* e = getenv("SB_SV");
  if (!(e && e[0] == '1')) return false;  // opt-in: measured slower than k_astep
  if (tma_disabled() || sharded(dd)) return false;
  if (!vec_ok(dd, PL) || !vec_ok(dd, QL)) return false;
  const size_t rb = (size_t)dd->V * elem_size(dd);
  if (rb % 16 || rb > (size_t)1024 * kSegBytes) return false;
  if (dd->B > kSvMaxB || (size_t)dd->B * dd->K * (dd->G + 1) > (size_t)kSvPartRowsMax) return false;
  return num_sms() * kSvW * 32 + 64 <= kSvPartCap;  // one partial record per lane (sb_host.h)
}

sb_status sv_run(const sb_dims* dd, const Workspace& w, const Workspace* cw, const void* PL, const void* QL,
                 const int32_t* tok, const float* u, const float* us, const int32_t* gamma, const int32_t* branch_pos,
                 sb_select_rule rule, float eps, int32_t k_max, float* c_top1, int32_t* c_id, float* c_ent,
                 float* c_stat, int32_t* c_stop, int32_t* c_knext, int32_t* c_gamma, float* lse_p, float* lse_q,
                 float* p_tok, float* q_tok, uint32_t* acc_mask, int32_t* n_acc, float* top1_q, int32_t* top1_id_q,
                 float* entropy_q, int32_t* status, const CommitOut& co, cudaStream_t s) {
  const Dims d = to_dims(dd);
  SvParams sp{};
  RowsParams& p = sp.r;
  p.d = d; p.PL = PL; p.QL = QL; p.tok = tok; p.u = u;
  p.info = w.info; p.unit_off = w.unit_off; p.seqpk = w.seqpk; p.cnt = w.cnt; p.rowstat = w.rowstat;
  p.pflag = w.pflag;
  p.lse_p = lse_p; p.lse_q = lse_q; p.p_tok = p_tok; p.q_tok = q_tok;
  p.top1_q = top1_q; p.entropy_q = entropy_q; p.top1_id_q = top1_id_q;
  p.acc_mask = acc_mask; p.n_acc = n_acc; p.status = status;
  const int nvec = (int)((size_t)dd->V * elem_size(dd) / 16);
  const int lanes = num_sms() * kSvW * 32 - 32;
  if (cw) {
    p.qreuse = cw->qrs;
    ConfParams& c = sp.c;
    c.d = d;
    c.d.K = 1;  // slot-0 view of the draft rows
    c.QL = QL; c.tok = nullptr; c.mode = SB_CONF_TOP1; c.eps = eps; c.lambda = 1.f; c.k_max = k_max;
    c.top1_prob = c_top1; c.entropy = c_ent; c.tok_prob = nullptr; c.stat = c_stat; c.top1_id = c_id;
    c.stop = c_stop; c.k_next = c_knext; c.gamma_next = c_gamma;
    c.cnt = cw->conf_cnt; c.ws_stat = cw->conf_stat; c.ws_c = cw->conf_c; c.qrs = cw->qrs;
    const int rows = dd->B * dd->G;
    sp.nsl_c = std::max(1, std::min(std::min(kSvMaxSl, std::max(1, nvec / kSvMinV)), lanes / rows));
  }
  sp.co = co;
  sp.us = us; sp.bpos = branch_pos; sp.gamma_in = gamma;
  sp.adaptive = cw != nullptr;
  sp.rule = rule;
  sp.part_p = w.sv_part_p; sp.part_q = w.sv_part_q;
  sp.desc = reinterpret_cast<SvDesc*>(w.sv_desc);
  sp.seg = w.sv_seg; sp.segm = w.sv_segm; sp.ctr = w.sv_ctr;
  return dd->dtype == SB_BF16 ? launch_sv<__nv_bfloat16>(sp, s) : launch_sv<float>(sp, s);
}

}  // namespace sb
