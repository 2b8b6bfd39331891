// sb_confidence.cu — sb_draft_confidence: the implicit draft-confidence statistic
// (§4.2 P170: max_x q(x) or 1 - sqrt(lambda H); App. E.6 P954/P965), the Eq. 6 stop
// (keep q(x) > eps, P198; Alg. 1 "Mask" P517) and Eq. 7's adaptive branch count
// k = max(1, floor(k_max (1 - q(x_b)))) at the stop row (P218).  SURVEY §8.1 row a6.
//
// One unit = one q row; persistent CTAs stream it once (same online state as the
// verify kernel), write the per-row statistics; the CTA finishing a (b,k) group takes
// the first row whose statistic is <= eps (ballot/ffs over <= 31 rows).
#include <algorithm>

#include "sb_host.h"
#include "sb_ring.cuh"
#include "sb_conf.cuh"
#include "sb_stream.cuh"

#ifdef SB_TRACE
SB_TRACE_TABLE(sb_trace_conf)
#endif

namespace sb {

// Register-staged fallback (any alignment / stride).
template <typename T, int NT, int U>
__global__ void __launch_bounds__(NT) k_conf(ConfParams p, bool vec_ok) {
  constexpr int NA = 4;
  __shared__ RowStat red[NT / 32];
  __shared__ int s_last;
  const Dims& d = p.d;
  const int tid = threadIdx.x, G = d.G;
  const int total = d.B * d.K * G;
  const T* QL = static_cast<const T*>(p.QL);
  for (int unit = blockIdx.x; unit < total; unit += gridDim.x) {
    const int grp = unit / G, i = unit % G;
    const int b = grp / d.K, k = grp % d.K;
    const T* row = QL + row_off(d, b, k, i);
    RowAcc<true, NA> a;
    a.init();
    stream_row<T, true, NA, NT, U>(row, d.V, vec_ok, a);
    const RowStat s = block_reduce<NT>(fold(a), red);
    conf_epilogue(p, grp, i, row, s, tid, &s_last, [] { __syncthreads(); });
  }
}

// TMA ring version (same warp roles as k_rows_tma): the producer warp streams cChunk-byte
// chunks of each q row, cCW consumer warps fold them, cNE epilogue warps finish the rows.
// 28 consumer warps x 7 stages of 28 KB, 2 epilogue warps (same box, C3's 4096 draft rows:
// 0.1995-0.2001 ms against 0.2162-0.2176 ms for 16 x 12 x 16 KB with 4 epilogue warps;
// 20 x 10: 0.210, 24 x 8: 0.208, 24 x 8 / 2: 0.206, 26 x 7: 0.212, 28 x 7 / 1: 0.204,
// 30 x 7 / 1: 0.217, 12 x 16: 0.237)
#ifndef SB_CONF_NS
#define SB_CONF_NS 7
#endif
#ifndef SB_CONF_CW
#define SB_CONF_CW 28
#endif
#ifndef SB_CONF_NE
#define SB_CONF_NE 2
#endif
constexpr int cNS = SB_CONF_NS;  // (macros: A/B experiment builds only)
constexpr int cCW = SB_CONF_CW;
constexpr int cCT = cCW * 32;
constexpr int cVPT = 2;
constexpr int cChunk = cCT * cVPT * 16;
constexpr int cNP = 4;
constexpr int cNE = SB_CONF_NE;  // epilogue warps, alternating units
constexpr int cThreads = cCT + 32 * (1 + cNE);
using ConfGeo = RC<cCW, cNS, cVPT, cNP>;  // ring geometry (resolve_argmax)

struct ConfSmem {
  uint64_t full[cNS], empty[cNS];
  uint64_t pfull[cNP], pempty[cNP];
  RowStat part[cNP][cCW];
  uint2 cand[cNP][cCW];
  int s_last[cNE];
  alignas(128) uint8_t buf[cNS][cChunk];
};

// One chunk of a q row into the accumulator; first: the row's first chunk (the peeled
// rescale test of LazyAcc, warp-uniform).
template <typename T>
__device__ __forceinline__ void conf_acc(LazyAcc<true, 4>& a, const uint4* x, int c, bool first) {
  constexpr int E = Vec<T>::E;
  if constexpr (sizeof(T) == 2) {
    if (first) acc_vecs_bf16<cVPT, true, true>(a, x, c);
    else acc_vecs_bf16<cVPT, true, false>(a, x, c);
  } else {
    float f[cVPT * E];
#pragma unroll
    for (int j = 0; j < cVPT; ++j) Vec<T>::unpack(x[j], f + j * E);
    if (first) a.template add<cVPT * E, true>(f, c);
    else a.template add<cVPT * E, false>(f, c);
  }
}

template <typename T>
__global__ void __launch_bounds__(cThreads, 1) k_conf_tma(ConfParams p) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  ConfSmem& S = *reinterpret_cast<ConfSmem*>(smem_raw);
  const Dims& d = p.d;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, G = d.G;
  if (tid == 0) {
    for (int s = 0; s < cNS; ++s) {
      mbar_init(&S.full[s], 1);
      mbar_init(&S.empty[s], cCW);
    }
    for (int s = 0; s < cNP; ++s) {
      mbar_init(&S.pfull[s], cCW);
      mbar_init(&S.pempty[s], 1);
    }
    fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0) SB_TRACE_AT(sb_trace_conf, 0, 0);
  pdl_wait();
  if (tid == 0) SB_TRACE_AT(sb_trace_conf, 0, 1);
  const int total = d.B * d.K * G;
  const T* QL = static_cast<const T*>(p.QL);
  const uint32_t row_bytes = (uint32_t)d.V * sizeof(T);
  const int nchunks = (row_bytes + cChunk - 1) / cChunk;
  const int nvec_last = (int)(row_bytes - (uint32_t)(nchunks - 1) * cChunk) / 16;
  if (warp == cCW) {
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      RingPos<cNS> rp;
      for (int unit = blockIdx.x; unit < total; unit += gridDim.x) {
        const int grp = unit / G, i = unit % G;
        const char* row =
            reinterpret_cast<const char*>(QL + row_off(d, grp / d.K, grp % d.K, i));
        for (int c = 0; c < nchunks; ++c) {
          const uint32_t bytes = min((uint32_t)cChunk, row_bytes - (uint32_t)c * cChunk);
          mbar_wait(&S.empty[rp.stage], rp.phase ^ 1u);
          mbar_expect_tx(&S.full[rp.stage], bytes);
          bulk_g2s(S.buf[rp.stage], row + (size_t)c * cChunk, bytes, &S.full[rp.stage], pol);
          rp.advance();
        }
      }
    }
    return;
  }
  if (warp > cCW) {  // epilogue warp e takes local units e, e + cNE, ...
    const int e = warp - cCW - 1;
    for (int li = e, unit = blockIdx.x + e * gridDim.x; unit < total; li += cNE, unit += cNE * gridDim.x) {
      const int grp = unit / G, i = unit % G;
      const int stage = li % cNP;
      mbar_wait_parked(&S.pfull[stage], (uint32_t)(li / cNP) & 1u);
      RowStat r = lane < cCW ? S.part[stage][lane] : rowstat_empty();
      const uint2 cand = lane < cCW ? S.cand[stage][lane] : make_uint2(0xffffffffu, 0u);
      __syncwarp();
      if (lane == 0) mbar_arrive(&S.pempty[stage]);
      const float mw = r.m;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) r = combine(r, shfl_xor(r, o));
      const T* row = QL + row_off(d, grp / d.K, grp % d.K, i);
      r.idx = resolve_argmax<ConfGeo, T>(mw, cand, r.m, row, nvec_last, nchunks);
      conf_epilogue(p, grp, i, row, r, lane, &S.s_last[e], [] { __syncwarp(); });
      if (lane == 0) SB_TRACE_AT(sb_trace_conf, 2, 2 + li);
    }
    if (lane == 0) SB_TRACE_AT(sb_trace_conf, 2, 63);
    return;
  }
  RingPos<cNS> rp;
  RingPos<cNP> up;
  for (int unit = blockIdx.x; unit < total; unit += gridDim.x) {
    LazyAcc<true, 4> a;
    a.init();
    for (int c = 0; c < nchunks - 1; ++c) {
      mbar_wait_spin(&S.full[rp.stage], rp.phase);
      uint4 x[cVPT];
#pragma unroll
      for (int j = 0; j < cVPT; ++j) x[j] = lds128(S.buf[rp.stage] + (tid + j * cCT) * 16);
      __syncwarp();
      if (lane == 0) mbar_arrive(&S.empty[rp.stage]);
      rp.advance();
      conf_acc<T>(a, x, c, c == 0);
    }
    {
      const int c = nchunks - 1;
      mbar_wait_spin(&S.full[rp.stage], rp.phase);
      uint4 x[cVPT];
#pragma unroll
      for (int j = 0; j < cVPT; ++j) {
        const int v = tid + j * cCT;
        x[j] = v < nvec_last ? lds128(S.buf[rp.stage] + v * 16) : neg_inf_vec<T>();
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&S.empty[rp.stage]);
      rp.advance();
      conf_acc<T>(a, x, c, nchunks == 1);
    }
    uint2 cand;
    const RowStat s = warp_part_deferred(a, cand);
    if (lane == 0) {
      mbar_wait(&S.pempty[up.stage], up.phase ^ 1u);
      S.part[up.stage][warp] = s;
      S.cand[up.stage][warp] = cand;
      mbar_arrive(&S.pfull[up.stage]);
    }
    __syncwarp();
    up.advance();
  }
}

__global__ void k_conf_empty(int n, int* stop, int* k_next, int* gamma_next) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g < n) {
    stop[g] = 0;
    if (k_next) k_next[g] = -1;
    if (gamma_next) gamma_next[g] = 1;
  }
}

template <typename T, int NT, int U>
static sb_status launch_conf(const ConfParams& p, bool vok, cudaStream_t s) {
  const int g = full_grid<k_conf<T, NT, U>>(NT);
  const int64_t units = (int64_t)p.d.B * p.d.K * p.d.G;
  const int grid = (int)std::min<int64_t>(g, units);
  k_conf<T, NT, U><<<grid, NT, 0, s>>>(p, vok);
  return cuda_status(cudaGetLastError());
}

template <typename T>
static sb_status launch_conf_tma(const ConfParams& p, cudaStream_t s) {
  const int smem = (int)sizeof(ConfSmem);
  if (ensure_smem<k_conf_tma<T>>(smem) != cudaSuccess) return SB_ERR_CUDA;
  const int64_t units = (int64_t)p.d.B * p.d.K * p.d.G;
  const int grid = (int)std::min<int64_t>(num_sms(), units);
  return cuda_status(launch_pdl(k_conf_tma<T>, dim3(grid), dim3(cThreads), smem, s, p));
}

}  // namespace sb

using namespace sb;

extern "C" sb_status sb_draft_confidence(const sb_dims* dd, const void* q_logits,
                                         const int32_t* tok, sb_conf_mode mode, float eps,
                                         float lambda, int32_t k_max, float* top1_prob,
                                         int32_t* top1_id, float* entropy, float* tok_prob,
                                         float* stat, int32_t* stop, int32_t* k_next,
                                         int32_t* gamma_next, void* comm, void* workspace,
                                         size_t workspace_bytes, sb_stream_t stream) {
  SB_NVTX("sb_draft_confidence");
  if (!dims_valid(dd) || !q_logits || !stop || !workspace) return SB_ERR_INVALID_ARG;
  if (mode != SB_CONF_TOP1 && mode != SB_CONF_TOKEN && mode != SB_CONF_ENTROPY)
    return SB_ERR_INVALID_ARG;
  if (mode == SB_CONF_TOKEN && !tok) return SB_ERR_INVALID_ARG;
  if (!(eps > 0.f && eps < 1.f) || !(lambda > 0.f) || k_max < 1) return SB_ERR_INVALID_ARG;
  if (comm || sharded(dd)) return SB_ERR_UNSUPPORTED;  // draft rows are not vocabulary-sharded
  if ((uintptr_t)workspace % 256) return SB_ERR_INVALID_ARG;
  const Workspace w = carve(*dd, workspace);
  if (workspace_bytes < w.bytes) return SB_ERR_WORKSPACE;
  cudaStream_t s = (cudaStream_t)stream;
  if (dd->G == 0) {
    const int n = dd->B * dd->K;
    k_conf_empty<<<(n + 255) / 256, 256, 0, s>>>(n, stop, k_next, gamma_next);
    return cuda_status(cudaGetLastError());
  }
  ConfParams p;
  p.d = to_dims(dd); p.QL = q_logits; p.tok = tok; p.mode = mode; p.eps = eps; p.lambda = lambda;
  p.k_max = k_max; p.top1_prob = top1_prob; p.entropy = entropy; p.tok_prob = tok_prob;
  p.stat = stat; p.top1_id = top1_id; p.stop = stop; p.k_next = k_next; p.gamma_next = gamma_next;
  p.cnt = w.conf_cnt; p.ws_stat = w.conf_stat; p.ws_c = w.conf_c; p.qrs = w.qrs;
  const bool vok = vec_ok(dd, q_logits);
  const size_t row_bytes = (size_t)dd->V * elem_size(dd);
  if (vok && row_bytes % 16 == 0 && !tma_disabled())
    return dd->dtype == SB_BF16 ? launch_conf_tma<__nv_bfloat16>(p, s) : launch_conf_tma<float>(p, s);
  if (dd->dtype == SB_BF16)
    return row_bytes <= 131072 ? launch_conf<__nv_bfloat16, 128, 4>(p, vok, s)
                               : launch_conf<__nv_bfloat16, 256, 4>(p, vok, s);
  return row_bytes <= 131072 ? launch_conf<float, 128, 4>(p, vok, s)
                             : launch_conf<float, 256, 4>(p, vok, s);
}
