// sb_tree.cu — sb_tree_verify: token-tree verification (the dense tree
// structure of Appendix F, P1057/P1073, that SpecBranch's sparse branches are compared
// against), read as Eq. 9 applied at every node (R31):
//   acc(j) = u_j Q_r[x_j] <= P_r[x_j] at the parent's context row r = parent[j] + 1 (P94),
//   walk from the root to the accepted child of largest raw target logit (P236-241),
//   y from the stop node's row: residual norm(max(0, p - q)) if it has children, else
//   the bonus p (P94, P554).
//
// Two launches:
//   k_tree_rows    one CTA per (sequence, context row); rows with no child exit at once
//                  (their q is never read, their p only if the walk ends there), the rest
//                  stream the (p, q) pair once -> softmax state (MS, Z) of both.
//   k_tree_select  one CTA per sequence: every node's test in fp64 from the states (one
//                  thread per node), the walk (thread 0), then the block sampler on the
//                  stop row (a leaf's p row first gets its own softmax pass).
#include "sb_block_sample.cuh"
#include "sb_host.h"

namespace sb {

constexpr int kTreeMaxN = 63;

struct TreeParams {
  Dims d;  // K = 1, G = N: rows [B][N+1]
  const void* PL;
  const void* QL;
  const int* parent;
  const int* tok;
  const float* u;
  const float* us;
  float4* rowstat;  // [B][N+1] (MS_p, Z_p, MS_q, Z_q); NaN Z for a non-finite row
  unsigned long long *acc_mask, *keep_mask;
  int *stop_node, *commit_len, *out_tok, *y_tok, *y_kind, *status;
  float* resid_mass;
};

template <typename T, int NT, int U>
__global__ void __launch_bounds__(NT) k_tree_rows(TreeParams p, bool vec_ok) {
  __shared__ RowStat red[NT / 32];
  const Dims& d = p.d;
  const int N = d.G, R1 = N + 1;
  const int b = blockIdx.x / R1, r = blockIdx.x % R1, lane = threadIdx.x & 31;
  // every warp decides alike whether context row r has a child (parent == r - 1)
  bool has = false;
  for (int j = lane; j < N; j += 32) has |= (__ldg(p.parent + (int64_t)b * N + j) == r - 1) && (r - 1 < j);
  if (!__any_sync(0xffffffffu, has)) return;
  const T* prow = static_cast<const T*>(p.PL) + row_off(d, b, 0, r);
  const T* qrow = static_cast<const T*>(p.QL) + row_off(d, b, 0, r);
  RowStat sp, sq;
  if (vec_ok && sizeof(T) == 2) {  // lazy-offset packed bf16 path (as the verify kernels)
    LazyAcc<false, 4> pa, qa;
    pa.init();
    qa.init();
    constexpr int E = Vec<T>::E;
    const int nvec = d.V / E;
    const uint4* pv = reinterpret_cast<const uint4*>(prow);
    const uint4* qv = reinterpret_cast<const uint4*>(qrow);
    const int nround = (nvec + U * NT - 1) / (U * NT) * (U * NT);
    for (int vb = threadIdx.x; vb < nround; vb += U * NT) {  // block-uniform trip count
      uint4 xp[U], xq[U];
#pragma unroll
      for (int j = 0; j < U; ++j) {
        const bool in = vb + j * NT < nvec;
        xp[j] = in ? ldg_stream(pv + vb + j * NT) : neg_inf_vec<T>();
        xq[j] = in ? ldg_stream(qv + vb + j * NT) : neg_inf_vec<T>();
      }
#pragma unroll
      for (int j = 0; j + 1 < U; j += 2) {
        acc_vecs_bf16<2>(pa, xp + j, 0);
        acc_vecs_bf16<2>(qa, xq + j, 0);
      }
    }
    RowAcc<false, 4> pt, qt;  // the V % 8 tail, exact-offset state, merged below
    pt.init();
    qt.init();
    for (int v = nvec * E + threadIdx.x; v < d.V; v += NT) {
      pt.add1(ld_scalar(prow + v), v);
      qt.add1(ld_scalar(qrow + v), v);
    }
    sp = block_reduce<NT>(combine(fold_lazy(pa), fold(pt)), red);
    sq = block_reduce<NT>(combine(fold_lazy(qa), fold(qt)), red);
  } else {
    RowAcc<false, 4> pa, qa;
    pa.init();
    qa.init();
    stream_pair<T, 4, NT, U, false>(prow, qrow, d.V, vec_ok, pa, qa);
    sp = block_reduce<NT>(fold(pa), red);
    sq = block_reduce<NT>(fold(qa), red);
  }
  if (threadIdx.x == 0) {
    const RowOut op = finish(sp), oq = finish(sq);
    p.rowstat[(int64_t)b * R1 + r] = make_float4(op.MS, z_store(op), oq.MS, z_store(oq));
  }
}

template <typename T, int NT>
__global__ void __launch_bounds__(NT) k_tree_select(TreeParams p, bool vec_ok) {
  constexpr int NW = NT / 32;
  __shared__ SampleSmem<NW> sm;
  __shared__ int spar[kTreeMaxN + 1], stok[kTreeMaxN + 1], path[kTreeMaxN + 1];
  __shared__ float skey[kTreeMaxN + 1];
  __shared__ unsigned sacc[2];
  __shared__ int sh_st, sh_stop, sh_kind, sh_npath;
  const Dims& d = p.d;
  const int N = d.G, R1 = N + 1;
  const int b = blockIdx.x, tid = threadIdx.x;
  const T* PL = static_cast<const T*>(p.PL);
  const T* QL = static_cast<const T*>(p.QL);
  if (tid == 0) { sh_st = 0; sacc[0] = sacc[1] = 0u; }
  __syncthreads();
  // the Match test of every node against its parent's context row (P94, P538)
  if (tid < 64) {
    const int j = tid;
    bool acc = false;
    int st = 0, pj = -3, x = -1;
    float key = -CUDART_INF_F;
    if (j < N) {
      pj = __ldg(p.parent + (int64_t)b * N + j);
      x = __ldg(p.tok + (int64_t)b * N + j);
      if (pj < -1 || pj >= j) {
        st |= SB_ST_BAD_PARENT;
        pj = -3;  // never anybody's child
      } else {
        const float4 rs = p.rowstat[(int64_t)b * R1 + pj + 1];
        const int cls = z_class(rs.y) | z_class(rs.w);
        if (cls) {
          st |= cls;
        } else if (x < 0 || x >= d.V) {
          st |= SB_ST_BAD_TOKEN;
        } else {
          const int64_t ro = row_off(d, b, 0, pj + 1);
          key = ld_scalar(PL + ro + x);
          const double P = tok_prob(key, rs.x, rs.y), Q = tok_prob(ld_scalar(QL + ro + x), rs.z, rs.w);
          acc = (double)__ldg(p.u + (int64_t)b * N + j) * Q <= P;  // Q = 0 accepts (S127)
        }
      }
      spar[j] = pj;
      stok[j] = x;
      skey[j] = key;
    }
    const unsigned m = __ballot_sync(0xffffffffu, acc);
    if ((tid & 31) == 0) sacc[tid >> 5] = m;
    if (st) atomicOr(&sh_st, st);
  }
  __syncthreads();
  const unsigned long long acc = (unsigned long long)sacc[0] | ((unsigned long long)sacc[1] << 32);
  if (tid == 0) {
    // the walk: Eq. 9 at every node (raw target logit; ties -> smaller token, smaller j)
    int c = -1, npath = 0, has_child;
    for (;;) {
      int best = -1;
      has_child = 0;
      for (int j = 0; j < N; ++j) {
        if (spar[j] != c) continue;
        has_child = 1;
        if (!((acc >> j) & 1ull)) continue;
        if (best < 0 || skey[j] > skey[best] || (skey[j] == skey[best] && stok[j] < stok[best])) best = j;
      }
      if (best < 0) break;
      path[npath++] = best;
      c = best;
    }
    sh_stop = c;
    sh_npath = npath;
    sh_kind = has_child ? 1 : 2;
  }
  __syncthreads();
  const int c = sh_stop, npath = sh_npath;
  int kind = sh_kind;
  int y = -1;
  double mass = 0.0;
  {
    Sampler<T, NT> smp;
    smp.prow = PL + row_off(d, b, 0, c + 1);
    smp.qrow = QL + row_off(d, b, 0, c + 1);
    smp.V = d.V;
    smp.vec_ok = vec_ok;
    float MSp, Zp, MSq = 0.f, Zq = 1.f;
    int cls;
    if (kind == 2) {  // a leaf's p row: never streamed by k_tree_rows
      float m;
      const RowOut o = block_row_stats<T, NT>(smp.prow, d.V, vec_ok, sm.red, &m);
      MSp = o.MS; Zp = (float)o.Z; cls = o.st;
    } else {
      const float4 rs = p.rowstat[(int64_t)b * R1 + c + 1];
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
  __syncthreads();
  int* out = p.out_tok + (int64_t)b * R1;
  for (int q = tid; q < R1; q += NT) out[q] = q < npath ? stok[path[q]] : (q == npath && kind != 0 ? y : -1);
  if (tid == 0) {
    unsigned long long keep = 0;
    for (int q = 0; q < npath; ++q) keep |= 1ull << path[q];
    p.acc_mask[b] = acc;
    p.keep_mask[b] = keep;
    p.stop_node[b] = c;
    p.commit_len[b] = npath + (kind != 0);
    p.y_tok[b] = kind != 0 ? y : -1;
    p.y_kind[b] = kind;
    if (p.resid_mass) p.resid_mass[b] = kind != 0 ? (float)mass : 0.f;
    p.status[b] = sh_st;
  }
}

static bool tree_dims_valid(const sb_dims* d) {
  if (!d || d->B < 1 || d->K != 1 || d->G < 1 || d->G > kTreeMaxN || d->V < 2 || d->row_stride < d->V) return false;
  if (d->dtype != SB_BF16 && d->dtype != SB_F32) return false;
  if (d->v_offset != 0 || (d->v_total != 0 && d->v_total != d->V) || d->reserved != 0) return false;
  return d->seq_stride == 0 || d->seq_stride >= (int64_t)(d->G + 1) * d->row_stride;
}

template <typename T>
static sb_status launch_tree(const TreeParams& p, bool vok, cudaStream_t s) {
  // 128-thread CTAs, 4 vectors in flight per thread (measured on 256 dense 30-node
  // trees, V = 32000: 256 threads 0.135 ms, 128 threads 0.119 ms, 64 threads 0.125 ms)
  k_tree_rows<T, 128, 4><<<p.d.B * (p.d.G + 1), 128, 0, s>>>(p, vok);
  k_tree_select<T, 256><<<p.d.B, 256, 0, s>>>(p, vok);
  return cuda_status(cudaGetLastError());
}

}  // namespace sb

using namespace sb;

extern "C" size_t sb_tree_workspace_bytes(const sb_dims* d) {
  if (!tree_dims_valid(d)) return 0;
  return align256((size_t)d->B * (d->G + 1) * sizeof(float4));
}

extern "C" sb_status sb_tree_verify(const sb_dims* dd, const void* p_logits, const void* q_logits,
                                    const int32_t* parent, const int32_t* tok, const float* u, const float* us,
                                    uint64_t* acc_mask, uint64_t* keep_mask, int32_t* stop_node,
                                    int32_t* commit_len, int32_t* out_tok, int32_t* y_tok, int32_t* y_kind,
                                    float* resid_mass, int32_t* status, void* workspace, size_t workspace_bytes,
                                    sb_stream_t stream) {
  SB_NVTX("sb_tree_verify");
  if (!tree_dims_valid(dd) || !p_logits || !q_logits || !parent || !tok || !u || !us || !acc_mask || !keep_mask ||
      !stop_node || !commit_len || !out_tok || !y_tok || !y_kind || !status || !workspace)
    return SB_ERR_INVALID_ARG;
  if ((uintptr_t)workspace % 16) return SB_ERR_INVALID_ARG;
  if (workspace_bytes < sb_tree_workspace_bytes(dd)) return SB_ERR_WORKSPACE;
  if (dd->dtype == SB_BF16 ? (dd->V + 256 * 8 - 1) / (256 * 8) > kMaxTiles
                           : (dd->V + 256 * 4 - 1) / (256 * 4) > kMaxTiles)
    return SB_ERR_UNSUPPORTED;
  TreeParams p;
  p.d = to_dims(dd); p.PL = p_logits; p.QL = q_logits; p.parent = parent; p.tok = tok; p.u = u; p.us = us;
  p.rowstat = static_cast<float4*>(workspace);
  p.acc_mask = reinterpret_cast<unsigned long long*>(acc_mask);
  p.keep_mask = reinterpret_cast<unsigned long long*>(keep_mask);
  p.stop_node = stop_node; p.commit_len = commit_len; p.out_tok = out_tok; p.y_tok = y_tok; p.y_kind = y_kind;
  p.resid_mass = resid_mass; p.status = status;
  const bool vok = vec_ok(dd, p_logits) && vec_ok(dd, q_logits);
  cudaStream_t s = (cudaStream_t)stream;
  return dd->dtype == SB_BF16 ? launch_tree<__nv_bfloat16>(p, vok, s) : launch_tree<float>(p, vok, s);
}
