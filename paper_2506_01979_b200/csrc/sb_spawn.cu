// sb_spawn.cu — sb_spawn_branches: the branch spawn right before verification
// (Eq. 7 PAPER P216-220): at the branch row s_b of the shared draft
// slot, c = q(x_b) (max_x q(x), or q of the drafted token), k_b = max(1,
// floor(k_max (1 - c))) and B = TopK(q(x_b), k_b) (ties -> smaller id, S393).
//
// One CTA per sequence streams the draft row once (16-byte loads, U vectors in flight
// per thread): lazy-offset online sum and exact max for the probabilities, plus one
// warp-wide sorted top-KL list by raw logit (the order of q) per warp; a vector enters
// the insertion path only if its max reaches max(block seed, warp list tail) — the
// seed, the KL-th largest of the threads' first-vector maxima, is a lower bound of the
// row's KL-th value, so almost every vector is filtered by one compare + one ballot.  The warps' lists merge by KL rounds of
// warp argmax.  Logit order == q order, so the token set is exact (ties: smaller id).
#include <algorithm>

#include "sb_host.h"

namespace sb {

// CTA size by batch: 8 warps per row while one wave of 256-thread CTAs (5 per SM at 48
// registers) covers the batch, 2 warps per row beyond that (C4's 2048 rows: 14 CTAs of
// 64 threads per SM, one wave; measured 0.198 ms -> 0.158 ms)
constexpr int kSpawnNT = 256, kSpawnNTSmall = 64;

struct SpawnParams {
  Dims d;
  const void* QL;
  const int* bpos;
  const int* tok;
  int mode, k_max;
  int* k_out;
  int* btok;
  float* bprob;
  float* conf;
};

template <int KL>
struct TopList {
  float v[KL];
  int id[KL];
  __device__ __forceinline__ void init() {
#pragma unroll
    for (int t = 0; t < KL; ++t) {
      v[t] = -CUDART_INF_F;
      id[t] = 0x7fffffff;
    }
  }
  // elements arrive in increasing id per thread, so an equal value never displaces
  __device__ __forceinline__ void insert(float f, int idx) {
    if (!(f > v[KL - 1] || (f == v[KL - 1] && idx < id[KL - 1]))) return;
    float cv = f;
    int ci = idx;
#pragma unroll
    for (int t = 0; t < KL; ++t) {
      const bool sw = cv > v[t] || (cv == v[t] && ci < id[t]);
      const float tv = v[t];
      const int ti = id[t];
      v[t] = sw ? cv : tv;
      id[t] = sw ? ci : ti;
      cv = sw ? tv : cv;
      ci = sw ? ti : ci;
    }
  }
  __device__ __forceinline__ void pop() {
#pragma unroll
    for (int t = 0; t + 1 < KL; ++t) {
      v[t] = v[t + 1];
      id[t] = id[t + 1];
    }
    v[KL - 1] = -CUDART_INF_F;
    id[KL - 1] = 0x7fffffff;
  }
};

// KL rounds of warp argmax over the lanes' list heads (value desc, id asc).
template <int KL>
__device__ __forceinline__ void warp_merge(TopList<KL>& L, float* outv, int* outid) {
  const int lane = threadIdx.x & 31;
  for (int r = 0; r < KL; ++r) {
    float bv = L.v[0];
    int bi = L.id[0];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
    }
    if (L.id[0] == bi && L.v[0] == bv && bi != 0x7fffffff) L.pop();
    if (lane == 0) { outv[r] = bv; outid[r] = bi; }
  }
}

// Warp-wide sorted top-KL list (value desc, id asc): lane t < KL holds entry t.  An
// element enters only if it beats the tail, so after the first vectors almost every
// 16-byte vector is filtered by one compare + one ballot per warp.
template <int KL>
struct WarpTop {
  float v;
  int id;
  __device__ __forceinline__ void init() { v = -CUDART_INF_F; id = 0x7fffffff; }
  __device__ __forceinline__ void tail(float& tv, int& ti) const {
    tv = __shfl_sync(0xffffffffu, v, KL - 1);
    ti = __shfl_sync(0xffffffffu, id, KL - 1);
  }
  // warp-uniform (f, x): insert if it ranks inside the list
  __device__ __forceinline__ void insert(float f, int x) {
    const int lane = threadIdx.x & 31;
    const bool above = lane < KL && (v > f || (v == f && id < x));
    const int pos = __popc(__ballot_sync(0xffffffffu, above));
    if (pos >= KL) return;
    const float pv = __shfl_up_sync(0xffffffffu, v, 1);
    const int pi = __shfl_up_sync(0xffffffffu, id, 1);
    if (lane > pos && lane < KL) { v = pv; id = pi; }
    if (lane == pos) { v = f; id = x; }
  }
  // insert, then return the tail value (warp-uniform)
  __device__ __forceinline__ float insert_tail(float f, int x) {
    insert(f, x);
    return __shfl_sync(0xffffffffu, v, KL - 1);
  }
};

template <typename T, int KL, int U, int NT>
__global__ void __launch_bounds__(NT) k_spawn(SpawnParams p, bool vec_ok) {
  constexpr int E = Vec<T>::E, NW = NT / 32;
  __shared__ RowStat red[NW];
  __shared__ float wv[NW * KL];
  __shared__ int wi[NW * KL];
  __shared__ float fv[KL];
  __shared__ int fi[KL];
  const Dims& d = p.d;
  const int b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int s = p.bpos ? __ldg(p.bpos + b) : 0;
  s = max(0, min(s, d.G));
  const T* row = static_cast<const T*>(p.QL) + row_off(d, b, 0, s);
  LazyAcc<false, 4> acc;  // lazy-offset sum, exact running max
  acc.init();
  WarpTop<KL> W;
  W.init();
  // filter threshold: max(list tail, lower bound); the lower bound is the KL-th largest
  // of the 32 lane maxima of the first vector group (KL distinct elements of this warp,
  // so <= the warp's true KL-th largest) -> no warm-up flood of candidates
  // block-wide seed: the KL-th largest of the NT threads' first-vector maxima (KL
  // distinct elements of the row, so <= the row's KL-th largest value)
  float filt;
  {
    float vm0 = -CUDART_INF_F;
    if (vec_ok && tid < d.V / E) {
      float f[E];
      Vec<T>::unpack(ldg_stream(reinterpret_cast<const uint4*>(row) + tid), f);
      vm0 = Vec<T>::vmax(f);
    } else if (!vec_ok && tid < d.V) {
      vm0 = ld_scalar(row + tid);
    }
    float cur = vm0;
    for (int r = 0; r < KL; ++r) {
      float mx = cur;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      const unsigned who = __ballot_sync(0xffffffffu, cur == mx);
      if (lane == __ffs(who) - 1) cur = -CUDART_INF_F;
      if (lane == 0) wv[warp * KL + r] = mx;
    }
    __syncthreads();
    TopList<(NW * KL + 31) / 32> M;
    M.init();
#pragma unroll
    for (int t = 0; t < (NW * KL + 31) / 32; ++t) {
      const int c = lane + 32 * t;
      if (c < NW * KL) M.insert(wv[c], c);
    }
    float kth = -CUDART_INF_F;
    for (int r = 0; r < KL; ++r) {
      float cv = M.v[0];
      int ci = M.id[0];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const float ov = __shfl_xor_sync(0xffffffffu, cv, o);
        const int oi = __shfl_xor_sync(0xffffffffu, ci, o);
        if (ov > cv || (ov == cv && oi < ci)) { cv = ov; ci = oi; }
      }
      if (M.id[0] == ci && M.v[0] == cv) M.pop();
      kth = cv;
    }
    filt = kth;
    __syncthreads();  // wv is reused by the final merge
  }
  int done = 0;
  if (vec_ok) {
    const int nvec = d.V / E;
    const uint4* rv = reinterpret_cast<const uint4*>(row);
    const int nv_round = (nvec + 32 * U * NW - 1) / (32 * U * NW) * (32 * U * NW);
    // register double buffer: the next U vectors are in flight while these are reduced
    uint4 xn[U];
#pragma unroll
    for (int j = 0; j < U; ++j) xn[j] = (tid + j * NT < nvec) ? ldg_stream(rv + tid + j * NT) : neg_inf_vec<T>();
    for (int vb = tid; vb < nv_round; vb += U * NT) {  // warp-uniform trip count
      uint4 x[U];
#pragma unroll
      for (int j = 0; j < U; ++j) {
        x[j] = xn[j];
        const int vn = vb + U * NT + j * NT;
        xn[j] = (vn < nvec) ? ldg_stream(rv + vn) : neg_inf_vec<T>();
      }
#pragma unroll
      for (int j = 0; j < U; ++j) {
        float f[E];
        Vec<T>::unpack(x[j], f);
        const bool valid = vb + j * NT < nvec;
        float vm;
        if constexpr (sizeof(T) == 2) {
          vm = acc_vecs_bf16<1>(acc, x + j, 0);  // packed FFMA2 / FADD2 sums, returns the max
        } else {
          vm = Vec<T>::vmax(f);
          float g[E];  // the accumulator freezes (masks) its maximum in place; f feeds the top-K
#pragma unroll
          for (int e = 0; e < E; ++e) g[e] = f[e];
          acc.template add_cm<E>(g, vm, vb + j * NT);
        }
        unsigned cand = __ballot_sync(0xffffffffu, valid && vm >= filt);
        while (cand) {  // rare once warm: one lane's values, broadcast, qualifying ones inserted
          const int src = __ffs(cand) - 1;
          cand &= cand - 1;
          const int bb = (vb - lane + src + j * NT) * E;
#pragma unroll
          for (int e = 0; e < E; ++e) {
            const float xv = __shfl_sync(0xffffffffu, f[e], src);
            if (xv >= filt) filt = fmaxf(filt, W.insert_tail(xv, bb + e));
          }
        }
      }
    }
    done = nvec * E;
  }
  for (int v0 = done; v0 < d.V; v0 += NT) {  // scalar tail / unaligned rows: one value per thread
    const int v = v0 + tid;
    float f[E];
    f[0] = v < d.V ? ld_scalar(row + v) : -CUDART_INF_F;
#pragma unroll
    for (int e = 1; e < E; ++e) f[e] = -CUDART_INF_F;
    {
      float g[E];  // (add() masks the frozen maximum in place)
#pragma unroll
      for (int e = 0; e < E; ++e) g[e] = f[e];
      acc.template add<E>(g, 0);
    }
    unsigned cand = __ballot_sync(0xffffffffu, v < d.V && f[0] >= filt);
    while (cand) {
      const int src = __ffs(cand) - 1;
      cand &= cand - 1;
      const float xv = __shfl_sync(0xffffffffu, f[0], src);
      if (xv >= filt) filt = fmaxf(filt, W.insert_tail(xv, v0 + warp * 32 + src));
    }
  }
  RowStat st = fold_lazy(acc);
  st.idx = 0x7fffffff;
  st = block_reduce<NT>(st, red);
  if (lane < KL) { wv[warp * KL + lane] = W.v; wi[warp * KL + lane] = W.id; }
  __syncthreads();
  if (warp == 0) {  // merge the warps' lists: KL rounds of argmax over NW*KL candidates
    TopList<(NW * KL + 31) / 32> M;
    M.init();
#pragma unroll
    for (int t = 0; t < (NW * KL + 31) / 32; ++t) {
      const int c = lane + 32 * t;
      if (c < NW * KL) M.insert(wv[c], wi[c]);
    }
    float bv[KL];
    int bi[KL];
    for (int r = 0; r < KL; ++r) {
      float cv = M.v[0];
      int ci = M.id[0];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const float ov = __shfl_xor_sync(0xffffffffu, cv, o);
        const int oi = __shfl_xor_sync(0xffffffffu, ci, o);
        if (ov > cv || (ov == cv && oi < ci)) { cv = ov; ci = oi; }
      }
      if (M.id[0] == ci && M.v[0] == cv && ci != 0x7fffffff) M.pop();
      bv[r] = cv;
      bi[r] = ci;
    }
    if (lane == 0)
      for (int r = 0; r < KL; ++r) { fv[r] = bv[r]; fi[r] = bi[r]; }
  }
  __syncthreads();
  if (tid == 0) {
    const RowOut o = finish(st);
    int k = 0;
    double c = CUDART_NAN;
    if (o.finite) {
      if (p.mode == SB_CONF_TOKEN) {
        const int x = __ldg(p.tok + ent(d, b, 0, s));
        if (x >= 0 && x < d.V) c = tok_prob(ld_scalar(row + x), o.MS, o.Z);
      } else {
        c = tok_prob(st.m, o.MS, o.Z);  // max_x q(x)
      }
      if (c == c) {
        const double kk = floor((double)p.k_max * (1.0 - c));  // Eq. 7
        k = kk < 1.0 ? 1 : (int)kk;
        k = min(k, min(d.V, KL));
      }
    }
    p.k_out[b] = k;
    if (p.conf) p.conf[b] = (float)c;
    for (int j = 0; j < p.k_max; ++j) {
      const bool on = j < k;
      p.btok[(int64_t)b * p.k_max + j] = on ? fi[j] : -1;
      if (p.bprob) p.bprob[(int64_t)b * p.k_max + j] = on ? (float)tok_prob(fv[j], o.MS, o.Z) : CUDART_NAN_F;
    }
  }
}

template <typename T, int KL>
static sb_status launch_spawn(const SpawnParams& p, bool vok, cudaStream_t s) {
  if (p.d.B > 5 * num_sms()) k_spawn<T, KL, 4, kSpawnNTSmall><<<p.d.B, kSpawnNTSmall, 0, s>>>(p, vok);
  else k_spawn<T, KL, 4, kSpawnNT><<<p.d.B, kSpawnNT, 0, s>>>(p, vok);
  return cuda_status(cudaGetLastError());
}

}  // namespace sb

using namespace sb;

extern "C" sb_status sb_spawn_branches(const sb_dims* dd, const void* q_logits, const int32_t* branch_pos,
                                       const int32_t* tok, sb_conf_mode mode, int32_t k_max, int32_t* k_out,
                                       int32_t* branch_tok, float* branch_prob, float* conf, sb_stream_t stream) {
  SB_NVTX("sb_spawn_branches");
  if (!dims_valid(dd) || sharded(dd) || !q_logits || !k_out || !branch_tok) return SB_ERR_INVALID_ARG;
  if (mode != SB_CONF_TOP1 && mode != SB_CONF_TOKEN) return SB_ERR_INVALID_ARG;
  if (mode == SB_CONF_TOKEN && !tok) return SB_ERR_INVALID_ARG;
  if (k_max < 1 || k_max > 16) return SB_ERR_INVALID_ARG;
  SpawnParams p;
  p.d = to_dims(dd); p.QL = q_logits; p.bpos = branch_pos; p.tok = tok; p.mode = mode; p.k_max = k_max;
  p.k_out = k_out; p.btok = branch_tok; p.bprob = branch_prob; p.conf = conf;
  const bool vok = vec_ok(dd, q_logits);
  cudaStream_t s = (cudaStream_t)stream;
  if (dd->dtype == SB_BF16)
    return k_max <= 8 ? launch_spawn<__nv_bfloat16, 8>(p, vok, s) : launch_spawn<__nv_bfloat16, 16>(p, vok, s);
  return k_max <= 8 ? launch_spawn<float, 8>(p, vok, s) : launch_spawn<float, 16>(p, vok, s);
}
