// sb_spawn.cu — sb_spawn_branches: the branch spawn right before verification
// (Eq. 7 PAPER P216-220): at the branch row s_b of the shared draft
// slot, c = q(x_b) (max_x q(x), or q of the drafted token), k_b = max(1,
// floor(k_max (1 - c))) and B = TopK(q(x_b), k_b) (ties -> smaller id, S393).
//
// One CTA per sequence streams the draft row once (16-byte loads, U vectors in flight
// per thread): online max / sum (exact-offset state) for the probabilities, plus a
// per-thread sorted top-KL list by raw logit (the order of q), insertion only when a
// vector's max beats the list's tail.  Lists merge by KL rounds of warp argmax, then
// once more across warps.  Logit order == q order, so the token set is exact.
#include <algorithm>

#include "sb_host.h"

namespace sb {

constexpr int kSpawnNT = 256;

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

template <typename T, int KL, int U>
__global__ void __launch_bounds__(kSpawnNT) k_spawn(SpawnParams p, bool vec_ok) {
  constexpr int E = Vec<T>::E, NT = kSpawnNT, NW = NT / 32;
  __shared__ RowStat red[NW];
  __shared__ float wv[NW][KL];
  __shared__ int wi[NW][KL];
  __shared__ float fv[KL];
  __shared__ int fi[KL];
  const Dims& d = p.d;
  const int b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int s = p.bpos ? __ldg(p.bpos + b) : 0;
  s = max(0, min(s, d.G));
  const T* row = static_cast<const T*>(p.QL) + row_off(d, b, 0, s);
  RowAcc<false, 4> acc;
  acc.init();
  TopList<KL> L;
  L.init();
  int done = 0;
  if (vec_ok) {
    const int nvec = d.V / E;
    const uint4* rv = reinterpret_cast<const uint4*>(row);
    for (int vb = tid; vb < nvec; vb += U * NT) {
      uint4 x[U];
#pragma unroll
      for (int j = 0; j < U; ++j)
        if (vb + j * NT < nvec) x[j] = ldg_stream(rv + vb + j * NT);
#pragma unroll
      for (int j = 0; j < U; ++j) {
        if (vb + j * NT >= nvec) break;
        float f[E];
        Vec<T>::unpack(x[j], f);
        const float vm = Vec<T>::vmax(f);
        const int base = (vb + j * NT) * E;
        acc.template add<E>(f, vm, base);
        if (vm > L.v[KL - 1] || vm == L.v[KL - 1]) {  // rare after the first vectors
#pragma unroll
          for (int e = 0; e < E; ++e) L.insert(f[e], base + e);
        }
      }
    }
    done = nvec * E;
  }
  for (int v = done + tid; v < d.V; v += NT) {
    const float f = ld_scalar(row + v);
    acc.add1(f, v);
    L.insert(f, v);
  }
  const RowStat st = block_reduce<NT>(fold(acc), red);
  warp_merge<KL>(L, wv[warp], wi[warp]);
  __syncthreads();
  if (warp == 0) {
    TopList<KL> M;
#pragma unroll
    for (int t = 0; t < KL; ++t) {
      M.v[t] = lane < NW ? wv[lane][t] : -CUDART_INF_F;
      M.id[t] = lane < NW ? wi[lane][t] : 0x7fffffff;
    }
    warp_merge<KL>(M, fv, fi);
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
  k_spawn<T, KL, 4><<<p.d.B, kSpawnNT, 0, s>>>(p, vok);
  return cuda_status(cudaGetLastError());
}

}  // namespace sb

using namespace sb;

extern "C" sb_status sb_spawn_branches(const sb_dims* dd, const void* q_logits, const int32_t* branch_pos,
                                       const int32_t* tok, sb_conf_mode mode, int32_t k_max, int32_t* k_out,
                                       int32_t* branch_tok, float* branch_prob, float* conf, sb_stream_t stream) {
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
