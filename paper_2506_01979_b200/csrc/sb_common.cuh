// sb_common.cuh — shared device helpers of libspecbranch (sm_100a only).
//
// Row softmax state in log2 units.  With c = fp32(log2 e) every element contributes
//   e_v = 2^(l_v * c - ms),   ms = m * c (one fp32 constant per running max m)
// computed as ex2.approx(fma(l_v, c, -ms)): the product l*c is exact inside the FMA,
// so the rounding of ms cancels between a row's normaliser Z = sum e_v and any single
// probability 2^(l_x c - MS) / Z evaluated later in fp64 with the same MS.  The
// entropy uses S1 = sum e_v * a_v (a_v the exponent), H = ln2 * (log2 Z - S1 / Z).
// Per-thread sums are fp32; every reduction across threads, warps and shards is fp64
// (RowStat), and q rows keep the element that set the current offset out of the fp32
// accumulators (LazyAcc / RowAcc "frozen" part), so the small terms of a peaked row are
// never rounded against its dominant term: H of a near one-hot row stays within
// 1e-5 |H| + 1e-7 nats (SURVEY §8.4 pass band).
// All reductions are fixed-order trees (no float atomics): bit-reproducible.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <math_constants.h>
#include <stdint.h>

#include "../../include/specbranch.h"

namespace sb {

constexpr float kC = 1.4426950408889634f;  // fp32(log2 e)
constexpr float kLn2 = 0.69314718055994531f;
constexpr float kInvC = 0.69314718055994531f;  // 1 / log2 e (the rescale test only)
constexpr int kMaxK = 32;
constexpr float kMsEmpty = -1e30f;  // exponent offset of a state that has seen no finite value
// Lazy offset: rescale only when max*c - ms exceeds the threshold.  q rows also sum
// S1 = sum e*a, whose fp32 rounding grows with the offset lag |a| of the largest terms,
// so they keep the lag <= 6.  p rows keep it <= 10 so that a peaked row's dominant
// element (p >= ~0.05: 2^10 above a thread's first-group maximum) raises the offset and
// is frozen (kept out of the fp32 sums, see RowAcc): with 2^20 of headroom it was
// summed in fp32 and every later small term rounded against it (Z off by up to ~1e-6
// relative, residual mass R by ~1e-6 absolute).  10 rather than 6: a bulk N(0, 2^2)
// logit exceeds its thread's first-group maximum by 10 / c only with probability ~2e-4,
// so the rescale branch (~150 instructions per warp) stays off the hot path.
#ifndef SB_RESCALE_P
#define SB_RESCALE_P 10.f
#endif
constexpr float kRescaleP = SB_RESCALE_P;
constexpr float kRescaleQ = 6.f;
constexpr int kMaxG = 31;
// Input domain (include/specbranch.h "Input domain"; DESIGN reading 34): a row is
// evaluated iff its maximum logit m (NaN entries ignored) is finite with |m| < 2^24,
// where the fp32 offset ms = fl(m c) is exact to within one unit of the exponent; other
// entries are unrestricted (-inf, -FLT_MAX, finfo(bf16).min masks contribute exactly 0).
constexpr float kLogitRange = 16777216.f;  // 2^24
// The bf16 q-row path clamps its inputs to -2^97 (one HMNMX2.NAN per two values, NaN
// kept) so the entropy sum e*a never meets 0 * -inf.  For any row with m > -2^97 this is
// exact (the clamped entries contribute 0 either way); a row whose clamped maximum is
// -2^97 is outside the domain or all -inf, told apart by row_has_finite() (rare path).
constexpr float kMaskedLogit = -1.5845632502852868e29f;  // -2^97, exact in bf16 (0xf000)
constexpr uint32_t kMaskedBf16x2 = 0xf000f000u;

struct Dims {
  int B, K, G, V;
  int64_t rs;  // row stride (elements)
  int64_t ss;  // sequence stride (elements)
  int dtype;
};

__host__ __device__ inline int64_t row_off(const Dims& d, int b, int slot, int i) {
  return (int64_t)b * d.ss + ((int64_t)slot * (d.G + 1) + i) * d.rs;
}
__host__ __device__ inline int64_t ent(const Dims& d, int b, int k, int i) {  // [B][K][G+1]
  return ((int64_t)b * d.K + k) * (d.G + 1) + i;
}

// ------------------------------------------------------------------ timeline tracing
// SB_TRACE builds only (diagnostics, scripts/step_trace.py): per CTA and role, the
// global timer at numbered events of the streaming kernels.  Each translation unit
// defines its own table (SB_TRACE_TABLE) and a C reader.
#ifdef SB_TRACE
constexpr int kTrCtas = 160, kTrRoles = 8, kTrEvents = 64;
#define SB_TRACE_TABLE(name)                                                              \
  __device__ unsigned long long name[::sb::kTrCtas][::sb::kTrRoles][::sb::kTrEvents];     \
  extern "C" int name##_read(void* host, size_t bytes) {                                  \
    return (int)cudaMemcpyFromSymbol(host, name, bytes < sizeof(name) ? bytes : sizeof(name)); \
  }
#define SB_TRACE_AT(table, role, ev)                                                      \
  do {                                                                                    \
    unsigned long long t_;                                                                \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                \
    if (blockIdx.x < ::sb::kTrCtas && (ev) < ::sb::kTrEvents && (ev) >= 0)                \
      table[blockIdx.x][role][ev] = t_;                                                   \
  } while (0)
#else
#define SB_TRACE_AT(table, role, ev) do {} while (0)
#endif

// ------------------------------------------------------------------ small PTX helpers
// Programmatic dependent launch (launch_pdl): wait for the predecessor grid's memory,
// then let the next grid be scheduled.
__device__ __forceinline__ void pdl_wait() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float fmax_nan(float a, float b) {  // NaN-propagating max
  float r;
  asm("max.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
  return r;
}
// 2^a for two values on the FMA pipe (FFMA2), as a stand-in for MUFU.EX2 on a share of
// the p-row elements: the streaming kernels issue one MUFU per element and the MUFU
// pipe (16 lanes / clk / SM) co-limits them at full HBM bandwidth.  a <= 2^7 (the lazy
// offsets keep a <= kRescale); a = round(a) + f, f in [-1/2, 1/2]; 2^f by a degree-5
// polynomial with p(0) = 1 (fit for relative error on [-1/2, 1/2]: max 1.7e-7, mean
// -2e-8 with fp32 Horner, about the accuracy of ex2.approx); 2^round(a) built in the
// exponent field (one IMAD: bits(a + 1.5 2^23) * 2^23 + bits(1.0)) and applied with
// one FMUL2, so NaN propagates.  Below 2^-126 it returns tiny normals instead of 0
// (a clamped at -126; masked -inf entries contribute <= 2^-125 each, far below the
// row's own maximum term 2^-kRescale).
__device__ __forceinline__ float2 ex2_poly2(float2 a) {
  a.x = fmax_nan(a.x, -126.f);
  a.y = fmax_nan(a.y, -126.f);
  const float2 M = make_float2(12582912.f, 12582912.f);  // 1.5 * 2^23
  const float2 t = __fadd2_rn(a, M);
  const float2 j = __fadd2_rn(t, make_float2(-12582912.f, -12582912.f));
  const float2 f = __ffma2_rn(j, make_float2(-1.f, -1.f), a);  // exact
  float2 q = make_float2(1.3264661e-3f, 1.3264661e-3f);
  q = __ffma2_rn(q, f, make_float2(9.6714906e-3f, 9.6714906e-3f));
  q = __ffma2_rn(q, f, make_float2(5.5507336e-2f, 5.5507336e-2f));
  q = __ffma2_rn(q, f, make_float2(2.4022242e-1f, 2.4022242e-1f));
  q = __ffma2_rn(q, f, make_float2(6.9314700e-1f, 6.9314700e-1f));
  q = __ffma2_rn(q, f, make_float2(1.f, 1.f));
  const float2 sc = make_float2(__int_as_float(__float_as_int(t.x) * 8388608 + 0x3f800000),
                                __int_as_float(__float_as_int(t.y) * 8388608 + 0x3f800000));
  return __fmul2_rn(q, sc);
}
// p-row exponentials (experiment builds: SB_POLY_P = n routes every n-th packed pair
// of a p row through ex2_poly2; 0 = all on MUFU.EX2)
#ifndef SB_POLY_P
#define SB_POLY_P 0
#endif
constexpr int kPolyP = SB_POLY_P;
__device__ __forceinline__ float fmax3(float a, float b, float c) {
  float r;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}
__device__ __forceinline__ uint4 ldg_stream(const void* p) {
  uint4 r;
  asm("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ uint32_t bf16x2_max_nan(uint32_t a, uint32_t b) {
  uint32_t r;
  asm("max.NaN.bf16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}
__device__ __forceinline__ float bf16_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf16_hi(uint32_t w) { return __uint_as_float(w & 0xffff0000u); }

template <typename T>
__device__ __forceinline__ float ld_scalar(const T* p);
template <>
__device__ __forceinline__ float ld_scalar<float>(const float* p) {
  return __ldg(p);
}
template <>
__device__ __forceinline__ float ld_scalar<__nv_bfloat16>(const __nv_bfloat16* p) {
  return __uint_as_float((uint32_t)__ldg(reinterpret_cast<const unsigned short*>(p)) << 16);
}

// Unpack one 16-byte vector into E fp32 values (exact widening).
template <typename T>
struct Vec;
template <>
struct Vec<__nv_bfloat16> {
  static constexpr int E = 8;
  __device__ __forceinline__ static void unpack(const uint4& v, float* f) {
    f[0] = bf16_lo(v.x); f[1] = bf16_hi(v.x); f[2] = bf16_lo(v.y); f[3] = bf16_hi(v.y);
    f[4] = bf16_lo(v.z); f[5] = bf16_hi(v.z); f[6] = bf16_lo(v.w); f[7] = bf16_hi(v.w);
  }
  __device__ __forceinline__ static float vmax(const float* f) {
    return fmax3(fmax3(f[0], f[1], f[2]), fmax3(f[3], f[4], f[5]), fmaxf(f[6], f[7]));
  }
};
template <>
struct Vec<float> {
  static constexpr int E = 4;
  __device__ __forceinline__ static void unpack(const uint4& v, float* f) {
    f[0] = __uint_as_float(v.x); f[1] = __uint_as_float(v.y);
    f[2] = __uint_as_float(v.z); f[3] = __uint_as_float(v.w);
  }
  __device__ __forceinline__ static float vmax(const float* f) {
    return fmaxf(fmax3(f[0], f[1], f[2]), f[3]);
  }
};

// ------------------------------------------------------------------ online row state
// Offset bookkeeping shared by the accumulators: the new offset clamped to the fp32
// range (a maximum beyond 2.36e38 overflows m*c; such a row is outside the input domain
// anyway) and the rescale exponent clamped to [-256, 0] (0 only when leaving the empty
// state, whose sums are 0), so no 0 * inf can poison a finite row.
__device__ __forceinline__ float offset_of(float m) {
  return fminf(fmaxf(m * kC, -3.4028234663852886e38f), 3.4028234663852886e38f);
}
__device__ __forceinline__ float rescale_exp(float ms, float nms) {
  return fminf(fmaxf(ms - nms, -256.f), 0.f);
}

// Per-thread running state of one row with the exact running maximum as offset.
// NA independent accumulators for ILP and a shorter fp32 summation chain.  kQ adds S1
// (entropy), the top-1 index and the frozen part: the element(s) equal to the current
// maximum are kept in (zf, s1f) instead of z[] (their e = 2^(m c - ms) from an accurate
// exp2 of the exactly representable residual m c - fl(m c)), and join z[] only when a
// larger maximum arrives.
template <bool kQ, int NA>
struct RowAcc {
  float m;       // running max (raw logit units), -inf until the first finite value
  float ms;      // m * c (fp32), the exponent offset used by every term
  float z[NA];   // sum of 2^(l c - ms)
  float s1[kQ ? NA : 1];
  float fa;      // exponent a = m c - ms of the frozen maximum element(s) ...
  int fn;        // ... and their count (0: none); their e = 2^a is evaluated in fp64
  int idx;       // smallest index attaining m (kQ only)

  __device__ __forceinline__ void init() {
    m = -CUDART_INF_F;
    ms = kMsEmpty;
#pragma unroll
    for (int j = 0; j < NA; ++j) z[j] = 0.f;
#pragma unroll
    for (int j = 0; j < (kQ ? NA : 1); ++j) s1[j] = 0.f;
    fa = 0.f;
    fn = 0;
    idx = 0x7fffffff;
  }

  // raise the running max to nm (> m); rare after the first few vectors
  __device__ __forceinline__ void rescale(float nm) {
    const float nms = offset_of(nm);
    const float dd = rescale_exp(ms, nms);
    const float sc = ex2(dd);  // 0 from the kMsEmpty sentinel
#pragma unroll
    for (int j = 0; j < NA; ++j) {
      if (kQ) s1[j] = sc * fmaf(z[j], dd, s1[j]);
      z[j] *= sc;
    }
    if (fn) {  // the previous maximum's element(s) become ordinary terms
      const float ef = (float)fn * exp2f(fa);
      if (kQ) s1[0] = fmaf(sc, ef * (fa + dd), s1[0]);
      z[0] = fmaf(sc, ef, z[0]);
    }
    m = nm;
    ms = nms;
  }
  // move the n elements equal to the new maximum into the frozen part
  __device__ __forceinline__ void freeze(int n) {
    fa = fmaf(m, kC, -ms);  // exact: the rounding residual of ms
    fn = n;
  }

  // accumulate E values f[] whose first element has index base
  template <int E>
  __device__ __forceinline__ void add(const float* fin, float vmax, int base) {
    float f[E];
#pragma unroll
    for (int j = 0; j < E; ++j) f[j] = fin[j];
    if (vmax > m) {
      rescale(vmax);
      int first = E, n = 0;
#pragma unroll
      for (int j = E - 1; j >= 0; --j)
        if (f[j] == vmax) { first = j; ++n; f[j] = kMaskedLogit; }
      if (kQ) idx = base + first;
      freeze(n);
    }
#pragma unroll
    for (int j = 0; j < E; ++j) {
      const float a = fmaf(f[j], kC, -ms);
      const float e = ex2(a);
      z[j % NA] += e;
      if (kQ) s1[j % NA] = fmaf(e, fmaxf(a, -200.f), s1[j % NA]);
    }
  }

  __device__ __forceinline__ void add1(float f, int index) {
    if (f > m) {
      rescale(f);
      if (kQ) idx = index;
      freeze(1);
      return;
    }
    const float a = fmaf(f, kC, -ms);
    const float e = ex2(a);
    z[0] += e;
    if (kQ) s1[0] = fmaf(e, fmaxf(a, -200.f), s1[0]);
  }
};

// Lazy-offset accumulator for the streaming (TMA) kernels.  Per group of N values:
// the exact running max m (one FMNMX), the group tag of its first occurrence (Q rows;
// one FSETP + SEL), and the exponent offset ms raised only when max*c - ms > 20 (p) / 6
// (q), a warp-uniform rare branch, so the hot path is unpack, FFMA, MUFU.EX2, FADD (+
// FMNMX, FFMA for the entropy sum of q rows).  q rows freeze the element(s) that raise
// the offset (see RowAcc): for a peaked row that is its dominant element, so the fp32
// sums z[] only ever hold terms far below it.
template <bool kQ, int NA>
struct LazyAcc {
  static constexpr float kT = kQ ? kRescaleQ : kRescaleP;
  float m;
  float ms;
  float lim;  // raw-logit form of the rescale test: a group maximum cm > lim ~ (ms + kT) / c
  float z[NA];
  float s1[kQ ? NA : 1];
  float fa;  // frozen element(s): exponent and count (see RowAcc)
  int fn;
  int tag;

  __device__ __forceinline__ void set_offset(float nms) {
    ms = nms;
    lim = (nms + kT) * kInvC;
  }
  __device__ __forceinline__ void init() {
    m = -CUDART_INF_F;
    ms = kMsEmpty;
    lim = -CUDART_INF_F;  // the empty state takes any finite maximum
#pragma unroll
    for (int j = 0; j < NA; ++j) z[j] = 0.f;
#pragma unroll
    for (int j = 0; j < (kQ ? NA : 1); ++j) s1[j] = 0.f;
    fa = 0.f;
    fn = 0;
    tag = -1;
  }
  __device__ __forceinline__ void rescale(float nms) {
    const float dd = rescale_exp(ms, nms);
    const float sc = ex2(dd);
#pragma unroll
    for (int j = 0; j < NA; ++j) {
      if (kQ) s1[j] = sc * fmaf(z[j], dd, s1[j]);
      z[j] *= sc;
    }
    if (fn) {
      const float ef = (float)fn * exp2f(fa);
      if (kQ) s1[0] = fmaf(sc, ef * (fa + dd), s1[0]);
      z[0] = fmaf(sc, ef, z[0]);
    }
    set_offset(nms);
  }
  // inside the rescale branch: the group's elements equal to its maximum cm (which
  // set the new offset) leave f[] for the frozen part
  template <int N>
  __device__ __forceinline__ void freeze(float* f, float cm) {
    int n = 0;
#pragma unroll
    for (int j = 0; j < N; ++j) {
      const bool eq = f[j] == cm;
      f[j] = eq ? kMaskedLogit : f[j];
      n += eq;
    }
    fa = fmaf(cm, kC, -ms);  // exact residual of ms = fl(cm c)
    fn = n;
  }
  // The rescale test of one group.  FIRST: the first group after init() (every lane
  // takes it together, so no vote, and an empty state needs no rescaling of its sums).
  template <int N, bool FIRST>
  __device__ __forceinline__ void raise(float* f, float cm) {
    if (FIRST) {
      if (cm > lim) {
        set_offset(offset_of(cm));
        freeze<N>(f, cm);
      }
      return;
    }
    bool up = cm > lim;
    // rare; written as a loop so the compiler keeps it a branch instead of predicating
    // the rescale into every iteration
    while (__builtin_expect(__any_sync(0xffffffffu, up), 0)) {
      if (up) {
        rescale(offset_of(cm));
        freeze<N>(f, cm);
      }
      up = false;
    }
  }
  template <int N, bool FIRST = false>
  __device__ __forceinline__ void add(float* f, int t) {
    float cm = f[0];
#pragma unroll
    for (int j = 1; j + 1 < N; j += 2) cm = fmax3(cm, f[j], f[j + 1]);
    if (N % 2 == 0) cm = fmaxf(cm, f[N - 1]);
    add_cm<N, FIRST>(f, cm, t);
  }
  // the same with the group maximum cm = max(f[0..N)) already known
  template <int N, bool FIRST = false>
  __device__ __forceinline__ void add_cm(float* f, float cm, int t) {
    if (kQ) tag = (cm > m) ? t : tag;
    m = fmaxf(m, cm);
    raise<N, FIRST>(f, cm);
#pragma unroll
    for (int j = 0; j < N; ++j) {
      const float a = fmaf(f[j], kC, -ms);
      const float e = ex2(a);
      z[j % NA] += e;
      if (kQ) s1[j % NA] = fmaf(e, fmaxf(a, -200.f), s1[j % NA]);
    }
  }

  // The same as add<2*NW>() on NW packed bf16 pairs, with the fp32 arithmetic paired
  // into FFMA2 / FADD2 (same IEEE fp32 operations, same accumulator order: element j
  // goes to z[j % 4]).  q rows clamp their inputs at -2^97 instead of clamping the
  // exponent: identical results for every logit > -2^97, since ex2.approx.ftz is 0
  // below 2^-126 either way.
  template <int NW, bool FIRST = false>
  __device__ __forceinline__ float add_bf16(const uint32_t* win, int t) {
    static_assert(NA == 4 && NW % 2 == 0, "pairs map to (z0,z1), (z2,z3)");
    constexpr int N = 2 * NW;
    float f[N];
#pragma unroll
    for (int j = 0; j < NW; ++j) {
      const uint32_t w = kQ ? bf16x2_max_nan(win[j], kMaskedBf16x2) : win[j];
      f[2 * j] = bf16_lo(w);
      f[2 * j + 1] = bf16_hi(w);
    }
    float cm = f[0];
#pragma unroll
    for (int j = 1; j + 1 < N; j += 2) cm = fmax3(cm, f[j], f[j + 1]);
    cm = fmaxf(cm, f[N - 1]);
    if (kQ) tag = (cm > m) ? t : tag;
    m = fmaxf(m, cm);
    raise<N, FIRST>(f, cm);
    const float2 c2 = make_float2(kC, kC), n2 = make_float2(-ms, -ms);
    float2 za = make_float2(z[0], z[1]), zb = make_float2(z[2], z[3]);
    float2 sa = make_float2(0.f, 0.f), sb = sa;
    if (kQ) {
      sa = make_float2(s1[0], s1[1]);
      sb = make_float2(s1[2], s1[3]);
    }
#pragma unroll
    for (int j = 0; j < NW; ++j) {
      const float2 a = __ffma2_rn(make_float2(f[2 * j], f[2 * j + 1]), c2, n2);
      float2 e;
#ifdef SB_P_NOEXP  // bandwidth-ceiling experiment only: p rows skip the exponential (wrong sums)
      if (!kQ) e = a; else
#endif
      if (!kQ && kPolyP > 0 && j % (kPolyP > 0 ? kPolyP : 1) == (kPolyP > 0 ? kPolyP : 1) - 1)
        e = ex2_poly2(a);
      else
        e = make_float2(ex2(a.x), ex2(a.y));
      if (j % 2 == 0) {
        za = __fadd2_rn(za, e);
        if (kQ) sa = __ffma2_rn(e, a, sa);
      } else {
        zb = __fadd2_rn(zb, e);
        if (kQ) sb = __ffma2_rn(e, a, sb);
      }
    }
    z[0] = za.x; z[1] = za.y; z[2] = zb.x; z[3] = zb.y;
    if (kQ) {
      s1[0] = sa.x; s1[1] = sa.y; s1[2] = sb.x; s1[3] = sb.y;
    }
    return cm;  // this group's maximum (of the clamped values for q rows)
  }
};

// A 16-byte vector of -inf (fill for lanes past the end of a row).
template <typename T>
__device__ __forceinline__ uint4 neg_inf_vec() {
  return sizeof(T) == 2 ? make_uint4(0xff80ff80u, 0xff80ff80u, 0xff80ff80u, 0xff80ff80u)
                        : make_uint4(0xff800000u, 0xff800000u, 0xff800000u, 0xff800000u);
}

// Accumulate NV 16-byte bf16 vectors of one row chunk (tag t) into a LazyAcc.
template <int NV, bool kQ, bool FIRST = false>
__device__ __forceinline__ float acc_vecs_bf16(LazyAcc<kQ, 4>& a, const uint4* x, int t) {
  uint32_t w[4 * NV];
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    w[4 * j] = x[j].x; w[4 * j + 1] = x[j].y; w[4 * j + 2] = x[j].z; w[4 * j + 3] = x[j].w;
  }
  return a.template add_bf16<4 * NV, FIRST>(w, t);
}

// Reduced row state (one per thread after folding accumulators, then across threads).
// The sums are fp64 from here on: a row's dominant term (the frozen part of the thread
// holding it) and everything else meet only in fp64 adds.
struct RowStat {
  float m, ms;
  double z, s1;
  int idx;
};

// The frozen element(s) of a q row, n * 2^a and their entropy term n * 2^a * a, in fp64
// (a is the exact rounding residual of the offset: a one-hot row gets H = 0 exactly).
// 2^a for the frozen residual a = fl(m c) rounding error: |a| <= ulp(m c) / 2, tiny
// for every in-domain row (|m| < 2^24), so a cubic Taylor series is exact to ~1e-16
// there (the library exp2 costs ~40 fp64 instructions per lane per row).
__device__ __forceinline__ double exp2_small(float a) {
  const double x = (double)a * 0.69314718055994530942;
  if (fabs(x) > 0x1p-12) return exp2((double)a);
  return fma(x, fma(x, fma(x, 1.0 / 6.0, 0.5), 1.0), 1.0);
}
template <bool kQ>
__device__ __forceinline__ void add_frozen(RowStat& r, int n, float a) {
  if (n) {
    const double e = (double)n * exp2_small(a);
    r.z += e;
    if (kQ) r.s1 += e * (double)a;
  }
}

template <bool kQ, int NA>
__device__ __forceinline__ RowStat fold_lazy(const LazyAcc<kQ, NA>& a) {
  RowStat r;
  r.m = a.m;
  r.ms = a.ms;
  float z = 0.f, s = 0.f;
#pragma unroll
  for (int j = 0; j < NA; ++j) z += a.z[j];
  if (kQ) {
#pragma unroll
    for (int j = 0; j < NA; ++j) s += a.s1[j];
  }
  r.z = (double)z;
  r.s1 = (double)s;
  add_frozen<kQ>(r, a.fn, a.fa);
  r.idx = 0x7fffffff;
  return r;
}

// Identity element of combine().
__device__ __forceinline__ RowStat rowstat_empty() {
  RowStat r;
  r.m = -CUDART_INF_F;
  r.ms = kMsEmpty;
  r.z = 0.0;
  r.s1 = 0.0;
  r.idx = 0x7fffffff;
  return r;
}

template <bool kQ, int NA>
__device__ __forceinline__ RowStat fold(const RowAcc<kQ, NA>& a) {
  RowStat r;
  r.m = a.m;
  r.ms = a.ms;
  float z = 0.f, s = 0.f;
#pragma unroll
  for (int j = 0; j < NA; ++j) z += a.z[j];
  if (kQ) {
#pragma unroll
    for (int j = 0; j < NA; ++j) s += a.s1[j];
  }
  r.z = (double)z;
  r.s1 = (double)s;
  add_frozen<kQ>(r, a.fn, a.fa);
  r.idx = kQ ? a.idx : 0;
  return r;
}

// Bring a state's sums to the offset MS >= s.ms (fp64; the scale 2^(s.ms - MS) is 1
// exactly for the state that holds MS).
__device__ __forceinline__ void shift_to(RowStat& s, float MS) {
  const float dd = rescale_exp(s.ms, MS);
  const double sc = (double)ex2(dd);
  s.s1 = sc * fma(s.z, (double)dd, s.s1);
  s.z = sc * s.z;
  s.ms = MS;
}

// Combine two states (called in a fixed tree order).  The exact max / first index
// follow the larger value (ties: smaller index); the sums are brought to the larger
// exponent offset.  Works for any offsets (lazy or exact), for empty states (kMsEmpty,
// z = 0) and keeps NaN poison (z = NaN) of non-finite rows.
__device__ __forceinline__ RowStat combine(RowStat a, RowStat b) {
  RowStat r;
  const bool bw = b.m > a.m || (b.m == a.m && b.idx < a.idx);
  r.m = bw ? b.m : a.m;
  r.idx = bw ? b.idx : a.idx;
  const float MS = fmaxf(a.ms, b.ms);
  shift_to(a, MS);
  shift_to(b, MS);
  r.z = a.z + b.z;
  r.s1 = a.s1 + b.s1;
  r.ms = MS;
  return r;
}

__device__ __forceinline__ RowStat shfl_xor(const RowStat& s, int o) {
  RowStat r;
  r.m = __shfl_xor_sync(0xffffffffu, s.m, o);
  r.ms = __shfl_xor_sync(0xffffffffu, s.ms, o);
  r.z = __shfl_xor_sync(0xffffffffu, s.z, o);
  r.s1 = __shfl_xor_sync(0xffffffffu, s.s1, o);
  r.idx = __shfl_xor_sync(0xffffffffu, s.idx, o);
  return r;
}

// Warp reduction of one lane state's (ms, z, s1), m and idx left to the caller: every
// lane first moves to the warp's largest offset (one ex2, as LazyAcc::rescale), then
// plain fp64 sums — two independent 5-round trees instead of 5 rounds of combine() on
// the consumers' per-unit critical path.
__device__ __forceinline__ RowStat warp_reduce_offsets(RowStat s) {
  float MS = s.ms;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) MS = fmaxf(MS, __shfl_xor_sync(0xffffffffu, MS, o));
  shift_to(s, MS);
  double z = s.z, s1 = s.s1;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    z += __shfl_xor_sync(0xffffffffu, z, o);
    s1 += __shfl_xor_sync(0xffffffffu, s1, o);
  }
  s.z = z;
  s.s1 = s1;
  return s;
}

// The same with the maximum reduced too (the lanes' idx are not combined: callers
// resolve the argmax separately).
__device__ __forceinline__ RowStat warp_reduce_state(RowStat s) {
  float m = s.m;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  s = warp_reduce_offsets(s);
  s.m = m;
  return s;
}

// Block-wide reduction of RowStat; result valid in every thread.  smem: NT/32 entries.
template <int NT>
__device__ __forceinline__ RowStat block_reduce(RowStat s, RowStat* smem) {
  constexpr int NW = NT / 32;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s = combine(s, shfl_xor(s, o));
  if (lane == 0) smem[w] = s;
  __syncthreads();
  RowStat r = smem[0];
#pragma unroll
  for (int j = 1; j < NW; ++j) r = combine(r, smem[j]);
  __syncthreads();  // smem reusable after return
  return r;
}

// Stream one row [0, V) into a per-thread accumulator (vector path if vec_ok).
template <typename T, bool kQ, int NA, int NT, int U>
__device__ __forceinline__ void stream_row(const T* __restrict__ row, int V, bool vec_ok,
                                           RowAcc<kQ, NA>& acc) {
  constexpr int E = Vec<T>::E;
  const int tid = threadIdx.x;
  int done = 0;
  if (vec_ok) {
    const int nvec = V / E;
    const uint4* rv = reinterpret_cast<const uint4*>(row);
    const int full = nvec / (U * NT) * (U * NT);
    for (int vb = tid; vb < full; vb += U * NT) {
      uint4 x[U];
#pragma unroll
      for (int j = 0; j < U; ++j) x[j] = ldg_stream(rv + vb + j * NT);
#pragma unroll
      for (int j = 0; j < U; ++j) {
        float f[E];
        Vec<T>::unpack(x[j], f);
        acc.template add<E>(f, Vec<T>::vmax(f), (vb + j * NT) * E);
      }
    }
    for (int vb = full + tid; vb < nvec; vb += NT) {
      float f[E];
      Vec<T>::unpack(ldg_stream(rv + vb), f);
      acc.template add<E>(f, Vec<T>::vmax(f), vb * E);
    }
    done = nvec * E;
  }
  for (int v = done + tid; v < V; v += NT) acc.add1(ld_scalar(row + v), v);
}

// Two rows (p and q) interleaved so both streams keep loads in flight.
template <typename T, int NA, int NT, int U, bool kQq = true>
__device__ __forceinline__ void stream_pair(const T* __restrict__ prow, const T* __restrict__ qrow,
                                            int V, bool vec_ok, RowAcc<false, NA>& pa,
                                            RowAcc<kQq, NA>& qa) {
  constexpr int E = Vec<T>::E;
  const int tid = threadIdx.x;
  int done = 0;
  if (vec_ok) {
    const int nvec = V / E;
    const uint4* pv = reinterpret_cast<const uint4*>(prow);
    const uint4* qv = reinterpret_cast<const uint4*>(qrow);
    const int full = nvec / (U * NT) * (U * NT);
    for (int vb = tid; vb < full; vb += U * NT) {
      uint4 xp[U], xq[U];
#pragma unroll
      for (int j = 0; j < U; ++j) {
        xp[j] = ldg_stream(pv + vb + j * NT);
        xq[j] = ldg_stream(qv + vb + j * NT);
      }
#pragma unroll
      for (int j = 0; j < U; ++j) {
        float f[E];
        Vec<T>::unpack(xp[j], f);
        pa.template add<E>(f, Vec<T>::vmax(f), (vb + j * NT) * E);
        Vec<T>::unpack(xq[j], f);
        qa.template add<E>(f, Vec<T>::vmax(f), (vb + j * NT) * E);
      }
    }
    for (int vb = full + tid; vb < nvec; vb += NT) {
      float f[E];
      Vec<T>::unpack(ldg_stream(pv + vb), f);
      pa.template add<E>(f, Vec<T>::vmax(f), vb * E);
      Vec<T>::unpack(ldg_stream(qv + vb), f);
      qa.template add<E>(f, Vec<T>::vmax(f), vb * E);
    }
    done = nvec * E;
  }
  for (int v = done + tid; v < V; v += NT) {
    pa.add1(ld_scalar(prow + v), v);
    qa.add1(ld_scalar(qrow + v), v);
  }
}

// Final per-row quantities from a reduced state.  st classifies the row (include/
// specbranch.h "Input domain"): SB_ST_NONFINITE for a +inf entry or no finite entry
// (m = +-inf), SB_ST_RANGE for a finite maximum with |m| >= 2^24, SB_ST_NONFINITE for a
// NaN entry of an in-range row (z poisoned); only st == 0 rows have a distribution.
// (bf16 q rows: a clamped maximum of exactly -2^97 is reported SB_ST_RANGE here; the
// caller tells "all -inf" apart with row_has_finite().)
struct RowOut {
  float MS;     // exponent offset (log2 units) of Z
  double Z;     // sum 2^(l c - MS)
  int st;       // 0, SB_ST_NONFINITE or SB_ST_RANGE
  bool finite;  // st == 0: the row has a distribution
};
__device__ __forceinline__ int row_class(float m, double z) {
  if (m == CUDART_INF_F || m == -CUDART_INF_F) return SB_ST_NONFINITE;
  if (!(fabsf(m) < kLogitRange)) return m == m ? SB_ST_RANGE : SB_ST_NONFINITE;
  if (!(z > 0.0) || z == CUDART_INF) return SB_ST_NONFINITE;  // NaN entry (or no mass)
  return 0;
}
__device__ __forceinline__ RowOut finish(const RowStat& r) {
  RowOut o;
  o.MS = r.ms;
  o.Z = r.z;
  o.st = row_class(r.m, r.z);
  o.finite = (o.st == 0);
  return o;
}

// The normaliser as stored in the float4 row-state records (MS_p, Z_p, MS_q, Z_q): Z of
// an evaluated row, NaN for SB_ST_NONFINITE, -1 for SB_ST_RANGE; z_class() reads it back.
__device__ __forceinline__ float z_store(const RowOut& o) {
  return o.finite ? (float)o.Z : (o.st == SB_ST_RANGE ? -1.f : CUDART_NAN_F);
}
__device__ __forceinline__ int z_class(float z) {
  return z > 0.f ? 0 : (z == -1.f ? (int)SB_ST_RANGE : (int)SB_ST_NONFINITE);
}
// Per-token flag bits (workspace pflag): 1 accepted, 2 bad token, 4 / 8 the rows'
// SB_ST_NONFINITE / SB_ST_RANGE.
__device__ __forceinline__ uint8_t st_flags(int st) {
  return (uint8_t)(((st & SB_ST_NONFINITE) ? 4 : 0) | ((st & SB_ST_RANGE) ? 8 : 0));
}
__device__ __forceinline__ int flags_st(uint32_t f) {
  return ((f & 2u) ? (int)SB_ST_BAD_TOKEN : 0) | ((f & 4u) ? (int)SB_ST_NONFINITE : 0) |
         ((f & 8u) ? (int)SB_ST_RANGE : 0);
}

// Probability of one token from the row state, in fp64: 2^(l_x c - MS) / Z.
__device__ __forceinline__ double tok_prob(float lx, float MS, double Z) {
  const double arg = (double)lx * (double)kC - (double)MS;  // exact product in fp64
  return exp2(arg) / Z;
}

// Does a bf16 row hold any finite entry?  (The rare tie-break of a q row whose clamped
// maximum is -2^97: out of the input domain if so, all -inf otherwise.)  One warp, any
// alignment; returns the answer in every lane.
__device__ __forceinline__ bool row_has_finite_bf16(const __nv_bfloat16* row, int V) {
  const unsigned short* r = reinterpret_cast<const unsigned short*>(row);
  bool any = false;
  for (int v = threadIdx.x & 31; v < V && !any; v += 32) any = (__ldg(r + v) & 0x7f80u) != 0x7f80u;
  return __any_sync(0xffffffffu, any);
}

// The class of a q row reduced from clamped bf16 inputs (LazyAcc::add_bf16): a clamped
// maximum of exactly -2^97 means "outside the input domain" if the row holds a finite
// entry and "all -inf" otherwise (one warp re-reads the row; never on a real row).
// Warp-uniform call.
template <typename T>
__device__ __forceinline__ RowOut finish_q(const RowStat& qs, const T* qrow, int V) {
  RowOut qo = finish(qs);
  if constexpr (sizeof(T) == 2) {
    if (qs.m == kMaskedLogit && !row_has_finite_bf16(reinterpret_cast<const __nv_bfloat16*>(qrow), V)) {
      qo.st = SB_ST_NONFINITE;
      qo.finite = false;
    }
  }
  return qo;
}

// Warp-level inclusive scan (Kogge-Stone), fixed order.
__device__ __forceinline__ float warp_incl_scan(float x) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const float y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  return x;
}

}  // namespace sb
