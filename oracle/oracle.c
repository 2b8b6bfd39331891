/*
 * oracle.c — plain fp64 CPU oracle for the SpecBranch verify-and-branch step.
 *
 * TEST INFRASTRUCTURE ONLY (see oracle.h).  No blocking, fusion or reordering beyond
 * the plain definitions: every path row recomputes its own two-pass softmax, every
 * scan is linear, every cumulative sum is sequential in ascending token id.
 *
 * Citations: P<n> = /root/reference/PAPER.md line n, S<n> = SPEC.md line n.
 * Pins that hold it to the paper live in tests/test_oracle_*.py; parity for every
 * function here is pinned except where DESIGN.md says "parity unpinned"
 * (the K >= 2 output law of the Eq. 9 rule, which the paper does not fix).
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
static int omp_default_threads(void) { return omp_get_max_threads(); }
#else
static int omp_default_threads(void) { return 1; }
#endif

#define TIE_BAND 1e-6

static int64_t seq_stride_of(const or_dims* d) {
  return d->seq_stride ? d->seq_stride : (int64_t)d->K * (d->G + 1) * d->row_stride;
}

/* Exact widening of the input bytes: bf16 is the top half of an fp32. */
double oracle_logit(const or_dims* d, const void* L, int b, int slot, int i, int v) {
  int64_t off = (int64_t)b * seq_stride_of(d) + ((int64_t)slot * (d->G + 1) + i) * d->row_stride + v;
  if (d->dtype == OR_BF16) {
    uint32_t bits = (uint32_t)((const uint16_t*)L)[off] << 16;
    float f;
    memcpy(&f, &bits, sizeof f);
    return (double)f;
  }
  return (double)((const float*)L)[off];
}

/* Softmax of one row, plain two-pass definition (SURVEY §8.0 "Per-row definitions"):
 * m = max l, Z = sum exp(l - m), lse = m + ln Z, P(v) = exp(l(v) - m) / Z.
 * A row containing NaN or +inf, or whose entries are all -inf, has no distribution:
 * NaN.  (Terms with l = -inf add exp(-inf) = 0, SURVEY reading 20.) */
double oracle_row_softmax(const or_dims* d, const void* L, int b, int slot, int i, double* P) {
  const int V = d->V;
  double m = -INFINITY;
  for (int v = 0; v < V; ++v) {
    double l = oracle_logit(d, L, b, slot, i, v);
    if (isnan(l) || l == INFINITY) return NAN;
    if (l > m) m = l;
  }
  if (m == -INFINITY) return NAN; /* all entries -inf */
  double Z = 0.0;
  for (int v = 0; v < V; ++v) Z += exp(oracle_logit(d, L, b, slot, i, v) - m);
  double lse = m + log(Z);
  /* P = exp(l - m) / Z (not exp(l - lse): at |m| >> 1 the sum m + ln Z rounds ln Z away) */
  if (P)
    for (int v = 0; v < V; ++v) P[v] = exp(oracle_logit(d, L, b, slot, i, v) - m) / Z;
  return lse;
}

/* Input-domain validation (include/specbranch.h "Input domain", DESIGN reading 34) — a
 * precondition of the library, checked here as its own step before the softmax: the
 * maximum of the non-NaN entries must be finite with |m| < 2^24.  Order of the checks:
 * +inf entry or no finite entry -> NONFINITE; |m| >= 2^24 -> RANGE; NaN -> NONFINITE. */
uint32_t oracle_row_domain(const or_dims* d, const void* L, int b, int slot, int i) {
  double m = -INFINITY;
  int has_nan = 0, has_pinf = 0;
  for (int v = 0; v < d->V; ++v) {
    const double l = oracle_logit(d, L, b, slot, i, v);
    if (isnan(l)) has_nan = 1;
    else if (l == INFINITY) has_pinf = 1;
    else if (l > m) m = l;
  }
  if (has_pinf || m == -INFINITY) return OR_ST_NONFINITE;
  if (fabs(m) >= OR_LOGIT_RANGE) return OR_ST_RANGE;
  if (has_nan) return OR_ST_NONFINITE;
  return 0;
}

/* Validation, then the plain softmax of an in-domain row; NaN lse (and the status bit
 * in *st) for a row that is not evaluated. */
static double row_eval(const or_dims* d, const void* L, int b, int slot, int i, double* P, uint32_t* st) {
  const uint32_t dom = oracle_row_domain(d, L, b, slot, i);
  if (dom) {
    if (st) *st |= dom;
    return NAN;
  }
  return oracle_row_softmax(d, L, b, slot, i, P);
}

/* top-1 probability, smallest argmax id, entropy H = -sum Q ln Q (nats) of a q row
 * (§4.2 P170 "confidence max_x q(x)" and the entropy statistic; ties -> smaller id,
 * S393/S443). */
static void q_row_confidence(const or_dims* d, const void* QL, int b, int slot, int i,
                             const double* Q, double* top1, int32_t* top1_id, double* H) {
  double m = -INFINITY;
  int id = -1;
  for (int v = 0; v < d->V; ++v) {
    double l = oracle_logit(d, QL, b, slot, i, v);
    if (l > m) { m = l; id = v; }
  }
  double best = -1.0, h = 0.0;
  for (int v = 0; v < d->V; ++v) {
    if (Q[v] > best) best = Q[v];
    if (Q[v] > 0.0) h -= Q[v] * log(Q[v]);
  }
  *top1 = best;
  *top1_id = id;
  *H = h;
}

/* Inverse-CDF draw from the unnormalised non-negative vector r (SURVEY §8.0
 * "Inverse CDF"): F(j) = sum_{v<=j} r(v), t = us * R, j* = min{j : F(j) > t};
 * if rounding leaves t >= F(V-1), j* = max{v : r(v) > 0}.  Reports the distance of t
 * to the nearest CDF breakpoint adjacent to j* (the near-tie margin). */
static int inverse_cdf(const double* r, int V, double us, double* R_out, double* margin) {
  double R = 0.0;
  for (int v = 0; v < V; ++v) R += r[v];
  *R_out = R;
  double t = us * R, F = 0.0, Fprev = 0.0;
  int pick = -1;
  for (int v = 0; v < V; ++v) {
    Fprev = F;
    F += r[v];
    if (F > t) { pick = v; break; }
  }
  if (pick < 0) {
    for (int v = V - 1; v >= 0; --v)
      if (r[v] > 0.0) { pick = v; break; }
    *margin = 0.0;
    return pick;
  }
  double a = fabs(t - F), c = fabs(t - Fprev);
  *margin = a < c ? a : c;
  return pick;
}

static void verify_one(const or_dims* d, const void* PL, const void* QL, const int32_t* tok,
                       const double* u, const double* us, const int32_t* gamma,
                       const int32_t* branch_pos, int rule, or_verify_out* o, int b) {
  const int K = d->K, G = d->G, V = d->V, R1 = G + 1;
  uint32_t st = 0, ties = 0;
  double margin_acc = INFINITY, margin_sample = INFINITY;

  /* gamma_b in [0,G], s_b in [0,gamma_b] (SURVEY §8.0 Shapes); out of range -> clamp+flag */
  int g = gamma ? gamma[b] : G;
  if (g > G) { g = G; st |= OR_ST_GAMMA_CLAMPED; }
  if (g < 0) { g = 0; st |= OR_ST_GAMMA_CLAMPED; }
  int s = branch_pos ? branch_pos[b] : 0;
  if (s > g) { s = g; st |= OR_ST_BRANCH_CLAMPED; }
  if (s < 0) { s = 0; st |= OR_ST_BRANCH_CLAMPED; }
  /* path length: bonus row gamma_b verified next round if s_b < gamma_b; Alg.-1 form
   * (branch token at p_{gamma+1}, P538) if s_b == gamma_b */
  const int L = (s < g) ? g : g + 1;

  double* P = (double*)malloc(sizeof(double) * V);
  double* Q = (double*)malloc(sizeof(double) * V);
  double* r = (double*)malloc(sizeof(double) * V);

  /* sentinels */
  for (int k = 0; k < K; ++k)
    for (int i = 0; i < R1; ++i) {
      int64_t e = ((int64_t)b * K + k) * R1 + i;
      o->lse_p[e] = NAN; o->lse_q[e] = NAN; o->top1_q[e] = NAN; o->entropy_q[e] = NAN;
      o->top1_id_q[e] = -1; o->p_tok[e] = NAN; o->q_tok[e] = NAN;
    }

  /* Match along each branch path (P94; Alg. 1 P530-534; per-branch tests P538) */
  int32_t n[64];
  uint32_t mask[64];
  for (int k = 0; k < K; ++k) {
    mask[k] = 0;
    n[k] = L;
    for (int i = 0; i < L; ++i) {
      const int ls = (i <= s) ? 0 : k; /* logits shared up to the branch row (Eq. 7-8) */
      const int ts = (i < s) ? 0 : k;  /* own token and uniform from the branch row    */
      const int64_t er = ((int64_t)b * K + ls) * R1 + i; /* physical row entry  */
      const int64_t et = ((int64_t)b * K + ts) * R1 + i; /* token-slot entry    */
      double lse_p = row_eval(d, PL, b, ls, i, P, &st);
      double lse_q = row_eval(d, QL, b, ls, i, Q, &st);
      o->lse_p[er] = lse_p;
      o->lse_q[er] = lse_q;
      int acc = 0;
      if (isnan(lse_p) || isnan(lse_q)) {
        /* no distribution on one side: the test fails (reading 25); status set above */
      } else {
        q_row_confidence(d, QL, b, ls, i, Q, &o->top1_q[er], &o->top1_id_q[er], &o->entropy_q[er]);
        int x = tok[et];
        if (x < 0 || x >= V) {
          st |= OR_ST_BAD_TOKEN;
        } else {
          double Px = P[x], Qx = Q[x], ui = u[et];
          o->p_tok[et] = Px;
          o->q_tok[et] = Qx;
          /* accept iff r <= p/q (P534, P538), written u*Q[x] <= P[x]; Q[x] = 0 accepts (S127) */
          acc = (ui * Qx <= Px);
          if (Qx > 0.0) {
            double gap = fabs(ui - Px / Qx);
            if (gap < TIE_BAND) ties |= OR_TIE_ACC_MASK;
            if (n[k] == L && gap < margin_acc) margin_acc = gap; /* rows up to the first rejection */
            if (n[k] == L && gap < TIE_BAND) ties |= OR_TIE_ACC_DEC;
          }
        }
      }
      if (acc) mask[k] |= 1u << i;
      else if (n[k] == L) n[k] = i; /* first rejection: n_k = min{i : not acc} U {L} */
    }
    o->acc_mask[(int64_t)b * K + k] = mask[k];
    o->n_acc[(int64_t)b * K + k] = n[k];
  }

  /* Branch-point verification and selection (Eq. 9, P236-241; Alg. 1 P540) */
  int ksel = -1;
  double bestkey = 0.0;
  int besttok = 0;
  for (int k = 0; k < K; ++k) {
    if (n[k] <= s) continue; /* A = {k : n_k > s_b}: branch token accepted */
    int xk = tok[((int64_t)b * K + k) * R1 + s];
    double key = (rule == 1) ? (double)u[((int64_t)b * K + k) * R1 + s]
                             : oracle_logit(d, PL, b, 0, s, xk); /* raw target logit */
    int better;
    if (ksel < 0) better = 1;
    else if (rule == 1) better = key > bestkey;
    else better = key > bestkey || (key == bestkey && xk < besttok);
    if (better) { ksel = k; bestkey = key; besttok = xk; }
  }

  /* Commit (SURVEY §8.0 "Commit"): path tokens, then y from residual or bonus */
  int npath, yrow = -1, yslot = 0, ykind = 0, kpath;
  if (ksel < 0) {
    kpath = 0;
    npath = n[0] < s ? n[0] : s; /* rejection in the shared prefix or at the branch row (P655) */
    yrow = npath; yslot = 0; ykind = 1;
  } else {
    kpath = ksel;
    npath = n[ksel];
    if (npath < L) { yrow = npath; yslot = (npath <= s) ? 0 : ksel; ykind = 1; }
    else if (s < g) { yrow = g; yslot = ksel; ykind = 2; } /* bonus from p_{gamma+1} (P94) */
    else ykind = 0; /* branch token accepted; continuation carried by the caller (P237) */
  }

  int32_t* out = o->out_tok + (int64_t)b * (G + 2);
  for (int i = 0; i < G + 2; ++i) out[i] = -1;
  for (int k = 0; k < K; ++k) o->keep_mask[(int64_t)b * K + k] = 0;
  for (int i = 0; i < npath; ++i) {
    int ts = (i < s) ? 0 : kpath;
    out[i] = tok[((int64_t)b * K + ts) * R1 + i];
    o->keep_mask[(int64_t)b * K + ts] |= 1u << i;
  }

  int y = -1;
  double mass = 0.0;
  if (ykind != 0) {
    double lp = row_eval(d, PL, b, yslot, yrow, P, &st);
    double lq = (ykind == 1) ? row_eval(d, QL, b, yslot, yrow, Q, &st) : 0.0;
    if (isnan(lp) || isnan(lq)) {
      ykind = 0;
    } else {
      /* norm(max(0, p - q)) at the first rejected position (P94, P554); bonus: p */
      for (int v = 0; v < V; ++v) r[v] = (ykind == 1) ? fmax(0.0, P[v] - Q[v]) : P[v];
      double R = 0.0, mg = 0.0;
      for (int v = 0; v < V; ++v) R += r[v];
      if (ykind == 1 && R == 0.0) { /* "no residual mass" (S134-140): fall back to p */
        st |= OR_ST_ZERO_RESID;
        for (int v = 0; v < V; ++v) r[v] = P[v];
      }
      y = inverse_cdf(r, V, us[b], &R, &mg);
      mass = R;
      margin_sample = mg;
      if (mg < TIE_BAND) ties |= OR_TIE_SAMPLE;
      if (ykind == 1 && R < 1e-4) ties |= OR_TIE_ILLCOND;
    }
  }
  if (ykind != 0) out[npath] = y;

  o->sel_k[b] = ksel;
  o->commit_len[b] = npath + (ykind != 0);
  o->y_tok[b] = (ykind != 0) ? y : -1;
  o->y_kind[b] = ykind;
  o->path_rolled[b] = L - npath;            /* paper's RB numerator (P317) */
  o->branch_discarded[b] = (K - 1) * (L - s); /* excluded from RB (P734)   */
  o->resid_mass[b] = mass;
  o->status[b] = (int32_t)st;
  o->ties[b] = ties;
  o->margin_acc[b] = margin_acc;
  o->margin_sample[b] = margin_sample;
  free(P); free(Q); free(r);
}

static int dims_ok(const or_dims* d) {
  return d && d->B >= 1 && d->K >= 1 && d->K <= 64 && d->G >= 0 && d->G <= 31 && d->V >= 2 &&
         d->row_stride >= d->V && (d->dtype == OR_BF16 || d->dtype == OR_F32);
}

int oracle_verify_f64u(const or_dims* d, const void* PL, const void* QL, const int32_t* tok,
                       const double* u, const double* us, const int32_t* gamma,
                       const int32_t* branch_pos, int rule, int nthreads, or_verify_out* o) {
  if (!dims_ok(d) || !PL || !QL || !tok || !u || !us || !o) return -1;
#pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads > 0 ? nthreads : omp_default_threads())
  for (int b = 0; b < d->B; ++b) verify_one(d, PL, QL, tok, u, us, gamma, branch_pos, rule, o, b);
  /* exclusive scan of commit_len and the packed commit stream */
  o->offsets[0] = 0;
  for (int b = 0; b < d->B; ++b) o->offsets[b + 1] = o->offsets[b] + o->commit_len[b];
  if (o->packed_tok)
    for (int b = 0; b < d->B; ++b)
      for (int i = 0; i < o->commit_len[b]; ++i)
        o->packed_tok[o->offsets[b] + i] = o->out_tok[(int64_t)b * (d->G + 2) + i];
  return 0;
}

int oracle_verify(const or_dims* d, const void* PL, const void* QL, const int32_t* tok,
                  const float* u, const float* us, const int32_t* gamma,
                  const int32_t* branch_pos, int rule, int nthreads, or_verify_out* o) {
  if (!dims_ok(d) || !u || !us) return -1;
  const int64_t n = (int64_t)d->B * d->K * (d->G + 1);
  double* ud = (double*)malloc(sizeof(double) * n);
  double* usd = (double*)malloc(sizeof(double) * d->B);
  for (int64_t e = 0; e < n; ++e) ud[e] = (double)u[e]; /* exact widening */
  for (int b = 0; b < d->B; ++b) usd[b] = (double)us[b];
  int rc = oracle_verify_f64u(d, PL, QL, tok, ud, usd, gamma, branch_pos, rule, nthreads, o);
  free(ud); free(usd);
  return rc;
}

int oracle_adaptive_k(double c, int k_max) {
  double k = floor((double)k_max * (1.0 - c)); /* Eq. 7, P218 */
  return k < 1.0 ? 1 : (int)k;
}

int oracle_confidence(const or_dims* d, const void* QL, const int32_t* tok, int mode,
                      double eps, double lambda, int k_max, int nthreads, or_conf_out* o) {
  if (!dims_ok(d) || !QL || !o || (mode == 1 && !tok) || mode < 0 || mode > 2) return -1;
  const int K = d->K, G = d->G, R1 = G + 1, V = d->V;
#pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads > 0 ? nthreads : omp_default_threads())
  for (int bk = 0; bk < d->B * K; ++bk) {
    const int b = bk / K, k = bk % K;
    double* Q = (double*)malloc(sizeof(double) * V);
    int stop = G;
    uint32_t ties = 0;
    for (int i = 0; i < G; ++i) {
      const int64_t e = ((int64_t)b * K + k) * G + i;
      double lse = row_eval(d, QL, b, k, i, Q, NULL);
      double top1 = NAN, H = NAN, tp = NAN, stat = NAN;
      int32_t id = -1;
      if (!isnan(lse)) {
        q_row_confidence(d, QL, b, k, i, Q, &top1, &id, &H);
        if (tok) {
          int x = tok[((int64_t)b * K + k) * R1 + i];
          tp = (x >= 0 && x < V) ? Q[x] : NAN;
        }
        if (mode == 0) stat = top1;                     /* max_x q(x) (P170, P954) */
        else if (mode == 1) stat = tp;                  /* q(x_i) (Eq. 6 P198)     */
        else stat = 1.0 - sqrt(lambda * H);             /* AdaEDL form (P170)      */
      }
      o->top1_prob[e] = top1; o->top1_id[e] = id; o->entropy[e] = H;
      o->tok_prob[e] = tp; o->stat[e] = stat;
      if (stop == G) {
        if (!isnan(stat) && fabs(stat - eps) < TIE_BAND) ties |= OR_TIE_CONF;
        if (stat <= eps) stop = i; /* Eq. 6 keeps q(x) > eps: stop at the first <= eps */
      }
    }
    int kn = -1;
    if (stop < G) {
      const int64_t e = ((int64_t)b * K + k) * G + stop;
      double c = (mode == 1) ? o->tok_prob[e] : o->top1_prob[e];
      double a = (double)k_max * (1.0 - c);
      if (fabs(a - nearbyint(a)) < TIE_BAND) ties |= OR_TIE_EQ7;
      kn = oracle_adaptive_k(c, k_max);
    }
    o->stop[bk] = stop;
    o->k_next[bk] = kn;
    o->gamma_next[bk] = stop > 1 ? stop : 1;
    o->ties[bk] = ties;
    free(Q);
  }
  return 0;
}

/* Eq. 7 branch spawn, plain (k_b argmax scans over the fp64 draft distribution). */
int oracle_spawn(const or_dims* d, const void* QL, const int32_t* branch_pos, const int32_t* tok,
                 int mode, int k_max, int nthreads, or_spawn_out* o) {
  if (!dims_ok(d) || !QL || !o || k_max < 1 || (mode == 1 && !tok) || mode < 0 || mode > 1) return -1;
  const int V = d->V, R1 = d->G + 1;
#pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads > 0 ? nthreads : omp_default_threads())
  for (int b = 0; b < d->B; ++b) {
    int s = branch_pos ? branch_pos[b] : 0;
    if (s < 0) s = 0;
    if (s > d->G) s = d->G;
    double* Q = (double*)malloc(sizeof(double) * V);
    char* taken = (char*)calloc(V, 1);
    for (int j = 0; j < k_max; ++j) {
      o->btok[(int64_t)b * k_max + j] = -1;
      o->bprob[(int64_t)b * k_max + j] = NAN;
    }
    double lse = row_eval(d, QL, b, 0, s, Q, NULL);
    uint32_t ties = 0;
    int k = 0;
    double c = NAN;
    if (!isnan(lse)) {
      if (mode == 0) {
        c = -1.0;
        for (int v = 0; v < V; ++v)
          if (Q[v] > c) c = Q[v];
      } else {
        const int x = tok[((int64_t)b * d->K + 0) * R1 + s];
        c = (x >= 0 && x < V) ? Q[x] : NAN;
      }
      if (!isnan(c)) {
        const double a = (double)k_max * (1.0 - c);
        if (fabs(a - nearbyint(a)) < TIE_BAND) ties |= OR_TIE_EQ7;
        k = oracle_adaptive_k(c, k_max); /* Eq. 7 */
        if (k > V) k = V;
        for (int j = 0; j < k; ++j) { /* TopK(q(x_b), k): highest q, ties -> smaller id */
          int best = -1;
          for (int v = 0; v < V; ++v)
            if (!taken[v] && (best < 0 || Q[v] > Q[best])) best = v;
          taken[best] = 1;
          o->btok[(int64_t)b * k_max + j] = best;
          o->bprob[(int64_t)b * k_max + j] = Q[best];
        }
      }
    }
    o->k[b] = k;
    o->conf[b] = c;
    o->ties[b] = ties;
    free(Q);
    free(taken);
  }
  return 0;
}

/* Tree verify, one sequence (oracle.h; R31).  Every context row that is read
 * gets its own two-pass softmax; children are scanned linearly in node order. */
static void tree_one(const or_dims* d, const void* PL, const void* QL, const int32_t* parent,
                     const int32_t* tok, const float* u, const float* us, or_tree_out* o, int b) {
  const int N = d->G, V = d->V;
  const int32_t* par = parent + (int64_t)b * N;
  const int32_t* tk = tok + (int64_t)b * N;
  const float* ub = u + (int64_t)b * N;
  uint32_t st = 0, ties = 0;
  double* P = (double*)malloc(sizeof(double) * V);
  double* Q = (double*)malloc(sizeof(double) * V);
  double* r = (double*)malloc(sizeof(double) * V);
  uint64_t acc = 0;
  double* gap = (double*)malloc(sizeof(double) * (N + 1));
  /* the Match test of every node against its parent's context row (P94, P538) */
  for (int j = 0; j < N; ++j) {
    gap[j] = INFINITY;
    const int pj = par[j];
    if (pj < -1 || pj >= j) { st |= OR_ST_BAD_PARENT; continue; }
    const int row = pj + 1;
    double lp = row_eval(d, PL, b, 0, row, P, &st);
    double lq = row_eval(d, QL, b, 0, row, Q, &st);
    if (isnan(lp) || isnan(lq)) continue;
    const int x = tk[j];
    if (x < 0 || x >= V) { st |= OR_ST_BAD_TOKEN; continue; }
    const double ui = (double)ub[j];
    if (ui * Q[x] <= P[x]) acc |= 1ull << j; /* Q[x] = 0 accepts (S127) */
    if (Q[x] > 0.0) gap[j] = fabs(ui - P[x] / Q[x]);
  }
  /* the walk: Eq. 9 at every node, no backtracking */
  int c = -1, npath = 0;
  uint64_t keep = 0;
  int32_t* out = o->out_tok + (int64_t)b * (N + 1);
  for (int i = 0; i <= N; ++i) out[i] = -1;
  for (;;) {
    int best = -1, has_child = 0;
    for (int j = 0; j < N; ++j) {
      if (par[j] != c || par[j] >= j) continue;
      has_child = 1;
      if (gap[j] < TIE_BAND) ties |= OR_TIE_ACC_DEC; /* every child of a walked node decides */
      if (!((acc >> j) & 1)) continue;
      if (best < 0) { best = j; continue; }
      const double kj = oracle_logit(d, PL, b, 0, c + 1, tk[j]);
      const double kb = oracle_logit(d, PL, b, 0, c + 1, tk[best]);
      if (kj > kb || (kj == kb && tk[j] < tk[best])) best = j; /* raw target logit (P241) */
    }
    if (best < 0) {
      /* y from row c+1: residual if c has children (all rejected), else bonus */
      int ykind = has_child ? 1 : 2, y = -1;
      double mass = 0.0;
      double lp = row_eval(d, PL, b, 0, c + 1, P, &st);
      double lq = ykind == 1 ? row_eval(d, QL, b, 0, c + 1, Q, &st) : 0.0;
      if (isnan(lp) || isnan(lq)) {
        ykind = 0;
      } else {
        for (int v = 0; v < V; ++v) r[v] = (ykind == 1) ? fmax(0.0, P[v] - Q[v]) : P[v];
        double R = 0.0, mg = 0.0;
        for (int v = 0; v < V; ++v) R += r[v];
        if (ykind == 1 && R == 0.0) {
          st |= OR_ST_ZERO_RESID;
          for (int v = 0; v < V; ++v) r[v] = P[v];
        }
        y = inverse_cdf(r, V, (double)us[b], &R, &mg);
        mass = R;
        if (mg < TIE_BAND) ties |= OR_TIE_SAMPLE;
        if (ykind == 1 && R < 1e-4) ties |= OR_TIE_ILLCOND;
      }
      if (ykind != 0) out[npath] = y;
      o->stop_node[b] = c;
      o->commit_len[b] = npath + (ykind != 0);
      o->y_tok[b] = ykind ? y : -1;
      o->y_kind[b] = ykind;
      o->resid_mass[b] = mass;
      break;
    }
    out[npath++] = tk[best];
    keep |= 1ull << best;
    c = best;
  }
  o->acc_mask[b] = acc;
  o->keep_mask[b] = keep;
  o->status[b] = (int32_t)st;
  o->ties[b] = ties;
  free(P); free(Q); free(r); free(gap);
}

int oracle_tree_verify(const or_dims* d, const void* PL, const void* QL, const int32_t* parent,
                       const int32_t* tok, const float* u, const float* us, int nthreads, or_tree_out* o) {
  if (!d || d->K != 1 || d->G < 1 || d->G > 63 || d->V < 2 || d->row_stride < d->V ||
      (d->dtype != OR_BF16 && d->dtype != OR_F32) || !PL || !QL || !parent || !tok || !u || !us || !o)
    return -1;
#pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads > 0 ? nthreads : omp_default_threads())
  for (int b = 0; b < d->B; ++b) tree_one(d, PL, QL, parent, tok, u, us, o, b);
  return 0;
}

/* ---------------------------------------------------------------- H-RAD (f4)
 * Eq. 4-5 (P190-191) with the architecture of P745 (two hidden layers of 256 and 64
 * ReLU units, a 3-way classification layer; dropout is a training-time operation and
 * absent at inference):
 *   h1 = relu(W1 z + b1), h2 = relu(W2 h1 + b2), l = W3 h2 + b3,
 *   s_t = argmax softmax(l) = argmax l (softmax is monotone; ties -> smaller class).
 * H_t (P194-201, read with the stage-transition cases of P669, DESIGN reading 35):
 *   s_t = 0 (all reject)  -> gamma_b = 0,    s_b = 0     (branch at this round's first token)
 *   s_t = 1 (confidence)  -> gamma_b = stop, s_b = stop  (branch at the first q(x) <= eps)
 *   s_t = 2 (all accept)  -> gamma_b = G,    s_b = G     (branch at the next round's first token)
 * z and W1 are the exact bf16 bytes (widened exactly), the rest fp32; all sums fp64,
 * in index order.  margin[b] = l(best) - l(second) (the near-tie distance). */
static double bf16_to_double(uint16_t h) {
  uint32_t bits = (uint32_t)h << 16;
  float f;
  memcpy(&f, &bits, sizeof f);
  return (double)f;
}

int oracle_hrad(int B, int Dz, const uint16_t* z, const uint16_t* w1, const float* b1, const float* w2,
                const float* b2, const float* w3, const float* b3, const int32_t* stop, int G, int nthreads,
                double* h1_out, double* logits, int32_t* s_t, int32_t* gamma, int32_t* branch_pos,
                double* margin) {
  if (B < 1 || Dz < 1 || !z || !w1 || !b1 || !w2 || !b2 || !w3 || !b3 || !logits || !s_t || G < 0)
    return -1;
#pragma omp parallel for schedule(dynamic, 8) num_threads(nthreads > 0 ? nthreads : omp_default_threads())
  for (int b = 0; b < B; ++b) {
    double h1[256], h2[64], l[3];
    for (int j = 0; j < 256; ++j) {
      double acc = 0.0;
      for (int c = 0; c < Dz; ++c)
        acc += bf16_to_double(w1[(int64_t)j * Dz + c]) * bf16_to_double(z[(int64_t)b * Dz + c]);
      acc += (double)b1[j];
      h1[j] = acc > 0.0 ? acc : 0.0;
      if (h1_out) h1_out[(int64_t)b * 256 + j] = h1[j];
    }
    for (int j = 0; j < 64; ++j) {
      double acc = 0.0;
      for (int c = 0; c < 256; ++c) acc += (double)w2[j * 256 + c] * h1[c];
      acc += (double)b2[j];
      h2[j] = acc > 0.0 ? acc : 0.0;
    }
    for (int k = 0; k < 3; ++k) {
      double acc = 0.0;
      for (int c = 0; c < 64; ++c) acc += (double)w3[k * 64 + c] * h2[c];
      l[k] = acc + (double)b3[k];
      logits[(int64_t)b * 3 + k] = l[k];
    }
    int best = 0;
    for (int k = 1; k < 3; ++k)
      if (l[k] > l[best]) best = k;
    double second = -INFINITY;
    for (int k = 0; k < 3; ++k)
      if (k != best && l[k] > second) second = l[k];
    if (margin) margin[b] = l[best] - second;
    s_t[b] = best;
    if (gamma && branch_pos) {
      int st = stop ? stop[b] : G;
      if (st < 0) st = 0;
      if (st > G) st = G;
      const int g = best == 0 ? 0 : (best == 1 ? st : G);
      gamma[b] = g;
      branch_pos[b] = g;
    }
  }
  return 0;
}
