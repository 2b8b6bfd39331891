/*
 * oracle.h — plain, slow, fp64 CPU oracle for the SpecBranch verify-and-branch step.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load or call this library.  The product
 * path (paper_2506_01979_b200/, libspecbranch.so) never links, imports or executes it,
 * and this file shares no code, header, table or constant with the CUDA path.
 *
 * What it computes is the plain definition of SURVEY.md §8.0, which restates:
 *   - §3 "Speculative Decoding", PAPER.md P94: beta = min(1, p/q), Match, residual
 *     norm(max(0, p - q)) at the first rejected position, bonus token from p_{gamma+1};
 *   - Algorithm 1 VERIFICATION branch, PAPER.md P523-557 (n = min{i-1 : r_i > p_i/q_i}
 *     U {gamma}; branch check P538; b* P540; residual P547/P554);
 *   - Eq. 9 branch-point verification, PAPER.md P236-241 (argmax p over Match-accepted
 *     branches, "maximum logits" P241);
 *   - Eq. 6 confidence filter q(x) > eps, PAPER.md P194-202, and the implicit
 *     statistics of §4.2 P170 (max_x q(x), 1 - sqrt(lambda H));
 *   - Eq. 7 adaptive branch count k = max(1, floor(k_max (1 - q(x_b)))), P218.
 * Every reading the paper leaves open is listed in DESIGN.md §"Readings".
 *
 * Everything is fp64, two-pass softmax, linear scans, sequential cumulative sums.
 * Inputs are the exact bytes the GPU path consumes (bf16 or fp32 logits, widened
 * exactly to double).  OpenMP is used across independent sequences only (timing).
 */
#ifndef SB_ORACLE_H
#define SB_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OR_BF16 0
#define OR_F32 1

/* status bits (same meaning as the library's, defined independently here) */
#define OR_ST_GAMMA_CLAMPED 1u  /* gamma_b > G  -> clamped to G                  */
#define OR_ST_BRANCH_CLAMPED 2u /* s_b > gamma_b or < 0 -> clamped               */
#define OR_ST_BAD_TOKEN 4u      /* a path token outside [0, V): counted rejected */
#define OR_ST_NONFINITE 8u      /* a row read has +inf, no finite entry, or NaN  */
#define OR_ST_ZERO_RESID 16u    /* residual mass R == 0 after a rejection -> P   */
#define OR_ST_BAD_PARENT 32u    /* tree: parent[j] outside [-1, j): node rejected */
#define OR_ST_RANGE 64u         /* a row read is outside the input domain        */

/* Input-domain validation (a separate, explicit step before any softmax; the library's
 * documented precondition, include/specbranch.h "Input domain"): the maximum m of the
 * row's non-NaN entries must be finite with |m| < 2^24.  Returns 0 (in domain),
 * OR_ST_NONFINITE (+inf entry, or no finite entry, or NaN in an in-range row) or
 * OR_ST_RANGE (finite maximum with |m| >= 2^24).  Rows that fail are not evaluated: the
 * contract gives them NaN outputs and the status bit; oracle_row_softmax itself is the
 * plain definition and is never bent to the kernel. */
#define OR_LOGIT_RANGE 16777216.0 /* 2^24 */

/* near-tie flags (oracle only): the decision is within the fp32 error band */
#define OR_TIE_ACC_MASK 1u  /* |u - P/Q| < 1e-6 at some tested row             */
#define OR_TIE_ACC_DEC 2u   /* ... at a row that decides some n_k (i <= n_k)   */
#define OR_TIE_SAMPLE 4u    /* |t - F(j*)| or |t - F(j*-1)| < 1e-6 (mass)      */
#define OR_TIE_ILLCOND 8u   /* R < 1e-4                                        */
#define OR_TIE_CONF 16u     /* |stat - eps| < 1e-6                             */
#define OR_TIE_EQ7 32u      /* k_max (1 - c) within 1e-6 of an integer         */

typedef struct {
  int32_t B, K, G, V;   /* G = gamma_max; V = vocabulary columns               */
  int64_t row_stride;   /* elements between consecutive rows (>= V)            */
  int64_t seq_stride;   /* elements between sequences; 0 -> K*(G+1)*row_stride */
  int32_t dtype;        /* OR_BF16 (raw uint16 bf16) or OR_F32                 */
  int32_t pad_;
} or_dims;

/* Outputs of one verify-and-branch round.  Index conventions:
 *   row arrays  [B][K][G+1] at physical logit rows (b, ls(k,i), i), NaN / -1 elsewhere;
 *   path arrays [B][K][G+1] at token slots (b, ts(k,i), i), NaN elsewhere. */
typedef struct {
  double *lse_p, *lse_q;          /* row arrays                                  */
  double *top1_q, *entropy_q;     /* row arrays (q rows)                         */
  int32_t *top1_id_q;             /* row array                                   */
  double *p_tok, *q_tok;          /* path arrays: P_i[x], Q_i[x]                 */
  uint32_t *acc_mask;             /* [B][K] bit i = acc(k, i), i < L_b           */
  int32_t *n_acc;                 /* [B][K]                                      */
  int32_t *sel_k;                 /* [B] k* or -1                                */
  int32_t *commit_len;            /* [B]                                         */
  int32_t *out_tok;               /* [B][G+2], -1 padded                         */
  int32_t *y_tok, *y_kind;        /* [B]; kind 0 none, 1 residual, 2 bonus       */
  int32_t *offsets;               /* [B+1] exclusive scan of commit_len          */
  int32_t *packed_tok;            /* [sum commit_len]                            */
  int32_t *path_rolled;           /* [B] L_b - n                                 */
  int32_t *branch_discarded;      /* [B] (K-1)(L_b - s_b)                        */
  uint32_t *keep_mask;            /* [B][K] committed draft positions per slot   */
  double *resid_mass;             /* [B] mass of the sampled distribution        */
  int32_t *status;                /* [B]                                         */
  uint32_t *ties;                 /* [B] OR_TIE_* flags                          */
  double *margin_acc;             /* [B] min |u - P/Q| over deciding rows        */
  double *margin_sample;          /* [B] min distance of t to a CDF breakpoint   */
} or_verify_out;

/* Outputs of the draft-confidence statistic over rows 0..G-1 of each (b,k) group. */
typedef struct {
  double *top1_prob;    /* [B][K][G]    max_x q(x)                  (P170, P954)   */
  int32_t *top1_id;     /* [B][K][G]    smallest argmax id                          */
  double *entropy;      /* [B][K][G]    H = -sum q ln q (nats)      (P170)         */
  double *tok_prob;     /* [B][K][G]    q(x_i) of the drafted token (P198, P517)   */
  double *stat;         /* [B][K][G]    the statistic compared with eps            */
  int32_t *stop;        /* [B][K]       min{i : stat_i <= eps} U {G}   (Eq. 6)     */
  int32_t *k_next;      /* [B][K]       Eq. 7 at the stop row; -1 if stop == G     */
  int32_t *gamma_next;  /* [B][K]       max(1, stop)                               */
  uint32_t *ties;       /* [B][K]       OR_TIE_CONF | OR_TIE_EQ7                    */
} or_conf_out;

/* Widen one logit to double exactly. */
double oracle_logit(const or_dims* d, const void* L, int b, int slot, int i, int v);

/* Softmax of one physical row in fp64 (two passes): writes P[V] and returns lse.
 * Plain definition: NaN lse for a row holding NaN or +inf, or whose entries are all
 * -inf (no distribution); every other row, at any magnitude, gets its softmax. */
double oracle_row_softmax(const or_dims* d, const void* L, int b, int slot, int i, double* P);

/* The input-domain validation above for one row: 0, OR_ST_NONFINITE or OR_ST_RANGE. */
uint32_t oracle_row_domain(const or_dims* d, const void* L, int b, int slot, int i);

/* One verify-and-branch round for all B sequences; uniforms in fp32
 * (widened exactly).  rule: 0 = Eq. 9 (default), 1 = Algorithm 1 argmax r_b.
 * nthreads <= 0 -> OpenMP default.  Returns 0, or -1 on invalid arguments. */
int oracle_verify(const or_dims* d, const void* PL, const void* QL, const int32_t* tok,
                  const float* u, const float* us, const int32_t* gamma,
                  const int32_t* branch_pos, int rule, int nthreads, or_verify_out* o);

/* Same, with the uniforms given in fp64 (used by the exact enumeration pins). */
int oracle_verify_f64u(const or_dims* d, const void* PL, const void* QL, const int32_t* tok,
                       const double* u, const double* us, const int32_t* gamma,
                       const int32_t* branch_pos, int rule, int nthreads, or_verify_out* o);

/* Draft confidence over rows 0..G-1 of every (b,k) group of q logits.
 * mode: 0 TOP1 (max q), 1 TOKEN (q(x_i), needs tok), 2 ENTROPY (1 - sqrt(lambda H)). */
int oracle_confidence(const or_dims* d, const void* QL, const int32_t* tok, int mode,
                      double eps, double lambda, int k_max, int nthreads, or_conf_out* o);

/* Eq. 7 alone (for the SPEC pins): max(1, floor(k_max (1 - c))). */
int oracle_adaptive_k(double c, int k_max);

/* Branch spawn (Eq. 7 P216-220): at the branch row s_b of slot 0,
 * c = q(x_b) (mode 0: max_x q(x); mode 1: q of tok[b][0][s_b]),
 * k_b = min(V, max(1, floor(k_max (1 - c)))), and the k_b tokens of highest q
 * (ties -> smaller id, S393), found by k_b plain argmax scans. */
typedef struct {
  int32_t *k;       /* [B]                                   */
  int32_t *btok;    /* [B][k_max], -1 padded                 */
  double *bprob;    /* [B][k_max], NaN padded                */
  double *conf;     /* [B] c = q(x_b)                        */
  uint32_t *ties;   /* [B] OR_TIE_EQ7                        */
} or_spawn_out;
int oracle_spawn(const or_dims* d, const void* QL, const int32_t* branch_pos, const int32_t* tok,
                 int mode, int k_max, int nthreads, or_spawn_out* o);

/* Tree-structured verify (the dense-tree structure of Appendix F,
 * P1057, that the paper compares against), read as Eq. 9 applied at every node
 * (reading R31).  Per sequence: N draft nodes j with token tok[j], parent
 * parent[j] in [-1, j) (-1 = the committed context), uniform u[j].  Logit rows are
 * contexts: row 0 = the committed context, row j+1 = the context after node j; d->K
 * must be 1 and d->G = N (rows [B][N+1]).
 *   acc(j)  = u_j Q_r[x_j] <= P_r[x_j], r = parent[j] + 1            (P94 Match, P538)
 *   walk:   c = -1; while some child of c is accepted: c = the accepted child of
 *           largest raw target logit P-logit_r[x_j] (ties: smaller token, smaller j)
 *                                                                   (Eq. 9, P236-241)
 *   commit: the path's tokens, then y from row c+1: norm(max(0, p - q)) if c has a
 *           child (all rejected), else the bonus p (c is a leaf).     (P94, P554) */
typedef struct {
  uint64_t *acc_mask;   /* [B] bit j = acc(j)                               */
  uint64_t *keep_mask;  /* [B] bit j = node j is on the committed path      */
  int32_t *stop_node;   /* [B] c (-1 = the root)                            */
  int32_t *commit_len;  /* [B] path length + [y]                            */
  int32_t *out_tok;     /* [B][N+1] path tokens, then y; -1 padded          */
  int32_t *y_tok, *y_kind; /* [B] kind 1 residual, 2 bonus, 0 none (bad row) */
  double *resid_mass;   /* [B]                                              */
  int32_t *status;      /* [B] OR_ST_*                                      */
  uint32_t *ties;       /* [B] OR_TIE_ACC_DEC | OR_TIE_SAMPLE | OR_TIE_ILLCOND */
} or_tree_out;
int oracle_tree_verify(const or_dims* d, const void* PL, const void* QL, const int32_t* parent,
                       const int32_t* tok, const float* u, const float* us, int nthreads, or_tree_out* o);

/* H-RAD MLP (Eq. 4-5 P190-191, architecture P745, H_t P194-201 with
 * the cases of P669): z [B][Dz] and W1 [256][Dz] raw bf16, b1 [256], W2 [64][256],
 * b2 [64], W3 [3][64], b3 [3] fp32; stop [B] (a6's confidence stop, may be NULL -> G).
 * Outputs: h1 [B][256] (may be NULL), logits [B][3], s_t [B], gamma / branch_pos [B]
 * (may be NULL), margin [B] (top-2 logit gap, may be NULL). */
int oracle_hrad(int B, int Dz, const uint16_t* z, const uint16_t* w1, const float* b1, const float* w2,
                const float* b2, const float* w3, const float* b3, const int32_t* stop, int G, int nthreads,
                double* h1_out, double* logits, int32_t* s_t, int32_t* gamma, int32_t* branch_pos,
                double* margin);

#ifdef __cplusplus
}
#endif
#endif
