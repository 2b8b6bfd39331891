/*
 * specbranch.h — C ABI of the B200 (sm_100a) verify-and-branch step of SpecBranch
 * (arXiv 2506.01979).  Library: paper_2506_01979_b200/libspecbranch.so.
 *
 * Citations: P<n> = PAPER.md line n (the paper), S<n> = SPEC.md line n, SURVEY §8.0 =
 * the contract restated from those passages.  DESIGN.md lists every reading taken
 * where the paper is silent or ambiguous.
 *
 * Problem statement the arguments follow (Alg. 1 inputs P480-492, §3 P94, Eq. 7 P218,
 * Eq. 9 P239): target logits p and draft logits q for B sequences x K branches x
 * (G+1) rows, the draft tokens (including the K branch tokens at the branch row), the
 * per-position uniforms r_i ~ U(0,1) (P531), the draft length gamma_b, the branch row
 * s_b, and the confidence threshold eps / k_max of Eq. 6-7.
 *
 * Conventions common to every entry point
 *   - All array pointers are DEVICE pointers, caller-owned (e.g. torch tensors), and
 *     must stay valid until the stream work completes.  The library allocates nothing
 *     and never synchronises the host; every call is stream-ordered on `stream`.
 *   - Layouts (row-major, 0-based):
 *       logits  [B][K][G+1][row_stride]  element (b,slot,i,v) at
 *               b*seq_stride + (slot*(G+1) + i)*row_stride + v   (bf16 or fp32)
 *       tok     int32 [B][K][G+1]   token of branch slot k at row i (ts map below)
 *       u       fp32  [B][K][G+1]   uniforms in [0,1) at the same slots as tok
 *       "row arrays"  [B][K][G+1] indexed by the physical logit row (b, ls(k,i), i)
 *       "path arrays" [B][K][G+1] indexed by the token slot      (b, ts(k,i), i)
 *     Slot maps (Eq. 7-8 P218-222, Alg. 1 P538):
 *       ls(k,i) = (i <= s_b) ? 0 : k     rows up to the branch row share slot 0
 *       ts(k,i) = (i <  s_b) ? 0 : k     each branch owns its token/uniform from s_b on
 *     Path length L_b = gamma_b if s_b < gamma_b (bonus row gamma_b), else gamma_b + 1
 *     (Algorithm-1 form: the branch token sits at the target's p_{gamma+1}, P538).
 *   - Entries of row / path arrays that are not on any tested path are written NaN
 *     (float) or -1 (int).  Rows >= L_b are never read.
 *   - Host-checkable argument errors return SB_ERR_INVALID_ARG before any launch.
 *     Data errors found on the device never fail the call: they are clamped or
 *     skipped and reported per sequence in status[b] (SB_ST_* bits).
 *   - workspace: device buffer of sb_workspace_bytes(d) bytes, 256-byte aligned, that
 *     must be ZERO-FILLED before its first use; every call leaves it re-usable.  The
 *     same workspace must be passed to sb_select_branch after sb_verify_branches (it
 *     carries the per-row softmax state between them) and must not be shared by calls
 *     in flight on different streams.
 *   - Functions are stateless apart from `workspace` and thread-safe across streams.
 *   - Input domain (precondition on every logit row the call reads): the row's maximum
 *     logit m (NaN entries ignored) is finite with |m| < 2^24 (SB_LOGIT_RANGE).  Entries
 *     below the maximum are unrestricted: -inf, -FLT_MAX or finfo(bf16).min masks
 *     contribute exactly 0, as in the plain definition softmax(l)_v = exp(l_v - m) / Z.
 *     Why: the kernels evaluate every term as 2^(l c - fl(m c)) in fp32 (c = log2 e),
 *     exact up to the rounding of fl(m c), which stays below one unit of the exponent
 *     only while |m| < 2^24.  A row outside the domain is not evaluated: its row / path
 *     outputs are NaN (as for a row with no distribution) and SB_ST_RANGE is set.  A
 *     row holding +inf, no finite entry (all -inf), or NaN (in-range rows) sets
 *     SB_ST_NONFINITE instead.  (Real logits lie within a few hundred of 0.)
 */
#ifndef SPECBRANCH_H
#define SPECBRANCH_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SB_LOGIT_RANGE 16777216.0f /* 2^24: input domain bound on |row maximum| (above) */

typedef struct CUstream_st* sb_stream_t; /* identical to cudaStream_t; NULL = default */

typedef enum {
  SB_OK = 0,
  SB_ERR_INVALID_ARG = 1, /* bad dims, null required pointer, misaligned workspace   */
  SB_ERR_UNSUPPORTED = 2, /* valid request this build does not implement            */
  SB_ERR_CUDA = 3,        /* a CUDA launch or runtime call failed                   */
  SB_ERR_NCCL = 4,        /* an NCCL call of the vocabulary-sharded exchange failed */
  SB_ERR_WORKSPACE = 5    /* workspace_bytes < sb_workspace_bytes(d)                */
} sb_status;

typedef enum { SB_BF16 = 0, SB_F32 = 1 } sb_dtype;
typedef enum { SB_SELECT_EQ9 = 0, SB_SELECT_ALG1 = 1 } sb_select_rule;
typedef enum { SB_CONF_TOP1 = 0, SB_CONF_TOKEN = 1, SB_CONF_ENTROPY = 2 } sb_conf_mode;

/* per-sequence status bits (status[b]) */
#define SB_ST_GAMMA_CLAMPED 1u  /* gamma_b outside [0,G]: clamped                        */
#define SB_ST_BRANCH_CLAMPED 2u /* s_b outside [0,gamma_b]: clamped                      */
#define SB_ST_BAD_TOKEN 4u      /* a path token outside [0,V): that test counts rejected */
#define SB_ST_NONFINITE 8u      /* a row read holds +inf, no finite entry, or (in-range
                                   rows) a NaN: it has no distribution                  */
#define SB_ST_ZERO_RESID 16u    /* residual mass R == 0 after a rejection: sampled from p */
#define SB_ST_BAD_PARENT 32u    /* tree: parent[j] outside [-1, j): node j counts rejected */
#define SB_ST_RANGE 64u         /* a row read violates the input domain (below): its
                                   maximum is finite with |max| >= 2^24; not evaluated  */

typedef struct {
  int32_t B;          /* sequences, >= 1                                              */
  int32_t K;          /* branch slots, 1..32                                          */
  int32_t G;          /* gamma_max, 0..31 (rows per slot = G+1)                       */
  int32_t V;          /* vocabulary columns, >= 2                                     */
  int32_t v_offset;   /* vocabulary shard offset; unsharded: 0                        */
  int32_t v_total;    /* full vocabulary (token ids are global); unsharded: V or 0    */
  int64_t row_stride; /* elements between rows, >= V                                  */
  int64_t seq_stride; /* elements between sequences; 0 -> K*(G+1)*row_stride         */
  int32_t dtype;      /* sb_dtype of the logits                                       */
  int32_t reserved;   /* must be 0                                                    */
} sb_dims;

/* Library version string, and a static message for a status code. */
const char* sb_version(void);
const char* sb_status_string(sb_status s);

/* Device bytes the caller must provide as `workspace` for dims d (0 if d invalid). */
size_t sb_workspace_bytes(const sb_dims* d);

/*
 * sb_verify_branches — row statistics, acceptance test and first rejection.
 *   (§3 P94 beta = min(1, p/q) and Match; Alg. 1 P523-534; branch tests P538)
 *
 * For every physical row pair (p row, q row) on a tested path — slot 0 rows
 * 0..min(s_b, L_b-1), plus rows s_b+1..L_b-1 of every slot — computes in one streaming
 * pass: lse = m + ln sum exp(l - m) of both rows, and for the q row the top-1
 * probability, its smallest id and the entropy H = -sum q ln q in nats (§4.2 P170).
 * Then for every path token x through the row: P[x], Q[x] and the acceptance bit
 * acc = (u * Q[x] <= P[x])   (accept iff r <= p/q, P534/P538; Q[x] = 0 accepts, S127),
 * and per branch k the accepted prefix n_k = min({i < L_b : !acc(k,i)} U {L_b}).
 *
 * Inputs : p_logits, q_logits  logits (layout above);
 *          tok, u              path tokens / uniforms [B][K][G+1];
 *          gamma               [B] draft lengths, NULL -> G for all;
 *          branch_pos          [B] branch rows s_b, NULL -> 0 for all.
 * Outputs: lse_p, lse_q        row arrays (natural log);
 *          top1_q, top1_id_q, entropy_q  row arrays (q rows), each nullable;
 *          p_tok, q_tok        path arrays, P_i[x], Q_i[x];
 *          acc_mask            [B][K] uint32, bit i = acc(k,i) for i < L_b;
 *          n_acc               [B][K] accepted prefix lengths;
 *          status              [B] SB_ST_* bits (overwritten).
 * comm: NULL for an unsharded call; a communicator from sb_comm_create for a vocabulary
 * shard (d->v_offset / d->v_total describe this rank's slice): the library then runs
 * sb_shard_verify_local, an NCCL all-gather of the partials and sb_shard_verify_combine
 * on `stream` (a7).  Sharded dims without a communicator are SB_ERR_INVALID_ARG.
 */
typedef struct sb_comm sb_comm; /* opaque NCCL communicator of the vocabulary-shard ranks */

sb_status sb_verify_branches(const sb_dims* d, const void* p_logits, const void* q_logits,
                             const int32_t* tok, const float* u, const int32_t* gamma,
                             const int32_t* branch_pos, float* lse_p, float* lse_q,
                             float* p_tok, float* q_tok, uint32_t* acc_mask, int32_t* n_acc,
                             float* top1_q, int32_t* top1_id_q, float* entropy_q,
                             int32_t* status, void* comm, void* workspace,
                             size_t workspace_bytes, sb_stream_t stream);

/*
 * sb_select_branch — branch-point verification, correction/bonus sample, commit.
 *   (Eq. 9 P236-241; Alg. 1 P536-557; residual P94/P547/P554; rollback P655; RB P317/P734)
 *
 * Per sequence b with A = {k : n_k > s_b}:
 *   SB_SELECT_EQ9  k* = argmax_{k in A} p_logits[b][0][s_b][tok[b][k][s_b]] (raw target
 *                  logits = argmax p within the row, "maximum logits" P241); ties ->
 *                  smaller token id, then smaller k;
 *   SB_SELECT_ALG1 k* = argmax_{k in A} u[b][k][s_b], ties -> smaller k (P540).
 *   A empty: k* = -1; commit tok[b][0][0..j-1], j = min(n_0, s_b), and y drawn from
 *            norm(max(0, P_j - Q_j)) of slot 0 (P547, P554, P655).
 *   else n = n_{k*}: commit k*'s path tokens 0..n-1, then
 *            n <  L_b            -> y ~ norm(max(0, P_n - Q_n)) at row n of slot ls(k*,n);
 *            n == L_b, s_b<gamma -> y ~ P_{gamma_b} of slot k* (bonus, P94);
 *            n == L_b, s_b==gamma-> no y (branch token accepted, P237).
 *   Sampling: inverse CDF over ascending token id with the one uniform us[b]:
 *   j* = min{j : F(j) > us*R}, F(j) = sum_{v<=j} r(v); if rounding leaves us*R >= F(V-1)
 *   the last v with r(v) > 0.  R == 0 after a rejection samples from P instead
 *   (SB_ST_ZERO_RESID; SPEC "no residual mass", S134-140).
 *
 * Inputs : p_logits, q_logits, tok, u as for sb_verify_branches; us [B] in [0,1);
 *          gamma, branch_pos as before; n_acc from sb_verify_branches; rule.
 * Outputs: sel_k [B] (k* or -1); commit_len [B]; out_tok [B][G+2] committed tokens
 *          (-1 padded); y_tok [B] (-1 none); y_kind [B] (0 none, 1 residual, 2 bonus);
 *          offsets [B+1] exclusive scan of commit_len; packed_tok [B*(G+2)] nullable,
 *          the commits concatenated at offsets; path_rolled [B] = L_b - n (RB
 *          numerator, P317); branch_discarded [B] = (K-1)(L_b - s_b) (excluded from RB,
 *          P734); keep_mask [B][K] bit i of slot k set iff the draft token at (k,i) is
 *          committed (the KV rows to keep, P241); resid_mass [B] nullable, the mass R of
 *          the sampled vector (1 for a bonus, 0 for none); status [B] (bits OR-ed in).
 * comm: as for sb_verify_branches (sharded: local masses, NCCL all-gather, owner
 * sample, NCCL all-reduce MAX of the token, commit).
 */
sb_status sb_select_branch(const sb_dims* d, const void* p_logits, const void* q_logits,
                           const int32_t* tok, const float* u, const float* us,
                           const int32_t* gamma, const int32_t* branch_pos,
                           const int32_t* n_acc, sb_select_rule rule, int32_t* sel_k,
                           int32_t* commit_len, int32_t* out_tok, int32_t* y_tok,
                           int32_t* y_kind, int32_t* offsets, int32_t* packed_tok,
                           int32_t* path_rolled, int32_t* branch_discarded,
                           uint32_t* keep_mask, float* resid_mass, int32_t* status,
                           void* comm, void* workspace, size_t workspace_bytes,
                           sb_stream_t stream);

/*
 * sb_verify_select — sb_verify_branches followed by sb_select_branch: every output of
 * both calls, with the same meaning, in one call (one workspace, one stream).  The two
 * streaming kernels run back to back (PDL-chained).  Experiment switches (environment):
 * SB_FUSED_STEP=1 runs the single persistent TMA-ring launch k_step_tma, SB_ASTEP=1 the
 * persistent work-queue launch k_astep with plan items (both correct, both measured
 * slower on B200).  Unsharded only.
 */
sb_status sb_verify_select(const sb_dims* d, const void* p_logits, const void* q_logits,
                           const int32_t* tok, const float* u, const float* us,
                           const int32_t* gamma, const int32_t* branch_pos, sb_select_rule rule,
                           float* lse_p, float* lse_q, float* p_tok, float* q_tok,
                           uint32_t* acc_mask, int32_t* n_acc, float* top1_q, int32_t* top1_id_q,
                           float* entropy_q, int32_t* status, int32_t* sel_k, int32_t* commit_len,
                           int32_t* out_tok, int32_t* y_tok, int32_t* y_kind, int32_t* offsets,
                           int32_t* packed_tok, int32_t* path_rolled, int32_t* branch_discarded,
                           uint32_t* keep_mask, float* resid_mass, void* workspace,
                           size_t workspace_bytes, sb_stream_t stream);

/*
 * sb_step_adaptive — the whole adaptive-gamma step in one call:
 * sb_draft_confidence on the slot-0 draft rows (SB_CONF_TOP1, lambda unused, Eq. 6 stop
 * with eps, Eq. 7 k with k_max), gamma_b = max(1, stop_b) (written to c_gamma_next), then
 * sb_verify_branches and sb_select_branch with that gamma and branch_pos.  Every output
 * has the meaning of the corresponding call (c_* arrays [B][G] / [B] as sb_draft_confidence
 * with K = 1).  Small problems (16-byte aligned rows of 16-byte multiples up to 1 MB,
 * B * K * (G+1) <= 4096) run as ONE persistent launch (k_astep: confidence items, then
 * each sequence's verify items as soon as its gamma is known, then its sample item as
 * soon as its n_k is known; SB_ASTEP=0 / 1 forces it off / on); larger ones as the three
 * streaming kernels, the verify reusing the confidence pass's row states.  All CTAs of
 * the persistent launch must be co-resident (one per SM; SB_ERR_UNSUPPORTED if the
 * occupancy check fails).  conf_workspace: sb_workspace_bytes of the slot-0
 * dims (K = 1, seq_stride of d), zero-filled once; workspace: sb_workspace_bytes(d).
 * Errors as the three calls; G must be >= 1.
 */
sb_status sb_step_adaptive(const sb_dims* d, const void* p_logits, const void* q_logits, const int32_t* tok,
                           const float* u, const float* us, const int32_t* branch_pos, sb_select_rule rule,
                           float eps, int32_t k_max, float* c_top1_prob, int32_t* c_top1_id, float* c_entropy,
                           float* c_stat, int32_t* c_stop, int32_t* c_k_next, int32_t* c_gamma_next, float* lse_p,
                           float* lse_q, float* p_tok, float* q_tok, uint32_t* acc_mask, int32_t* n_acc,
                           float* top1_q, int32_t* top1_id_q, float* entropy_q, int32_t* status, int32_t* sel_k,
                           int32_t* commit_len, int32_t* out_tok, int32_t* y_tok, int32_t* y_kind,
                           int32_t* offsets, int32_t* packed_tok, int32_t* path_rolled,
                           int32_t* branch_discarded, uint32_t* keep_mask, float* resid_mass,
                           void* conf_workspace, size_t conf_workspace_bytes, void* workspace,
                           size_t workspace_bytes, sb_stream_t stream);

/*
 * sb_verify_branches_reuse — sb_verify_branches for the adaptive-gamma step (SURVEY §8.4
 * C2/C3): conf_workspace is the workspace of a preceding sb_draft_confidence call on the
 * slot-0 view of the same q_logits (K = 1, seq_stride = this call's sequence stride,
 * same B, G, V, row_stride, dtype; e.g. api.conf_dims(d)).  That call already streamed
 * draft rows 0..G-1 of slot 0 and left their reduced softmax state in its workspace;
 * this call reads those states back instead of re-reading the rows (only their p rows
 * and the token logits are read).  Outputs and errors as sb_verify_branches; the q
 * statistics of those rows come from the confidence pass (same arithmetic, a
 * different summation order: within the 1e-5 tolerance, not bit-identical).  Not for
 * vocabulary shards (SB_ERR_INVALID_ARG).
 */
sb_status sb_verify_branches_reuse(const sb_dims* d, const void* p_logits, const void* q_logits,
                                   const int32_t* tok, const float* u, const int32_t* gamma,
                                   const int32_t* branch_pos, float* lse_p, float* lse_q, float* p_tok,
                                   float* q_tok, uint32_t* acc_mask, int32_t* n_acc, float* top1_q,
                                   int32_t* top1_id_q, float* entropy_q, int32_t* status,
                                   const void* conf_workspace, void* workspace, size_t workspace_bytes,
                                   sb_stream_t stream);

/*
 * sb_draft_confidence — the implicit draft-confidence statistic and adaptive gamma.
 *   (§4.2 P170; Eq. 6 P194-202; Eq. 7 P218; Alg. 1 P517; App. E.6 P954/P965)
 *
 * Over rows i = 0..G-1 of every (b,k) group of q_logits:
 *   top1_prob = max_x q(x), top1_id (smallest), entropy H (nats), tok_prob = q(x_i)
 *   of tok[b][k][i] (TOKEN mode; nullable otherwise), and
 *   stat_i = top1_prob (TOP1) | tok_prob (TOKEN) | 1 - sqrt(lambda * H) (ENTROPY);
 *   stop = min({i : stat_i <= eps} U {G})   (Eq. 6 keeps q(x) > eps);
 *   k_next = max(1, floor(k_max (1 - c))) with c the top-1 (TOKEN: token) probability
 *   at the stop row (Eq. 7), -1 when stop == G;  gamma_next = max(1, stop).
 * Output arrays [B][K][G] (rows) and [B][K] (groups); all but stop nullable.
 * To score only slot 0 of a [B][K'][G+1] tensor pass K = 1 and seq_stride of K'.
 */
sb_status sb_draft_confidence(const sb_dims* d, const void* q_logits, const int32_t* tok,
                              sb_conf_mode mode, float eps, float lambda, int32_t k_max,
                              float* top1_prob, int32_t* top1_id, float* entropy,
                              float* tok_prob, float* stat, int32_t* stop, int32_t* k_next,
                              int32_t* gamma_next, void* comm, void* workspace,
                              size_t workspace_bytes, sb_stream_t stream);

/*
 * sb_spawn_branches — branch spawn at the branch point (Eq. 7 P216-220).
 * For each sequence, on the shared draft row s_b of slot 0 (branch_pos, NULL -> 0):
 *   c = q(x_b): max_x q(x) (SB_CONF_TOP1) or q of tok[b][0][s_b] (SB_CONF_TOKEN);
 *   k_b = min(V, max(1, floor(k_max (1 - c))))  (Eq. 7, k_max <= 16);
 *   branch_tok[b][0..k_b) = TopK(q(x_b), k_b) in descending q, ties -> smaller id (S393),
 *   -1 padded to k_max; branch_prob the matching q (nullable); conf[b] = c (nullable).
 * A non-finite row gives k_b = 0.  The tokens feed tok[b][k][s_b] of the next verify.
 */
sb_status sb_spawn_branches(const sb_dims* d, const void* q_logits, const int32_t* branch_pos,
                            const int32_t* tok, sb_conf_mode mode, int32_t k_max, int32_t* k_out,
                            int32_t* branch_tok, float* branch_prob, float* conf,
                            sb_stream_t stream);

/*
 * sb_kv_rollback — keep the surviving branch's draft KV rows (P241,
 * shared-prefix KV P220).  kv: the draft KV of the round, [B][K][G+1] positions of
 * row_bytes each (16-byte multiple) at row_stride_bytes, token-slot layout (as tok).
 * keep_mask [B][K] (device, from sb_select_branch): bit i of keep_mask[b][k] set iff the
 * draft token at slot k, position i is committed; at most one slot per position (the
 * slot ts(k*, i) = (i < s_b ? 0 : k*) of the clamped layout, slot 0 when k* = -1).
 *   out_kv != NULL: out_kv[b][i] (layout [B][G+1] at row_stride_bytes) = that row;
 *   out_kv == NULL: in place, kept rows of slots k > 0 are moved into slot 0.
 * Positions with no kept bit are not touched (the rolled-back positions).
 * Errors: SB_ERR_INVALID_ARG (dims, NULL kv / keep_mask, row sizes or pointers not
 * 16-byte multiples / aligned), SB_ERR_CUDA (launch).
 */
sb_status sb_kv_rollback(int32_t B, int32_t K, int32_t G, const void* kv, int64_t row_bytes,
                         int64_t row_stride_bytes, const uint32_t* keep_mask, void* out_kv,
                         sb_stream_t stream);

/*
 * sb_tree_verify — token-tree verification (the dense-tree structure of
 * Appendix F, P1057/P1073), read as Eq. 9 (P236-241) applied at every node
 * (R31).  Per sequence: N = d->G draft nodes (1 <= N <= 63, d->K must be 1),
 * node j with token tok[b][j], parent[b][j] in [-1, j) (-1 = the committed context;
 * topological order), uniform u[b][j]; us[b] for the sample.  Logit rows are contexts,
 * [B][N+1][row_stride] (seq_stride 0 -> (N+1)*row_stride): row 0 = the committed context,
 * row j+1 = the context after node j.  The q row of a childless context is never read.
 *   acc(j) = u_j Q_r[x_j] <= P_r[x_j], r = parent[j] + 1                        (P94)
 *   walk:  c = -1; while a child of c is accepted, c = the accepted child of largest
 *          raw target logit at row c+1 (ties: smaller token, then smaller j)   (Eq. 9)
 *   y:     from row c+1, residual norm(max(0,p-q)) if c has a child, else bonus p.
 * Outputs (device, overwritten): acc_mask [B] (bit j = acc(j)), keep_mask [B] (bit j =
 * node j committed), stop_node [B] (c), commit_len [B], out_tok [B][N+1] (path tokens,
 * y, -1 padded), y_tok, y_kind [B] (1 residual, 2 bonus, 0 none), resid_mass [B] (may be
 * NULL), status [B] (SB_ST_*).  workspace: >= sb_tree_workspace_bytes(d), 16-byte aligned.
 * Errors: SB_ERR_INVALID_ARG (dims / pointers), SB_ERR_WORKSPACE, SB_ERR_UNSUPPORTED
 * (V too large for the sampler's tile table), SB_ERR_CUDA (launch).
 */
size_t sb_tree_workspace_bytes(const sb_dims* d);
sb_status sb_tree_verify(const sb_dims* d, const void* p_logits, const void* q_logits, const int32_t* parent,
                         const int32_t* tok, const float* u, const float* us, uint64_t* acc_mask,
                         uint64_t* keep_mask, int32_t* stop_node, int32_t* commit_len, int32_t* out_tok,
                         int32_t* y_tok, int32_t* y_kind, float* resid_mass, int32_t* status, void* workspace,
                         size_t workspace_bytes, sb_stream_t stream);

/*
 * sb_hrad_predict — H-RAD draft-length predictor inference: the
 * lightweight MLP of Eq. 4-5 (P190-191) with the architecture of P745 and the hybrid
 * strategy H_t (P194-201) mapped onto this library's branch layout (P669; DESIGN.md
 * reading 35):
 *   h1 = relu(W1 z + b1), h2 = relu(W2 h1 + b2), l = W3 h2 + b3, s_t = argmax l
 *   (softmax is monotone; ties -> smaller class); (gamma_b, branch_pos_b) =
 *   (0, 0) if s_t = 0 (all reject), (stop_b, stop_b) if s_t = 1 (confidence; stop_b
 *   from sb_draft_confidence, clamped to [0, G]; NULL stop -> G), (G, G) if s_t = 2.
 * z: [B][Dz] bf16 row-major (features Concat(h^1..h^4, e_t), Eq. 4), w1: [256][Dz] bf16,
 * b1 [256], w2 [64][256], b2 [64], w3 [3][64], b3 [3] fp32 — all device pointers,
 * caller-owned, z / w1 / b1 / w2 16-byte aligned.  Outputs (device, overwritten): s_t [B];
 * logits [B][3], gamma [B], branch_pos [B] may be NULL.  Layer 1 runs on the tensor
 * cores (tcgen05, fp32 accumulation, split along K; the split partials — the
 * workspace, sb_hrad_workspace_bytes(B, Dz) bytes, 16-byte aligned, no initialisation
 * needed — are summed in a fixed order, so results are run-to-run deterministic);
 * layers 2-3 in fp32.  Errors: SB_ERR_INVALID_ARG (B < 1, G outside [0, 31], NULL
 * required pointer), SB_ERR_UNSUPPORTED (Dz not a multiple of 64, misaligned z / w1 / b1 / w2),
 * SB_ERR_WORKSPACE (too small), SB_ERR_CUDA (tensor-map encode or launch).
 * Stream-ordered, no host synchronisation.
 */
size_t sb_hrad_workspace_bytes(int32_t B, int32_t Dz);
sb_status sb_hrad_predict(int32_t B, int32_t Dz, int32_t G, const void* z, const void* w1, const float* b1,
                          const float* w2, const float* b2, const float* w3, const float* b3,
                          const int32_t* stop, float* logits, int32_t* s_t, int32_t* gamma,
                          int32_t* branch_pos, void* workspace, size_t workspace_bytes,
                          sb_stream_t stream);

/*
 * ---- Vocabulary-sharded variant (a7) ----------------------
 * Rank g of G holds the contiguous slice [v_offset, v_offset + V) of the v_total-token
 * vocabulary; slices are in rank order (so global ascending-id order = rank order).
 * tok (global ids), u, us, gamma, branch_pos are identical on every rank.  All outputs
 * are identical on every rank (decisions are replicated after each exchange).  The
 * split-phase calls let a caller run the three exchanges itself (tests use an
 * in-process loopback); sb_comm_* + the comm argument above run them with NCCL.
 *
 *   1. sb_shard_verify_local   -> partial (sb_shard_partial_bytes bytes, device)
 *      exchange: all-gather the G partials, rank-major, contiguous
 *   2. sb_shard_verify_combine -> the sb_verify_branches outputs
 *   3. sb_shard_select_local   -> mass [B][2] fp64 (this shard's residual and p mass)
 *      exchange: all-gather the G mass arrays, rank-major -> gathered_mass [G][B][2]
 *   4. sb_shard_select_sample  -> ycand [B] (the sampled global id on the owner, -1 else)
 *      exchange: all-reduce MAX of ycand -> y
 *   5. sb_shard_select_commit  -> the sb_select_branch outputs
 * The same workspace (sized by sb_workspace_bytes of the shard dims) must be used by
 * all five calls of one round.  In sharded mode the verify phase also reads every
 * branch's bonus row (statistics only) so that the sample needs no extra exchange.
 */
size_t sb_shard_partial_bytes(const sb_dims* d);
sb_status sb_shard_verify_local(const sb_dims* d, const void* p_logits, const void* q_logits,
                                const int32_t* tok, const float* u, const int32_t* gamma,
                                const int32_t* branch_pos, void* partial, void* workspace,
                                size_t workspace_bytes, sb_stream_t stream);
sb_status sb_shard_verify_combine(const sb_dims* d, const void* gathered, int32_t nranks,
                                  const int32_t* tok, const float* u, float* lse_p, float* lse_q,
                                  float* p_tok, float* q_tok, uint32_t* acc_mask, int32_t* n_acc,
                                  float* top1_q, int32_t* top1_id_q, float* entropy_q,
                                  int32_t* status, void* workspace, size_t workspace_bytes,
                                  sb_stream_t stream);
sb_status sb_shard_select_local(const sb_dims* d, const void* p_logits, const void* q_logits,
                                const int32_t* tok, const float* u, const int32_t* n_acc,
                                sb_select_rule rule, double* mass, void* workspace,
                                size_t workspace_bytes, sb_stream_t stream);
sb_status sb_shard_select_sample(const sb_dims* d, const double* gathered_mass, int32_t nranks,
                                 int32_t rank, const void* p_logits, const void* q_logits,
                                 const float* us, int32_t* ycand, void* workspace,
                                 size_t workspace_bytes, sb_stream_t stream);
sb_status sb_shard_select_commit(const sb_dims* d, const int32_t* y, const int32_t* tok,
                                 int32_t* sel_k, int32_t* commit_len, int32_t* out_tok,
                                 int32_t* y_tok, int32_t* y_kind, int32_t* offsets,
                                 int32_t* packed_tok, int32_t* path_rolled,
                                 int32_t* branch_discarded, uint32_t* keep_mask,
                                 float* resid_mass, int32_t* status, void* workspace,
                                 size_t workspace_bytes, sb_stream_t stream);

/* NCCL communicator of the G shard ranks (one process per GPU).  Rank 0 creates the
 * unique id (sb_comm_unique_id, sb_comm_unique_id_bytes() bytes, host memory) and the
 * caller broadcasts it (e.g. with torch.distributed); every rank then calls
 * sb_comm_create with the largest dims it will use (scratch is allocated here, never
 * on the hot path).  sb_comm_destroy frees it. */
size_t sb_comm_unique_id_bytes(void);
sb_status sb_comm_unique_id(void* unique_id_out);
sb_status sb_comm_create(const void* unique_id, int32_t nranks, int32_t rank,
                         const sb_dims* max_dims, sb_comm** out);
sb_status sb_comm_destroy(sb_comm* comm);
/* Failure detection: SB_ERR_NCCL if the communicator has recorded an
 * asynchronous NCCL error (ncclCommGetAsyncError; a failed peer or link), SB_OK
 * otherwise.  Host-only, never blocks.  The sharded calls perform the same check before
 * enqueueing their collectives.  After SB_ERR_NCCL the communicator is unusable:
 * sb_comm_abort (ncclCommAbort) releases it without waiting for pending collectives,
 * which sb_comm_destroy would. */
sb_status sb_comm_check(sb_comm* comm);
sb_status sb_comm_abort(sb_comm* comm);

#ifdef __cplusplus
}
#endif
#endif /* SPECBRANCH_H */
