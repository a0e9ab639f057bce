/*
 * propd.h — C ABI of libpropd.so, the B200 (sm_100a) kernels of the batched
 * ProPD token-tree decode step.
 *
 * Conventions
 *   - Every pointer is a DEVICE pointer unless its name ends in _host.
 *   - `stream` is a cudaStream_t passed as void*; every call is asynchronous
 *     on that stream and allocates nothing persistent.
 *   - Return value: 0 on success; nonzero on a launch/argument error, with a
 *     message available from propd_last_error() (thread-local).  The Python
 *     host layer raises ValueError/RuntimeError from it.
 *   - dtype codes: PROPD_F32 = 0 (fp32 parity mode), PROPD_BF16 = 1.
 *   - KV cache layout per layer: [slot][head][Lmax][dh], so one (sequence,
 *     head) K or V block is a contiguous [Lmax, dh] tile.  Tree nodes of the
 *     current pass live at slots seq_len[slot] + node (original tree index).
 *   - Tree templates are shared by every sequence of a step (the tree SHAPE
 *     is global per step, engine.py:246): parent[n], depth[n], rank[n] and an
 *     ancestor bitset mask[n][W], W = ceil(n/64).
 *
 * Reference interfaces replaced (paths relative to
 * /root/reference/pkg/src/treedecode/):
 *   ModelBackend.forward_tree / commit / draft / next_argmax  backends.py:53-95
 *   TinyTransformer._block (attention + projections)           backends.py:202-237
 *   build_tree / make_mask / positions                         token_tree.py:125-185, engine.py:260
 *   prune (+ early head top-K)                                 pruning.py:40-66, backends.py:320-327
 *   verify + commit                                            verification.py:30-53, backends.py:337-348
 *   AcceptanceStats.update + select_best_nodes                 acceptance.py:96-113, 186-206
 */
#ifndef PROPD_H
#define PROPD_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PROPD_F32 0
#define PROPD_BF16 1

/* Last error message of the calling thread ("" if none). */
const char* propd_last_error(void);
/* ABI version; bumped on any signature change. */
int propd_abi_version(void);
/* Number of SMs of the current device (0 if no device). */
int propd_num_sms(void);
/* One-time kernel attribute setup and occupancy queries (the weight-streaming
 * GEMM's grid barriers are only launched when every CTA can be co-resident);
 * call before capturing CUDA graphs. */
int propd_prepare(void);
/* Largest grid of a weight-streaming launch with in-kernel phases (grid
 * barriers) whose CTAs are all resident at once on this device: resident CTAs
 * per SM (computed from the kernel's resources, confirmed by a bounded probe
 * launch in propd_prepare) x SMs.  0 if the probe failed to run. */
int propd_gemm_ws_barrier_ctas(void);
/* Measurement hook (bench.py in-step view): install (buf) or remove (NULL) a
 * device buffer that receives one timeline record per CTA of the GEMM and
 * attention kernels (layout in csrc/common.cuh).  Off by default. */
int propd_debug_timeline(void* buf);

/* ---- K1: tree materialisation (token_tree.py:125-170, engine.py:260) ----
 * For sequence b and template node i (row m = b*n + i):
 *   tokens[m]    = draft_tok[b][depth[i]-1][rank[i]-1]
 *   positions[m] = seq_len[seq_slot[b]] + depth[i] - 1
 *   x[m,:]       = emb[tokens[m]] + pos[positions[m]]        (fp32 residual)
 *   row_seq[m] = b, row_node[m] = i, row_off[b] = b*n (row_off[B] = B*n).   */
int propd_tree_embed(int dtype, int B, int n, int D, int kmax, int H,
                     const int32_t* depth, const int32_t* rank, const int32_t* draft_tok,
                     const int32_t* seq_slot, const int32_t* seq_len,
                     const void* emb, const void* pos,
                     int32_t* tokens, int32_t* positions, float* x,
                     int32_t* row_seq, int32_t* row_node, int32_t* row_off, void* stream);

/* Generic row embedding: x[m] = emb[tokens[m]] + pos[positions[m]]. */
int propd_embed_rows(int dtype, int M, int H, const int32_t* tokens, const int32_t* positions,
                     const void* emb, const void* pos, float* x, void* stream);

/* Bonus rows (one per sequence): tokens[b] = bonus[b],
 * positions[b] = seq_len[seq_slot[b]], x[b] = emb + pos; row_seq[b] = b,
 * row_node[b] = 0, row_off[b] = b. */
int propd_bonus_embed(int dtype, int B, int H, const int32_t* bonus, const int32_t* seq_slot,
                      const int32_t* seq_len, const void* emb, const void* pos, float* x,
                      int32_t* positions, int32_t* row_seq, int32_t* row_node, int32_t* row_off,
                      void* stream);

/* ---- dense helpers (backends.py:135-142, 216, 234-236) ----
 * x += delta (if delta != NULL, dtype-typed); out = LN(x) (no affine, eps 1e-5,
 * population variance).  in_idx/out_idx (nullable) gather/scatter rows:
 * row m reads x[in_idx ? in_idx[m] : m], writes out[out_idx ? out_idx[m] : m].
 * When delta is given the residual update is written back to x (in place).
 * rows_dev (nullable, device int32; also on argmax_rows / qkv_finish /
 * gelu_finish): only rows m < *rows_dev are processed — the live row count of
 * a pass launched for a padded capacity M. */
int propd_add_ln(int dtype, int M, const int32_t* rows_dev, int H, float* x, const void* delta, void* out,
                 const int32_t* in_idx, const int32_t* out_idx, void* stream);
/* In-place tanh-GELU over count elements. */
int propd_gelu(int dtype, int64_t count, void* buf, void* stream);
/* x += delta (residual add, fp32 += dtype). */
int propd_residual_add(int dtype, int64_t count, float* x, const void* delta, void* stream);
/* dst[m] = (dtype) src[idx ? idx[m] : m] for fp32 rows of width H (gather + cast). */
int propd_gather_rows(int dtype, int M, int H, const float* src, const int32_t* idx, void* dst,
                      void* stream);
/* First-max argmax per row of an fp32 [M, V] matrix (row stride ld). */
int propd_argmax_rows(int M, const int32_t* rows_dev, int V, int ld, const float* logits, int32_t* out, void* stream);
/* Stable descending top-k per row (ties -> lower index; == numpy
 * argsort(-x, kind="stable")[:k]), k <= 1024. */
int propd_topk_rows(int R, int V, int ld, int k, const float* logits, int32_t* out_idx,
                    float* out_val, void* stream);

/* ---- KV cache ---- */
/* Scatter K/V of rows into the layer cache: row m of sequence b = row_seq[m]
 * goes to slot seq_len[seq_slot[b]] + row_node[m].  k/v are columns
 * [H,2H) and [2H,3H) of the fused qkv buffer (row stride ldqkv). */
int propd_kv_append(int dtype, int M, int A, int dh, int Lmax, const void* qkv, int ldqkv,
                    const int32_t* row_seq, const int32_t* row_node, const int32_t* seq_slot,
                    const int32_t* seq_len, void* kcache, void* vcache, void* stream);

/* ---- K2: tree-masked verification attention (backends.py:216-233) ----
 * Rows [row_off[b], row_off[b+1]) belong to sequence b; row m sees cache keys
 * [0, L_b) plus tree keys L_b + j for every bit j set in mask[row_node[m]]
 * (mask == NULL: causal new rows, j visible iff j <= row_node[m]; keys
 * beyond L_b + n_tmpl are never visible).
 * q = columns [0,H) of qkv.  out[m, a*dh:(a+1)*dh] = softmax(q k^T / sqrt(dh)) v.
 * `workspace` must hold propd_attn_workspace_bytes(...) bytes.
 * impl: 0 = auto, 1 = CUDA-core split-KV kernel, 4 = tcgen05/TMA row-major kernel (64-key
 * blocks, 6+6-stage K/V rings, two softmax warpgroups; auto for > 64 rows and
 * for latency-bound > 32-row launches), 5 = transposed tcgen05 kernel
 * (S^T = K Q^T, O^T += V^T P^T, keys on the MMA M dimension; <= 64 rows per
 * sequence; auto for 5..64 rows), 3 = streaming decode kernel (<= 4 rows per
 * sequence; auto for the bonus pass).  impls 3-5 need bf16 and dh = 128.  n_slots = number of [A, Lmax, dh] slot blocks in the
 * cache layer (bounds of the TMA tensor map).
 * impl | PROPD_ATTN_SCRATCH_LAST: the last batch entry holds only the pad rows
 * of a pass captured at a padded row capacity (the scratch slot, a few keys):
 * it is excluded from the launch-geometry heuristics (key splits per
 * sequence), so a B-sequence step gets the splits of B, not B + 1. */
#define PROPD_ATTN_SCRATCH_LAST 0x100
/* impl | PROPD_ATTN_QKV_F32: qkv is the fp32 QKV accumulator [M, 3H] of a QKV
 * launch without a tail (row stride ldqkv floats): Q and the tree rows' K/V
 * are read from it (bf16-rounded as propd_qkv_finish would store them), and
 * the kernel itself writes the tree rows' K/V into the layer cache (slot
 * seq_len + row_node); the accumulator is left as it is.  Decode kernel
 * (<= 4 rows per sequence) or transposed kernel (<= 64); bf16, dh = 128, a
 * mask (the single-node mask for one-row passes). */
#define PROPD_ATTN_QKV_F32 0x200
int64_t propd_attn_workspace_bytes(int M, int A, int dh, int max_splits);
int propd_tree_attention(int dtype, int impl, int B, int M, int A, int dh, int Lmax, int n_slots,
                         int max_rows_per_seq, int max_keys,
                         const void* qkv, int ldqkv, const void* kcache, const void* vcache,
                         const int32_t* seq_slot, const int32_t* seq_len,
                         const int32_t* row_off, const int32_t* row_node,
                         const uint64_t* mask, int n_tmpl, int W,
                         void* out, int ldout, void* workspace, int64_t workspace_bytes,
                         void* stream);

/* ---- weight-streaming projections for few tokens (bf16, M <= 128) ----
 * Y[M,N] (+)= X[M,K] . W[K,N] on tcgen05 (W row-major [K,N], X row-major
 * [M,K], Y fp32 row stride ldy).  accumulate = 1: split-K partial sums are
 * added with fp32 reductions into Y (Y must hold the addend, e.g. the
 * residual stream or a zeroed accumulator); 0: Y is overwritten.  N % 128 ==
 * 0, K % 64 == 0.  max_split <= 0: automatic.  rows_dev (nullable, device
 * int32): only rows < min(M, *rows_dev) of Y are written — the live row count
 * of a pass whose size is known only on the device (post-prune survivors),
 * so the launch can be captured once for the padded size M. */
int propd_gemm_ws(int M, const int32_t* rows_dev, int N, int K, const void* X, int ldx, const void* W, int ldw,
                  float* Y, int ldy, int accumulate, int max_split, void* stream);
/* In-kernel phases of a weight-streaming GEMM launch (all CTAs co-resident:
 * tiles x splits <= 2 x SMs; phases meet at grid barriers on `bar`, 4 zeroed
 * uint32 that every launch leaves zeroed).  They replace the small kernels
 * between projections, so a layer is five launches and the weight stream of
 * a launch keeps flowing while its prologue runs:
 *   prologue PROPD_PRO_LN:   X[t] = bf16(LN(pro_src[t])) (no affine, eps 1e-5,
 *            population variance; backends.py:135-142), pro_cols = K <= 4096;
 *            at <= 2 live rows every CTA normalises them itself and writes its
 *            own k-range of X (no grid barrier)
 *   prologue PROPD_PRO_GELU: X = bf16(tanh-GELU(pro_src)), pro_src re-zeroed
 *            (the previous launch's split-K accumulator)
 *   (X = pro_dst must be this launch's X operand, row stride pro_ldd = ldx)
 *   tail PROPD_TAIL_QKV:     after the split-K reduction into Y (= the zeroed
 *            fp32 QKV accumulator, N = 3H): Q rows -> tail_q (bf16, stride
 *            tail_ldq), K/V rows -> the layer cache exactly as
 *            propd_qkv_finish; Y re-zeroed.
 * Barrier-free prologue (the X operand is converted per ring stage inside
 * every CTA from fp32 pro_src [M, K] (row stride pro_ld, pro_cols = K), no
 * grid barrier, no bf16 X buffer):
 *   PROPD_PRO_XGELU: X = bf16(tanh-GELU(pro_src)) (pro_src is not re-zeroed:
 *            a later launch zeroes it through zero_buf: rows [0, M) x
 *            zero_cols of zero_buf, stride zero_ld, zeroed after the launch's
 *            dependency wait).  With pro_dst = X (bf16, stride pro_ldd = ldx)
 *            given, launches with more than 20 live rows (or fewer than 4
 *            ring slots) run the PROPD_PRO_GELU grid-barrier phase instead
 *            (and re-zero pro_src). */
#define PROPD_PRO_NONE 0
#define PROPD_PRO_LN 1
#define PROPD_PRO_GELU 2
#define PROPD_PRO_XGELU 4
/* Fused one-row attention (bonus / autoregressive passes at small batch):
 *   QKV launch, attn_splits = S > 0 (with PROPD_TAIL_QKV, one row per
 *            sequence): after the tail, the CTAs also compute the attention
 *            of every (row t, head a) over its sequence's keys 0..seq_len
 *            (the committed cache rows, streamed by bulk copies issued before
 *            the tail barrier, and the row's own K/V from Y) in S key splits,
 *            writing (m, l, -, -, o[dh]) partials (log2 domain, o unnormalised)
 *            to attn_part[t][a][S][4 + dh]; Y is not re-zeroed (the W_o launch's
 *            zero_buf duty does it).  M * A * S <= the launch's CTAs.
 *   PROPD_PRO_XATTN (W_o launch): X = bf16(combine of the S partials), built
 *            per ring stage inside every CTA (pro_src = attn_part,
 *            attn_splits = S, A, dh). */
#define PROPD_PRO_XATTN 5
#define PROPD_TAIL_NONE 0
#define PROPD_TAIL_QKV 1
typedef struct propd_ws_phases {
  int pro_mode;
  float* pro_src;
  int pro_ld;
  void* pro_dst;
  int pro_ldd, pro_cols;
  int tail_mode;
  void* tail_q;
  int tail_ldq;
  int A, dh, Lmax;
  const int32_t* row_seq;
  const int32_t* row_node;
  const int32_t* seq_slot;
  const int32_t* seq_len;
  void* kcache;
  void* vcache;
  uint32_t* bar;
  float* zero_buf;
  int zero_ld, zero_cols;
  int attn_splits;
  float* attn_part;
} propd_ws_phases;
int propd_gemm_ws_ph(int M, const int32_t* rows_dev, int N, int K, const void* X, int ldx, const void* W, int ldw,
                     float* Y, int ldy, int accumulate, int max_split, const propd_ws_phases* phases, void* stream);
/* K splits of an accumulating weight-streaming launch over W [K, N] (its grid
 * is N / 128 x splits CTAs; 0 for an invalid shape). */
int propd_ws_split_count(int N, int K);
/* ---- projections over many rows (> 128): Y = epilogue(X[M,K] . W[K,N]) ----
 * (backends.py:217-219, 234-236, 281, 321, 329).  bf16: persistent tcgen05
 * kernel (128 x 256 tiles, TMA, TMEM double-buffered accumulator; N % 32 == 0,
 * K % 64 == 0, 16-byte aligned rows); fp32 (parity mode): CUDA-core SGEMM.
 * rows_dev (nullable): live row count on the device (rows past it untouched).
 * ADD_F32 at few 128 x 256 tiles: K split across CTAs, reduced into Y.
 * Epilogue modes:
 *   STORE_F32  Y fp32 [M, N] = acc          (logits)
 *   ADD_F32    Y fp32 += acc                 (residual stream: W_o, W_2)
 *   STORE      Y [M, N] = acc in dtype       (bf16 / fp32 operand)
 *   GELU       Y = tanh-GELU(acc) in dtype   (W_1)
 *   QKV        N = 3H: columns < H -> Y (Q operand), K / V columns -> the layer
 *              cache at slot seq_len[seq_slot[row_seq[m]]] + row_node[m]. */
enum { PROPD_EPI_STORE = 0, PROPD_EPI_STORE_F32 = 1, PROPD_EPI_ADD_F32 = 2, PROPD_EPI_GELU = 3, PROPD_EPI_QKV = 4 };
typedef struct propd_gemm_epi {
  int mode;
  void* Y;
  int ldy;
  int A, dh, Lmax;
  const int32_t* row_seq;
  const int32_t* row_node;
  const int32_t* seq_slot;
  const int32_t* seq_len;
  void* kcache;
  void* vcache;
} propd_gemm_epi;
int propd_gemm(int dtype, int M, const int32_t* rows_dev, int N, int K, const void* X, int ldx, const void* W,
               int ldw, const propd_gemm_epi* epi, void* stream);
/* acc[M, 3H] fp32 -> qkv bf16 [M, 3H] and K/V rows into the layer cache
 * (slot seq_len[seq_slot[row_seq[m]]] + row_node[m]); acc re-zeroed. */
int propd_qkv_finish(int M, const int32_t* rows_dev, int A, int dh, int Lmax, float* acc, int ldacc, void* qkv, int ldqkv,
                     const int32_t* row_seq, const int32_t* row_node, const int32_t* seq_slot, const int32_t* seq_len,
                     void* kcache, void* vcache, void* stream);
/* out = bf16(tanh-GELU(acc)) for acc[M, N] fp32; acc re-zeroed. */
int propd_gelu_finish(int M, const int32_t* rows_dev, int N, float* acc, int ldacc, void* out, int ldout, void* stream);

/* ---- probability statistics (probability pruning, typical acceptance) ----
 * stats[r] = (log-sum-exp, entropy) in fp64 of z = logits[idx ? idx[r] : r] / temp
 * (fp32 rows of width V, row stride ld); rows_dev as above. */
int propd_row_lse(int R, const int32_t* rows_dev, int V, int ld, const float* logits, const int32_t* idx,
                  double temp, double* stats, void* stream);
/* Probability-based early pruning (the reference disables
 * it, pruning.py:76-82; definition = oracle probability_prune):
 * member[b*n+i] = depth-1, or sum over the path of (l_parent[token] - lse_parent)
 * >= log_tau, summed top-down in fp64.  early_stats = propd_row_lse of the
 * early rows (temp 1); row layout as propd_early_member. */
int propd_early_prob_member(int B, int n, int P, int V, double log_tau, const float* early_logits,
                            const double* early_stats, const int32_t* parent, const int32_t* parent_slot,
                            const int32_t* tokens, uint8_t* member, void* stream);

/* ---- K3: early prune (pruning.py:40-66, backends.py:320-327) ----
 * early_logits: fp32 [R, V], one row per (sequence, parent-slot): row
 * b*P + parent_slot[p] holds the early head output of node p of sequence b.
 * member[b*n+i] = (parent[i] < 0) or rank of tokens[b*n+i] in its parent's
 * row < topk, rank(t) = #{v: l[v] > l[t]} + #{v < t: l[v] == l[t]}. */
int propd_early_member(int B, int n, int P, int V, int topk, const float* early_logits,
                       const int32_t* parent, const int32_t* parent_slot, const int32_t* tokens,
                       uint8_t* member, void* stream);
/* Top-down closure + compaction of surviving rows (ballot/prefix sum):
 * alive[b*n+i] = member && (parent < 0 || alive[parent]); new rows are the
 * survivors in (b, i) order: new_row_seq/new_row_node/new_row_src (old row
 * index b*n+i), new_row_off[B+1]; node_row[b*n+i] = new row or -1;
 * surv_cnt[b]; *total = sum. */
int propd_prune_compact(int B, int n, const int32_t* parent, const uint8_t* member, uint8_t* alive,
                        int32_t* new_row_seq, int32_t* new_row_node, int32_t* new_row_src,
                        int32_t* new_row_off, int32_t* node_row, int32_t* surv_cnt, int32_t* total,
                        void* stream);

/* Typical acceptance for propd_verify_commit_ex (definition = oracle
 * typical_verify): candidate x is typical under row p = softmax(logits / T)
 * iff log p(x) > min(log_eps, log_alpha - H(p)); accepted = typical and parent
 * accepted (depth 1: under the root row); the path to the deepest accepted
 * node (ties: lowest index) is committed, bonus = its row argmax.
 * row_logits/row_stats: the tree pass's LM rows (survivor order) and their
 * propd_row_lse; root_logits: per sequence SLOT (stride root_ld), root_stats:
 * per batch entry; depth: template depths. */
typedef struct propd_typical {
  const float* row_logits;
  int ld;
  const double* row_stats;
  const float* root_logits;
  int root_ld;
  const double* root_stats;
  double log_eps, log_alpha, temperature;
  const int32_t* depth;
} propd_typical;
int propd_verify_commit_ex(int dtype, int B, int n, int D, int kmax, int layers, int A, int dh, int Lmax,
                           int64_t layer_stride, const int32_t* parent, const int32_t* tokens, const uint8_t* alive,
                           const int32_t* node_row, const int32_t* row_argmax, const int32_t* root,
                           const int32_t* draft_tok, const int32_t* seq_slot, int32_t* seq_len, void* kcache,
                           void* vcache, int32_t* acc_node, int32_t* acc_surv, int32_t* acc_len, int32_t* bonus,
                           int32_t* committed, int8_t* ranks, const propd_typical* typical, void* stream);
/* ---- K5: greedy accept + in-place KV compaction (verification.py:30-53,
 * backends.py:337-348) ----
 * Walks each sequence's (pruned) tree from root[slot]; accepted nodes
 * (original indices) -> acc_node[b][D], survivor-row indices -> acc_surv[b][D],
 * acc_len[b]; bonus[b]; committed[b][0..acc_len] = accepted tokens + bonus;
 * ranks[b][d] (int8) = 1-based rank of committed[b][d] in draft head d+1's
 * list, -1 if absent, 0 for depths beyond acc_len+1 (the acceptance record).
 * Then moves K/V of accepted node j from slot L+acc_node[j] to L+j in every
 * layer/head (read-before-write per element) and sets seq_len += acc_len.
 * alive may be NULL (no pruning); node_row may be NULL (row = b*n+i).
 * kcache/vcache: base of layer 0; layer_stride in elements. */
int propd_verify_commit(int dtype, int B, int n, int D, int kmax, int layers, int A, int dh, int Lmax,
                        int64_t layer_stride, const int32_t* parent, const int32_t* tokens,
                        const uint8_t* alive, const int32_t* node_row, const int32_t* row_argmax,
                        const int32_t* root, const int32_t* draft_tok, const int32_t* seq_slot,
                        int32_t* seq_len, void* kcache, void* vcache,
                        int32_t* acc_node, int32_t* acc_surv, int32_t* acc_len, int32_t* bonus,
                        int32_t* committed, int8_t* ranks, void* stream);

/* Explicit-index compaction (per-sequence commit path): same move as in
 * propd_verify_commit for given acc_node/acc_len, plus seq_len += acc_len. */
int propd_kv_compact(int dtype, int B, int D, int layers, int A, int dh, int Lmax, int64_t layer_stride,
                     const int32_t* seq_slot, int32_t* seq_len, const int32_t* acc_node,
                     const int32_t* acc_len, void* kcache, void* vcache, void* stream);

/* Padding for graph-captured passes: rows [*total, S_pad) of the compacted
 * tables get row_seq = B, row_node = 0, row_src = 0.  pad_seq = 1: they form
 * batch entry B (the scratch sequence, row_off[B+1] = S_pad) and are computed
 * like real rows; pad_seq = 0: they belong to no sequence (row_off[B+1] =
 * *total) and the pass's kernels skip them via rows_dev. */
int propd_pad_rows(int B, int S_pad, int pad_seq, const int32_t* total, int32_t* row_seq, int32_t* row_node, int32_t* row_src,
                   int32_t* row_off, void* stream);

/* seq_len[seq_slot[b]] += delta (delta_dev[b] if non-NULL, else delta). */
int propd_seq_advance(int B, const int32_t* seq_slot, int32_t* seq_len, const int32_t* delta_dev,
                      int delta, void* stream);
/* root[seq_slot[b]] = argmax[b] (first max of each bonus row). */
int propd_scatter_i32(int B, const int32_t* idx, const int32_t* src, int32_t* dst, void* stream);

/* ---- K4: dynamic tree generation (acceptance.py:96-206) ----
 * Replays acceptance records in global sequence order into P[D][k] (fp64,
 * in/out) and counts[D] (int64): for each record r = ranks[s][d] != 0,
 * counts[d] += 1, step = alpha > 0 ? alpha : 1/counts[d],
 * P[d][j] = (1-step)*P[d][j] + step*[j >= r-1 and r > 0]  (no FMA contraction).
 * Then scores the grid universe (1,..,1,r): contrib = spine[d]*m[d][r] with
 * m = diff(P, prepend 0), spine = cumprod(m[:,0]) and writes the selection
 * order (candidate c = d*k + r, sorted by (-contrib, depth, rank)) and the
 * expected-length curve l[s-1] = sum of the first s contributions. */
int propd_stats_replay_select(int S, int D, int k, const int8_t* ranks, double alpha, double* P,
                              int64_t* counts, int32_t* order, double* lcurve, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* PROPD_H */
