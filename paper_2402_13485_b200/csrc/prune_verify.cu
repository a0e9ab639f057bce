// K3 early prune, K5 greedy accept + in-place KV compaction, K4 acceptance
// statistics replay + grid node selection.
//
// Reference semantics (paths relative to /root/reference/pkg/src/treedecode/):
//   prune: depth-1 exempt, child alive iff parent alive and token in the
//          parent's early top-K (stable argsort)      pruning.py:40-66, backends.py:320-323
//   verify: greedy root-chain walk, bonus = last target verification.py:30-53
//   commit: accepted rows + bonus join the context    backends.py:337-348 (the
//          recompute is replaced by compaction of the tree-pass K/V rows; the
//          two are bit-identical in the reference)
//   stats update / marginals / selection             acceptance.py:96-117, 186-206
//   realized ranks per depth                          engine.py:283-288, acceptance.py:53-57
#include "common.cuh"

namespace propd {

// ---------------------------------------------------------------- K3 ------
// One thread-block cluster per (sequence, parent row): the parent's
// early-logit row is split across the cluster's CTAs (a row of 32000 logits
// scanned by one CTA took ~50 us at batch 1, three parent rows on three SMs),
// every child of that parent is ranked against each slice in the same pass,
// and the per-CTA partial ranks are summed through distributed shared memory
// by CTA rank 0.  Counting rank of child token t: the number of vocabulary
// entries a stable descending argsort places before t,
// #{v: l[v] > l[t]} + #{v < t: l[v] == l[t]}; the child is a member iff that
// rank is < K (the parent's K-th order statistic under the (value desc,
// index asc) order).  Depth-1 nodes are exempt (pruning.py:60-61) and
// written by the clusters of parent row 0.
constexpr int K3_THREADS = 512, K3_CH = 16, K3_MAXN = 1024, K3_MAXCL = 8;
__device__ __forceinline__ uint32_t k3_cl_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t k3_cl_size() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void k3_cl_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ int k3_cl_ld(const int* p, uint32_t rank) {
  uint32_t a, v;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(a) : "r"((uint32_t)__cvta_generic_to_shared(p)), "r"(rank));
  asm volatile("ld.shared::cluster.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
  return (int)v;
}
__global__ void __launch_bounds__(K3_THREADS) early_member_kernel(int n, int P, int V, int topk,
                                                                  const float* __restrict__ early,
                                                                  const int32_t* __restrict__ parent,
                                                                  const int32_t* __restrict__ parent_slot,
                                                                  const int32_t* __restrict__ tokens,
                                                                  uint8_t* __restrict__ member) {
  __shared__ int s_idx[K3_MAXN];
  __shared__ int s_cnt;
  __shared__ int red[K3_THREADS / 32][K3_CH];
  __shared__ int s_part[K3_CH];
  const int Pe = P > 0 ? P : 1;
  const int cs = (int)k3_cl_size(), cr = (int)k3_cl_rank();
  const int pr = blockIdx.x / cs;  // (sequence, parent row) of this cluster
  const int b = pr / Pe, j = pr - b * Pe;
  if (threadIdx.x == 0) s_cnt = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const int par = parent[i];
    if (par < 0) {
      if (j == 0 && cr == 0) member[b * n + i] = 1;
    } else if (parent_slot[par] == j) {
      s_idx[atomicAdd(&s_cnt, 1)] = i;
    }
  }
  __syncthreads();
  const int nc = s_cnt;  // (the same on every CTA of the cluster)
  if (nc == 0) return;
  const float* row = early + ((size_t)b * P + j) * V;
  const bool vec = (V & 3) == 0 && (reinterpret_cast<uintptr_t>(early) & 15) == 0;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  // this CTA's slice of the row (float4 units when vectorised)
  const int units = vec ? (V >> 2) : V, per = (units + cs - 1) / cs;
  const int u0 = min(units, cr * per), u1 = min(units, u0 + per);
  for (int c0 = 0; c0 < nc; c0 += K3_CH) {  // children in chunks held in registers (one slice pass each)
    float tv[K3_CH];
    int tk[K3_CH], cnt[K3_CH];
#pragma unroll
    for (int c = 0; c < K3_CH; ++c) {
      const bool live = c0 + c < nc;
      tk[c] = live ? tokens[b * n + s_idx[c0 + c]] : 0;
      tv[c] = live ? __ldg(row + tk[c]) : INFINITY;
      cnt[c] = 0;
    }
    if (vec) {
      const float4* r4 = reinterpret_cast<const float4*>(row);
      for (int i = u0 + threadIdx.x; i < u1; i += blockDim.x) {
        const float4 f = __ldg(r4 + i);
        const int v = 4 * i;
#pragma unroll
        for (int c = 0; c < K3_CH; ++c) {
          cnt[c] += (f.x > tv[c]) || (f.x == tv[c] && v < tk[c]);
          cnt[c] += (f.y > tv[c]) || (f.y == tv[c] && v + 1 < tk[c]);
          cnt[c] += (f.z > tv[c]) || (f.z == tv[c] && v + 2 < tk[c]);
          cnt[c] += (f.w > tv[c]) || (f.w == tv[c] && v + 3 < tk[c]);
        }
      }
    } else {
      for (int v = u0 + threadIdx.x; v < u1; v += blockDim.x) {
        const float x = row[v];
#pragma unroll
        for (int c = 0; c < K3_CH; ++c) cnt[c] += (x > tv[c]) || (x == tv[c] && v < tk[c]);
      }
    }
#pragma unroll
    for (int c = 0; c < K3_CH; ++c) {
      const int s = warp_isum(cnt[c]);
      if (lane == 0) red[wid][c] = s;
    }
    __syncthreads();
    if (threadIdx.x < K3_CH) {
      int s = 0;
      for (int w = 0; w < K3_THREADS / 32; ++w) s += red[w][threadIdx.x];
      s_part[threadIdx.x] = s;
    }
    if (cs > 1) k3_cl_sync();  // every slice's partial ranks are visible cluster-wide
    else __syncthreads();
    if (cr == 0 && threadIdx.x < K3_CH && c0 + (int)threadIdx.x < nc) {
      int s = 0;
      for (int r = 0; r < cs; ++r) s += r == 0 ? s_part[threadIdx.x] : k3_cl_ld(&s_part[threadIdx.x], r);
      member[b * n + s_idx[c0 + threadIdx.x]] = s < topk ? 1 : 0;
    }
    if (cs > 1) k3_cl_sync();  // s_part / red reused by the next chunk (and read remotely until here)
    else __syncthreads();
  }
}

// Single CTA: closure per sequence, block-wide exclusive scan of survivor
// counts, scatter of the compacted row tables.
__global__ void prune_compact_kernel(int B, int n, const int32_t* __restrict__ parent,
                                     const uint8_t* __restrict__ member, uint8_t* __restrict__ alive,
                                     int32_t* new_row_seq, int32_t* new_row_node, int32_t* new_row_src,
                                     int32_t* new_row_off, int32_t* node_row, int32_t* surv_cnt, int32_t* total) {
  __shared__ int scan[1024];
  const int b = threadIdx.x;
  int cnt = 0;
  if (b < B) {
    for (int i = 0; i < n; ++i) {
      const int par = parent[i];
      const bool ok = member[b * n + i] && (par < 0 || alive[b * n + par]);
      alive[b * n + i] = ok;
      cnt += ok;
    }
  }
  scan[threadIdx.x] = cnt;
  __syncthreads();
  for (int off = 1; off < (int)blockDim.x; off <<= 1) {  // Hillis-Steele inclusive scan
    int v = threadIdx.x >= off ? scan[threadIdx.x - off] : 0;
    __syncthreads();
    scan[threadIdx.x] += v;
    __syncthreads();
  }
  if (b < B) {
    int o = scan[b] - cnt;
    new_row_off[b] = o;
    surv_cnt[b] = cnt;
    for (int i = 0; i < n; ++i) {
      if (alive[b * n + i]) {
        new_row_seq[o] = b;
        new_row_node[o] = i;
        new_row_src[o] = b * n + i;
        node_row[b * n + i] = o++;
      } else {
        node_row[b * n + i] = -1;
      }
    }
    if (b == B - 1) {
      new_row_off[B] = o;
      *total = o;
    }
  }
}

// Same outputs with the tree staged in shared memory (B * n <= K5S_MAX): the
// closure of every (sequence, node) is an independent walk up its ancestor
// chain (a node is alive iff it and all its ancestors are members), so it
// runs on all threads at once instead of one dependent global-memory chain
// per sequence; counts, scan and the row scatter then read shared memory.
constexpr int K5S_MAX = 16384;
__global__ void __launch_bounds__(1024) prune_compact_smem_kernel(
    int B, int n, const int32_t* __restrict__ parent, const uint8_t* __restrict__ member, uint8_t* __restrict__ alive,
    int32_t* new_row_seq, int32_t* new_row_node, int32_t* new_row_src, int32_t* new_row_off, int32_t* node_row,
    int32_t* surv_cnt, int32_t* total) {
  __shared__ int scan[1024];
  __shared__ int s_par[1024];
  __shared__ uint8_t s_mem[K5S_MAX], s_alive[K5S_MAX];
  const int BN = B * n;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s_par[i] = parent[i];
  for (int e = threadIdx.x; e < BN; e += blockDim.x) s_mem[e] = member[e];
  __syncthreads();
  for (int e = threadIdx.x; e < BN; e += blockDim.x) {
    const int b = e / n, i = e - b * n;
    bool ok = s_mem[e] != 0;
    for (int a = s_par[i]; ok && a >= 0; a = s_par[a]) ok = s_mem[b * n + a] != 0;
    s_alive[e] = ok;
    alive[e] = ok;
  }
  __syncthreads();
  const int b = threadIdx.x;
  int cnt = 0;
  if (b < B)
    for (int i = 0; i < n; ++i) cnt += s_alive[b * n + i];
  scan[threadIdx.x] = cnt;
  __syncthreads();
  for (int off = 1; off < (int)blockDim.x; off <<= 1) {  // Hillis-Steele inclusive scan
    int v = threadIdx.x >= off ? scan[threadIdx.x - off] : 0;
    __syncthreads();
    scan[threadIdx.x] += v;
    __syncthreads();
  }
  if (b < B) {
    int o = scan[b] - cnt;
    new_row_off[b] = o;
    surv_cnt[b] = cnt;
    for (int i = 0; i < n; ++i) {
      if (s_alive[b * n + i]) {
        new_row_seq[o] = b;
        new_row_node[o] = i;
        new_row_src[o] = b * n + i;
        node_row[b * n + i] = o++;
      } else {
        node_row[b * n + i] = -1;
      }
    }
    if (b == B - 1) {
      new_row_off[B] = o;
      *total = o;
    }
  }
}

// Graph-captured passes run layers > p on a padded row count: rows
// [total, S_pad) become batch entry B (the scratch slot, node 0).
__global__ void pad_rows_kernel(int B, int S_pad, int pad_seq, const int32_t* __restrict__ total, int32_t* row_seq,
                                int32_t* row_node, int32_t* row_src, int32_t* row_off) {
  const int S = *total;
  for (int i = S + blockIdx.x * blockDim.x + threadIdx.x; i < S_pad; i += gridDim.x * blockDim.x) {
    row_seq[i] = B;
    row_node[i] = 0;
    row_src[i] = 0;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) row_off[B + 1] = pad_seq ? S_pad : S;
}

// ---------------------------------------------------------------- K5 ------
constexpr int MAX_D = 32;

// Moves accepted rows j (slot L + node[j]) to L + j.  One CTA per (sequence,
// layer); each thread owns a fixed 16-byte column chunk of one head's block
// and walks j upward: since node[j] >= j and node is increasing, dst L+j never
// aliases a source still to be read (read-before-write per element).  seq_len
// has already been advanced by the accepted count: L = seq_len - acc_len.
template <typename T>
__global__ void compact_rows_kernel(int D, int A, int dh, int Lmax, int64_t layer_stride,
                                    const int32_t* __restrict__ seq_slot, const int32_t* __restrict__ seq_len,
                                    const int32_t* __restrict__ acc_node, const int32_t* __restrict__ acc_len, T* kc,
                                    T* vc) {
  __shared__ int s_acc[MAX_D];
  const int b = blockIdx.x, l = blockIdx.y;
  const int len = acc_len[b];
  if (len == 0) return;
  const int slot = seq_slot[b];
  const int L = seq_len[slot] - len;
  if (threadIdx.x < len) s_acc[threadIdx.x] = acc_node[b * D + threadIdx.x];
  __syncthreads();
  constexpr int VEC = 16 / sizeof(T);
  const int chunks = dh / VEC;
  for (int w = threadIdx.x; w < A * chunks; w += blockDim.x) {
    const int c = w % chunks, a = w / chunks;
    const size_t base = (size_t)l * layer_stride + ((size_t)slot * A + a) * Lmax * dh + (size_t)c * VEC;
    for (int j = 0; j < len; ++j) {
      const int src = s_acc[j];
      if (src == j) continue;
      const size_t so = base + (size_t)(L + src) * dh, dof = base + (size_t)(L + j) * dh;
      *reinterpret_cast<uint4*>(kc + dof) = *reinterpret_cast<const uint4*>(kc + so);
      *reinterpret_cast<uint4*>(vc + dof) = *reinterpret_cast<const uint4*>(vc + so);
    }
  }
}

__global__ void advance_by_acc_kernel(int B, const int32_t* seq_slot, int32_t* seq_len, const int32_t* acc_len) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b < B) seq_len[seq_slot[b]] += acc_len[b];
}

// Typical acceptance (oracle typical_verify): candidate token x of a node is
// typical under its parent's row p = softmax(z), z = logits / T, iff
// z[x] - lse > min(log eps, log alpha - H); a node is accepted iff typical and
// its parent accepted (depth 1: under the root row); the path to the deepest
// accepted node (ties: lowest index) is committed, bonus = that row's argmax.
// Evaluated level by level by one warp (parents precede children in the
// canonical order and depth <= D).
__device__ __forceinline__ bool typical_ok(const float* row, int tok, const double* st, const propd_typical& t) {
  const double lp = __dsub_rn(__ddiv_rn((double)row[tok], t.temperature), st[0]);
  return lp > fmin(t.log_eps, __dsub_rn(t.log_alpha, st[1]));
}

__device__ int typical_walk(int b, int slot, int n, int D, const int32_t* parent, const int32_t* tokens,
                            const uint8_t* alive, const int32_t* node_row, const propd_typical& t, int* s_acc,
                            uint8_t* s_ok, int lane) {
  for (int i = lane; i < n; i += 32) s_ok[i] = 0;
  __syncwarp();
  for (int d = 1; d <= D; ++d) {
    for (int base = 0; base < n; base += 32) {
      const int i = base + lane;
      if (i < n && t.depth[i] == d && (alive == nullptr || alive[b * n + i])) {
        const int p = parent[i];
        bool ok;
        if (p < 0) {
          ok = typical_ok(t.root_logits + (size_t)slot * t.root_ld, tokens[b * n + i], t.root_stats + 2 * b, t);
        } else if (s_ok[p]) {
          const int r = node_row ? node_row[b * n + p] : b * n + p;
          ok = typical_ok(t.row_logits + (size_t)r * t.ld, tokens[b * n + i], t.row_stats + 2 * r, t);
        } else {
          ok = false;
        }
        s_ok[i] = ok ? 1 : 0;
      }
    }
    __syncwarp();
  }
  // deepest accepted node, ties -> lowest index
  int best = -1, best_d = 0;
  for (int i = lane; i < n; i += 32)
    if (s_ok[i] && t.depth[i] > best_d) {
      best = i;
      best_d = t.depth[i];
    }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const int ob = __shfl_xor_sync(0xffffffffu, best, o), od = __shfl_xor_sync(0xffffffffu, best_d, o);
    if (od > best_d || (od == best_d && ob >= 0 && (best < 0 || ob < best))) {
      best = ob;
      best_d = od;
    }
  }
  if (lane == 0)
    for (int j = best, k = best_d - 1; j >= 0; j = parent[j], --k) s_acc[k] = j;
  __syncwarp();
  return best;
}

// One warp per sequence: walk, committed tokens, acceptance records; seq_len
// advanced by the accepted count (the K/V rows move in compact_rows_kernel).
__global__ void __launch_bounds__(32) verify_commit_kernel(int n, int D, int kmax, const int32_t* __restrict__ parent, const int32_t* __restrict__ tokens,
                                     const uint8_t* __restrict__ alive, const int32_t* __restrict__ node_row,
                                     const int32_t* __restrict__ row_argmax, const int32_t* __restrict__ root,
                                     const int32_t* __restrict__ draft_tok, const int32_t* __restrict__ seq_slot,
                                     int32_t* seq_len, int32_t* acc_node, int32_t* acc_surv,
                                     int32_t* acc_len, int32_t* bonus, int32_t* committed, int8_t* ranks,
                                     propd_typical typ) {
  __shared__ int s_acc[MAX_D];
  __shared__ int s_len, s_L;
  __shared__ uint8_t s_ok[1024];
  const int b = blockIdx.x;
  const int slot = seq_slot[b];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    const int L = seq_len[slot];
    int target = root[slot];
    int cur = -1, len = 0;
    if (typ.depth != nullptr) {  // typical acceptance: the walk fills s_acc, D steps skipped below
      const int best = typical_walk(b, slot, n, D, parent, tokens, alive, node_row, typ, s_acc, s_ok, lane);
      if (best >= 0) {
        len = typ.depth[best];
        target = row_argmax[node_row ? node_row[b * n + best] : b * n + best];
      }
    }
    for (int step = 0; step < D && typ.depth == nullptr; ++step) {
      int found = -1;
      for (int base = 0; base < n; base += 32) {
        const int i = base + lane;
        const bool ok = i < n && parent[i] == cur && (alive == nullptr || alive[b * n + i]) &&
                        tokens[b * n + i] == target;
        const unsigned bal = __ballot_sync(0xffffffffu, ok);
        if (bal) { found = base + __ffs(bal) - 1; break; }
      }
      if (found < 0) break;
      if (lane == 0) s_acc[len] = found;
      const int row = node_row ? node_row[b * n + found] : b * n + found;
      target = row_argmax[row];
      cur = found;
      ++len;
    }
    __syncwarp();
    // survivor-row index of each accepted node = #alive nodes before it
    for (int j = 0; j < len; ++j) {
      const int node = s_acc[j];
      int cnt = 0;
      for (int base = 0; base < node; base += 32) {
        const int i = base + lane;
        const bool ok = i < node && (alive == nullptr || alive[b * n + i]);
        cnt += __popc(__ballot_sync(0xffffffffu, ok));
      }
      if (lane == 0) {
        acc_node[b * D + j] = node;
        acc_surv[b * D + j] = cnt;
      }
    }
    if (lane == 0) {
      for (int j = len; j < D; ++j) { acc_node[b * D + j] = -1; acc_surv[b * D + j] = -1; }
      s_len = len;
      s_L = L;
      acc_len[b] = len;
      bonus[b] = target;
      int32_t* cm = committed + (size_t)b * (D + 1);
      for (int j = 0; j < len; ++j) cm[j] = tokens[b * n + s_acc[j]];
      cm[len] = target;
      for (int j = len + 1; j <= D; ++j) cm[j] = -1;
      // acceptance record: realized[d] = newly[d-1], d <= min(len+1, D)
      for (int d = 0; d < D; ++d) {
        int8_t r = 0;
        if (d <= len) {
          const int tok = cm[d];
          const int32_t* lst = draft_tok + ((size_t)b * D + d) * kmax;
          r = -1;
          for (int k = 0; k < kmax; ++k)
            if (lst[k] == tok) { r = (int8_t)(k + 1); break; }
        }
        ranks[(size_t)b * D + d] = r;
      }
    }
  }
  if (threadIdx.x == 0) seq_len[slot] = s_L + s_len;  // compaction: compact_rows_kernel (L = seq_len - acc_len)
}

// ---------------------------------------------------------------- K4 ------
// fp64 with explicit round-to-nearest intrinsics: no FMA contraction, so the
// results are bit-identical to numpy's separate multiply and add.
__global__ void stats_replay_select_kernel(int S, int D, int k, const int8_t* __restrict__ ranks, double alpha,
                                           double* P, int64_t* counts, int32_t* order, double* lcurve) {
  extern __shared__ double sm[];
  double* Ps = sm;               // D*k
  double* contrib = sm + D * k;  // D*k
  double* spine = contrib + D * k;  // D+1
  __shared__ long long cnt_s[MAX_D];
  const int N = D * k;
  for (int i = threadIdx.x; i < N; i += blockDim.x) Ps[i] = P[i];
  if (threadIdx.x < D) cnt_s[threadIdx.x] = counts[threadIdx.x];
  __syncthreads();
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    for (int s = 0; s < S; ++s) {
      for (int d = 0; d < D; ++d) {
        const int r = ranks[(size_t)s * D + d];
        if (r == 0) continue;
        const long long c = cnt_s[d] + 1;
        __syncwarp();
        if (lane == 0) cnt_s[d] = c;
        const double step = alpha > 0.0 ? alpha : __ddiv_rn(1.0, (double)c);
        const double keep = __dsub_rn(1.0, step);
        for (int j = lane; j < k; j += 32) {
          const double hit = (r > 0 && j >= r - 1) ? 1.0 : 0.0;
          Ps[d * k + j] = __dadd_rn(__dmul_rn(keep, Ps[d * k + j]), __dmul_rn(step, hit));
        }
        __syncwarp();
      }
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < N; i += blockDim.x) P[i] = Ps[i];
  if (threadIdx.x < D) counts[threadIdx.x] = cnt_s[threadIdx.x];
  if (threadIdx.x == 0) {
    spine[0] = 1.0;
    for (int d = 0; d < D; ++d) spine[d + 1] = __dmul_rn(spine[d], __dsub_rn(Ps[d * k], 0.0));
  }
  __syncthreads();
  for (int c = threadIdx.x; c < N; c += blockDim.x) {
    const int d = c / k, r = c - d * k;
    const double m = __dsub_rn(Ps[c], r > 0 ? Ps[c - 1] : 0.0);
    contrib[c] = __dmul_rn(spine[d], m);
  }
  __syncthreads();
  for (int c = threadIdx.x; c < N; c += blockDim.x) {
    const double v = contrib[c];
    int pos = 0;
    for (int c2 = 0; c2 < N; ++c2) {
      const double w = contrib[c2];
      pos += (w > v) || (w == v && c2 < c);
    }
    order[pos] = c;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    // l(s) = Python sum() of the first s contributions.  CPython >= 3.12 sums
    // floats with Neumaier compensation (bltinmodule.c builtin_sum_impl):
    // the first term seeds the running sum, later terms update (f, c), and
    // the result is f + c when c is non-zero and finite.
    double f = contrib[order[0]], c = 0.0;
    lcurve[0] = f;
    for (int s = 1; s < N; ++s) {
      const double x = contrib[order[s]];
      const double t = __dadd_rn(f, x);
      if (fabs(f) >= fabs(x))
        c = __dadd_rn(c, __dadd_rn(__dsub_rn(f, t), x));
      else
        c = __dadd_rn(c, __dadd_rn(__dsub_rn(x, t), f));
      f = t;
      lcurve[s] = (c != 0.0 && isfinite(c)) ? __dadd_rn(f, c) : f;
    }
  }
}

}  // namespace propd

using namespace propd;

extern "C" {

int propd_early_member(int B, int n, int P, int V, int topk, const float* early_logits, const int32_t* parent,
                       const int32_t* parent_slot, const int32_t* tokens, uint8_t* member, void* stream) {
  if (B == 0 || n == 0) return 0;
  PROPD_REQUIRE(topk >= 1, "early_member: topk must be positive");
  PROPD_REQUIRE(n <= K3_MAXN, "early_member: tree of %d nodes > %d", n, K3_MAXN);
  // cluster size: up to 8 slices per parent row while the clusters fit in about two waves of CTAs
  const int rows = B * (P > 0 ? P : 1);
  int cs = 1;
  while (cs < K3_MAXCL && rows * cs * 2 <= 2 * propd_num_sms() && V / (cs * 2) >= 4 * K3_THREADS) cs *= 2;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(rows * cs);
  cfg.blockDim = dim3(K3_THREADS);
  cfg.stream = as_stream(stream);
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cs;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, early_member_kernel, n, P, V, topk, early_logits, parent,
                                           parent_slot, tokens, member);
  if (e != cudaSuccess) {
    (void)cudaGetLastError();
    return fail("early_member: %s", cudaGetErrorString(e));
  }
  return check_launch("early_member");
}

int propd_prune_compact(int B, int n, const int32_t* parent, const uint8_t* member, uint8_t* alive,
                        int32_t* new_row_seq, int32_t* new_row_node, int32_t* new_row_src, int32_t* new_row_off,
                        int32_t* node_row, int32_t* surv_cnt, int32_t* total, void* stream) {
  if (B == 0) return 0;
  PROPD_REQUIRE(B <= 1024, "prune_compact: batch %d > 1024", B);
  if ((long long)B * n <= K5S_MAX && n <= 1024) {
    prune_compact_smem_kernel<<<1, 1024, 0, as_stream(stream)>>>(B, n, parent, member, alive, new_row_seq,
                                                                  new_row_node, new_row_src, new_row_off, node_row,
                                                                  surv_cnt, total);
    return check_launch("prune_compact");
  }
  int threads = ((B + 31) / 32) * 32;
  prune_compact_kernel<<<1, threads, 0, as_stream(stream)>>>(B, n, parent, member, alive, new_row_seq, new_row_node,
                                                             new_row_src, new_row_off, node_row, surv_cnt, total);
  return check_launch("prune_compact");
}

int propd_pad_rows(int B, int S_pad, int pad_seq, const int32_t* total, int32_t* row_seq, int32_t* row_node, int32_t* row_src,
                   int32_t* row_off, void* stream) {
  pad_rows_kernel<<<1, 256, 0, as_stream(stream)>>>(B, S_pad, pad_seq, total, row_seq, row_node, row_src, row_off);
  return check_launch("pad_rows");
}

int propd_verify_commit(int dtype, int B, int n, int D, int kmax, int layers, int A, int dh, int Lmax,
                        int64_t layer_stride, const int32_t* parent, const int32_t* tokens, const uint8_t* alive,
                        const int32_t* node_row, const int32_t* row_argmax, const int32_t* root,
                        const int32_t* draft_tok, const int32_t* seq_slot, int32_t* seq_len, void* kcache,
                        void* vcache, int32_t* acc_node, int32_t* acc_surv, int32_t* acc_len, int32_t* bonus,
                        int32_t* committed, int8_t* ranks, void* stream) {
  return propd_verify_commit_ex(dtype, B, n, D, kmax, layers, A, dh, Lmax, layer_stride, parent, tokens, alive,
                                node_row, row_argmax, root, draft_tok, seq_slot, seq_len, kcache, vcache, acc_node,
                                acc_surv, acc_len, bonus, committed, ranks, nullptr, stream);
}

// K/V rows of the accepted nodes -> positions L + j (seq_len already advanced)
static int launch_compact(int dtype, int B, int D, int layers, int A, int dh, int Lmax, int64_t layer_stride,
                          const int32_t* seq_slot, const int32_t* seq_len, const int32_t* acc_node,
                          const int32_t* acc_len, void* kcache, void* vcache, cudaStream_t st) {
  return PROPD_DISPATCH_DTYPE(dtype, T, [&] {
    PROPD_REQUIRE((dh * (int)sizeof(T)) % 16 == 0, "kv compaction: dh*sizeof must be a multiple of 16");
    compact_rows_kernel<T><<<dim3(B, layers), 256, 0, st>>>(D, A, dh, Lmax, layer_stride, seq_slot, seq_len, acc_node,
                                                           acc_len, (T*)kcache, (T*)vcache);
    return check_launch("kv compaction");
  });
}

int propd_verify_commit_ex(int dtype, int B, int n, int D, int kmax, int layers, int A, int dh, int Lmax,
                           int64_t layer_stride, const int32_t* parent, const int32_t* tokens, const uint8_t* alive,
                           const int32_t* node_row, const int32_t* row_argmax, const int32_t* root,
                           const int32_t* draft_tok, const int32_t* seq_slot, int32_t* seq_len, void* kcache,
                           void* vcache, int32_t* acc_node, int32_t* acc_surv, int32_t* acc_len, int32_t* bonus,
                           int32_t* committed, int8_t* ranks, const propd_typical* typical, void* stream) {
  if (B == 0) return 0;
  PROPD_REQUIRE(D >= 1 && D <= MAX_D, "verify_commit: D=%d outside 1..%d", D, MAX_D);
  // acceptance records hold rank + 1 in an int8 (propd_stats_replay_select)
  PROPD_REQUIRE(kmax >= 1 && kmax <= 127, "verify_commit: draft top-k %d outside 1..127 (int8 acceptance records)",
                kmax);
  PROPD_REQUIRE(typical == nullptr || (n <= 1024 && typical->depth && typical->row_logits && typical->row_stats &&
                                       typical->root_logits && typical->root_stats),
                "verify_commit: typical acceptance needs depth, row and root logits + statistics (n <= 1024)");
  cudaStream_t st = as_stream(stream);
  verify_commit_kernel<<<B, 32, 0, st>>>(n, D, kmax, parent, tokens, alive, node_row, row_argmax, root, draft_tok,
                                         seq_slot, seq_len, acc_node, acc_surv, acc_len, bonus, committed, ranks,
                                         typical ? *typical : propd_typical{});
  if (int e = check_launch("verify_commit")) return e;
  return launch_compact(dtype, B, D, layers, A, dh, Lmax, layer_stride, seq_slot, seq_len, acc_node, acc_len, kcache,
                        vcache, st);
}

int propd_kv_compact(int dtype, int B, int D, int layers, int A, int dh, int Lmax, int64_t layer_stride,
                     const int32_t* seq_slot, int32_t* seq_len, const int32_t* acc_node, const int32_t* acc_len,
                     void* kcache, void* vcache, void* stream) {
  if (B == 0) return 0;
  PROPD_REQUIRE(D >= 1 && D <= MAX_D, "kv_compact: D=%d outside 1..%d", D, MAX_D);
  cudaStream_t st = as_stream(stream);
  advance_by_acc_kernel<<<(B + 127) / 128, 128, 0, st>>>(B, seq_slot, seq_len, acc_len);
  if (int e = check_launch("kv_compact")) return e;
  return launch_compact(dtype, B, D, layers, A, dh, Lmax, layer_stride, seq_slot, seq_len, acc_node, acc_len, kcache,
                        vcache, st);
}

int propd_stats_replay_select(int S, int D, int k, const int8_t* ranks, double alpha, double* P, int64_t* counts,
                              int32_t* order, double* lcurve, void* stream) {
  PROPD_REQUIRE(D >= 1 && D <= MAX_D && k >= 1 && k <= 127 && D * k <= 4096,
                "stats_replay_select: bad grid D=%d k=%d (k <= 127: int8 acceptance records)", D, k);
  const size_t smem = (size_t)(2 * D * k + D + 1) * sizeof(double);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(stats_replay_select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return fail("stats_replay_select: %s", cudaGetErrorString(e));
  }
  stats_replay_select_kernel<<<1, 256, smem, as_stream(stream)>>>(S, D, k, ranks, alpha, P, counts, order, lcurve);
  return check_launch("stats_replay_select");
}

}  // extern "C"
