// K2: tree-masked verification attention, CUDA-core split-KV variant
// (fp32 parity path + generic fallback for any dh in {16,32,64,128}).
//
// Reference: TinyTransformer._block attention (backends.py:216-233): every
// new row attends to all committed cache rows plus the tree rows its
// ancestor mask allows, softmax(q k^T / sqrt(dh)) v per head.
//
// Decomposition: grid (split, head, sequence).  One CTA streams one KV chunk
// [k_begin, k_end) of one (sequence, head) through shared memory and serves
// every query row of that sequence from it (rows in groups of 4 warps x
// 8 rows (4 for dh=128); lane j <-> key j of a 32-key tile).  Online softmax per row with
// warp shuffles; splits are merged by attn_combine_kernel (flash-decoding).
// Keys t < L are cache rows (always visible); t = L + j is tree node j,
// visible iff bit j of the row's ancestor bitset is set.
#include "common.cuh"

namespace propd {

constexpr int ATT_THREADS = 128;
constexpr int ATT_TILE = 32;
constexpr int ATT_MAXW = 4;  // <= 256 tree nodes

struct AttnArgs {
  const void* qkv;
  int ldq;
  const void* kc;
  const void* vc;
  const int32_t* seq_slot;
  const int32_t* seq_len;
  const int32_t* row_off;
  const int32_t* row_node;
  const uint64_t* mask;
  int n_tmpl, W;
  int A, Lmax;
  float scale;
  int split_len, nsplit;
  float* part_o;   // [M][A][nsplit][dh]
  float* part_ml;  // [M][A][nsplit][2]
  void* out;
  int ldout;
};

template <typename T, int DH>
__global__ void __launch_bounds__(ATT_THREADS) attn_core_kernel(AttnArgs p) {
  constexpr int DPL = DH >= 32 ? DH / 32 : 1;
  constexpr int ATT_ROWS_PER_WARP = DH >= 128 ? 4 : 8;   // static smem < 48 KB
  constexpr int ATT_GROUP = 4 * ATT_ROWS_PER_WARP;
  __shared__ float q_s[ATT_GROUP][DH];
  __shared__ float k_s[ATT_TILE][DH + 1];
  __shared__ float v_s[ATT_TILE][DH];
  __shared__ uint64_t msk_s[ATT_GROUP][ATT_MAXW];

  const int s = blockIdx.x, a = blockIdx.y, b = blockIdx.z;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int slot = p.seq_slot[b];
  const int L = p.seq_len[slot];
  const int r0 = p.row_off[b], r1 = p.row_off[b + 1];
  const int nkeys = L + p.n_tmpl;
  const int k_begin = s * p.split_len;
  const int k_end = min(nkeys, k_begin + p.split_len);
  const T* q = reinterpret_cast<const T*>(p.qkv);
  const T* kb = reinterpret_cast<const T*>(p.kc) + ((size_t)slot * p.A + a) * p.Lmax * DH;
  const T* vb = reinterpret_cast<const T*>(p.vc) + ((size_t)slot * p.A + a) * p.Lmax * DH;
  const int H = p.A * DH;

  for (int g0 = r0; g0 < r1; g0 += ATT_GROUP) {
    const int nrows = min(ATT_GROUP, r1 - g0);
    for (int i = threadIdx.x; i < ATT_GROUP * DH; i += ATT_THREADS) {
      const int r = i / DH, d = i - r * DH;
      q_s[r][d] = r < nrows ? to_f(q[(size_t)(g0 + r) * p.ldq + a * DH + d]) : 0.f;
    }
    for (int i = threadIdx.x; i < ATT_GROUP * ATT_MAXW; i += ATT_THREADS) {
      const int r = i / ATT_MAXW, w = i - r * ATT_MAXW;
      if (p.mask == nullptr)  // causal new rows (prefill / extend): node j visible iff j <= row_node
        msk_s[r][w] = (r < nrows && w == 0) ? (uint64_t)p.row_node[g0 + r] : 0ull;
      else
        msk_s[r][w] = (r < nrows && w < p.W) ? p.mask[(size_t)p.row_node[g0 + r] * p.W + w] : 0ull;
    }
    float m_run[ATT_ROWS_PER_WARP], l_run[ATT_ROWS_PER_WARP], o[ATT_ROWS_PER_WARP][DPL];
#pragma unroll
    for (int j = 0; j < ATT_ROWS_PER_WARP; ++j) {
      m_run[j] = -INFINITY;
      l_run[j] = 0.f;
#pragma unroll
      for (int c = 0; c < DPL; ++c) o[j][c] = 0.f;
    }
    __syncthreads();
    for (int kt = k_begin; kt < k_end; kt += ATT_TILE) {
      for (int i = threadIdx.x; i < ATT_TILE * DH; i += ATT_THREADS) {
        const int j = i / DH, d = i - j * DH;
        const int key = kt + j;
        float kv = 0.f, vv = 0.f;
        if (key < k_end) {
          kv = to_f(kb[(size_t)key * DH + d]);
          vv = to_f(vb[(size_t)key * DH + d]);
        }
        k_s[j][d] = kv;
        v_s[j][d] = vv;
      }
      __syncthreads();
      const int key = kt + lane;
#pragma unroll
      for (int j = 0; j < ATT_ROWS_PER_WARP; ++j) {
        const int r = warp * ATT_ROWS_PER_WARP + j;
        if (r >= nrows) break;  // warp-uniform
        bool vis;
        if (key >= k_end) vis = false;
        else if (key < L) vis = true;
        else {
          const int t = key - L;
          vis = p.mask == nullptr ? (t <= (int)msk_s[r][0]) : (bool)((msk_s[r][t >> 6] >> (t & 63)) & 1ull);
        }
        float sc = -INFINITY;
        if (vis) {
          float acc = 0.f;
#pragma unroll
          for (int d = 0; d < DH; ++d) acc = fmaf(q_s[r][d], k_s[lane][d], acc);
          sc = acc * p.scale;
        }
        const float tmax = warp_max(sc);
        if (tmax == -INFINITY) continue;  // warp-uniform: nothing visible in this tile
        const float mnew = fmaxf(m_run[j], tmax);
        const float corr = expf(m_run[j] - mnew);
        const float pr = vis ? expf(sc - mnew) : 0.f;
        l_run[j] = l_run[j] * corr + warp_sum(pr);
        m_run[j] = mnew;
#pragma unroll
        for (int c = 0; c < DPL; ++c) o[j][c] *= corr;
#pragma unroll 8
        for (int jj = 0; jj < ATT_TILE; ++jj) {
          const float pj = __shfl_sync(0xffffffffu, pr, jj);
#pragma unroll
          for (int c = 0; c < DPL; ++c) {
            const int d = (lane + 32 * c) % DH;
            o[j][c] = fmaf(pj, v_s[jj][d], o[j][c]);
          }
        }
      }
      __syncthreads();
    }
    // epilogue
#pragma unroll
    for (int j = 0; j < ATT_ROWS_PER_WARP; ++j) {
      const int r = warp * ATT_ROWS_PER_WARP + j;
      if (r >= nrows) break;
      const int row = g0 + r;
      if (p.nsplit == 1) {
        T* out = reinterpret_cast<T*>(p.out) + (size_t)row * p.ldout + a * DH;
        const float inv = l_run[j] > 0.f ? 1.f / l_run[j] : 0.f;
#pragma unroll
        for (int c = 0; c < DPL; ++c) {
          const int d = lane + 32 * c;
          if (d < DH) out[d] = from_f<T>(o[j][c] * inv);
        }
      } else {
        const size_t base = ((size_t)row * p.A + a) * p.nsplit + s;
        float* po = p.part_o + base * DH;
#pragma unroll
        for (int c = 0; c < DPL; ++c) {
          const int d = lane + 32 * c;
          if (d < DH) po[d] = o[j][c];
        }
        if (lane == 0) {
          p.part_ml[base * 2] = m_run[j];
          p.part_ml[base * 2 + 1] = l_run[j];
        }
      }
    }
    __syncthreads();
  }
  (void)H;
}

// Merge the per-split (o, m, l) partials of every (row, head).
template <typename T>
__global__ void attn_combine_kernel(int A, int dh, int nsplit, const float* __restrict__ part_o,
                                    const float* __restrict__ part_ml, T* __restrict__ out, int ldout) {
  pdl_trigger();  // early: the dependent only prefetches weights before its own wait
  pdl_wait();
  const int row = blockIdx.x, a = blockIdx.y;
  const size_t base = ((size_t)row * A + a) * nsplit;
  float mx = -INFINITY;
  for (int s = 0; s < nsplit; ++s) mx = fmaxf(mx, part_ml[(base + s) * 2]);
  float l = 0.f;
  for (int s = 0; s < nsplit; ++s) {
    const float ms = part_ml[(base + s) * 2];
    if (ms != -INFINITY) l += part_ml[(base + s) * 2 + 1] * expf(ms - mx);
  }
  const float inv = l > 0.f ? 1.f / l : 0.f;
  for (int d = threadIdx.x; d < dh; d += blockDim.x) {
    float acc = 0.f;
    for (int s = 0; s < nsplit; ++s) {
      const float ms = part_ml[(base + s) * 2];
      if (ms != -INFINITY) acc += part_o[(base + s) * dh + d] * expf(ms - mx);
    }
    out[(size_t)row * ldout + a * dh + d] = from_f<T>(acc * inv);
  }
}

template <typename T, int DH>
static int launch_core(const AttnArgs& p, int B, int M, cudaStream_t st) {
  dim3 grid(p.nsplit, p.A, B);
  attn_core_kernel<T, DH><<<grid, ATT_THREADS, 0, st>>>(p);
  if (int e = check_launch("tree_attention(core)")) return e;
  if (p.nsplit > 1) {
    attn_combine_kernel<T><<<dim3(M, p.A), 128, 0, st>>>(p.A, DH, p.nsplit, p.part_o, p.part_ml,
                                                         reinterpret_cast<T*>(p.out), p.ldout);
    if (int e = check_launch("tree_attention(combine)")) return e;
  }
  return 0;
}

// Split heuristic: aim for ~2 waves of CTAs over 148 SMs, >= 64 keys per split.
static int choose_splits(int B, int A, int max_keys, int max_splits) {
  const int ctas = B * A;
  int want = (2 * 148 + ctas - 1) / ctas;
  int cap = (max_keys + 63) / 64;
  if (want > cap) want = cap;
  if (want > max_splits) want = max_splits;
  return want < 1 ? 1 : want;
}

int attention_tc2_bf16(int B, int Bg, int M, int A, int Lmax, int n_slots, int max_rows_per_seq, int max_keys,
                       const void* qkv, int ldqkv, const void* kc, const void* vc, const int32_t* seq_slot,
                       const int32_t* seq_len, const int32_t* row_off, const int32_t* row_node, const uint64_t* mask,
                       int n_tmpl, int W, void* out, int ldout, void* ws, int64_t ws_bytes, cudaStream_t st,
                       bool* handled, bool qy = false);
int attention_tct_bf16(int B, int Bg, int A, int Lmax, int n_slots, int max_rows_per_seq, int max_keys, const void* qkv,
                       int ldqkv, const void* kc, const void* vc, const int32_t* seq_slot, const int32_t* seq_len,
                       const int32_t* row_off, const int32_t* row_node, const uint64_t* mask, int n_tmpl, int W,
                       void* out, int ldout, cudaStream_t st, bool force, bool* handled, bool qy = false);

int attention_decode_bf16(int B, int Bg, int M, int A, int Lmax, int max_rows_per_seq, int max_keys, const void* qkv,
                          int ldqkv, const void* kc, const void* vc, const int32_t* seq_slot, const int32_t* seq_len,
                          const int32_t* row_off, const int32_t* row_node, const uint64_t* mask, int n_tmpl, int W,
                          void* out, int ldout, void* ws, int64_t ws_bytes, cudaStream_t st, bool* handled, bool qy = false);

}  // namespace propd

using namespace propd;

static constexpr int kMaxSplits = 64;

namespace propd {
int attention_tc2_prepare();
int gemm_ws_prepare();
int gemm_ws_barrier_ctas();
}  // namespace propd

extern "C" {

int propd_prepare(void) {  // one-time function attributes + occupancy queries (before any graph capture)
  if (int e = propd::attention_tc2_prepare()) return e;
  return propd::gemm_ws_prepare();
}

int propd_gemm_ws_barrier_ctas(void) { return propd::gemm_ws_barrier_ctas(); }

int64_t propd_attn_workspace_bytes(int M, int A, int dh, int max_splits) {
  if (max_splits <= 0 || max_splits > kMaxSplits) max_splits = kMaxSplits;
  return (int64_t)M * A * max_splits * (dh + 2) * (int64_t)sizeof(float) + 256;
}

int propd_tree_attention(int dtype, int impl, int B, int M, int A, int dh, int Lmax, int n_slots,
                         int max_rows_per_seq, int max_keys, const void* qkv, int ldqkv, const void* kcache, const void* vcache,
                         const int32_t* seq_slot, const int32_t* seq_len, const int32_t* row_off,
                         const int32_t* row_node, const uint64_t* mask, int n_tmpl, int W, void* out, int ldout,
                         void* workspace, int64_t workspace_bytes, void* stream) {
  if (B == 0 || M == 0) return 0;
  // launch geometry counts the sequences with a real KV cache (not the scratch entry)
  const int Bg = (impl & PROPD_ATTN_SCRATCH_LAST) && B > 1 ? B - 1 : B;
  const bool qy = (impl & PROPD_ATTN_QKV_F32) != 0;
  impl &= 0xFF;
  if (qy) {  // fp32 QKV accumulator input: the decode (<= 4 rows) or the transposed kernel
    PROPD_REQUIRE(dtype == PROPD_BF16 && dh == 128 && mask != nullptr && (impl == 0 || impl == 3 || impl == 5),
                  "tree_attention: QKV_F32 input needs bf16, dh = 128, a mask and the decode / transposed kernel");
    bool handled = false;
    if (impl != 5 && max_rows_per_seq <= 4) {
      int e = attention_decode_bf16(B, Bg, M, A, Lmax, max_rows_per_seq, max_keys, qkv, ldqkv, kcache, vcache,
                                    seq_slot, seq_len, row_off, row_node, mask, n_tmpl, W, out, ldout, workspace,
                                    workspace_bytes, as_stream(stream), &handled, true);
      if (e || handled) return e;
    }
    // the transposed kernel, or the row-major one where its latency heuristic routes the shape (impl 0)
    int e = attention_tct_bf16(B, Bg, A, Lmax, n_slots, max_rows_per_seq, max_keys, qkv, ldqkv, kcache, vcache,
                               seq_slot, seq_len, row_off, row_node, mask, n_tmpl, W, out, ldout, as_stream(stream),
                               impl == 5, &handled, true);
    if (e || handled) return e;
    e = attention_tc2_bf16(B, Bg, M, A, Lmax, n_slots, max_rows_per_seq, max_keys, qkv, ldqkv, kcache, vcache,
                           seq_slot, seq_len, row_off, row_node, mask, n_tmpl, W, out, ldout, workspace,
                           workspace_bytes, as_stream(stream), &handled, true);
    if (e) return e;
    PROPD_REQUIRE(handled, "tree_attention: QKV_F32 input serves <= 64 rows per sequence (one row tile)");
    return 0;
  }
  PROPD_REQUIRE(mask == nullptr || (W <= ATT_MAXW && W * 64 >= n_tmpl),
                "tree_attention: template of %d nodes needs W=%d <= %d", n_tmpl, W, ATT_MAXW);
  PROPD_REQUIRE(max_keys >= 1, "tree_attention: max_keys must be positive");
  cudaStream_t st = as_stream(stream);
  if (impl == 3 || (impl == 0 && dtype == PROPD_BF16 && dh == 128 && max_rows_per_seq <= 4)) {
    bool handled = false;
    int e = attention_decode_bf16(B, Bg, M, A, Lmax, max_rows_per_seq, max_keys, qkv, ldqkv, kcache, vcache, seq_slot,
                                  seq_len, row_off, row_node, mask, n_tmpl, W, out, ldout, workspace,
                                  workspace_bytes, st, &handled);
    if (e || handled) return e;
    PROPD_REQUIRE(impl != 3, "tree_attention: decode kernel cannot serve this shape");
  }
  if (impl == 5 || (impl == 0 && dtype == PROPD_BF16 && dh == 128)) {  // <= 64 rows: transposed kernel
    bool handled = false;
    int e = attention_tct_bf16(B, Bg, A, Lmax, n_slots, max_rows_per_seq, max_keys, qkv, ldqkv, kcache, vcache, seq_slot,
                               seq_len, row_off, row_node, mask, n_tmpl, W, out, ldout, st, impl == 5, &handled);
    if (e || handled) return e;
    PROPD_REQUIRE(impl != 5, "tree_attention: transposed tcgen05 kernel serves <= 64 rows per sequence");
  }
  if (impl == 4 || (impl == 0 && dtype == PROPD_BF16 && dh == 128)) {
    bool handled = false;
    int e = attention_tc2_bf16(B, Bg, M, A, Lmax, n_slots, max_rows_per_seq, max_keys, qkv, ldqkv, kcache, vcache,
                               seq_slot, seq_len, row_off, row_node, mask, n_tmpl, W, out, ldout, workspace,
                               workspace_bytes, st, &handled);
    if (e || handled) return e;
    PROPD_REQUIRE(impl != 4, "tree_attention: tcgen05 v2 kernel cannot serve this shape");
  }
  AttnArgs p{};
  p.qkv = qkv;
  p.ldq = ldqkv;
  p.kc = kcache;
  p.vc = vcache;
  p.seq_slot = seq_slot;
  p.seq_len = seq_len;
  p.row_off = row_off;
  p.row_node = row_node;
  p.mask = mask;
  p.n_tmpl = n_tmpl;
  p.W = W;
  p.A = A;
  p.Lmax = Lmax;
  p.scale = 1.0f / sqrtf((float)dh);
  p.out = out;
  p.ldout = ldout;
  int nsplit = choose_splits(B, A, max_keys, kMaxSplits);
  const int64_t need = propd_attn_workspace_bytes(M, A, dh, nsplit);
  if (nsplit > 1 && (workspace == nullptr || workspace_bytes < need)) nsplit = 1;
  int split_len = (max_keys + nsplit - 1) / nsplit;
  split_len = ((split_len + ATT_TILE - 1) / ATT_TILE) * ATT_TILE;
  nsplit = (max_keys + split_len - 1) / split_len;
  p.split_len = split_len;
  p.nsplit = nsplit;
  p.part_o = reinterpret_cast<float*>(workspace);
  p.part_ml = p.part_o + (size_t)M * A * nsplit * dh;
  (void)max_rows_per_seq;
  return PROPD_DISPATCH_DTYPE(dtype, T, [&] {
    switch (dh) {
      case 16: return launch_core<T, 16>(p, B, M, st);
      case 32: return launch_core<T, 32>(p, B, M, st);
      case 64: return launch_core<T, 64>(p, B, M, st);
      case 128: return launch_core<T, 128>(p, B, M, st);
      default: return fail("tree_attention: head dim %d not in {16,32,64,128}", dh);
    }
  });
}

}  // extern "C"
