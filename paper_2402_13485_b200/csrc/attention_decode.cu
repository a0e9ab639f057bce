// K2 for few query rows per sequence (the bonus pass: 1 row; tiny trees):
// a streaming split-KV decode kernel on the CUDA cores.
//
// With one row per sequence there is no GEMM to feed a tensor core; the work
// is a pure stream of the sequence's K/V cache (backends.py:216-233 with
// n = 1).  A half-warp covers one key (16 lanes x 8 bf16 = the 256-byte
// row), so one warp-wide 16-byte load fetches two keys; scores are reduced
// with 4 shuffles, softmax is online per 8-key batch, and each lane
// accumulates 8 output dims.  Up to ROWS query rows share every K/V load.
#include "common.cuh"

namespace propd {

template <typename T>
__global__ void attn_combine_kernel(int A, int dh, int nsplit, const float* __restrict__ part_o,
                                    const float* __restrict__ part_ml, T* __restrict__ out, int ldout);

namespace dec {

constexpr int DH = 128, THREADS = 128, KB = 8;  // keys per half-warp batch

struct Args {
  const __nv_bfloat16* qkv;
  int ldq;
  const __nv_bfloat16* kc;
  const __nv_bfloat16* vc;
  const int32_t* seq_slot;
  const int32_t* seq_len;
  const int32_t* row_off;
  const int32_t* row_node;
  const uint64_t* mask;
  int n_tmpl, W, A, Lmax;
  float scale_log2;
  int split_len, nsplit;
  float* part_o;
  float* part_ml;
  __nv_bfloat16* out;
  int ldout;
  unsigned long long* tl;  // development timeline (common.cuh)
  unsigned int tag;
};

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ void bf16x8_to_f32(const uint4& u, float* f) {
  const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    f[2 * i] = __uint_as_float(w[i] << 16);
    f[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
  }
}

template <int ROWS>
__global__ void __launch_bounds__(THREADS) decode_kernel(Args p) {
  __shared__ float red_m[4][ROWS], red_l[4][ROWS];
  __shared__ float red_o[4][ROWS][DH];
  const int s = blockIdx.x, a = blockIdx.y, b = blockIdx.z;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int half = lane >> 4, hl = lane & 15;  // half-warp, lane within it (dims 8*hl .. 8*hl+7)
  const unsigned long long t_entry = p.tl ? gtimer() : 0ull;
  pdl_wait();
  const unsigned long long t_wait = p.tl ? gtimer() : 0ull;
  pdl_trigger();
  const int slot = p.seq_slot[b];
  const int L = p.seq_len[slot];
  const int r0 = p.row_off[b];
  const int nrows = p.row_off[b + 1] - r0;
  if (nrows <= 0) return;
  const int nkeys = L + p.n_tmpl;
  const int k_begin = s * p.split_len;
  const int k_end = min(nkeys, k_begin + p.split_len);

  // query rows (8 dims per lane) and their tree-visibility bitsets
  float q[ROWS][8];
  uint64_t bits[ROWS][4];
  int node[ROWS];
#pragma unroll
  for (int r = 0; r < ROWS; ++r) {
    node[r] = 0;
#pragma unroll
    for (int w = 0; w < 4; ++w) bits[r][w] = 0ull;
    if (r < nrows) {
      const uint4 u = *reinterpret_cast<const uint4*>(p.qkv + (size_t)(r0 + r) * p.ldq + a * DH + hl * 8);
      bf16x8_to_f32(u, q[r]);
      node[r] = p.row_node[r0 + r];
      if (p.mask != nullptr)
#pragma unroll
        for (int w = 0; w < 4; ++w)
          if (w < p.W) bits[r][w] = p.mask[(size_t)node[r] * p.W + w];
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) q[r][i] = 0.f;
    }
  }
  float m[ROWS], l[ROWS], o[ROWS][8];
#pragma unroll
  for (int r = 0; r < ROWS; ++r) {
    m[r] = -INFINITY;
    l[r] = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) o[r][i] = 0.f;
  }
  const size_t base = ((size_t)slot * p.A + a) * p.Lmax * DH + hl * 8;
  // each warp handles 2*KB consecutive keys per iteration (KB per half-warp)
  for (int k0 = k_begin + warp * 2 * KB; k0 < k_end; k0 += 4 * 2 * KB) {
    uint4 kr[KB], vr[KB];
#pragma unroll
    for (int t = 0; t < KB; ++t) {
      const int key = k0 + half * KB + t;
      const int kk = key < k_end ? key : k_end - 1;  // clamp: masked below
      kr[t] = *reinterpret_cast<const uint4*>(p.kc + base + (size_t)kk * DH);
      vr[t] = *reinterpret_cast<const uint4*>(p.vc + base + (size_t)kk * DH);
    }
#pragma unroll
    for (int r = 0; r < ROWS; ++r) {
      if (r >= nrows) break;
      float sc[KB];
#pragma unroll
      for (int t = 0; t < KB; ++t) {
        float kf[8];
        bf16x8_to_f32(kr[t], kf);
        float d = 0.f;
#pragma unroll
        for (int i = 0; i < 8; ++i) d = fmaf(q[r][i], kf[i], d);
#pragma unroll
        for (int off = 8; off > 0; off >>= 1) d += __shfl_xor_sync(0xffffffffu, d, off);
        const int key = k0 + half * KB + t;
        bool vis;
        if (key >= k_end) vis = false;
        else if (key < L) vis = true;
        else {
          const int tt = key - L;
          vis = p.mask == nullptr ? (tt <= node[r]) : (bool)((bits[r][tt >> 6] >> (tt & 63)) & 1ull);
        }
        sc[t] = vis ? d * p.scale_log2 : -INFINITY;
      }
      float mx = sc[0];
#pragma unroll
      for (int t = 1; t < KB; ++t) mx = fmaxf(mx, sc[t]);
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 16));  // both half-warps share (m, l)
      if (mx == -INFINITY) continue;
      const float mn = fmaxf(m[r], mx);
      const float corr = ex2(m[r] - mn);
      m[r] = mn;
      float ps = 0.f;
#pragma unroll
      for (int i = 0; i < 8; ++i) o[r][i] *= corr;
#pragma unroll
      for (int t = 0; t < KB; ++t) {
        const float pt = ex2(sc[t] - mn);
        ps += pt;
        float vf[8];
        bf16x8_to_f32(vr[t], vf);
#pragma unroll
        for (int i = 0; i < 8; ++i) o[r][i] = fmaf(pt, vf[i], o[r][i]);
      }
      ps += __shfl_xor_sync(0xffffffffu, ps, 16);
      l[r] = l[r] * corr + ps;
    }
  }
  // merge the two half-warps (same dims, different keys), then the 4 warps
#pragma unroll
  for (int r = 0; r < ROWS; ++r)
#pragma unroll
    for (int i = 0; i < 8; ++i) o[r][i] += __shfl_xor_sync(0xffffffffu, o[r][i], 16);
  if (half == 0) {
#pragma unroll
    for (int r = 0; r < ROWS; ++r) {
#pragma unroll
      for (int i = 0; i < 8; ++i) red_o[warp][r][hl * 8 + i] = o[r][i];
      if (hl == 0) {
        red_m[warp][r] = m[r];
        red_l[warp][r] = l[r];
      }
    }
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < ROWS * DH; idx += THREADS) {
    const int r = idx / DH, d = idx - r * DH;
    if (r >= nrows) continue;
    float mx = -INFINITY;
#pragma unroll
    for (int w = 0; w < 4; ++w) mx = fmaxf(mx, red_m[w][r]);
    float lsum = 0.f, acc = 0.f;
    if (mx != -INFINITY) {
#pragma unroll
      for (int w = 0; w < 4; ++w) {
        const float f = red_m[w][r] == -INFINITY ? 0.f : ex2(red_m[w][r] - mx);
        lsum += red_l[w][r] * f;
        acc += red_o[w][r][d] * f;
      }
    }
    const int row = r0 + r;
    if (p.nsplit == 1) {
      p.out[(size_t)row * p.ldout + a * DH + d] = __float2bfloat16_rn(lsum > 0.f ? acc / lsum : 0.f);
    } else {
      const size_t pb = ((size_t)row * p.A + a) * p.nsplit + s;
      p.part_o[pb * DH + d] = acc;
      if (d == 0) {
        p.part_ml[pb * 2] = mx == -INFINITY ? -INFINITY : mx * 0.69314718055994531f;
        p.part_ml[pb * 2 + 1] = lsum;
      }
    }
  }
  if (p.tl && threadIdx.x == 0) trace_record(p.tl, p.tag, t_entry, t_wait, t_wait);
}

}  // namespace dec

// Called by propd_tree_attention for bf16 / dh = 128 with <= 4 rows per sequence.
int attention_decode_bf16(int B, int M, int A, int Lmax, int max_rows_per_seq, int max_keys, const void* qkv,
                          int ldqkv, const void* kc, const void* vc, const int32_t* seq_slot, const int32_t* seq_len,
                          const int32_t* row_off, const int32_t* row_node, const uint64_t* mask, int n_tmpl, int W,
                          void* out, int ldout, void* ws, int64_t ws_bytes, cudaStream_t st, bool* handled) {
  *handled = false;
  if (max_rows_per_seq > 4 || W > 4 || (ldqkv % 8) != 0) return 0;
  // enough CTAs for ~4 per SM; >= 256 keys per split
  const int ctas = B * A;
  int nsplit = (4 * 148 + ctas - 1) / ctas;
  const int cap = (max_keys + 255) / 256;
  if (nsplit > cap) nsplit = cap;
  if (nsplit > 64) nsplit = 64;
  if (nsplit < 1) nsplit = 1;
  const int64_t need = (int64_t)M * A * nsplit * (dec::DH + 2) * (int64_t)sizeof(float);
  if (nsplit > 1 && (ws == nullptr || ws_bytes < need)) nsplit = 1;
  int split_len = (max_keys + nsplit - 1) / nsplit;
  split_len = ((split_len + 63) / 64) * 64;
  nsplit = (max_keys + split_len - 1) / split_len;
  dec::Args p{};
  p.qkv = reinterpret_cast<const __nv_bfloat16*>(qkv);
  p.ldq = ldqkv;
  p.kc = reinterpret_cast<const __nv_bfloat16*>(kc);
  p.vc = reinterpret_cast<const __nv_bfloat16*>(vc);
  p.seq_slot = seq_slot;
  p.seq_len = seq_len;
  p.row_off = row_off;
  p.row_node = row_node;
  p.mask = mask;
  p.n_tmpl = n_tmpl;
  p.W = W;
  p.A = A;
  p.Lmax = Lmax;
  p.scale_log2 = 1.4426950408889634f / sqrtf(128.f);
  p.split_len = split_len;
  p.nsplit = nsplit;
  p.part_o = reinterpret_cast<float*>(ws);
  p.part_ml = p.part_o + (size_t)M * A * nsplit * dec::DH;
  p.out = reinterpret_cast<__nv_bfloat16*>(out);
  p.ldout = ldout;
  p.tl = g_dbg_trace;
  p.tag = g_dbg_tag++;
  *handled = true;
  dim3 grid(nsplit, A, B);
  int e = 0;
  switch (max_rows_per_seq) {
    case 1: e = launch_pdl("tree_attention(decode)", dec::decode_kernel<1>, grid, dim3(dec::THREADS), 0, st, p); break;
    case 2: e = launch_pdl("tree_attention(decode)", dec::decode_kernel<2>, grid, dim3(dec::THREADS), 0, st, p); break;
    default: e = launch_pdl("tree_attention(decode)", dec::decode_kernel<4>, grid, dim3(dec::THREADS), 0, st, p); break;
  }
  if (e) return e;
  if (nsplit > 1) {
    if (int e2 = launch_pdl("tree_attention(decode combine)", attn_combine_kernel<__nv_bfloat16>, dim3(M, A),
                            dim3(128), 0, st, A, dec::DH, nsplit, (const float*)p.part_o, (const float*)p.part_ml,
                            p.out, ldout))
      return e2;
  }
  return 0;
}

}  // namespace propd
