#include <cstring>
// Row-level kernels of the tree pass: K1 tree materialisation + embedding,
// residual/LN/GELU helpers, KV append, argmax and stable top-k.
//
// Reference semantics (paths relative to /root/reference/pkg/src/treedecode/):
//   build_tree canonical order + positions  token_tree.py:125-170, engine.py:260
//   x = emb[tok] + pos[pos]                 backends.py:315
//   _ln / _gelu                              backends.py:135-142
//   argmax (first max)                       backends.py:288, 333
//   stable argsort top-k                     backends.py:282, 323
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <string>

#include "common.cuh"

namespace propd {

static thread_local std::string g_error;

void set_error(const std::string& msg) { g_error = msg; }

int fail(const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_error = buf;
  return 1;
}

bool pdl_enabled() {
  static const bool on = [] {
    const char* v = getenv("PROPD_PDL");
    return !(v && v[0] == '0');
  }();
  return on;
}

bool pdl_skip(const char* what) {
  static const char* skip = getenv("PROPD_PDL_SKIP");
  return skip != nullptr && strstr(skip, what) != nullptr;
}

int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail("%s: %s", what, cudaGetErrorString(e));
  return 0;
}

// x row = emb row + pos row (fp32 out): 16-byte loads of 8 bf16 (or 4 fp32)
// elements per thread when the width allows it (the K1 / bonus / prefill
// embeds: one dependent gather per row, latency-bound at small batch)
template <typename T>
__device__ __forceinline__ void embed_add_row(const T* __restrict__ e, const T* __restrict__ q, float* __restrict__ o,
                                              int H) {
  constexpr int VW = 16 / sizeof(T);  // elements per 16-byte load
  if (H % VW == 0 && (reinterpret_cast<uintptr_t>(e) & 15) == 0 && (reinterpret_cast<uintptr_t>(q) & 15) == 0 &&
      (reinterpret_cast<uintptr_t>(o) & 15) == 0) {
    for (int h = threadIdx.x * VW; h < H; h += blockDim.x * VW) {
      const uint4 ev = __ldg(reinterpret_cast<const uint4*>(e + h));
      const uint4 qv = __ldg(reinterpret_cast<const uint4*>(q + h));
      const T* ea = reinterpret_cast<const T*>(&ev);
      const T* qa = reinterpret_cast<const T*>(&qv);
#pragma unroll
      for (int k = 0; k < VW; k += 4)
        *reinterpret_cast<float4*>(o + h + k) = make_float4(to_f(ea[k]) + to_f(qa[k]), to_f(ea[k + 1]) + to_f(qa[k + 1]),
                                                            to_f(ea[k + 2]) + to_f(qa[k + 2]),
                                                            to_f(ea[k + 3]) + to_f(qa[k + 3]));
    }
  } else {
    for (int h = threadIdx.x; h < H; h += blockDim.x) o[h] = to_f(e[h]) + to_f(q[h]);
  }
}

// ---------------------------------------------------------------- K1 ------
template <typename T>
__global__ void tree_embed_kernel(int n, int D, int kmax, int H, const int32_t* __restrict__ depth,
                                  const int32_t* __restrict__ rank, const int32_t* __restrict__ draft_tok,
                                  const int32_t* __restrict__ seq_slot, const int32_t* __restrict__ seq_len,
                                  const T* __restrict__ emb, const T* __restrict__ pos,
                                  int32_t* tokens, int32_t* positions, float* __restrict__ x,
                                  int32_t* row_seq, int32_t* row_node, int32_t* row_off, int B) {
  const int m = blockIdx.x;
  const int b = m / n, i = m - b * n;
  const int d = depth[i], r = rank[i];
  const int tok = draft_tok[((size_t)b * D + (d - 1)) * kmax + (r - 1)];
  const int p = seq_len[seq_slot[b]] + d - 1;
  if (threadIdx.x == 0) {
    tokens[m] = tok;
    positions[m] = p;
    row_seq[m] = b;
    row_node[m] = i;
    if (i == 0) row_off[b] = b * n;
    if (m == 0) row_off[B] = B * n;
  }
  const T* e = emb + (size_t)tok * H;
  const T* q = pos + (size_t)p * H;
  float* o = x + (size_t)m * H;
  embed_add_row(e, q, o, H);
}

template <typename T>
__global__ void embed_rows_kernel(int H, const int32_t* __restrict__ tokens, const int32_t* __restrict__ positions,
                                  const T* __restrict__ emb, const T* __restrict__ pos, float* __restrict__ x) {
  const int m = blockIdx.x;
  const T* e = emb + (size_t)tokens[m] * H;
  const T* q = pos + (size_t)positions[m] * H;
  float* o = x + (size_t)m * H;
  embed_add_row(e, q, o, H);
}

template <typename T>
__global__ void bonus_embed_kernel(int B, int H, const int32_t* __restrict__ bonus,
                                   const int32_t* __restrict__ seq_slot, const int32_t* __restrict__ seq_len,
                                   const T* __restrict__ emb, const T* __restrict__ pos, float* __restrict__ x,
                                   int32_t* positions, int32_t* row_seq, int32_t* row_node, int32_t* row_off) {
  const int b = blockIdx.x;
  const int p = seq_len[seq_slot[b]];
  const int tok = bonus[b];
  if (threadIdx.x == 0) {
    positions[b] = p;
    row_seq[b] = b;
    row_node[b] = 0;
    row_off[b] = b;
    if (b == 0) row_off[B] = B;
  }
  const T* e = emb + (size_t)tok * H;
  const T* q = pos + (size_t)p * H;
  float* o = x + (size_t)b * H;
  embed_add_row(e, q, o, H);
}

// ------------------------------------------------------------- dense ------
// One row per CTA at a time, the row held in registers (8 floats per thread
// per chunk): x (+ delta) is read once, the residual written back once, the
// normalised row written once.  Two-pass mean / variance like numpy's
// x.var() (the second pass runs over registers).  The grid is capped at a
// few CTAs per SM and strides over the live rows: a capacity-sized grid of
// thousands of one-row CTAs (post-prune passes at B >= 16, mostly dead rows)
// is CTA-launch-rate bound and held the next many-row GEMM's CTAs off ~1/3
// of the SMs for ~15 us (measured at B=32).
template <typename T, int CHUNKS>
__global__ void __launch_bounds__(512) add_ln_vec_kernel(int M, int H, float* __restrict__ x,
                                                          const T* __restrict__ delta, T* __restrict__ out,
                                                          const int32_t* __restrict__ in_idx,
                                                          const int32_t* __restrict__ out_idx,
                                                          const int32_t* __restrict__ rows_dev,
                                                          unsigned long long* trace, unsigned int tag) {
  __shared__ float red[32];
  const unsigned long long t_entry = trace ? gtimer() : 0ull;
  pdl_trigger();  // early: the dependent only prefetches weights before its own wait
  pdl_wait();
  const unsigned long long t_wait = trace ? gtimer() : 0ull;
  const int rows = rows_dev ? min(M, *rows_dev) : M;
  for (int m = blockIdx.x; m < rows; m += gridDim.x) {
  const int src = in_idx ? in_idx[m] : m;
  const int dst = out_idx ? out_idx[m] : m;
  float* xr = x + (size_t)src * H;
  float v[CHUNKS][8];
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < CHUNKS; ++c) {
    const int h = (c * blockDim.x + threadIdx.x) * 8;
    if (h < H) {
      const float4 a = *reinterpret_cast<const float4*>(xr + h);
      const float4 b = *reinterpret_cast<const float4*>(xr + h + 4);
      v[c][0] = a.x; v[c][1] = a.y; v[c][2] = a.z; v[c][3] = a.w;
      v[c][4] = b.x; v[c][5] = b.y; v[c][6] = b.z; v[c][7] = b.w;
      if (delta) {
        const T* dr = delta + (size_t)src * H + h;
#pragma unroll
        for (int i = 0; i < 8; ++i) v[c][i] += to_f(dr[i]);
        *reinterpret_cast<float4*>(xr + h) = make_float4(v[c][0], v[c][1], v[c][2], v[c][3]);
        *reinterpret_cast<float4*>(xr + h + 4) = make_float4(v[c][4], v[c][5], v[c][6], v[c][7]);
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) s += v[c][i];
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) v[c][i] = 0.f;
    }
  }
  const float mu = block_sum(s, red) / (float)H;
  float ss = 0.f;
#pragma unroll
  for (int c = 0; c < CHUNKS; ++c) {
    const int h = (c * blockDim.x + threadIdx.x) * 8;
    if (h < H) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float d = v[c][i] - mu;
        ss += d * d;
      }
    }
  }
  const float den = sqrtf(block_sum(ss, red) / (float)H + 1e-5f);
  T* o = out + (size_t)dst * H;
#pragma unroll
  for (int c = 0; c < CHUNKS; ++c) {
    const int h = (c * blockDim.x + threadIdx.x) * 8;
    if (h < H) {
#pragma unroll
      for (int i = 0; i < 8; ++i) o[h + i] = from_f<T>((v[c][i] - mu) / den);
    }
  }
  }
  if (trace && threadIdx.x == 0) trace_record(trace, tag, t_entry, t_wait, t_wait, 6ull);
}

// Wide rows (H % (128 * WPR) == 0, <= 32 float4 per lane): WPR warps per row
// (one at H = 4096), the row in registers, no CTA-wide barrier per row
// (warp shuffles; WPR > 1 exchanges two partial sums through shared memory
// with a named barrier per row group), 16- / 8-byte vector loads and stores,
// rows strided over a grid of a few CTAs per SM.  Measured standalone at
// 512 live rows: 11.4 us for the one-row-per-CTA kernel above.
template <typename T, int WPR, int NV4>
__global__ void __launch_bounds__(64 * WPR) add_ln_warp_kernel(int M, int H, float* __restrict__ x,
                                                          const T* __restrict__ delta, T* __restrict__ out,
                                                          const int32_t* __restrict__ in_idx,
                                                          const int32_t* __restrict__ out_idx,
                                                          const int32_t* __restrict__ rows_dev,
                                                          unsigned long long* trace, unsigned int tag) {
  constexpr int RPC = 2;  // rows per CTA pass (64 * WPR threads)
  __shared__ float red[2 * WPR][2];
  const unsigned long long t_entry = trace ? gtimer() : 0ull;
  pdl_trigger();
  pdl_wait();
  const unsigned long long t_wait = trace ? gtimer() : 0ull;
  const int rows = rows_dev ? min(M, *rows_dev) : M;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, grp = warp / WPR, wr = warp % WPR;
  for (int m = blockIdx.x * RPC + grp; m < rows; m += gridDim.x * RPC) {
    const int src = in_idx ? in_idx[m] : m;
    const int dst = out_idx ? out_idx[m] : m;
    float4* xr = reinterpret_cast<float4*>(x + (size_t)src * H) + wr * NV4 * 32;
    float4 v[NV4];
#pragma unroll
    for (int j = 0; j < NV4; ++j) v[j] = xr[j * 32 + lane];
    if (delta) {
      const T* dr = delta + (size_t)src * H + (size_t)wr * NV4 * 128;
#pragma unroll
      for (int j = 0; j < NV4; ++j) {
        const int e = (j * 32 + lane) * 4;
        v[j].x += to_f(dr[e]);
        v[j].y += to_f(dr[e + 1]);
        v[j].z += to_f(dr[e + 2]);
        v[j].w += to_f(dr[e + 3]);
        xr[j * 32 + lane] = v[j];
      }
    }
    float s = 0.f;
#pragma unroll
    for (int j = 0; j < NV4; ++j) s += (v[j].x + v[j].y) + (v[j].z + v[j].w);
    s = warp_sum(s);
    if (WPR > 1) {
      if (lane == 0) red[warp][0] = s;
      asm volatile("bar.sync %0, %1;" ::"r"(1 + grp), "r"(32 * WPR) : "memory");
      s = 0.f;
#pragma unroll
      for (int i = 0; i < WPR; ++i) s += red[grp * WPR + i][0];
    }
    const float mu = s / (float)H;
    float ss = 0.f;
#pragma unroll
    for (int j = 0; j < NV4; ++j) {
      const float a = v[j].x - mu, b = v[j].y - mu, c = v[j].z - mu, d = v[j].w - mu;
      ss += (a * a + b * b) + (c * c + d * d);
    }
    ss = warp_sum(ss);
    if (WPR > 1) {
      if (lane == 0) red[warp][1] = ss;
      asm volatile("bar.sync %0, %1;" ::"r"(1 + grp), "r"(32 * WPR) : "memory");
      ss = 0.f;
#pragma unroll
      for (int i = 0; i < WPR; ++i) ss += red[grp * WPR + i][1];
    }
    const float inv = 1.f / sqrtf(ss / (float)H + 1e-5f);
    T* o = out + (size_t)dst * H + (size_t)wr * NV4 * 128;
#pragma unroll
    for (int j = 0; j < NV4; ++j) {
      const int e = (j * 32 + lane) * 4;
      if constexpr (sizeof(T) == 2) {
        __nv_bfloat162 lo = __floats2bfloat162_rn((v[j].x - mu) * inv, (v[j].y - mu) * inv);
        __nv_bfloat162 hi = __floats2bfloat162_rn((v[j].z - mu) * inv, (v[j].w - mu) * inv);
        *reinterpret_cast<uint2*>(o + e) =
            make_uint2(*reinterpret_cast<uint32_t*>(&lo), *reinterpret_cast<uint32_t*>(&hi));
      } else {
        *reinterpret_cast<float4*>(o + e) =
            make_float4((v[j].x - mu) * inv, (v[j].y - mu) * inv, (v[j].z - mu) * inv, (v[j].w - mu) * inv);
      }
    }
    if (WPR > 1) asm volatile("bar.sync %0, %1;" ::"r"(1 + grp), "r"(32 * WPR) : "memory");  // red reuse
  }
  if (trace && threadIdx.x == 0) trace_record(trace, tag, t_entry, t_wait, t_wait, 6ull);
}

// Scalar fallback for widths that are not a multiple of 8.
template <typename T>
__global__ void add_ln_kernel(int H, float* __restrict__ x, const T* __restrict__ delta, T* __restrict__ out,
                              const int32_t* __restrict__ in_idx, const int32_t* __restrict__ out_idx) {
  __shared__ float red[32];
  const int m = blockIdx.x;
  const int src = in_idx ? in_idx[m] : m;
  const int dst = out_idx ? out_idx[m] : m;
  float* xr = x + (size_t)src * H;
  float s = 0.f;
  if (delta) {
    const T* dr = delta + (size_t)src * H;
    for (int h = threadIdx.x; h < H; h += blockDim.x) {
      float v = xr[h] + to_f(dr[h]);
      xr[h] = v;
      s += v;
    }
  } else {
    for (int h = threadIdx.x; h < H; h += blockDim.x) s += xr[h];
  }
  const float mu = block_sum(s, red) / (float)H;
  float ss = 0.f;
  for (int h = threadIdx.x; h < H; h += blockDim.x) {
    float c = xr[h] - mu;
    ss += c * c;
  }
  const float var = block_sum(ss, red) / (float)H;
  const float den = sqrtf(var + 1e-5f);
  T* o = out + (size_t)dst * H;
  for (int h = threadIdx.x; h < H; h += blockDim.x) o[h] = from_f<T>((xr[h] - mu) / den);
}

template <typename T>
__global__ void gelu_kernel(int64_t count, T* __restrict__ buf) {
  const float c = 0.7978845608028654f;  // sqrt(2/pi)
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
    float v = to_f(buf[i]);
    buf[i] = from_f<T>(0.5f * v * (1.f + tanhf(c * (v + 0.044715f * v * v * v))));
  }
}

template <typename T>
__global__ void residual_add_kernel(int64_t count, float* __restrict__ x, const T* __restrict__ d) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
    x[i] += to_f(d[i]);
}

template <typename T>
__global__ void gather_rows_kernel(int H, const float* __restrict__ src, const int32_t* __restrict__ idx,
                                   T* __restrict__ dst) {
  const int m = blockIdx.x;
  const float* s = src + (size_t)(idx ? idx[m] : m) * H;
  T* d = dst + (size_t)m * H;
  if (H % 4 == 0 && (reinterpret_cast<uintptr_t>(s) & 15) == 0 && (reinterpret_cast<uintptr_t>(d) & 7) == 0) {
    for (int h = threadIdx.x * 4; h < H; h += blockDim.x * 4) {  // 16-byte loads, 4 elements per thread
      const float4 v = __ldg(reinterpret_cast<const float4*>(s + h));
      d[h] = from_f<T>(v.x);
      d[h + 1] = from_f<T>(v.y);
      d[h + 2] = from_f<T>(v.z);
      d[h + 3] = from_f<T>(v.w);
    }
  } else {
    for (int h = threadIdx.x; h < H; h += blockDim.x) d[h] = from_f<T>(s[h]);
  }
}

// First maximum of each row (numpy argmax semantics).  The scan is latency-bound (one row per CTA,
// ~20 rows at batch 1), so every thread keeps 4 float4 loads in flight; each
// thread still visits its indices in increasing order, so "first max" per
// thread plus the (value, lower index) reduction is the first max of the row.
__device__ __forceinline__ void argmax_take(float t, int v, float& best, int& bi) {
  if (t > best) {
    best = t;
    bi = v;
  }
}
__global__ void __launch_bounds__(512) argmax_rows_kernel(int M, int V, int ld, const float* __restrict__ logits,
                                                            int32_t* __restrict__ out,
                                                            const int32_t* __restrict__ rows_dev) {
  __shared__ float sv[32];
  __shared__ int si[32];
  // rows strided over a grid of <= 2 CTAs per SM (a capacity-sized grid of
  // mostly dead rows is CTA-launch-rate bound at large batch)
  const int rows = rows_dev ? min((int)M, *rows_dev) : (int)M;
  for (int row = blockIdx.x; row < rows; row += gridDim.x) {
  const float* x = logits + (size_t)row * ld;
  float best = -INFINITY;
  int bi = 0x7fffffff;
  const bool vec = ((ld & 3) == 0) && ((reinterpret_cast<uintptr_t>(logits) & 15) == 0);
  const int V4 = vec ? (V >> 2) : 0;
  const float4* x4 = reinterpret_cast<const float4*>(x);
  constexpr int U = 4;
  for (int base = threadIdx.x; base < V4; base += U * blockDim.x) {
    float4 f[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = base + u * blockDim.x;
      f[u] = i < V4 ? __ldg(x4 + i) : make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int v = 4 * (base + u * blockDim.x);
      argmax_take(f[u].x, v, best, bi);
      argmax_take(f[u].y, v + 1, best, bi);
      argmax_take(f[u].z, v + 2, best, bi);
      argmax_take(f[u].w, v + 3, best, bi);
    }
  }
  for (int v = 4 * V4 + threadIdx.x; v < V; v += blockDim.x) argmax_take(x[v], v, best, bi);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    float ov = __shfl_xor_sync(0xffffffffu, best, o);
    int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) { sv[wid] = best; si[wid] = bi; }
  __syncthreads();
  if (wid == 0) {
    const int nw = blockDim.x >> 5;
    best = lane < nw ? sv[lane] : -INFINITY;
    bi = lane < nw ? si[lane] : 0x7fffffff;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      float ov = __shfl_xor_sync(0xffffffffu, best, o);
      int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
    }
    if (lane == 0) out[row] = bi;
  }
  __syncthreads();  // sv / si reused by the next row
  }
}

// Stable descending top-k: radix select on the unique 64-bit key
// (float_key(x) << 32) | ~index, then bitonic sort of the k winners.
constexpr int TOPK_MAX = 1024;
// The row is staged once in shared memory when it fits (every radix pass
// re-reads it; V = 32000 is 125 KB), read from global memory otherwise.
constexpr int TOPK_SMEM_MAX = 48 * 1024;  // floats staged (192 KB)
__global__ void __launch_bounds__(512) topk_rows_kernel(int V, int ld, int k, const float* __restrict__ logits,
                                                          int32_t* __restrict__ out_idx, float* __restrict__ out_val) {
  __shared__ unsigned hist[256];
  __shared__ unsigned long long cand[TOPK_MAX];
  __shared__ unsigned long long s_prefix;
  __shared__ int s_shift, s_need, s_done, s_cnt;
  extern __shared__ float4 row_s[];
  const float* xg = logits + (size_t)blockIdx.x * ld;
  const float* x = xg;
  if (V <= TOPK_SMEM_MAX) {
    float* rs = reinterpret_cast<float*>(row_s);
    if (((ld & 3) == 0) && ((reinterpret_cast<uintptr_t>(logits) & 15) == 0)) {
      const float4* g4 = reinterpret_cast<const float4*>(xg);
      for (int i = threadIdx.x; i < (V >> 2); i += blockDim.x) row_s[i] = __ldg(g4 + i);
      for (int v = 4 * (V >> 2) + threadIdx.x; v < V; v += blockDim.x) rs[v] = xg[v];
    } else {
      for (int v = threadIdx.x; v < V; v += blockDim.x) rs[v] = xg[v];
    }
    x = rs;
    __syncthreads();
  }
  auto key_of = [&](int v) -> unsigned long long {
    return ((unsigned long long)float_key(x[v]) << 32) | (unsigned long long)(0xffffffffu - (unsigned)v);
  };
  if (threadIdx.x == 0) { s_prefix = 0ull; s_need = k; s_done = 0; s_shift = 56; s_cnt = 0; }
  __syncthreads();
  for (int pass = 0; pass < 8; ++pass) {
    const int shift = 56 - 8 * pass;
    for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0u;
    __syncthreads();
    const unsigned long long pre = s_prefix;
    for (int v = threadIdx.x; v < V; v += blockDim.x) {
      unsigned long long kk = key_of(v);
      if (pass == 0 || (kk >> (shift + 8)) == (pre >> (shift + 8))) atomicAdd(&hist[(kk >> shift) & 255u], 1u);
    }
    __syncthreads();
    if (threadIdx.x < 32) {
      // the bin holding the need-th largest key: lane l owns bins 255-8l .. 248-8l
      // (descending), a warp scan of the lane totals finds the lane, the lane
      // walks its 8 bins (a serial scan of 256 bins cost ~1-2 us per pass)
      const int lane = threadIdx.x, need = s_need;
      unsigned c[8], tot = 0;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        c[i] = hist[255 - 8 * lane - i];
        tot += c[i];
      }
      unsigned incl = tot;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const unsigned t = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= off) incl += t;
      }
      const unsigned excl = incl - tot;
      if (excl < (unsigned)need && (unsigned)need <= incl) {
        unsigned cum = excl;
        int bsel = 255 - 8 * lane - 7;
        unsigned cnt = c[7];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          if (cum + c[i] >= (unsigned)need) {
            bsel = 255 - 8 * lane - i;
            cnt = c[i];
            break;
          }
          cum += c[i];
        }
        const int left = need - (int)cum;  // still needed from bucket bsel
        s_prefix = pre | ((unsigned long long)bsel << shift);
        s_shift = shift;
        s_need = left;
        if (cnt == (unsigned)left) s_done = 1;
      }
    }
    __syncthreads();
    if (s_done) break;
  }
  // winners: top (64 - shift) bits >= prefix bits  (exactly k elements)
  const int shift = s_shift;
  const unsigned long long thr = s_prefix >> shift;
  for (int v = threadIdx.x; v < V; v += blockDim.x) {
    unsigned long long kk = key_of(v);
    if ((kk >> shift) >= thr) {
      int p = atomicAdd(&s_cnt, 1);
      if (p < TOPK_MAX) cand[p] = kk;
    }
  }
  __syncthreads();
  int P2 = 1;
  while (P2 < k) P2 <<= 1;
  for (int i = k + threadIdx.x; i < P2; i += blockDim.x) cand[i] = 0ull;
  __syncthreads();
  // bitonic sort, descending
  for (int size = 2; size <= P2; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = threadIdx.x; i < P2; i += blockDim.x) {
        int j = i ^ stride;
        if (j > i) {
          bool desc = ((i & size) == 0);
          unsigned long long a = cand[i], c = cand[j];
          if (desc ? (a < c) : (a > c)) { cand[i] = c; cand[j] = a; }
        }
      }
      __syncthreads();
    }
  }
  for (int i = threadIdx.x; i < k; i += blockDim.x) {
    int v = (int)(0xffffffffu - (unsigned)(cand[i] & 0xffffffffull));
    out_idx[(size_t)blockIdx.x * k + i] = v;
    if (out_val) out_val[(size_t)blockIdx.x * k + i] = x[v];
  }
}

// ------------------------------------------------------------ KV cache ----
template <typename T>
__global__ void kv_append_kernel(int A, int dh, int Lmax, const T* __restrict__ qkv, int ld,
                                 const int32_t* __restrict__ row_seq, const int32_t* __restrict__ row_node,
                                 const int32_t* __restrict__ seq_slot, const int32_t* __restrict__ seq_len,
                                 T* __restrict__ kc, T* __restrict__ vc) {
  // blockIdx.x = row, blockIdx.y = 0 (K) / 1 (V); 16-byte vectors
  constexpr int VEC = 16 / sizeof(T);
  const int m = blockIdx.x;
  const int b = row_seq[m];
  const int slot = seq_slot[b];
  const int t = seq_len[slot] + row_node[m];
  const int H = A * dh;
  const T* src = qkv + (size_t)m * ld + (1 + blockIdx.y) * H;
  T* dst = blockIdx.y == 0 ? kc : vc;
  for (int e = threadIdx.x * VEC; e < H; e += blockDim.x * VEC) {
    const int a = e / dh, d = e - a * dh;
    *reinterpret_cast<uint4*>(dst + (((size_t)slot * A + a) * Lmax + t) * dh + d) =
        *reinterpret_cast<const uint4*>(src + e);
  }
}

__global__ void seq_advance_kernel(int B, const int32_t* seq_slot, int32_t* seq_len, const int32_t* delta_dev, int delta) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b < B) seq_len[seq_slot[b]] += delta_dev ? delta_dev[b] : delta;
}

__global__ void scatter_i32_kernel(int B, const int32_t* idx, const int32_t* src, int32_t* dst) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b < B) dst[idx[b]] = src[b];
}

static int threads_for(int H) {
  int t = ((H + 31) / 32) * 32;
  return t < 256 ? t : 256;
}

}  // namespace propd

using namespace propd;

namespace propd {
unsigned long long* g_dbg_trace = nullptr;
unsigned int g_dbg_tag = 0;
}  // namespace propd

extern "C" {

int propd_debug_timeline(void* buf) {  // development aid: per-CTA timeline records (common.cuh)
  propd::g_dbg_trace = reinterpret_cast<unsigned long long*>(buf);
  propd::g_dbg_tag = 0;
  return 0;
}

const char* propd_last_error(void) { return g_error.c_str(); }
int propd_abi_version(void) { return 5; }
int propd_num_sms(void) {
  static int cached = 0;  // launch heuristics call this per launch
  if (cached > 0) return cached;
  int dev = 0, n = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) { cudaGetLastError(); return 0; }
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) { cudaGetLastError(); return 0; }
  cached = n;
  return n;
}

int propd_tree_embed(int dtype, int B, int n, int D, int kmax, int H, const int32_t* depth, const int32_t* rank,
                     const int32_t* draft_tok, const int32_t* seq_slot, const int32_t* seq_len, const void* emb,
                     const void* pos, int32_t* tokens, int32_t* positions, float* x, int32_t* row_seq,
                     int32_t* row_node, int32_t* row_off, void* stream) {
  PROPD_REQUIRE(B > 0 && n > 0 && H > 0, "tree_embed: empty batch/tree (B=%d n=%d H=%d)", B, n, H);
  return PROPD_DISPATCH_DTYPE(dtype, T, [&] {
    tree_embed_kernel<T><<<B * n, threads_for(H), 0, as_stream(stream)>>>(
        n, D, kmax, H, depth, rank, draft_tok, seq_slot, seq_len, (const T*)emb, (const T*)pos, tokens, positions,
        x, row_seq, row_node, row_off, B);
    return check_launch("tree_embed");
  });
}

int propd_embed_rows(int dtype, int M, int H, const int32_t* tokens, const int32_t* positions, const void* emb,
                     const void* pos, float* x, void* stream) {
  if (M == 0) return 0;
  return PROPD_DISPATCH_DTYPE(dtype, T, [&] {
    embed_rows_kernel<T><<<M, threads_for(H), 0, as_stream(stream)>>>(H, tokens, positions, (const T*)emb,
                                                                        (const T*)pos, x);
    return check_launch("embed_rows");
  });
}

int propd_bonus_embed(int dtype, int B, int H, const int32_t* bonus, const int32_t* seq_slot, const int32_t* seq_len,
                      const void* emb, const void* pos, float* x, int32_t* positions, int32_t* row_seq,
                      int32_t* row_node, int32_t* row_off, void* stream) {
  if (B == 0) return 0;
  return PROPD_DISPATCH_DTYPE(dtype, T, [&] {
    bonus_embed_kernel<T><<<B, threads_for(H), 0, as_stream(stream)>>>(B, H, bonus, seq_slot, seq_len, (const T*)emb,
                                                                        (const T*)pos, x, positions, row_seq,
                                                                        row_node, row_off);
    return check_launch("bonus_embed");
  });
}

int propd_add_ln(int dtype, int M, const int32_t* rows_dev, int H, float* x, const void* delta, void* out,
                 const int32_t* in_idx, const int32_t* out_idx, void* stream) {
  if (M == 0) return 0;
  return PROPD_DISPATCH_DTYPE(dtype, T, [&] {
    cudaStream_t st = as_stream(stream);
    const int wgrid = (M + 1) / 2 < 4 * propd_num_sms() ? (M + 1) / 2 : 4 * propd_num_sms();  // 2 rows per CTA
    const bool aligned = (reinterpret_cast<uintptr_t>(x) & 15) == 0 && (reinterpret_cast<uintptr_t>(out) & 15) == 0;
    if (aligned && H == 4096)
      return launch_pdl("add_ln", add_ln_warp_kernel<T, 1, 32>, dim3(wgrid), dim3(64), 0, st, M, H, x,
                        (const T*)delta, (T*)out, in_idx, out_idx, rows_dev, g_dbg_trace, g_dbg_tag++);
    if (aligned && H == 6656)  // 33B shape: two warps per row
      return launch_pdl("add_ln", add_ln_warp_kernel<T, 2, 26>, dim3(wgrid), dim3(128), 0, st, M, H, x,
                        (const T*)delta, (T*)out, in_idx, out_idx, rows_dev, g_dbg_trace, g_dbg_tag++);
    if (H % 8 == 0 && H <= 8 * 512 * 4) {
      // 8 elements per thread per chunk; pick threads so that <= 4 chunks
      int threads = 32;
      while (threads * 8 * 4 < H) threads *= 2;
      if (threads > 512) threads = 512;
      const int chunks = (H + threads * 8 - 1) / (threads * 8);
      const int grid = M < 4 * propd_num_sms() ? M : 4 * propd_num_sms();  // rows strided over the CTAs
      switch (chunks) {
        case 1: return launch_pdl("add_ln", add_ln_vec_kernel<T, 1>, dim3(grid), dim3(threads), 0, st, M, H, x, (const T*)delta, (T*)out, in_idx, out_idx, rows_dev, g_dbg_trace, g_dbg_tag++);
        case 2: return launch_pdl("add_ln", add_ln_vec_kernel<T, 2>, dim3(grid), dim3(threads), 0, st, M, H, x, (const T*)delta, (T*)out, in_idx, out_idx, rows_dev, g_dbg_trace, g_dbg_tag++);
        case 3: return launch_pdl("add_ln", add_ln_vec_kernel<T, 3>, dim3(grid), dim3(threads), 0, st, M, H, x, (const T*)delta, (T*)out, in_idx, out_idx, rows_dev, g_dbg_trace, g_dbg_tag++);
        default: return launch_pdl("add_ln", add_ln_vec_kernel<T, 4>, dim3(grid), dim3(threads), 0, st, M, H, x, (const T*)delta, (T*)out, in_idx, out_idx, rows_dev, g_dbg_trace, g_dbg_tag++);
      }
    } else {
      PROPD_REQUIRE(rows_dev == nullptr, "add_ln: rows_dev needs H %% 8 == 0");
      add_ln_kernel<T><<<M, threads_for(H), 0, st>>>(H, x, (const T*)delta, (T*)out, in_idx, out_idx);
    }
    return check_launch("add_ln");
  });
}

int propd_gelu(int dtype, int64_t count, void* buf, void* stream) {
  if (count == 0) return 0;
  int blocks = (int)((count + 255) / 256);
  if (blocks > 148 * 16) blocks = 148 * 16;
  return PROPD_DISPATCH_DTYPE(dtype, T, [&] {
    gelu_kernel<T><<<blocks, 256, 0, as_stream(stream)>>>(count, (T*)buf);
    return check_launch("gelu");
  });
}

int propd_residual_add(int dtype, int64_t count, float* x, const void* delta, void* stream) {
  if (count == 0) return 0;
  int blocks = (int)((count + 255) / 256);
  if (blocks > 148 * 16) blocks = 148 * 16;
  return PROPD_DISPATCH_DTYPE(dtype, T, [&] {
    residual_add_kernel<T><<<blocks, 256, 0, as_stream(stream)>>>(count, x, (const T*)delta);
    return check_launch("residual_add");
  });
}

int propd_gather_rows(int dtype, int M, int H, const float* src, const int32_t* idx, void* dst, void* stream) {
  if (M == 0) return 0;
  return PROPD_DISPATCH_DTYPE(dtype, T, [&] {
    gather_rows_kernel<T><<<M, threads_for(H), 0, as_stream(stream)>>>(H, src, idx, (T*)dst);
    return check_launch("gather_rows");
  });
}

int propd_argmax_rows(int M, const int32_t* rows_dev, int V, int ld, const float* logits, int32_t* out, void* stream) {
  if (M == 0) return 0;
  PROPD_REQUIRE(V > 0 && ld >= V, "argmax_rows: bad V=%d ld=%d", V, ld);
  const int grid = M < 2 * propd_num_sms() ? M : 2 * propd_num_sms();
  argmax_rows_kernel<<<grid, 512, 0, as_stream(stream)>>>(M, V, ld, logits, out, rows_dev);
  return check_launch("argmax_rows");
}

int propd_topk_rows(int R, int V, int ld, int k, const float* logits, int32_t* out_idx, float* out_val, void* stream) {
  if (R == 0) return 0;
  PROPD_REQUIRE(k >= 1 && k <= TOPK_MAX && k <= V, "topk_rows: k=%d outside 1..min(%d, V=%d)", k, TOPK_MAX, V);
  const int smem = V <= TOPK_SMEM_MAX ? V * 4 : 0;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(topk_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         TOPK_SMEM_MAX * 4);
    if (e != cudaSuccess) return fail("topk_rows: %s", cudaGetErrorString(e));
    attr = true;
  }
  topk_rows_kernel<<<R, 512, smem, as_stream(stream)>>>(V, ld, k, logits, out_idx, out_val);
  return check_launch("topk_rows");
}

int propd_kv_append(int dtype, int M, int A, int dh, int Lmax, const void* qkv, int ldqkv, const int32_t* row_seq,
                    const int32_t* row_node, const int32_t* seq_slot, const int32_t* seq_len, void* kcache,
                    void* vcache, void* stream) {
  if (M == 0) return 0;
  return PROPD_DISPATCH_DTYPE(dtype, T, [&] {
    PROPD_REQUIRE((dh * (int)sizeof(T)) % 16 == 0 && (ldqkv * (int)sizeof(T)) % 16 == 0,
                  "kv_append: rows must be 16-byte aligned");
    kv_append_kernel<T><<<dim3(M, 2), 128, 0, as_stream(stream)>>>(
        A, dh, Lmax, (const T*)qkv, ldqkv, row_seq, row_node, seq_slot, seq_len, (T*)kcache, (T*)vcache);
    return check_launch("kv_append");
  });
}

int propd_seq_advance(int B, const int32_t* seq_slot, int32_t* seq_len, const int32_t* delta_dev, int delta,
                      void* stream) {
  if (B == 0) return 0;
  seq_advance_kernel<<<(B + 127) / 128, 128, 0, as_stream(stream)>>>(B, seq_slot, seq_len, delta_dev, delta);
  return check_launch("seq_advance");
}

int propd_scatter_i32(int B, const int32_t* idx, const int32_t* src, int32_t* dst, void* stream) {
  if (B == 0) return 0;
  scatter_i32_kernel<<<(B + 127) / 128, 128, 0, as_stream(stream)>>>(B, idx, src, dst);
  return check_launch("scatter_i32");
}

}  // extern "C"
