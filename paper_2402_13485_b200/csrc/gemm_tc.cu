// Projections of the many-row passes: Y = epilogue(X[M,K] . W[K,N]) for
// M > 128 token rows (the pre-prune tree pass at batch >= 3, the post-prune
// pass once survivors exceed 128 rows, prefill), and the LM / early / draft
// heads over such row counts (backends.py:217-219, 234-236, 256, 281, 321,
// 329).  At these row counts the projection is tensor-bound (intensity = rows
// flop/B, the ridge is ~210 rows), so the tile is the largest single-CTA
// tcgen05 shape: 128 token rows (MMA M) x 256 output features (MMA N).
//
// bf16 (tcgen05): persistent kernel, one CTA per SM, tiles rasterised M-fastest
// (the ~148 concurrently running tiles share a few W column blocks in L2).
//   warp 0     TMA producer: X tile [128 rows x 64 k] K-major (SW128) + W tile
//              [64 k x 256 features] MN-major (4 SW128 boxes), 4-stage ring
//   warp 1     TMEM allocation (2 x 256 columns: double-buffered accumulator)
//              and the MMA issuer (tcgen05.mma kind::f16, M128 N256 K16)
//   warps 2-5  epilogue: TMEM -> registers (lane = token row, 32 features per
//              tcgen05.ld) -> fused output op, overlapping the next tile's MMAs
// fp32 (parity mode): a CUDA-core SGEMM (true fp32 FMA) with the same epilogues.
//
// Epilogues: fp32 store (logits), fp32 add into the residual stream (W_o, W_2),
// store in the activation dtype, tanh-GELU (W_1), QKV split (Q rows -> the
// attention operand, K/V rows -> their cache slots seq_len + node, replacing
// propd_kv_append).
#include <unordered_map>

#include "tc_common.cuh"

namespace propd {
namespace gtc {
using namespace propd::tc;

constexpr int BM = 128, BN = 256, BK = 64, STAGES = 4, THREADS = 192;
constexpr int A_BYTES = BM * BK * 2;         // 16 KB: [128 rows x 64 k] SW128 K-major
constexpr int B_BYTES = BK * BN * 2;         // 32 KB: 4 x [64 k x 64 features] SW128 MN-major
constexpr int B_BLOCK = BK * 64 * 2;         // 8 KB per 64-feature block
constexpr int STAGE = A_BYTES + B_BYTES;     // 48 KB
constexpr int SMEM = STAGES * STAGE + 256 + 1024;
constexpr int TMEM_COLS = 2 * BN;            // two accumulators of 256 fp32 columns

struct Args {
  int M, N, K;
  int split;  // K splits (ADD_F32 only: partial sums are reduced into Y by red.global.add)
  const int32_t* rows_dev;
  propd_gemm_epi epi;
  unsigned long long* trace;
  unsigned int tag;
};

__device__ __forceinline__ float gelu_tanh(float v) {
  return 0.5f * v * (1.f + tanhf(0.7978845608028654f * (v + 0.044715f * v * v * v)));
}

template <typename T>
__device__ __forceinline__ void store32(T* dst, const float* v);
template <>
__device__ __forceinline__ void store32<__nv_bfloat16>(__nv_bfloat16* dst, const float* v) {
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    uint4 u;
    uint32_t* w = reinterpret_cast<uint32_t*>(&u);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      __nv_bfloat162 h = __floats2bfloat162_rn(v[q * 8 + 2 * j], v[q * 8 + 2 * j + 1]);
      w[j] = *reinterpret_cast<uint32_t*>(&h);
    }
    reinterpret_cast<uint4*>(dst)[q] = u;
  }
}
template <>
__device__ __forceinline__ void store32<float>(float* dst, const float* v) {
#pragma unroll
  for (int q = 0; q < 8; ++q)
    reinterpret_cast<float4*>(dst)[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
}

// 32 consecutive output features f0.. of token row `row` (f0 % 32 == 0, f0 + 32 <= N).
template <typename T>
__device__ __forceinline__ void epilogue32(const propd_gemm_epi& e, int split, int row, int f0, float* v) {
  switch (e.mode) {
    case PROPD_EPI_STORE_F32:
      store32<float>(reinterpret_cast<float*>(e.Y) + (size_t)row * e.ldy + f0, v);
      break;
    case PROPD_EPI_ADD_F32: {
      float* y = reinterpret_cast<float*>(e.Y) + (size_t)row * e.ldy + f0;
      if (split > 1 || split < 0) {  // K splits add into the same rows (or one tile per CTA): fire-and-forget reductions
#pragma unroll
        for (int q = 0; q < 8; ++q)
          asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(y + 4 * q), "f"(v[4 * q]),
                       "f"(v[4 * q + 1]), "f"(v[4 * q + 2]), "f"(v[4 * q + 3])
                       : "memory");
      } else {  // the only writer of these rows: plain read-modify-write (cheaper than reductions)
        float4* y4 = reinterpret_cast<float4*>(y);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          float4 a = __ldcg(y4 + q);
          a.x += v[4 * q];
          a.y += v[4 * q + 1];
          a.z += v[4 * q + 2];
          a.w += v[4 * q + 3];
          y4[q] = a;
        }
      }
      break;
    }
    case PROPD_EPI_GELU:
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = gelu_tanh(v[i]);
      store32<T>(reinterpret_cast<T*>(e.Y) + (size_t)row * e.ldy + f0, v);
      break;
    case PROPD_EPI_QKV: {
      const int H = e.A * e.dh;
      if (f0 < H) {
        store32<T>(reinterpret_cast<T*>(e.Y) + (size_t)row * e.ldy + f0, v);
      } else {
        const int kv = f0 >= 2 * H;
        const int ee = f0 - (kv ? 2 * H : H);
        const int head = ee / e.dh, d = ee - head * e.dh;
        const int slot = e.seq_slot[e.row_seq[row]];
        const int pos = e.seq_len[slot] + e.row_node[row];
        T* cache = reinterpret_cast<T*>(kv ? e.vcache : e.kcache);
        store32<T>(cache + (((size_t)slot * e.A + head) * e.Lmax + pos) * e.dh + d, v);
      }
      break;
    }
    default:  // PROPD_EPI_STORE
      store32<T>(reinterpret_cast<T*>(e.Y) + (size_t)row * e.ldy + f0, v);
  }
}

// K splits of a residual-add launch over `tiles` output tiles on `ctas`
// persistent CTAs: minimises waves / split + a small per-split cost for the
// reductions, >= 4 k-blocks per split, no empty split (host and device).
__host__ __device__ inline int choose_split(int tiles, int kb, int ctas) {
  int split = 1;
  double best = 1e30;
  for (int s = 1; s <= 8 && kb / s >= 4; ++s) {
    const double cost = (double)((tiles * s + ctas - 1) / ctas) / s + 0.04 * (s - 1);
    if (cost < best - 1e-9) {
      best = cost;
      split = s;
    }
  }
  const int kper = (kb + split - 1) / split;
  return (kb + kper - 1) / kper;
}

__global__ void __launch_bounds__(THREADS, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap xmap, const __grid_constant__ CUtensorMap wmap, Args p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE);
  uint64_t* empty = full + STAGES;
  uint64_t* acc_full = empty + STAGES;  // [2]
  uint64_t* acc_empty = acc_full + 2;   // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);
  const unsigned long long t_entry = p.trace ? gtimer() : 0ull;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_empty[i], 128);
    }
    fence_barrier_init();
    asm volatile("prefetch.tensormap [%0];" ::"l"(&xmap) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&wmap) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_before_sync();
  __syncthreads();
  tc_after_sync();
  const uint32_t tmem = *tmem_slot;
  pdl_trigger();  // after the TMEM allocation (see common.cuh)
  pdl_wait();
  const unsigned long long t_wait = p.trace ? gtimer() : 0ull;
  const int M = p.rows_dev ? min(p.M, *p.rows_dev) : p.M;
  const int Mb = (M + BM - 1) / BM, Nb = (p.N + BN - 1) / BN, Kb = p.K / BK;
  const int tiles = Mb * Nb;
  // a pass captured at a padded row capacity learns its live rows here: the
  // residual-add split is chosen for them (the host's split assumed the capacity)
  const int split = (p.rows_dev && p.epi.mode == PROPD_EPI_ADD_F32) ? choose_split(tiles, Kb, gridDim.x) : p.split;
  const int units = tiles * split;
  const int kper = (Kb + split - 1) / split;  // k-blocks per split
  if (warp == 0) {
    if (lane == 0) {
      int it = 0;
      for (int u = blockIdx.x; u < units; u += gridDim.x) {
        const int t = u % tiles, s = u / tiles;
        const int mb = t % Mb, nb = t / Mb;
        const int kb1 = min(Kb, (s + 1) * kper);
        for (int kb = s * kper; kb < kb1; ++kb, ++it) {
          const int st = it % STAGES;
          mbar_wait(&empty[st], ((it / STAGES) & 1) ^ 1, 81);
          mbar_expect_tx(&full[st], STAGE);
          uint8_t* a = smem + st * STAGE;
          tma_load_2d(a, &xmap, &full[st], kb * BK, mb * BM);
#pragma unroll
          for (int j = 0; j < 4; ++j) tma_load_2d(a + A_BYTES + j * B_BLOCK, &wmap, &full[st], nb * BN + j * 64, kb * BK);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // A = X K-major, B = W MN-major (features contiguous); M = 128, N = 256
      constexpr uint32_t idesc = idesc_bf16(true, BN, BM);
      int it = 0, i = 0;
      for (int u = blockIdx.x; u < units; u += gridDim.x, ++i) {
        const int s = u / tiles;
        const int kb0 = s * kper, kb1 = min(Kb, (s + 1) * kper);
        const int buf = i & 1;
        mbar_wait(&acc_empty[buf], ((i >> 1) & 1) ^ 1, 82);
        tc_after_sync();
        const uint32_t d = tmem + buf * BN;
        for (int kb = kb0; kb < kb1; ++kb, ++it) {
          const int st = it % STAGES;
          mbar_wait(&full[st], (it / STAGES) & 1, 83);
          tc_after_sync();
          const uint32_t a = smem_u32(smem + st * STAGE);
          const uint32_t b = a + A_BYTES;
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk) {
            const uint64_t ad = sw128_desc(a + kk * 32, 16, 1024);
            const uint64_t bd = sw128_desc(b + kk * 2048, B_BLOCK, 1024);
            mma_bf16(d, ad, bd, idesc, (kb > kb0 || kk > 0) ? 1u : 0u);
          }
          mma_commit(&empty[st]);
        }
        mma_commit(&acc_full[buf]);
      }
    }
  } else {
    // epilogue: TMEM lane quarter q4 = warp % 4 holds token rows q4*32 .. q4*32+31
    const int q4 = warp & 3, tid = threadIdx.x - 64;
    int i = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x, ++i) {
      const int t = u % tiles;
      const int mb = t % Mb, nb = t / Mb;
      const int buf = i & 1;
      mbar_wait(&acc_full[buf], (i >> 1) & 1, 84);
      tc_after_sync();
      const int row = mb * BM + q4 * 32 + lane;
      const uint32_t base = tmem + buf * BN + ((uint32_t)(q4 * 32) << 16);
#pragma unroll 1
      for (int c = 0; c < BN / 32; ++c) {
        uint32_t r[32];
        TMEM_LD32(base + c * 32, r);
        tmem_wait_ld();
        const int f0 = nb * BN + c * 32;
        if (row < M && f0 < p.N) {
          float v[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
          // with fewer than two units per CTA the residual add cannot hide a read-modify-write
          // behind the next tile's MMAs: fire-and-forget reductions (W_o at 1024 rows 56.6 -> 30.5 us)
          epilogue32<__nv_bfloat16>(p.epi, units < 2 * (int)gridDim.x ? -1 : split, row, f0, v);
        }
      }
      tc_before_sync();
      mbar_arrive(&acc_empty[buf]);  // the accumulator is free for the unit after next
    }
  }
  tc_before_sync();
  __syncthreads();
  tc_after_sync();
  if (warp == 1) {
    __syncwarp();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
  }
  if (p.trace && threadIdx.x == 0)  // kind 5 + shape: bench.py computes this launch's algorithmic bytes / flops
    trace_record(p.trace, p.tag, t_entry, t_wait, t_wait,
                 5ull | ((unsigned long long)(p.N / 32) << 8) | ((unsigned long long)(p.K / 64) << 24) |
                     ((unsigned long long)min(M, 65535) << 40));
}

// ---- fp32 parity mode: CUDA-core SGEMM (64 x 64 tiles, 4 x 4 per thread)
constexpr int SB = 64, SK = 16;
__global__ void __launch_bounds__(256) sgemm_kernel(int M, int N, int K, const float* __restrict__ X, int ldx,
                                                    const float* __restrict__ W, int ldw, propd_gemm_epi e,
                                                    const int32_t* rows_dev) {
  __shared__ float xs[SK][SB + 4];
  __shared__ float ws[SK][SB + 4];
  pdl_wait();
  if (rows_dev) M = min(M, *rows_dev);
  const int m0 = blockIdx.y * SB, n0 = blockIdx.x * SB;
  if (m0 >= M) return;
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < K; k0 += SK) {
    for (int i = threadIdx.x; i < SB * SK; i += 256) {
      const int r = i / SK, c = i % SK;  // X tile: row r, k c
      xs[c][r] = (m0 + r < M && k0 + c < K) ? X[(size_t)(m0 + r) * ldx + k0 + c] : 0.f;
      const int kr = i / SB, nc = i % SB;  // W tile: k kr, feature nc
      ws[kr][nc] = (k0 + kr < K && n0 + nc < N) ? W[(size_t)(k0 + kr) * ldw + n0 + nc] : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < SK; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        a[i] = xs[kk][ty * 4 + i];
        b[i] = ws[kk][tx * 4 + i];
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
  const int H = e.A * e.dh;
  for (int i = 0; i < 4; ++i) {
    const int row = m0 + ty * 4 + i;
    if (row >= M) continue;
    for (int j = 0; j < 4; ++j) {
      const int f = n0 + tx * 4 + j;
      if (f >= N) continue;
      float v = acc[i][j];
      float* y = reinterpret_cast<float*>(e.Y);
      switch (e.mode) {
        case PROPD_EPI_ADD_F32: y[(size_t)row * e.ldy + f] += v; break;
        case PROPD_EPI_GELU: y[(size_t)row * e.ldy + f] = gelu_tanh(v); break;
        case PROPD_EPI_QKV:
          if (f < H) {
            y[(size_t)row * e.ldy + f] = v;
          } else {
            const int kv = f >= 2 * H;
            const int ee = f - (kv ? 2 * H : H);
            const int head = ee / e.dh, d = ee - head * e.dh;
            const int slot = e.seq_slot[e.row_seq[row]];
            const int pos = e.seq_len[slot] + e.row_node[row];
            float* cache = reinterpret_cast<float*>(kv ? e.vcache : e.kcache);
            cache[(((size_t)slot * e.A + head) * e.Lmax + pos) * e.dh + d] = v;
          }
          break;
        default: y[(size_t)row * e.ldy + f] = v;  // STORE / STORE_F32
      }
    }
  }
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

// 2D bf16 map of a row-major [rows, cols] matrix, box [64 cols x box_rows], SW128.
static bool map2d(CUtensorMap* m, const void* base, uint64_t rows, uint64_t cols, uint64_t ld, uint32_t box_rows) {
  struct Key {
    uint64_t p, r, c, l, b;
    bool operator==(const Key& o) const { return p == o.p && r == o.r && c == o.c && l == o.l && b == o.b; }
  };
  struct Hs {
    size_t operator()(const Key& k) const { return k.p ^ (k.r * 1315423911u) ^ (k.c << 7) ^ (k.b << 17); }
  };
  static std::unordered_map<Key, CUtensorMap, Hs> cache;
  static EncodeFn enc = nullptr;
  const Key key{(uint64_t)(uintptr_t)base, rows, cols, ld, box_rows};
  auto it = cache.find(key);
  if (it != cache.end()) {
    *m = it->second;
    return true;
  }
  if (!enc) {
    cudaDriverEntryPointQueryResult q;
    void* fp = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return false;
    enc = reinterpret_cast<EncodeFn>(fp);
  }
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {ld * 2};
  cuuint32_t box[2] = {64, box_rows};
  cuuint32_t es[2] = {1, 1};
  if (enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return false;
  cache[key] = *m;
  return true;
}

}  // namespace gtc
}  // namespace propd

using namespace propd;

extern "C" {

int propd_gemm(int dtype, int M, const int32_t* rows_dev, int N, int K, const void* X, int ldx, const void* W,
               int ldw, const propd_gemm_epi* epi, void* stream) {
  if (M == 0) return 0;
  PROPD_REQUIRE(epi != nullptr && epi->Y != nullptr, "gemm: needs an epilogue with an output");
  PROPD_REQUIRE(M > 0 && N > 0 && K > 0, "gemm: bad shape %d x %d x %d", M, N, K);
  PROPD_REQUIRE(epi->mode != PROPD_EPI_QKV || (N == 3 * epi->A * epi->dh && epi->kcache && epi->vcache &&
                                                epi->row_seq && epi->row_node && epi->seq_slot && epi->seq_len),
                "gemm: the QKV epilogue needs N = 3H and the cache tables");
  cudaStream_t st = as_stream(stream);
  if (dtype == PROPD_F32) {
    dim3 grid((N + gtc::SB - 1) / gtc::SB, (M + gtc::SB - 1) / gtc::SB);
    return launch_pdl("gemm(fp32)", gtc::sgemm_kernel, grid, dim3(256), 0, st, M, N, K,
                      reinterpret_cast<const float*>(X), ldx, reinterpret_cast<const float*>(W), ldw, *epi, rows_dev);
  }
  PROPD_REQUIRE(dtype == PROPD_BF16, "gemm: dtype %d", dtype);
  PROPD_REQUIRE(N % 32 == 0 && K % gtc::BK == 0, "gemm: N=%d must be a multiple of 32, K=%d of 64", N, K);
  PROPD_REQUIRE(ldx % 8 == 0 && ldw % 8 == 0 && (reinterpret_cast<uintptr_t>(X) & 15) == 0 &&
                    (reinterpret_cast<uintptr_t>(W) & 15) == 0,
                "gemm: X / W need 16-byte aligned rows (TMA)");
  PROPD_REQUIRE((reinterpret_cast<uintptr_t>(epi->Y) & 15) == 0 && epi->ldy % 8 == 0 &&
                    (epi->mode != PROPD_EPI_QKV || epi->dh % 32 == 0),
                "gemm: Y needs 16-byte aligned rows (vector epilogue), head dim a multiple of 32");
  CUtensorMap xm, wm;
  PROPD_REQUIRE(gtc::map2d(&xm, X, (uint64_t)M, (uint64_t)K, (uint64_t)ldx, gtc::BM) &&
                    gtc::map2d(&wm, W, (uint64_t)K, (uint64_t)N, (uint64_t)ldw, gtc::BK),
                "gemm: tensor map encode failed");
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(gtc::gemm_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, gtc::SMEM);
    if (e != cudaSuccess) return fail("gemm: %s", cudaGetErrorString(e));
    attr = true;
  }
  const int tiles = ((M + gtc::BM - 1) / gtc::BM) * ((N + gtc::BN - 1) / gtc::BN);
  const int sms = propd_num_sms();
  // Few tiles (a few hundred rows) leave SMs idle or a short last wave: for the
  // residual-stream epilogue K is split so the work units fill the waves
  // (partial sums reduced into Y).  split minimises waves / split + a small
  // per-split cost for the reductions, >= 4 k-blocks per split.  (A split
  // through an fp32 workspace for the other epilogues was measured slower:
  // the reductions and the last-split finish cost more than the wave fill.)
  const int split = epi->mode == PROPD_EPI_ADD_F32 ? gtc::choose_split(tiles, K / gtc::BK, sms) : 1;
  gtc::Args p{M, N, K, split, rows_dev, *epi, g_dbg_trace, g_dbg_tag++};
  const int units = tiles * split;
  // with a device row count the residual-add split is re-chosen in the kernel
  // for the live rows: launch every SM
  const int grid = (rows_dev && epi->mode == PROPD_EPI_ADD_F32) || units >= sms ? sms : units;
  return launch_pdl("gemm(tcgen05)", gtc::gemm_tc_kernel, dim3(grid), dim3(gtc::THREADS), gtc::SMEM, st, xm, wm, p);
}

}  // extern "C"
