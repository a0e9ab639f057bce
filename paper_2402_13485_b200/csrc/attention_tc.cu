// K2 on the 5th-generation tensor cores: tree-masked verification attention
// for bf16 K/V with head dim 128 (the 7B/33B shapes).
//
// Reference semantics: TinyTransformer._block attention (backends.py:216-233);
// every tree row attends to all committed cache rows and to its tree
// ancestors (+ itself), softmax(q k^T / sqrt(dh)) v.
//
// One CTA = (split of the key range, 128-row query tile, head, sequence).
// Warp roles (192 threads):
//   warp 0     TMA producer: streams K and V blocks of 128 keys x 128 dh from
//              the sequence's contiguous [Lmax, dh] cache tile (SWIZZLE_128B)
//              through a 2-stage mbarrier ring;
//   warp 1     TMEM allocator + single-thread tcgen05.mma issuer:
//              S_j = Q K_j^T (M=128, N=128, K=128, both K-major) into a
//              double-buffered TMEM S, then O += P_j V_j (P K-major from smem,
//              V MN-major) into a TMEM O accumulator;
//   warps 2-5  softmax: thread = query row (TMEM lane), tcgen05.ld of the S
//              row, ancestor-bitset mask, online softmax in the log2 domain
//              with a lazily updated reference max (O rescaled in TMEM only
//              when the row max grows by more than 2^8), bf16 P written to
//              smem in the UMMA SW128 K-major layout.
// Splits of the key range are merged by attn_combine_kernel (attention.cu).
#include <unordered_map>

#include "tc_common.cuh"

namespace propd {

template <typename T>
__global__ void attn_combine_kernel(int A, int dh, int nsplit, const float* __restrict__ part_o,
                                    const float* __restrict__ part_ml, T* __restrict__ out, int ldout);

namespace tc {

constexpr int BM = 128, BN = 128, DH = 128, STAGES = 2, THREADS = 192;
constexpr int TILE_BYTES = 128 * 128 * 2;  // one [128 x 128] bf16 operand = 2 SW128 column blocks
constexpr int SMEM_Q = 0;
constexpr int SMEM_K = SMEM_Q + TILE_BYTES;
constexpr int SMEM_V = SMEM_K + STAGES * TILE_BYTES;
constexpr int SMEM_P = SMEM_V + STAGES * TILE_BYTES;
constexpr int SMEM_MASK = SMEM_P + TILE_BYTES;        // [128 rows][8] u32 ancestor bitsets
constexpr int SMEM_BAR = SMEM_MASK + BM * 8 * 4;
constexpr int SMEM_TOTAL = SMEM_BAR + 256 + 1024;  // + barriers + alignment slack
constexpr uint32_t TMEM_COLS = 512;               // O: [0,128), S buffers: [128,256), [256,384)

struct Args {
  const __nv_bfloat16* qkv;
  int ldq;
  const int32_t* seq_slot;
  const int32_t* seq_len;
  const int32_t* row_off;
  const int32_t* row_node;
  const uint64_t* mask;
  int n_tmpl, W, A, Lmax;
  float scale_log2;  // log2(e) / sqrt(dh)
  int split_len, nsplit, mtiles;
  float* part_o;
  float* part_ml;
  __nv_bfloat16* out;
  int ldout;
  unsigned long long* trace;  // debug: phase timestamps of CTA (0,0,0), or null
};

static unsigned long long* g_trace = nullptr;

__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define TRACE(k)                                                                          \
  do {                                                                                    \
    if (p.trace && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0) p.trace[k] = gtime(); \
  } while (0)

// ------------------------------------------------------------------ kernel --
__global__ void __launch_bounds__(THREADS, 1)
    attn_tc_kernel(const __grid_constant__ CUtensorMap kmap, const __grid_constant__ CUtensorMap vmap, Args p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + SMEM_BAR);
  uint64_t* kv_full = bars;            // [STAGES]
  uint64_t* kv_empty = bars + STAGES;  // [STAGES]
  uint64_t* s_full = bars + 2 * STAGES;  // [2]
  uint64_t* p_full = bars + 2 * STAGES + 2;
  uint64_t* o_done = p_full + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_done + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) TRACE(0);
  const int s = blockIdx.x / p.mtiles, mt = blockIdx.x % p.mtiles;
  const int a = blockIdx.y, b = blockIdx.z;
  const int slot = p.seq_slot[b];
  const int L = p.seq_len[slot];
  const int r0 = p.row_off[b] + mt * BM;
  const int nrows = min(BM, p.row_off[b + 1] - r0);
  if (nrows <= 0) return;  // uniform: this query tile is empty for this sequence
  const int nkeys = L + p.n_tmpl;
  const int k_begin = s * p.split_len;
  const int k_end = min(nkeys, k_begin + p.split_len);
  const int nblk = k_end > k_begin ? (k_end - k_begin + BN - 1) / BN : 0;
  if (nblk == 0) {  // uniform: empty split contributes nothing
    if (p.nsplit > 1) {
      for (int r = threadIdx.x; r < nrows; r += blockDim.x) {
        const size_t base = ((size_t)(r0 + r) * p.A + a) * p.nsplit + s;
        p.part_ml[base * 2] = -INFINITY;
        p.part_ml[base * 2 + 1] = 0.f;
      }
    }
    return;
  }

  // ---- setup: barriers, TMEM, Q tile -------------------------------------
  if (threadIdx.x == 0) {
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&kv_full[i], 1);
      mbar_init(&kv_empty[i], 1);
    }
    mbar_init(&s_full[0], 1);
    mbar_init(&s_full[1], 1);
    mbar_init(p_full, 32 * min(4, (nrows + 31) / 32));  // softmax warps that own rows
    mbar_init(o_done, 1);
    fence_barrier_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  {  // Q rows -> SW128 K-major smem with cp.async (manual swizzle; rows past nrows are zero)
    const __nv_bfloat16* qbase = p.qkv + a * DH;
    for (int i = threadIdx.x; i < BM * 16; i += THREADS) {
      const int r = i >> 4, c = i & 15;
      uint8_t* dst = smem + SMEM_Q + sw128_chunk(r, c);
      if (r < nrows) {
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)),
                     "l"(qbase + (size_t)(r0 + r) * p.ldq + c * 8)
                     : "memory");
      } else {
        *reinterpret_cast<uint4*>(dst) = make_uint4(0, 0, 0, 0);
      }
    }
    uint32_t* msk = reinterpret_cast<uint32_t*>(smem + SMEM_MASK);
    for (int i = threadIdx.x; i < BM * 8; i += THREADS) {
      const int r = i >> 3, w = i & 7;
      uint32_t v = 0u;
      if (r < nrows) {
        if (p.mask != nullptr) {
          if ((w >> 1) < p.W) {
            const uint64_t word = p.mask[(size_t)p.row_node[r0 + r] * p.W + (w >> 1)];
            v = (w & 1) ? (uint32_t)(word >> 32) : (uint32_t)word;
          }
        } else {  // causal: tree nodes 0..row_node visible
          const int node = p.row_node[r0 + r];
          v = low_bits(node + 1 - 32 * w);
        }
      }
      msk[i] = v;
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
  }
  fence_proxy_async();
  tc_before_sync();
  __syncthreads();
  tc_after_sync();
  const uint32_t tmem = *tmem_slot;
  if (threadIdx.x == 0) TRACE(1);

  const size_t row_base = ((size_t)slot * p.A + a) * p.Lmax;
  if (warp == 0) {
    // ================= TMA producer =================
    if (lane == 0) {
      for (int j = 0; j < nblk; ++j) {
        const int st = j % STAGES;
        mbar_wait(&kv_empty[st], ((j / STAGES) & 1) ^ 1, 1);
        mbar_expect_tx(&kv_full[st], 2 * TILE_BYTES);
        const int row = (int)(row_base + k_begin + j * BN);
        uint8_t* kd = smem + SMEM_K + st * TILE_BYTES;
        uint8_t* vd = smem + SMEM_V + st * TILE_BYTES;
        tma_load_2d(kd, &kmap, &kv_full[st], 0, row);
        tma_load_2d(kd + HALF, &kmap, &kv_full[st], 64, row);
        tma_load_2d(vd, &vmap, &kv_full[st], 0, row);
        tma_load_2d(vd + HALF, &vmap, &kv_full[st], 64, row);
      }
    }
  } else if (warp == 1) {
    // ================= MMA issuer =================
    if (lane == 0) {
      const uint32_t id_s = idesc_bf16(false), id_o = idesc_bf16(true);
      const uint32_t q_addr = smem_u32(smem + SMEM_Q), p_addr = smem_u32(smem + SMEM_P);
      auto issue_pv = [&](int jj) {
        const int st = jj % STAGES;
        mbar_wait(p_full, jj & 1, 2);
        tc_after_sync();
        if (jj == 0) TRACE(6);
        const uint32_t v_addr = smem_u32(smem + SMEM_V + st * TILE_BYTES);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {  // K = 128 keys in steps of 16
          const uint64_t ad = sw128_desc(p_addr + (kk >> 2) * HALF + (kk & 3) * 32, 16, 1024);
          const uint64_t bd = sw128_desc(v_addr + kk * 2048, HALF, 1024);
          mma_bf16(tmem, ad, bd, id_o, (jj > 0 || kk > 0) ? 1u : 0u);
        }
        mma_commit(&kv_empty[st]);
        mma_commit(o_done);
      };
      for (int j = 0; j < nblk; ++j) {
        const int st = j % STAGES;
        mbar_wait(&kv_full[st], (j / STAGES) & 1, 3);
        tc_after_sync();
        if (j == 0) TRACE(2);
        const uint32_t k_addr = smem_u32(smem + SMEM_K + st * TILE_BYTES);
        const uint32_t s_tmem = tmem + 128 + 128 * (j & 1);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {  // K = dh 128 in steps of 16
          const uint64_t ad = sw128_desc(q_addr + (kk >> 2) * HALF + (kk & 3) * 32, 16, 1024);
          const uint64_t bd = sw128_desc(k_addr + (kk >> 2) * HALF + (kk & 3) * 32, 16, 1024);
          mma_bf16(s_tmem, ad, bd, id_s, kk > 0 ? 1u : 0u);
        }
        mma_commit(&s_full[j & 1]);
        if (j == 0) TRACE(3);
        if (j > 0) issue_pv(j - 1);
      }
      issue_pv(nblk - 1);
    }
  } else {
    // ================= softmax warps =================
    const int q4 = warp & 3;  // TMEM lane quadrant this warp may access
    const int r = q4 * 32 + lane;
    const bool valid = r < nrows;
    const bool warp_live = q4 * 32 < nrows;
    const int row = r0 + r;
    const uint32_t* mrow = reinterpret_cast<const uint32_t*>(smem + SMEM_MASK) + r * 8;
    const uint32_t lane_addr = tmem + ((uint32_t)(q4 * 32) << 16);
    const float scale = p.scale_log2;
    float m_ref = -INFINITY, l_sum = 0.f;
    uint8_t* prow = smem + SMEM_P;
    for (int j = 0; j < nblk && warp_live; ++j) {
      float sv[128];
      mbar_wait(&s_full[j & 1], (j >> 1) & 1, 4);
      tc_after_sync();
      if (j == 0 && r == 0) TRACE(4);
      const uint32_t sa = lane_addr + 128 + 128 * (j & 1);
      {  // four 32-column loads in flight, one wait
        uint32_t* rv = reinterpret_cast<uint32_t*>(sv);
        TMEM_LD32(sa, rv);
        TMEM_LD32(sa + 32, (rv + 32));
        TMEM_LD32(sa + 64, (rv + 64));
        TMEM_LD32(sa + 96, (rv + 96));
        tmem_wait_ld();
      }
      // visibility of the block's 128 keys as 4 x 32-bit words (all uniform
      // except the row's own ancestor bits): cache keys, tree keys, range end
      const int key0 = k_begin + j * BN;
      const int ncache = L - key0, nvalid = k_end - key0;
      uint32_t vis[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint32_t cache_bits = low_bits(ncache - 32 * q);
        const uint32_t tree_bits = mask_bits32(mrow, key0 + 32 * q - L);
        vis[q] = valid ? ((cache_bits | tree_bits) & low_bits(nvalid - 32 * q)) : 0u;
      }
      // masked max with 8 independent accumulators (no 128-long dependency chain)
      float mx8[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) mx8[u] = -INFINITY;
      const bool all_vis = __all_sync(0xffffffffu, (vis[0] & vis[1] & vis[2] & vis[3]) == 0xffffffffu);
      if (all_vis) {
#pragma unroll
        for (int i = 0; i < 128; ++i) mx8[i & 7] = fmaxf(mx8[i & 7], sv[i]);
      } else {
#pragma unroll
        for (int i = 0; i < 128; ++i) {
          sv[i] = ((vis[i >> 5] >> (i & 31)) & 1u) ? sv[i] : -INFINITY;
          mx8[i & 7] = fmaxf(mx8[i & 7], sv[i]);
        }
      }
      float mx = fmaxf(fmaxf(fmaxf(mx8[0], mx8[1]), fmaxf(mx8[2], mx8[3])),
                       fmaxf(fmaxf(mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7])));
      mx *= scale;  // scale > 0: max commutes with scaling (-inf stays -inf)
      if (j > 0) {  // PV_{j-1} finished: P buffer free, O stable
        mbar_wait(o_done, (j - 1) & 1, 5);
        tc_after_sync();
      }
      // lazy max update (exact: O and l always share m_ref); the decision is
      // per row but tcgen05.ld/st are warp-collective, so the O rescale
      // runs for the whole warp with corr = 1 on rows that keep their max
      float corr = 1.f;
      const bool grow = mx > m_ref + 8.f;
      if (grow) {
        corr = ex2(m_ref - mx);
        l_sum *= corr;
        m_ref = mx;
      }
      if (j > 0 && __any_sync(0xffffffffu, grow)) {
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          uint32_t rr[32];
          TMEM_LD32(lane_addr + c * 32, rr);
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 32; ++i) rr[i] = __float_as_uint(__uint_as_float(rr[i]) * corr);
          TMEM_ST32(lane_addr + c * 32, rr);
        }
        tmem_wait_st();
      }
      const float mneg = m_ref == -INFINITY ? 0.f : -m_ref;  // masked keys: ex2(-inf) = 0
      float ls8[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) ls8[u] = 0.f;
#pragma unroll
      for (int c = 0; c < 16; ++c) {
        uint32_t pk[4];
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          const float2 pp = ex2x2(fmaf(sv[c * 8 + 2 * h], scale, mneg), fmaf(sv[c * 8 + 2 * h + 1], scale, mneg));
          ls8[(2 * h) & 7] += pp.x;
          ls8[(2 * h + 1) & 7] += pp.y;
          __nv_bfloat162 v2 = __floats2bfloat162_rn(pp.x, pp.y);
          pk[h] = *reinterpret_cast<uint32_t*>(&v2);
        }
        *reinterpret_cast<uint4*>(prow + sw128_chunk(r, c)) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
      }
      l_sum += ((ls8[0] + ls8[1]) + (ls8[2] + ls8[3])) + ((ls8[4] + ls8[5]) + (ls8[6] + ls8[7]));
      fence_proxy_async();
      tc_before_sync();
      mbar_arrive(p_full);
      if (j == 0 && r == 0) TRACE(5);
    }
    // epilogue: O row from TMEM
    if (warp_live) {
      mbar_wait(o_done, (nblk - 1) & 1, 6);
      tc_after_sync();
      if (r == 0) TRACE(7);
      float o[128];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t rr[32];
        TMEM_LD32(lane_addr + c * 32, rr);
        tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 32; ++i) o[c * 32 + i] = __uint_as_float(rr[i]);
      }
      if (valid) {
        if (p.nsplit == 1) {
          const float inv = l_sum > 0.f ? 1.f / l_sum : 0.f;
          __nv_bfloat16* dst = p.out + (size_t)row * p.ldout + a * DH;
#pragma unroll
          for (int c = 0; c < 16; ++c) {
            uint32_t pk[4];
#pragma unroll
            for (int h = 0; h < 4; ++h) {
              __nv_bfloat162 v2 = __floats2bfloat162_rn(o[c * 8 + 2 * h] * inv, o[c * 8 + 2 * h + 1] * inv);
              pk[h] = *reinterpret_cast<uint32_t*>(&v2);
            }
            *reinterpret_cast<uint4*>(dst + c * 8) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
          }
        } else {
          const size_t base = ((size_t)row * p.A + a) * p.nsplit + s;
          float4* po = reinterpret_cast<float4*>(p.part_o + base * DH);
#pragma unroll
          for (int c = 0; c < 32; ++c) po[c] = make_float4(o[4 * c], o[4 * c + 1], o[4 * c + 2], o[4 * c + 3]);
          p.part_ml[base * 2] = m_ref * 0.69314718055994531f;  // back to natural-log units
          p.part_ml[base * 2 + 1] = l_sum;
        }
      }
    }
  }
  if (threadIdx.x == 128) TRACE(8);
  tc_before_sync();
  __syncthreads();
  tc_after_sync();
  if (threadIdx.x == 0) TRACE(9);
  if (warp == 1) {
    __syncwarp();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
  }
}

// ------------------------------------------------------------------ host --
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeFn get_encode() {
  static EncodeFn fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* f = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(f);
  }
  return fn;
}

// [rows, 128] bf16 view of a K or V cache layer; box 64 x 128, SWIZZLE_128B.
static bool kv_map(CUtensorMap* m, const void* base, uint64_t rows) {
  static std::unordered_map<uint64_t, std::pair<uint64_t, CUtensorMap>> cache;
  const uint64_t key = (uint64_t)(uintptr_t)base;
  auto it = cache.find(key);
  if (it != cache.end() && it->second.first == rows) {
    *m = it->second.second;
    return true;
  }
  EncodeFn enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {128, rows};
  cuuint64_t strides[1] = {128 * 2};
  cuuint32_t box[2] = {64, 128};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return false;
  cache[key] = {rows, *m};
  return true;
}

}  // namespace tc

// Called by propd_tree_attention for bf16 / dh = 128.
int attention_tc_bf16(int B, int M, int A, int Lmax, int n_slots, int max_rows_per_seq, int max_keys, const void* qkv,
                      int ldqkv, const void* kc, const void* vc, const int32_t* seq_slot, const int32_t* seq_len,
                      const int32_t* row_off, const int32_t* row_node, const uint64_t* mask, int n_tmpl, int W,
                      void* out, int ldout, void* ws, int64_t ws_bytes, cudaStream_t st, bool* handled) {
  *handled = false;
  if (n_slots <= 0 || W > 4 || (ldqkv % 8) != 0 || (ldout % 8) != 0) return 0;
  CUtensorMap km, vm;
  const uint64_t rows = (uint64_t)n_slots * A * Lmax;
  if (!tc::kv_map(&km, kc, rows) || !tc::kv_map(&vm, vc, rows)) return 0;
  const int mtiles = (max_rows_per_seq + tc::BM - 1) / tc::BM;
  // split the key range so that one wave (one CTA per SM) covers the grid
  const int ctas = B * A * mtiles;
  const int nblk_max = (max_keys + tc::BN - 1) / tc::BN;
  int nsplit = 148 / ctas;
  if (nsplit > nblk_max) nsplit = nblk_max;
  if (nsplit > 64) nsplit = 64;
  if (nsplit < 1) nsplit = 1;
  const int64_t need = (int64_t)M * A * nsplit * (tc::DH + 2) * (int64_t)sizeof(float);
  if (nsplit > 1 && (ws == nullptr || ws_bytes < need)) nsplit = 1;
  int blocks_per_split = (nblk_max + nsplit - 1) / nsplit;
  nsplit = (nblk_max + blocks_per_split - 1) / blocks_per_split;
  tc::Args p{};
  p.qkv = reinterpret_cast<const __nv_bfloat16*>(qkv);
  p.ldq = ldqkv;
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
  p.split_len = blocks_per_split * tc::BN;
  p.nsplit = nsplit;
  p.mtiles = mtiles;
  p.part_o = reinterpret_cast<float*>(ws);
  p.part_ml = p.part_o + (size_t)M * A * nsplit * tc::DH;
  p.out = reinterpret_cast<__nv_bfloat16*>(out);
  p.ldout = ldout;
  p.trace = tc::g_trace;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(tc::attn_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         tc::SMEM_TOTAL);
    if (e != cudaSuccess) return fail("tree_attention(tc): %s", cudaGetErrorString(e));
    attr = true;
  }
  *handled = true;
  dim3 grid(nsplit * mtiles, A, B);
  tc::attn_tc_kernel<<<grid, tc::THREADS, tc::SMEM_TOTAL, st>>>(km, vm, p);
  if (int e = check_launch("tree_attention(tc)")) return e;
  if (nsplit > 1) {
    attn_combine_kernel<__nv_bfloat16><<<dim3(M, A), 128, 0, st>>>(A, tc::DH, nsplit, p.part_o, p.part_ml, p.out,
                                                                  ldout);
    if (int e = check_launch("tree_attention(tc combine)")) return e;
  }
  return 0;
}

}  // namespace propd

namespace propd {
int attention_tc2_prepare();
}

extern "C" int propd_prepare(void) {  // one-time function attributes (before any graph capture)
  cudaError_t e = cudaFuncSetAttribute(propd::tc::attn_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       propd::tc::SMEM_TOTAL);
  if (e != cudaSuccess) return propd::fail("prepare: %s", cudaGetErrorString(e));
  return propd::attention_tc2_prepare();
}

extern "C" int propd_debug_trace(void* buf) {  // development aid: phase timestamps of one CTA
  propd::tc::g_trace = reinterpret_cast<unsigned long long*>(buf);
  return 0;
}
