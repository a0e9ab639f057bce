// K2 v2 on tcgen05: tree-masked verification attention (bf16, dh = 128)
// built to keep HBM busy.  Reference semantics as in attention_tc.cu
// (backends.py:216-233).
//
// v1 (attention_tc.cu) serialises every 128-key block through one softmax
// warpgroup and a 2-stage ring, so a block costs ~2 us of chain latency
// against ~1.5 us of HBM time.  v2:
//   - 64-key blocks streamed by two TMA producers into separate 6-stage rings:
//     K (released as soon as S = QK^T completes) and V (released after PV),
//     192 KB of shared memory for K/V (P never touches smem: the bf16
//     probabilities are written with tcgen05.st over the consumed S buffer
//     and P V reads its A operand straight from TMEM);
//   - two softmax warpgroups (A: even blocks, B: odd blocks), each with its
//     own TMEM accumulator O_g, running max/sum and P buffer, so two blocks
//     are in softmax at once; the MMA thread is an event loop that issues
//     S_j = Q K_j^T (M=128, N=64) as soon as K_j and an S buffer are free
//     (up to four blocks ahead) and O_g += P_g V_j (M=128, N=128, K=64) as
//     soon as P_j and V_j are ready;
//   - the two partial softmax states are merged in-kernel at the end; the key
//     splits of one (sequence, head, row tile) are one thread-block cluster
//     and are merged through distributed shared memory (no combine launch).
// Warp roles (352 threads): warp 0 TMA (K), warp 10 TMA (V), warp 1 TMEM
// alloc + MMA issue, warps 2-5 group A, warps 6-9 group B.
#include <unordered_map>

#include "tc_common.cuh"

namespace propd {

namespace tc2 {
using namespace propd::tc;

constexpr int BM = 128, BN = 64, DH = 128, KS = 6, VS = 6, THREADS = 352;
constexpr int QBYTES = 128 * 128 * 2;      // Q: two SW128 blocks of [128 rows x 128 B]
constexpr int KV_HALF = BN * 128;          // one [64 rows x 128 B] SW128 block = 8 KB
constexpr int KV_TILE = 2 * KV_HALF;       // K (or V) of one 64-key block = 16 KB

constexpr int SMEM_Q = 0;
constexpr int SMEM_K = SMEM_Q + QBYTES;         // K ring: KS x 16 KB (released after S)
constexpr int SMEM_V = SMEM_K + KS * KV_TILE;     // V ring: VS x 16 KB (released after PV)
constexpr int SMEM_ML = SMEM_V + VS * KV_TILE;    // [2 groups][2][128] floats (m, l)
constexpr int SMEM_BAR = SMEM_ML + 2 * 2 * 128 * 4;
constexpr int SMEM_TOTAL = SMEM_BAR + 512;  // 32 mbarriers + TMEM slot; smem is declared 1024-aligned
// O_A [0,128), O_B [128,256), S buffers 256 + 64*{A0,A1,B0,B1}; the bf16 P of a
// block overwrites the first 32 columns of its own S buffer (A operand of PV)
constexpr uint32_t TMEM_COLS = 512;

struct Args {
  const __nv_bfloat16* qkv;
  int ldq;
  const int32_t* seq_slot;
  const int32_t* seq_len;
  const int32_t* row_off;
  const int32_t* row_node;
  const uint64_t* mask;
  int n_tmpl, W, A, Lmax;
  float scale_log2;
  int nsplit, mtiles;  // key splits per row tile; boundaries from the device length
  __nv_bfloat16* out;
  int ldout;
  unsigned long long* tl;     // development timeline (common.cuh)
  unsigned int tag;
  // PROPD_ATTN_QKV_F32 (one row tile per sequence): Q and the tree rows' K/V
  // from the fp32 QKV accumulator (row stride ldy floats, bf16-rounded); the
  // CTA writes the tree rows of its key range into the cache before its TMA
  // stream reads them
  const float* y;
  int ldy;
  __nv_bfloat16* kc;
  __nv_bfloat16* vc;
};

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

// Bits [t0, t0+32) of a row's visibility over tree nodes (0 outside [0, 64W)).
__device__ __forceinline__ uint32_t tree_bits32(const uint64_t* mrow, int W, int node, int t0) {
  if (mrow == nullptr) return low_bits(node + 1 - t0);  // causal: nodes 0..node
  if (t0 >= 64 * W || t0 <= -32) return 0u;
  const uint32_t* m = reinterpret_cast<const uint32_t*>(mrow);
  const int w = (t0 + 32) / 32 - 1;
  const int sh = t0 - 32 * w;
  const uint32_t lo = (w >= 0) ? m[w] : 0u;
  const uint32_t hi = (w + 1 < 2 * W) ? m[w + 1] : 0u;
  return sh ? __funnelshift_r(lo, hi, sh) : lo;
}

__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n)); }

// ---- split-KV combine inside a thread-block cluster (the key splits of one
// (sequence, head, row tile) are the cluster's CTAs): every CTA parks its
// unnormalised O and (m, l) in its now idle K ring; rank q finishes rows
// [q * ceil(nrows / splits), ...) reading all ranks through DSMEM.
constexpr int SMEM_PO = SMEM_K;                  // [128 rows][128] fp32 partial O (64 KB)
constexpr int SMEM_PM = SMEM_K + BM * DH * 4;    // [128] m (log2 domain)
constexpr int SMEM_PL = SMEM_PM + BM * 4;        // [128] l
static_assert(SMEM_PL + BM * 4 <= SMEM_V, "partial state must fit in the K ring");
__device__ __forceinline__ uint32_t cl_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cl_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t cl_map(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
__device__ __forceinline__ float cl_ld(uint32_t a) {
  float v;
  asm("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ float4 cl_ld4(uint32_t a) {
  float4 v;
  asm("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
  return v;
}
constexpr int MAX_SPLIT = 8;

__device__ __forceinline__ void cluster_combine(const uint8_t* smem, int nsplit, int nrows, int r0, int a,
                                                __nv_bfloat16* out, int ldout) {
  cl_sync();  // every split's partial state is visible cluster-wide
  const int rank = (int)cl_rank();
  const int per = (nrows + nsplit - 1) / nsplit;
  const int rb = rank * per, re = min(nrows, rb + per);
  uint32_t po[MAX_SPLIT], pm[MAX_SPLIT], pl[MAX_SPLIT];
#pragma unroll
  for (int q = 0; q < MAX_SPLIT; ++q) {
    const uint32_t rk = q < nsplit ? q : 0;
    po[q] = cl_map(smem_u32(smem + SMEM_PO), rk);
    pm[q] = cl_map(smem_u32(smem + SMEM_PM), rk);
    pl[q] = cl_map(smem_u32(smem + SMEM_PL), rk);
  }
  for (int e = threadIdx.x; e < (re - rb) * (DH / 4); e += blockDim.x) {
    const int r = rb + e / (DH / 4), d4 = (e % (DH / 4)) * 4;
    float ms[MAX_SPLIT], mx = -INFINITY;
#pragma unroll
    for (int q = 0; q < MAX_SPLIT; ++q) {
      ms[q] = q < nsplit ? cl_ld(pm[q] + r * 4) : -INFINITY;
      mx = fmaxf(mx, ms[q]);
    }
    float l = 0.f;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    if (mx != -INFINITY) {
#pragma unroll
      for (int q = 0; q < MAX_SPLIT; ++q) {
        if (q < nsplit && ms[q] != -INFINITY) {
          const float f = ex2(ms[q] - mx);
          l += cl_ld(pl[q] + r * 4) * f;
          const float4 o = cl_ld4(po[q] + (r * DH + d4) * 4);
          acc.x += o.x * f;
          acc.y += o.y * f;
          acc.z += o.z * f;
          acc.w += o.w * f;
        }
      }
    }
    const float inv = l > 0.f ? 1.f / l : 0.f;
    __nv_bfloat162 lo = __floats2bfloat162_rn(acc.x * inv, acc.y * inv), hi = __floats2bfloat162_rn(acc.z * inv, acc.w * inv);
    *reinterpret_cast<uint2*>(out + (size_t)(r0 + r) * ldout + a * DH + d4) =
        make_uint2(*reinterpret_cast<uint32_t*>(&lo), *reinterpret_cast<uint32_t*>(&hi));
  }
  cl_sync();  // peers may still be reading this CTA's state
}

__global__ void __launch_bounds__(THREADS, 1)
    attn_tc2_kernel(const __grid_constant__ CUtensorMap kmap, const __grid_constant__ CUtensorMap vmap, Args p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw;  // SW128 operands need 1024-byte alignment
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + SMEM_BAR);
  uint64_t* k_full = bars;                 // [KS]
  uint64_t* k_empty = k_full + KS;         // [KS]
  uint64_t* v_full = k_empty + KS;         // [VS]
  uint64_t* v_empty = v_full + VS;         // [VS]
  uint64_t* s_full = v_empty + VS;         // [4] A0 A1 B0 B1
  uint64_t* p_full = s_full + 4;           // [2] per group
  uint64_t* o_done = p_full + 2;           // [2] per group
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_done + 2);
  float* ml = reinterpret_cast<float*>(smem + SMEM_ML);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const unsigned long long t_entry = p.tl ? gtimer() : 0ull;
  pdl_wait();
  const unsigned long long t_wait = p.tl ? gtimer() : 0ull;
  const int s = blockIdx.x % p.nsplit, mt = blockIdx.x / p.nsplit;  // the splits of a row tile are one cluster
  const int a = blockIdx.y, b = blockIdx.z;
  const int slot = p.seq_slot[b];
  const int L = p.seq_len[slot];
  const int r0 = p.row_off[b] + mt * BM;
  const int nrows = min(BM, p.row_off[b + 1] - r0);
  if (nrows <= 0) return;
  const int nkeys = L + p.n_tmpl;
  // split boundaries from this sequence's device length (BN-key multiples;
  // launch geometry independent of the KV length)
  const int split_len = (((nkeys + BN - 1) / BN + p.nsplit - 1) / p.nsplit) * BN;
  const int k_begin = s * split_len;
  const int k_end = min(nkeys, k_begin + split_len);
  const int nblk = k_end > k_begin ? (k_end - k_begin + BN - 1) / BN : 0;
  if (nblk == 0) {  // no keys in this split: contribute an empty state to the cluster combine
    if (p.nsplit > 1) {
      float* pmv = reinterpret_cast<float*>(smem + SMEM_PM);
      float* plv = reinterpret_cast<float*>(smem + SMEM_PL);
      for (int r = threadIdx.x; r < BM; r += blockDim.x) {
        pmv[r] = -INFINITY;
        plv[r] = 0.f;
      }
      __syncthreads();
      cluster_combine(smem, p.nsplit, nrows, r0, a, p.out, p.ldout);
    }
    return;
  }
  const int nlive = min(4, (nrows + 31) / 32);

  if (threadIdx.x == 0) {
    for (int i = 0; i < KS; ++i) {
      mbar_init(&k_full[i], 1);
      mbar_init(&k_empty[i], 1);
    }
    for (int i = 0; i < VS; ++i) {
      mbar_init(&v_full[i], 1);
      mbar_init(&v_empty[i], 1);
    }
    for (int i = 0; i < 4; ++i) mbar_init(&s_full[i], 1);
    mbar_init(&p_full[0], 32 * nlive);
    mbar_init(&p_full[1], 32 * nlive);
    mbar_init(&o_done[0], 1);
    mbar_init(&o_done[1], 1);
    fence_barrier_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (p.y) {  // Q rows from the fp32 accumulator; this split's tree rows -> the cache
    const int H = p.A * DH;
    const size_t rb = ((size_t)slot * p.A + a) * p.Lmax;
    for (int i = threadIdx.x; i < BM * 16; i += THREADS) {
      const int r = i >> 4, c = i & 15;
      uint4 v = make_uint4(0, 0, 0, 0);
      if (r < nrows) {
        const float4* src = reinterpret_cast<const float4*>(p.y + (size_t)(r0 + r) * p.ldy + a * DH + c * 8);
        const float4 f0 = __ldcg(src), f1 = __ldcg(src + 1);
        v = make_uint4(pack_bf16(f0.x, f0.y), pack_bf16(f0.z, f0.w), pack_bf16(f1.x, f1.y), pack_bf16(f1.z, f1.w));
      }
      *reinterpret_cast<uint4*>(smem + SMEM_Q + sw128_chunk(r, c)) = v;
    }
    bool wrote = false;
    for (int i = threadIdx.x; i < nrows * 32; i += THREADS) {
      const int r = i >> 5, kv = (i >> 4) & 1, c = i & 15;
      const int pos = L + p.row_node[r0 + r];
      if (pos < k_begin || pos >= k_end) continue;
      wrote = true;
      const float4* src =
          reinterpret_cast<const float4*>(p.y + (size_t)(r0 + r) * p.ldy + (1 + kv) * H + a * DH + c * 8);
      const float4 f0 = __ldcg(src), f1 = __ldcg(src + 1);
      *reinterpret_cast<uint4*>((kv ? p.vc : p.kc) + (rb + pos) * DH + c * 8) =
          make_uint4(pack_bf16(f0.x, f0.y), pack_bf16(f0.z, f0.w), pack_bf16(f1.x, f1.y), pack_bf16(f1.z, f1.w));
    }
    if (wrote) asm volatile("fence.proxy.async.global;" ::: "memory");  // generic cache writes -> the TMA reads
  } else {  // Q rows -> SW128 K-major smem (cp.async; rows past nrows zero)
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
    asm volatile("cp.async.wait_all;" ::: "memory");
  }
  fence_proxy_async();
  tc_before_sync();
  __syncthreads();
  tc_after_sync();
  const uint32_t tmem = *tmem_slot;
  pdl_trigger();  // after the TMEM allocation (see common.cuh)
  const size_t row_base = ((size_t)slot * p.A + a) * p.Lmax;

  if (warp == 0 || warp == 10) {
    // ================= TMA producers: warp 0 streams K, warp 10 streams V =================
    if (lane == 0) {
      const bool isk = warp == 0;
      const int NS = isk ? KS : VS;
      uint64_t* full = isk ? k_full : v_full;
      uint64_t* empty = isk ? k_empty : v_empty;
      const CUtensorMap* map = isk ? &kmap : &vmap;
      uint8_t* ring = smem + (isk ? SMEM_K : SMEM_V);
      for (int j = 0; j < nblk; ++j) {
        const int st = j % NS;
        mbar_wait(&empty[st], ((j / NS) & 1) ^ 1, isk ? 11 : 17);
        mbar_expect_tx(&full[st], KV_TILE);
        const int row = (int)(row_base + k_begin + j * BN);
        uint8_t* d = ring + st * KV_TILE;
        tma_load_2d(d, map, &full[st], 0, row);
        tma_load_2d(d + KV_HALF, map, &full[st], 64, row);
      }
    }
  } else if (warp == 1) {
    // ================= MMA issuer =================
    if (lane == 0) {
      const uint32_t id_s = idesc_bf16(false, BN, 128), id_o = idesc_bf16(true, 128, 128);
      const uint32_t q_addr = smem_u32(smem + SMEM_Q);
      // Event loop: S_j = Q K_j^T is issued as soon as K_j has landed and its
      // S buffer is free (PV_{j-4}, the previous user of the buffer, issued),
      // O_g += P_j V_j as soon as P_j and V_j are ready; so S runs up to four
      // blocks ahead and each softmax group finds its next S already computed.
      // Every barrier is polled in phase order (no phase is ever skipped).
      int ns = 0, np = 0;
      uint32_t idle = 0;
      while (np < nblk) {
        bool prog = false;
        if (ns < nblk && ns < np + 4 && mbar_try(&k_full[ns % KS], (ns / KS) & 1)) {
          const int st = ns % KS;
          tc_after_sync();
          const int sb = (ns & 1) * 2 + ((ns >> 1) & 1);
          const uint32_t k_addr = smem_u32(smem + SMEM_K + st * KV_TILE);
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {  // K = dh 128 in steps of 16
            const uint64_t ad = sw128_desc(q_addr + (kk >> 2) * HALF + (kk & 3) * 32, 16, 1024);
            const uint64_t bd = sw128_desc(k_addr + (kk >> 2) * KV_HALF + (kk & 3) * 32, 16, 1024);
            mma_bf16(tmem + 256 + 64 * sb, ad, bd, id_s, kk > 0 ? 1u : 0u);
          }
          mma_commit(&s_full[sb]);
          mma_commit(&k_empty[st]);  // K is only needed by S: release its stage now
          ++ns;
          prog = true;
        }
        if (np < ns) {
          const int g = np & 1, i = np >> 1, st = np % VS;
          if (mbar_try(&p_full[g], i & 1) && mbar_try(&v_full[st], (np / VS) & 1)) {
            tc_after_sync();
            const int sb = g * 2 + (i & 1);
            const uint32_t p_tmem = tmem + 256 + 64 * sb;  // P (bf16 pairs) over its S buffer
            const uint32_t v_addr = smem_u32(smem + SMEM_V + st * KV_TILE);
#pragma unroll
            for (int kk = 0; kk < BN / 16; ++kk) {
              const uint64_t bd = sw128_desc(v_addr + kk * 2048, KV_HALF, 1024);
              mma_bf16_ts(tmem + g * 128, p_tmem + 8 * kk, bd, id_o, (i > 0 || kk > 0) ? 1u : 0u);
            }
            mma_commit(&v_empty[st]);
            mma_commit(&o_done[g]);
            ++np;
            prog = true;
          }
        }
        if (prog) {
          idle = 0;
        } else if (++idle > (1u << 28)) {
          mbar_timeout(12, (uint32_t)np);
        }
      }
    }
  } else {
    // ================= softmax warpgroups =================
    const int g = (warp - 2) >> 2;  // 0: even blocks, 1: odd blocks
    const int q4 = warp & 3;        // TMEM lane quadrant
    const int r = q4 * 32 + lane;
    const bool valid = r < nrows;
    const bool warp_live = q4 * 32 < nrows;
    const int row = r0 + r;
    const int node = valid ? p.row_node[row] : 0;
    const uint64_t* mrow = (valid && p.mask != nullptr) ? p.mask + (size_t)node * p.W : nullptr;
    const bool causal = p.mask == nullptr;
    const uint32_t lane_addr = tmem + ((uint32_t)(q4 * 32) << 16);
    const uint32_t o_addr = lane_addr + g * 128;
    const float scale = p.scale_log2;
    float m_ref = -INFINITY, l_sum = 0.f;
    const int nb = (nblk - g + 1) >> 1;  // blocks j = g, g+2, ...
    for (int i = 0; i < nb && warp_live; ++i) {
      const int j = 2 * i + g;
      const int sb = g * 2 + (i & 1);
      float sv[64];
      mbar_wait(&s_full[sb], (i >> 1) & 1, 14);
      tc_after_sync();
      {
        uint32_t* rv = reinterpret_cast<uint32_t*>(sv);
        TMEM_LD32(lane_addr + 256 + 64 * sb, rv);
        TMEM_LD32(lane_addr + 256 + 64 * sb + 32, (rv + 32));
        tmem_wait_ld();
      }
      const int key0 = k_begin + j * BN;
      const int ncache = L - key0, nvalid = k_end - key0;
      uint32_t vis[2];
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int t0 = key0 + 32 * q - L;
        uint32_t tb = 0u;
        if (valid && t0 > -32) tb = causal ? low_bits(node + 1 - t0) : tree_bits32(mrow, p.W, node, t0);
        vis[q] = valid ? ((low_bits(ncache - 32 * q) | tb) & low_bits(nvalid - 32 * q)) : 0u;
      }
      float mx8[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) mx8[u] = -INFINITY;
      if (__all_sync(0xffffffffu, (vis[0] & vis[1]) == 0xffffffffu)) {
#pragma unroll
        for (int k = 0; k < 64; ++k) mx8[k & 7] = fmaxf(mx8[k & 7], sv[k]);
      } else {
#pragma unroll
        for (int k = 0; k < 64; ++k) {
          sv[k] = ((vis[k >> 5] >> (k & 31)) & 1u) ? sv[k] : -INFINITY;
          mx8[k & 7] = fmaxf(mx8[k & 7], sv[k]);
        }
      }
      float mx = fmaxf(fmaxf(fmaxf(mx8[0], mx8[1]), fmaxf(mx8[2], mx8[3])),
                       fmaxf(fmaxf(mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7])));
      mx *= scale;
      float corr = 1.f;
      const bool grow = mx > m_ref + 8.f;
      if (grow) {
        corr = ex2(m_ref - mx);
        l_sum *= corr;
        m_ref = mx;
      }
      const float mneg = m_ref == -INFINITY ? 0.f : -m_ref;
      float ls8[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) ls8[u] = 0.f;
      uint32_t pk[32];  // P row as 32 bf16 pairs -> TMEM (A operand of O_g += P V)
#pragma unroll
      for (int k2 = 0; k2 < 32; ++k2) {
        const float2 pp = ex2x2(fmaf(sv[2 * k2], scale, mneg), fmaf(sv[2 * k2 + 1], scale, mneg));
        ls8[(2 * k2) & 7] += pp.x;
        ls8[(2 * k2 + 1) & 7] += pp.y;
        __nv_bfloat162 v2 = __floats2bfloat162_rn(pp.x, pp.y);
        pk[k2] = *reinterpret_cast<uint32_t*>(&v2);
      }
      TMEM_ST32(lane_addr + 256 + 64 * sb, pk);  // P_i goes to its own S buffer: no conflict with PV_{i-1}
      // Only now wait for this group's previous PV (it overlapped the exp
      // work above): O_g must be stable before a rescale, and the phase of
      // every PV is observed in order.
      if (i > 0) {
        mbar_wait(&o_done[g], (i - 1) & 1, 15);
        tc_after_sync();
      }
      if (i > 0 && __any_sync(0xffffffffu, grow)) {  // warp-collective O_g rescale
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          uint32_t rr[32];
          TMEM_LD32(o_addr + c * 32, rr);
          tmem_wait_ld();
#pragma unroll
          for (int k = 0; k < 32; ++k) rr[k] = __float_as_uint(__uint_as_float(rr[k]) * corr);
          TMEM_ST32(o_addr + c * 32, rr);
        }
      }
      tmem_wait_st();
      l_sum += ((ls8[0] + ls8[1]) + (ls8[2] + ls8[3])) + ((ls8[4] + ls8[5]) + (ls8[6] + ls8[7]));
      tc_before_sync();
      mbar_arrive(&p_full[g]);
    }
    // ---- epilogue: merge the two groups' (m, l, O) and write ----
    if (warp_live && nb > 0) {
      mbar_wait(&o_done[g], (nb - 1) & 1, 16);
      tc_after_sync();
    }
    ml[(g * 2 + 0) * 128 + r] = m_ref;
    ml[(g * 2 + 1) * 128 + r] = l_sum;
    tc_before_sync();
    named_sync(1, 256);  // both groups' last PV observed complete
    tc_after_sync();
    if (warp_live) {
      const float mA = ml[r], lA = ml[128 + r];
      const bool hasB = nblk > 1;
      const float mB = hasB ? ml[256 + r] : -INFINITY, lB = hasB ? ml[384 + r] : 0.f;
      const float m = fmaxf(mA, mB);
      const float fA = mA == -INFINITY ? 0.f : ex2(mA - m);
      const float fB = mB == -INFINITY ? 0.f : ex2(mB - m);
      const float l = lA * fA + lB * fB;
      const float inv = l > 0.f ? 1.f / l : 0.f;
#pragma unroll
      for (int c = 0; c < 2; ++c) {  // this group writes columns [64g, 64g + 64)
        const int col = 64 * g + 32 * c;
        uint32_t ra[32], rb[32];
        TMEM_LD32(lane_addr + col, ra);
        if (hasB) TMEM_LD32(lane_addr + 128 + col, rb);
        tmem_wait_ld();
        float o[32];
#pragma unroll
        for (int k = 0; k < 32; ++k)
          o[k] = __uint_as_float(ra[k]) * fA + (hasB ? __uint_as_float(rb[k]) * fB : 0.f);
        if (valid) {
          if (p.nsplit == 1) {
            __nv_bfloat16* dst = p.out + (size_t)row * p.ldout + a * DH + col;
#pragma unroll
            for (int k8 = 0; k8 < 4; ++k8) {
              uint32_t pk[4];
#pragma unroll
              for (int h = 0; h < 4; ++h) {
                __nv_bfloat162 v2 = __floats2bfloat162_rn(o[k8 * 8 + 2 * h] * inv, o[k8 * 8 + 2 * h + 1] * inv);
                pk[h] = *reinterpret_cast<uint32_t*>(&v2);
              }
              *reinterpret_cast<uint4*>(dst + k8 * 8) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
            }
          } else {  // unnormalised partial state of this split -> own shared memory
            float4* po = reinterpret_cast<float4*>(smem + SMEM_PO + ((size_t)r * DH + col) * 4);
#pragma unroll
            for (int k4 = 0; k4 < 8; ++k4) po[k4] = make_float4(o[4 * k4], o[4 * k4 + 1], o[4 * k4 + 2], o[4 * k4 + 3]);
            if (g == 0 && c == 0) {
              reinterpret_cast<float*>(smem + SMEM_PM)[r] = m;
              reinterpret_cast<float*>(smem + SMEM_PL)[r] = l;
            }
          }
        }
      }
    }
  }
  tc_before_sync();
  __syncthreads();
  tc_after_sync();
  if (warp == 1) {
    __syncwarp();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
  }
  if (p.nsplit > 1) {
    __syncwarp();
    cluster_combine(smem, p.nsplit, nrows, r0, a, p.out, p.ldout);
  }
  if (p.tl && threadIdx.x == 0) trace_record(p.tl, p.tag, t_entry, t_wait, t_wait, 2);
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

// [rows, 128] bf16 view of a K or V cache layer; box 64 x BN rows, SWIZZLE_128B.
static bool kv_map64(CUtensorMap* m, const void* base, uint64_t rows) {
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
  cuuint32_t box[2] = {64, (cuuint32_t)BN};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return false;
  cache[key] = {rows, *m};
  return true;
}

}  // namespace tc2


int attention_tc2_prepare() {
  cudaError_t e = cudaFuncSetAttribute(tc2::attn_tc2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       tc2::SMEM_TOTAL);
  return e == cudaSuccess ? 0 : fail("prepare(tc2): %s", cudaGetErrorString(e));
}

int attention_tc2_bf16(int B, int Bg, int M, int A, int Lmax, int n_slots, int max_rows_per_seq, int max_keys,
                       const void* qkv, int ldqkv, const void* kc, const void* vc, const int32_t* seq_slot,
                       const int32_t* seq_len, const int32_t* row_off, const int32_t* row_node, const uint64_t* mask,
                       int n_tmpl, int W, void* out, int ldout, void* ws, int64_t ws_bytes, cudaStream_t st,
                       bool* handled, bool qy) {
  *handled = false;
  if (n_slots <= 0 || W > 4 || (ldqkv % (qy ? 4 : 8)) != 0 || (ldout % 8) != 0) return 0;
  if (qy && max_rows_per_seq > tc2::BM) return 0;  // (a second row tile would need the first tile's tree rows)
  CUtensorMap km, vm;
  const uint64_t rows = (uint64_t)n_slots * A * Lmax;
  if (!tc2::kv_map64(&km, kc, rows) || !tc2::kv_map64(&vm, vc, rows)) return 0;
  const int mtiles = (max_rows_per_seq + tc2::BM - 1) / tc2::BM;
  const int ctas = Bg * A * mtiles;  // sequences with a KV cache (Bg <= B)
  const int nblk_max = (max_keys + tc2::BN - 1) / tc2::BN;
  // key splits per row tile (one cluster each, <= 8): one wave of one CTA
  // per SM at small batch (more, shorter splits measured slower at B=8-16)
  int nsplit = propd_num_sms() / ctas;
  if (nsplit > nblk_max) nsplit = nblk_max;
  if (nsplit > tc2::MAX_SPLIT) nsplit = tc2::MAX_SPLIT;
  if (nsplit < 1) nsplit = 1;
  (void)ws;
  (void)ws_bytes;
  const int blocks_per_split = (nblk_max + nsplit - 1) / nsplit;
  nsplit = (nblk_max + blocks_per_split - 1) / blocks_per_split;
  tc2::Args p{};
  p.qkv = qy ? nullptr : reinterpret_cast<const __nv_bfloat16*>(qkv);
  p.ldq = ldqkv;
  p.y = qy ? reinterpret_cast<const float*>(qkv) : nullptr;
  p.ldy = ldqkv;
  p.kc = reinterpret_cast<__nv_bfloat16*>(const_cast<void*>(kc));
  p.vc = reinterpret_cast<__nv_bfloat16*>(const_cast<void*>(vc));
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
  p.nsplit = nsplit;
  p.mtiles = mtiles;
  p.out = reinterpret_cast<__nv_bfloat16*>(out);
  p.ldout = ldout;
  p.tl = g_dbg_trace;
  p.tag = g_dbg_tag++;
  static bool attr = false;
  if (!attr) {
    if (int e = attention_tc2_prepare()) return e;
    attr = true;
  }
  *handled = true;
  (void)M;
  dim3 grid(nsplit * mtiles, A, B);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(tc2::THREADS);
  cfg.dynamicSmemBytes = tc2::SMEM_TOTAL;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  int na = 0;
  if (nsplit > 1) {
    at[na].id = cudaLaunchAttributeClusterDimension;
    at[na].val.clusterDim.x = nsplit;
    at[na].val.clusterDim.y = 1;
    at[na].val.clusterDim.z = 1;
    ++na;
  }
  if (pdl_enabled()) {
    at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.attrs = at;
  cfg.numAttrs = na;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, tc2::attn_tc2_kernel, km, vm, p);
  if (e != cudaSuccess) {
    (void)cudaGetLastError();
    return fail("tree_attention(tc2): %s", cudaGetErrorString(e));
  }
  return check_launch("tree_attention(tc2)");
}

}  // namespace propd
