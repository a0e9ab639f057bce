// K2 for trees of <= 64 rows per (sequence, head): the transposed tcgen05
// kernel ("tcT").  Reference semantics as attention_tc2.cu (backends.py:216-233).
//
// Why transposed: with M = 128 query rows per MMA (tc2) a pruned tree of ~20
// rows wastes 84% of every S = Q K^T and O += P V instruction, the tensor
// pipe re-reads a 32 KB zero-padded Q tile from shared memory for every
// 64-key block, and one warp per softmax group does all the exponentials.
// Measured (scripts/attn_probe.py with the MMAs stubbed out): the S MMA alone
// holds tc2 at 0.84 of the copy bandwidth at B = 64, KV 4096.  Here keys run
// along M instead:
//   S^T_j = K_j Q^T     (M = 128 keys, N = 32 rows, K = 128 dims; A = K_j
//                        K-major, B = Q K-major, both SW128 from TMA/cp.async)
//   O^T  += V_j^T P_j^T (M = 128 dims, N = 32 rows, K = 128 keys; A = V_j
//                        MN-major straight from the same TMA tile, B = P^T
//                        K-major written by the softmax warps)
// so each MMA is 4x (2x at 64 rows) smaller, Q is 8-16 KB, and the softmax of
// a block is spread over four warps (TMEM lane = key: warp q owns keys
// 32q..32q+31 of the block, 32 row values per thread and 32-row half).  Row maxima / sums are lane
// transposes: a 5-step butterfly leaves lane l with row l's maximum over the
// warp's keys, one named barrier merges the four warps.  l stays as per-thread
// partial sums (one per row) until the end.
//
// Warp roles: warp 0 TMA K, warp 1 TMEM alloc + MMA issue (event loop), one
// softmax warpgroup per 32-row half (warps 2-5, 6-9), then the V TMA warp
// (224 threads at 32 rows, 352 at 64).  Key splits of one (sequence,
// head) form a thread-block cluster merged through distributed shared memory.
#include <unordered_map>

#include "tc_common.cuh"

namespace propd {
namespace tct {
using namespace propd::tc;

constexpr int BK = 128;   // keys per block (M of S^T)
constexpr int DH = 128;
constexpr int NSB = 4;         // S^T buffers in TMEM (S runs up to NSB blocks ahead of PV)
constexpr int MAX_SPLIT = 8;
constexpr int KV_HALF = BK * 128;     // [128 keys x 64 dims] SW128 = 16 KB
constexpr int KV_TILE = 2 * KV_HALF;  // 32 KB

// Shared-memory / TMEM plan for NR query rows per tile (32 or 64) and RING
// K / V ring stages (32 KB each): 3 with one CTA per SM; 1 with two CTAs per
// SM (32 rows: 90 KB, 256 TMEM columns, <= 146 registers) for launches of
// more tiles than SMs (one wave instead of two at B = 5-9, and the other CTA of
// an SM hides each CTA's exposed K/V latency at larger batch).
template <int NR_, int RING = 3>
struct Cfg {
  static constexpr int NR = NR_;
  static constexpr int KS = RING, VS = RING;
  static constexpr int MINB = RING == 1 ? 2 : 1;  // CTAs per SM (launch bounds)
  static_assert(RING >= 3 || NR == 32, "two CTAs per SM: 32-row tiles only");
  static constexpr int NH = NR / 32;             // softmax warpgroups, one per 32-row half
  static constexpr int NPB = NR == 32 ? 2 : 1;   // P^T buffers (one at 64 rows: shared memory)
  static constexpr int VWARP = 2 + 4 * NH;       // V producer warp (after the softmax warps)
  static constexpr int THREADS = 32 * (VWARP + 1);
  static constexpr int Q_HALF = NR * 128;        // [NR rows x 64 dims]
  static constexpr int P_HALF = NR * 128;        // [NR rows x 64 keys]
  static constexpr int P_TILE = 2 * P_HALF;
  static constexpr int SMEM_K = 0;
  static constexpr int SMEM_V = SMEM_K + KS * KV_TILE;
  static constexpr int SMEM_Q = SMEM_V + VS * KV_TILE;
  static constexpr int SMEM_P = SMEM_Q + 2 * Q_HALF;
  // [NH][2][4 warps][32] floats: block-max exchange per group (double
  // buffered; the final row sums reuse the buffer the last block left idle)
  static constexpr int SMEM_RED = SMEM_P + NPB * P_TILE;
  static constexpr int SMEM_NODE = SMEM_RED + NH * 2 * 4 * 32 * 4;  // [NR] template node of each row
  static constexpr int SMEM_BAR = SMEM_NODE + NR * 4;
  static constexpr int SMEM_TOTAL = SMEM_BAR + 192;
  // cluster combine state parks in the idle K ring after the main loop
  static constexpr int SMEM_PO = SMEM_K;              // [NR rows][128] fp32
  static constexpr int SMEM_PM = SMEM_PO + NR * DH * 4;  // [NR] m (log2 domain)
  static constexpr int SMEM_PL = SMEM_PM + NR * 4;       // [NR] l
  static_assert(SMEM_PL + NR * 4 <= SMEM_V, "partial state must fit in the K ring");
  static_assert(SMEM_TOTAL <= 227 * 1024, "shared memory");
  // TMEM: O^T [0, NR), S^T buffers NR + NR * b
  static constexpr uint32_t O_COL = 0, S_COL = NR, TMEM_COLS = NR == 32 ? 256 : 512;
};

struct Args {
  const __nv_bfloat16* qkv;
  int ldq;
  // PROPD_ATTN_QKV_F32: Q and the tree rows' K/V from the fp32 QKV accumulator
  // (row stride ldy floats; bf16-rounded as the QKV tail would store them); the
  // CTA writes the tree rows of its key range into the cache itself
  const float* y;
  int ldy;
  __nv_bfloat16* kc;
  __nv_bfloat16* vc;
  const int32_t* seq_slot;
  const int32_t* seq_len;
  const int32_t* row_off;
  const int32_t* row_node;
  const uint64_t* mask;
  int n_tmpl, W, A, Lmax;
  float scale_log2;
  int nsplit;  // key splits per (sequence, head); boundaries from the device length
  __nv_bfloat16* out;
  int ldout;
  unsigned long long* tl;  // development timeline (common.cuh)
  unsigned int tag;
};

__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n)); }
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
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

// Merge the key splits of one (sequence, head): rank q finishes rows
// [q * ceil(nrows / splits), ...) from every rank's parked (O, m, l).
template <class C>
__device__ __forceinline__ void cluster_combine(const uint8_t* smem, int nsplit, int nrows, int r0, int a,
                                                __nv_bfloat16* out, int ldout) {
  cl_sync();
  const int rank = (int)cl_rank();
  const int per = (nrows + nsplit - 1) / nsplit;
  const int rb = rank * per, re = min(nrows, rb + per);
  uint32_t po[MAX_SPLIT], pm[MAX_SPLIT], pl[MAX_SPLIT];
#pragma unroll
  for (int q = 0; q < MAX_SPLIT; ++q) {
    const uint32_t rk = q < nsplit ? q : 0;
    po[q] = cl_map(smem_u32(smem + C::SMEM_PO), rk);
    pm[q] = cl_map(smem_u32(smem + C::SMEM_PM), rk);
    pl[q] = cl_map(smem_u32(smem + C::SMEM_PL), rk);
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
    *reinterpret_cast<uint2*>(out + (size_t)(r0 + r) * ldout + a * DH + d4) =
        make_uint2(pack_bf16(acc.x * inv, acc.y * inv), pack_bf16(acc.z * inv, acc.w * inv));
  }
  cl_sync();  // peers may still be reading this CTA's state
}

// Butterfly transpose-reduce of 32 per-lane values: lane l ends with the
// reduction over the warp's 32 lanes of value index l (in t[0]).
template <bool MAX>
__device__ __forceinline__ void lane_transpose_reduce(float (&t)[32], int lane) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    const bool up = (lane & o) != 0;
#pragma unroll
    for (int i = 0; i < o; ++i) {
      const float send = up ? t[i] : t[i + o];
      const float keep = up ? t[i + o] : t[i];
      const float recv = __shfl_xor_sync(0xffffffffu, send, o);
      t[i] = MAX ? fmaxf(keep, recv) : keep + recv;
    }
  }
}

template <class C>
__global__ void __launch_bounds__(C::THREADS, C::MINB)
    attn_tct_kernel(const __grid_constant__ CUtensorMap kmap, const __grid_constant__ CUtensorMap vmap, Args p) {
  constexpr int NR = C::NR, NH = C::NH, NPB = C::NPB;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::SMEM_BAR);
  uint64_t* k_full = bars;
  uint64_t* k_empty = k_full + C::KS;
  uint64_t* v_full = k_empty + C::KS;
  uint64_t* v_empty = v_full + C::VS;
  uint64_t* s_full = v_empty + C::VS;   // [NSB]
  uint64_t* p_full = s_full + NSB;   // [NPB]
  uint64_t* pv_done = p_full + NPB;  // [NPB]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(pv_done + NPB);
  float* red = reinterpret_cast<float*>(smem + C::SMEM_RED);
  int* rnode = reinterpret_cast<int*>(smem + C::SMEM_NODE);
  // development timeline (first S seen, softmax loop end): the tail of the
  // barrier block (static shared memory would push the 64-row plan past 227 KB)
  unsigned long long* s_t = reinterpret_cast<unsigned long long*>(smem + C::SMEM_BAR + 176);
  static_assert(8 * (2 * C::KS + 2 * C::VS + NSB + 2 * C::NPB) + 4 <= 176, "barrier block");

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // independent of the predecessor: barriers, tensor-map prefetch
  if (threadIdx.x == 0) {
    for (int i = 0; i < C::KS; ++i) {
      mbar_init(&k_full[i], 1);
      mbar_init(&k_empty[i], 1);
    }
    for (int i = 0; i < C::VS; ++i) {
      mbar_init(&v_full[i], 1);
      mbar_init(&v_empty[i], 1);
    }
    for (int i = 0; i < NSB; ++i) mbar_init(&s_full[i], 1);
    for (int i = 0; i < NPB; ++i) mbar_init(&pv_done[i], 1);
    fence_barrier_init();
    asm volatile("prefetch.tensormap [%0];" ::"l"(&kmap) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&vmap) : "memory");
  }
  __syncthreads();
  pdl_wait();
  const unsigned long long t_wait = p.tl ? gtimer() : 0ull;
  const int s = blockIdx.x, a = blockIdx.y, b = blockIdx.z;
  const int slot = p.seq_slot[b];
  const int L = p.seq_len[slot];
  const int r0 = p.row_off[b];
  const int nrows = min(NR, p.row_off[b + 1] - r0);
  if (nrows <= 0) return;  // uniform over the cluster (same sequence)
  const int nkeys = L + p.n_tmpl;
  // split boundaries from this sequence's device length (64-key multiples):
  // the launch geometry does not depend on the KV length, so captured graphs
  // stay valid as sequences grow
  const int split_len = ((((nkeys + 63) >> 6) + p.nsplit - 1) / p.nsplit) * 64;
  const int k_begin = s * split_len;
  const int k_end = min(nkeys, k_begin + split_len);
  const int nblk = k_end > k_begin ? (k_end - k_begin + BK - 1) / BK : 0;
  if (nblk == 0) {  // no keys in this split: an empty state for the cluster combine
    if (p.nsplit > 1) {
      for (int r = threadIdx.x; r < NR; r += blockDim.x) {
        reinterpret_cast<float*>(smem + C::SMEM_PM)[r] = -INFINITY;
        reinterpret_cast<float*>(smem + C::SMEM_PL)[r] = 0.f;
      }
      __syncthreads();
      cluster_combine<C>(smem, p.nsplit, nrows, r0, a, p.out, p.ldout);
    }
    return;
  }
  const size_t row_base = ((size_t)slot * p.A + a) * p.Lmax;
  // the first ring fill goes out before anything else (its latency overlaps
  // the Q load, the TMEM allocation and the block-wide sync)
  const bool producer = (warp == 0 || warp == C::VWARP) && lane == 0;
  // (with the tree rows written by this CTA below, only blocks wholly below L go out early)
  const int npre = p.y ? max(0, min(min(C::KS, nblk), (L - k_begin) / BK)) : min(C::KS, nblk);  // C::KS == C::VS
  if (producer) {
    const bool isk = warp == 0;
    uint64_t* full = isk ? k_full : v_full;
    const CUtensorMap* map = isk ? &kmap : &vmap;
    uint8_t* ring = smem + (isk ? C::SMEM_K : C::SMEM_V);
    for (int j = 0; j < npre; ++j) {
      mbar_expect_tx(&full[j], KV_TILE);
      const int row = (int)(row_base + k_begin + j * BK);
      tma_load_2d(ring + j * KV_TILE, map, &full[j], 0, row);
      tma_load_2d(ring + j * KV_TILE + KV_HALF, map, &full[j], 64, row);
    }
  }

  // live 32-row halves: a 64-row launch whose sequence has <= 32 surviving
  // rows runs N = 32 MMAs and one softmax group (row capacities are host
  // upper bounds; the survivor counts live on the device)
  const int live_h = NH == 1 ? 1 : (nrows + 31) >> 5;
  if (threadIdx.x == 32) {
    for (int i = 0; i < NPB; ++i) mbar_init(&p_full[i], 128 * live_h);
    fence_barrier_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(C::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (p.y) {  // Q rows from the fp32 accumulator; this split's tree rows -> the cache
    const int H = p.A * DH;
    for (int i = threadIdx.x; i < NR * 16; i += C::THREADS) {
      const int r = i >> 4, c = i & 15;
      uint8_t* dst =
          smem + C::SMEM_Q + (c >> 3) * C::Q_HALF + (r >> 3) * 1024 + (r & 7) * 128 + (((c & 7) ^ (r & 7)) << 4);
      uint4 v = make_uint4(0, 0, 0, 0);
      if (r < nrows) {
        const float4* src = reinterpret_cast<const float4*>(p.y + (size_t)(r0 + r) * p.ldy + a * DH + c * 8);
        const float4 f0 = __ldcg(src), f1 = __ldcg(src + 1);
        v = make_uint4(pack_bf16(f0.x, f0.y), pack_bf16(f0.z, f0.w), pack_bf16(f1.x, f1.y), pack_bf16(f1.z, f1.w));
      }
      *reinterpret_cast<uint4*>(dst) = v;
    }
    bool wrote = false;
    for (int i = threadIdx.x; i < nrows * 32; i += C::THREADS) {
      const int r = i >> 5, kv = (i >> 4) & 1, c = i & 15;
      const int pos = L + p.row_node[r0 + r];
      if (pos < k_begin || pos >= k_end) continue;
      wrote = true;
      const float4* src =
          reinterpret_cast<const float4*>(p.y + (size_t)(r0 + r) * p.ldy + (1 + kv) * H + a * DH + c * 8);
      const float4 f0 = __ldcg(src), f1 = __ldcg(src + 1);
      __nv_bfloat16* dst = (kv ? p.vc : p.kc) + (row_base + pos) * DH + c * 8;
      *reinterpret_cast<uint4*>(dst) =
          make_uint4(pack_bf16(f0.x, f0.y), pack_bf16(f0.z, f0.w), pack_bf16(f1.x, f1.y), pack_bf16(f1.z, f1.w));
    }
    if (wrote) asm volatile("fence.proxy.async.global;" ::: "memory");  // generic cache writes -> the TMA reads below
    for (int r = threadIdx.x; r < NR; r += C::THREADS) rnode[r] = r < nrows ? p.row_node[r0 + r] : 0;
  } else {  // Q rows -> SW128 K-major [NR rows x 128 dims] (rows past nrows zero)
    const __nv_bfloat16* qbase = p.qkv + a * DH;
    for (int i = threadIdx.x; i < NR * 16; i += C::THREADS) {
      const int r = i >> 4, c = i & 15;
      uint8_t* dst =
          smem + C::SMEM_Q + (c >> 3) * C::Q_HALF + (r >> 3) * 1024 + (r & 7) * 128 + (((c & 7) ^ (r & 7)) << 4);
      if (r < nrows)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)),
                     "l"(qbase + (size_t)(r0 + r) * p.ldq + c * 8)
                     : "memory");
      else
        *reinterpret_cast<uint4*>(dst) = make_uint4(0, 0, 0, 0);
    }
    for (int r = threadIdx.x; r < NR; r += C::THREADS) rnode[r] = r < nrows ? p.row_node[r0 + r] : 0;
    asm volatile("cp.async.wait_all;" ::: "memory");
  }
  fence_proxy_async();
  tc_before_sync();
  __syncthreads();
  tc_after_sync();
  const uint32_t tmem = *tmem_slot;
  pdl_trigger();  // after the TMEM allocation (see common.cuh)

  if (warp == 0 || warp == C::VWARP) {
    // ================= TMA producers: warp 0 streams K, warp VWARP streams V =================
    if (lane == 0) {
      const bool isk = warp == 0;
      const int NS = isk ? C::KS : C::VS;
      uint64_t* full = isk ? k_full : v_full;
      uint64_t* empty = isk ? k_empty : v_empty;
      const CUtensorMap* map = isk ? &kmap : &vmap;
      uint8_t* ring = smem + (isk ? C::SMEM_K : C::SMEM_V);
      for (int j = npre; j < nblk; ++j) {
        const int st = j % NS;
        mbar_wait(&empty[st], ((j / NS) & 1) ^ 1, isk ? 61 : 67);
        mbar_expect_tx(&full[st], KV_TILE);
        const int row = (int)(row_base + k_begin + j * BK);
        uint8_t* d = ring + st * KV_TILE;
        tma_load_2d(d, map, &full[st], 0, row);
        tma_load_2d(d + KV_HALF, map, &full[st], 64, row);
      }
    }
  } else if (warp == 1) {
    // ================= MMA issuer =================
    if (lane == 0) {
      const uint32_t nn = 32u * live_h;
      const uint32_t id_s = idesc_bf16(false, nn, BK);
      const uint32_t id_o = idesc_bf16(false, nn, DH) | (1u << 15);  // A = V^T read MN-major from the V tile
      const uint32_t q_addr = smem_u32(smem + C::SMEM_Q);
      int ns = 0, np = 0;
      uint32_t idle = 0;
      while (np < nblk) {
        bool prog = false;
        if (ns < nblk && ns < np + NSB && mbar_try(&k_full[ns % C::KS], (ns / C::KS) & 1)) {
          const int st = ns % C::KS;
          tc_after_sync();
          const uint32_t k_addr = smem_u32(smem + C::SMEM_K + st * KV_TILE);
#pragma unroll
          for (int kk = 0; kk < DH / 16; ++kk) {
            const uint64_t ad = sw128_desc(k_addr + (kk >> 2) * KV_HALF + (kk & 3) * 32, 16, 1024);
            const uint64_t bd = sw128_desc(q_addr + (kk >> 2) * C::Q_HALF + (kk & 3) * 32, 16, 1024);
            mma_bf16(tmem + C::S_COL + NR * (ns % NSB), ad, bd, id_s, kk > 0 ? 1u : 0u);
          }
          mma_commit(&s_full[ns % NSB]);
          mma_commit(&k_empty[st]);
          ++ns;
          prog = true;
        }
        if (np < ns) {
          const int st = np % C::VS, pb = np % NPB;
          if (mbar_try(&p_full[pb], (np / NPB) & 1) && mbar_try(&v_full[st], (np / C::VS) & 1)) {
            tc_after_sync();
            const uint32_t v_addr = smem_u32(smem + C::SMEM_V + st * KV_TILE);
            const uint32_t p_addr = smem_u32(smem + C::SMEM_P + pb * C::P_TILE);
#pragma unroll
            for (int kk = 0; kk < BK / 16; ++kk) {
              const uint64_t ad = sw128_desc(v_addr + kk * 2048, KV_HALF, 1024);
              const uint64_t bd = sw128_desc(p_addr + (kk >> 2) * C::P_HALF + (kk & 3) * 32, 16, 1024);
              mma_bf16(tmem + C::O_COL, ad, bd, id_o, (np > 0 || kk > 0) ? 1u : 0u);
            }
            mma_commit(&v_empty[st]);
            mma_commit(&pv_done[pb]);
            ++np;
            prog = true;
          }
        }
        if (prog) {
          idle = 0;
        } else if (++idle > (1u << 28)) {
          mbar_timeout(62, (uint32_t)np);
        }
      }
    }
  } else if (warp < C::VWARP && (NH == 1 || ((warp - 2) >> 2) < live_h)) {
    // ============ softmax: group h = rows 32h..32h+31, warp q owns keys 32q..32q+31 of each block ============
    const int h = NH == 1 ? 0 : (warp - 2) >> 2, q = warp & 3;
    const uint32_t lane_base = tmem + ((uint32_t)(q * 32) << 16);
    const float scale = p.scale_log2;
    float m_ref = -INFINITY;  // running reference max of row 32h + lane (log2 domain; same in the group's warps)
    float lpart[32];          // this thread's key-lane partial sums of rows 32h..32h+31
#pragma unroll
    for (int n = 0; n < 32; ++n) lpart[n] = 0.f;
    const int kin = (q & 1) * 32 + (lane & ~1);  // even key of this lane pair within its 64-key half
    const int pchunk = kin >> 3, pbyte = (kin & 7) * 2;
    const bool odd = lane & 1;
    float* red_g = red + h * 256;
    for (int j = 0; j < nblk; ++j) {
      const int sb = j % NSB, pb = j % NPB;
      mbar_wait(&s_full[sb], (j / NSB) & 1, 63);
      tc_after_sync();
      if (p.tl && j == 0 && threadIdx.x == 64) s_t[0] = gtimer();
      const int key = k_begin + j * BK + q * 32 + lane;
      float v[32];
      TMEM_LD32(lane_base + C::S_COL + NR * sb + 32 * h, reinterpret_cast<uint32_t*>(v));
      tmem_wait_ld();
      // visibility of key `key` for rows 32h + n
      if (key >= k_end) {
#pragma unroll
        for (int n = 0; n < 32; ++n) v[n] = -INFINITY;
      } else if (key >= L) {
        const int t = key - L;  // tree node index of this key
#pragma unroll
        for (int n = 0; n < 32; ++n) {
          const int r = 32 * h + n;
          bool vis = r < nrows;
          if (vis) {
            const int node = rnode[r];
            vis = p.mask != nullptr ? ((__ldg(p.mask + (size_t)node * p.W + (t >> 6)) >> (t & 63)) & 1ull) != 0
                                    : t <= node;
          }
          v[n] = vis ? v[n] * scale : -INFINITY;
        }
      } else {
#pragma unroll
        for (int n = 0; n < 32; ++n) v[n] = 32 * h + n < nrows ? v[n] * scale : -INFINITY;
      }
      // block maximum of every row: butterfly transpose (lane l ends with row 32h + l) + 4-warp merge
      float tr[32];
#pragma unroll
      for (int n = 0; n < 32; ++n) tr[n] = v[n];
      lane_transpose_reduce<true>(tr, lane);
      float* rb = red_g + (j & 1) * 128;
      rb[q * 32 + lane] = tr[0];
      named_sync(1 + h, 128);
      const float bm = fmaxf(fmaxf(rb[lane], rb[32 + lane]), fmaxf(rb[64 + lane], rb[96 + lane]));
      // lazy rescale: move the reference only when the block max exceeds it by > 2^8
      const bool grow = bm > m_ref + 8.f;
      float corr = 1.f;
      if (grow) {
        corr = ex2(m_ref - bm);
        m_ref = bm;
      }
      const bool any_grow = __any_sync(0xffffffffu, grow);
      const float mneg = m_ref == -INFINITY ? 0.f : -m_ref;
#pragma unroll
      for (int n = 0; n < 32; n += 2) {
        const float2 pp = ex2x2(v[n] + __shfl_sync(0xffffffffu, mneg, n), v[n + 1] + __shfl_sync(0xffffffffu, mneg, n + 1));
        v[n] = pp.x;
        v[n + 1] = pp.y;
      }
      if (any_grow) {
#pragma unroll
        for (int n = 0; n < 32; ++n) lpart[n] *= __shfl_sync(0xffffffffu, corr, n);
      }
#pragma unroll
      for (int n = 0; n < 32; ++n) lpart[n] += v[n];
      // P^T (K-major [NR rows x 128 keys], SW128): lane pairs exchange so
      // each stores one 4-byte word (keys 2i, 2i+1) for 16 rows
      if (j >= NPB) mbar_wait(&pv_done[pb], ((j / NPB) - 1) & 1, 64);  // PV_{j-NPB} has read this buffer
      uint8_t* pbase = smem + C::SMEM_P + pb * C::P_TILE + (q >> 1) * C::P_HALF;
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const float send = odd ? v[i] : v[16 + i];
        const float recv = __shfl_xor_sync(0xffffffffu, send, 1);
        const int n = 32 * h + (odd ? 16 + i : i);
        const uint32_t w = odd ? pack_bf16(recv, v[16 + i]) : pack_bf16(v[i], recv);
        *reinterpret_cast<uint32_t*>(pbase + (n >> 3) * 1024 + (n & 7) * 128 + ((pchunk ^ (n & 7)) << 4) + pbyte) = w;
      }
      if (any_grow && j > 0) {  // O^T columns (rows) whose reference moved: rescale after PV_{j-1}
        mbar_wait(&pv_done[(j - 1) % NPB], ((j - 1) / NPB) & 1, 65);
        tc_after_sync();
        uint32_t o[32];
        TMEM_LD32(lane_base + C::O_COL + 32 * h, o);
        tmem_wait_ld();
#pragma unroll
        for (int n = 0; n < 32; ++n) o[n] = __float_as_uint(__uint_as_float(o[n]) * __shfl_sync(0xffffffffu, corr, n));
        TMEM_ST32(lane_base + C::O_COL + 32 * h, o);
        tmem_wait_st();
      }
      fence_proxy_async();  // P^T stores -> visible to the tensor core
      tc_before_sync();
      mbar_arrive(&p_full[pb]);
    }
    // ---- epilogue: row sums, then O^T (lane = dim) -> rows ----
    if (p.tl && threadIdx.x == 64) s_t[1] = gtimer();
    lane_transpose_reduce<false>(lpart, lane);
    float* lred = red_g + (nblk & 1) * 128;  // the exchange buffer the last block did not use
    lred[q * 32 + lane] = lpart[0];
    mbar_wait(&pv_done[(nblk - 1) % NPB], ((nblk - 1) / NPB) & 1, 66);
    tc_after_sync();
    named_sync(1 + h, 128);
    const float lrow = (lred[lane] + lred[32 + lane]) + (lred[64 + lane] + lred[96 + lane]);  // row 32h + lane
    const int d = q * 32 + lane;
    uint32_t o[32];
    TMEM_LD32(lane_base + C::O_COL + 32 * h, o);
    tmem_wait_ld();
    if (p.nsplit == 1) {
      const float inv = lrow > 0.f ? 1.f / lrow : 0.f;
#pragma unroll
      for (int n = 0; n < 32; ++n) {
        const float f = __shfl_sync(0xffffffffu, inv, n);
        if (32 * h + n < nrows)
          p.out[(size_t)(r0 + 32 * h + n) * p.ldout + a * DH + d] = __float2bfloat16_rn(__uint_as_float(o[n]) * f);
      }
    } else {  // park the unnormalised state; the K ring is idle (every S has completed)
      float* po = reinterpret_cast<float*>(smem + C::SMEM_PO);
#pragma unroll
      for (int n = 0; n < 32; ++n) po[(32 * h + n) * DH + d] = __uint_as_float(o[n]);
      if (q == 0) {
        reinterpret_cast<float*>(smem + C::SMEM_PM)[32 * h + lane] = m_ref;
        reinterpret_cast<float*>(smem + C::SMEM_PL)[32 * h + lane] = lrow;
      }
    }
  }
  tc_before_sync();
  __syncthreads();
  tc_after_sync();
  if (warp == 1) {
    __syncwarp();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(C::TMEM_COLS));
  }
  if (p.nsplit > 1) cluster_combine<C>(smem, p.nsplit, nrows, r0, a, p.out, p.ldout);
  // kind 4: (first S seen, dependency release, softmax loop end, exit)
  if (p.tl && threadIdx.x == 0) trace_record(p.tl, p.tag, s_t[0], t_wait, s_t[1], 4);
}

// ------------------------------------------------------------------ host --
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncodeFn encode_fn() {
  static EncodeFn fn = nullptr;
  if (!fn) {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(f);
  }
  return fn;
}

// [rows, 128] bf16 view of a K or V cache layer; box 64 dims x 128 keys, SWIZZLE_128B.
static bool kv_map128(CUtensorMap* m, const void* base, uint64_t rows) {
  static std::unordered_map<uint64_t, std::pair<uint64_t, CUtensorMap>> cache;
  const uint64_t key = (uint64_t)(uintptr_t)base;
  auto it = cache.find(key);
  if (it != cache.end() && it->second.first == rows) {
    *m = it->second.second;
    return true;
  }
  EncodeFn enc = encode_fn();
  if (!enc) return false;
  cuuint64_t dims[2] = {128, rows};
  cuuint64_t strides[1] = {128 * 2};
  cuuint32_t box[2] = {64, (cuuint32_t)BK};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return false;
  cache[key] = {rows, *m};
  return true;
}

}  // namespace tct

// PROPD_TCT: 0 = never (tc2 for every multi-row launch), 2 = whenever the
// shape fits (no latency heuristic), unset / other = auto
static int tct_mode() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("PROPD_TCT");
    v = (e != nullptr && e[0] == '0') ? 0 : ((e != nullptr && e[0] == '2') ? 2 : 1);
  }
  return v;
}

template <class C>
static int tct_launch(const CUtensorMap& km, const CUtensorMap& vm, const tct::Args& p, int nsplit, int A, int B,
                      cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(tct::attn_tct_kernel<C>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         C::SMEM_TOTAL);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(tct::attn_tct_kernel<C>, cudaFuncAttributePreferredSharedMemoryCarveout,
                               cudaSharedmemCarveoutMaxShared);
    if (e != cudaSuccess) return fail("prepare(tcT): %s", cudaGetErrorString(e));
    attr = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(nsplit, A, B);
  cfg.blockDim = dim3(C::THREADS);
  cfg.dynamicSmemBytes = C::SMEM_TOTAL;
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
  const cudaError_t e = cudaLaunchKernelEx(&cfg, tct::attn_tct_kernel<C>, km, vm, p);
  if (e != cudaSuccess) {
    (void)cudaGetLastError();
    return fail("tree_attention(tcT): %s", cudaGetErrorString(e));
  }
  return check_launch("tree_attention(tcT)");
}

int attention_tct_bf16(int B, int Bg, int A, int Lmax, int n_slots, int max_rows_per_seq, int max_keys, const void* qkv,
                       int ldqkv, const void* kc, const void* vc, const int32_t* seq_slot, const int32_t* seq_len,
                       const int32_t* row_off, const int32_t* row_node, const uint64_t* mask, int n_tmpl, int W,
                       void* out, int ldout, cudaStream_t st, bool force, bool* handled, bool qy) {
  *handled = false;
  if (!force && tct_mode() == 0) return 0;
  if (n_slots <= 0 || max_rows_per_seq > 64 || W > 4 || (ldqkv % (qy ? 4 : 8)) != 0) return 0;
  // > 32-row capacity with few 128-key blocks per SM (B=1-4 at KV <= 2K) is
  // latency-bound, where the row-major tc2 kernel's shorter per-block chain
  // wins (measured: 11.2 vs 14.7 us at B=1/KV 512, 22.2 vs 25.0 at B=4/KV 1K)
  if (!force && tct_mode() != 2 && max_rows_per_seq > 32 &&
      (long long)Bg * A * ((max_keys + 127) / 128) < 16LL * propd_num_sms())
    return 0;
  CUtensorMap km, vm;
  const uint64_t rows = (uint64_t)n_slots * A * Lmax;
  if (!tct::kv_map128(&km, kc, rows) || !tct::kv_map128(&vm, vc, rows)) return 0;
  const int ctas = Bg * A;  // sequences with a KV cache (Bg <= B)
  // <= 32-row tiles over more tiles than SMs: the 1-stage shape at two CTAs per SM
  static const int two_override = env_int("PROPD_TCT_TWO");  // -1: never, 1: whenever the tiles fit (A/B)
  // (measured, scripts/attn_probe.py at 16 rows: 0.58 -> 0.75 of the copy peak at B=8 / KV 1024, 0.74 -> 0.91
  // at B=64 / KV 1024, 1.04 -> 1.08 at B=64 / KV 4096; equal at B=1)
  const bool two = two_override != -1 && max_rows_per_seq <= 32 && (two_override == 1 || ctas > propd_num_sms());
  // key splits per (sequence, head), one cluster each (<= 8): one wave of one
  // CTA per SM at small batch; split boundaries on 64-key multiples (a
  // split's last 128-key block may be partly masked)
  int nsplit = propd_num_sms() / ctas;
  const int nh = (max_keys + 63) / 64;
  if (nsplit > nh) nsplit = nh;
  if (nsplit > tct::MAX_SPLIT) nsplit = tct::MAX_SPLIT;
  if (nsplit < 1) nsplit = 1;
  static const int split_override = env_int("PROPD_TCT_SPLIT");
  if (split_override > 0) nsplit = split_override < tct::MAX_SPLIT ? split_override : tct::MAX_SPLIT;
  const int per = (nh + nsplit - 1) / nsplit;  // 64-key units per split at max_keys
  nsplit = (nh + per - 1) / per;               // no split empty at max_keys
  tct::Args p{};
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
  p.out = reinterpret_cast<__nv_bfloat16*>(out);
  p.ldout = ldout;
  p.tl = g_dbg_trace;
  p.tag = g_dbg_tag++;
  *handled = true;
  if (two) return tct_launch<tct::Cfg<32, 1>>(km, vm, p, nsplit, A, B, st);
  return max_rows_per_seq <= 32 ? tct_launch<tct::Cfg<32>>(km, vm, p, nsplit, A, B, st)
                                : tct_launch<tct::Cfg<64>>(km, vm, p, nsplit, A, B, st);
}

}  // namespace propd
