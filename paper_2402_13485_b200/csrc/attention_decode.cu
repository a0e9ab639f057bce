// K2 for few query rows per sequence (the bonus pass: 1 row; tiny trees):
// a streaming split-KV decode kernel on the CUDA cores with the split-KV
// combine done inside a thread-block cluster.
//
// With one row per sequence there is no GEMM to feed a tensor core; the work
// is a pure stream of the sequence's K/V cache (backends.py:216-233 with
// n = 1).  Design for B200:
//   - every (sequence, head) is cut into <= 8 key splits that form ONE
//     cluster (grid.x = splits), so that even batch 1 puts ~2 CTAs on every
//     SM and the whole cache of a launch is in flight at once;
//   - each CTA streams its split in 64-key chunks (K and V of a chunk are two
//     contiguous 16 KB rows of the [Lmax, 128] cache tile) with bulk async
//     copies into a 3-deep shared-memory ring, one mbarrier per stage;
//   - a half-warp covers one key (16 lanes x 8 bf16 = the 256-byte row) for
//     up to ROWS query rows; scores are reduced with 4 shuffles and softmax is
//     online per 8-key batch;
//   - the per-split (m, l, o) states are merged through distributed shared
//     memory by the cluster (each rank finishes a slice of the output), so
//     there is no workspace and no second combine launch.
#include "tc_common.cuh"

namespace propd {
namespace dec {
using namespace propd::tc;

constexpr int CHUNK = 64, RING = 3, MAX_SPLIT = 8;
constexpr int DH = 128, NW = 8, THREADS = 32 * NW, KB = CHUNK / (2 * NW);  // keys per half-warp batch

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
  __nv_bfloat16* out;
  int ldout;
  unsigned long long* tl;  // development timeline (common.cuh)
  unsigned int tag;
  // PROPD_ATTN_QKV_F32: Q and the rows' own K/V from the fp32 QKV accumulator
  // (row stride ldy floats, bf16-rounded); the CTA whose key range holds a
  // row's cache slot writes its K/V there before the bulk copies read it
  const float* y;
  int ldy;
};

__device__ __forceinline__ void bf16x8_to_f32(const uint4& u, float* f) {
  const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    f[2 * i] = __uint_as_float(w[i] << 16);
    f[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
  }
}

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_nrank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t map_rank(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
__device__ __forceinline__ float ld_dsmem(uint32_t addr) {
  float v;
  asm("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(addr));
  return v;
}
// contiguous global -> shared bulk copy completing on an mbarrier
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

template <int ROWS>
struct Smem {
  __nv_bfloat16 k[RING][CHUNK * DH];
  __nv_bfloat16 v[RING][CHUNK * DH];
  float red_m[NW][ROWS], red_l[NW][ROWS];
  float red_o[NW][ROWS][DH];
  float part_m[ROWS], part_l[ROWS];  // this split's merged state (read by the cluster)
  float part_o[ROWS][DH];
  uint64_t full[RING];
};

template <int ROWS>
__global__ void __launch_bounds__(THREADS) decode_kernel(Args p) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  Smem<ROWS>& sm = *reinterpret_cast<Smem<ROWS>*>(smem_raw);
  const int s = blockIdx.x, a = blockIdx.y, b = blockIdx.z;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int half = lane >> 4, hl = lane & 15;  // half-warp, lane within it (dims 8*hl .. 8*hl+7)
  const unsigned long long t_entry = p.tl ? gtimer() : 0ull;
  if (threadIdx.x == 0) {
    for (int i = 0; i < RING; ++i) mbar_init(&sm.full[i], 1);
    fence_barrier_init();
  }
  __syncthreads();
  pdl_wait();
  pdl_trigger();
  const unsigned long long t_wait = p.tl ? gtimer() : 0ull;
  const int slot = p.seq_slot[b];
  const int L = p.seq_len[slot];
  const int r0 = p.row_off[b];
  const int nrows = min(ROWS, p.row_off[b + 1] - r0);
  const int nkeys = L + p.n_tmpl;
  // split boundaries from this sequence's device length (16-key multiples;
  // launch geometry independent of the KV length)
  const int nspl = (int)gridDim.x;
  const int split_len = (((nkeys + nspl - 1) / nspl + 15) / 16) * 16;
  const int k_begin = s * split_len;
  const int k_end = nrows > 0 ? min(nkeys, k_begin + split_len) : k_begin;
  const int nchunk = k_end > k_begin ? (k_end - k_begin + CHUNK - 1) / CHUNK : 0;
  const size_t tile = ((size_t)slot * p.A + a) * p.Lmax;  // first cache row of this (sequence, head)
  if (p.y) {  // this split's rows -> the cache (their K/V exist only in the accumulator)
    const int H = p.A * DH;
    bool wrote = false;
    for (int i = threadIdx.x; i < nrows * 32; i += THREADS) {
      const int r = i >> 5, kv = (i >> 4) & 1, c = i & 15;
      const int pos = L + p.row_node[r0 + r];
      if (pos < k_begin || pos >= k_end) continue;
      wrote = true;
      const float4* src =
          reinterpret_cast<const float4*>(p.y + (size_t)(r0 + r) * p.ldy + (1 + kv) * H + a * DH + c * 8);
      const float4 f0 = __ldcg(src), f1 = __ldcg(src + 1);
      __nv_bfloat162 h0 = __floats2bfloat162_rn(f0.x, f0.y), h1 = __floats2bfloat162_rn(f0.z, f0.w);
      __nv_bfloat162 h2 = __floats2bfloat162_rn(f1.x, f1.y), h3 = __floats2bfloat162_rn(f1.z, f1.w);
      *reinterpret_cast<uint4*>(const_cast<__nv_bfloat16*>(kv ? p.vc : p.kc) + (tile + pos) * DH + c * 8) =
          make_uint4(*reinterpret_cast<uint32_t*>(&h0), *reinterpret_cast<uint32_t*>(&h1),
                     *reinterpret_cast<uint32_t*>(&h2), *reinterpret_cast<uint32_t*>(&h3));
    }
    if (wrote) asm volatile("fence.proxy.async.global;" ::: "memory");  // generic cache writes -> the bulk copies below
    __syncthreads();
  }
  auto issue = [&](int c) {
    const int st = c % RING;
    const int key0 = k_begin + c * CHUNK;
    const int nk = min(CHUNK, k_end - key0);  // the split's last chunk loads only its own keys
    const uint32_t bytes = (uint32_t)nk * DH * 2;
    mbar_expect_tx(&sm.full[st], 2 * bytes);
    bulk_load(sm.k[st], p.kc + (tile + key0) * DH, bytes, &sm.full[st]);
    bulk_load(sm.v[st], p.vc + (tile + key0) * DH, bytes, &sm.full[st]);
  };
  if (threadIdx.x == 0)
    for (int c = 0; c < min(RING, nchunk); ++c) issue(c);

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
      if (p.y) {  // bf16-rounded as the Q operand would hold it
        const float4* src = reinterpret_cast<const float4*>(p.y + (size_t)(r0 + r) * p.ldy + a * DH + hl * 8);
        const float4 f0 = __ldcg(src), f1 = __ldcg(src + 1);
        const float fv[8] = {f0.x, f0.y, f0.z, f0.w, f1.x, f1.y, f1.z, f1.w};
#pragma unroll
        for (int i = 0; i < 8; ++i) q[r][i] = __bfloat162float(__float2bfloat16_rn(fv[i]));
      } else {
        const uint4 u = *reinterpret_cast<const uint4*>(p.qkv + (size_t)(r0 + r) * p.ldq + a * DH + hl * 8);
        bf16x8_to_f32(u, q[r]);
      }
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
  for (int c = 0; c < nchunk; ++c) {
    const int st = c % RING;
    mbar_wait(&sm.full[st], (c / RING) & 1, 41);
    // warp w: keys [2KB w, 2KB (w + 1)) of the chunk, half-warp h: KB of them
    const int kc0 = warp * 2 * KB + half * KB;
    uint4 kr[KB], vr[KB];
#pragma unroll
    for (int t = 0; t < KB; ++t) {
      kr[t] = *reinterpret_cast<const uint4*>(&sm.k[st][(kc0 + t) * DH + hl * 8]);
      vr[t] = *reinterpret_cast<const uint4*>(&sm.v[st][(kc0 + t) * DH + hl * 8]);
    }
    const int kbase = k_begin + c * CHUNK + kc0;
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
        const int key = kbase + t;
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
        // masked keys are skipped, not multiplied by 0: the ring tail past
        // the cache tile holds stale shared memory (possibly NaN patterns)
        if (sc[t] == -INFINITY) continue;
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
    __syncthreads();  // every warp is done with stage st
    if (threadIdx.x == 0 && c + RING < nchunk) issue(c + RING);
  }
  // merge the two half-warps (same dims, different keys), then the warps
#pragma unroll
  for (int r = 0; r < ROWS; ++r)
#pragma unroll
    for (int i = 0; i < 8; ++i) o[r][i] += __shfl_xor_sync(0xffffffffu, o[r][i], 16);
  if (half == 0) {
#pragma unroll
    for (int r = 0; r < ROWS; ++r) {
#pragma unroll
      for (int i = 0; i < 8; ++i) sm.red_o[warp][r][hl * 8 + i] = o[r][i];
      if (hl == 0) {
        sm.red_m[warp][r] = m[r];
        sm.red_l[warp][r] = l[r];
      }
    }
  }
  __syncthreads();
  const unsigned long long t_loop = p.tl ? gtimer() : 0ull;
  const int nsplit = (int)cluster_nrank();
  for (int idx = threadIdx.x; idx < ROWS * DH; idx += THREADS) {
    const int r = idx / DH, d = idx - r * DH;
    if (r >= nrows) continue;
    float mx = -INFINITY;
#pragma unroll
    for (int w = 0; w < NW; ++w) mx = fmaxf(mx, sm.red_m[w][r]);
    float lsum = 0.f, acc = 0.f;
    if (mx != -INFINITY) {
#pragma unroll
      for (int w = 0; w < NW; ++w) {
        const float f = sm.red_m[w][r] == -INFINITY ? 0.f : ex2(sm.red_m[w][r] - mx);
        lsum += sm.red_l[w][r] * f;
        acc += sm.red_o[w][r][d] * f;
      }
    }
    if (nsplit == 1) {
      p.out[(size_t)(r0 + r) * p.ldout + a * DH + d] = __float2bfloat16_rn(lsum > 0.f ? acc / lsum : 0.f);
    } else {
      sm.part_o[r][d] = acc;
      if (d == 0) {
        sm.part_m[r] = mx;
        sm.part_l[r] = lsum;
      }
    }
  }
  if (nsplit > 1) {
    // cluster combine: rank q finishes elements [q * per, (q + 1) * per) of the
    // nrows x 128 output through distributed shared memory
    cluster_sync_all();
    const int rank = (int)cluster_rank();
    const int total = nrows * DH;
    const int per = (total + nsplit - 1) / nsplit;
    uint32_t base_m[MAX_SPLIT], base_l[MAX_SPLIT], base_o[MAX_SPLIT];
#pragma unroll
    for (int qq = 0; qq < MAX_SPLIT; ++qq) {
      const uint32_t rk = qq < nsplit ? qq : 0;
      base_m[qq] = map_rank(smem_u32(sm.part_m), rk);
      base_l[qq] = map_rank(smem_u32(sm.part_l), rk);
      base_o[qq] = map_rank(smem_u32(&sm.part_o[0][0]), rk);
    }
    for (int e = rank * per + threadIdx.x; e < min(total, (rank + 1) * per); e += THREADS) {
      const int r = e / DH, d = e - r * DH;
      float ms[MAX_SPLIT], mx = -INFINITY;
#pragma unroll
      for (int qq = 0; qq < MAX_SPLIT; ++qq) {
        ms[qq] = qq < nsplit ? ld_dsmem(base_m[qq] + r * 4) : -INFINITY;
        mx = fmaxf(mx, ms[qq]);
      }
      float lsum = 0.f, acc = 0.f;
      if (mx != -INFINITY) {
#pragma unroll
        for (int qq = 0; qq < MAX_SPLIT; ++qq) {
          if (qq < nsplit && ms[qq] != -INFINITY) {
            const float f = ex2(ms[qq] - mx);
            lsum += ld_dsmem(base_l[qq] + r * 4) * f;
            acc += ld_dsmem(base_o[qq] + (r * DH + d) * 4) * f;
          }
        }
      }
      p.out[(size_t)(r0 + r) * p.ldout + a * DH + d] = __float2bfloat16_rn(lsum > 0.f ? acc / lsum : 0.f);
    }
    cluster_sync_all();  // peers may still read this CTA's state
  }
  if (p.tl && threadIdx.x == 0) trace_record(p.tl, p.tag, t_entry, t_wait, t_loop, 2);
}

// Clusters of `cs` decode CTAs resident at once (cudaOccupancyMaxActiveClusters,
// cached per (rows variant, cluster size)); 0 on a query error.
template <int ROWS>
static int max_clusters_t(int cs) {
  static int cache[MAX_SPLIT + 1] = {};
  if (cs < 1 || cs > MAX_SPLIT) return 0;
  if (cache[cs] == 0) {
    constexpr int smem = (int)sizeof(Smem<ROWS>);
    if (cudaFuncSetAttribute(decode_kernel<ROWS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess ||
        cudaFuncSetAttribute(decode_kernel<ROWS>, cudaFuncAttributePreferredSharedMemoryCarveout,
                             cudaSharedmemCarveoutMaxShared) != cudaSuccess) {
      (void)cudaGetLastError();
      return 0;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs, 1, 1);
    cfg.blockDim = dim3(THREADS);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, decode_kernel<ROWS>, &cfg) != cudaSuccess) {
      (void)cudaGetLastError();
      return 0;
    }
    cache[cs] = n > 0 ? n : -1;
  }
  return cache[cs] > 0 ? cache[cs] : 0;
}
static int max_clusters(int rows, int cs) {
  if (cs <= 1) return 1 << 30;
  return rows <= 1 ? max_clusters_t<1>(cs) : (rows <= 2 ? max_clusters_t<2>(cs) : max_clusters_t<4>(cs));
}

template <int ROWS>
static int launch(const Args& p, dim3 grid, cudaStream_t st) {
  static bool attr = false;
  constexpr int smem = (int)sizeof(Smem<ROWS>);
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(decode_kernel<ROWS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(decode_kernel<ROWS>, cudaFuncAttributePreferredSharedMemoryCarveout,
                               cudaSharedmemCarveoutMaxShared);
    if (e != cudaSuccess) return fail("tree_attention(decode): %s", cudaGetErrorString(e));
    attr = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  int na = 0;
  if (grid.x > 1) {  // the key splits of one (sequence, head) form a cluster
    at[na].id = cudaLaunchAttributeClusterDimension;
    at[na].val.clusterDim.x = grid.x;
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
  const cudaError_t e = cudaLaunchKernelEx(&cfg, decode_kernel<ROWS>, p);
  if (e != cudaSuccess) {
    (void)cudaGetLastError();
    return fail("tree_attention(decode): %s", cudaGetErrorString(e));
  }
  return check_launch("tree_attention(decode)");
}

}  // namespace dec

// Called by propd_tree_attention for bf16 / dh = 128 with <= 4 rows per sequence.
int attention_decode_bf16(int B, int Bg, int M, int A, int Lmax, int max_rows_per_seq, int max_keys, const void* qkv,
                          int ldqkv, const void* kc, const void* vc, const int32_t* seq_slot, const int32_t* seq_len,
                          const int32_t* row_off, const int32_t* row_node, const uint64_t* mask, int n_tmpl, int W,
                          void* out, int ldout, void* ws, int64_t ws_bytes, cudaStream_t st, bool* handled,
                          bool qy) {
  *handled = false;
  (void)M;
  (void)ws;
  (void)ws_bytes;
  if (max_rows_per_seq > 4 || W > 4 || (ldqkv % (qy ? 4 : 8)) != 0) return 0;
  // splits per (sequence, head), one cluster each: enough CTAs for ~2 per SM
  // at small batch; at large batch (>= one wave of pairs) one split unless
  // its last wave leaves over 20 % of the CTA slots idle, then the split
  // count whose last wave is fullest (measured at B=32 x 32 heads, KV 1024:
  // 1 split 110 us per launch vs 127 us for the 2 splits wave filling picks)
  const int pairs = Bg * A;  // sequences with a KV cache (Bg <= B)
  const int slots = 2 * propd_num_sms();
  int nsplit = (slots + pairs - 1) / pairs;
  if (2 * pairs > slots) {
    const int waves = (pairs + slots - 1) / slots;
    nsplit = (double)pairs / ((double)waves * slots) >= 0.8 ? 1 : wave_split(pairs, slots, 2);
  }
  const int cap = (max_keys + dec::CHUNK - 1) / dec::CHUNK;
  if (nsplit > cap) nsplit = cap;
  if (nsplit > dec::MAX_SPLIT) nsplit = dec::MAX_SPLIT;
  if (nsplit < 1) nsplit = 1;
  // all clusters of one wave must fit at once (clusters of s CTAs are placed
  // within a GPC: at B = 1, 32 clusters of 8 do not, and the second wave
  // costs ~5 us per launch): the largest split whose clusters are co-resident
  if (Bg * A * nsplit <= slots)
    while (nsplit > 1) {
      const int mc = dec::max_clusters(max_rows_per_seq, nsplit);
      if (mc == 0 || pairs <= mc) break;  // (0: query failed, keep the split)
      --nsplit;
    }
  static const int split_override = env_int("PROPD_DEC_SPLIT");
  if (split_override > 0) nsplit = split_override < dec::MAX_SPLIT ? split_override : dec::MAX_SPLIT;
  // boundaries: any multiple of 16 keys from the device length (chunks start
  // at the split's first key and the last one loads only the keys left, so
  // splits stay balanced across SMs); no split empty at max_keys
  const int split_len = (((max_keys + nsplit - 1) / nsplit + 15) / 16) * 16;
  nsplit = (max_keys + split_len - 1) / split_len;
  dec::Args p{};
  p.qkv = qy ? nullptr : reinterpret_cast<const __nv_bfloat16*>(qkv);
  p.ldq = ldqkv;
  p.y = qy ? reinterpret_cast<const float*>(qkv) : nullptr;
  p.ldy = ldqkv;
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
  p.out = reinterpret_cast<__nv_bfloat16*>(out);
  p.ldout = ldout;
  p.tl = g_dbg_trace;
  p.tag = g_dbg_tag++;
  *handled = true;
  dim3 grid(nsplit, A, B);
  switch (max_rows_per_seq) {
    case 1: return dec::launch<1>(p, grid, st);
    case 2: return dec::launch<2>(p, grid, st);
    default: return dec::launch<4>(p, grid, st);
  }
}

}  // namespace propd
