// Shared device helpers for libpropd (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <cstdlib>
#include <string>
#include <utility>

#include "../../include/propd.h"

namespace propd {

// ---- error plumbing (C ABI returns int, message via propd_last_error) ----
void set_error(const std::string& msg);
int fail(const char* fmt, ...);
int check_launch(const char* what);

#define PROPD_REQUIRE(cond, ...)                 \
  do {                                           \
    if (!(cond)) return ::propd::fail(__VA_ARGS__); \
  } while (0)

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// ---- programmatic dependent launch (PDL) ----
// The per-layer kernels are launched with programmatic stream serialisation:
// a kernel may be scheduled while its predecessor drains, runs its
// independent prologue (barrier init, TMEM alloc, weight prefetch), then
// blocks in pdl_wait() until the predecessor grid has completed and its
// writes are visible.  Every kernel launched through launch_pdl MUST call
// pdl_wait() before it touches memory written by earlier kernels, and must
// call pdl_trigger() only after its own TMEM allocation (a dependent CTA that
// grabbed the SM's TMEM first would otherwise deadlock it).  Kernels without
// TMEM trigger before their own wait, so the next weight-streaming GEMM is
// launched early and prefetches its weights while they run (its pre-wait
// section touches nothing but the weights).  Both are no-ops for a normal
// launch.  PROPD_PDL=0 in the environment disables it.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
bool pdl_enabled();
bool pdl_skip(const char* what);  // PROPD_PDL_SKIP="name,..." (dev A/B): launches of these names without PDL

template <typename... Exp, typename... Act>
inline int launch_pdl(const char* what, void (*kern)(Exp...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                      Act&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = (pdl_enabled() && !pdl_skip(what)) ? 1 : 0;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, std::forward<Act>(args)...);
  if (e != cudaSuccess) {
    (void)cudaGetLastError();
    return fail("%s: %s", what, cudaGetErrorString(e));
  }
  return check_launch(what);
}

// ---- development trace (scripts/kernel_timeline.py) ----
// When a trace buffer is installed (propd_debug_timeline), instrumented kernels
// append one record per CTA: [tag, cta, smid, t_entry, t_after_pdl_wait,
// t_main_done, t_exit] (globaltimer ns); buf[0] is the record counter, buf[1]
// the capacity in records, records
// start at buf[8].  tag = host launch sequence number, slot 7 = kernel kind.  Off (NULL) normally.
extern unsigned long long* g_dbg_trace;
extern unsigned int g_dbg_tag;
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned int smid() {
  unsigned int s;
  asm volatile("mov.u32 %0, %smid;" : "=r"(s));
  return s;
}
// kind (record slot 7, low byte): 1 = weight-streaming GEMM, 2 = attention, 4 = transposed attention;
// GEMM records carry their shape above it (gemm_ws.cu: N / 128, K / 64, live rows, accumulate)
__device__ __forceinline__ void trace_record(unsigned long long* buf, unsigned int tag, unsigned long long t0,
                                             unsigned long long t1, unsigned long long t2,
                                             unsigned long long kind = 0, unsigned long long slot2 = ~0ull) {
  if (buf == nullptr) return;
  const unsigned long long t3 = gtimer();
  const unsigned long long i = atomicAdd(buf, 1ull);
  if (i >= buf[1]) return;  // capacity (records) in buf[1]
  unsigned long long* r = buf + 8 + i * 8;
  r[0] = tag;
  r[1] = blockIdx.x + (unsigned long long)gridDim.x * (blockIdx.y + (unsigned long long)gridDim.y * blockIdx.z);
  r[2] = slot2 != ~0ull ? slot2 : smid();  // (debug builds may put a timestamp here)
  r[3] = t0;
  r[4] = t1;
  r[5] = t2;
  r[6] = t3;
  r[7] = kind;
}

// ---- key-split count of a split-KV attention launch ----
// units = (sequence, head, row-tile) work items, slots = co-resident CTAs of
// the kernel on the device.  If every unit can get max_split splits within
// one wave, take as many as fit (latency-bound small batches); otherwise the
// split count in [1, max_split] whose grid fills its last wave best
// (>= 95 %, else the best fill), so large batches do not lose a partial wave.
// development override of a launch heuristic's split count (0 = unset)
inline int env_int(const char* name) {
  const char* e = getenv(name);
  return e != nullptr ? atoi(e) : 0;
}

inline int wave_split(int units, int slots, int max_split) {
  if (max_split < 1) return 1;
  if (units * max_split <= slots) return max_split;
  if (2 * units <= slots) return slots / units;  // one wave, as many splits as fit
  int best = 1;
  double best_eff = 0.0;
  for (int ns = 1; ns <= max_split; ++ns) {
    const long long ctas = (long long)units * ns;
    const long long waves = (ctas + slots - 1) / slots;
    const double eff = (double)ctas / (double)(waves * slots);
    if (eff >= 0.95) return ns;
    if (eff > best_eff + 1e-9) {
      best_eff = eff;
      best = ns;
    }
  }
  return best;
}

// ---- element conversion ----
__device__ __forceinline__ float to_f(float v) { return v; }
__device__ __forceinline__ float to_f(__nv_bfloat16 v) { return __bfloat162float(v); }
template <typename T> __device__ __forceinline__ T from_f(float v);
template <> __device__ __forceinline__ float from_f<float>(float v) { return v; }
template <> __device__ __forceinline__ __nv_bfloat16 from_f<__nv_bfloat16>(float v) { return __float2bfloat16_rn(v); }

// ---- warp / block reductions ----
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ int warp_isum(int v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// block-wide sum for blockDim.x a multiple of 32 (<= 1024); red has >= 32 floats
__device__ __forceinline__ float block_sum(float v, float* red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) red[wid] = v;
  __syncthreads();
  float t = (lane < nw) ? red[lane] : 0.f;
  t = warp_sum(t);
  return t;
}

// Order-preserving key of an fp32 value (+0 and -0 map to the same key).
__device__ __forceinline__ uint32_t float_key(float f) {
  uint32_t u = __float_as_uint(f);
  if ((u & 0x7fffffffu) == 0u) u = 0u;  // canonicalise -0.0 -> +0.0
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

}  // namespace propd

#define PROPD_DISPATCH_DTYPE(dtype, T, ...)                              \
  [&]() -> int {                                                         \
    if ((dtype) == PROPD_F32) { using T = float; return __VA_ARGS__(); } \
    if ((dtype) == PROPD_BF16) { using T = __nv_bfloat16; return __VA_ARGS__(); } \
    return ::propd::fail("unsupported dtype code %d", (int)(dtype));     \
  }()
