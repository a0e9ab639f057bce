// Probability-based early pruning and typical acceptance — the two north-star
// criteria the reference does not ship (pruning.py:76-82 disables the
// probability threshold; verification.py:30-53 is greedy only).  Their
// definitions are the fp64 restatements oracle/treedecode_port.py
// probability_prune / typical_verify (PAPER.md:401-405 for the marginal path
// probability; Medusa's typical acceptance).  Probabilities are evaluated in
// fp64 from the fp32 logits, so a decision only differs from the oracle's when
// its margin is below the logits' own rounding.
#include "common.cuh"

namespace propd {

constexpr int MAX_PATH = 32;  // tree depth bound = MAX_D draft heads (prune_verify.cu)

// Per row of z = logits / temp: stats[r] = (log-sum-exp, entropy) in fp64.
// idx (nullable) gathers rows: row r reads logits[idx[r]].
__global__ void __launch_bounds__(256) row_lse_kernel(int V, int ld, const float* __restrict__ logits,
                                                      const int32_t* __restrict__ idx, double temp,
                                                      double* __restrict__ stats, const int32_t* __restrict__ rows_dev) {
  __shared__ float redf[32];
  __shared__ double redd[2][32];
  const int r = blockIdx.x;
  if (rows_dev && r >= *rows_dev) return;
  const float* row = logits + (size_t)(idx ? idx[r] : r) * ld;
  float mx = -INFINITY;
  for (int v = threadIdx.x; v < V; v += blockDim.x) mx = fmaxf(mx, row[v]);
  mx = warp_max(mx);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if (lane == 0) redf[wid] = mx;
  __syncthreads();
  if (wid == 0) {
    float t = lane < nw ? redf[lane] : -INFINITY;
    t = warp_max(t);
    if (lane == 0) redf[0] = t;
  }
  __syncthreads();
  const double zm = __ddiv_rn((double)redf[0], temp);
  double s = 0.0, sz = 0.0;
  for (int v = threadIdx.x; v < V; v += blockDim.x) {
    const double z = __ddiv_rn((double)row[v], temp);
    const double e = exp(z - zm);
    s += e;
    sz += e * z;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    s += __shfl_xor_sync(0xffffffffu, s, o);
    sz += __shfl_xor_sync(0xffffffffu, sz, o);
  }
  if (lane == 0) {
    redd[0][wid] = s;
    redd[1][wid] = sz;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0, b = 0.0;
    for (int w = 0; w < nw; ++w) {
      a += redd[0][w];
      b += redd[1][w];
    }
    const double lse = zm + log(a);
    stats[2 * r] = lse;
    stats[2 * r + 1] = lse - b / a;
  }
}

// member[b*n+i] = depth-1, or log P(path to i) >= log_tau where log P sums
// (l_parent[token] - lse_parent) over the path, top-down (fp64, no FMA).
__global__ void early_prob_member_kernel(int B, int n, int P, int V, double log_tau, const float* __restrict__ early,
                                         const double* __restrict__ early_stats, const int32_t* __restrict__ parent,
                                         const int32_t* __restrict__ parent_slot, const int32_t* __restrict__ tokens,
                                         uint8_t* __restrict__ member) {
  const int m = blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= B * n) return;
  const int b = m / n, i = m - b * n;
  if (parent[i] < 0) {
    member[m] = 1;
    return;
  }
  double terms[MAX_PATH];
  int d = 0;
  for (int a = i; parent[a] >= 0 && d < MAX_PATH; a = parent[a]) {
    const int prow = b * P + parent_slot[parent[a]];
    terms[d++] = __dsub_rn((double)early[(size_t)prow * V + tokens[b * n + a]], early_stats[2 * prow]);
  }
  double lp = 0.0;
  for (int k = d - 1; k >= 0; --k) lp = __dadd_rn(lp, terms[k]);
  member[m] = lp >= log_tau ? 1 : 0;
}

}  // namespace propd

using namespace propd;

extern "C" {

int propd_row_lse(int R, const int32_t* rows_dev, int V, int ld, const float* logits, const int32_t* idx,
                  double temp, double* stats, void* stream) {
  if (R == 0) return 0;
  PROPD_REQUIRE(temp > 0.0, "row_lse: temperature must be positive");
  row_lse_kernel<<<R, 256, 0, as_stream(stream)>>>(V, ld, logits, idx, temp, stats, rows_dev);
  return check_launch("row_lse");
}

int propd_early_prob_member(int B, int n, int P, int V, double log_tau, const float* early_logits,
                            const double* early_stats, const int32_t* parent, const int32_t* parent_slot,
                            const int32_t* tokens, uint8_t* member, void* stream) {
  if (B * n == 0) return 0;
  early_prob_member_kernel<<<(B * n + 127) / 128, 128, 0, as_stream(stream)>>>(
      B, n, P, V, log_tau, early_logits, early_stats, parent, parent_slot, tokens, member);
  return check_launch("early_prob_member");
}

}  // extern "C"
