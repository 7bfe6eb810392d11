// K3: cumulant recursion over packed blocks (bc/cumulants.py:53-136).
//
//   C_m[key][o] = ((M_m[key][o] - B_2) - B_3) - ...,
//   B_sigma     = sum over min-2 partitions zeta (bc/partitions.py:63-98 order)
//                 of prod_{part in zeta} C_|part|[key|part][o|part]
//
// key|part is sorted because key is sorted and parts list modes ascending, so
// every factor is an element of a stored lower-order block (bc/cumulants.py:
// 9-12); its block index is precomputed on the host (Plan::sub_rank).  One CTA
// per output block; the block's slot offsets live in shared memory, lower
// orders are read through L1/L2 (they total <= a few % of M_m).  The product
// and sums are evaluated in the reference's order with explicit round-to-
// nearest intrinsics (no FMA contraction), i.e. the same float operations as
// the reference's einsum loop.
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.h"

namespace bcg {

// SMEM_SLOTS: the block's slot offsets staged in shared memory (nslots <=
// 25600, i.e. m <= 9); otherwise (m = 10..12: up to 2.5e6 slots per block)
// each factor's lower-block offset is looked up in the plan tables directly
template <bool SMEM_SLOTS>
__global__ void __launch_bounds__(256) k_recursion(RecursionArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  int64_t *slot_base = reinterpret_cast<int64_t *>(smem_raw);  // nslots
  __shared__ int edges[16];
  const int m = a.m;
  const int64_t k = a.klist ? (int64_t)a.klist[blockIdx.x] : a.k0 + blockIdx.x;
  const int tid = threadIdx.x;
  const int32_t *key = a.keys + k * m;
  if (tid < m) {
    const int64_t j = key[tid];
    const int64_t hi = j * a.b < a.n ? j * a.b : a.n;
    edges[tid] = (int)(hi - (j - 1) * a.b);
  }
  // slot s -> offset of its lower block (the slot's order = popcount(mask))
  if constexpr (SMEM_SLOTS) {
    int s = 0;
    for (int p = 0; p < a.p_end; ++p) {
      for (int i = 0; i < 8; ++i) {
        const int mask = a.part_mask[p * 8 + i];
        if (!mask) continue;
        if (s % blockDim.x == tid) {
          const int ord = __popc(mask);
          slot_base[s] = a.lower_offs[ord][a.sub_rank[k * a.nslots + s]];
        }
        ++s;
      }
    }
  }
  __syncthreads();
  int64_t E = 1;
  for (int q = 0; q < m; ++q) E *= edges[q];
  double *blk = a.mk + a.offs[k];  // (boff below)
  // first slot of p_begin
  int slot0 = 0;
  for (int p = 0; p < a.p_begin; ++p)
    for (int i = 0; i < 8; ++i) slot0 += a.part_mask[p * 8 + i] != 0;

  const int64_t boff = a.offs[k];
  for (int64_t e = tid; e < E; e += blockDim.x) {
    if (boff + e < a.e0 || boff + e >= a.e1) continue;  // outside this caller's element span
    int o[16];
    int64_t rem = e;
    for (int q = m - 1; q >= 0; --q) {
      o[q] = (int)(rem % edges[q]);
      rem /= edges[q];
    }
    double res = a.mode == 0 ? blk[e] : 0.0;
    int s = slot0;
    for (int sigma = a.sigma_lo; sigma <= a.sigma_hi; ++sigma) {
      const int pb = a.sigma_first[sigma], pe = a.sigma_first[sigma + 1];
      double bsum = 0.0;
      for (int p = pb; p < pe; ++p) {
        double prod = 1.0;
        for (int i = 0; i < sigma; ++i, ++s) {
          int mask = a.part_mask[p * 8 + i];
          const int ord = __popc(mask);
          int64_t lin = 0;
          while (mask) {
            const int q = __ffs(mask) - 1;
            mask &= mask - 1;
            lin = lin * edges[q] + o[q];
          }
          int64_t base;
          if constexpr (SMEM_SLOTS) {
            base = slot_base[s];
          } else {
            base = a.lower_offs[ord][a.sub_rank[k * a.nslots + s]];
          }
          const double v = __ldg(a.lower[ord] + base + lin);
          prod = i == 0 ? v : __dmul_rn(prod, v);
        }
        bsum = __dadd_rn(bsum, prod);
      }
      res = a.mode == 0 ? __dsub_rn(res, bsum) : bsum;
    }
    blk[e] = res;
  }
}

cudaError_t launch_recursion(const RecursionArgs &args, cudaStream_t stream) {
  if (args.K <= 0) return cudaSuccess;
  if (args.k1 <= args.k0) return cudaSuccess;
  const size_t smem = (size_t)args.nslots * sizeof(int64_t);
  if (smem <= 200 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(k_recursion<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k_recursion<true><<<(unsigned)(args.k1 - args.k0), 256, smem, stream>>>(args);
  } else {
    k_recursion<false><<<(unsigned)(args.k1 - args.k0), 256, 0, stream>>>(args);
  }
  g_launches++;
  return cudaGetLastError();
}

}  // namespace bcg
