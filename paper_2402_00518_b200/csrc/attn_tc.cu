// attn_tc.cu -- causal GQA flash-attention forward on the 5th-generation
// tensor cores (tcgen05 + TMEM + TMA) for the Layer exit and the backbone
// (Llama-2 attention; Layer exit P:210).
//
// One CTA per (128-query tile, query head, sequence); head dim 128.
//   warp 0      TMA producer of Q and K_j (128 keys, 2-stage ring; a stage is
//               released as soon as its QK MMA completes)
//   warp 3      TMA producer of V_j (3-stage ring, released after its PV MMA)
//   warp 1      MMA issuer (one thread): S_j = Q K_j^T into one of two TMEM
//               S buffers, then O (+)= P_j V_j into the TMEM O accumulator
//   warps 4..7  softmax, one thread per query row (= TMEM lane): reads S_j,
//               keeps the running max m and sum l in registers, writes
//               P_j = 2^(s log2e/sqrt(d) - m) as bf16 into shared memory in the
//               SWIZZLE_128B K-major layout the MMA reads as its A operand;
//               finally O / l -> bf16 and lse2 = m + log2 l.
// The MMA of S_{j+1} runs while the softmax threads work on S_j.  O lives in
// TMEM for the whole key loop; it is rescaled (TMEM ld/st) only when a row's
// max grows by more than 2^8 over the reference max used so far -- with a
// fixed reference m, O / l is exact whatever m is, and P stays <= 2^8 in bf16.
// Causal mask on the diagonal tile only (key > query); tiles past a short
// sequence's end are excluded by the same mask, so T need only be a multiple
// of 64.  Heavy (late) query tiles are scheduled first.
#include <cmath>
#include "internal.cuh"

namespace ee {

namespace {
constexpr int FA_BM = 128;                        // queries per CTA
constexpr int FA_BN = 128;                        // keys per tile
constexpr int FA_D = 128;                         // head dim
constexpr int FA_TILE = FA_BM * FA_D * 2;         // 32 KB: two 16 KB SW128 atoms
constexpr int FA_ATOM = 16384;
constexpr int FA_KST = 2;                         // K ring stages
constexpr int FA_VST = 3;                         // V ring stages
constexpr int FA_SMEM = 1024 + FA_TILE * (2 + FA_KST + FA_VST) + 256;
constexpr float FA_RESCALE = 8.0f;                // log2 headroom before O is rescaled
#ifndef EE_FA_P_TMEM
#define EE_FA_P_TMEM 1                            // P as a TMEM A operand (else swizzled smem)
#endif
}  // namespace

__global__ void __launch_bounds__(256, 1)
    attn_fwd_tc_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                       const __grid_constant__ CUtensorMap tmV, __nv_bfloat16* __restrict__ o,
                       float* __restrict__ lse2, int T, int Hq, int Hkv, float scale_log2) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint8_t* sQ = smem;
  uint8_t* sK = sQ + FA_TILE;
  uint8_t* sV = sK + FA_KST * FA_TILE;
  uint8_t* sP = sV + FA_VST * FA_TILE;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sP + FA_TILE);
  uint64_t* q_full = bars;
  uint64_t* k_full = bars + 1;               // [KST]
  uint64_t* k_empty = k_full + FA_KST;       // [KST]
  uint64_t* v_full = k_empty + FA_KST;       // [VST]
  uint64_t* v_empty = v_full + FA_VST;       // [VST]
  uint64_t* s_full = v_empty + FA_VST;       // [2]
  uint64_t* p_full = s_full + 2;
  uint64_t* o_done = p_full + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_done + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nqt = (T + FA_BM - 1) / FA_BM;
  const int qt = nqt - 1 - (int)blockIdx.x;  // longest causal rows first
  const int hq = blockIdx.y, b = blockIdx.z;
  const int hk = hq / (Hq / Hkv);
  const int q_row0 = b * T + qt * FA_BM;
  const int n_kt = qt + 1;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmQ);
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
    mbar_init(q_full, 1);
    for (int s = 0; s < FA_KST; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&k_empty[s], 1);
    }
    for (int s = 0; s < FA_VST; ++s) {
      mbar_init(&v_full[s], 1);
      mbar_init(&v_empty[s], 1);
    }
    mbar_init(&s_full[0], 1);
    mbar_init(&s_full[1], 1);
    mbar_init(p_full, 128);
    mbar_init(o_done, 1);
    fence_barrier_init();
  }
  if (warp == 2) {
    tmem_alloc(tmem_slot, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const uint32_t tS0 = tmem_base, tO = tmem_base + 2 * FA_BN;

  if (warp == 0) {
    // ---------------------------------------------------------------- TMA: Q, K
    if (lane == 0) {
      tma_load_2d(sQ, &tmQ, q_full, hq * FA_D, q_row0);
      tma_load_2d(sQ + FA_ATOM, &tmQ, q_full, hq * FA_D + 64, q_row0);
      mbar_arrive_expect_tx(q_full, FA_TILE);
      for (int j = 0; j < n_kt; ++j) {
        const int s = j % FA_KST;
        mbar_wait(&k_empty[s], ((j / FA_KST) & 1) ^ 1);
        uint8_t* k = sK + s * FA_TILE;
        const int k_row0 = b * T + j * FA_BN;
        tma_load_2d(k, &tmK, &k_full[s], hk * FA_D, k_row0);
        tma_load_2d(k + FA_ATOM, &tmK, &k_full[s], hk * FA_D + 64, k_row0);
        mbar_arrive_expect_tx(&k_full[s], FA_TILE);
      }
    }
  } else if (warp == 3) {
    // ---------------------------------------------------------------- TMA: V
    if (lane == 0) {
      for (int j = 0; j < n_kt; ++j) {
        const int s = j % FA_VST;
        mbar_wait(&v_empty[s], ((j / FA_VST) & 1) ^ 1);
        uint8_t* v = sV + s * FA_TILE;
        const int k_row0 = b * T + j * FA_BN;
        tma_load_2d(v, &tmV, &v_full[s], hk * FA_D, k_row0);
        tma_load_2d(v + FA_ATOM, &tmV, &v_full[s], hk * FA_D + 64, k_row0);
        mbar_arrive_expect_tx(&v_full[s], FA_TILE);
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc_qk = make_idesc_bf16(FA_BM, FA_BN, false, false);
      constexpr uint32_t idesc_pv = make_idesc_bf16(FA_BM, FA_D, false, true);
      const uint32_t aq = smem_u32(sQ), ap = smem_u32(sP);
      mbar_wait(q_full, 0);
      auto issue_qk = [&](int j) {
        const int s = j % FA_KST;
        mbar_wait(&k_full[s], (j / FA_KST) & 1);
        tc_fence_after();
        const uint32_t bk = smem_u32(sK + s * FA_TILE);
#pragma unroll
        for (int k = 0; k < FA_D / 16; ++k) {  // K-major A and B: 4 k-steps per 64-wide atom
          const uint32_t off = (k >> 2) * FA_ATOM + (k & 3) * 32;
          tc_mma_f16(tS0 + (j & 1) * FA_BN, make_sdesc(aq + off, 16, 1024),
                     make_sdesc(bk + off, 16, 1024), idesc_qk, k != 0 ? 1u : 0u);
        }
        tc_commit(&s_full[j & 1]);
        tc_commit(&k_empty[s]);  // K_j is free once S_j is computed
      };
      issue_qk(0);
      for (int j = 0; j < n_kt; ++j) {
        if (j + 1 < n_kt) issue_qk(j + 1);
        const int sv = j % FA_VST;
        mbar_wait(&v_full[sv], (j / FA_VST) & 1);
        mbar_wait(p_full, j & 1);
        tc_fence_after();
        const uint32_t bv = smem_u32(sV + sv * FA_TILE);
#pragma unroll
        for (int k = 0; k < FA_BN / 16; ++k) {  // A = P, B = V (MN-major: keys x d)
#if EE_FA_P_TMEM
          tc_mma_f16_ts(tO, tS0 + (j & 1) * FA_BN + k * 8, make_sdesc(bv + k * 2048, FA_ATOM, 1024),
                        idesc_pv, (j | k) != 0 ? 1u : 0u);
#else
          const uint32_t offa = (k >> 2) * FA_ATOM + (k & 3) * 32;
          tc_mma_f16(tO, make_sdesc(ap + offa, 16, 1024), make_sdesc(bv + k * 2048, FA_ATOM, 1024),
                     idesc_pv, (j | k) != 0 ? 1u : 0u);
#endif
        }
        tc_commit(o_done);
        tc_commit(&v_empty[sv]);
      }
    }
  } else if (warp >= 4) {
    // ---------------------------------------------------------------- softmax
    const int ew = warp - 4;
    const int r = ew * 32 + lane;  // query row within the tile = TMEM lane
    const uint32_t lane_off = static_cast<uint32_t>(ew * 32) << 16;
    float m_ref = -INFINITY, l = 0.f;
    const uint32_t prow = smem_u32(sP) + r * 128;
    for (int j = 0; j < n_kt; ++j) {
      mbar_wait(&s_full[j & 1], (j >> 1) & 1);
      tc_fence_after();
      // all four 32-column TMEM loads in flight, one wait (outputs are only
      // read after tcgen05.wait::ld)
      uint32_t sr[FA_BN];
      const uint32_t ts = tS0 + (j & 1) * FA_BN + lane_off;
      tmem_ld_32x32b_x32(ts, *reinterpret_cast<uint32_t(*)[32]>(sr));
      tmem_ld_32x32b_x32(ts + 32, *reinterpret_cast<uint32_t(*)[32]>(sr + 32));
      tmem_ld_32x32b_x32(ts + 64, *reinterpret_cast<uint32_t(*)[32]>(sr + 64));
      tmem_ld_32x32b_x32(ts + 96, *reinterpret_cast<uint32_t(*)[32]>(sr + 96));
      tmem_ld_wait();
      float sv[FA_BN];
#pragma unroll
      for (int i = 0; i < FA_BN; ++i) sv[i] = __uint_as_float(sr[i]);
      if (j == qt) {  // diagonal tile: key column > query row is in the future
#pragma unroll
        for (int i = 0; i < FA_BN; ++i)
          if (i > r) sv[i] = -INFINITY;
      }
      // row max with 8 independent chains (latency, not throughput, bound)
      float m8[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) m8[e] = sv[e];
#pragma unroll
      for (int i = 8; i < FA_BN; i += 8)
#pragma unroll
        for (int e = 0; e < 8; ++e) m8[e] = fmaxf(m8[e], sv[i + e]);
      float mx = fmaxf(fmaxf(fmaxf(m8[0], m8[1]), fmaxf(m8[2], m8[3])),
                       fmaxf(fmaxf(m8[4], m8[5]), fmaxf(m8[6], m8[7])));
      mx *= scale_log2;
      // reference max: set on the first tile, raised only past the 2^8 headroom
      // (warp-uniform, since the O rescale below is a warp-collective TMEM op)
      bool grow = false;
      float alpha = 1.0f;
      if (j == 0) {
        m_ref = mx;
      } else {
        grow = mx > m_ref + FA_RESCALE;
        if (grow) {
          alpha = ex2_approx(m_ref - mx);
          l *= alpha;
          m_ref = mx;
        }
      }
      const bool any_grow = __any_sync(0xffffffffu, grow);
      // P = 2^(s * scale - m_ref): computed BEFORE waiting for PV_{j-1}, so the
      // exp2 work overlaps the tensor core (one FFMA + one MUFU per element)
      uint32_t pk[FA_BN / 2];
      float l8[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int i = 0; i < FA_BN / 2; ++i) {
        const float p0 = ex2_approx(fmaf(sv[2 * i], scale_log2, -m_ref));
        const float p1 = ex2_approx(fmaf(sv[2 * i + 1], scale_log2, -m_ref));
        l8[(2 * i) & 7] += p0;
        l8[(2 * i + 1) & 7] += p1;
        pk[i] = pack_bf16(p0, p1);
      }
      l += ((l8[0] + l8[1]) + (l8[2] + l8[3])) + ((l8[4] + l8[5]) + (l8[6] + l8[7]));
      if (j > 0) {
        mbar_wait(o_done, (j - 1) & 1);  // PV_{j-1} done: O stable, P buffer free
        tc_fence_after();
      }
      if (any_grow) {
#pragma unroll 1
        for (int c = 0; c < FA_D / 32; ++c) {
          uint32_t v[32];
          tmem_ld_32x32b_x32(tO + lane_off + c * 32, v);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = __float_as_uint(__uint_as_float(v[i]) * alpha);
          tmem_st_32x32b_x32(tO + lane_off + c * 32, v);
        }
        tmem_st_wait();
      }
#if EE_FA_P_TMEM
      // P -> TMEM over the first 64 columns of S_j's own buffer (S_j is in
      // registers now; S_{j+2} reuses the buffer only after PV_j, in issue order)
      tmem_st_32x32b_x32(ts, *reinterpret_cast<const uint32_t(*)[32]>(pk));
      tmem_st_32x32b_x32(ts + 32, *reinterpret_cast<const uint32_t(*)[32]>(pk + 32));
      tmem_st_wait();
#else
      // P -> smem, K-major SWIZZLE_128B: 16-byte chunk cc of row r sits at
      // chunk (cc ^ (r & 7)) of the row's 128-byte line
#pragma unroll
      for (int c8 = 0; c8 < FA_BN / 8; ++c8) {
        const int cc = c8 & 7;
        st_shared_v4(prow + (c8 >> 3) * FA_ATOM + ((cc ^ (r & 7)) << 4), pk[4 * c8],
                     pk[4 * c8 + 1], pk[4 * c8 + 2], pk[4 * c8 + 3]);
      }
      fence_proxy_async_smem();
#endif
      tc_fence_before();
      mbar_arrive(p_full);
    }
    // ---------------------------------------------------------------- epilogue
    mbar_wait(o_done, (n_kt - 1) & 1);
    tc_fence_after();
    const int pos = qt * FA_BM + r;
    const bool ok = pos < T;
    const float inv_l = 1.0f / l;
    __nv_bfloat16* orow = o + (long long)(q_row0 + r) * Hq * FA_D + hq * FA_D;
#pragma unroll 1
    for (int c = 0; c < FA_D / 32; ++c) {
      uint32_t v[32];
      tmem_ld_32x32b_x32(tO + lane_off + c * 32, v);
      tmem_ld_wait();
      if (ok) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          uint32_t w[8];
#pragma unroll
          for (int q = 0; q < 8; ++q)
            w[q] = pack_bf16(__uint_as_float(v[h * 16 + 2 * q]) * inv_l,
                             __uint_as_float(v[h * 16 + 2 * q + 1]) * inv_l);
          __nv_bfloat16* dst = orow + c * 32 + h * 16;
          if (aligned32(dst)) {
            st_global_v8(dst, w);
          } else {
            *reinterpret_cast<uint4*>(dst) = make_uint4(w[0], w[1], w[2], w[3]);
            *reinterpret_cast<uint4*>(dst + 8) = make_uint4(w[4], w[5], w[6], w[7]);
          }
        }
      }
    }
    if (ok && lse2 != nullptr) lse2[(long long)(q_row0 + r) * Hq + hq] = m_ref + log2f(l);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem_base, 512);
  }
}

cudaError_t launch_attn_fwd_tc(const __nv_bfloat16* q, const __nv_bfloat16* k,
                               const __nv_bfloat16* v, __nv_bfloat16* o, long long N, int T,
                               int Hq, int Hkv, float* lse2, cudaStream_t s) {
  if (N == 0) return cudaSuccess;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(attn_fwd_tc_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, FA_SMEM);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  CUtensorMap tq, tk, tv;
  const Mat Q{q, N, (long long)Hq * FA_D, (long long)Hq * FA_D};
  const Mat K{k, N, (long long)Hkv * FA_D, (long long)Hkv * FA_D};
  const Mat V{v, N, (long long)Hkv * FA_D, (long long)Hkv * FA_D};
  if (!make_tmap(&tq, Q, 64, FA_BM) || !make_tmap(&tk, K, 64, FA_BN) || !make_tmap(&tv, V, 64, FA_BN))
    return cudaErrorInvalidValue;
  const float scale_log2 = 1.4426950408889634f / sqrtf((float)FA_D);
  dim3 grid((T + FA_BM - 1) / FA_BM, Hq, (unsigned)(N / T));
  attn_fwd_tc_kernel<<<grid, 256, FA_SMEM, s>>>(tq, tk, tv, o, lse2, T, Hq, Hkv, scale_log2);
  return cudaGetLastError();
}

// ============================================================================
// Forward, two query tiles per CTA (tiles 2p and 2p + 1 of one head): the
// FA4-style ping-pong.  The one-tile kernel above is MUFU-bound by
// construction -- 128 x 128 exp2 per key tile at 16/clk/SM take as long as the
// tile's QK^T + PV MMAs, and PV_j must wait for softmax_j -- so the tensor core
// idles about a third of the time.  Here two softmax warpgroups (warps 4-7:
// tile A, warps 8-11: tile B) alternate with the MMA issuer:
//   S_A(0) S_B(0) | PV_A(j) S_A(j+1) PV_B(j) S_B(j+1) | ...
// so softmax A(j+1) runs under PV_B(j) + S_B(j+1) and vice versa.  K_j and V_j
// are loaded once for both tiles.  TMEM: S_A | S_B | O_A | O_B (4 x 128
// columns); P_X(j) is written as bf16 over the first 64 columns of S_X (the
// TMEM A operand of PV_X(j)); S_X(j+1) is issued after PV_X(j), so the tensor
// pipe's issue order protects P.  setmaxnreg moves registers from the
// producer / MMA warpgroup to the softmax warpgroups, which hold a whole S row.
// Same arithmetic, rounding points and outputs as the one-tile kernel
// (bitwise: the per-row operations and their order are unchanged).
// 2^x on the FMA pipe (FA4's trick to take part of the exp2 load off the
// 16/clk/SM MUFU unit): x = n + f with n = rint(x) from the 1.5 * 2^23 magic
// constant, 2^f by a degree-3 minimax polynomial on [-0.5, 0.5] (max relative
// error 7.5e-5, below the bf16 rounding of P, 2^-9), and 2^n added to the
// exponent field with one integer multiply-add (the magic constant has zero
// low 22 bits, so bits(t) << 23 = n << 23 mod 2^32).  x >= -125 (clamped):
// only used on tiles without masked (-inf) entries, where x >= -(2^8 + ...).
__device__ __forceinline__ float ex2_poly(float x) {
  x = fmaxf(x, -125.0f);
  const float t = x + 12582912.0f;
  const float f = x - (t - 12582912.0f);
  const float p = fmaf(fmaf(fmaf(0.0551716685f, f, 0.2426111549f), f, 0.6932609677f), f,
                       0.9999280572f);
  return __int_as_float(__float_as_int(t) * (1 << 23) + __float_as_int(p));
}

// Blackwell packed / 3-input fp32 ops (FMNMX3, FFMA2, FADD2): the two-tile
// softmax is issue-bound, and these halve its max / scale / sum instructions
// with the same per-element IEEE roundings as fmaxf / fmaf / fadd.
__device__ __forceinline__ float fmax3f(float a, float b, float c) {
  float d;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}
__device__ __forceinline__ unsigned long long f2pack(float a, float b) {
  unsigned long long v;
  asm("mov.b64 %0, {%1, %2};" : "=l"(v) : "f"(a), "f"(b));
  return v;
}
__device__ __forceinline__ void f2unpack(unsigned long long v, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
__device__ __forceinline__ unsigned long long ffma2(unsigned long long a, unsigned long long b,
                                                    unsigned long long c) {
  unsigned long long d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ unsigned long long fadd2(unsigned long long a, unsigned long long b) {
  unsigned long long d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ unsigned long long fmul2(unsigned long long a, unsigned long long b) {
  unsigned long long d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}

namespace {
constexpr int FA2_KST = 2, FA2_VST = 2;
constexpr int FA2_SMEM = 1024 + FA_TILE * (2 + FA2_KST + FA2_VST) + 512;
}  // namespace

template <int POLY>
__global__ void __launch_bounds__(384, 1)
    attn_fwd_tc2_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                        const __grid_constant__ CUtensorMap tmV, __nv_bfloat16* __restrict__ o,
                        float* __restrict__ lse2, int T, int Hq, int Hkv, float scale_log2) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint8_t* sQ = smem;                        // [2] tiles A, B
  uint8_t* sK = sQ + 2 * FA_TILE;
  uint8_t* sV = sK + FA2_KST * FA_TILE;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sV + FA2_VST * FA_TILE);
  uint64_t* q_full = bars;                   // [2]
  uint64_t* k_full = bars + 2;               // [KST]
  uint64_t* k_empty = k_full + FA2_KST;      // [KST]
  uint64_t* v_full = k_empty + FA2_KST;      // [VST]
  uint64_t* v_empty = v_full + FA2_VST;      // [VST]
  uint64_t* s_full = v_empty + FA2_VST;      // [2] per tile
  uint64_t* p_full = s_full + 2;             // [2] per tile
  uint64_t* o_done = p_full + 2;             // [2] per tile
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_done + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nqt = (T + FA_BM - 1) / FA_BM;
  const int npair = (nqt + 1) / 2;
  const int pr = npair - 1 - (int)blockIdx.x;  // longest causal rows first
  const int qtA = 2 * pr, qtB = 2 * pr + 1;
  const bool hasB = qtB < nqt;
  const int n_ktA = qtA + 1, n_kt = hasB ? qtB + 1 : n_ktA;
  const int hq = blockIdx.y, b = blockIdx.z;
  const int hk = hq / (Hq / Hkv);

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmQ);
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
    for (int x = 0; x < 2; ++x) {
      mbar_init(&q_full[x], 1);
      mbar_init(&s_full[x], 1);
      mbar_init(&p_full[x], 128);
      mbar_init(&o_done[x], 1);
    }
    for (int s = 0; s < FA2_KST; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&k_empty[s], 1);
    }
    for (int s = 0; s < FA2_VST; ++s) {
      mbar_init(&v_full[s], 1);
      mbar_init(&v_empty[s], 1);
    }
    fence_barrier_init();
  }
  if (warp == 2) {
    tmem_alloc(tmem_slot, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  // registers: 56 for the producer / MMA warpgroup, 224 for the two softmax
  // warpgroups (4 x 32 x 56 + 8 x 32 x 224 <= 64 K), which hold a whole
  // 128-column S row each
  if (warp == 0) {
    // ---------------------------------------------------------------- TMA: Q_A, Q_B, K
    asm volatile("setmaxnreg.dec.sync.aligned.u32 56;\n" ::: "memory");
    if (lane == 0) {
      for (int x = 0; x < (hasB ? 2 : 1); ++x) {
        const int row0 = b * T + (qtA + x) * FA_BM;
        tma_load_2d(sQ + x * FA_TILE, &tmQ, &q_full[x], hq * FA_D, row0);
        tma_load_2d(sQ + x * FA_TILE + FA_ATOM, &tmQ, &q_full[x], hq * FA_D + 64, row0);
        mbar_arrive_expect_tx(&q_full[x], FA_TILE);
      }
      for (int j = 0; j < n_kt; ++j) {
        const int s = j % FA2_KST;
        mbar_wait(&k_empty[s], ((j / FA2_KST) & 1) ^ 1);
        uint8_t* k = sK + s * FA_TILE;
        const int k_row0 = b * T + j * FA_BN;
        tma_load_2d(k, &tmK, &k_full[s], hk * FA_D, k_row0);
        tma_load_2d(k + FA_ATOM, &tmK, &k_full[s], hk * FA_D + 64, k_row0);
        mbar_arrive_expect_tx(&k_full[s], FA_TILE);
      }
    }
  } else if (warp == 3) {
    // ---------------------------------------------------------------- TMA: V
    asm volatile("setmaxnreg.dec.sync.aligned.u32 56;\n" ::: "memory");
    if (lane == 0) {
      for (int j = 0; j < n_kt; ++j) {
        const int s = j % FA2_VST;
        mbar_wait(&v_empty[s], ((j / FA2_VST) & 1) ^ 1);
        uint8_t* v = sV + s * FA_TILE;
        const int k_row0 = b * T + j * FA_BN;
        tma_load_2d(v, &tmV, &v_full[s], hk * FA_D, k_row0);
        tma_load_2d(v + FA_ATOM, &tmV, &v_full[s], hk * FA_D + 64, k_row0);
        mbar_arrive_expect_tx(&v_full[s], FA_TILE);
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer
    // (the whole warp runs the loop; elect.sync issues: ptx.cuh tc_mma_f16_w)
    asm volatile("setmaxnreg.dec.sync.aligned.u32 56;\n" ::: "memory");
    {
      constexpr uint32_t idesc_qk = make_idesc_bf16(FA_BM, FA_BN, false, false);
      constexpr uint32_t idesc_pv = make_idesc_bf16(FA_BM, FA_D, false, true);
      int k_ready = -1, v_ready = -1;
      auto ensure_k = [&](int j) {
        if (k_ready < j) {
          mbar_wait(&k_full[j % FA2_KST], (j / FA2_KST) & 1);
          tc_fence_after();
          k_ready = j;
        }
      };
      auto ensure_v = [&](int j) {
        if (v_ready < j) {
          mbar_wait(&v_full[j % FA2_VST], (j / FA2_VST) & 1);
          tc_fence_after();
          v_ready = j;
        }
      };
      auto issue_s = [&](int x, int j) {  // S_x(j) = Q_x K_j^T
        ensure_k(j);
        const uint32_t aq = smem_u32(sQ + x * FA_TILE);
        const uint32_t bk = smem_u32(sK + (j % FA2_KST) * FA_TILE);
#pragma unroll
        for (int k = 0; k < FA_D / 16; ++k) {
          const uint32_t off = (k >> 2) * FA_ATOM + (k & 3) * 32;
          tc_mma_f16_w(tmem_base + x * FA_BN, make_sdesc(aq + off, 16, 1024),
                     make_sdesc(bk + off, 16, 1024), idesc_qk, k != 0 ? 1u : 0u);
        }
        tc_commit_w(&s_full[x]);
      };
      auto issue_pv = [&](int x, int j) {  // O_x (+)= P_x(j) V_j, P in TMEM
        ensure_v(j);
        mbar_wait(&p_full[x], j & 1);
        tc_fence_after();
        const uint32_t bv = smem_u32(sV + (j % FA2_VST) * FA_TILE);
        const uint32_t tO = tmem_base + 2 * FA_BN + x * FA_D;
#pragma unroll
        for (int k = 0; k < FA_BN / 16; ++k)
          tc_mma_f16_ts_w(tO, tmem_base + x * FA_BN + k * 8,
                        make_sdesc(bv + k * 2048, FA_ATOM, 1024), idesc_pv,
                        (j | k) != 0 ? 1u : 0u);
        tc_commit_w(&o_done[x]);
      };
      mbar_wait(&q_full[0], 0);
      if (hasB) mbar_wait(&q_full[1], 0);
      issue_s(0, 0);
      if (hasB) issue_s(1, 0);
      tc_commit_w(&k_empty[0]);
      for (int j = 0; j < n_kt; ++j) {
        if (j < n_ktA) {
          issue_pv(0, j);
          if (!hasB) tc_commit_w(&v_empty[j % FA2_VST]);
          if (j + 1 < n_ktA) {
            issue_s(0, j + 1);
            if (!hasB) tc_commit_w(&k_empty[(j + 1) % FA2_KST]);
          }
        }
        if (hasB) {
          issue_pv(1, j);
          tc_commit_w(&v_empty[j % FA2_VST]);
          if (j + 1 < n_kt) {
            issue_s(1, j + 1);
            tc_commit_w(&k_empty[(j + 1) % FA2_KST]);
          }
        }
      }
    }
  } else if (warp == 2) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 56;\n" ::: "memory");
  } else {
    // ---------------------------------------------------------------- softmax (tile x)
    asm volatile("setmaxnreg.inc.sync.aligned.u32 224;\n" ::: "memory");
    const int x = (warp - 4) >> 2;
    if (x == 1 && !hasB) goto done;
    {
      const int qt = qtA + x, nk = qt + 1;
      const int ew = (warp - 4) & 3;
      const int r = ew * 32 + lane;  // query row within the tile = TMEM lane
      const uint32_t lane_off = static_cast<uint32_t>(ew * 32) << 16;
      const uint32_t ts = tmem_base + x * FA_BN + lane_off;
      const uint32_t tO = tmem_base + 2 * FA_BN + x * FA_D + lane_off;
      float m_ref = -INFINITY, l = 0.f;
      for (int j = 0; j < nk; ++j) {
        mbar_wait(&s_full[x], j & 1);
        tc_fence_after();
        const bool diag = j == qt;
        // the whole 128-column row in registers (setmaxnreg above): four TMEM
        // loads in flight, one wait; the causal mask only on the diagonal tile
        uint32_t sr[FA_BN];
        tmem_ld_32x32b_x32(ts, *reinterpret_cast<uint32_t(*)[32]>(sr));
        tmem_ld_32x32b_x32(ts + 32, *reinterpret_cast<uint32_t(*)[32]>(sr + 32));
        tmem_ld_32x32b_x32(ts + 64, *reinterpret_cast<uint32_t(*)[32]>(sr + 64));
        tmem_ld_32x32b_x32(ts + 96, *reinterpret_cast<uint32_t(*)[32]>(sr + 96));
        tmem_ld_wait();
        float sv[FA_BN];
#pragma unroll
        for (int i = 0; i < FA_BN; ++i) sv[i] = __uint_as_float(sr[i]);
        if (diag) {
#pragma unroll
          for (int i = 0; i < FA_BN; ++i)
            if (i > r) sv[i] = -INFINITY;
        }
        // row max: 8 independent chains of 3-input max (exact, so the same
        // value as the one-tile kernel's 2-input chains)
        float m8[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) m8[e] = sv[e];
#pragma unroll
        for (int i = 8; i + 16 <= FA_BN; i += 16)
#pragma unroll
          for (int e = 0; e < 8; ++e) m8[e] = fmax3f(m8[e], sv[i + e], sv[i + 8 + e]);
#pragma unroll
        for (int e = 0; e < 8; ++e) m8[e] = fmaxf(m8[e], sv[FA_BN - 8 + e]);
        float mx = fmaxf(fmaxf(fmaxf(m8[0], m8[1]), fmaxf(m8[2], m8[3])),
                         fmaxf(fmaxf(m8[4], m8[5]), fmaxf(m8[6], m8[7])));
        mx *= scale_log2;
        bool grow = false;
        float alpha = 1.0f;
        if (j == 0) {
          m_ref = mx;
        } else {
          grow = mx > m_ref + FA_RESCALE;
          if (grow) {
            alpha = ex2_approx(m_ref - mx);
            l *= alpha;
            m_ref = mx;
          }
        }
        const bool any_grow = __any_sync(0xffffffffu, grow);
        uint32_t pk[FA_BN / 2];
        float l8[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        if (POLY == 0) {  // packed: x = s * scale - m (FFMA2), l chains (FADD2)
          const unsigned long long sc2 = f2pack(scale_log2, scale_log2);
          const unsigned long long nm2 = f2pack(-m_ref, -m_ref);
          unsigned long long l2[4] = {0ull, 0ull, 0ull, 0ull};
#pragma unroll
          for (int i = 0; i < FA_BN / 2; ++i) {
            float x0, x1;
            f2unpack(ffma2(f2pack(sv[2 * i], sv[2 * i + 1]), sc2, nm2), x0, x1);
            const float p0 = ex2_approx(x0), p1 = ex2_approx(x1);
            l2[i & 3] = fadd2(l2[i & 3], f2pack(p0, p1));   // chains (2i)&7, (2i+1)&7
            pk[i] = pack_bf16(p0, p1);
          }
#pragma unroll
          for (int c = 0; c < 4; ++c) f2unpack(l2[c], l8[2 * c], l8[2 * c + 1]);
        } else if (!diag) {  // every POLY-th pair of exp2 on the FMA pipe
#pragma unroll
          for (int i = 0; i < FA_BN / 2; ++i) {
            const bool poly = (i % (POLY > 0 ? POLY : 1)) == (POLY > 0 ? POLY : 1) - 1;
            const float x0 = fmaf(sv[2 * i], scale_log2, -m_ref);
            const float x1 = fmaf(sv[2 * i + 1], scale_log2, -m_ref);
            const float p0 = poly ? ex2_poly(x0) : ex2_approx(x0);
            const float p1 = poly ? ex2_poly(x1) : ex2_approx(x1);
            l8[(2 * i) & 7] += p0;
            l8[(2 * i + 1) & 7] += p1;
            pk[i] = pack_bf16(p0, p1);
          }
        } else {
#pragma unroll
          for (int i = 0; i < FA_BN / 2; ++i) {
            const float p0 = ex2_approx(fmaf(sv[2 * i], scale_log2, -m_ref));
            const float p1 = ex2_approx(fmaf(sv[2 * i + 1], scale_log2, -m_ref));
            l8[(2 * i) & 7] += p0;
            l8[(2 * i + 1) & 7] += p1;
            pk[i] = pack_bf16(p0, p1);
          }
        }
        // P over the first 64 columns of S_x (read into registers above)
        tmem_st_32x32b_x32(ts, *reinterpret_cast<const uint32_t(*)[32]>(pk));
        tmem_st_32x32b_x32(ts + 32, *reinterpret_cast<const uint32_t(*)[32]>(pk + 32));
        l += ((l8[0] + l8[1]) + (l8[2] + l8[3])) + ((l8[4] + l8[5]) + (l8[6] + l8[7]));
        if (j > 0) {
          mbar_wait(&o_done[x], (j - 1) & 1);  // PV_x(j-1) done (implied by s_full; explicit)
          tc_fence_after();
        }
        if (any_grow) {
#pragma unroll 1
          for (int c = 0; c < FA_D / 32; ++c) {
            uint32_t v[32];
            tmem_ld_32x32b_x32(tO + c * 32, v);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = __float_as_uint(__uint_as_float(v[i]) * alpha);
            tmem_st_32x32b_x32(tO + c * 32, v);
          }
        }
        tmem_st_wait();
        tc_fence_before();
        mbar_arrive(&p_full[x]);
      }
      // ---------------------------------------------------------------- epilogue
      mbar_wait(&o_done[x], (nk - 1) & 1);
      tc_fence_after();
      const int q_row0 = b * T + qt * FA_BM;
      const int pos = qt * FA_BM + r;
      const bool ok = pos < T;
      const float inv_l = 1.0f / l;
      __nv_bfloat16* orow = o + (long long)(q_row0 + r) * Hq * FA_D + hq * FA_D;
#pragma unroll 1
      for (int c = 0; c < FA_D / 32; ++c) {
        uint32_t v[32];
        tmem_ld_32x32b_x32(tO + c * 32, v);
        tmem_ld_wait();
        if (ok) {
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            uint32_t w[8];
#pragma unroll
            for (int q = 0; q < 8; ++q)
              w[q] = pack_bf16(__uint_as_float(v[h * 16 + 2 * q]) * inv_l,
                               __uint_as_float(v[h * 16 + 2 * q + 1]) * inv_l);
            __nv_bfloat16* dst = orow + c * 32 + h * 16;
            if (aligned32(dst)) {
              st_global_v8(dst, w);
            } else {
              *reinterpret_cast<uint4*>(dst) = make_uint4(w[0], w[1], w[2], w[3]);
              *reinterpret_cast<uint4*>(dst + 8) = make_uint4(w[4], w[5], w[6], w[7]);
            }
          }
        }
      }
      if (ok && lse2 != nullptr) lse2[(long long)(q_row0 + r) * Hq + hq] = m_ref + log2f(l);
    }
  }
done:
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem_base, 512);
  }
}

cudaError_t launch_attn_fwd_tc2(const __nv_bfloat16* q, const __nv_bfloat16* k,
                                const __nv_bfloat16* v, __nv_bfloat16* o, long long N, int T,
                                int Hq, int Hkv, float* lse2, cudaStream_t s) {
  if (N == 0) return cudaSuccess;
  // EE_ATTN_POLY = k: every k-th pair of exp2 of the off-diagonal tiles on the
  // FMA pipe (0 = all on MUFU: bitwise the one-tile kernel's outputs)
  static const int poly = [] {
    const char* e = getenv("EE_ATTN_POLY");
    return e ? atoi(e) : 0;
  }();
  auto kern = poly == 2 ? attn_fwd_tc2_kernel<2> : poly == 3 ? attn_fwd_tc2_kernel<3>
            : poly == 4 ? attn_fwd_tc2_kernel<4> : attn_fwd_tc2_kernel<0>;
  static bool attr[5] = {false, false, false, false, false};
  const int pi = (poly >= 2 && poly <= 4) ? poly : 0;
  if (!attr[pi]) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, FA2_SMEM);
    if (e != cudaSuccess) return e;
    attr[pi] = true;
  }
  CUtensorMap tq, tk, tv;
  const Mat Q{q, N, (long long)Hq * FA_D, (long long)Hq * FA_D};
  const Mat K{k, N, (long long)Hkv * FA_D, (long long)Hkv * FA_D};
  const Mat V{v, N, (long long)Hkv * FA_D, (long long)Hkv * FA_D};
  if (!make_tmap(&tq, Q, 64, FA_BM) || !make_tmap(&tk, K, 64, FA_BN) || !make_tmap(&tv, V, 64, FA_BN))
    return cudaErrorInvalidValue;
  const float scale_log2 = 1.4426950408889634f / sqrtf((float)FA_D);
  const int nqt = (T + FA_BM - 1) / FA_BM;
  dim3 grid((nqt + 1) / 2, Hq, (unsigned)(N / T));
  kern<<<grid, 384, FA2_SMEM, s>>>(tq, tk, tv, o, lse2, T, Hq, Hkv, scale_log2);
  return cudaGetLastError();
}

// ============================================================================
// Backward (FlashAttention-2 split, deterministic: no float atomics).  With
// lse2 from the forward and Dv = rowsum(dO * O) (attn_bwd_dot_kernel):
//   P = 2^(s S - lse2), dP = dO V^T, dS = P (dP - Dv),
//   dQ = c dS K, dK = c dS^T Q, dV = P^T dO   (c = 1/sqrt(d), s = c log2 e)
// and RoPE^T applied to dQ, dK in fp32 before their single bf16 rounding.
// ============================================================================
namespace {
constexpr int FB_BQ = 64;                       // queries per step of the dK/dV kernel
constexpr int FB_QT = FB_BQ * FA_D * 2;         // 16 KB: two 8 KB SW128 atoms
#ifndef EE_FB_QST
#define EE_FB_QST 4                                 // Q / dO ring stages of the dK/dV kernel
#endif
constexpr int FB_QST = EE_FB_QST;
constexpr int FB_SMEM_KV = 1024 + 2 * FA_TILE + FB_QST * 2 * FB_QT + 2 * 2 * FB_BQ * 4 + 512;
constexpr int FQ_BK = 64;                       // keys per step of the dQ kernel
constexpr int FQ_KT = FQ_BK * FA_D * 2;         // 16 KB K or V tile
constexpr int FQ_STAGES = 4;
constexpr int FB_SMEM_Q = 1024 + 2 * FA_TILE + FQ_STAGES * 2 * FQ_KT + 256;

// RoPE^T (rotation by -angle) of 32 columns [c0, c0 + 32) (c0 < 64) paired
// with [c0 + 64, c0 + 96) of one row at position pos.
// tab: the (cos, sin) row of `pos` of launch_rope_table's table, or NULL
// (then computed with powf + sincosf in fp32).
__device__ __forceinline__ void rope_t_32(float* a, float* b, int c0, float pos, float theta,
                                          const float2* tab) {
#pragma unroll
  for (int i = 0; i < 32; i += 2) {
    float csn[4];
    if (tab) {
      const float4 t4 = *reinterpret_cast<const float4*>(tab + c0 + i);
      csn[0] = t4.x; csn[1] = t4.y; csn[2] = t4.z; csn[3] = t4.w;
    } else {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const float inv = powf(theta, -2.0f * (float)(c0 + i + e) / 128.0f);
        sincosf(pos * inv, &csn[2 * e + 1], &csn[2 * e]);
      }
    }
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const float cs = csn[2 * e], sn = csn[2 * e + 1];
      const float x = a[i + e], y = b[i + e];
      a[i + e] = x * cs + y * sn;
      b[i + e] = y * cs - x * sn;
    }
  }
}

// Row r of a [rows x 128] fp32 TMEM accumulator -> scale, optional RoPE^T at
// `pos`, bf16, 256 bytes at dst.
__device__ __forceinline__ void store_row_bf16(uint32_t tacc, __nv_bfloat16* dst, bool ok,
                                               float scale, float pos, float theta, int c0 = 0,
                                               int c1 = 2, const float2* tab = nullptr) {
#pragma unroll 1
  for (int c = c0; c < c1; ++c) {
    uint32_t va[32], vb[32];
    tmem_ld_32x32b_x32(tacc + c * 32, va);
    tmem_ld_wait();
    tmem_ld_32x32b_x32(tacc + 64 + c * 32, vb);
    tmem_ld_wait();
    float a[32], b[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      a[i] = __uint_as_float(va[i]) * scale;
      b[i] = __uint_as_float(vb[i]) * scale;
    }
    if (theta > 0.f) rope_t_32(a, b, c * 32, pos, theta, tab);
    if (ok) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        uint32_t wa[8], wb[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          wa[q] = pack_bf16(a[h * 16 + 2 * q], a[h * 16 + 2 * q + 1]);
          wb[q] = pack_bf16(b[h * 16 + 2 * q], b[h * 16 + 2 * q + 1]);
        }
        __nv_bfloat16* pa = dst + c * 32 + h * 16;
        __nv_bfloat16* pb = pa + 64;
        if (aligned32(pa) && aligned32(pb)) {
          st_global_v8(pa, wa);
          st_global_v8(pb, wb);
        } else {
          *reinterpret_cast<uint4*>(pa) = make_uint4(wa[0], wa[1], wa[2], wa[3]);
          *reinterpret_cast<uint4*>(pa + 8) = make_uint4(wa[4], wa[5], wa[6], wa[7]);
          *reinterpret_cast<uint4*>(pb) = make_uint4(wb[0], wb[1], wb[2], wb[3]);
          *reinterpret_cast<uint4*>(pb + 8) = make_uint4(wb[4], wb[5], wb[6], wb[7]);
        }
      }
    }
  }
}
}  // namespace

// dK, dV: one CTA per (128-key tile, kv head, sequence); loops over the query
// heads of the GQA group and the 64-query tiles at or after the key tile.
//   warp 0 TMA (K, V once; Q_i, dO_i in a FB_QST-stage ring), warp 1 MMA,
//   warps 4..7 one thread per key row (TMEM lane).
// TMEM: S^T [128 x 64] | dP^T [128 x 64] | dK [128 x 128] | dV [128 x 128].
__global__ void __launch_bounds__(384, 1)
    attn_bwd_dkdv_tc_kernel(const __grid_constant__ CUtensorMap tmQ,
                            const __grid_constant__ CUtensorMap tmK,
                            const __grid_constant__ CUtensorMap tmV,
                            const __grid_constant__ CUtensorMap tmDO,
                            const float* __restrict__ lse2, const float* __restrict__ Dv,
                            __nv_bfloat16* __restrict__ dk, __nv_bfloat16* __restrict__ dv,
                            int T, int Hq, int Hkv, float scale_log2, float scale,
                            float rope_theta, const float2* __restrict__ rope_tab) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint8_t* sK = smem;
  uint8_t* sV = sK + FA_TILE;
  uint8_t* sQ = sV + FA_TILE;          // [FB_QST] x 16 KB
  uint8_t* sDO = sQ + FB_QST * FB_QT;  // [FB_QST] x 16 KB
  float* sL = reinterpret_cast<float*>(sDO + FB_QST * FB_QT);  // [2][64]
  float* sD = sL + 2 * FB_BQ;                              // [2][64]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sD + 2 * FB_BQ);
  uint64_t* kv_full = bars;
  uint64_t* qd_full = bars + 1;              // [FB_QST]
  uint64_t* qd_empty = qd_full + FB_QST;     // [FB_QST]
  uint64_t* sdp_full = qd_empty + FB_QST;    // [2]
  uint64_t* pds_full = sdp_full + 2;         // [2], per P^T/dS^T buffer (see attn_bwd_dq_tc_kernel)
  uint64_t* acc_done = pds_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_done + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int kt = blockIdx.x, hk = blockIdx.y, b = blockIdx.z;
  const int grp = Hq / Hkv;
  const int nq64 = (T + FB_BQ - 1) / FB_BQ;
  const int q64_0 = kt * (FA_BN / FB_BQ);           // first 64-query tile touching this key tile
  const int per_head = nq64 - q64_0;
  const int n_it = grp * per_head;
  const int k_row0 = b * T + kt * FA_BN;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmQ);
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
    tma_prefetch_desc(&tmDO);
    mbar_init(kv_full, 1);
    for (int s = 0; s < FB_QST; ++s) {
      mbar_init(&qd_full[s], 1);
      mbar_init(&qd_empty[s], 1);
    }
    mbar_init(&sdp_full[0], 1);
    mbar_init(&sdp_full[1], 1);
    mbar_init(&pds_full[0], 256);
    mbar_init(&pds_full[1], 256);
    mbar_init(acc_done, 1);
    fence_barrier_init();
  }
  if (warp == 2) {
    tmem_alloc(tmem_slot, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // S^T[b] at b*128, dP^T[b] at b*128 + 64 (b = step parity); dK, dV after
  const uint32_t tDK = tmem_base + 256, tDV = tmem_base + 384;

  if (warp == 0) {
    if (lane == 0) {
      tma_load_2d(sK, &tmK, kv_full, hk * FA_D, k_row0);
      tma_load_2d(sK + FA_ATOM, &tmK, kv_full, hk * FA_D + 64, k_row0);
      tma_load_2d(sV, &tmV, kv_full, hk * FA_D, k_row0);
      tma_load_2d(sV + FA_ATOM, &tmV, kv_full, hk * FA_D + 64, k_row0);
      mbar_arrive_expect_tx(kv_full, 2 * FA_TILE);
      for (int it = 0; it < n_it; ++it) {
        const int s = it % FB_QST;
        const int hq = hk * grp + it / per_head;
        const int q_row0 = b * T + (q64_0 + it % per_head) * FB_BQ;
        mbar_wait(&qd_empty[s], ((it / FB_QST) & 1) ^ 1);
        uint8_t* q = sQ + s * FB_QT;
        uint8_t* d = sDO + s * FB_QT;
        tma_load_2d(q, &tmQ, &qd_full[s], hq * FA_D, q_row0);
        tma_load_2d(q + FB_QT / 2, &tmQ, &qd_full[s], hq * FA_D + 64, q_row0);
        tma_load_2d(d, &tmDO, &qd_full[s], hq * FA_D, q_row0);
        tma_load_2d(d + FB_QT / 2, &tmDO, &qd_full[s], hq * FA_D + 64, q_row0);
        mbar_arrive_expect_tx(&qd_full[s], 2 * FB_QT);
      }
    }
  } else if (warp == 1) {
    {  // whole warp; elect.sync issues (ptx.cuh tc_mma_f16_w)
      constexpr uint32_t idesc_s = make_idesc_bf16(FA_BN, FB_BQ, false, false);   // 128 x 64
      constexpr uint32_t idesc_acc = make_idesc_bf16(FA_BN, FA_D, false, true);   // 128 x 128
      const uint32_t ak = smem_u32(sK), av = smem_u32(sV);
      mbar_wait(kv_full, 0);
      tc_fence_after();
      // S^T / dP^T of step `it` into TMEM buffer it & 1, issued one step ahead
      // so the tensor core works while the softmax threads process the last one
      auto issue_sdp = [&](int it) {
        const int qs = it % FB_QST;
        mbar_wait(&qd_full[qs], (it / FB_QST) & 1);
        tc_fence_after();
        const uint32_t bq = smem_u32(sQ + qs * FB_QT), bd = smem_u32(sDO + qs * FB_QT);
        const uint32_t tS = tmem_base + (it & 1) * 128, tDP = tS + 64;
        // descriptors built once; the k-step offsets (< 64 KB, 16-byte units)
        // are added to the start-address field (no carry out of its 14 bits)
        const uint64_t dk0 = make_sdesc(ak, 16, 1024), dv0 = make_sdesc(av, 16, 1024);
        const uint64_t dq0 = make_sdesc(bq, 16, 1024), ddo0 = make_sdesc(bd, 16, 1024);
#pragma unroll
        for (int k = 0; k < FA_D / 16; ++k) {  // S^T = K Q^T, dP^T = V dO^T (K-major, K = d)
          const uint32_t offa = ((k >> 2) * FA_ATOM + (k & 3) * 32) >> 4;
          const uint32_t offb = ((k >> 2) * (FB_QT / 2) + (k & 3) * 32) >> 4;
          tc_mma_f16_w(tS, dk0 + offa, dq0 + offb, idesc_s, k != 0 ? 1u : 0u);
          tc_mma_f16_w(tDP, dv0 + offa, ddo0 + offb, idesc_s, k != 0 ? 1u : 0u);
        }
        tc_commit_w(&sdp_full[it & 1]);
      };
      if (n_it > 0) issue_sdp(0);
      for (int it = 0; it < n_it; ++it) {
        const int s = it & 1;
        if (it + 1 < n_it) issue_sdp(it + 1);
        mbar_wait(&pds_full[s], (it >> 1) & 1);
        tc_fence_after();
        const int qs = it % FB_QST;
        const uint32_t bq = smem_u32(sQ + qs * FB_QT), bd = smem_u32(sDO + qs * FB_QT);
        const uint32_t tPt = tmem_base + s * 128, tDSt = tPt + 64;
        const uint64_t ddo0 = make_sdesc(bd, FB_QT / 2, 1024), dq0 = make_sdesc(bq, FB_QT / 2, 1024);
#pragma unroll
        for (int k = 0; k < FB_BQ / 16; ++k) {  // dV += P^T dO, dK += dS^T Q (A in TMEM, K = q)
          // queries 16k.. sit at column 32*(k/2) + 8*(k%2) (each warpgroup's slab)
          const uint32_t offa = (k >> 1) * 32 + (k & 1) * 8;
          const uint32_t offb = (k * 2048) >> 4;
#ifndef EE_EXPT_NO_DVDK  // timing experiment (profiles/r02attn), never in the product build
          tc_mma_f16_ts_w(tDV, tPt + offa, ddo0 + offb, idesc_acc, (it | k) != 0 ? 1u : 0u);
          tc_mma_f16_ts_w(tDK, tDSt + offa, dq0 + offb, idesc_acc, (it | k) != 0 ? 1u : 0u);
#endif
        }
        tc_commit_w(&qd_empty[qs]);
      }
      tc_commit_w(acc_done);
    }
  } else if (warp >= 4) {
    // two softmax warpgroups: warps w and w + 4 share TMEM lanes 32 (w % 4) ..
    // and take query columns [0, 32) and [32, 64) of every step
    const int ew = (warp - 4) & 3, half = (warp - 4) >> 2;
    const int kr = ew * 32 + lane;  // key row = TMEM lane
    const int kpos = kt * FA_BN + kr;
    const uint32_t lane_off = static_cast<uint32_t>(ew * 32) << 16;
    const int tid = threadIdx.x - 128;
    // thread tid < 64 stages lse2 of query tid of the step, tid >= 64 stages Dv;
    // the global load for step it + 1 is issued during step it
    auto stat_of = [&](int it) -> float {
      const int hq = hk * grp + it / per_head;
      const int qpos0 = (q64_0 + it % per_head) * FB_BQ;
      const int t = tid & (FB_BQ - 1);
      if (qpos0 + t >= T) return 0.f;
      const long long idx = (long long)(b * T + qpos0 + t) * Hq + hq;
      return tid < FB_BQ ? lse2[idx] : Dv[idx];
    };
    float stat_next = (n_it > 0 && tid < 2 * FB_BQ) ? stat_of(0) : 0.f;
    for (int it = 0; it < n_it; ++it) {
      // P^T / dS^T overwrite S^T / dP^T of buffer it & 1 once read; S^T(it+2)
      // reuses the buffer only after dV/dK(it) (tensor-pipe issue order)
      const uint32_t tS = tmem_base + (it & 1) * 128, tDP = tS + 64;
      const int qpos0 = (q64_0 + it % per_head) * FB_BQ;
      float* L = sL + (it & 1) * FB_BQ;
      float* D = sD + (it & 1) * FB_BQ;
      if (tid < 2 * FB_BQ) {  // staged negated: the packed FMA / add below take -lse2, -Dv
        (tid < FB_BQ ? L : D)[tid & (FB_BQ - 1)] = -stat_next;
        if (it + 1 < n_it) stat_next = stat_of(it + 1);
      }
      asm volatile("bar.sync 1, 256;" ::: "memory");
      mbar_wait(&sdp_full[it & 1], (it >> 1) & 1);
      tc_fence_after();
#ifdef EE_EXPT_NO_SOFTMAX  // timing experiment (profiles/r02attn), never in the product build
      if (true) {
        tc_fence_before();
        mbar_arrive(&pds_full[it & 1]);
        continue;
      }
#endif
      {
        const int c = half;
        uint32_t vs[32], vp[32];
        tmem_ld_32x32b_x32(tS + lane_off + c * 32, vs);
        tmem_ld_32x32b_x32(tDP + lane_off + c * 32, vp);
        tmem_ld_wait();
        uint32_t wp[16], wd[16];
        // the causal / sequence-end mask only on the tiles that need it
        // (CTA-uniform); packed f32x2 FMA / add / mul with the same per-element
        // roundings as fmaf / fadd / fmul (the softmax is issue-bound: ncu,
        // profiles/r02attn)
        const bool need_mask = qpos0 < kt * FA_BN + FA_BN || qpos0 + FB_BQ > T;
        const unsigned long long sc2 = f2pack(scale_log2, scale_log2);
        // -lse2 / -Dv of this half's 32 query columns: explicit shared loads (the
        // generic float2 loads compiled to LD.E through the global path, ncu
        // stall_lg, profiles/r02attn)
        float nlv[32], ndv[32];
        const uint32_t la = smem_u32(L + c * 32), da = smem_u32(D + c * 32);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];"
                       : "=f"(nlv[4 * q]), "=f"(nlv[4 * q + 1]), "=f"(nlv[4 * q + 2]), "=f"(nlv[4 * q + 3])
                       : "r"(la + 16 * q));
          asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];"
                       : "=f"(ndv[4 * q]), "=f"(ndv[4 * q + 1]), "=f"(ndv[4 * q + 2]), "=f"(ndv[4 * q + 3])
                       : "r"(da + 16 * q));
        }
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          const float2 nl = make_float2(nlv[2 * q], nlv[2 * q + 1]);
          const float2 nd = make_float2(ndv[2 * q], ndv[2 * q + 1]);
          float x0, x1, p0, p1, d0, d1;
          f2unpack(ffma2(f2pack(__uint_as_float(vs[2 * q]), __uint_as_float(vs[2 * q + 1])), sc2,
                         f2pack(nl.x, nl.y)), x0, x1);
          p0 = ex2_approx(x0);
          p1 = ex2_approx(x1);
          if (need_mask) {
            const int qpos = qpos0 + c * 32 + 2 * q;
            if (qpos < kpos || qpos >= T) p0 = 0.f;
            if (qpos + 1 < kpos || qpos + 1 >= T) p1 = 0.f;
          }
          const unsigned long long t2 = fadd2(
              f2pack(__uint_as_float(vp[2 * q]), __uint_as_float(vp[2 * q + 1])), f2pack(nd.x, nd.y));
          f2unpack(fmul2(f2pack(p0, p1), t2), d0, d1);
          wp[q] = pack_bf16(p0, p1);
          wd[q] = pack_bf16(d0, d1);
        }
        // P^T and dS^T as TMEM A operands: this warpgroup's 32 query columns,
        // packed bf16x2, over the first 16 columns of its own fp32 slab of the
        // S^T / dP^T buffers (already read into registers above)
        tmem_st_32x32b_x16(tS + lane_off + c * 32, wp);
        tmem_st_32x32b_x16(tDP + lane_off + c * 32, wd);
        tmem_st_wait();
      }
      tc_fence_before();
      mbar_arrive(&pds_full[it & 1]);
    }
    mbar_wait(acc_done, 0);
    tc_fence_after();
    const bool ok = kpos < T;
    const long long ldk = (long long)Hkv * FA_D;
    if (half == 0)
      store_row_bf16(tDK + lane_off, dk + (long long)(k_row0 + kr) * ldk + hk * FA_D, ok, scale,
                     (float)kpos, rope_theta, 0, 2,
                     rope_tab && ok ? rope_tab + (long long)kpos * 64 : nullptr);
    else
      store_row_bf16(tDV + lane_off, dv + (long long)(k_row0 + kr) * ldk + hk * FA_D, ok, 1.0f,
                     0.f, 0.f);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem_base, 512);
  }
}

// dQ: one CTA per (128-query tile, query head, sequence); loops over the
// 64-key tiles at or before the query tile (4-stage K/V ring).  TMEM: three
// [S | dP] buffers of 128 columns (S/dP of steps j+1 and j+2 are queued on
// the tensor core while the softmax threads form dS_j) and dQ (128 columns).
// dS in smem is double-buffered.
__global__ void __launch_bounds__(384, 1)
    attn_bwd_dq_tc_kernel(const __grid_constant__ CUtensorMap tmQ,
                          const __grid_constant__ CUtensorMap tmK,
                          const __grid_constant__ CUtensorMap tmV,
                          const __grid_constant__ CUtensorMap tmDO,
                          const float* __restrict__ lse2, const float* __restrict__ Dv,
                          __nv_bfloat16* __restrict__ dq, int T, int Hq, int Hkv, float scale_log2,
                          float scale, float rope_theta, const float2* __restrict__ rope_tab) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint8_t* sQ = smem;
  uint8_t* sDO = sQ + FA_TILE;
  uint8_t* sK = sDO + FA_TILE;                  // [STAGES] x 16 KB (64 keys x 128 d)
  uint8_t* sV = sK + FQ_STAGES * FQ_KT;         // [STAGES]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sV + FQ_STAGES * FQ_KT);
  uint64_t* qo_full = bars;
  uint64_t* kv_full = bars + 1;                 // [STAGES]
  uint64_t* kv_empty = kv_full + FQ_STAGES;     // [STAGES]
  uint64_t* sdp_full = kv_empty + FQ_STAGES;    // [3]
  // ds_full[j % 3]: dS of step j written (into S buffer j % 3).  One barrier
  // per buffer: step j + 3 needs S/dP(j + 3), issued only after the MMA
  // thread has observed ds_full(j), so no barrier can run two phases ahead
  // of its waiter
  uint64_t* ds_full = sdp_full + 3;             // [3]
  uint64_t* acc_done = ds_full + 3;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_done + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nqt = (T + FA_BM - 1) / FA_BM;
  const int qt = nqt - 1 - (int)blockIdx.x;
  const int hq = blockIdx.y, b = blockIdx.z;
  const int hk = hq / (Hq / Hkv);
  const int q_row0 = b * T + qt * FA_BM;
  const int n_kt = (qt + 1) * (FA_BM / FQ_BK);   // 64-key tiles up to the diagonal

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmQ);
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
    tma_prefetch_desc(&tmDO);
    mbar_init(qo_full, 1);
    for (int s = 0; s < FQ_STAGES; ++s) {
      mbar_init(&kv_full[s], 1);
      mbar_init(&kv_empty[s], 1);
    }
    for (int bb = 0; bb < 3; ++bb) mbar_init(&sdp_full[bb], 1);
    for (int bb = 0; bb < 3; ++bb) mbar_init(&ds_full[bb], 256);
    mbar_init(acc_done, 1);
    fence_barrier_init();
  }
  if (warp == 2) {
    tmem_alloc(tmem_slot, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const uint32_t tDQ = tmem_base + 384;          // S[b] at b*128, dP[b] at b*128 + 64, b < 3

  if (warp == 0) {
    if (lane == 0) {
      tma_load_2d(sQ, &tmQ, qo_full, hq * FA_D, q_row0);
      tma_load_2d(sQ + FA_ATOM, &tmQ, qo_full, hq * FA_D + 64, q_row0);
      tma_load_2d(sDO, &tmDO, qo_full, hq * FA_D, q_row0);
      tma_load_2d(sDO + FA_ATOM, &tmDO, qo_full, hq * FA_D + 64, q_row0);
      mbar_arrive_expect_tx(qo_full, 2 * FA_TILE);
      for (int j = 0; j < n_kt; ++j) {
        const int s = j % FQ_STAGES;
        mbar_wait(&kv_empty[s], ((j / FQ_STAGES) & 1) ^ 1);
        const int k_row0 = b * T + j * FQ_BK;
        uint8_t* k = sK + s * FQ_KT;
        uint8_t* v = sV + s * FQ_KT;
        tma_load_2d(k, &tmK, &kv_full[s], hk * FA_D, k_row0);
        tma_load_2d(k + FQ_KT / 2, &tmK, &kv_full[s], hk * FA_D + 64, k_row0);
        tma_load_2d(v, &tmV, &kv_full[s], hk * FA_D, k_row0);
        tma_load_2d(v + FQ_KT / 2, &tmV, &kv_full[s], hk * FA_D + 64, k_row0);
        mbar_arrive_expect_tx(&kv_full[s], 2 * FQ_KT);
      }
    }
  } else if (warp == 1) {
    {  // whole warp; elect.sync issues (ptx.cuh tc_mma_f16_w)
      constexpr uint32_t idesc_s = make_idesc_bf16(FA_BM, FQ_BK, false, false);   // 128 x 64
      constexpr uint32_t idesc_dq = make_idesc_bf16(FA_BM, FA_D, false, true);    // 128 x 128
      const uint32_t aq = smem_u32(sQ), ado = smem_u32(sDO);
      mbar_wait(qo_full, 0);
      auto issue_sdp = [&](int j) {
        const int s = j % FQ_STAGES;
        mbar_wait(&kv_full[s], (j / FQ_STAGES) & 1);
        tc_fence_after();
        const uint32_t bk = smem_u32(sK + s * FQ_KT), bv = smem_u32(sV + s * FQ_KT);
        const uint32_t tS = tmem_base + (j % 3) * 128, tDP = tS + 64;
        const uint64_t dq0 = make_sdesc(aq, 16, 1024), ddo0 = make_sdesc(ado, 16, 1024);
        const uint64_t dk0 = make_sdesc(bk, 16, 1024), dv0 = make_sdesc(bv, 16, 1024);
#pragma unroll
        for (int k = 0; k < FA_D / 16; ++k) {  // S = Q K^T, dP = dO V^T  (K = d)
          const uint32_t offa = ((k >> 2) * FA_ATOM + (k & 3) * 32) >> 4;
          const uint32_t offb = ((k >> 2) * (FQ_KT / 2) + (k & 3) * 32) >> 4;
          tc_mma_f16_w(tS, dq0 + offa, dk0 + offb, idesc_s, k != 0 ? 1u : 0u);
          tc_mma_f16_w(tDP, ddo0 + offa, dv0 + offb, idesc_s, k != 0 ? 1u : 0u);
        }
        tc_commit_w(&sdp_full[j % 3]);
      };
      issue_sdp(0);
      if (n_kt > 1) issue_sdp(1);
      for (int j = 0; j < n_kt; ++j) {
        // buffer (j + 2) % 3 held S/dP of step j - 1, whose dS the softmax has
        // published (ds_full(j - 1) waited in the previous iteration)
        if (j + 2 < n_kt) issue_sdp(j + 2);
        mbar_wait(&ds_full[j % 3], (j / 3) & 1);
        tc_fence_after();
        const int s = j % FQ_STAGES;
        const uint32_t bk = smem_u32(sK + s * FQ_KT), tDS = tmem_base + (j % 3) * 128;
        const uint64_t dkm = make_sdesc(bk, FQ_KT / 2, 1024);
#pragma unroll
        for (int k = 0; k < FQ_BK / 16; ++k)  // dQ += dS K  (dS in TMEM; K MN-major, LBO 8 KB)
          tc_mma_f16_ts_w(tDQ, tDS + (k >> 1) * 32 + (k & 1) * 8, dkm + ((k * 2048) >> 4),
                          idesc_dq, (j | k) != 0 ? 1u : 0u);
        tc_commit_w(&kv_empty[s]);
      }
      tc_commit_w(acc_done);
    }
  } else if (warp >= 4) {
    // two softmax warpgroups: key columns [0, 32) and [32, 64) of every step
    const int ew = (warp - 4) & 3, half = (warp - 4) >> 2;
    const int r = ew * 32 + lane;
    const int pos = qt * FA_BM + r;
    const uint32_t lane_off = static_cast<uint32_t>(ew * 32) << 16;
    const bool ok = pos < T;
    const float Lr = ok ? lse2[(long long)(q_row0 + r) * Hq + hq] : 0.f;
    const float Dr = ok ? Dv[(long long)(q_row0 + r) * Hq + hq] : 0.f;
    for (int j = 0; j < n_kt; ++j) {
      mbar_wait(&sdp_full[j % 3], (j / 3) & 1);
      tc_fence_after();
      const uint32_t tS = tmem_base + (j % 3) * 128 + lane_off, tDP = tS + 64;
      {
        const int c = half;
        uint32_t vs[32], vp[32];
        tmem_ld_32x32b_x32(tS + c * 32, vs);
        tmem_ld_32x32b_x32(tDP + c * 32, vp);
        tmem_ld_wait();
        uint32_t wd[16];
        // mask only on the key tiles at the diagonal or rows past T (CTA-uniform);
        // packed f32x2 ops, same per-element roundings (profiles/r02attn)
        const bool need_mask = j * FQ_BK + FQ_BK - 1 > qt * FA_BM || qt * FA_BM + FA_BM > T;
        const unsigned long long sc2 = f2pack(scale_log2, scale_log2);
        const unsigned long long nl2 = f2pack(-Lr, -Lr), nd2 = f2pack(-Dr, -Dr);
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          float x0, x1, p0, p1, d0, d1;
          f2unpack(ffma2(f2pack(__uint_as_float(vs[2 * q]), __uint_as_float(vs[2 * q + 1])), sc2,
                         nl2), x0, x1);
          p0 = ex2_approx(x0);
          p1 = ex2_approx(x1);
          if (need_mask) {
            const int kpos = j * FQ_BK + c * 32 + 2 * q;
            if (kpos > pos || !ok) p0 = 0.f;
            if (kpos + 1 > pos || !ok) p1 = 0.f;
          }
          const unsigned long long t2 =
              fadd2(f2pack(__uint_as_float(vp[2 * q]), __uint_as_float(vp[2 * q + 1])), nd2);
          f2unpack(fmul2(f2pack(p0, p1), t2), d0, d1);
          wd[q] = pack_bf16(d0, d1);
        }
        // dS as a TMEM A operand: packed into the first 16 columns of this
        // warpgroup's fp32 slab of the S buffer (read above)
        tmem_st_32x32b_x16(tS + c * 32, wd);
        tmem_st_wait();
      }
      tc_fence_before();
      mbar_arrive(&ds_full[j % 3]);
    }
    mbar_wait(acc_done, 0);
    tc_fence_after();
    store_row_bf16(tDQ + lane_off, dq + (long long)(q_row0 + r) * Hq * FA_D + hq * FA_D, ok, scale,
                   (float)pos, rope_theta, half, half + 1,
                   rope_tab && ok ? rope_tab + (long long)pos * 64 : nullptr);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem_base, 512);
  }
}

cudaError_t launch_attn_bwd_tc(const __nv_bfloat16* q, const __nv_bfloat16* k,
                               const __nv_bfloat16* v, const __nv_bfloat16* dout,
                               const float* lse2, const float* Dv, __nv_bfloat16* dq,
                               __nv_bfloat16* dk, __nv_bfloat16* dv, long long N, int T, int Hq,
                               int Hkv, float rope_theta, cudaStream_t s,
                               const float2* rope_tab) {
  if (N == 0) return cudaSuccess;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(attn_bwd_dkdv_tc_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, FB_SMEM_KV);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(attn_bwd_dq_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             FB_SMEM_Q);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const Mat Q{q, N, (long long)Hq * FA_D, (long long)Hq * FA_D};
  const Mat DO{dout, N, (long long)Hq * FA_D, (long long)Hq * FA_D};
  const Mat K{k, N, (long long)Hkv * FA_D, (long long)Hkv * FA_D};
  const Mat V{v, N, (long long)Hkv * FA_D, (long long)Hkv * FA_D};
  CUtensorMap tq64, tdo64, tq128, tdo128, tk, tv, tk64, tv64;
  if (!make_tmap(&tq64, Q, 64, FB_BQ) || !make_tmap(&tdo64, DO, 64, FB_BQ) ||
      !make_tmap(&tq128, Q, 64, FA_BM) || !make_tmap(&tdo128, DO, 64, FA_BM) ||
      !make_tmap(&tk, K, 64, FA_BN) || !make_tmap(&tv, V, 64, FA_BN) ||
      !make_tmap(&tk64, K, 64, FQ_BK) || !make_tmap(&tv64, V, 64, FQ_BK))
    return cudaErrorInvalidValue;
  const float scale = 1.0f / sqrtf((float)FA_D);
  const float scale_log2 = 1.4426950408889634f * scale;
  const unsigned B = (unsigned)(N / T);
  dim3 g1((T + FA_BN - 1) / FA_BN, Hkv, B);
  attn_bwd_dkdv_tc_kernel<<<g1, 384, FB_SMEM_KV, s>>>(tq64, tk, tv, tdo64, lse2, Dv, dk, dv, T, Hq,
                                                      Hkv, scale_log2, scale, rope_theta,
                                                      rope_tab);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  dim3 g2((T + FA_BM - 1) / FA_BM, Hq, B);
  attn_bwd_dq_tc_kernel<<<g2, 384, FB_SMEM_Q, s>>>(tq128, tk64, tv64, tdo128, lse2, Dv, dq, T, Hq,
                                                   Hkv, scale_log2, scale, rope_theta,
                                                   rope_tab);
  return cudaGetLastError();
}

}  // namespace ee
