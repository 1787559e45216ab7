// tcgen05 tensor-core GEMM for sm_100a with the decoder/LM epilogues.
//
//   C[m, n] = acc_scale * sum_p sum_k A_p[m, k] * W[n, k]   (p over the planes)
//
// A is the fp32 activation split into operand planes (common.cuh: by default
// two fp16 planes of x 2^8, 22 significant bits; or three bf16 planes), written
// by fb_pack_rows and by the LSTM epilogues; W holds the weights exactly
// (power-of-two scaled fp16, or bf16); accumulation is fp32 in TMEM -- an
// fp32-accurate product on the 5th-gen tensor cores (SURVEY.md §7 "GEMM
// precision").  Algorithmic FLOPs count the product once.
//
// Accuracy: the tensor core's fp32 accumulation in TMEM is not IEEE
// round-to-nearest -- its error grows ~k^1.5 (7.5x an fp32 dot product at
// k = 4096, scripts/gemm_accuracy2.py).  So K is consumed in chunks of
// TC_KCB * 64 = 256: each chunk is accumulated in its own TMEM slot (a ring of
// TC_NACC slots) and the epilogue warps drain every chunk into fp32 registers
// (round-to-nearest adds).  The MMA issuer runs up to TC_NACC chunks ahead.
//
// Structure (persistent, one CTA per SM, 10 warps):
//   warp 0 lane 0 : TMA producer, 3-stage smem ring (128B swizzle, K block 64)
//   warp 1 lane 0 : MMA issuer (tcgen05.mma.cta_group::1.kind::f16, M=128)
//   warp 1        : TMEM allocator (TC_NACC x BN fp32 columns: the chunk ring)
//   warps 2..9    : chunk drains + epilogue, tcgen05.ld 32x32b (warp w owns TMEM
//                   lanes 32(w%4).., column half (w-2)/4 of the tile)
#include "common.cuh"

#include <cstdlib>

#include <cuda.h>
#include <cuda_bf16.h>
#include <cudaTypedefs.h>

namespace fb {

#ifdef FB_GEMM_TRACE
// dev experiment: per-k-block event times (ns, %globaltimer) of CTA 0
__device__ unsigned long long g_trace[10][256];
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define TRACE(slot, i) do { if (blockIdx.x == 0 && (i) < 256 && (threadIdx.x & 31) == 0) g_trace[slot][i] = gtime(); } while (0)
// per-CTA stamp of one chosen step (recurrence skew)
#define TRACE_CTA(slot, t, t0) do { if ((t) == (t0) && blockIdx.x < 256) g_trace[slot][blockIdx.x] = gtime(); } while (0)
#else
#define TRACE(slot, i) do {} while (0)
#define TRACE_CTA(slot, t, t0) do {} while (0)
#endif

constexpr int TC_BM = 128;
constexpr int TC_BK = 64;            // 64 bf16 = 128 B = one swizzle atom
constexpr int TC_STAGES = kPlanes == 2 ? 4 : 3;   // smem ring: 4 x 48 KB or 3 x 64 KB
// stages of the GEMM ring for a tile width (4 x 48 KB or 3 x 64 KB, + the 33 KB
// epilogue staging within the 227 KB of a CTA)
constexpr int tc_stages(int bn) {
  return (kPlanes * 128 * 64 * 2 + bn * 64 * 2) <= 48 * 1024 ? 4
         : (kPlanes * 128 * 64 * 2 + bn * 64 * 2) <= 64 * 1024 ? 3 : 2;
}
constexpr int TC_KCB = 4;            // K blocks per accumulation chunk (K = 256)
constexpr int TC_NACC = 4;           // TMEM chunk slots (4 x 128 columns = all of TMEM)
#ifndef FB_GEMM_GROUP
#define FB_GEMM_GROUP 1              // chunks per slot-group handshake (1, 2 or 4)
#endif
constexpr int TC_EPI_THREADS = 256;
// instruction descriptor operand formats (kind::f16): a/b = F16 (0) or BF16 (1)
constexpr uint32_t kIdescAB = FB_OPERAND_FP16X2 ? 0u : ((1u << 7) | (1u << 10));     // 8 epilogue warps: 2 per TMEM lane quarter
constexpr int TC_THREADS = 64 + TC_EPI_THREADS;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra DONE_%=;\n\t"
      "bra WAIT_%=;\n"
      "DONE_%=:\n\t}" ::"r"(bar),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, uint32_t bar,
                                            int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar)
      : "memory");
}

__device__ __forceinline__ uint64_t smem_desc_sw128(uint32_t saddr) {
  // K-major, SWIZZLE_128B: start>>4 | SBO (8 rows x 128 B = 1024 B)>>4 << 32 |
  // version 1 << 46 | layout 2 << 61 (cute::UMMA::SmemDescriptor)
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}

__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                         uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

// warp-uniform issue: every lane runs the loop (descriptors stay in uniform
// registers), one elected lane issues -- avoids a per-MMA R2UR/ELECT sequence
__device__ __forceinline__ void mma_bf16_elect(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                               uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit_elect(uint32_t bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(
          bar)
      : "memory");
}

__device__ __forceinline__ void mma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   bar)
               : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float* v) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32"
      " {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// 64 consecutive columns of this warp's 32 lanes, no wait (the caller issues
// tcgen05.wait::ld before reading r)
__device__ __forceinline__ void tmem_ld64_nowait(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x64.b32"
      " {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,%47,%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63}, [%64];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31]), "=r"(r[32]), "=r"(r[33]), "=r"(r[34]), "=r"(r[35]), "=r"(r[36]), "=r"(r[37]), "=r"(r[38]), "=r"(r[39]), "=r"(r[40]), "=r"(r[41]), "=r"(r[42]), "=r"(r[43]), "=r"(r[44]), "=r"(r[45]), "=r"(r[46]), "=r"(r[47]), "=r"(r[48]), "=r"(r[49]), "=r"(r[50]), "=r"(r[51]), "=r"(r[52]), "=r"(r[53]), "=r"(r[54]), "=r"(r[55]), "=r"(r[56]), "=r"(r[57]), "=r"(r[58]), "=r"(r[59]), "=r"(r[60]), "=r"(r[61]), "=r"(r[62]), "=r"(r[63])
      : "r"(taddr));
}

__device__ __forceinline__ float sigm_tc(float x) { return 1.0f / (1.0f + expf(-x)); }

// MUFU ex2 + rcp; __fdividef returns 0 for denominators > 2^126, which is the
// correct limit here (sigmoid -> 0, tanh -> -1)
#ifdef FB_PRECISE_ACT
__device__ __forceinline__ float fsig(float x) { return 1.0f / (1.0f + expf(-x)); }
__device__ __forceinline__ float ftanh(float x) { return tanhf(x); }
#else
__device__ __forceinline__ float fsig(float x) { return __fdividef(1.0f, 1.0f + __expf(-x)); }

__device__ __forceinline__ float ftanh(float x) {
  return 1.0f - __fdividef(2.0f, 1.0f + __expf(2.0f * x));
}
#endif

__device__ __forceinline__ void store_split(const fb_gemm_t& g, int64_t row, int col, float x) {
  // operand planes of an fp32 value (the next GEMM's A operand)
  uint16_t* o = reinterpret_cast<uint16_t*>(g.h_split) + row * g.ld_hs + col;
  uint16_t e[3];
  split_operand(x, e);
#pragma unroll
  for (int q = 0; q < kPlanes; ++q) o[q * g.hs_plane_rows * g.ld_hs] = e[q];
}

// One warp drains its 32 TMEM lanes (rows) chunk by chunk; each 32x32 chunk is
// transposed through shared memory so global loads/stores are row-contiguous
// across the warp (plain mode: lane = column; LSTM mode: lane = (row, unit)).
template <int BN>
__device__ __forceinline__ void epilogue_tile(const fb_gemm_t& g, int M, int row0, int n0,
                                              const float (*acc)[32],
                                              float* st /* [32][33] */, int half,
                                              const CUtensorMap* tmC = nullptr,
                                              const CUtensorMap* tmH = nullptr,
                                              const CUtensorMap* tmS = nullptr) {
  const int lane = threadIdx.x & 31;
  // {max_all, sum_all, max_words, sum_words} of this lane's row over the
  // warp's half of the tile (BN/2 columns)
  float4 st_stats = make_float4(-INFINITY, 0.f, -INFINITY, 0.f);
  constexpr int CH = BN / 64;                 // 32-column chunks per half
  // vectorised LSTM cell when every per-row access is 16-byte aligned
  const bool vec_cell =
      g.mode == 1 && (g.hidden % 8) == 0 && (g.ld_cin % 4) == 0 && (g.ld_cout % 4) == 0 &&
      (g.ld_h % 4) == 0 && (g.ld_res % 4) == 0 && (g.ld_add % 4) == 0 && (g.ld_hs % 8) == 0 &&
      (g.hs_plane_rows * g.ld_hs) % 8 == 0 &&
      ((reinterpret_cast<uintptr_t>(g.c_in) | reinterpret_cast<uintptr_t>(g.c_out) |
        reinterpret_cast<uintptr_t>(g.h_out) | reinterpret_cast<uintptr_t>(g.h_res) |
        reinterpret_cast<uintptr_t>(g.addend) | reinterpret_cast<uintptr_t>(g.h_split) |
        reinterpret_cast<uintptr_t>(g.bias)) % 16) == 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    const int cb = half * CH + c;
    float v[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = acc[c][j] * g.acc_scale;     // exact power of 2
    __syncwarp();
    const int nb = n0 + cb * 32;
    if (g.mode == 0 && g.bias) {
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] += (nb + j < g.n) ? __ldg(g.bias + nb + j) : 0.f;
    }
    if (g.row_stats) {
      // lane = row: online (max, sum exp) over this chunk's valid columns
      float mw = -INFINITY, ma = -INFINITY;
      float sw = 0.f, sa = 0.f;
      if (nb + 32 <= g.stats_vw) {
        // all 32 columns are words (every chunk but the row's last): the
        // word and all-output statistics coincide -- one exp per element
#pragma unroll
        for (int j = 0; j < 32; ++j) mw = fmaxf(mw, v[j]);
#pragma unroll
        for (int j = 0; j < 32; ++j) sw += __expf(v[j] - mw);
        ma = mw;
        sa = sw;
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          if (nb + j < g.n) ma = fmaxf(ma, v[j]);
          if (nb + j < g.stats_vw) mw = fmaxf(mw, v[j]);
        }
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          if (nb + j < g.n) sa += __expf(v[j] - ma);
          if (nb + j < g.stats_vw) sw += __expf(v[j] - mw);
        }
      }
      if (ma > -INFINITY) {
        const float m2 = fmaxf(st_stats.x, ma);
        st_stats.y = st_stats.y * __expf(st_stats.x - m2) + sa * __expf(ma - m2);
        st_stats.x = m2;
      }
      if (mw > -INFINITY) {
        const float m2 = fmaxf(st_stats.z, mw);
        st_stats.w = st_stats.w * __expf(st_stats.z - m2) + sw * __expf(mw - m2);
        st_stats.z = m2;
      }
      if (c & 1) {
        // one 64-column statistics group done (n0/64 + half for BN = 128); a
        // group wholly past n (the second half of the last tile when n % 128
        // <= 64) has no slot: writing it would land on the next row's group 0
        if (row0 + lane < M && n0 + (cb - 1) * 32 < g.n) {
          const int orow = g.rows ? g.rows[row0 + lane] : row0 + lane;
          const int ntiles = (g.n + 63) / 64;
          reinterpret_cast<float4*>(g.row_stats)[(int64_t)orow * ntiles + (n0 + (cb - 1) * 32) / 64] =
              st_stats;
        }
        st_stats = make_float4(-INFINITY, 0.f, -INFINITY, 0.f);
      }
    }
    // the staging buffer is about to be rewritten: the previous chunk's TMA
    // store must have read it (waited here, not right after that store, so the
    // wait overlaps this chunk's scaling / statistics and, at a tile boundary,
    // the next tile's TMEM drain)
    if (tmC || tmS) {
      if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      __syncwarp();
    }
    if constexpr (BN == 64) {
      if (g.out_logsoftmax) {
        // the whole row is this tile: lane = row, this warp holds columns
        // [32 half, 32 half + 32), the partner warp (other half) the rest.
        // Same arithmetic as log_softmax_kernel (asr.cu): per-lane partials
        // e_l + e_{l+32}, then its xor-butterfly order.
        const int q = (threadIdx.x >> 5) & 3;
        float* other = st + (half ? -4 : 4) * (32 * 33);
#pragma unroll
        for (int j = 0; j < 32; ++j) st[lane * 33 + j] = v[j];
        asm volatile("bar.sync %0, 64;" ::"r"(2 + q));
        float lo[32], hi[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          lo[j] = half ? other[lane * 33 + j] : v[j];
          hi[j] = half ? v[j] : other[lane * 33 + j];
        }
        asm volatile("bar.sync %0, 64;" ::"r"(2 + q));
        float mx = -INFINITY;
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          if (j < g.n) mx = fmaxf(mx, lo[j]);
          if (j + 32 < g.n) mx = fmaxf(mx, hi[j]);
        }
        // fp64 normaliser, the exact sum order of log_softmax_kernel: lane l's
        // e_l + e_{l+32}, then the xor butterfly -- a binary tree over the 32
        // partials in bit-reversed leaf order, merged on a 5-deep stack
        double stk[5];
#pragma unroll
        for (int k = 0; k < 32; ++k) {
          const int j = ((k & 1) << 4) | ((k & 2) << 2) | (k & 4) | ((k & 8) >> 2) | ((k & 16) >> 4);
          double d = 0.0;
          if (j < g.n) d += (double)expf(lo[j] - mx);
          if (j + 32 < g.n) d += (double)expf(hi[j] - mx);
          int depth = __popc(k) ;                      // stack height before this leaf
#pragma unroll
          for (int c = k, t = depth; c & 1; c >>= 1) d = stk[--t] + d;
          stk[__popc(k + 1) - 1] = d;
          (void)depth;
        }
        const double lse = log(stk[0]);
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = (float)((double)(v[j] - mx) - lse);
      }
    }
    if (nb >= g.n) continue;
    if (g.mode == 1 && vec_cell) {
      // lane = row and its 32 accumulator columns = 8 whole units (gates 4u+q),
      // straight from the TMEM load: vector loads/stores per row, no transpose
      const int row = row0 + lane;
      const int unit0 = nb >> 2;
      if (row < M) {
        const int slot = g.rows ? __ldg(g.rows + row) : row;
        const int pr = g.parent ? __ldg(g.parent + slot) : slot;
        float cp[8], hr[8], hv[8], cv[8];
        if (g.c_in) {
          const float4* s4 = reinterpret_cast<const float4*>(g.c_in + (int64_t)pr * g.ld_cin + unit0);
          const float4 a = __ldg(s4), b = __ldg(s4 + 1);
          cp[0] = a.x; cp[1] = a.y; cp[2] = a.z; cp[3] = a.w;
          cp[4] = b.x; cp[5] = b.y; cp[6] = b.z; cp[7] = b.w;
        } else {
#pragma unroll
          for (int u = 0; u < 8; ++u) cp[u] = 0.f;
        }
        if (g.h_res) {
          const float4* s4 = reinterpret_cast<const float4*>(g.h_res + (int64_t)slot * g.ld_res + unit0);
          const float4 a = __ldg(s4), b = __ldg(s4 + 1);
          hr[0] = a.x; hr[1] = a.y; hr[2] = a.z; hr[3] = a.w;
          hr[4] = b.x; hr[5] = b.y; hr[6] = b.z; hr[7] = b.w;
        } else {
#pragma unroll
          for (int u = 0; u < 8; ++u) hr[u] = 0.f;
        }
        // bias (+ addend) fetched per unit at its use: the bias is the same
        // for every row (L1 hits after the first warp); holding all eight
        // float4 of both beside the accumulator spilled registers
        const float4* b4p = g.bias ? reinterpret_cast<const float4*>(g.bias) + unit0 : nullptr;
        const float4* a4p = g.addend
            ? reinterpret_cast<const float4*>(g.addend + (int64_t)row * g.ld_add) + unit0 : nullptr;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          float4 b = b4p ? __ldg(b4p + u) : make_float4(0.f, 0.f, 0.f, 0.f);
          if (a4p) {
            const float4 a = __ldg(a4p + u);
            b.x += a.x; b.y += a.y; b.z += a.z; b.w += a.w;
          }
          const float gi = v[4 * u] + b.x, gf = v[4 * u + 1] + b.y;
          const float gg = v[4 * u + 2] + b.z, go = v[4 * u + 3] + b.w;
          cv[u] = fsig(gf) * cp[u] + fsig(gi) * ftanh(gg);
          hv[u] = fsig(go) * ftanh(cv[u]) + hr[u];
        }
        const bool tma = tmC && tmH && row0 + 32 <= M;   // warp-uniform; slot == row here
        if (tma) {
          // stage [32 rows][8 units] c and h tiles (and the h planes) for TMA
          float4* sc = reinterpret_cast<float4*>(st) + lane * 2;
          sc[0] = make_float4(cv[0], cv[1], cv[2], cv[3]);
          sc[1] = make_float4(cv[4], cv[5], cv[6], cv[7]);
          float4* sh = reinterpret_cast<float4*>(st + 256) + lane * 2;
          sh[0] = make_float4(hv[0], hv[1], hv[2], hv[3]);
          sh[1] = make_float4(hv[4], hv[5], hv[6], hv[7]);
        } else {
        float4* c4 = reinterpret_cast<float4*>(g.c_out + (int64_t)slot * g.ld_cout + unit0);
        c4[0] = make_float4(cv[0], cv[1], cv[2], cv[3]);
        c4[1] = make_float4(cv[4], cv[5], cv[6], cv[7]);
        float4* h4 = reinterpret_cast<float4*>(g.h_out + (int64_t)slot * g.ld_h + unit0);
        h4[0] = make_float4(hv[0], hv[1], hv[2], hv[3]);
        h4[1] = make_float4(hv[4], hv[5], hv[6], hv[7]);
        }
        if (g.h_split) {
          uint16_t pl[3][8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            uint16_t e[3];
            split_operand(hv[u], e);
#pragma unroll
            for (int q = 0; q < kPlanes; ++q) pl[q][u] = e[q];
          }
          if (tmS && row0 + 32 <= M) {
            uint4* ss = reinterpret_cast<uint4*>(st + 512);        // [planes][32 rows][16 B]
#pragma unroll
            for (int q = 0; q < kPlanes; ++q) ss[q * 32 + lane] = *reinterpret_cast<const uint4*>(pl[q]);
          } else {
          uint16_t* o = reinterpret_cast<uint16_t*>(g.h_split) +
                        (int64_t)(g.hs_row_mode ? row : slot) * g.ld_hs + unit0;
#pragma unroll
          for (int q = 0; q < kPlanes; ++q)
            *reinterpret_cast<uint4*>(o + (int64_t)q * g.hs_plane_rows * g.ld_hs) =
                *reinterpret_cast<const uint4*>(pl[q]);
          }
        }
      }
      if ((tmC && tmH) || tmS) {
       if (row0 + 32 <= M) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) {
          if (tmC && tmH) {
          asm volatile(
              "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                  tmC), "r"(unit0), "r"(row0), "r"(smem_u32(st)) : "memory");
          asm volatile(
              "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                  tmH), "r"(unit0), "r"(row0), "r"(smem_u32(st + 256)) : "memory");
          }
          if (g.h_split && tmS)
            asm volatile(
                "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];"
                ::"l"(tmS), "r"(unit0), "r"(row0), "r"(0), "r"(smem_u32(st + 512)) : "memory");
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
        __syncwarp();
       }
      }
      continue;
    }
    TRACE(8, 2 * c);
#pragma unroll
    for (int j = 0; j < 32; ++j) st[lane * 33 + j] = v[j];
    __syncwarp();
    if (g.mode == 1) {
      const int u = lane & 7, rs = lane >> 3;
      const int unit = (nb >> 2) + u;
      const bool uok = unit * 4 < g.n;
      float4 b4 = make_float4(0.f, 0.f, 0.f, 0.f);
      if (g.bias && uok) b4 = *reinterpret_cast<const float4*>(g.bias + 4 * unit);
      // gather everything the 8 rows of this lane need before any math, so the
      // dependent loads (rows -> parent -> c_in) are in flight together
      int slot[8];
      bool ok[8];
#pragma unroll
      for (int it = 0; it < 8; ++it) {
        const int row = row0 + it * 4 + rs;
        ok[it] = uok && row < M;
        slot[it] = ok[it] ? (g.rows ? __ldg(g.rows + row) : row) : 0;
      }
      int pr[8];
#pragma unroll
      for (int it = 0; it < 8; ++it) pr[it] = (ok[it] && g.parent) ? __ldg(g.parent + slot[it]) : slot[it];
      float cp[8], hr[8];
      float4 ad[8];
#pragma unroll
      for (int it = 0; it < 8; ++it) {
        cp[it] = (ok[it] && g.c_in) ? __ldg(g.c_in + (int64_t)pr[it] * g.ld_cin + unit) : 0.f;
        hr[it] = (ok[it] && g.h_res) ? __ldg(g.h_res + (int64_t)slot[it] * g.ld_res + unit) : 0.f;
        ad[it] = (ok[it] && g.addend)
                     ? __ldg(reinterpret_cast<const float4*>(
                           g.addend + (int64_t)(row0 + it * 4 + rs) * g.ld_add + 4 * unit))
                     : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int it = 0; it < 8; ++it) {
        if (!ok[it]) continue;
        const int r = it * 4 + rs;
        const float gi = st[r * 33 + 4 * u] + b4.x + ad[it].x;
        const float gf = st[r * 33 + 4 * u + 1] + b4.y + ad[it].y;
        const float gg = st[r * 33 + 4 * u + 2] + b4.z + ad[it].z;
        const float go = st[r * 33 + 4 * u + 3] + b4.w + ad[it].w;
        const float c = fsig(gf) * cp[it] + fsig(gi) * ftanh(gg);
        const float h = fsig(go) * ftanh(c) + hr[it];
        g.c_out[(int64_t)slot[it] * g.ld_cout + unit] = c;
        g.h_out[(int64_t)slot[it] * g.ld_h + unit] = h;
        if (g.h_split) store_split(g, g.hs_row_mode ? row0 + r : slot[it], unit, h);
      }
    } else if (tmC && row0 + 32 <= M) {
      // plain rows, all 32 live: the chunk leaves as one TMA tensor store
      // (the SM's store path is the epilogue's bottleneck, scripts/micro/)
      float x[32];
#pragma unroll
      for (int r = 0; r < 32; ++r) {
        x[r] = st[r * 33 + lane];
        if (g.out_exp2) x[r] = expf(2.0f * x[r]);          // == query_exp_kernel
      }
      __syncwarp();
#pragma unroll
      for (int r = 0; r < 32; ++r) st[r * 32 + lane] = x[r];     // unpadded [32][32] box
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (g.rows) {
        // gathered output rows: eight 4-row TMA scatters (box {32, 1})
        const int orow = __ldg(g.rows + row0 + lane);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int a0 = __shfl_sync(0xffffffffu, orow, 4 * q);
          const int a1 = __shfl_sync(0xffffffffu, orow, 4 * q + 1);
          const int a2 = __shfl_sync(0xffffffffu, orow, 4 * q + 2);
          const int a3 = __shfl_sync(0xffffffffu, orow, 4 * q + 3);
          if (lane == 0)
            asm volatile(
                "cp.async.bulk.tensor.2d.global.shared::cta.tile::scatter4.bulk_group "
                "[%0, {%1, %2, %3, %4, %5}], [%6];" ::"l"(tmC),
                "r"(nb), "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(smem_u32(st + q * 128))
                : "memory");
        }
      } else if (lane == 0) {
        asm volatile(
            "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                tmC),
            "r"(nb), "r"(row0), "r"(smem_u32(st))
            : "memory");
      }
      if (lane == 0) asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      __syncwarp();
    } else {
      const int col = nb + lane;
      for (int r = 0; r < 32; ++r) {
        const int row = row0 + r;
        if (row >= M) break;
        if (col < g.n) {
          float x = st[r * 33 + lane];
          if (g.addend) x += g.addend[(int64_t)row * g.ld_add + col];
          if (g.out_exp2) x = expf(2.0f * x);          // == query_exp_kernel
          const int orow = g.rows ? g.rows[row] : row;
          g.c[(int64_t)orow * g.ldc + col] = x;
        }
      }
      TRACE(8, 2 * c + 1);
    }
  }
  __syncwarp();
}

// Work decomposition of one launch.  Plain: CTA b takes tiles b, b+G, ...
// whole K.  Stream-K (g.splitk_ws set and fewer tiles than CTAs): the
// tile x K-block space [0, tiles*num_kb) is cut into `ctas` equal ranges, CTA b
// taking range b -- up to one partial segment at each end plus whole tiles in
// between.  Every role (TMA, MMA, epilogue) walks the same segment list.
struct TcWork {
  int num_tiles, num_kb, ctas, lo, hi;
  bool sk;
  __device__ __forceinline__ int owner(int64_t p) const {   // CTA whose range holds p
    const int64_t total = (int64_t)num_tiles * num_kb;
    return (int)(((p + 1) * ctas - 1) / total);
  }
  __device__ __forceinline__ int range_lo(int c) const {
    return (int)((int64_t)c * num_tiles * num_kb / ctas);
  }
  // i-th segment of this CTA: tile, K blocks [kb_lo, kb_hi)
  __device__ __forceinline__ bool seg(int i, int& tile, int& kb_lo, int& kb_hi) const {
    if (!sk) {
      tile = (int)blockIdx.x + i * (int)gridDim.x;
      kb_lo = 0;
      kb_hi = num_kb;
      return tile < num_tiles;
    }
    const int t0 = lo / num_kb;
    tile = t0 + i;
    const int s0 = tile * num_kb;
    if (s0 + (i == 0 ? lo - s0 : 0) >= hi) return false;
    kb_lo = i == 0 ? lo - s0 : 0;
    kb_hi = min(num_kb, hi - s0);
    return true;
  }
};

constexpr int TC_SK_MIN_KB = 8;      // stream-K: at least 8 K blocks (K = 512) per CTA

// Persistent, warp-specialized: warp 0 = TMA producer, warp 1 = MMA issuer
// (+ TMEM owner), warps 2..5 = epilogue.  Two TMEM accumulators (2 x BN
// columns) let the epilogue of tile i overlap the MMAs of tile i+1.  The tile
// count follows the device-side row count, so graph replays with few live rows
// cost only the tiles they need.
template <int BN>
__global__ void __launch_bounds__(TC_THREADS, 1)   // 10 warps: <= 168 registers (3 warps per SMSP)
gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmW,
               const __grid_constant__ CUtensorMap tmC, const __grid_constant__ CUtensorMap tmH,
               const __grid_constant__ CUtensorMap tmS, int tma_c,
               fb_gemm_t g, int a_planes, int a_plane_rows, int num_kb, int kcb) {
  constexpr int NACC = TC_NACC;
  constexpr int GRP = FB_GEMM_GROUP;         // accumulation chunks per TMEM handshake
  constexpr int NGRP = NACC / GRP;
  static_assert(NACC % GRP == 0, "slot groups must tile the TMEM slots");
  constexpr int STAGES = tc_stages(BN);
  pdl_entry();
  const int M = row_count(g.m_max, g.m_dev);
  const int m_tiles = (M + TC_BM - 1) / TC_BM;
  const int n_tiles = (g.n + BN - 1) / BN;
  const int num_tiles = m_tiles * n_tiles;
  TcWork wk;
  wk.num_tiles = num_tiles;
  wk.num_kb = num_kb;
  wk.sk = g.splitk_ws != nullptr && num_tiles < (int)gridDim.x;
  if (wk.sk) {
    wk.ctas = min((int)gridDim.x, max(num_tiles, num_tiles * num_kb / TC_SK_MIN_KB));
    wk.sk = wk.ctas > num_tiles;
  }
  if (!wk.sk) wk.ctas = num_tiles;
  if ((int)blockIdx.x >= wk.ctas) return;
  wk.lo = wk.range_lo(blockIdx.x);
  wk.hi = wk.range_lo(blockIdx.x + 1);

  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* base = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  constexpr int A_TILE = TC_BM * TC_BK * 2;         // 16 KB
  constexpr int W_TILE = BN * TC_BK * 2;
  const int stage_bytes = a_planes * A_TILE + W_TILE;
  __shared__ __align__(8) uint64_t bar_full[STAGES], bar_empty[STAGES];
  __shared__ __align__(8) uint64_t bar_tfull[NACC], bar_tempty[NACC];
  __shared__ uint32_t tmem_base_sh;
  __shared__ int sk_last_sh;
  __shared__ __align__(128) float epi_stage[8][32 * 33];   // 33 * 128 B per warp

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(smem_u32(&bar_full[s]), 1);
      mbar_init(smem_u32(&bar_empty[s]), 1);
    }
    for (int a = 0; a < NACC; ++a) {
      mbar_init(smem_u32(&bar_tfull[a]), 1);
      mbar_init(smem_u32(&bar_tempty[a]), TC_EPI_THREADS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tmem_base_sh)),
                 "r"(NACC * BN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base_sh;

  if (warp == 0) {
    // ---- TMA producer: lane p issues A plane p, lane a_planes the W tile ----
    int gk = 0, tile, kb_lo, kb_hi;
    for (int si = 0; wk.seg(si, tile, kb_lo, kb_hi); ++si) {
      const int m0 = (tile % m_tiles) * TC_BM, n0 = (tile / m_tiles) * BN;
      for (int kb = kb_lo; kb < kb_hi; ++kb, ++gk) {
        const int s = gk % STAGES;
        const uint32_t ph = (gk / STAGES) & 1;
        TRACE(0, gk);
        if (lane == 0) {
          mbar_wait(smem_u32(&bar_empty[s]), ph ^ 1);
          mbar_expect_tx(smem_u32(&bar_full[s]), stage_bytes);
        }
        TRACE(1, gk);
        __syncwarp();
        const uint32_t full = smem_u32(&bar_full[s]);
        unsigned char* st = base + (size_t)s * stage_bytes;
        if (lane < a_planes)
          tma_load_2d(smem_u32(st + lane * A_TILE), &tmA, full, kb * TC_BK,
                      lane * a_plane_rows + m0);
        else if (lane == a_planes)
          tma_load_2d(smem_u32(st + a_planes * A_TILE), &tmW, full, kb * TC_BK, n0);
      }
    }
  } else if (warp == 1) {
    {
      // ---- MMA issuer: bf16 x bf16 -> f32, K-major, M = 128, N = BN ----
      const uint32_t idesc = kIdescAB | (1u << 4) | ((uint32_t)(BN >> 3) << 17) |
                             ((uint32_t)(TC_BM >> 4) << 24);
      int gk = 0, gc = 0, tile, kb_lo, kb_hi;
      for (int si = 0; wk.seg(si, tile, kb_lo, kb_hi); ++si) {
        const int nch = (kb_hi - kb_lo + kcb - 1) / kcb;
        for (int c0 = 0; c0 < nch; c0 += GRP, ++gc) {
          // a group of GRP chunks: one slot-group wait and one commit (the
          // per-chunk handshake, not the MMAs, paced 64-K chunks)
          const int grp = gc % NGRP;
          mbar_wait(smem_u32(&bar_tempty[grp]), ((gc / NGRP) & 1) ^ 1);
          asm volatile("tcgen05.fence::after_thread_sync;");
          for (int j = 0; j < GRP && c0 + j < nch; ++j) {
          const uint32_t d = tmem + (grp * GRP + j) * BN;
          const int kb0 = kb_lo + (c0 + j) * kcb;
          const int kb1 = min(kb0 + kcb, kb_hi);
          for (int kb = kb0; kb < kb1; ++kb, ++gk) {
            const int s = gk % STAGES;
            const uint32_t ph = (gk / STAGES) & 1;
            TRACE(2, gk);
            mbar_wait(smem_u32(&bar_full[s]), ph);
            TRACE(3, gk);
            asm volatile("tcgen05.fence::after_thread_sync;");
            unsigned char* st = base + (size_t)s * stage_bytes;
            const uint64_t bdesc0 = smem_desc_sw128(smem_u32(st + a_planes * A_TILE));
            // smallest plane first: lo/mid products are summed while the
            // accumulator is still small, so its rounding loses less of them
            for (int p = a_planes - 1; p >= 0; --p) {
              const uint64_t adesc0 = smem_desc_sw128(smem_u32(st + p * A_TILE));
#pragma unroll
              for (int k = 0; k < TC_BK / 16; ++k) {  // 16 elements = 32 B per UMMA_K
#ifdef FB_GEMM_NOMMA
                if (kb != kb0 || p != a_planes - 1 || k != 0) continue;   // dev: feed-only timing
#endif
                mma_bf16_elect(d, adesc0 + 2 * k, bdesc0 + 2 * k, idesc,
                         ((kb - kb0) | (a_planes - 1 - p) | k) != 0);
              }
            }
            mma_commit_elect(smem_u32(&bar_empty[s]));
            TRACE(4, gk);
          }
          }
          mma_commit_elect(smem_u32(&bar_tfull[grp]));
        }
      }
    }
  } else {
    // ---- epilogue warps 2..9: lane quarter = warp % 4, column half = (warp-2)/4 ----
    const int quarter = warp & 3;
    const int half = (warp - 2) >> 2;
    constexpr int CH = BN / 64;
    const uint32_t tl = tmem + ((uint32_t)(quarter * 32) << 16);
    int gc = 0, tile, kb_lo, kb_hi;
    for (int si = 0; wk.seg(si, tile, kb_lo, kb_hi); ++si) {
      const int m0 = (tile % m_tiles) * TC_BM, n0 = (tile / m_tiles) * BN;
      float acc[CH][32];
      const int nch = (kb_hi - kb_lo + kcb - 1) / kcb;
      for (int c0 = 0; c0 < nch; c0 += GRP, ++gc) {
        const int grp = gc % NGRP;
        mbar_wait(smem_u32(&bar_tfull[grp]), (gc / NGRP) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
        for (int j = 0; j < GRP && c0 + j < nch; ++j) {
        const int slot = grp * GRP + j;
        const bool first = c0 + j == 0;
        if constexpr (CH == 2) {
          // both 32-column chunks in flight before one wait::ld (the drain
          // runs once per accumulation chunk, so its latency matters)
          uint32_t r[64];
          tmem_ld64_nowait(tl + slot * BN + half * 64, r);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
          for (int c = 0; c < 2; ++c)
#pragma unroll
            for (int jj = 0; jj < 32; ++jj)
              acc[c][jj] = first ? __uint_as_float(r[c * 32 + jj])
                                 : acc[c][jj] + __uint_as_float(r[c * 32 + jj]);
        } else {
#pragma unroll
          for (int c = 0; c < CH; ++c) {
            float v[32];
            tmem_ld32(tl + slot * BN + (half * CH + c) * 32, v);
            if (first) {
#pragma unroll
              for (int jj = 0; jj < 32; ++jj) acc[c][jj] = v[jj];
            } else {
#pragma unroll
              for (int jj = 0; jj < 32; ++jj) acc[c][jj] += v[jj];
            }
          }
        }
        }
        asm volatile("tcgen05.fence::before_thread_sync;");
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&bar_tempty[grp]))
                     : "memory");
        TRACE(9, gc);
      }
      TRACE(5, si);
      if (wk.sk) {
        const int c0 = wk.owner((int64_t)tile * num_kb);
        const int c1 = wk.owner((int64_t)(tile + 1) * num_kb - 1);
        if (c0 != c1) {
          // partial tile: publish, count arrivals; the last CTA sums the
          // partials in K order (c0..c1) -- the same result whoever is last
          constexpr int WS_WARP = CH * 32 * 32;
          auto slot_of = [&](int cta) {
            return 2 * cta + (tile == wk.range_lo(cta) / num_kb ? 0 : 1);
          };
          float* mine = g.splitk_ws + (size_t)slot_of(blockIdx.x) * (8 * WS_WARP) +
                        (warp - 2) * WS_WARP + lane;
#pragma unroll
          for (int c = 0; c < CH; ++c)
#pragma unroll
            for (int j = 0; j < 32; ++j) __stcg(mine + (c * 32 + j) * 32, acc[c][j]);
          __threadfence();
          asm volatile("bar.sync 1, %0;" ::"n"(TC_EPI_THREADS));
          if (threadIdx.x == 64) {
            const unsigned old = atomicAdd(&g.splitk_cnt[tile], 1u);
            const int last = old == (unsigned)(c1 - c0);
            if (last) atomicExch(&g.splitk_cnt[tile], 0u);
            sk_last_sh = last;
          }
          asm volatile("bar.sync 1, %0;" ::"n"(TC_EPI_THREADS));
          if (!sk_last_sh) continue;
          __threadfence();
          // (own partial re-read too: the sum order must not depend on who is last)
          for (int cta = c0; cta <= c1; ++cta) {
            const float* src = g.splitk_ws + (size_t)slot_of(cta) * (8 * WS_WARP) +
                               (warp - 2) * WS_WARP + lane;
#pragma unroll
            for (int c = 0; c < CH; ++c)
#pragma unroll
              for (int j = 0; j < 32; ++j) {
                const float v = __ldcg(src + (c * 32 + j) * 32);
                acc[c][j] = cta == c0 ? v : acc[c][j] + v;
              }
          }
        }
      }
      TRACE(6, si);
      epilogue_tile<BN>(g, M, m0 + quarter * 32, n0, acc, epi_stage[warp - 2], half,
                        (tma_c == 1 || tma_c == 2) ? &tmC : nullptr,
                        tma_c == 2 ? &tmH : nullptr,
                        (tma_c == 2 || tma_c == 3) && g.h_split ? &tmS : nullptr);
      TRACE(7, si);
    }
    // the TMA stores' global writes complete before the CTA retires
    if (tma_c && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(NACC * BN));
  }
}

// Encoder LSTM recurrence as ONE persistent launch per direction (PAPER.md:
// 105-110): CTA = fixed (m-tile, n-tile) of gates = xp[:, t] + h_{t-1} W_hh^T,
// looping over t with a grid barrier between steps (a cooperative launch: all
// CTAs co-resident, one per SM).  The CTA's W_hh slice (128 gate rows x K) is
// loaded into shared memory ONCE and stays resident for all steps; only the
// previous step's h planes stream through the A ring.  The dedicated cell
// epilogue writes h -> y and -> the next step's operand planes.
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ unsigned ld_relaxed_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
#ifndef FB_REC_POLL
#define FB_REC_POLL 0        // barrier poll: 0 acquire + nanosleep, 1 acquire spin, 2 relaxed spin + fence
#endif

constexpr int REC_MAX_STAGES = 4;
#ifndef FB_REC_SYNC_STRIDE
#define FB_REC_SYNC_STRIDE 32
#endif
// one 128-byte line per row tile's step counter (its 10 CTAs' atomics and
// polls do not contend with the other tiles')
constexpr int kRecSyncStride = FB_REC_SYNC_STRIDE;
#ifndef FB_REC_EARLY_PUB
#define FB_REC_EARLY_PUB 1   // publish h planes before storing the fp32 output
#endif
#ifndef FB_REC_XA_AFTER_PASS
#define FB_REC_XA_AFTER_PASS 1   // input-projection loads wait for the step barrier
#endif
#ifndef FB_REC_PF
#define FB_REC_PF 1          // L2 prefetch of the next step's input projection
#endif
#ifndef FB_REC_CELL7
#define FB_REC_CELL7 1       // LSTM cell with 5 ex2 + 2 rcp (instead of 5 + 5)
#endif

// LSTM cell sharing reciprocals: with e_i = exp(-i), e_f = exp(-f),
// E_g = exp(2g),  c' = c sig(f) + sig(i) tanh(g)
//   = [c (1+e_i)(1+E_g) + (E_g-1)(1+e_f)] / [(1+e_f)(1+e_i)(1+E_g)],
// h = sig(o) tanh(c') = (E_c-1) / [(1+e_o)(1+E_c)], E_c = exp(2c').
// Arguments are clamped where the functions are saturated in fp32 (sigmoid
// below 1e-13, |tanh| within 3e-8 of 1) so the products stay below 1e34.
__device__ __forceinline__ void rec_cell(float gi, float gf, float gg, float go, float& c,
                                         float& h) {
  const float ei = __expf(-fmaxf(gi, -30.f)), ef = __expf(-fmaxf(gf, -30.f));
  const float eg = __expf(2.f * fminf(fmaxf(gg, -9.f), 9.f));
  const float pi = 1.f + ei, pg = 1.f + eg, pf = 1.f + ef;
  const float pig = pi * pg;
  c = __fdividef(fmaf(c, pig, (eg - 1.f) * pf), pig * pf);
  const float eo = __expf(-fmaxf(go, -30.f));
  const float ec = __expf(2.f * fminf(fmaxf(c, -9.f), 9.f));
  const float pc = 1.f + ec;
  h = __fdividef(ec - 1.f, (1.f + eo) * pc);
}

__global__ void __launch_bounds__(TC_THREADS, 1)
lstm_rec_kernel(const __grid_constant__ CUtensorMap tmA0, const __grid_constant__ CUtensorMap tmA1,
                const __grid_constant__ CUtensorMap tmW, fb_gemm_t g0, int steps, int num_kb,
                int kcb, const float* xp, int64_t step_xp, float* y, int64_t ld_y,
                int64_t step_y, uint16_t* rec, int64_t plane, unsigned* sync, int nst,
                const int32_t* t_rev, int wide) {
  constexpr int BN = 128;
  const int batch = g0.m_max;
  const int m_tiles = (batch + TC_BM - 1) / TC_BM;
  // rows of different m-tiles never interact: each m-tile's n-tile CTAs
  // synchronise among themselves (one counter per m-tile), not grid-wide
  const int n_peers = gridDim.x / m_tiles;
  unsigned* msync = sync + (blockIdx.x % m_tiles) * kRecSyncStride;
  const int tile = blockIdx.x;
  const int m0 = (tile % m_tiles) * TC_BM, n0 = (tile / m_tiles) * BN;

  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* base = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  constexpr int A_TILE = TC_BM * TC_BK * 2;
  constexpr int W_TILE = BN * TC_BK * 2;
  constexpr int stage_bytes = kPlanes * A_TILE;          // A planes only
  unsigned char* wres = base;                             // resident W_hh: num_kb tiles
  unsigned char* ring = base + (size_t)num_kb * W_TILE;
  __shared__ __align__(8) uint64_t bar_full[REC_MAX_STAGES], bar_empty[REC_MAX_STAGES];
  __shared__ __align__(8) uint64_t bar_tfull[TC_NACC], bar_tempty[TC_NACC], bar_w, bar_pass;
  __shared__ uint32_t tmem_base_sh;
#if FB_REC_POLL == 3
  __shared__ __align__(8) uint64_t bar_poll;
  __shared__ __align__(16) unsigned poll_buf[4];
  uint32_t poll_ph = 0;
#endif

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < nst; ++s) {
      mbar_init(smem_u32(&bar_full[s]), 1);
      mbar_init(smem_u32(&bar_empty[s]), 1);
    }
    mbar_init(smem_u32(&bar_w), 1);
    mbar_init(smem_u32(&bar_pass), 1);
#if FB_REC_POLL == 3
    mbar_init(smem_u32(&bar_poll), 1);
#endif
    for (int a = 0; a < TC_NACC; ++a) {
      mbar_init(smem_u32(&bar_tfull[a]), 1);
      mbar_init(smem_u32(&bar_tempty[a]), TC_EPI_THREADS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tmem_base_sh)),
                 "r"(TC_NACC * BN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base_sh;

  if (warp == 0) {
    if (lane == 0) {
      // the CTA's W_hh slice, once
      mbar_expect_tx(smem_u32(&bar_w), (uint32_t)(num_kb * W_TILE));
      for (int kb = 0; kb < num_kb; ++kb)
        tma_load_2d(smem_u32(wres + (size_t)kb * W_TILE), &tmW, smem_u32(&bar_w), kb * TC_BK, n0);
      int gk = 0;
      for (int t = 0; t < steps; ++t) {
        // h_{t-1} complete in every CTA (grid barrier), then visible to TMA
        const unsigned target = (unsigned)(n_peers * t);
        TRACE(0, t);
        TRACE_CTA(6, t, 101);
#if FB_REC_POLL == 3
        // poll through the TMA unit (async proxy, L2): the epilogue warps'
        // input-projection loads fill the SM's load queue at this moment, and
        // a generic load of the counter waits behind them for microseconds
        for (;;) {
          mbar_expect_tx(smem_u32(&bar_poll), 16);
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 16, [%2];"
              ::"r"(smem_u32(poll_buf)), "l"(msync), "r"(smem_u32(&bar_poll)) : "memory");
          mbar_wait(smem_u32(&bar_poll), poll_ph);
          poll_ph ^= 1;
          if (*reinterpret_cast<volatile unsigned*>(poll_buf) >= target) break;
        }
#elif FB_REC_POLL == 1
        while (ld_acquire_u32(msync) < target) {}
#elif FB_REC_POLL == 2
        while (ld_relaxed_u32(msync) < target) {}
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
#else
        while (ld_acquire_u32(msync) < target) __nanosleep(32);
#endif
        TRACE(1, t);
        TRACE_CTA(7, t, 101);
#if FB_REC_XA_AFTER_PASS
        // step t's barrier passed: the epilogue may now load its input
        // projection (overlapping the A loads and the MMA, not the poll)
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&bar_pass)) : "memory");
#endif
#ifdef FB_GEMM_TRACE
        if (t == 101) {
          unsigned smid;
          asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
          g_trace[8][blockIdx.x] = smid;
        }
#endif
        asm volatile("fence.proxy.async.global;" ::: "memory");
        const CUtensorMap* tmA = (t & 1) ? &tmA1 : &tmA0;
        for (int kb = 0; kb < num_kb; ++kb, ++gk) {
          const int s = gk % nst;
          const uint32_t ph = (gk / nst) & 1;
          mbar_wait(smem_u32(&bar_empty[s]), ph ^ 1);
          const uint32_t full = smem_u32(&bar_full[s]);
          mbar_expect_tx(full, stage_bytes);
          unsigned char* st = ring + (size_t)s * stage_bytes;
          for (int p = 0; p < kPlanes; ++p)
            tma_load_2d(smem_u32(st + p * A_TILE), tmA, full, kb * TC_BK, p * batch + m0);
        }
      }
    }
  } else if (warp == 1) {
    {
      const uint32_t idesc = kIdescAB | (1u << 4) | ((uint32_t)(BN >> 3) << 17) |
                             ((uint32_t)(TC_BM >> 4) << 24);
      int gk = 0, cc = 0;
      mbar_wait(smem_u32(&bar_w), 0);
      for (int t = 0; t < steps; ++t) {
        for (int kb0 = 0; kb0 < num_kb; kb0 += kcb, ++cc) {
          const int slot = cc % TC_NACC;
          mbar_wait(smem_u32(&bar_tempty[slot]), ((cc / TC_NACC) & 1) ^ 1);
          asm volatile("tcgen05.fence::after_thread_sync;");
          const uint32_t d = tmem + slot * BN;
          const int kb1 = min(kb0 + kcb, num_kb);
          for (int kb = kb0; kb < kb1; ++kb, ++gk) {
            const int s = gk % nst;
            const uint32_t ph = (gk / nst) & 1;
            mbar_wait(smem_u32(&bar_full[s]), ph);
            asm volatile("tcgen05.fence::after_thread_sync;");
            unsigned char* st = ring + (size_t)s * stage_bytes;
            const uint64_t bdesc0 = smem_desc_sw128(smem_u32(wres + (size_t)kb * W_TILE));
            for (int p = kPlanes - 1; p >= 0; --p) {
              const uint64_t adesc0 = smem_desc_sw128(smem_u32(st + p * A_TILE));
#pragma unroll
              for (int k = 0; k < TC_BK / 16; ++k)
                mma_bf16_elect(d, adesc0 + 2 * k, bdesc0 + 2 * k, idesc,
                               ((kb - kb0) | (kPlanes - 1 - p) | k) != 0);
            }
            mma_commit_elect(smem_u32(&bar_empty[s]));
          }
          mma_commit_elect(smem_u32(&bar_tfull[slot]));
        }
      }
    }
  } else {
    // dedicated cell epilogue: lane = row, 16 units per warp half; the cell
    // state stays in registers across steps and the step's input projection
    // is fetched before the accumulator is ready (off the MMA critical path)
    const int quarter = warp & 3;
    const int half = (warp - 2) >> 2;
    const uint32_t tl = tmem + ((uint32_t)(quarter * 32) << 16);
    const int row = m0 + quarter * 32 + lane;
    const bool ok = row < batch;
    // backward direction: step t of row b reads / writes frame T_b - 1 - t
    // (frames past T_b map to themselves: the reversal is a per-row permutation)
    const int t_row = (t_rev && ok) ? t_rev[row] : 0;
    const int unitb = (n0 >> 2) + half * 16;
    float cst[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) cst[u] = 0.f;
    int cc = 0;
    for (int t = 0; t < steps; ++t) {
      float4 xa[16];
#if FB_REC_XA_AFTER_PASS
      mbar_wait(smem_u32(&bar_pass), t & 1);
#endif
      const float4* xr =
          reinterpret_cast<const float4*>(xp + (int64_t)(t < t_row ? t_row - 1 - t : t) * step_xp +
                                          (int64_t)(ok ? row : 0) * g0.ld_add) +
          unitb;
      if (wide & 1) {
        // 256-bit loads (sm_100): each lane is a different row, so every load
        // instruction costs the L1 one request per lane; half the instructions
        // halve this step's request burst (which also delays the barrier poll)
#pragma unroll
        for (int u = 0; u < 16; u += 2)
          asm volatile("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                       : "=f"(xa[u].x), "=f"(xa[u].y), "=f"(xa[u].z), "=f"(xa[u].w),
                         "=f"(xa[u + 1].x), "=f"(xa[u + 1].y), "=f"(xa[u + 1].z), "=f"(xa[u + 1].w)
                       : "l"(xr + u));
      } else {
#pragma unroll
        for (int u = 0; u < 16; ++u) xa[u] = __ldg(xr + u);
      }
      // K in chunks of kcb blocks, each in its own TMEM slot, summed here with
      // round-to-nearest adds (the in-TMEM adds truncate: a whole-K slot
      // biases every gate pre-activation toward zero).  The input projection
      // joins the first chunk (divided by the exact power-of-two scale), so
      // its registers are free before the remaining chunks arrive.
      const float sc = g0.acc_scale, inv_sc = 1.0f / sc;
      float acc[2][32];
      {
        // chunk 0 (+ the input projection)
        const int slot = cc % TC_NACC;
        mbar_wait(smem_u32(&bar_tfull[slot]), (cc / TC_NACC) & 1);
        ++cc;
        asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          float v[32];
          tmem_ld32(tl + slot * BN + (half * 2 + c) * 32, v);
#pragma unroll
          for (int u8 = 0; u8 < 8; ++u8) {
            const float4 x4 = xa[c * 8 + u8];
            acc[c][4 * u8] = v[4 * u8] + x4.x * inv_sc;
            acc[c][4 * u8 + 1] = v[4 * u8 + 1] + x4.y * inv_sc;
            acc[c][4 * u8 + 2] = v[4 * u8 + 2] + x4.z * inv_sc;
            acc[c][4 * u8 + 3] = v[4 * u8 + 3] + x4.w * inv_sc;
          }
        }
        asm volatile("tcgen05.fence::before_thread_sync;");
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&bar_tempty[slot]))
                     : "memory");
      }
      for (int kb0 = kcb; kb0 < num_kb; kb0 += kcb) {
        const int slot = cc % TC_NACC;
        mbar_wait(smem_u32(&bar_tfull[slot]), (cc / TC_NACC) & 1);
        ++cc;
        asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          float v[32];
          tmem_ld32(tl + slot * BN + (half * 2 + c) * 32, v);
#pragma unroll
          for (int j = 0; j < 32; ++j) acc[c][j] += v[j];
        }
        asm volatile("tcgen05.fence::before_thread_sync;");
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&bar_tempty[slot]))
                     : "memory");
      }
      TRACE(2, t);
#if FB_REC_PF
      // next step's input projection into L2 now: the fetch from HBM overlaps
      // this step's cell / publish / barrier, and the loads at the top of the
      // next step hit L2 -- a burst of HBM misses there delays the barrier
      // poll's reply for microseconds (prefetches return no data to the SM)
      if (t + 1 < steps && ok) {
        const char* nx = reinterpret_cast<const char*>(
            xp + (int64_t)(t + 1 < t_row ? t_row - 2 - t : t + 1) * step_xp + (int64_t)row * g0.ld_add +
            4 * unitb);
        asm volatile("prefetch.global.L2 [%0];" ::"l"(nx));
        asm volatile("prefetch.global.L2 [%0];" ::"l"(nx + 128));
      }
#endif
      float hv[16];
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const float* v = acc[c];
#pragma unroll
        for (int u8 = 0; u8 < 8; ++u8) {
          const int u = c * 8 + u8;
          const float gi = v[4 * u8] * sc, gf = v[4 * u8 + 1] * sc;
          const float gg = v[4 * u8 + 2] * sc, go = v[4 * u8 + 3] * sc;
#if FB_REC_CELL7
          rec_cell(gi, gf, gg, go, cst[u], hv[u]);
#else
          cst[u] = fsig(gf) * cst[u] + fsig(gi) * ftanh(gg);
          hv[u] = fsig(go) * ftanh(cst[u]);
#endif
        }
      }
      float* yrow = y + (int64_t)(t < t_row ? t_row - 1 - t : t) * step_y + (int64_t)row * ld_y + unitb;
#if !FB_REC_EARLY_PUB
      if (ok) {
        float4* yo = reinterpret_cast<float4*>(yrow);
#pragma unroll
        for (int q = 0; q < 4; ++q)
          yo[q] = make_float4(hv[4 * q], hv[4 * q + 1], hv[4 * q + 2], hv[4 * q + 3]);
      }
#endif
      if (ok) {
        uint16_t pl[3][16];
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          uint16_t e[3];
          split_operand(hv[u], e);
#pragma unroll
          for (int q = 0; q < kPlanes; ++q) pl[q][u] = e[q];
        }
        uint16_t* o = rec + (int64_t)((t & 1) ^ 1) * kPlanes * plane + (int64_t)row * g0.ld_hs + unitb;
#pragma unroll
        for (int q = 0; q < kPlanes; ++q) {
          if (wide & 4) {
            const uint32_t* w = reinterpret_cast<const uint32_t*>(&pl[q][0]);
            asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(o + (int64_t)q * plane),
                         "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]),
                         "r"(w[7]) : "memory");
          } else {
            uint4* d = reinterpret_cast<uint4*>(o + (int64_t)q * plane);
            d[0] = *reinterpret_cast<const uint4*>(&pl[q][0]);
            d[1] = *reinterpret_cast<const uint4*>(&pl[q][8]);
          }
        }
      }
      TRACE(4, t);
      // publish h_t: every epilogue thread's stores, then one release-increment
      __threadfence();
      TRACE(5, t);
      asm volatile("bar.sync 1, %0;" ::"n"(TC_EPI_THREADS));
      if (warp == 2 && lane == 0) {
        asm volatile("fence.proxy.async.global;" ::: "memory");
        atomicAdd(msync, 1u);
        TRACE_CTA(9, t, 100);
      }
      TRACE(3, t);
#if FB_REC_EARLY_PUB
      // the fp32 output is not read by the peers: stored after the publish
      if (ok && (wide & 2)) {
#pragma unroll
        for (int q = 0; q < 16; q += 8)
          asm volatile("st.global.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(yrow + q),
                       "f"(hv[q]), "f"(hv[q + 1]), "f"(hv[q + 2]), "f"(hv[q + 3]), "f"(hv[q + 4]),
                       "f"(hv[q + 5]), "f"(hv[q + 6]), "f"(hv[q + 7]) : "memory");
      } else if (ok) {
        float4* yo = reinterpret_cast<float4*>(yrow);
#pragma unroll
        for (int q = 0; q < 4; ++q)
          yo[q] = make_float4(hv[4 * q], hv[4 * q + 1], hv[4 * q + 2], hv[4 * q + 3]);
      }
#endif
    }
  }
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(TC_NACC * BN));
  }
}

// ---- host: tensor maps through the driver entry point (no -lcuda needed) ----
static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

constexpr CUtensorMapDataType kOperandMapType =
    FB_OPERAND_FP16X2 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;

static int make_map(CUtensorMap* m, const void* ptr, uint64_t rows, uint64_t cols, uint64_t ld,
                    uint32_t box_rows) {
  auto enc = get_encode();
  if (!enc) return fail(FB_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {ld * 2};
  cuuint32_t box[2] = {TC_BK, box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(m, kOperandMapType, 2, const_cast<void*>(ptr), dims, strides,
                   box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(FB_ERR_VALUE, "cuTensorMapEncodeTiled failed (alignment?)");
  return FB_OK;
}

// fp32 output map for the epilogue's TMA stores: 32 x 32 boxes, no swizzle
static int make_map_c(CUtensorMap* m, const fb_gemm_t* g) {
  auto enc = get_encode();
  if (!enc) return fail(FB_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  // gathered rows (g->rows) go out as 4-row scatters: box {32, 1}, and the row
  // extent is the caller's contract on rows[] (no clipping needed)
  cuuint64_t dims[2] = {(cuuint64_t)g->n, g->rows ? (cuuint64_t)1 << 24 : (cuuint64_t)g->m_max};
  cuuint64_t strides[1] = {(cuuint64_t)g->ldc * 4};
  cuuint32_t box[2] = {32, g->rows ? 1u : 32u};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, g->c, dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? FB_OK : FB_ERR_VALUE;
}

// LSTM-cell outputs (mode 1, rows in GEMM order): c/h fp32 [rows][hidden]
// boxes of 8 units x 32 rows; h planes bf16 [3][plane rows][hidden] boxes
static int make_map_2d(CUtensorMap* m, CUtensorMapDataType dt, int esize, const void* p,
                       uint64_t cols, uint64_t rows, uint64_t ld) {
  auto enc = get_encode();
  if (!enc) return FB_ERR_CUDA;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {ld * esize};
  cuuint32_t box[2] = {8, 32};
  cuuint32_t es[2] = {1, 1};
  return enc(m, dt, 2, const_cast<void*>(p), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS ? FB_OK : FB_ERR_VALUE;
}

static int make_map_planes(CUtensorMap* m, const fb_gemm_t* g) {
  auto enc = get_encode();
  if (!enc) return FB_ERR_CUDA;
  cuuint64_t dims[3] = {(cuuint64_t)g->hidden, (cuuint64_t)g->hs_plane_rows, (cuuint64_t)kPlanes};
  cuuint64_t strides[2] = {(cuuint64_t)g->ld_hs * 2, (cuuint64_t)g->hs_plane_rows * g->ld_hs * 2};
  cuuint32_t box[3] = {8, 32, (cuuint32_t)kPlanes};
  cuuint32_t es[3] = {1, 1, 1};
  return enc(m, kOperandMapType, 3, g->h_split, dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
             CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS
             ? FB_OK : FB_ERR_VALUE;
}

template <int BN>
static int launch_tc_maps(const CUtensorMap& ta, const CUtensorMap& tw, const fb_gemm_t* g,
                          int a_planes, int64_t a_plane_rows, cudaStream_t s) {
  const int stage_bytes = a_planes * TC_BM * TC_BK * 2 + BN * TC_BK * 2;
  const size_t smem = (size_t)tc_stages(BN) * stage_bytes + 1024;
  auto k = gemm_tc_kernel<BN>;
  static size_t smem_set = 0;                       // set once (graph-capture safe)
  if (smem > smem_set) {
    const int full = tc_stages(BN) * (kPlanes * TC_BM * TC_BK * 2 + BN * TC_BK * 2) + 1024;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, full);
    smem_set = full;
  }
  const int tiles = ((g->m_max + TC_BM - 1) / TC_BM) * ((g->n + BN - 1) / BN);
  static const int kcb_env = [] {                   // dev override of the default
    const char* e = getenv("FB_GEMM_KCB");
    return e ? std::max(1, atoi(e)) : TC_KCB;
  }();
  const int kcb = g->kcb > 0 ? g->kcb : kcb_env;
  const int grid = g->splitk_ws ? kNumSMs : std::min(tiles, kNumSMs);
  // plain fp32 rows (no gather, no fused transform): TMA stores
#ifndef FB_NO_TMA_STORE
  // bit 0: plain fp32 tiles, bit 1: LSTM-cell outputs (dev override FB_GEMM_TMA_STORE)
  static const int tma_env = getenv("FB_GEMM_TMA_STORE") ? atoi(getenv("FB_GEMM_TMA_STORE")) : 15;
  // bit 2: the h planes of row-gathered LSTM cells, bit 3: gathered plain rows (TMA scatter4)
#else
  static const int tma_env = 0;
#endif
  CUtensorMap tc = ta, th = ta, ts = ta;
  int tma_c = (tma_env & 1) && g->mode == 0 && (!g->rows || (tma_env & 8)) && !g->addend &&
              (g->ldc % 4) == 0 && ((uintptr_t)g->c % 16) == 0;
  if (tma_c && make_map_c(&tc, g) != FB_OK) tma_c = 0;
  // LSTM cell with rows in GEMM order (the word LM): c, h and h planes by TMA
  const bool a16 = ((uintptr_t)g->c_out % 16) == 0 && ((uintptr_t)g->h_out % 16) == 0 &&
                   (g->ld_cout % 4) == 0 && (g->ld_h % 4) == 0 && (g->hidden % 8) == 0;
  const bool s16 = !g->h_split || (((uintptr_t)g->h_split % 16) == 0 && (g->ld_hs % 8) == 0);
  if ((tma_env & 2) && g->mode == 1 && !g->rows && a16 && s16 &&
      make_map_2d(&tc, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, g->c_out, g->hidden, g->m_max,
                  g->ld_cout) == FB_OK &&
      make_map_2d(&th, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, g->h_out, g->hidden, g->m_max,
                  g->ld_h) == FB_OK &&
      (!g->h_split || make_map_planes(&ts, g) == FB_OK))
    tma_c = 2;
  // rows gathered (the acoustic decoder): only the row-ordered h planes by TMA
  else if ((tma_env & 4) && g->mode == 1 && g->rows && g->h_split && g->hs_row_mode && a16 &&
           s16 && make_map_planes(&ts, g) == FB_OK)
    tma_c = 3;
  launch_pdl(k, dim3(grid), dim3(TC_THREADS), smem, s, ta, tw, tc, th, ts, tma_c, *g, a_planes,
             (int)a_plane_rows, g->k / TC_BK, kcb);
  count_launch();
  return check_launch("gemm_tc");
}

template <int BN>
static int launch_tc(const fb_gemm_t* g, int a_planes, int64_t a_plane_rows, int64_t w_rows,
                     cudaStream_t s) {
  CUtensorMap ta, tw;
  int rc = make_map(&ta, g->a, (uint64_t)a_planes * a_plane_rows, g->k, g->lda, TC_BM);
  if (rc) return rc;
  rc = make_map(&tw, g->w, w_rows, g->k, g->ldw, BN);
  if (rc) return rc;
  return launch_tc_maps<BN>(ta, tw, g, a_planes, a_plane_rows, s);
}

}  // namespace fb

using namespace fb;

#ifdef FB_GEMM_TRACE
extern "C" int fb_gemm_trace_read(unsigned long long* out) {
  return cudaMemcpyFromSymbol(out, g_trace, sizeof(g_trace)) == cudaSuccess ? 0 : 3;
}
#endif

extern "C" int fb_gemm_tc(const fb_gemm_t* g, int32_t a_planes, int64_t a_plane_rows,
                          void* stream) {
  FB_CHECK_ARG(g && g->a && g->w, "null GEMM operands");
  FB_CHECK_ARG(a_planes >= 1 && a_planes <= kPlanes, "a_planes must be 1..operand planes");
  FB_CHECK_ARG(g->k % TC_BK == 0 && g->k > 0, "tensor-core GEMM needs k % 64 == 0");
  FB_CHECK_ARG(g->lda % 8 == 0 && g->ldw % 8 == 0, "leading dims must be multiples of 8");
  FB_CHECK_ARG(((uintptr_t)g->a % 16) == 0 && ((uintptr_t)g->w % 16) == 0, "16B alignment");
  FB_CHECK_ARG(a_plane_rows >= g->m_max, "plane stride smaller than m_max");
  FB_CHECK_ARG(g->mode == 0 || g->mode == 1, "unknown GEMM epilogue");
  FB_CHECK_ARG(g->mode != 1 || (g->n == 4 * g->hidden && g->h_out && g->c_out),
               "LSTM epilogue needs n == 4*hidden and state outputs");
  FB_CHECK_ARG(g->mode != 0 || g->c, "GEMM output is null");
  FB_CHECK_ARG(!g->splitk_ws || g->splitk_cnt, "stream-K workspace without counters");
  FB_CHECK_ARG(!g->out_logsoftmax || (g->mode == 0 && g->n <= 64 && !g->row_stats &&
                                      !g->splitk_ws && !g->addend),
               "fused log-softmax needs mode 0, n <= 64, no stats/addend/stream-K");
  FB_CHECK_ARG(g->mode != 1 || g->bias == nullptr || ((uintptr_t)g->bias % 16) == 0,
               "LSTM bias must be 16B aligned");
  FB_CHECK_ARG(g->mode != 1 || g->addend == nullptr ||
                   (((uintptr_t)g->addend % 16) == 0 && g->ld_add % 4 == 0),
               "LSTM addend must be 16B aligned");
  if (g->m_max <= 0) return FB_OK;
  fb_gemm_t gs = *g;
  if (gs.acc_scale == 0.f) gs.acc_scale = 1.f / kActScale;
  g = &gs;
  // small problems: half-width tiles so more SMs take part
  static const int force_bn = [] {
    const char* e = getenv("FB_GEMM_BN");
    return e ? atoi(e) : 0;
  }();
  const int tiles128 = ((g->m_max + TC_BM - 1) / TC_BM) * ((g->n + 127) / 128);
  // 128-wide tiles beat 64-wide ones at the decoder shapes with n > 64 once
  // the grid holds more than a third of the SMs; below that (the word LM's
  // LSTM GEMMs with <= 128 event rows, the acoustic LSTM GEMMs in the
  // lock-step tail) twice the CTAs win: 160x4800x2432 33 -> 47 us, but
  // 64x4800x2432 32 -> 27 us and 512x1280x320 12 -> 8.8 us (graph-timed
  // scripts/bench_gemm.py via scripts/sweep_bn.sh).  Same K loop per output,
  // so the result is bit-identical either way.
  static const int few_env = getenv("FB_GEMM_FEW") ? atoi(getenv("FB_GEMM_FEW")) : 1;  // dev A/B
  const bool few_tiles = few_env && force_bn == 0 && !g->splitk_ws && 3 * tiles128 <= kNumSMs;
  // n <= 64 (the acoustic output projection): a 64-wide tile is the whole N
  const bool want64 = force_bn == 64 || (force_bn == 0 && g->n <= 64) || g->out_logsoftmax ||
                      few_tiles;
  if (want64 && !g->row_stats)
    return launch_tc<64>(g, a_planes, a_plane_rows, g->n, (cudaStream_t)stream);
  return launch_tc<128>(g, a_planes, a_plane_rows, g->n, (cudaStream_t)stream);
}

// LSTM recurrence over `steps` time steps for one direction (the encoder):
// h_t = cell(xp[:, t] + h_{t-1} W_hh^T), h written to y[:, t] and, split into
// bf16 planes, to rec[(t+1)%2] (the next step's A operand).  The host loop
// lives here so a layer costs one C call; tensor maps are built once.
extern "C" int fb_lstm_recurrence(int32_t steps, int32_t batch, int32_t hidden,
                                  const void* w_hh, int32_t k, const float* xp, int64_t ld_xp,
                                  int64_t step_xp, float* y, int64_t ld_y, int64_t step_y,
                                  void* rec, uint32_t* sync_ws, float acc_scale,
                                  const int32_t* t_rev, void* stream) {
  FB_CHECK_ARG(w_hh && xp && y && rec && sync_ws, "null recurrence buffers");
  FB_CHECK_ARG(ld_xp % 4 == 0 && step_xp % 4 == 0 && ld_y % 4 == 0 && step_y % 4 == 0 &&
                   k % 8 == 0 && ((uintptr_t)xp % 16) == 0 && ((uintptr_t)y % 16) == 0,
               "recurrence layouts must be 16-byte aligned");
  FB_CHECK_ARG(k % TC_BK == 0 && k >= hidden, "recurrence k must be a multiple of 64 >= hidden");
  FB_CHECK_ARG(steps >= 0 && batch > 0, "bad recurrence sizes");
  FB_CHECK_ARG((4 * hidden) % 128 == 0 && hidden % 32 == 0, "hidden must be a multiple of 32");
  const int n_tiles = 4 * hidden / 128;
  if (steps == 0) return FB_OK;
  cudaStream_t s = (cudaStream_t)stream;
  // shared memory: the resident W_hh slice + a ring of A-plane stages
  const int num_kb = k / TC_BK;
  const size_t w_bytes = (size_t)num_kb * 128 * TC_BK * 2;
  const size_t a_stage = (size_t)kPlanes * TC_BM * TC_BK * 2;
  int dev = 0, max_optin = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&max_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const size_t budget = (size_t)max_optin - 1024 - 256;    // static barriers
  const int nst = (int)std::min<size_t>(REC_MAX_STAGES, budget > w_bytes ? (budget - w_bytes) / a_stage : 0);
  if (nst < 2) return fail(FB_ERR_CONFIG, "recurrence W_hh slice does not fit shared memory");
  const size_t smem = w_bytes + (size_t)nst * a_stage + 1024;
  if (cudaFuncSetAttribute(lstm_rec_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)smem) != cudaSuccess)
    return check_launch("lstm_rec attributes");
  // the step barrier needs every CTA of a launch resident: the device's
  // capacity (SM count and occupancy read at run time, not a constant) bounds
  // the row tiles per cooperative launch; a larger batch runs as several
  // launches over row blocks (rows never interact), each from h = c = 0
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, lstm_rec_kernel, TC_THREADS, smem);
  int max_mt = per_sm * sms / n_tiles;
  const char* cap_s = getenv("FB_REC_MAX_ROWS");      // read per call (tests toggle it)
  const int cap_env = cap_s ? atoi(cap_s) : 0;
  if (cap_env > 0) max_mt = std::min(max_mt, std::max(1, cap_env / TC_BM));   // test knob
  if (max_mt < 1) return fail(FB_ERR_CONFIG, "recurrence tile row cannot be co-resident on this device");
  // TMEM accumulation chunk of the recurrence (K blocks; dev override FB_REC_KCB)
  static const int kcb_env = getenv("FB_REC_KCB") ? std::max(1, atoi(getenv("FB_REC_KCB"))) : 1;
  int nkb = num_kb, kcb = std::min(kcb_env, num_kb);
  static const int wide_env = getenv("FB_REC_WIDE") ? atoi(getenv("FB_REC_WIDE")) : 7;
  uint16_t* r = reinterpret_cast<uint16_t*>(rec);
  int rc = 0;
  for (int b0 = 0; b0 < batch; b0 += max_mt * TC_BM) {
    const int nb = std::min(batch - b0, max_mt * TC_BM);
    const int m_tiles = (nb + TC_BM - 1) / TC_BM;
    // rec is scratch: this block's two steps of planes packed as [2][planes][nb][k]
    const int64_t plane = (int64_t)nb * k;
    if (b0 > 0) cudaMemsetAsync(r, 0, sizeof(uint16_t) * kPlanes * plane, s);   // h_{-1} = 0
    const float* xpb = xp + (int64_t)b0 * ld_xp;
    float* yb = y + (int64_t)b0 * ld_y;
    const int32_t* trb = t_rev ? t_rev + b0 : nullptr;
    fb_gemm_t g{};
    g.acc_scale = acc_scale > 0.f ? acc_scale : 1.f / kActScale;
    g.m_max = nb; g.m_dev = nullptr; g.n = 4 * hidden; g.k = k;
    g.lda = k; g.w = w_hh; g.ldw = k; g.bias = nullptr;
    g.mode = 1; g.hidden = hidden;
    g.ld_cin = hidden; g.ld_cout = hidden; g.ld_h = ld_y; g.ld_add = ld_xp;
    g.hs_plane_rows = nb; g.ld_hs = k;
    CUtensorMap ta[2], tw;
    for (int p = 0; p < 2; ++p) {
      rc = make_map(&ta[p], r + (int64_t)p * kPlanes * plane, (uint64_t)kPlanes * nb, k, k, TC_BM);
      if (rc) return rc;
    }
    rc = make_map(&tw, w_hh, g.n, k, k, 128);
    if (rc) return rc;
    cudaMemsetAsync(sync_ws, 0, sizeof(uint32_t) * m_tiles * kRecSyncStride, s);
    // 256-bit accesses where the layouts are 32-byte aligned: bit 0 xp loads,
    // bit 1 y stores, bit 2 operand-plane stores (dev override FB_REC_WIDE)
    int wide = wide_env &
               ((((uintptr_t)xpb % 32) == 0 && ld_xp % 8 == 0 && step_xp % 8 == 0 ? 1 : 0) |
                (((uintptr_t)yb % 32) == 0 && ld_y % 8 == 0 && step_y % 8 == 0 ? 2 : 0) |
                (((uintptr_t)rec % 32) == 0 && k % 16 == 0 ? 4 : 0));
    void* args[] = {(void*)&ta[0], (void*)&ta[1], (void*)&tw, (void*)&g, (void*)&steps,
                    (void*)&nkb, (void*)&kcb, (void*)&xpb, (void*)&step_xp, (void*)&yb,
                    (void*)&ld_y, (void*)&step_y, (void*)&r, (void*)&plane, (void*)&sync_ws,
                    (void*)&nst, (void*)&trb, (void*)&wide};
    const cudaError_t e = cudaLaunchCooperativeKernel((const void*)lstm_rec_kernel,
                                                      dim3(m_tiles * n_tiles), dim3(TC_THREADS),
                                                      args, smem, s);
    count_launch();
    if (e != cudaSuccess) {
      cudaGetLastError();
      return fail(FB_ERR_CUDA, std::string("lstm_rec cooperative launch: ") + cudaGetErrorString(e));
    }
  }
  return FB_OK;
}

extern "C" int fb_operand_format(int32_t* planes, int32_t* is_fp16, float* act_scale) {
  FB_CHECK_ARG(planes && is_fp16 && act_scale, "null outputs");
  *planes = kPlanes;
  *is_fp16 = FB_OPERAND_FP16X2;
  *act_scale = kActScale;
  return FB_OK;
}
