// gs_gemm.cu — Darknet-style layers on the 5th-generation tensor cores.
//
// The reference models Darknet jobs as catalog entries (conv1 / conv2 / fc /
// backbone ..., gpushare/data/neural_catalog.json:6-57) with no code; here
// they run for real.  A Darknet convolution is im2col + GEMM (Darknet's
// gemm_gpu path); on B200 the GEMM is a tcgen05 kernel:
//
//   D[M x N] = act(A[M x K] . B[N x K]^T + bias[N])      (bf16 in, fp32 acc)
//
// A = activation patches (NHWC im2row: one row per output pixel, K =
// kh*kw*C_in contiguous), B = filters [C_out x K] (Darknet's weight layout),
// D = the next NHWC activation.  Both operands are K-major and arrive by TMA
// (128-byte swizzle) into a 4-stage shared-memory ring; one elected thread
// issues tcgen05.mma (M = 128, N = BN, K = 16 per instruction) into a TMEM
// accumulator; all four warps drain TMEM with tcgen05.ld and apply the bias +
// leaky-ReLU epilogue (Darknet's activate_array LEAKY, slope 0.1).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include <atomic>
#include <mutex>
#include <string>
#include <vector>

#include "gs_tc.cuh"
#include "gs_work_internal.h"

namespace gsw {

struct GemmArgs {
  int m, n;              // valid rows / columns of D
  int m_tiles, n_tiles, k_blocks;
  const float *bias;     // [n] or nullptr
  void *out;             // D + column offset
  int64_t ldo;           // row pitch of D (elements)
  int out_f32;           // 1: fp32 D, 0: bf16 D
  int act;               // 0 linear, 1 leaky (0.1), 2 YOLO logistic, 3 ReLU
  const __nv_bfloat16 *res;  // residual added before the activation (bf16, pitch ldr) or nullptr
  int64_t ldr;
  unsigned *tk;          // the job's tile tickets (gs_kernels.cuh grab_tile) or nullptr: static striding
  // implicit convolution (gemm_bf16_tc<BN, true>): A is not a matrix in
  // memory but the im2row view of an NHWC activation, gathered per stage
  const __nv_bfloat16 *cin;  // the activation (its channel offset applied)
  int cn, ch, cw, cpitch;    // batch, input height / width, pixel pitch (elements)
  int clog2c;                // log2(channels): channels are a power of two >= 8
  int coh, cow, ck, cstride, cpad, ckdim;  // output h / w, kernel (1 or 3), stride, pad, k*k*C
};

// 3 stages x (16 KB A + <= 16 KB B) <= 99 KB: two CTAs per SM, so one CTA's
// epilogue overlaps the other's mainloop and a Darknet job's kernels all
// fit a 2 x 148 grid (the mgb-sm probe rule, see gs_darknet.cu grid_for)
constexpr int kGemmBM = 128, kGemmBK = 64, kGemmStages = 3;

template <int BN>
constexpr size_t gemm_smem_bytes() {
  return (size_t)kGemmStages * (kGemmBM + BN) * kGemmBK * 2 + 1024 + 256;
}

constexpr int kGemmThreads = 192;  // warp 0 TMA, warp 1 MMA, warps 2-5 epilogue
constexpr int kGatherWarps = 2;    // implicit convolution: warps 6.. gather A (4 measured no faster)
constexpr int kGatherThreads = 32 * kGatherWarps;
constexpr int kGatherRows = kGemmBM / kGatherThreads;  // tile rows per gather thread
constexpr int kConvThreads = kGemmThreads + kGatherThreads;

__device__ __forceinline__ float leaky(float v) { return v > 0.0f ? v : 0.1f * v; }
// YOLO layer (Darknet yolo_layer forward): logistic on x, y, objectness and
// class scores of each 85-channel anchor group; w, h (entries 2, 3) linear.
__device__ __forceinline__ float yolo_act(float v, int col) {
  const int e = col % 85;
  return (e == 2 || e == 3) ? v : 1.0f / (1.0f + expf(-v));
}

// 16-byte global -> shared copy, zero-filled when src_bytes == 0 (padding,
// rows past M, columns past K)
__device__ __forceinline__ void cp_async16_zfill(uint32_t dst, const void *src, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(src_bytes) : "memory");
}
// arrive on `bar` when every cp.async this thread issued so far has landed
// (the barrier's expected count includes these arrivals)
__device__ __forceinline__ void cp_async_mbar_arrive(uint64_t *bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(tc::smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tc::smem_u32(bar)) : "memory");
}

// Bias + activation of one row's 32 columns, stored as bf16 or fp32.
__device__ __forceinline__ void epilogue_store(const GemmArgs &g, int row, int col0, float (&v)[32]) {
  if (row >= g.m || col0 >= g.n) return;
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    float x = v[i];
    if (g.bias && col0 + i < g.n) x += __ldg(g.bias + col0 + i);
    v[i] = x;
  }
  if (g.res) {  // ResNet shortcut: D = act(A.B^T + bias + R)
    const __nv_bfloat16 *r = g.res + (int64_t)row * g.ldr + col0;
    if (col0 + 32 <= g.n && ((reinterpret_cast<uintptr_t>(r) & 15) == 0)) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint4 u = *reinterpret_cast<const uint4 *>(r + 8 * q);
        const __nv_bfloat162 *h = reinterpret_cast<const __nv_bfloat162 *>(&u);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 f = __bfloat1622float2(h[e]);
          v[8 * q + 2 * e] += f.x;
          v[8 * q + 2 * e + 1] += f.y;
        }
      }
    } else {
#pragma unroll
      for (int i = 0; i < 32; ++i)
        if (col0 + i < g.n) v[i] += __bfloat162float(r[i]);
    }
  }
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    const float x = v[i];
    v[i] = g.act == 1 ? leaky(x) : (g.act == 2 ? yolo_act(x, col0 + i) : (g.act == 3 ? fmaxf(x, 0.0f) : x));
  }
  const bool whole = col0 + 32 <= g.n;
  if (g.out_f32) {
    float *o = reinterpret_cast<float *>(g.out) + (int64_t)row * g.ldo + col0;
    if (whole && ((reinterpret_cast<uintptr_t>(o) & 15) == 0)) {
#pragma unroll
      for (int i = 0; i < 32; i += 4) *reinterpret_cast<float4 *>(o + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
    } else if (whole) {
      // rows of an odd pitch (the YOLO heads: 255 fp32 columns): scalars up
      // to the next 16-byte boundary, then float4s (32 scalar stores per row
      // made the heads store-bound)
      const int lead = (int)((16 - (reinterpret_cast<uintptr_t>(o) & 15)) & 15) >> 2;
#pragma unroll
      for (int i = 0; i < 3; ++i)
        if (i < lead) o[i] = v[i];
#pragma unroll
      for (int q = 0; q < 7; ++q) {
#pragma unroll
        for (int a4 = 0; a4 < 4; ++a4)
          if (lead == a4) {
            const int i = a4 + 4 * q;
            *reinterpret_cast<float4 *>(o + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
          }
      }
#pragma unroll
      for (int i = 28; i < 32; ++i)
        if (i >= lead + 28) o[i] = v[i];
    } else {
#pragma unroll
      for (int i = 0; i < 32; ++i)
        if (col0 + i < g.n) o[i] = v[i];
    }
  } else {
    __nv_bfloat16 *o = reinterpret_cast<__nv_bfloat16 *>(g.out) + (int64_t)row * g.ldo + col0;
    if (whole && ((reinterpret_cast<uintptr_t>(o) & 15) == 0)) {
#pragma unroll
      for (int i = 0; i < 32; i += 8) {
        uint4 q;
        __nv_bfloat162 p0 = __floats2bfloat162_rn(v[i], v[i + 1]), p1 = __floats2bfloat162_rn(v[i + 2], v[i + 3]);
        __nv_bfloat162 p2 = __floats2bfloat162_rn(v[i + 4], v[i + 5]), p3 = __floats2bfloat162_rn(v[i + 6], v[i + 7]);
        q.x = *reinterpret_cast<uint32_t *>(&p0);
        q.y = *reinterpret_cast<uint32_t *>(&p1);
        q.z = *reinterpret_cast<uint32_t *>(&p2);
        q.w = *reinterpret_cast<uint32_t *>(&p3);
        *reinterpret_cast<uint4 *>(o + i) = q;
      }
    } else {
#pragma unroll
      for (int i = 0; i < 32; ++i)
        if (col0 + i < g.n) o[i] = __float2bfloat16_rn(v[i]);
    }
  }
}

// The producer's next tile: a ticket from the job's counter (co-location
// friendly: a CTA that starts late behind another job's kernel finds fewer
// tiles left instead of owing a fixed share), or static striding without
// one.  The retirement protocol is grab_tile's: the last CTA out resets the
// counter for the next kernel on the job's stream.
__device__ __forceinline__ int gemm_next_tile(const GemmArgs &g, int i, int tiles) {
  if (!g.tk) return blockIdx.x + i * gridDim.x;
  const unsigned t = atomicAdd(&g.tk[0], 1u);
  if ((int64_t)t < tiles) return (int)t;
  __threadfence();
  if (atomicAdd(&g.tk[1], 1u) == gridDim.x - 1) {
    atomicExch(&g.tk[0], 0u);
    atomicExch(&g.tk[1], 0u);
  }
  return tiles;
}

// Persistent, warp-specialized: the TMA producer takes tiles (tickets or
// static striding) and publishes each tile index through a 4-slot smem queue
// to the MMA warp and the epilogue warps; it runs ahead through the 3-stage
// operand ring across tile boundaries, the MMA warp alternates between two
// TMEM accumulators, and the four epilogue warps drain accumulator t while
// the MMAs of tile t+1 run.
//
// CONV = true: the implicit convolution.  A's stage is gathered by
// kGatherWarps extra warps (6, ...) straight from the NHWC activation with 16-byte cp.async into
// the 128-byte-swizzled K-major layout the TMA would have written (chunk j of
// tile row r at r * 128 + ((j ^ (r & 7)) << 4)), zero-filled at the padding
// and past M / K; each gather thread's cp.async completion arrives on the
// stage's barrier (expected count 1 + kGatherThreads), and the MMA thread issues a proxy
// fence before its tensor-core reads.  K order (ky, kx, c) is im2row's, so
// the products equal im2row + GEMM's exactly — without writing and
// re-reading the im2row matrix (30-39 % of a Darknet job).
template <int BN, bool CONV = false>
__global__ void __launch_bounds__(CONV ? kConvThreads : kGemmThreads, 2)
    gemm_bf16_tc(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb, GemmArgs g) {
  using namespace tc;
  constexpr uint32_t A_BYTES = kGemmBM * kGemmBK * 2, B_BYTES = BN * kGemmBK * 2;
  constexpr uint32_t TM_COLS = 2 * BN < 32 ? 32 : 2 * BN;  // two accumulators
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t *sa = smem;
  uint8_t *sb = smem + kGemmStages * A_BYTES;
  uint64_t *full = reinterpret_cast<uint64_t *>(sb + kGemmStages * B_BYTES);
  uint64_t *empty = full + kGemmStages;
  uint64_t *acc_full = empty + kGemmStages;  // [2]
  uint64_t *acc_empty = acc_full + 2;        // [2]
  uint64_t *tq_full = acc_empty + 2;         // [4] tile index published
  uint64_t *tq_empty = tq_full + 4;          // [4] read by the MMA thread and the 4 epilogue warps
  volatile int *tq = reinterpret_cast<volatile int *>(tq_empty + 4);  // [4]
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tq_empty + 4) + 4;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    if (!CONV) tma_prefetch(&ta);
    tma_prefetch(&tb);
    for (int s = 0; s < kGemmStages; ++s) {
      mbar_init(&full[s], CONV ? 1 + kGatherThreads : 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&acc_full[a], 1);
      mbar_init(&acc_empty[a], 4);  // one arrival per epilogue warp
    }
    for (int s = 0; s < 4; ++s) {
      mbar_init(&tq_full[s], 1);
      mbar_init(&tq_empty[s], CONV ? 5 + kGatherWarps : 5);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<TM_COLS>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  constexpr uint32_t idesc = idesc_bf16_f32(kGemmBM, BN);
  const int tiles = g.m_tiles * g.n_tiles;

  if (warp == 0) {
    if (lane == 0) {  // TMA producer
      uint32_t stage = 0, phase = 0;
      for (int i = 0;; ++i) {
        mbar_wait(&tq_empty[i & 3], ((i >> 2) & 1) ^ 1);
        const int tile = gemm_next_tile(g, i, tiles);
        tq[i & 3] = tile;
        mbar_arrive(&tq_full[i & 3]);
        if (tile >= tiles) break;
        const int mt = tile / g.n_tiles, nt = tile % g.n_tiles;
        for (int kb = 0; kb < g.k_blocks; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_expect_tx(&full[stage], CONV ? B_BYTES : A_BYTES + B_BYTES);
          if (!CONV) tma_load_2d(sa + stage * A_BYTES, &ta, &full[stage], kb * kGemmBK, mt * kGemmBM);
          tma_load_2d(sb + stage * B_BYTES, &tb, &full[stage], kb * kGemmBK, nt * BN);
          if (++stage == kGemmStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // MMA issuer
      uint32_t stage = 0, phase = 0;
      for (int t = 0;; ++t) {
        mbar_wait(&tq_full[t & 3], (t >> 2) & 1);
        const int tile = tq[t & 3];
        mbar_arrive(&tq_empty[t & 3]);
        if (tile >= tiles) break;
        const int acc = t & 1;
        mbar_wait(&acc_empty[acc], ((t >> 1) & 1) ^ 1);  // epilogue drained this accumulator
        tc_fence_after();
        const uint32_t d = tmem + acc * BN;
        for (int kb = 0; kb < g.k_blocks; ++kb) {
          mbar_wait(&full[stage], phase);
          if (CONV) fence_proxy_async_smem();  // the gathered A was written by cp.async (generic proxy)
          tc_fence_after();
          const uint64_t ad = sdesc_k_sw128(sa + stage * A_BYTES);
          const uint64_t bd = sdesc_k_sw128(sb + stage * B_BYTES);
#pragma unroll
          for (int k = 0; k < kGemmBK / 16; ++k) mma_bf16(d, ad + 2 * k, bd + 2 * k, idesc, (kb | k) != 0);
          mma_commit(&empty[stage]);  // frees the smem slot when these MMAs finish
          if (++stage == kGemmStages) {
            stage = 0;
            phase ^= 1;
          }
        }
        mma_commit(&acc_full[acc]);  // accumulator ready for the epilogue
      }
    }
  } else if (CONV && warp >= 6) {
    // A gather (implicit im2row): kGatherThreads threads, tile rows gt + kGatherThreads * h
    const int gt = (int)threadIdx.x - 192;
    const int cmask = (1 << g.clog2c) - 1;
    uint32_t stage = 0, phase = 0;
    for (int i = 0;; ++i) {
      mbar_wait(&tq_full[i & 3], (i >> 2) & 1);
      const int tile = tq[i & 3];
      __syncwarp();
      if (lane == 0) mbar_arrive(&tq_empty[i & 3]);
      if (tile >= tiles) break;
      const int mt = tile / g.n_tiles;
      int iy0[kGatherRows], ix0[kGatherRows];
      bool valid[kGatherRows];
      const __nv_bfloat16 *img[kGatherRows];
#pragma unroll
      for (int h = 0; h < kGatherRows; ++h) {
        const int m = mt * kGemmBM + gt + kGatherThreads * h;
        valid[h] = m < g.m;
        const int mm = valid[h] ? m : 0;
        const int t2 = mm / g.cow, ox = mm - t2 * g.cow;
        const int b = t2 / g.coh, oy = t2 - b * g.coh;
        iy0[h] = oy * g.cstride - g.cpad;
        ix0[h] = ox * g.cstride - g.cpad;
        img[h] = g.cin + (int64_t)b * g.ch * g.cw * g.cpitch;
      }
      for (int kb = 0; kb < g.k_blocks; ++kb) {
        mbar_wait(&empty[stage], phase ^ 1);
        const uint32_t dst = smem_u32(sa + stage * A_BYTES);
#pragma unroll
        for (int h = 0; h < kGatherRows; ++h) {
          const int r = gt + kGatherThreads * h;
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const int k = kb * kGemmBK + j * 8;
            const int tap = k >> g.clog2c, c = k & cmask;
            const int ky = g.ck == 1 ? 0 : (tap * 11) >> 5;  // tap / 3 for tap < 9
            const int kx = tap - ky * g.ck;
            const int iy = iy0[h] + ky, ix = ix0[h] + kx;
            const bool ok = valid[h] && k < g.ckdim && iy >= 0 && iy < g.ch && ix >= 0 && ix < g.cw;
            const __nv_bfloat16 *src = ok ? img[h] + ((int64_t)iy * g.cw + ix) * g.cpitch + c : g.cin;
            cp_async16_zfill(dst + r * 128 + ((j ^ (r & 7)) << 4), src, ok ? 16 : 0);
          }
        }
        cp_async_mbar_arrive(&full[stage]);
        if (++stage == kGemmStages) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
  } else {
    // epilogue warps 2..5: TMEM lane quarter (warp % 4) = tile rows 32q .. 32q+31
    const int q = warp & 3;
    for (int t = 0;; ++t) {
      mbar_wait(&tq_full[t & 3], (t >> 2) & 1);
      const int tile = tq[t & 3];
      __syncwarp();
      if (lane == 0) mbar_arrive(&tq_empty[t & 3]);
      if (tile >= tiles) break;
      const int mt = tile / g.n_tiles, nt = tile % g.n_tiles;
      const int acc = t & 1;
      mbar_wait(&acc_full[acc], (t >> 1) & 1);
      tc_fence_after();
      const int row = mt * kGemmBM + q * 32 + lane;
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += 32) {
        float v[32];
        tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + acc * BN + c0, v);
        epilogue_store(g, row, nt * BN + c0, v);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[acc]);
    }
  }
  __syncthreads();
  if (warp == 1) tmem_dealloc<TM_COLS>(tmem);
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------

typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

// K-major bf16 matrix [rows x k] (row pitch ld elements), box [box_rows x 64],
// 128-byte swizzle; out-of-bounds rows / columns read as zero.
static int make_tmap(CUtensorMap *m, const void *ptr, int64_t rows, int64_t k, int64_t ld, int box_rows) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return err(GS_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  if ((ld * 2) % 16 || (reinterpret_cast<uintptr_t>(ptr) & 15))
    return err(GS_ERR_CONFIG, "gemm operands need 16-byte aligned rows (K % 8 == 0)");
  cuuint64_t dims[2] = {(cuuint64_t)k, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * 2)};
  cuuint32_t box[2] = {(cuuint32_t)kGemmBK, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void *>(ptr), dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return err(GS_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
  return GS_OK;
}

// Row-major fp32 matrix [rows x cols] (row pitch cols), box [box_rows x
// box_cols], no swizzle; out-of-bounds elements read as zero.
int make_tmap_f32(CUtensorMap *m, const void *ptr, int64_t rows, int64_t cols, int box_cols, int box_rows) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return err(GS_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  if ((cols * 4) % 16 || (reinterpret_cast<uintptr_t>(ptr) & 15))
    return err(GS_ERR_CONFIG, "fp32 tensor map needs 16-byte aligned rows");
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(cols * 4)};
  cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void *>(ptr), dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return err(GS_ERR_CUDA, "cuTensorMapEncodeTiled (f32) failed (" + std::to_string((int)r) + ")");
  return GS_OK;
}

template <int BN, bool CONV = false>
static int launch_bn(const CUtensorMap &ta, const CUtensorMap &tb, GemmArgs g, int max_ctas, cudaStream_t st) {
  // the attribute is per device (the executor may drive several); set it on
  // a device's first launch only -- a driver call per launch serializes the
  // executor's worker threads on the context lock
  static std::atomic<uint64_t> configured{0};  // (one per <BN, CONV> instance)
  int dev = 0;
  cudaGetDevice(&dev);
  const uint64_t bit = 1ull << (dev & 63);
  if (!(configured.load(std::memory_order_acquire) & bit)) {
    const cudaError_t attr_rc = cudaFuncSetAttribute(gemm_bf16_tc<BN, CONV>,
                                                     cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                     (int)gemm_smem_bytes<BN>());
    if (attr_rc != cudaSuccess)
      return err(GS_ERR_CUDA, std::string("gemm smem attribute: ") + cudaGetErrorString(attr_rc));
    configured.fetch_or(bit, std::memory_order_acq_rel);
  }
  g.n_tiles = (g.n + BN - 1) / BN;
  const int tiles = g.m_tiles * g.n_tiles;
  const int grid = tiles < max_ctas ? tiles : max_ctas;
  gemm_bf16_tc<BN, CONV><<<grid, CONV ? kConvThreads : kGemmThreads, gemm_smem_bytes<BN>(), st>>>(ta, tb, g);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return err(GS_ERR_CUDA, std::string("gemm launch: ") + cudaGetErrorString(e));
  return GS_OK;
}

int gemm_pick_bn(int m, int n) {
  (void)m;
  if (n <= 32) return 32;
  if (n <= 64) return 64;
  return 128;
}

// D = act(A . B^T + bias): A [m x k] (pitch lda), B [n x k] (pitch ldb), D
// [m x n] at `out` (pitch ldo).  max_ctas bounds the grid (the job's SM share).
int gemm_bf16(const void *A, int64_t lda, const void *B, int64_t ldb, const float *bias, void *out, int64_t ldo,
              int m, int n, int k, int out_f32, int act, int max_ctas, cudaStream_t st, const void *res, int64_t ldr,
              unsigned *tk) {
  if (m <= 0 || n <= 0 || k <= 0) return err(GS_ERR_CONFIG, "gemm dims must be positive");
  if (k % 8) return err(GS_ERR_CONFIG, "gemm K must be a multiple of 8");
  const int bn = gemm_pick_bn(m, n);
  CUtensorMap ta, tb;
  int rc = make_tmap(&ta, A, m, k, lda, kGemmBM);
  if (rc) return rc;
  rc = make_tmap(&tb, B, n, k, ldb, bn);
  if (rc) return rc;
  GemmArgs g;
  memset(&g, 0, sizeof g);
  g.m = m;
  g.n = n;
  g.m_tiles = (m + kGemmBM - 1) / kGemmBM;
  g.n_tiles = 0;
  g.k_blocks = (k + kGemmBK - 1) / kGemmBK;
  g.bias = bias;
  g.out = out;
  g.ldo = ldo;
  g.out_f32 = out_f32;
  g.act = act;
  g.res = reinterpret_cast<const __nv_bfloat16 *>(res);
  g.ldr = ldr;
  g.tk = tk;
  if (max_ctas <= 0) max_ctas = 2 * sm_count();
  switch (bn) {
    case 32: return launch_bn<32>(ta, tb, g, max_ctas, st);
    case 64: return launch_bn<64>(ta, tb, g, max_ctas, st);
    case 128: return launch_bn<128>(ta, tb, g, max_ctas, st);
    default: return launch_bn<256>(ta, tb, g, max_ctas, st);
  }
}

// Implicit convolution: D[pixels x cout] = act(conv(in, W) + bias), the
// im2row matrix never materialized.  `in` is an NHWC view (pitch elements
// per pixel, C = 2^log2c channels, C >= 8), W [cout x k*k*C] (pitch ldb),
// k = 1 (with a stride) or 3.
int conv_gemm_bf16(const void *in, int nb, int h, int w, int pitch, int log2c, int oh, int ow, int k, int stride,
                   int pad, const void *B, int64_t ldb, const float *bias, void *out, int64_t ldo, int cout,
                   int out_f32, int act, int max_ctas, cudaStream_t st, const void *res, int64_t ldr, unsigned *tk) {
  if (log2c < 3 || (k != 1 && k != 3)) return err(GS_ERR_CONFIG, "implicit conv needs C = 2^k >= 8 and k in {1, 3}");
  if (pitch % 8 || (reinterpret_cast<uintptr_t>(in) & 15)) return err(GS_ERR_CONFIG, "implicit conv needs 16-byte pixels");
  const int64_t m64 = (int64_t)nb * oh * ow;
  if (m64 >= (1ll << 31)) return err(GS_ERR_CONFIG, "implicit conv: too many output pixels");
  const int m = (int)m64, kdim = k * k * (1 << log2c);
  const int bn = gemm_pick_bn(m, cout);
  CUtensorMap tb;
  int rc = make_tmap(&tb, B, cout, kdim, ldb, bn);
  if (rc) return rc;
  GemmArgs g;
  memset(&g, 0, sizeof g);
  g.m = m;
  g.n = cout;
  g.m_tiles = (m + kGemmBM - 1) / kGemmBM;
  g.k_blocks = (kdim + kGemmBK - 1) / kGemmBK;
  g.bias = bias;
  g.out = out;
  g.ldo = ldo;
  g.out_f32 = out_f32;
  g.act = act;
  g.res = reinterpret_cast<const __nv_bfloat16 *>(res);
  g.ldr = ldr;
  g.tk = tk;
  g.cin = reinterpret_cast<const __nv_bfloat16 *>(in);
  g.cn = nb;
  g.ch = h;
  g.cw = w;
  g.cpitch = pitch;
  g.clog2c = log2c;
  g.coh = oh;
  g.cow = ow;
  g.ck = k;
  g.cstride = stride;
  g.cpad = pad;
  g.ckdim = kdim;
  if (max_ctas <= 0) max_ctas = 2 * sm_count();
  switch (bn) {
    case 32: return launch_bn<32, true>(tb, tb, g, max_ctas, st);
    case 64: return launch_bn<64, true>(tb, tb, g, max_ctas, st);
    case 128: return launch_bn<128, true>(tb, tb, g, max_ctas, st);
    default: return launch_bn<256, true>(tb, tb, g, max_ctas, st);
  }
}

const void *conv_kernel_fn(int bn) {
  switch (bn) {
    case 32: return (const void *)gemm_bf16_tc<32, true>;
    case 64: return (const void *)gemm_bf16_tc<64, true>;
    case 128: return (const void *)gemm_bf16_tc<128, true>;
    default: return (const void *)gemm_bf16_tc<256, true>;
  }
}
int conv_block_threads() { return kConvThreads; }

int gemm_block_threads() { return kGemmThreads; }

size_t gemm_smem_for(int bn) {
  switch (bn) {
    case 32: return gemm_smem_bytes<32>();
    case 64: return gemm_smem_bytes<64>();
    case 128: return gemm_smem_bytes<128>();
    default: return gemm_smem_bytes<256>();
  }
}

const void *gemm_kernel_fn(int bn) {
  switch (bn) {
    case 32: return (const void *)gemm_bf16_tc<32>;
    case 64: return (const void *)gemm_bf16_tc<64>;
    case 128: return (const void *)gemm_bf16_tc<128>;
    default: return (const void *)gemm_bf16_tc<256>;
  }
}

}  // namespace gsw

extern "C" int gs_gemm_bf16(const void *A, int64_t lda, const void *B, int64_t ldb, const float *bias, void *out,
                            int64_t ldo, int32_t m, int32_t n, int32_t k, int32_t out_f32, int32_t act, void *stream) {
  return gsw::gemm_bf16(A, lda, B, ldb, bias, out, ldo, m, n, k, out_f32, act, 0, (cudaStream_t)stream);
}
