// gs_darknet.cu — Darknet-style inference jobs: YOLOv3-tiny on B200.
//
// The reference's neural catalog (gpushare/data/neural_catalog.json:6-57)
// stands Darknet jobs in as footprints + durations; BASELINE cfg 2 names
// YOLOv3-tiny (random init, batch 1-64).  This is that network, layer for
// layer as Darknet's yolov3-tiny.cfg defines it (13 convolutions with folded
// batch-norm + leaky ReLU, 6 max-pools, a route / upsample / concat to the
// second head, two 255-channel YOLO heads), run Darknet's way: every
// convolution is im2col + GEMM, and every layer keeps its own resident
// output buffer (Darknet's l.output), so a job's footprint is the sum of its
// activations — which is what makes large batches exercise memory-safe
// placement.
//
// Layout is NHWC bf16 (a 3x3 tap's channels are contiguous, so im2row moves
// 16-byte vectors); the GEMM is the tcgen05 kernel of gs_gemm.cu with the
// bias + leaky (or YOLO logistic) epilogue fused; route/concat is free (the
// producing GEMM writes into a channel slice of the concat tensor) and the
// 2x upsample writes straight into its slice.
//
// The same layer machinery runs ResNet-50 (BASELINE cfg 2's other network:
// 7x7/2 stem, 3x3/2 max-pool, 16 bottleneck blocks with 1x1 / 3x3 / 1x1
// convolutions and identity or strided-projection shortcuts, global average
// pool, 1000-way fully connected layer; batch-norm folded into the bias):
// strided convolutions are im2row with a stride, and each block's residual
// add + ReLU is fused into the last GEMM's epilogue.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include <algorithm>
#include <string>
#include <vector>

#include "../../include/gs_work.h"
#include "gs_work_internal.h"

namespace gsw {

namespace {

constexpr int kThr = 256;
enum LType { CONV = 0, MAXPOOL = 1, UPSAMPLE = 2, AVGPOOL = 3 };
enum Act { LINEAR = 0, LEAKY = 1, YOLO = 2, RELU = 3 };

// A tensor view: NHWC with a per-pixel pitch and a channel offset inside buffer `buf`.
struct TView {
  int buf;
  int64_t off;  // element offset (channel offset)
  int n, h, w, c, pitch;
  bool f32;
};

struct LPlan {
  int type;
  TView in, out, res;        // res.buf < 0: no residual
  int k, stride, pad, cout, act;
  int kdim, kpad;            // im2row width (k*k*cin) and its 8-aligned pitch
  int64_t woff, boff;        // weight (bf16 elements) / bias (floats) offsets
};

struct NetPlan {
  std::vector<Buf> bufs;
  std::vector<LPlan> layers;
  int64_t flops = 0;
};

constexpr int B_IMG = 0, B_W = 1, B_BIAS = 2, B_DET = 3, B_WS = 4;

int64_t elems(const TView &v) { return (int64_t)v.n * v.h * v.w * v.pitch; }

// Layer-by-layer plan builder: every layer output is its own resident buffer
// (Darknet's l.output), weights / biases are packed into one buffer each.
struct NetBuilder {
  NetPlan P;
  int N;
  int64_t wcount = 0, bcount = 0, ws = 0;
  explicit NetBuilder(int batch, int64_t img_elems) : N(batch) {
    P.bufs.resize(5);
    P.bufs[B_IMG] = {img_elems * 2, IN};
  }
  TView act(int h, int w, int c, bool f32 = false) {
    TView v{(int)P.bufs.size(), 0, N, h, w, c, c, f32};
    P.bufs.push_back({elems(v) * (f32 ? 4 : 2), WRK});
    return v;
  }
  static TView none() { return TView{-1, 0, 0, 0, 0, 0, 0, false}; }
  TView conv(const TView &in, TView out, int k, int stride, int cout, int a, TView res = none()) {
    LPlan L{};
    L.type = CONV;
    L.in = in;
    L.out = out;
    L.res = res;
    L.k = k;
    L.stride = stride;
    L.pad = k / 2;
    L.cout = cout;
    L.act = a;
    L.kdim = k * k * in.c;
    L.kpad = (L.kdim + 7) / 8 * 8;
    L.woff = wcount;
    L.boff = bcount;
    wcount += (int64_t)cout * L.kpad;
    wcount = (wcount + 7) / 8 * 8;  // 16-byte aligned next layer
    bcount += cout;
    const int64_t opix = (int64_t)out.n * out.h * out.w;
    if (!direct_gemm(L) && !implicit_conv(L)) ws = std::max(ws, opix * L.kpad * 2);  // the im2row matrix
    P.flops += 2 * opix * (int64_t)L.kdim * cout;
    P.layers.push_back(L);
    return out;
  }
  // a 1x1 / stride-1 convolution reads the activation itself as the GEMM's A
  static bool direct_gemm(const LPlan &L) {
    return L.k == 1 && L.stride == 1 && L.in.pitch % 8 == 0 && L.in.off % 8 == 0;
  }
  // a k = 1 / 3 convolution over 2^j = 8 .. 128 channels runs as an
  // implicit GEMM (gemm_bf16_tc<BN, true> gathers A from the activation; no
  // im2row).  Measured per YOLO layer at 608^2 x 32 (ncu, us, im2row + GEMM
  // -> implicit): C 16: 713 -> 472, 32: 334 -> 200, 64: 212 -> 116, 128:
  // 126 -> 112, but 256: 80 -> 116 and 512: 158 -> 330 — with deep K the
  // two gather warps cannot feed the tensor cores the way the TMA does, so
  // wide layers keep im2row + the TMA GEMM.
  static bool implicit_conv(const LPlan &L) {
    static const bool off = [] {
      const char *e = getenv("GS_IM2ROW");
      return e && e[0] == '1';
    }();
    static const int cmax = [] {  // widest layer run implicitly (GS_IMPLICIT_CMAX, for measurement)
      const char *e = getenv("GS_IMPLICIT_CMAX");
      return e ? atoi(e) : 128;
    }();
    const int c = L.in.c;
    return !off && !direct_gemm(L) && (L.k == 1 || L.k == 3) && c >= 8 && c <= cmax && (c & (c - 1)) == 0 &&
           L.in.pitch % 8 == 0 && L.in.off % 8 == 0 && L.kpad == L.kdim;
  }
  TView pool(const TView &in, int k, int stride, int pad, int ho, int wo) {
    TView out = act(ho, wo, in.c);
    LPlan L{};
    L.type = MAXPOOL;
    L.in = in;
    L.out = out;
    L.res = none();
    L.k = k;
    L.stride = stride;
    L.pad = pad;
    P.layers.push_back(L);
    return out;
  }
  void finish(int64_t det_bytes) {
    P.bufs[B_W] = {wcount * 2, IN};
    P.bufs[B_BIAS] = {bcount * 4, IN};
    P.bufs[B_DET] = {det_bytes, OUT};
    P.bufs[B_WS] = {std::max<int64_t>(ws, 16), WRK};
  }
};

NetPlan yolo_plan(const gs_job_desc &j) {
  const int S = (int)j.n, N = (int)j.m;
  NetBuilder B(N, (int64_t)N * S * S * 3);
  // Darknet maxpool size 2: stride 2 halves the map, stride 1 keeps it
  // (window [i, i+1] clipped at the edge: Darknet's pad = size - 1, offset 0)
  auto pool2 = [&](const TView &in, int stride) {
    return B.pool(in, 2, stride, 0, stride == 2 ? in.h / 2 : in.h, stride == 2 ? in.w / 2 : in.w);
  };
  TView x{B_IMG, 0, N, S, S, 3, 3, false};
  // yolov3-tiny.cfg
  x = B.conv(x, B.act(S, S, 16), 3, 1, 16, LEAKY);                      // 0
  x = pool2(x, 2);                                                      // 1
  x = B.conv(x, B.act(S / 2, S / 2, 32), 3, 1, 32, LEAKY);              // 2
  x = pool2(x, 2);                                                      // 3
  x = B.conv(x, B.act(S / 4, S / 4, 64), 3, 1, 64, LEAKY);              // 4
  x = pool2(x, 2);                                                      // 5
  x = B.conv(x, B.act(S / 8, S / 8, 128), 3, 1, 128, LEAKY);            // 6
  x = pool2(x, 2);                                                      // 7
  // route target: [upsampled layer 18 (128) | layer 8 (256)] at S/16
  TView cat = B.act(S / 16, S / 16, 384);
  TView l8 = cat;
  l8.off = 128;
  l8.c = 256;
  x = B.conv(x, l8, 3, 1, 256, LEAKY);                                  // 8 -> concat[128:384]
  x = pool2(x, 2);                                                      // 9
  x = B.conv(x, B.act(S / 32, S / 32, 512), 3, 1, 512, LEAKY);          // 10
  x = pool2(x, 1);                                                      // 11 (size 2, stride 1)
  x = B.conv(x, B.act(S / 32, S / 32, 1024), 3, 1, 1024, LEAKY);        // 12
  TView l13 = B.conv(x, B.act(S / 32, S / 32, 256), 1, 1, 256, LEAKY);  // 13
  x = B.conv(l13, B.act(S / 32, S / 32, 512), 3, 1, 512, LEAKY);        // 14
  // 15 + 16: conv 255 linear, YOLO head 1 -> det[0 : N*(S/32)^2*255]
  TView det1{B_DET, 0, N, S / 32, S / 32, 255, 255, true};
  B.conv(x, det1, 1, 1, 255, YOLO);
  // 17 route 13; 18 conv 128 1x1; 19 upsample -> concat[0:128]
  TView l18 = B.conv(l13, B.act(S / 32, S / 32, 128), 1, 1, 128, LEAKY);
  {
    TView up = cat;
    up.c = 128;
    LPlan L{};
    L.type = UPSAMPLE;
    L.in = l18;
    L.out = up;
    L.res = NetBuilder::none();
    L.stride = 2;
    B.P.layers.push_back(L);
  }
  // 20 route 19, 8 (= cat); 21 conv 256 3x3; 22 conv 255 linear; 23 YOLO head 2
  x = B.conv(cat, B.act(S / 16, S / 16, 256), 3, 1, 256, LEAKY);        // 21
  TView det2{B_DET, (int64_t)N * (S / 32) * (S / 32) * 255, N, S / 16, S / 16, 255, 255, true};
  B.conv(x, det2, 1, 1, 255, YOLO);                                     // 22 + 23
  B.finish(((int64_t)N * (S / 32) * (S / 32) + (int64_t)N * (S / 16) * (S / 16)) * 255 * 4);
  return B.P;
}

// ResNet-50 (v1.5: stride on the 3x3 of the bottleneck), batch-norm folded
NetPlan resnet50_plan(const gs_job_desc &j) {
  const int S = (int)j.n, N = (int)j.m;
  NetBuilder B(N, (int64_t)N * S * S * 3);
  TView x{B_IMG, 0, N, S, S, 3, 3, false};
  x = B.conv(x, B.act(S / 2, S / 2, 64), 7, 2, 64, RELU);      // stem 7x7/2
  x = B.pool(x, 3, 2, 1, S / 4, S / 4);                        // max-pool 3x3/2, pad 1
  const int mids[4] = {64, 128, 256, 512}, blocks[4] = {3, 4, 6, 3};
  int hw = S / 4;
  for (int st = 0; st < 4; ++st) {
    const int mid = mids[st], outc = 4 * mid;
    for (int bi = 0; bi < blocks[st]; ++bi) {
      const int stride = (st > 0 && bi == 0) ? 2 : 1;
      const int ohw = hw / stride;
      TView a = B.conv(x, B.act(hw, hw, mid), 1, 1, mid, RELU);
      TView b = B.conv(a, B.act(ohw, ohw, mid), 3, stride, mid, RELU);
      TView sc = x;
      if (bi == 0) sc = B.conv(x, B.act(ohw, ohw, outc), 1, stride, outc, LINEAR);  // projection
      x = B.conv(b, B.act(ohw, ohw, outc), 1, 1, outc, RELU, sc);                  // + shortcut, ReLU
      hw = ohw;
    }
  }
  TView pooled = B.act(1, 1, 2048);
  {
    LPlan L{};
    L.type = AVGPOOL;
    L.in = x;
    L.out = pooled;
    L.res = NetBuilder::none();
    B.P.layers.push_back(L);
  }
  TView logits{B_DET, 0, N, 1, 1, 1000, 1000, true};
  B.conv(pooled, logits, 1, 1, 1000, LINEAR);                  // fully connected
  B.finish((int64_t)N * 1000 * 4);
  return B.P;
}

NetPlan net_plan(const gs_job_desc &j) { return j.kind == GS_JOB_RESNET ? resnet50_plan(j) : yolo_plan(j); }

// ---- kernels ------------------------------------------------------------------

__device__ __forceinline__ float unitf(uint64_t seed, uint64_t i) { return gs_unit(seed, i); }

__global__ void gen_image(__nv_bfloat16 *x, int64_t n, uint64_t seed) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    x[i] = __float2bfloat16_rn(unitf(seed, (uint64_t)i));
}

// one layer's filters [cout x kpad]: U(-s, s), s = sqrt(6 / fan_in) (He
// uniform, so activations stay O(1) through the stack); padding columns 0.
__global__ void gen_filters(__nv_bfloat16 *w, int cout, int kdim, int kpad, float s, uint64_t seed) {
  const int64_t total = (int64_t)cout * kpad;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int col = (int)(i % kpad);
    const float v = col < kdim ? (2.0f * unitf(seed, (uint64_t)i) - 1.0f) * s : 0.0f;
    w[i] = __float2bfloat16_rn(v);
  }
}

__global__ void gen_bias(float *b, int n, uint64_t seed) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    b[i] = 0.1f * (2.0f * unitf(seed, (uint64_t)i) - 1.0f);
}

struct ViewArgs {
  const __nv_bfloat16 *p;
  int n, h, w, c, pitch;
};

// im2row for a k x k / stride / pad convolution: ws[out pixel][(kh*k + kw)*C
// + c], zero outside the image and in the pad columns; 16-byte vectors when
// C % 8 == 0 (all layers but the first).
// Vector layers work per (output pixel, tap): the pixel's input row segment
// of C channels is copied as 16-byte chunks (a warp per unit, lane = chunk,
// when C >= 256; a thread per unit otherwise), and blocks walk output rows
// so the index arithmetic is 32-bit and per unit (a thread per 16-byte
// chunk with 64-bit div / mod per chunk was ALU bound: im2row was half of
// a YOLO / ResNet job).
__global__ void __launch_bounds__(kThr) im2row(ViewArgs in, __nv_bfloat16 *ws, int k, int stride, int pad, int oh,
                                               int ow, int kdim, int kpad) {
  const int C = in.c;
  const bool vec = (C % 8 == 0) && (in.pitch % 8 == 0);
  if (vec) {
    const int taps = k * k, cch = C / 8, tail = (kpad - kdim) / 8;
    const int rows = in.n * oh, per_row = ow * taps;
    const uint4 zero = make_uint4(0, 0, 0, 0);
    const bool warp_units = cch >= 32;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int r = blockIdx.x; r < rows; r += gridDim.x) {
      const int b = r / oh, oy = r - b * oh;
      const int u0 = warp_units ? warp : (int)threadIdx.x, us = warp_units ? nw : (int)blockDim.x;
      for (int u = u0; u < per_row; u += us) {
        const int ox = u / taps, tap = u - ox * taps;
        const int ky = tap / k, kx = tap - ky * k;
        const int iy = oy * stride + ky - pad, ix = ox * stride + kx - pad;
        uint4 *dst = reinterpret_cast<uint4 *>(ws + ((int64_t)r * ow + ox) * kpad + (int64_t)tap * C);
        const bool inside = iy >= 0 && iy < in.h && ix >= 0 && ix < in.w;
        const uint4 *src =
            reinterpret_cast<const uint4 *>(in.p + (((int64_t)b * in.h + iy) * in.w + ix) * in.pitch);
        if (warp_units) {
          for (int q = lane; q < cch; q += 32) dst[q] = inside ? src[q] : zero;
        } else {
          // all of the segment's loads before its stores (up to 16 chunks in
          // flight per thread instead of one load-store pair at a time)
          for (int q0 = 0; q0 < cch; q0 += 16) {
            uint4 v[16];
#pragma unroll
            for (int q = 0; q < 16; ++q) v[q] = (inside && q0 + q < cch) ? src[q0 + q] : zero;
#pragma unroll
            for (int q = 0; q < 16; ++q)
              if (q0 + q < cch) dst[q0 + q] = v[q];
          }
        }
        if (tap == taps - 1)
          for (int q = warp_units ? lane : 0; q < tail; q += warp_units ? 32 : 1)
            dst[cch + q] = zero;  // pad columns kdim .. kpad
      }
    }
    return;
  }
  // scalar layers (the 3-channel image): blocks walk output rows, threads
  // take (output column, 8-column chunk) units, 32-bit index arithmetic
  const int chunks = kpad / 8;
  const int rows = in.n * oh, per_row = ow * chunks;
  for (int r = blockIdx.x; r < rows; r += gridDim.x) {
    const int b = r / oh, oy = r - b * oh;
    for (int u = threadIdx.x; u < per_row; u += blockDim.x) {
      const int ox = u / chunks, col0 = (u - ox * chunks) * 8;
      __align__(16) __nv_bfloat16 v[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int col = col0 + q;
        float x = 0.0f;
        if (col < kdim) {
          const int tap = col / C, c = col - tap * C;
          const int ky = tap / k, kx = tap - ky * k;
          const int iy = oy * stride + ky - pad, ix = ox * stride + kx - pad;
          if (iy >= 0 && iy < in.h && ix >= 0 && ix < in.w)
            x = __bfloat162float(in.p[(((int64_t)b * in.h + iy) * in.w + ix) * in.pitch + c]);
        }
        v[q] = __float2bfloat16_rn(x);
      }
      *reinterpret_cast<uint4 *>(ws + ((int64_t)r * ow + ox) * kpad + col0) = *reinterpret_cast<uint4 *>(v);
    }
  }
}

// max-pool k x k / stride, window origin oy*stride - pad, taps outside the
// map skipped (Darknet's size-2 pools: pad 0; ResNet's 3x3/2: pad 1)
__global__ void __launch_bounds__(kThr) maxpool(ViewArgs in, __nv_bfloat16 *out, int oh, int ow, int opitch, int k,
                                                int stride, int pad) {
  const int cv = in.c / 8;
  const int64_t total = (int64_t)in.n * oh * ow * cv;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(t % cv) * 8;
    const int64_t p = t / cv;
    const int ox = (int)(p % ow), oy = (int)((p / ow) % oh), b = (int)(p / ((int64_t)ow * oh));
    __nv_bfloat162 m[4];
    bool first = true;
    for (int dy = 0; dy < k; ++dy)
      for (int dx = 0; dx < k; ++dx) {
        const int iy = oy * stride - pad + dy, ix = ox * stride - pad + dx;
        if (iy < 0 || iy >= in.h || ix < 0 || ix >= in.w) continue;
        const uint4 v = *reinterpret_cast<const uint4 *>(in.p + (((int64_t)b * in.h + iy) * in.w + ix) * in.pitch + c);
        const __nv_bfloat162 *h = reinterpret_cast<const __nv_bfloat162 *>(&v);
#pragma unroll
        for (int q = 0; q < 4; ++q) m[q] = first ? h[q] : __hmax2(m[q], h[q]);
        first = false;
      }
    *reinterpret_cast<uint4 *>(out + p * opitch + c) = *reinterpret_cast<uint4 *>(m);
  }
}

// global average pool: [N, H, W, C] -> [N, 1, 1, C] (fp32 sums in pixel order)
__global__ void __launch_bounds__(kThr) avgpool(ViewArgs in, __nv_bfloat16 *out, int opitch) {
  const int64_t total = (int64_t)in.n * in.c;
  const int hw = in.h * in.w;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(t % in.c);
    const int64_t b = t / in.c;
    const __nv_bfloat16 *src = in.p + b * hw * in.pitch + c;
    float s = 0.0f;
    for (int q = 0; q < hw; ++q) s += __bfloat162float(src[(int64_t)q * in.pitch]);
    out[b * opitch + c] = __float2bfloat16_rn(s / (float)hw);
  }
}

// nearest 2x upsample into a channel slice of the route tensor
__global__ void __launch_bounds__(kThr) upsample2(ViewArgs in, __nv_bfloat16 *out, int opitch) {
  const int cv = in.c / 8, oh = in.h * 2, ow = in.w * 2;
  const int64_t total = (int64_t)in.n * oh * ow * cv;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(t % cv) * 8;
    const int64_t p = t / cv;
    const int ox = (int)(p % ow), oy = (int)((p / ow) % oh), b = (int)(p / ((int64_t)ow * oh));
    *reinterpret_cast<uint4 *>(out + p * opitch + c) = *reinterpret_cast<const uint4 *>(
        in.p + (((int64_t)b * in.h + oy / 2) * in.w + ox / 2) * in.pitch + c);
  }
}

// Direct 3x3 convolution (stride 1, pad 1) for the thin first layer
// (C_in = 3 -> 16: K = 27, N = 16): an im2row matrix and a tensor-core GEMM
// with N = 16 move far more bytes than the math needs (measured 4.2 ms of a
// 7.5 ms job at 608^2 x 32), so it runs on the CUDA cores: one thread per
// output pixel, all C_out accumulators in registers (fp32 FMAs on the same
// bf16 inputs / filters), filters in shared memory as fp32, bias + leaky
// fused, 16-byte stores.
template <int CIN, int COUT>
__global__ void __launch_bounds__(kThr, 2) conv3x3_direct(ViewArgs in, const __nv_bfloat16 *__restrict__ w, int kpad,
                                                       const float *__restrict__ bias, __nv_bfloat16 *out, int opitch) {
  __shared__ __align__(16) float sW[9 * CIN][COUT];
  __shared__ float sb[COUT];
  for (int i = threadIdx.x; i < 9 * CIN * COUT; i += blockDim.x) {
    const int k = i / COUT, co = i % COUT;
    sW[k][co] = __bfloat162float(w[(int64_t)co * kpad + k]);
  }
  if (threadIdx.x < COUT) sb[threadIdx.x] = bias[threadIdx.x];
  __syncthreads();
  // pixel index -> (b, y, x) in 32-bit arithmetic (64-bit div / mod per
  // pixel cost as much as the 432 FMAs; every Darknet input here has
  // fewer than 2^31 pixels, gemm_validate's size limits)
  const unsigned pix = (unsigned)((int64_t)in.n * in.h * in.w);
  for (unsigned p = blockIdx.x * blockDim.x + threadIdx.x; p < pix; p += gridDim.x * blockDim.x) {
    const unsigned q = p / (unsigned)in.w;
    const int x = (int)(p - q * (unsigned)in.w);
    const unsigned bq = q / (unsigned)in.h;
    const int y = (int)(q - bq * (unsigned)in.h);
    const int64_t b = bq;
    float acc[COUT];
#pragma unroll
    for (int co = 0; co < COUT; ++co) acc[co] = 0.0f;
#pragma unroll
    for (int tap = 0; tap < 9; ++tap) {
      const int iy = y + tap / 3 - 1, ix = x + tap % 3 - 1;
      if (iy < 0 || iy >= in.h || ix < 0 || ix >= in.w) continue;
      const __nv_bfloat16 *src = in.p + ((b * in.h + iy) * in.w + ix) * in.pitch;
      float v[CIN];
      if constexpr (CIN % 8 == 0) {
#pragma unroll
        for (int q = 0; q < CIN / 8; ++q) {
          const uint4 u = *reinterpret_cast<const uint4 *>(src + 8 * q);
          const __nv_bfloat162 *h = reinterpret_cast<const __nv_bfloat162 *>(&u);
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float2 f = __bfloat1622float2(h[e]);
            v[8 * q + 2 * e] = f.x;
            v[8 * q + 2 * e + 1] = f.y;
          }
        }
      } else {
#pragma unroll
        for (int c = 0; c < CIN; ++c) v[c] = __bfloat162float(src[c]);
      }
#pragma unroll
      for (int c = 0; c < CIN; ++c) {
        const float4 *wr = reinterpret_cast<const float4 *>(&sW[tap * CIN + c][0]);
#pragma unroll
        for (int q = 0; q < COUT / 4; ++q) {
          const float4 ww = wr[q];
          acc[4 * q] = fmaf(v[c], ww.x, acc[4 * q]);
          acc[4 * q + 1] = fmaf(v[c], ww.y, acc[4 * q + 1]);
          acc[4 * q + 2] = fmaf(v[c], ww.z, acc[4 * q + 2]);
          acc[4 * q + 3] = fmaf(v[c], ww.w, acc[4 * q + 3]);
        }
      }
    }
    __nv_bfloat16 *dst = out + (int64_t)p * opitch;
#pragma unroll
    for (int q = 0; q < COUT / 8; ++q) {
      __align__(16) __nv_bfloat162 o[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        float a0 = acc[8 * q + 2 * e] + sb[8 * q + 2 * e], a1 = acc[8 * q + 2 * e + 1] + sb[8 * q + 2 * e + 1];
        a0 = a0 > 0.0f ? a0 : 0.1f * a0;
        a1 = a1 > 0.0f ? a1 : 0.1f * a1;
        o[e] = __floats2bfloat162_rn(a0, a1);
      }
      *reinterpret_cast<uint4 *>(dst + 8 * q) = *reinterpret_cast<const uint4 *>(o);
    }
  }
}

// YOLO layer 0 fused with the 2x2/2 max-pool that follows it: a thread owns
// one pooled pixel, i.e. a 2 x 2 block of conv outputs.  The block's 4 x 4 x 3
// input window is loaded once (48 values), every filter row of the shared
// fp32 weights (2 x float4 per 8-channel pass) feeds the 4 pixels at once
// (32 FMAs per 2 shared loads, not 8), and the pooled maximum is taken from the
// bf16 conv outputs in registers — the max-pool's re-read of the 378 MB conv
// output (608^2 x 32) is gone.  Per output pixel the FMA chain is
// conv3x3_direct's exactly (taps in order, channels inner, padding taps
// skipped), so both outputs are bit-identical to conv3x3_direct + maxpool.
template <int CIN, int COUT>
__global__ void __launch_bounds__(128, 2) conv3x3_pool2(ViewArgs in, const __nv_bfloat16 *__restrict__ w, int kpad,
                                                     const float *__restrict__ bias, __nv_bfloat16 *out, int opitch,
                                                     __nv_bfloat16 *pout, int ppitch) {
  __shared__ __align__(16) float sW[9 * CIN][COUT];
  __shared__ float sb[COUT];
  for (int i = threadIdx.x; i < 9 * CIN * COUT; i += blockDim.x) {
    const int k = i / COUT, co = i % COUT;
    sW[k][co] = __bfloat162float(w[(int64_t)co * kpad + k]);
  }
  if (threadIdx.x < COUT) sb[threadIdx.x] = bias[threadIdx.x];
  __syncthreads();
  const int ph = in.h / 2, pw = in.w / 2;
  const unsigned pix = (unsigned)((int64_t)in.n * ph * pw);
  for (unsigned p = blockIdx.x * blockDim.x + threadIdx.x; p < pix; p += gridDim.x * blockDim.x) {
    const unsigned q = p / (unsigned)pw;
    const int px = (int)(p - q * (unsigned)pw);
    const unsigned bq = q / (unsigned)ph;
    const int py = (int)(q - bq * (unsigned)ph);
    const int64_t b = bq;
    const int y0 = 2 * py - 1, x0 = 2 * px - 1;  // window origin (4 x 4)
    bool rin[4], cin[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      rin[i] = y0 + i >= 0 && y0 + i < in.h;
      cin[i] = x0 + i >= 0 && x0 + i < in.w;
    }
    float win[4][4][CIN];
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const bool ok = rin[r] && cin[c];
        const __nv_bfloat16 *src = in.p + (((b * in.h + (ok ? y0 + r : 0)) * in.w) + (ok ? x0 + c : 0)) * in.pitch;
#pragma unroll
        for (int ch = 0; ch < CIN; ++ch) win[r][c][ch] = ok ? __bfloat162float(src[ch]) : 0.0f;
      }
    auto bits = [](__nv_bfloat162 v) {
      return (uint32_t)__bfloat16_as_ushort(v.x) | ((uint32_t)__bfloat16_as_ushort(v.y) << 16);
    };
    // 8 output channels per pass (64 accumulators for all 16 spilled)
#pragma unroll 1
    for (int h8 = 0; h8 < COUT / 8; ++h8) {
      float acc[4][8];
#pragma unroll
      for (int o = 0; o < 4; ++o)
#pragma unroll
        for (int co = 0; co < 8; ++co) acc[o][co] = 0.0f;
#pragma unroll
      for (int tap = 0; tap < 9; ++tap) {
        const int ky = tap / 3, kx = tap % 3;
#pragma unroll
        for (int ch = 0; ch < CIN; ++ch) {
          const float4 *wr = reinterpret_cast<const float4 *>(&sW[tap * CIN + ch][8 * h8]);
          const float4 t0 = wr[0], t1 = wr[1];
          const float ww[8] = {t0.x, t0.y, t0.z, t0.w, t1.x, t1.y, t1.z, t1.w};
#pragma unroll
          for (int o = 0; o < 4; ++o) {
            const int r = (o >> 1) + ky, c = (o & 1) + kx;
            if (!(rin[r] && cin[c])) continue;  // conv3x3_direct skips padding taps
            const float v = win[r][c][ch];
#pragma unroll
            for (int co = 0; co < 8; ++co) acc[o][co] = fmaf(v, ww[co], acc[o][co]);
          }
        }
      }
      __nv_bfloat162 mx[4];
#pragma unroll
      for (int o = 0; o < 4; ++o) {
        const int oy = 2 * py + (o >> 1), ox = 2 * px + (o & 1);
        uint32_t ow[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int c0 = 8 * h8 + 2 * e;
          float a0 = acc[o][2 * e] + sb[c0], a1 = acc[o][2 * e + 1] + sb[c0 + 1];
          a0 = a0 > 0.0f ? a0 : 0.1f * a0;
          a1 = a1 > 0.0f ? a1 : 0.1f * a1;
          const __nv_bfloat162 v = __floats2bfloat162_rn(a0, a1);
          mx[e] = o == 0 ? v : __hmax2(mx[e], v);
          ow[e] = bits(v);
        }
        reinterpret_cast<uint4 *>(out + ((b * in.h + oy) * (int64_t)in.w + ox) * opitch)[h8] =
            make_uint4(ow[0], ow[1], ow[2], ow[3]);
      }
      reinterpret_cast<uint4 *>(pout + ((b * ph + py) * (int64_t)pw + px) * ppitch)[h8] =
          make_uint4(bits(mx[0]), bits(mx[1]), bits(mx[2]), bits(mx[3]));
    }
  }
}

ViewArgs vargs(const TView &v, const std::vector<void *> &buf) {
  return {reinterpret_cast<const __nv_bfloat16 *>(buf[v.buf]) + v.off, v.n, v.h, v.w, v.c, v.pitch};
}

// Two CTAs per SM for every kernel of the job: the GEMM's shared-memory ring
// (<= 99 KB) and the direct convolution's registers (<= 128) allow two, and
// mgb-sm places a job by its widest launch under the most demanding
// kernel's occupancy (task_builder.py:272-289 aggregation), so no grid may
// exceed 2 x 148.
int grid_for(int64_t total) { return (int)std::min<int64_t>((total + kThr - 1) / kThr, 2 * sm_count()); }

}  // namespace

// ---- job hooks (gs_work_internal.h) ------------------------------------------

int gemm_validate(const gs_job_desc &j) {
  if (j.n < 32 || j.n % 32) return err(GS_ERR_CONFIG, "network input size must be a positive multiple of 32");
  if (j.m < 1 || j.m > 1024) return err(GS_ERR_CONFIG, "network batch must be 1..1024");
  if (j.m * j.n * j.n >= (1ll << 31))  // pixel indices (GEMM rows, direct-conv pixels) are 32-bit
    return err(GS_ERR_CONFIG, "network batch x input pixels must be below 2^31");
  if (j.iters < 1) return err(GS_ERR_CONFIG, "a network job needs at least one forward pass");
  return GS_OK;
}

std::vector<Buf> gemm_buffers(const gs_job_desc &j) { return net_plan(j).bufs; }

// launch shapes for the probe: the widest launch (im2row / pool grids) and
// the GEMM's dynamic shared memory (largest tile variant the net can pick)
std::vector<Shape> gemm_launches(const gs_job_desc &j) {
  const NetPlan P = net_plan(j);
  int bn_max = 32;
  for (const LPlan &L : P.layers)
    if (L.type == CONV)
      bn_max = std::max(bn_max, gemm_pick_bn((int)((int64_t)L.out.n * L.out.h * L.out.w), L.cout));
  const int64_t pix0 = (int64_t)j.m * j.n * j.n;
  Shape g{gemm_kernel_fn(bn_max), 2 * sm_count(), gemm_block_threads()};
  g.dsmem = (int)gemm_smem_for(bn_max);
  Shape gc{conv_kernel_fn(bn_max), 2 * sm_count(), conv_block_threads()};
  gc.dsmem = (int)gemm_smem_for(bn_max);
  std::vector<Shape> v = {g, gc, {(const void *)im2row, grid_for(pix0 * 4), kThr},
                          {(const void *)maxpool, grid_for(pix0), kThr}};
  if (j.kind == GS_JOB_YOLO) {
    v.push_back({(const void *)conv3x3_direct<3, 16>, grid_for(pix0), kThr});
    v.push_back({(const void *)conv3x3_pool2<3, 16>,
                 (int)std::min<int64_t>((pix0 / 4 + 127) / 128, 2 * sm_count()), 128});
  }
  else v.push_back({(const void *)avgpool, grid_for(pix0), kThr});
  return v;
}

int gemm_generate(const gs_job_desc &j, const std::vector<void *> &dst, cudaStream_t st) {
  const NetPlan P = net_plan(j);
  const int64_t nimg = (int64_t)j.m * j.n * j.n * 3;
  gen_image<<<grid_for(nimg), kThr, 0, st>>>((__nv_bfloat16 *)dst[B_IMG], nimg, j.seed);
  int li = 0;
  for (const LPlan &L : P.layers) {
    if (L.type != CONV) continue;
    const float s = sqrtf(6.0f / (float)L.kdim);
    gen_filters<<<grid_for((int64_t)L.cout * L.kpad), kThr, 0, st>>>((__nv_bfloat16 *)dst[B_W] + L.woff, L.cout,
                                                                      L.kdim, L.kpad, s, j.seed + 100 + li);
    gen_bias<<<grid_for(L.cout), kThr, 0, st>>>((float *)dst[B_BIAS] + L.boff, L.cout, j.seed + 200 + li);
    ++li;
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return err(GS_ERR_CUDA, std::string("network generate: ") + cudaGetErrorString(e));
  return GS_OK;
}

// the YOLO layer-0 convolution followed by a 2x2/2 max-pool of its output
static bool fuse_pool(const LPlan &L, const LPlan &M) {
  static const bool off = [] {
    const char *e = getenv("GS_NO_POOL_FUSION");
    return e && e[0] == '1';
  }();
  return !off && M.type == MAXPOOL && M.k == 2 && M.stride == 2 && M.pad == 0 && M.in.buf == L.out.buf &&
         M.in.off == L.out.off && L.in.h % 2 == 0 && L.in.w % 2 == 0 && !M.out.f32 && M.out.off % 8 == 0 &&
         M.out.pitch % 8 == 0;
}
static int pool2_grid(const LPlan &L) {
  const int64_t units = (int64_t)L.in.n * (L.in.h / 2) * (L.in.w / 2);
  return (int)std::min<int64_t>((units + 127) / 128, 2 * sm_count());
}

int gemm_run(const gs_job_desc &j, std::vector<void *> &buf, cudaStream_t st, int *out_idx, int64_t *launches,
             unsigned *tk) {
  const NetPlan P = net_plan(j);
  for (int pass = 0; pass < j.iters; ++pass) {
    for (size_t li = 0; li < P.layers.size(); ++li) {
      const LPlan &L = P.layers[li];
      const ViewArgs in = vargs(L.in, buf);
      __nv_bfloat16 *obf = L.out.f32 ? nullptr : (__nv_bfloat16 *)buf[L.out.buf] + L.out.off;
      if (L.type == MAXPOOL) {
        maxpool<<<grid_for((int64_t)L.out.n * L.out.h * L.out.w * (L.in.c / 8)), kThr, 0, st>>>(
            in, obf, L.out.h, L.out.w, L.out.pitch, L.k, L.stride, L.pad);
        ++*launches;
        continue;
      }
      if (L.type == UPSAMPLE) {
        upsample2<<<grid_for((int64_t)L.in.n * L.in.h * L.in.w * 4 * (L.in.c / 8)), kThr, 0, st>>>(in, obf,
                                                                                                    L.out.pitch);
        ++*launches;
        continue;
      }
      if (L.type == AVGPOOL) {
        avgpool<<<grid_for((int64_t)L.in.n * L.in.c), kThr, 0, st>>>(in, obf, L.out.pitch);
        ++*launches;
        continue;
      }
      const int64_t opix = (int64_t)L.out.n * L.out.h * L.out.w;
      if (L.k == 3 && L.stride == 1 && L.act == LEAKY && !L.out.f32 && L.out.off % 8 == 0 && L.out.pitch % 8 == 0 &&
          L.in.c == 3 && L.cout == 16) {
        // YOLO layer 0 (K = 27): direct convolution (measured 0.6 ms vs 4.2 ms
        // for im2row + GEMM at 608^2 x 32; for 16 -> 32 the GEMM path is faster)
        if (li + 1 < P.layers.size() && fuse_pool(L, P.layers[li + 1])) {
          const LPlan &M = P.layers[li + 1];
          conv3x3_pool2<3, 16><<<pool2_grid(L), 128, 0, st>>>(
              in, (const __nv_bfloat16 *)buf[B_W] + L.woff, L.kpad, (const float *)buf[B_BIAS] + L.boff, obf,
              L.out.pitch, (__nv_bfloat16 *)buf[M.out.buf] + M.out.off, M.out.pitch);
          ++*launches;
          ++li;  // the max-pool's output is written too
          continue;
        }
        conv3x3_direct<3, 16><<<grid_for(opix), kThr, 0, st>>>(in, (const __nv_bfloat16 *)buf[B_W] + L.woff, L.kpad,
                                                               (const float *)buf[B_BIAS] + L.boff, obf, L.out.pitch);
        ++*launches;
        continue;
      }
      void *cout_p = L.out.f32 ? (void *)((float *)buf[L.out.buf] + L.out.off) : (void *)obf;
      const void *cres =
          L.res.buf >= 0 ? (const void *)((const __nv_bfloat16 *)buf[L.res.buf] + L.res.off) : nullptr;
      if (NetBuilder::implicit_conv(L)) {
        int rc = conv_gemm_bf16(in.p, L.in.n, L.in.h, L.in.w, L.in.pitch, __builtin_ctz(L.in.c), L.out.h, L.out.w,
                                L.k, L.stride, L.pad, (const __nv_bfloat16 *)buf[B_W] + L.woff, L.kpad,
                                (const float *)buf[B_BIAS] + L.boff, cout_p, L.out.pitch, L.cout, L.out.f32 ? 1 : 0,
                                L.act, 2 * sm_count(), st, cres, L.res.pitch, tk);
        if (rc) return rc;
        ++*launches;
        continue;
      }
      const void *A;
      int64_t lda;
      if (NetBuilder::direct_gemm(L)) {
        A = in.p;  // 1x1 / stride 1: the activation is already the im2row matrix
        lda = L.in.pitch;
      } else {
        const int grid = (int)std::min<int64_t>((int64_t)L.in.n * L.out.h, 2 * sm_count());  // blocks walk output rows
        im2row<<<grid, kThr, 0, st>>>(in, (__nv_bfloat16 *)buf[B_WS], L.k, L.stride, L.pad, L.out.h, L.out.w,
                                      L.kdim, L.kpad);
        ++*launches;
        A = buf[B_WS];
        lda = L.kpad;
      }
      void *out = L.out.f32 ? (void *)((float *)buf[L.out.buf] + L.out.off) : (void *)obf;
      const void *res = L.res.buf >= 0 ? (const void *)((const __nv_bfloat16 *)buf[L.res.buf] + L.res.off) : nullptr;
      int rc = gemm_bf16(A, lda, (const __nv_bfloat16 *)buf[B_W] + L.woff, L.kpad, (const float *)buf[B_BIAS] + L.boff,
                         out, L.out.pitch, (int)opix, L.cout, L.kpad, L.out.f32 ? 1 : 0, L.act, 2 * sm_count(), st, res,
                         L.res.pitch, tk);
      if (rc) return rc;
      ++*launches;
    }
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return err(GS_ERR_CUDA, std::string("network run: ") + cudaGetErrorString(e));
  *out_idx = B_DET;
  return GS_OK;
}

}  // namespace gsw
