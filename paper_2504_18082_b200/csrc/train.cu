// train.cu -- NEXT-4: the loss and the optimizer step that close one training
// step of the paper's 3-layer GraphSAGE.  PAPER.md P:503: "The goal of training is to learn the
// layer parameters W^1 .. W^{L-1} by minimizing the loss between the labels of all labeled nodes
// and the node embeddings of the last layer"; DGL's GraphSAGE defaults, learning rate 1e-3,
// weight decay 5e-4.  Readings R33 (softmax cross-entropy, mean over the batch's roots) and R34
// (Adam with L2 weight decay added to the gradient, DGL's optimizer) in DESIGN.md.
#include <cuda_bf16.h>

#include <cmath>
#include <cstdint>

#include "common.cuh"

namespace cmb {
namespace tr {

constexpr unsigned kFull = 0xffffffffu;

// R33: for root i < n (label_i = node_labels[nodes[i]]; the roots are the prefix of `nodes`),
//     loss = (1/n) sum_i [ lse_i - Y[i, label_i] ],  lse_i = m_i + log sum_c exp(Y[i, c] - m_i),
//     dY[i, c] = (exp(Y[i, c] - lse_i) - 1[c == label_i]) / n     (c < C; columns C.. of dY = 0).
// k_xent_rows: one warp per root (a row is one latency chain: loads, max and sum shuffles, log),
// lane j owning columns j, j + 32, ... (C <= 256); the row's loss term goes to row_loss[i] (fp64).
// k_xent_sum: one block sums row_loss in a fixed order (below) -- deterministic.  A label outside [0, C)
// sets the status word (CMB_ERR_INVALID_ARGUMENT); that row contributes nothing.
constexpr int kRowWarps = 8;
__global__ void __launch_bounds__(kRowWarps * 32)
    k_xent_rows(const float* __restrict__ logits, int64_t ld, const int32_t* __restrict__ node_labels,
                const int32_t* __restrict__ nodes, const int64_t* __restrict__ n_dev, int64_t n_cap,
                int C, __nv_bfloat16* __restrict__ dy, int64_t dy_ld, int dy_cols,
                double* __restrict__ row_loss, int32_t* __restrict__ status) {
  const int lane = threadIdx.x & 31;
  const int64_t n = min(*n_dev, n_cap);
  const int64_t i = static_cast<int64_t>(blockIdx.x) * kRowWarps + (threadIdx.x >> 5);
  if (i >= n) return;  // warp-uniform
  const float inv_n = 1.0f / static_cast<float>(n);
  const int32_t lab = __ldg(node_labels + __ldg(nodes + i));
  const bool ok = lab >= 0 && lab < C;
  if (!ok && lane == 0 && status) atomicCAS(status, 0, CMB_ERR_INVALID_ARGUMENT);
  float y[8];
  float m = -INFINITY;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int c = lane + 32 * k;
    y[k] = c < C ? __ldg(logits + i * ld + c) : -INFINITY;
    m = fmaxf(m, y[k]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(kFull, m, o));
  float s = 0.f, ylab = 0.f;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    s += lane + 32 * k < C ? expf(y[k] - m) : 0.f;
    if (lane + 32 * k == lab) ylab = y[k];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    s += __shfl_xor_sync(kFull, s, o);
    ylab += __shfl_xor_sync(kFull, ylab, o);
  }
  const float lse = m + logf(s);
  if (lane == 0) row_loss[i] = ok ? static_cast<double>(lse) - static_cast<double>(ylab) : 0.0;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int c = lane + 32 * k;
    if (c < dy_cols) {
      float g = 0.f;
      if (c < C && ok) g = (expf(y[k] - lse) - (c == lab ? 1.f : 0.f)) * inv_n;
      dy[i * dy_ld + c] = __float2bfloat16_rn(g);
    }
  }
}

constexpr int kSumThreads = 256;
__global__ void __launch_bounds__(kSumThreads)
    k_xent_sum(const double* __restrict__ row_loss, const int64_t* __restrict__ n_dev,
               int64_t n_cap, double* __restrict__ loss) {
  // fixed order: thread t adds rows t, t + 256, ... in order; a fixed xor-shuffle tree per warp;
  // thread 0 adds the 8 warp sums in warp order (deterministic, no serial 1024-term loop)
  __shared__ double wsum[kSumThreads / 32];
  const int64_t n = min(*n_dev, n_cap);
  double t = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += kSumThreads) t += row_loss[i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(kFull, t, o);
  if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = t;
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0;
    for (int w = 0; w < kSumThreads / 32; ++w) a += wsum[w];
    *loss = n > 0 ? a / static_cast<double>(n) : 0.0;
  }
}

// R34: Adam (torch.optim.Adam semantics, the optimizer of DGL's GraphSAGE example) with L2 weight
// decay added to the gradient, on a flat fp32 parameter buffer:
//     g = dW + wd * w;  m = b1 m + (1 - b1) g;  v = b2 v + (1 - b2) g^2;
//     w -= lr * (m * c1) / (sqrt(v * c2) + eps),  c1 = 1 / (1 - b1^t), c2 = 1 / (1 - b2^t).
// 1 - b1, 1 - b2 and the bias corrections are computed on the host in fp64 and rounded once
// (1 - 0.999f in fp32 would be off by 1.3e-5 relative).  HBM-bound elementwise (16 bytes read +
// 12 written per parameter), float4 per thread.
__global__ void __launch_bounds__(256)
    k_adam(float4* __restrict__ w, const float4* __restrict__ g, float4* __restrict__ m,
           float4* __restrict__ v, int64_t n4, float lr, float b1, float b2, float omb1,
           float omb2, float eps, float wd, float c1, float c2) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n4;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    float4 W = w[i], G = __ldg(g + i), M = m[i], V = v[i];
    float* pw = &W.x;
    const float* pg = &G.x;
    float* pm = &M.x;
    float* pv = &V.x;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float gk = __fmaf_rn(wd, pw[k], pg[k]);
      pm[k] = __fmaf_rn(b1, pm[k], omb1 * gk);
      pv[k] = __fmaf_rn(b2, pv[k], omb2 * gk * gk);
      const float den = __fsqrt_rn(pv[k] * c2) + eps;
      pw[k] = pw[k] - lr * __fdiv_rn(pm[k] * c1, den);
    }
    w[i] = W;
    m[i] = M;
    v[i] = V;
  }
}

// cmb_adam_step_pack: the Adam update of k_adam, then every updated W element rounded to bf16
// and stored at its place in the layer's forward image (row n = output column, K column c, half
// h) and transposed image (row c, K column n, half h).  Element-per-thread over the flat buffer.
constexpr int kMaxPackLayers = 8;
struct PackTable {
  int n_layers;
  int64_t offset[kMaxPackLayers + 1];
  int in_dim[kMaxPackLayers], out_dim[kMaxPackLayers];
  __nv_bfloat16* img[kMaxPackLayers];
  __nv_bfloat16* img_t[kMaxPackLayers];
  int dense[kMaxPackLayers];  // img in the dense.cu layout: row (h * Fp + c), column o
};

// step_dev != NULL: the step number is read on the device (after k_step_next advanced it) and
// the bias corrections c1, c2 formed from it in fp64 there -- the form a captured CUDA graph
// replays (no host value baked into the launch)
__global__ void k_step_next(int32_t* step) { *step += 1; }

__global__ void __launch_bounds__(256)
    k_adam_pack(float* __restrict__ w, const float* __restrict__ g, float* __restrict__ m,
                float* __restrict__ v, int64_t n, float lr, float b1, float b2, float omb1,
                float omb2, float eps, float wd, float c1, float c2,
                const __grid_constant__ PackTable t, const int32_t* __restrict__ step_dev,
                double b1d, double b2d) {
  if (step_dev) {
    __shared__ float c12[2];
    if (threadIdx.x == 0) {
      const int s = *step_dev;
      c12[0] = static_cast<float>(1.0 / (1.0 - pow(b1d, s)));
      c12[1] = static_cast<float>(1.0 / (1.0 - pow(b2d, s)));
    }
    __syncthreads();
    c1 = c12[0];
    c2 = c12[1];
  }
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const float gk = __fmaf_rn(wd, w[i], __ldg(g + i));
    const float mk = __fmaf_rn(b1, m[i], omb1 * gk);
    const float vk = __fmaf_rn(b2, v[i], omb2 * gk * gk);
    const float den = __fsqrt_rn(vk * c2) + eps;
    const float wk = w[i] - lr * __fdiv_rn(mk * c1, den);
    w[i] = wk;
    m[i] = mk;
    v[i] = vk;
    int l = 0;
    while (l + 1 < t.n_layers && i >= t.offset[l + 1]) ++l;
    const int F = t.in_dim[l], fo = t.out_dim[l];
    const int64_t j = i - t.offset[l];
    const int64_t per = static_cast<int64_t>(F) * fo;
    if (j < 2 * per) {  // a weight (the bias has no image)
      const int h = static_cast<int>(j / per);
      const int r = static_cast<int>(j - h * per);
      const int c = r / fo, o = r - c * fo;
      const __nv_bfloat16 bv = __float2bfloat16_rn(wk);
      if (t.dense[l]) {
        const int64_t fp = (F + 7) / 8 * 8;
        t.img[l][(h * fp + c) * fo + o] = bv;
        continue;
      }
      t.img[l][sw128_off(o, h, c, (F + 63) / 64, fo) >> 1] = bv;
      if (t.img_t[l]) t.img_t[l][sw128_off(c, h, o, (fo + 63) / 64, F) >> 1] = bv;
    }
  }
}

}  // namespace tr
}  // namespace cmb

using namespace cmb;

extern "C" {

cmb_status cmb_softmax_xent(const float* logits, int64_t ld, const int32_t* node_labels,
                            const int32_t* nodes, const int64_t* n_dev, int64_t n_cap,
                            int32_t num_classes, void* dy, int64_t dy_ld, int32_t dy_cols,
                            double* loss, double* row_loss, int32_t* status, void* stream) {
  CMB_NVTX("cmb.next4.softmax_xent");
  CMB_ARG(logits && node_labels && nodes && n_dev && dy && loss && row_loss,
          "cmb_softmax_xent: null argument");
  CMB_ARG(num_classes >= 1 && num_classes <= 256 && dy_cols >= num_classes && dy_cols <= 256 &&
              ld >= num_classes &&
              dy_ld >= dy_cols && n_cap >= 0,
          "cmb_softmax_xent: need 1 <= num_classes <= 256 <= ..., dy_cols >= num_classes, "
          "ld / dy_ld >= their widths (got C=%d, dy_cols=%d)", num_classes, dy_cols);
  cmb_status st = require_sm100();
  if (st != CMB_OK) return st;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (n_cap > 0) {
    tr::k_xent_rows<<<static_cast<int>((n_cap + tr::kRowWarps - 1) / tr::kRowWarps),
                      tr::kRowWarps * 32, 0, s>>>(logits, ld, node_labels, nodes, n_dev, n_cap,
                                                  num_classes, static_cast<__nv_bfloat16*>(dy),
                                                  dy_ld, dy_cols, row_loss, status);
    CMB_CUDA(cudaGetLastError());
  }
  tr::k_xent_sum<<<1, tr::kSumThreads, 0, s>>>(row_loss, n_dev, n_cap, loss);
  CMB_CUDA(cudaGetLastError());
  return CMB_OK;
}

cmb_status cmb_adam_step(float* w, const float* g, float* m, float* v, int64_t n, double lr,
                         double beta1, double beta2, double eps, double weight_decay, int32_t step,
                         void* stream) {
  CMB_NVTX("cmb.next4.adam_step");
  CMB_ARG(w && g && m && v, "cmb_adam_step: null argument");
  CMB_ARG(n >= 0 && n % 4 == 0 && step >= 1 && beta1 >= 0.0 && beta1 < 1.0 && beta2 >= 0.0 &&
              beta2 < 1.0,
          "cmb_adam_step: need n %% 4 == 0, step >= 1, betas in [0, 1)");
  CMB_ARG(((reinterpret_cast<uintptr_t>(w) | reinterpret_cast<uintptr_t>(g) |
            reinterpret_cast<uintptr_t>(m) | reinterpret_cast<uintptr_t>(v)) & 15u) == 0,
          "cmb_adam_step: buffers must be 16-byte aligned");
  if (n == 0) return CMB_OK;
  cmb_status st = require_sm100();
  if (st != CMB_OK) return st;
  const double c1 = 1.0 / (1.0 - std::pow(beta1, step));
  const double c2 = 1.0 / (1.0 - std::pow(beta2, step));
  const int64_t n4 = n / 4;
  const int grid = static_cast<int>(n4 / 256 + 1 < 148 * 8 ? n4 / 256 + 1 : 148 * 8);
  tr::k_adam<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<float4*>(w), reinterpret_cast<const float4*>(g),
      reinterpret_cast<float4*>(m), reinterpret_cast<float4*>(v), n4, static_cast<float>(lr),
      static_cast<float>(beta1), static_cast<float>(beta2), static_cast<float>(1.0 - beta1),
      static_cast<float>(1.0 - beta2), static_cast<float>(eps), static_cast<float>(weight_decay),
      static_cast<float>(c1), static_cast<float>(c2));
  CMB_CUDA(cudaGetLastError());
  return CMB_OK;
}

namespace {
cmb_status adam_step_pack(float* w, const float* g, float* m, float* v, int64_t n, double lr,
                          double beta1, double beta2, double eps, double weight_decay,
                          int32_t step, int32_t* step_dev, const cmb_layer_pack* layers,
                          int32_t n_layers, void* stream) {
  CMB_ARG(w && g && m && v && layers, "cmb_adam_step_pack: null argument");
  CMB_ARG(n >= 0 && (step >= 1 || step_dev) && beta1 >= 0.0 && beta1 < 1.0 && beta2 >= 0.0 &&
              beta2 < 1.0 &&
              n_layers >= 1 && n_layers <= tr::kMaxPackLayers,
          "cmb_adam_step_pack: need step >= 1, betas in [0, 1), 1 <= n_layers <= 8");
  tr::PackTable t{};
  t.n_layers = n_layers;
  int64_t at = 0;
  for (int l = 0; l < n_layers; ++l) {
    const cmb_layer_pack& L = layers[l];
    CMB_ARG(L.offset == at && L.in_dim >= 1 && (L.dense || L.in_dim <= 256) &&
                L.out_dim >= 16 && L.out_dim <= 256 && L.out_dim % 16 == 0 && L.img &&
                (!L.dense || !L.img_t),
            "cmb_adam_step_pack: layer %d: offsets must tile the buffer in order, 1 <= in_dim <= "
            "256 (any for a dense image), out_dim in [16, 256] a multiple of 16, img non-null, "
            "no transposed image with a dense one", l);
    t.offset[l] = L.offset;
    t.in_dim[l] = L.in_dim;
    t.out_dim[l] = L.out_dim;
    t.img[l] = static_cast<__nv_bfloat16*>(L.img);
    t.img_t[l] = static_cast<__nv_bfloat16*>(L.img_t);
    t.dense[l] = L.dense ? 1 : 0;
    at += 2ll * L.in_dim * L.out_dim + L.out_dim;
  }
  CMB_ARG(at == n, "cmb_adam_step_pack: the layers cover %lld parameters, n = %lld",
          static_cast<long long>(at), static_cast<long long>(n));
  t.offset[n_layers] = n;
  if (n == 0) return CMB_OK;
  cmb_status st = require_sm100();
  if (st != CMB_OK) return st;
  const double c1 = step_dev ? 1.0 : 1.0 / (1.0 - std::pow(beta1, step));
  const double c2 = step_dev ? 1.0 : 1.0 / (1.0 - std::pow(beta2, step));
  const int grid = static_cast<int>(n / 256 + 1 < 148 * 8 ? n / 256 + 1 : 148 * 8);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (step_dev) {
    tr::k_step_next<<<1, 1, 0, s>>>(step_dev);
    CMB_CUDA(cudaGetLastError());
  }
  tr::k_adam_pack<<<grid, 256, 0, s>>>(
      w, g, m, v, n, static_cast<float>(lr), static_cast<float>(beta1), static_cast<float>(beta2),
      static_cast<float>(1.0 - beta1), static_cast<float>(1.0 - beta2), static_cast<float>(eps),
      static_cast<float>(weight_decay), static_cast<float>(c1), static_cast<float>(c2), t,
      step_dev, beta1, beta2);
  CMB_CUDA(cudaGetLastError());
  return CMB_OK;
}
}  // namespace

cmb_status cmb_adam_step_pack(float* w, const float* g, float* m, float* v, int64_t n, double lr,
                              double beta1, double beta2, double eps, double weight_decay,
                              int32_t step, const cmb_layer_pack* layers, int32_t n_layers,
                              void* stream) {
  CMB_NVTX("cmb.next4.adam_step_pack");
  return adam_step_pack(w, g, m, v, n, lr, beta1, beta2, eps, weight_decay, step, nullptr, layers,
                        n_layers, stream);
}

cmb_status cmb_adam_step_pack_dev(float* w, const float* g, float* m, float* v, int64_t n,
                                  double lr, double beta1, double beta2, double eps,
                                  double weight_decay, int32_t* step,
                                  const cmb_layer_pack* layers, int32_t n_layers, void* stream) {
  CMB_NVTX("cmb.next4.adam_step_pack_dev");
  CMB_ARG(step != nullptr, "cmb_adam_step_pack_dev: null step counter");
  return adam_step_pack(w, g, m, v, n, lr, beta1, beta2, eps, weight_decay, 0, step, layers,
                        n_layers, stream);
}

}  // extern "C"
