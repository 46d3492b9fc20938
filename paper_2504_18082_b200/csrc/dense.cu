// dense.cu -- NEXT-4 for wide feature rows (F > 128, e.g. Reddit's F = 602): the
// input-side GraphSAGE layer (reading R26) and its weight gradients (reading R27) when the fused
// tcgen05 kernel (sage_layer.cu) cannot keep K = 2F resident in shared memory.
//
// The a4 + a5 outputs X_in / H come from the fused gather (cmb_gather_aggregate); then
//   pack    A = [bf16(X_dst) | bf16(H)]  rows < n (rows n .. cap zero), K = 2 * Fp (Fp = F
//           rounded up to 8, pad columns zero) -- bf16 operands as in the fused kernel (R26)
//   GEMM    Z = A W, W = [W_self; W_neigh] packed the same way (bf16, K x Fo)      (cuBLASLt)
//   epilogue Y = sigma(Z + b) -> bf16 / fp32, rows >= n zero
// and for the backward
//   mask    dZ = dY * 1[Y > 0] -> bf16 (rows >= n zero), column sums for db (fixed order)
//   GEMM    dW = A^T dZ (fp32 accumulation)                                           (cuBLASLt)
//   unpack  dW -> [dW_self | dW_neigh] (F x Fo each, the model's flat layout)
// The two GEMMs are plain dense products, the one place the library calls a library GEMM
// (cuBLASLt, bf16 x bf16 -> fp32); every other step is this file's kernels.  Bounds: R26 / R27
// (bf16 operands, fp32 accumulation), the same as the fused layer.
#include <cublasLt.h>
#include <cuda_bf16.h>

#include <map>
#include <mutex>

#include "common.cuh"

namespace cmb {
namespace dn {

inline int64_t padk(int32_t f) { return (f + 7) / 8 * 8; }

// A[r, 0:2Fp] = [bf16(x[r, 0:F]), 0.., bf16(h[r, 0:F]), 0..] for r < n, zero rows for r >= n.
__global__ void k_pack_a(const float* __restrict__ x, int64_t x_ld, const float* __restrict__ h,
                         int64_t h_ld, const int64_t* __restrict__ n_dev, int64_t cap, int f,
                         int64_t fp, __nv_bfloat16* __restrict__ a) {
  const int64_t n = min(*n_dev, cap);
  const int64_t k2 = 2 * fp;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < cap * k2;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / k2, c = i % k2;
    float v = 0.f;
    if (r < n) {
      if (c < f) v = x[r * x_ld + c];
      else if (c >= fp && c - fp < f) v = h[r * h_ld + (c - fp)];
    }
    a[i] = __float2bfloat16_rn(v);
  }
}

// W = [bf16(w_self); 0..; bf16(w_neigh); 0..], K = 2Fp rows of Fo (row-major)
__global__ void k_pack_w(const float* __restrict__ ws, const float* __restrict__ wn, int f,
                         int64_t fp, int fo, __nv_bfloat16* __restrict__ w) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < 2 * fp * fo;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = i / fo, o = i % fo;
    float v = 0.f;
    if (k < f) v = ws[k * fo + o];
    else if (k >= fp && k - fp < f) v = wn[(k - fp) * fo + o];
    w[i] = __float2bfloat16_rn(v);
  }
}

// Y = sigma(Z + b) for rows < n (bf16 or fp32), zero rows for n <= r < cap
__global__ void k_epilogue(const float* __restrict__ z, const float* __restrict__ bias,
                           const int64_t* __restrict__ n_dev, int64_t cap, int fo, int relu,
                           int out_bf16, void* __restrict__ out, int64_t out_ld) {
  const int64_t n = min(*n_dev, cap);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < cap * fo;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / fo;
    const int o = static_cast<int>(i % fo);
    float v = 0.f;
    if (r < n) {
      v = z[i] + (bias ? bias[o] : 0.f);
      if (relu) v = fmaxf(v, 0.f);
    }
    if (out_bf16)
      static_cast<__nv_bfloat16*>(out)[r * out_ld + o] = __float2bfloat16_rn(v);
    else
      static_cast<float*>(out)[r * out_ld + o] = v;
  }
}

// dZ = bf16(dY) * 1[Y > 0] (y == NULL: identity) for rows < n, zero rows beyond; per-block column
// partial sums of dZ for db (block b owns rows b, b + grid, ...; fixed order inside)
constexpr int kMaskThreads = 256;
__global__ void __launch_bounds__(kMaskThreads)
    k_mask_dz(const void* __restrict__ dy, int64_t dy_ld, int dy_f32,
              const __nv_bfloat16* __restrict__ y, int64_t y_ld, const int64_t* __restrict__ n_dev,
              int64_t cap, int fo, __nv_bfloat16* __restrict__ dz, float* __restrict__ part) {
  const int64_t n = min(*n_dev, cap);
  for (int o = threadIdx.x; o < fo; o += kMaskThreads) {
    float acc = 0.f;
    for (int64_t r = blockIdx.x; r < cap; r += gridDim.x) {
      float g = 0.f;
      if (r < n) {
        g = dy_f32 ? static_cast<const float*>(dy)[r * dy_ld + o]
                   : __bfloat162float(static_cast<const __nv_bfloat16*>(dy)[r * dy_ld + o]);
        g = __bfloat162float(__float2bfloat16_rn(g));  // the GEMM operand's value
        if (y && !(__bfloat162float(y[r * y_ld + o]) > 0.f)) g = 0.f;
      }
      dz[r * fo + o] = __float2bfloat16_rn(g);
      acc += g;
    }
    part[static_cast<int64_t>(blockIdx.x) * fo + o] = acc;
  }
}

// db[o] = sum of the block partials in fp64, fixed order; dW unpacked from the K = 2Fp rows
__global__ void k_finish(const float* __restrict__ part, int nparts, const float* __restrict__ dwk,
                         int f, int64_t fp, int fo, float* __restrict__ dw, float* __restrict__ db) {
  const int64_t total = 2ll * f * fo + fo;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (i < 2ll * f * fo) {
      const int64_t hf = i / fo, o = i % fo;  // hf = half * F + feature
      const int64_t half = hf / f, c = hf % f;
      dw[i] = dwk[(half * fp + c) * fo + o];
    } else {
      const int o = static_cast<int>(i - 2ll * f * fo);
      double s = 0.0;
      for (int p = 0; p < nparts; ++p) s += part[static_cast<int64_t>(p) * fo + o];
      db[o] = static_cast<float>(s);
    }
  }
}

constexpr int kMaskBlocks = 148;
constexpr size_t kLtWorkspace = 32u << 20;

// one cuBLASLt handle per device (created on first use, thread-safe)
cmb_status lt_handle(cublasLtHandle_t* out) {
  static std::mutex mu;
  static std::map<int, cublasLtHandle_t> handles;
  int dev = 0;
  CMB_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  auto it = handles.find(dev);
  if (it == handles.end()) {
    cublasLtHandle_t h = nullptr;
    if (cublasLtCreate(&h) != CUBLAS_STATUS_SUCCESS) {
      set_error("cuBLASLt: cublasLtCreate failed");
      return CMB_ERR_CUDA;
    }
    it = handles.emplace(dev, h).first;
  }
  *out = it->second;
  return CMB_OK;
}

#define CMB_LT(call)                                                        \
  do {                                                                      \
    const cublasStatus_t s_ = (call);                                       \
    if (s_ != CUBLAS_STATUS_SUCCESS) {                                      \
      ::cmb::set_error("cuBLASLt: %s failed (status %d)", #call, (int)s_); \
      st = CMB_ERR_CUDA;                                                    \
      goto done;                                                            \
    }                                                                       \
  } while (0)

// D (m x n, column-major, fp32, ld m) = op(A) (m x k) * op(B) (k x n), bf16 operands, fp32 accumulate
cmb_status lt_gemm(cublasOperation_t ta, cublasOperation_t tb, int64_t m, int64_t n, int64_t k,
                   const void* a, int64_t lda, const void* b, int64_t ldb, float* d,
                   void* ws, size_t ws_bytes, cudaStream_t s) {
  cublasLtHandle_t h;
  cmb_status st = lt_handle(&h);
  if (st != CMB_OK) return st;
  cublasLtMatmulDesc_t op = nullptr;
  cublasLtMatrixLayout_t la = nullptr, lb = nullptr, ld = nullptr;
  cublasLtMatmulPreference_t pref = nullptr;
  cublasLtMatmulHeuristicResult_t heur{};
  int found = 0;
  const float alpha = 1.f, beta = 0.f;
  CMB_LT(cublasLtMatmulDescCreate(&op, CUBLAS_COMPUTE_32F, CUDA_R_32F));
  CMB_LT(cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_TRANSA, &ta, sizeof(ta)));
  CMB_LT(cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_TRANSB, &tb, sizeof(tb)));
  CMB_LT(cublasLtMatrixLayoutCreate(&la, CUDA_R_16BF, ta == CUBLAS_OP_N ? m : k,
                                    ta == CUBLAS_OP_N ? k : m, lda));
  CMB_LT(cublasLtMatrixLayoutCreate(&lb, CUDA_R_16BF, tb == CUBLAS_OP_N ? k : n,
                                    tb == CUBLAS_OP_N ? n : k, ldb));
  CMB_LT(cublasLtMatrixLayoutCreate(&ld, CUDA_R_32F, m, n, m));
  CMB_LT(cublasLtMatmulPreferenceCreate(&pref));
  CMB_LT(cublasLtMatmulPreferenceSetAttribute(pref, CUBLASLT_MATMUL_PREF_MAX_WORKSPACE_BYTES,
                                              &ws_bytes, sizeof(ws_bytes)));
  CMB_LT(cublasLtMatmulAlgoGetHeuristic(h, op, la, lb, ld, ld, pref, 1, &heur, &found));
  if (found < 1) {
    set_error("cuBLASLt: no algorithm for a %lld x %lld x %lld bf16 GEMM", (long long)m,
              (long long)n, (long long)k);
    st = CMB_ERR_CUDA;
    goto done;
  }
  CMB_LT(cublasLtMatmul(h, op, &alpha, a, la, b, lb, &beta, d, ld, d, ld, &heur.algo, ws, ws_bytes,
                        s));
done:
  if (pref) cublasLtMatmulPreferenceDestroy(pref);
  if (ld) cublasLtMatrixLayoutDestroy(ld);
  if (lb) cublasLtMatrixLayoutDestroy(lb);
  if (la) cublasLtMatrixLayoutDestroy(la);
  if (op) cublasLtMatmulDescDestroy(op);
  return st;
}

// workspace: A image [cap x 2Fp] bf16 | fp32 scratch [cap x Fo] (Z, or dW [2Fp x Fo]) |
// dZ [cap x Fo] bf16 | db partials [kMaskBlocks x Fo] | cuBLASLt workspace
struct DenseWs {
  __nv_bfloat16* a;
  float* z;
  __nv_bfloat16* dz;
  float* part;
  void* lt;
};
DenseWs carve(void* base, int64_t cap, int32_t f, int32_t fo, size_t* bytes) {
  const int64_t fp = padk(f);
  Carver c(base);
  DenseWs w;
  w.a = c.take<__nv_bfloat16>(static_cast<size_t>(cap) * 2 * fp);
  const int64_t zr = cap > 2 * fp ? cap : 2 * fp;
  w.z = c.take<float>(static_cast<size_t>(zr) * fo);
  w.dz = c.take<__nv_bfloat16>(static_cast<size_t>(cap) * fo);
  w.part = c.take<float>(static_cast<size_t>(kMaskBlocks) * fo);
  w.lt = c.take<char>(kLtWorkspace);
  if (bytes) *bytes = c.bytes();
  return w;
}

}  // namespace dn
}  // namespace cmb

using namespace cmb;

extern "C" {

size_t cmb_sage_dense_weights_bytes(int32_t feat_dim, int32_t out_dim) {
  if (feat_dim < 1 || out_dim < 8 || out_dim % 8) return 0;
  return static_cast<size_t>(2 * dn::padk(feat_dim)) * out_dim * sizeof(__nv_bfloat16);
}

size_t cmb_sage_dense_workspace_bytes(int64_t n_rows_cap, int32_t feat_dim, int32_t out_dim) {
  if (n_rows_cap < 1 || cmb_sage_dense_weights_bytes(feat_dim, out_dim) == 0) return 0;
  size_t b = 0;
  dn::carve(nullptr, n_rows_cap, feat_dim, out_dim, &b);
  return b;
}

cmb_status cmb_sage_dense_pack_weights(const float* w_self, const float* w_neigh, int32_t feat_dim,
                                       int32_t out_dim, void* w_img, size_t w_img_bytes,
                                       void* stream) {
  CMB_NVTX("cmb.next4.sage_dense_pack_weights");
  CMB_ARG(w_self && w_neigh && w_img, "cmb_sage_dense_pack_weights: null argument");
  const size_t need = cmb_sage_dense_weights_bytes(feat_dim, out_dim);
  CMB_ARG(need != 0 && w_img_bytes >= need,
          "cmb_sage_dense_pack_weights: need feat_dim >= 1, out_dim a multiple of 8 and "
          "w_img_bytes >= %zu", need);
  const int64_t fp = dn::padk(feat_dim);
  dn::k_pack_w<<<148 * 4, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      w_self, w_neigh, feat_dim, fp, out_dim, static_cast<__nv_bfloat16*>(w_img));
  CMB_CUDA(cudaGetLastError());
  return CMB_OK;
}

cmb_status cmb_sage_dense_forward(const float* x_dst, int64_t x_ld, const float* h, int64_t h_ld,
                                  const int64_t* n_dev, int64_t n_rows_cap, int32_t feat_dim,
                                  const void* w_img, const float* bias, int32_t out_dim,
                                  int32_t relu, int32_t out_bf16, void* out, int64_t out_ld,
                                  void* workspace, size_t workspace_bytes, void* stream) {
  CMB_NVTX("cmb.next4.sage_dense_forward");
  CMB_ARG(x_dst && h && n_dev && w_img && out && workspace,
          "cmb_sage_dense_forward: null argument");
  CMB_ARG(n_rows_cap >= 1 && x_ld >= feat_dim && h_ld >= feat_dim && out_ld >= out_dim,
          "cmb_sage_dense_forward: bad n_rows_cap / leading dimension");
  const size_t need = cmb_sage_dense_workspace_bytes(n_rows_cap, feat_dim, out_dim);
  CMB_ARG(need != 0 && workspace_bytes >= need &&
              (reinterpret_cast<uintptr_t>(workspace) & 255) == 0,
          "cmb_sage_dense_forward: workspace must be 256-B aligned and >= %zu bytes", need);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int64_t fp = dn::padk(feat_dim);
  dn::DenseWs w = dn::carve(workspace, n_rows_cap, feat_dim, out_dim, nullptr);
  dn::k_pack_a<<<148 * 8, 256, 0, s>>>(x_dst, x_ld, h, h_ld, n_dev, n_rows_cap, feat_dim, fp, w.a);
  CMB_CUDA(cudaGetLastError());
  // column-major view: Z^T (Fo x cap) = W^T (Fo x 2Fp) * A^T (2Fp x cap); W row-major [2Fp][Fo]
  // is W^T column-major with ld Fo, A row-major [cap][2Fp] is A^T column-major with ld 2Fp
  cmb_status st = dn::lt_gemm(CUBLAS_OP_N, CUBLAS_OP_N, out_dim, n_rows_cap, 2 * fp, w_img,
                              out_dim, w.a, 2 * fp, w.z, w.lt, dn::kLtWorkspace, s);
  if (st != CMB_OK) return st;
  dn::k_epilogue<<<148 * 8, 256, 0, s>>>(w.z, bias, n_dev, n_rows_cap, out_dim, relu, out_bf16,
                                         out, out_ld);
  CMB_CUDA(cudaGetLastError());
  return CMB_OK;
}

cmb_status cmb_sage_dense_backward(const float* x_dst, int64_t x_ld, const float* h, int64_t h_ld,
                                   const int64_t* n_dev, int64_t n_rows_cap, int32_t feat_dim,
                                   const void* dy, int64_t dy_ld, int32_t dy_f32, const void* y,
                                   int64_t y_ld, int32_t out_dim, float* dw, float* db,
                                   void* workspace, size_t workspace_bytes, void* stream) {
  CMB_NVTX("cmb.next4.sage_dense_backward");
  CMB_ARG(x_dst && h && n_dev && dy && dw && db && workspace,
          "cmb_sage_dense_backward: null argument");
  CMB_ARG(n_rows_cap >= 1 && x_ld >= feat_dim && h_ld >= feat_dim && dy_ld >= out_dim &&
              (!y || y_ld >= out_dim),
          "cmb_sage_dense_backward: bad n_rows_cap / leading dimension");
  const size_t need = cmb_sage_dense_workspace_bytes(n_rows_cap, feat_dim, out_dim);
  CMB_ARG(need != 0 && workspace_bytes >= need &&
              (reinterpret_cast<uintptr_t>(workspace) & 255) == 0,
          "cmb_sage_dense_backward: workspace must be 256-B aligned and >= %zu bytes", need);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int64_t fp = dn::padk(feat_dim);
  dn::DenseWs w = dn::carve(workspace, n_rows_cap, feat_dim, out_dim, nullptr);
  dn::k_pack_a<<<148 * 8, 256, 0, s>>>(x_dst, x_ld, h, h_ld, n_dev, n_rows_cap, feat_dim, fp, w.a);
  CMB_CUDA(cudaGetLastError());
  dn::k_mask_dz<<<dn::kMaskBlocks, dn::kMaskThreads, 0, s>>>(
      dy, dy_ld, dy_f32, static_cast<const __nv_bfloat16*>(y), y_ld, n_dev, n_rows_cap, out_dim,
      w.dz, w.part);
  CMB_CUDA(cudaGetLastError());
  // column-major: dW^T (Fo x 2Fp) = dZ^T (Fo x cap) * A (cap x 2Fp); dZ row-major [cap][Fo] is
  // dZ^T column-major (ld Fo), A row-major [cap][2Fp] is A^T column-major (ld 2Fp), transposed
  cmb_status st = dn::lt_gemm(CUBLAS_OP_N, CUBLAS_OP_T, out_dim, 2 * fp, n_rows_cap, w.dz, out_dim,
                              w.a, 2 * fp, w.z, w.lt, dn::kLtWorkspace, s);
  if (st != CMB_OK) return st;
  dn::k_finish<<<148 * 4, 256, 0, s>>>(w.part, dn::kMaskBlocks, w.z, feat_dim, fp, out_dim, dw,
                                       db);
  CMB_CUDA(cudaGetLastError());
  return CMB_OK;
}

}  // extern "C"
