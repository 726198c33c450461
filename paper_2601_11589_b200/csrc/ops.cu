#include <cstdio>

#include "ops.cuh"
#include "synth.h"

namespace lp {

namespace {

constexpr int kRowThreads = 256;

__device__ __forceinline__ float block_sum(float v, float* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x / 32, l = threadIdx.x % 32;
  if (l == 0) red[w] = v;
  __syncthreads();
  float s = 0.f;
  if (threadIdx.x < 32) {
    s = threadIdx.x < blockDim.x / 32 ? red[threadIdx.x] : 0.f;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (threadIdx.x == 0) red[32] = s;
  }
  __syncthreads();
  const float r = red[32];
  __syncthreads();
  return r;
}

__global__ void init_weights_kernel(bf16* dst, size_t n, uint64_t seed, uint64_t tid, float scale,
                                    int inter_rows, int cols) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    uint64_t t = tid, idx = i;
    if (inter_rows > 0) {
      const size_t r = i / cols, c = i % cols;
      t = tid + (r & 1);
      idx = (r >> 1) * cols + c;
    }
    dst[i] = __float2bfloat16_rn(synth_weight_f32(seed, t, idx, scale));
  }
}

__global__ void fill_kernel(bf16* dst, size_t n, float v) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x)
    dst[i] = __float2bfloat16_rn(v);
}

// One CTA per token row. h is a multiple of 4.
__global__ void __launch_bounds__(kRowThreads)
    embed_rmsnorm_kernel(RowCtx c, const int* __restrict__ tokens, const bf16* __restrict__ embed,
                         const bf16* __restrict__ gamma, float* __restrict__ x_resid,
                         bf16* __restrict__ x_norm) {
  __shared__ float red[33];
  const int t = blockIdx.x;
  if (t >= *c.n_live) return;
  const bf16* e = embed + static_cast<size_t>(tokens[t]) * c.h;
  float* xr = x_resid + static_cast<size_t>(t) * c.h;
  float ss = 0.f;
  for (int i = threadIdx.x; i < c.h; i += blockDim.x) {
    const float v = __bfloat162float(e[i]);
    xr[i] = v;
    ss += v * v;
  }
  const float tot = block_sum(ss, red);
  const float inv = rsqrtf(tot / c.h + c.eps);
  bf16* xn = x_norm + static_cast<size_t>(t) * c.h;
  for (int i = threadIdx.x; i < c.h; i += blockDim.x)
    xn[i] = __float2bfloat16_rn(xr[i] * inv * __bfloat162float(gamma[i]));
}

__global__ void __launch_bounds__(kRowThreads)
    resid_rmsnorm_kernel(RowCtx c, const float* __restrict__ ws, int splits, size_t ws_stride_rows,
                         float* __restrict__ x_resid, const bf16* __restrict__ gamma,
                         bf16* __restrict__ x_norm) {
  __shared__ float red[33];
  const int t = blockIdx.x;
  if (t >= *c.n_live) return;
  float4* xr = reinterpret_cast<float4*>(x_resid + static_cast<size_t>(t) * c.h);
  const int h4 = c.h / 4;
  float ss = 0.f;
  for (int i = threadIdx.x; i < h4; i += blockDim.x) {
    float4 v = xr[i];
    for (int s = 0; s < splits; ++s) {
      const float4 p = reinterpret_cast<const float4*>(
          ws + (static_cast<size_t>(s) * ws_stride_rows + t) * c.h)[i];
      v.x += p.x; v.y += p.y; v.z += p.z; v.w += p.w;
    }
    xr[i] = v;
    ss += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
  }
  const float tot = block_sum(ss, red);
  const float inv = rsqrtf(tot / c.h + c.eps);
  __nv_bfloat162* xn = reinterpret_cast<__nv_bfloat162*>(x_norm + static_cast<size_t>(t) * c.h);
  const __nv_bfloat162* g2 = reinterpret_cast<const __nv_bfloat162*>(gamma);
  for (int i = threadIdx.x; i < h4; i += blockDim.x) {
    const float4 v = xr[i];
    const float2 ga = __bfloat1622float2(g2[2 * i]);
    const float2 gb = __bfloat1622float2(g2[2 * i + 1]);
    xn[2 * i] = __floats2bfloat162_rn(v.x * inv * ga.x, v.y * inv * ga.y);
    xn[2 * i + 1] = __floats2bfloat162_rn(v.z * inv * gb.x, v.w * inv * gb.y);
  }
}

// One CTA per token; thread j handles rotary pair (j, j + d/2) of one head.
__global__ void qkv_post_kernel(QkvCtx c) {
  const int t = blockIdx.x;
  if (t >= *c.n_live) return;
  const int half = c.d / 2;
  const int qkv_out = (c.nq + 2 * c.nkv) * c.d;
  const int pos = c.positions[t];
  const int slot = c.slot_mapping[t];
  const int page = slot / c.page_size, s_in = slot % c.page_size;
  const size_t page_elems = static_cast<size_t>(2) * c.nkv * c.page_size * c.d;
  const int n_rot_heads = c.nq + c.nkv;  // q and k heads get RoPE
  const int total = (c.nq + 2 * c.nkv) * half;
  for (int j = threadIdx.x; j < total; j += blockDim.x) {
    const int head = j / half, i = j % half;
    const int c0 = head * c.d + i, c1 = c0 + half;
    float x0 = __bfloat162float(c.bias[c0]), x1 = __bfloat162float(c.bias[c1]);
    for (int s = 0; s < c.splits; ++s) {
      const float* row = c.ws + (static_cast<size_t>(s) * c.ws_stride_rows + t) * qkv_out;
      x0 += row[c0];
      x1 += row[c1];
    }
    if (head < n_rot_heads) {
      float sn, cs;
      sincosf(static_cast<float>(pos) * c.inv_freq[i], &sn, &cs);
      const float r0 = x0 * cs - x1 * sn;
      const float r1 = x1 * cs + x0 * sn;
      x0 = r0;
      x1 = r1;
    }
    const bf16 b0 = __float2bfloat16_rn(x0), b1 = __float2bfloat16_rn(x1);
    if (head < c.nq) {
      bf16* q = c.q_out + static_cast<size_t>(t) * c.nq * c.d + head * c.d;
      q[i] = b0;
      q[i + half] = b1;
    } else {
      const bool is_v = head >= c.nq + c.nkv;
      const int g = is_v ? head - c.nq - c.nkv : head - c.nq;
      bf16* dst = c.kv_layer + page * page_elems +
                  ((static_cast<size_t>(is_v ? 1 : 0) * c.nkv + g) * c.page_size + s_in) * c.d;
      dst[i] = b0;
      dst[i + half] = b1;
    }
  }
}

__global__ void gather_rows_kernel(const int* n_rows, const int* idx, const bf16* src, bf16* dst,
                                   int h) {
  const int r = blockIdx.x;
  if (r >= *n_rows) return;
  const uint4* s = reinterpret_cast<const uint4*>(src + static_cast<size_t>(idx[r]) * h);
  uint4* d = reinterpret_cast<uint4*>(dst + static_cast<size_t>(r) * h);
  for (int i = threadIdx.x; i < h / 8; i += blockDim.x) d[i] = s[i];
}

__global__ void argmax_kernel(const int* n_rows, const float* logits, int vocab, int* out) {
  const int r = blockIdx.x;
  if (r >= *n_rows) return;
  const float* row = logits + static_cast<size_t>(r) * vocab;
  float best = -INFINITY;
  int bi = 0x7fffffff;
  for (int j = threadIdx.x; j < vocab; j += blockDim.x) {
    const float v = row[j];
    if (v > best || (v == best && j < bi)) { best = v; bi = j; }
  }
  __shared__ float sv[32];
  __shared__ int si[32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float ov = __shfl_xor_sync(0xffffffffu, best, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
  }
  const int w = threadIdx.x / 32;
  if (threadIdx.x % 32 == 0) { sv[w] = best; si[w] = bi; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 1; k < blockDim.x / 32; ++k)
      if (sv[k] > best || (sv[k] == best && si[k] < bi)) { best = sv[k]; bi = si[k]; }
    out[r] = bi;
  }
}

}  // namespace

void init_weights(bf16* dst, size_t n, uint64_t seed, uint64_t tensor_id, float scale,
                  int interleave_rows, int cols, cudaStream_t st) {
  init_weights_kernel<<<4096, 256, 0, st>>>(dst, n, seed, tensor_id, scale, interleave_rows, cols);
}

void fill_bf16(bf16* dst, size_t n, float v, cudaStream_t st) {
  fill_kernel<<<1024, 256, 0, st>>>(dst, n, v);
}

void embed_rmsnorm(const RowCtx& c, const int* tokens, const bf16* embed, const bf16* gamma,
                   float* x_resid, bf16* x_norm, cudaStream_t st) {
  embed_rmsnorm_kernel<<<c.t_cap, kRowThreads, 0, st>>>(c, tokens, embed, gamma, x_resid, x_norm);
}

void resid_rmsnorm(const RowCtx& c, const float* ws, int splits, size_t ws_stride_rows,
                   float* x_resid, const bf16* gamma, bf16* x_norm, cudaStream_t st) {
  resid_rmsnorm_kernel<<<c.t_cap, kRowThreads, 0, st>>>(c, ws, splits, ws_stride_rows, x_resid,
                                                        gamma, x_norm);
}

void qkv_post(const QkvCtx& c, cudaStream_t st) {
  qkv_post_kernel<<<c.t_cap, 256, 0, st>>>(c);
}

void gather_rows(const int* n_rows, int r_cap, const int* idx, const bf16* src, bf16* dst, int h,
                 cudaStream_t st) {
  gather_rows_kernel<<<r_cap, 128, 0, st>>>(n_rows, idx, src, dst, h);
}

void argmax_rows(const int* n_rows, int r_cap, const float* logits, int vocab, int* out,
                 cudaStream_t st) {
  argmax_kernel<<<r_cap, 1024, 0, st>>>(n_rows, logits, vocab, out);
}

}  // namespace lp
