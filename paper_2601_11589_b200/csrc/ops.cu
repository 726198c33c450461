#include <algorithm>
#include <cstdio>
#include <stdexcept>

#include "gemm_sm100.cuh"
#include "launch.cuh"
#include "ops.cuh"
#include "synth.h"

namespace lp {

namespace {

constexpr int kRowThreads = 256;
constexpr int kMaxVec = 8;  // float4 per thread: hidden <= 256*4*8 = 8192

__device__ __forceinline__ float block_sum(float v, float* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x / 32, l = threadIdx.x % 32;
  if (l == 0) red[w] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    float s = threadIdx.x < blockDim.x / 32 ? red[threadIdx.x] : 0.f;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (threadIdx.x == 0) red[32] = s;
  }
  __syncthreads();
  return red[32];
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

// One CTA per token row.
__global__ void __launch_bounds__(kRowThreads)
    embed_rmsnorm_kernel(RowCtx c, const int* __restrict__ tokens, const bf16* __restrict__ embed,
                         const bf16* __restrict__ gamma, float* __restrict__ x_resid,
                         bf16* __restrict__ x_norm) {
  KTL_SCOPE(kKtlEmbed, 0);
  __shared__ float red[33];
  pdl_trigger();
  const int t = blockIdx.x;
  const bool live = t < *c.n_live;
  pdl_wait();
  if (!live) return;
  const bf16* e = embed + static_cast<size_t>(tokens[t]) * c.h;
  float* xr = x_resid + static_cast<size_t>(t) * c.h;
  float ss = 0.f;
  for (int i = threadIdx.x; i < c.h; i += blockDim.x) {
    const float v = __bfloat162float(e[i]);
    xr[i] = v;
    ss += v * v;
  }
  const float inv = rsqrtf(block_sum(ss, red) / c.h + c.eps);
  bf16* xn = x_norm + static_cast<size_t>(t) * c.h;
  for (int i = threadIdx.x; i < c.h; i += blockDim.x)
    xn[i] = __float2bfloat16_rn(xr[i] * inv * __bfloat162float(gamma[i]));
}

// x_resid += sum of split partials; x_norm = bf16(rmsnorm(x_resid) * gamma).
// All of a thread's loads (residual + every split) are issued before use.
__global__ void __launch_bounds__(kRowThreads)
    resid_rmsnorm_kernel(RowCtx c, const float* __restrict__ ws, int splits, const int* splits_dev,
                         const int* __restrict__ sk_tab, size_t ws_stride_rows, float* __restrict__ x_resid,
                         const bf16* __restrict__ gamma, bf16* __restrict__ x_norm) {
  KTL_SCOPE(kKtlResidNorm, 0);
  __shared__ float red[33];
  pdl_trigger();
  const int t = blockIdx.x;
  const bool live = t < *c.n_live;
  if (splits_dev) splits = *splits_dev;  // pre-graph H2D metadata (< 0: stream-K)
  pdl_wait();
  if (!live) return;
  const int h4 = c.h / 4;
  float4* xr = reinterpret_cast<float4*>(x_resid + static_cast<size_t>(t) * c.h);
  float4 acc[kMaxVec];
#pragma unroll
  for (int k = 0; k < kMaxVec; ++k) {
    const int i = threadIdx.x + k * kRowThreads;
    acc[k] = i < h4 ? xr[i] : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  if (splits >= 0 || !sk_tab) {  // split-K: every element sums `splits` slices
    for (int s = 0; s < splits; ++s) {
      const float4* p = reinterpret_cast<const float4*>(ws + (static_cast<size_t>(s) * ws_stride_rows + t) * c.h);
#pragma unroll
      for (int k = 0; k < kMaxVec; ++k) {
        const int i = threadIdx.x + k * kRowThreads;
        if (i < h4) {
          const float4 q = p[i];
          acc[k].x += q.x; acc[k].y += q.y; acc[k].z += q.z; acc[k].w += q.w;
        }
      }
    }
  } else {  // stream-K: the segments of each element's output tile (table written by the GEMM)
    const int* seg = sk_tab + kSkTabHeader + t / sk_tab[0];
    const int tiles = sk_tab[1], rows = sk_tab[2];
    int nseg[kMaxVec];
    int smax = 1;
#pragma unroll
    for (int k = 0; k < kMaxVec; ++k) {
      const int i = threadIdx.x + k * kRowThreads;
      nseg[k] = i < h4 ? seg[(4 * i / rows) * tiles] : 0;
      smax = max(smax, nseg[k]);
    }
    for (int s = 0; s < smax; ++s) {
      const float4* p = reinterpret_cast<const float4*>(ws + (static_cast<size_t>(s) * ws_stride_rows + t) * c.h);
#pragma unroll
      for (int k = 0; k < kMaxVec; ++k) {
        const int i = threadIdx.x + k * kRowThreads;
        if (i < h4 && s < nseg[k]) {
          const float4 q = p[i];
          acc[k].x += q.x; acc[k].y += q.y; acc[k].z += q.z; acc[k].w += q.w;
        }
      }
    }
  }
  float ss = 0.f;
#pragma unroll
  for (int k = 0; k < kMaxVec; ++k) {
    const int i = threadIdx.x + k * kRowThreads;
    if (i < h4) {
      xr[i] = acc[k];
      ss += acc[k].x * acc[k].x + acc[k].y * acc[k].y + acc[k].z * acc[k].z + acc[k].w * acc[k].w;
    }
  }
  const float inv = rsqrtf(block_sum(ss, red) / c.h + c.eps);
  __nv_bfloat162* xn = reinterpret_cast<__nv_bfloat162*>(x_norm + static_cast<size_t>(t) * c.h);
  const __nv_bfloat162* g2 = reinterpret_cast<const __nv_bfloat162*>(gamma);
#pragma unroll
  for (int k = 0; k < kMaxVec; ++k) {
    const int i = threadIdx.x + k * kRowThreads;
    if (i < h4) {
      const float2 ga = __bfloat1622float2(g2[2 * i]);
      const float2 gb = __bfloat1622float2(g2[2 * i + 1]);
      xn[2 * i] = __floats2bfloat162_rn(acc[k].x * inv * ga.x, acc[k].y * inv * ga.y);
      xn[2 * i + 1] = __floats2bfloat162_rn(acc[k].z * inv * gb.x, acc[k].w * inv * gb.y);
    }
  }
}

// One CTA per token. A "unit" is 4 consecutive rotary pairs of one head:
// columns j..j+3 and j+d/2..j+d/2+3 (two float4 per split). Thread u owns
// units u, u + blockDim, ... (<= U), so a warp reads 2 x 256 B contiguous
// runs per load instruction. The d/2 rotary angles of the token are computed
// once into shared memory (q and k heads share them). Loads of U units x SU
// splits are issued before any add: U=4, SU=1 for large token counts (split-K
// <= 2, many CTAs per SM), U=1, SU=8 for short batches (deep split-K, few
// CTAs: all partials of a unit in flight at once).
constexpr int kQkvMaxHalf = 128;  // head_dim <= 256
__device__ __forceinline__ void add4(float4& a, const float4 b) {
  a.x += b.x; a.y += b.y; a.z += b.z; a.w += b.w;
}
__device__ __forceinline__ float4 bf4(const bf16* p) {
  const uint2 r = *reinterpret_cast<const uint2*>(p);
  const float2 lo = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&r.x));
  const float2 hi = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&r.y));
  return make_float4(lo.x, lo.y, hi.x, hi.y);
}
__device__ __forceinline__ void st_bf4(bf16* p, float a, float b, float c, float d) {
  const __nv_bfloat162 lo = __floats2bfloat162_rn(a, b), hi = __floats2bfloat162_rn(c, d);
  uint2 r;
  r.x = *reinterpret_cast<const uint32_t*>(&lo);
  r.y = *reinterpret_cast<const uint32_t*>(&hi);
  *reinterpret_cast<uint2*>(p) = r;
}
template <int U, int SU>
__global__ void qkv_post_kernel(QkvCtx c) {
  KTL_SCOPE(kKtlQkvPost, 0);
  __shared__ float s_cos[kQkvMaxHalf], s_sin[kQkvMaxHalf];
  pdl_trigger();
  const int t = blockIdx.x;
  if (t >= *c.n_live) {
    pdl_wait();
    return;
  }
  const int half = c.d / 2, upr = half / 4;  // units per head
  const int heads = c.nq + 2 * c.nkv;
  const int units = heads * upr;
  const int qkv_out = heads * c.d;
  // bias and rotary table: host-written metadata / static weights, safe before the wait
  float4 x0[U], x1[U];
#pragma unroll
  for (int k = 0; k < U; ++k) {
    const int u = threadIdx.x + k * blockDim.x;
    if (u < units) {
      const int c0 = (u / upr) * c.d + (u % upr) * 4;
      x0[k] = bf4(c.bias + c0);
      x1[k] = bf4(c.bias + c0 + half);
    }
  }
  if (threadIdx.x < half) {
    float sn, cs;
    sincosf(static_cast<float>(c.positions[t]) * c.inv_freq[threadIdx.x], &sn, &cs);
    s_cos[threadIdx.x] = cs;
    s_sin[threadIdx.x] = sn;
  }
  pdl_wait();
  const int raw = c.splits_dev ? *c.splits_dev : c.splits;
  // Sum `bound` slices; unit k takes the first nseg_of(k) of them.
  auto reduce = [&](int bound, auto nseg_of) {
    for (int s0 = 0; s0 < bound; s0 += SU) {
      float4 p0[SU][U], p1[SU][U];
#pragma unroll
      for (int e = 0; e < SU; ++e) {
        const float* row = c.ws + (static_cast<size_t>(s0 + e) * c.ws_stride_rows + t) * qkv_out;
#pragma unroll
        for (int k = 0; k < U; ++k) {
          const int u = threadIdx.x + k * blockDim.x;
          if (u < units && s0 + e < nseg_of(k)) {
            const int c0 = (u / upr) * c.d + (u % upr) * 4;
            p0[e][k] = *reinterpret_cast<const float4*>(row + c0);
            p1[e][k] = *reinterpret_cast<const float4*>(row + c0 + half);
          }
        }
      }
#pragma unroll
      for (int e = 0; e < SU; ++e) {
#pragma unroll
        for (int k = 0; k < U; ++k) {
          if (threadIdx.x + k * blockDim.x < units && s0 + e < nseg_of(k)) {
            add4(x0[k], p0[e][k]);
            add4(x1[k], p1[e][k]);
          }
        }
      }
    }
  };
  if (raw >= 0 || !c.sk_tab) {  // split-K: every unit sums the same slices
    const int splits = max(1, raw);
    reduce(splits, [&](int) { return splits; });
  } else {  // stream-K: the segments of each unit's output tile (table written by the GEMM)
    const int* seg = c.sk_tab + kSkTabHeader + t / c.sk_tab[0];
    const int tiles = c.sk_tab[1], rows = c.sk_tab[2];
    int nseg[U];
    int bound = 1;
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const int u = threadIdx.x + k * blockDim.x;
      nseg[k] = u < units ? seg[((u / upr) * c.d / rows) * tiles] : 0;
      bound = max(bound, nseg[k]);
    }
    reduce(bound, [&](int k) { return nseg[k]; });
  }
  __syncthreads();
  const int slot = c.slot_mapping[t];
  const int page = slot / c.page_size, s_in = slot % c.page_size;
  const size_t page_elems = static_cast<size_t>(2) * c.nkv * c.page_size * c.d;
#pragma unroll
  for (int k = 0; k < U; ++k) {
    const int u = threadIdx.x + k * blockDim.x;
    if (u >= units) continue;
    const int head = u / upr, j = (u % upr) * 4;
    float a[4] = {x0[k].x, x0[k].y, x0[k].z, x0[k].w};
    float b[4] = {x1[k].x, x1[k].y, x1[k].z, x1[k].w};
    if (head < c.nq + c.nkv) {  // RoPE on q and k heads (rotate-half pairing)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float cs = s_cos[j + e], sn = s_sin[j + e];
        const float r0 = a[e] * cs - b[e] * sn;
        const float r1 = b[e] * cs + a[e] * sn;
        a[e] = r0;
        b[e] = r1;
      }
    }
    bf16* dst;
    if (head < c.nq) {
      dst = c.q_out + static_cast<size_t>(t) * c.nq * c.d + head * c.d;
    } else {
      const bool is_v = head >= c.nq + c.nkv;
      const int g = is_v ? head - c.nq - c.nkv : head - c.nq;
      dst = c.kv_layer + page * page_elems +
            ((static_cast<size_t>(is_v ? 1 : 0) * c.nkv + g) * c.page_size + s_in) * c.d;
    }
    st_bf4(dst + j, a[0], a[1], a[2], a[3]);
    st_bf4(dst + j + half, b[0], b[1], b[2], b[3]);
  }
}

// Copies the last-token rows for the LM head and resets the argmax keys.
__global__ void gather_rows_kernel(const int* n_rows, const int* idx, const bf16* src, bf16* dst, int h,
                                   unsigned long long* keys) {
  KTL_SCOPE(kKtlGather, 0);
  pdl_trigger();
  const int r = blockIdx.x;
  const bool live = r < *n_rows;
  pdl_wait();
  if (!live) return;
  if (threadIdx.x == 0) keys[r] = 0ull;
  const uint4* s = reinterpret_cast<const uint4*>(src + static_cast<size_t>(idx[r]) * h);
  uint4* d = reinterpret_cast<uint4*>(dst + static_cast<size_t>(r) * h);
  for (int i = threadIdx.x; i < h / 8; i += blockDim.x) d[i] = s[i];
}

// Order-preserving key: larger value wins, ties -> lower index.
__device__ __forceinline__ unsigned long long argmax_key(float v, int j) {
  uint32_t u = __float_as_uint(v);
  u = (u & 0x80000000u) ? ~u : (u | 0x80000000u);
  return (static_cast<unsigned long long>(u) << 32) | static_cast<uint32_t>(0x7fffffff - j);
}

constexpr int kArgmaxChunks = 32;
__global__ void __launch_bounds__(256)
    argmax_kernel(const int* n_rows, const float* logits, int vocab, unsigned long long* keys) {
  KTL_SCOPE(kKtlArgmax, 0);
  pdl_trigger();
  const int r = blockIdx.x;
  const bool live = r < *n_rows;
  pdl_wait();
  if (!live) return;
  const float* row = logits + static_cast<size_t>(r) * vocab;
  const int per = ((vocab + kArgmaxChunks - 1) / kArgmaxChunks + 3) & ~3;
  const int b = blockIdx.y * per, e = min(vocab, b + per);
  unsigned long long best = 0;
  for (int j = b + 4 * threadIdx.x; j < e; j += 4 * blockDim.x) {
    if (j + 3 < e) {
      const float4 v = *reinterpret_cast<const float4*>(row + j);
      best = max(best, argmax_key(v.x, j));
      best = max(best, argmax_key(v.y, j + 1));
      best = max(best, argmax_key(v.z, j + 2));
      best = max(best, argmax_key(v.w, j + 3));
    } else {
      for (int k = j; k < e; ++k) best = max(best, argmax_key(row[k], k));
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) best = max(best, __shfl_xor_sync(0xffffffffu, best, o));
  __shared__ unsigned long long sm[8];
  if (threadIdx.x % 32 == 0) sm[threadIdx.x / 32] = best;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 1; k < blockDim.x / 32; ++k) best = max(best, sm[k]);
    atomicMax(keys + r, best);
  }
}

}  // namespace

void init_weights(bf16* dst, size_t n, uint64_t seed, uint64_t tensor_id, float scale,
                  int interleave_rows, int cols, cudaStream_t st) {
  init_weights_kernel<<<4096, 256, 0, st>>>(dst, n, seed, tensor_id, scale, interleave_rows, cols);
}

__global__ void kv_page_copy_kernel(const uint4* __restrict__ src_pool, size_t src_layer_stride,
                                    uint4* __restrict__ dst_pool, size_t dst_layer_stride, size_t page_vec,
                                    const int* __restrict__ src_pages, const int* __restrict__ dst_pages) {
  const int k = blockIdx.x, l = blockIdx.y;
  const uint4* s = src_pool + l * src_layer_stride + static_cast<size_t>(src_pages[k]) * page_vec;
  uint4* d = dst_pool + l * dst_layer_stride + static_cast<size_t>(dst_pages[k]) * page_vec;
  // All of a thread's loads in flight before its stores; streaming hints:
  // the pages are not re-read by this kernel.
  constexpr int kU = 4;
  for (size_t base = threadIdx.x; base < page_vec; base += size_t(blockDim.x) * kU) {
    uint4 r[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const size_t i = base + size_t(u) * blockDim.x;
      if (i < page_vec) r[u] = __ldcs(s + i);
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const size_t i = base + size_t(u) * blockDim.x;
      if (i < page_vec) __stcs(d + i, r[u]);
    }
  }
}

void kv_page_copy(const bf16* src_pool, size_t src_layer_stride, bf16* dst_pool, size_t dst_layer_stride,
                  size_t page_elems, const int* src_pages, const int* dst_pages, int n_pages, int layers,
                  cudaStream_t st) {
  if (n_pages <= 0) return;
  if (page_elems % 8 != 0 || src_layer_stride % 8 != 0 || dst_layer_stride % 8 != 0)
    throw std::runtime_error("kv_page_copy: pages must be 16-byte multiples");
  kv_page_copy_kernel<<<dim3(n_pages, layers), 512, 0, st>>>(
      reinterpret_cast<const uint4*>(src_pool), src_layer_stride / 8, reinterpret_cast<uint4*>(dst_pool),
      dst_layer_stride / 8, page_elems / 8, src_pages, dst_pages);
}

void fill_bf16(bf16* dst, size_t n, float v, cudaStream_t st) {
  fill_kernel<<<1024, 256, 0, st>>>(dst, n, v);
}

void embed_rmsnorm(const RowCtx& c, const int* tokens, const bf16* embed, const bf16* gamma,
                   float* x_resid, bf16* x_norm, cudaStream_t st) {
  launch_k(embed_rmsnorm_kernel, dim3(c.t_cap), dim3(kRowThreads), 0, st, c, tokens, embed, gamma,
           x_resid, x_norm);
}

__global__ void pdl_empty_kernel() {
  pdl_trigger();
  pdl_wait();
}

void launch_empty(dim3 grid, dim3 block, cudaStream_t st) { launch_k(pdl_empty_kernel, grid, block, 0, st); }

void resid_rmsnorm(const RowCtx& c, const float* ws, int splits, const int* splits_dev, const int* sk_tab,
                   size_t ws_stride_rows, float* x_resid, const bf16* gamma, bf16* x_norm, cudaStream_t st) {
  if (debug_empty("norm")) return launch_empty(dim3(c.t_cap), dim3(kRowThreads), st);
  launch_k(resid_rmsnorm_kernel, dim3(c.t_cap), dim3(kRowThreads), 0, st, c, ws, splits, splits_dev, sk_tab,
           ws_stride_rows, x_resid, gamma, x_norm);
}

void qkv_post(const QkvCtx& c, cudaStream_t st) {
  const int half = c.d / 2;
  if (half % 4 != 0 || half > kQkvMaxHalf)
    throw std::runtime_error("qkv_post: head_dim must be a multiple of 8 and <= 256");
  const int units = (c.nq + 2 * c.nkv) * (half / 4);
  // Deep split-K: all partials of a unit in flight (U=1, SU=8), or U=2, SU=4
  // when one unit per thread would exceed the register file (e.g. 56 heads).
  auto threads_for = [&](int per) { return std::max(((units + per - 1) / per + 31) / 32 * 32, half); };
  auto max_threads = [](const void* k) {
    cudaFuncAttributes a{};
    return cudaFuncGetAttributes(&a, k) == cudaSuccess ? a.maxThreadsPerBlock : 0;
  };
  static const int cap18 = max_threads(reinterpret_cast<const void*>(qkv_post_kernel<1, 8>));
  static const int cap24 = max_threads(reinterpret_cast<const void*>(qkv_post_kernel<2, 4>));
  static const int cap41 = max_threads(reinterpret_cast<const void*>(qkv_post_kernel<4, 1>));
  auto fits = [&](const void* k, int threads) {
    const int cap = k == reinterpret_cast<const void*>(qkv_post_kernel<1, 8>)   ? cap18
                    : k == reinterpret_cast<const void*>(qkv_post_kernel<2, 4>) ? cap24
                                                                                 : cap41;
    return threads <= cap;
  };
  // Deep split-K only happens below 256 live tokens (the tile planner charges
  // every extra split its fp32 partial round trip above that), so larger
  // capacities take the many-CTAs-per-SM <4, 1> variant.
  const bool deep = c.s_cap > 2 && c.t_cap < 256;
  if (debug_empty("qkv")) return launch_empty(dim3(c.t_cap), dim3(threads_for(deep ? 1 : 4)), st);
  if (deep && fits(reinterpret_cast<const void*>(qkv_post_kernel<1, 8>), threads_for(1))) {
    launch_k(qkv_post_kernel<1, 8>, dim3(c.t_cap), dim3(threads_for(1)), 0, st, c);
  } else if (deep && fits(reinterpret_cast<const void*>(qkv_post_kernel<2, 4>), threads_for(2))) {
    launch_k(qkv_post_kernel<2, 4>, dim3(c.t_cap), dim3(threads_for(2)), 0, st, c);
  } else if (fits(reinterpret_cast<const void*>(qkv_post_kernel<4, 1>), threads_for(4))) {
    launch_k(qkv_post_kernel<4, 1>, dim3(c.t_cap), dim3(threads_for(4)), 0, st, c);
  } else {
    throw std::runtime_error("qkv_post: too many heads for one CTA per token");
  }
}

void gather_rows(const int* n_rows, int r_cap, const int* idx, const bf16* src, bf16* dst, int h,
                 unsigned long long* argmax_keys, cudaStream_t st) {
  launch_k(gather_rows_kernel, dim3(r_cap), dim3(128), 0, st, n_rows, idx, src, dst, h, argmax_keys);
}

void argmax_rows(const int* n_rows, int r_cap, const float* logits, int vocab, unsigned long long* keys,
                 cudaStream_t st) {
  launch_k(argmax_kernel, dim3(r_cap, kArgmaxChunks), dim3(256), 0, st, n_rows, logits, vocab, keys);
}

}  // namespace lp

KTL_EXPORT(ops)
