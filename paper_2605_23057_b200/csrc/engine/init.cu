// K16: deterministic random-init weights generated on the device, bit-identical
// to the CPU oracle (integer hash -> exact fp32 -> IEEE RN fp16), plus the
// RTN quantisers (W8 per-channel, W4 g128 uint4b8) and the successor lm_head.
#include "kernels.cuh"

namespace msw {

__global__ void fill_fp16_kernel(half* dst, int64_t total, uint64_t key, float sc) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total;
       i += int64_t(gridDim.x) * blockDim.x)
    dst[i] = __float2half_rn(unif(key, uint64_t(i)) * sc);
}

void launch_fill_fp16(half* dst, int64_t rows, int64_t cols, uint64_t seed, uint64_t tid,
                      int scale_log2, cudaStream_t st) {
  const int64_t total = rows * cols;
  const int grid = int(std::min<int64_t>((total + 255) / 256, int64_t(kNumSMs) * 32));
  fill_fp16_kernel<<<grid, 256, 0, st>>>(dst, total, tensor_key(seed, tid),
                                         ldexpf(1.0f, -scale_log2));
  MSW_LAUNCH_CHECK();
}

__global__ void fill_norm_kernel(half* dst, int64_t n, uint64_t key) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    dst[i] = __float2half_rn(__fadd_rn(1.0f, __fmul_rn(unif(key, uint64_t(i)), 0.125f)));
}

void launch_fill_norm(half* dst, int64_t n, uint64_t seed, uint64_t tid, cudaStream_t st) {
  fill_norm_kernel<<<ceil_div(n, 256), 256, 0, st>>>(dst, n, tensor_key(seed, tid));
  MSW_LAUNCH_CHECK();
}

// One CTA per row: absmax, s = amax/127 (IEEE div), q = clamp(rint(w/s)).
__global__ void quant_int8_kernel(const half* w, int k, int8_t* q, float* s) {
  __shared__ float red[32];
  const size_t row = blockIdx.x;
  const half* src = w + row * k;
  float amax = 0.0f;
  for (int i = threadIdx.x; i < k; i += blockDim.x) amax = fmaxf(amax, fabsf(__half2float(src[i])));
  amax = block_max(amax, red);
  const float sc = amax / 127.0f;
  if (threadIdx.x == 0) s[row] = sc;
  for (int i = threadIdx.x; i < k; i += blockDim.x) {
    float v = 0.0f;
    if (amax > 0.0f) v = rintf(__half2float(src[i]) / sc);
    v = fminf(fmaxf(v, -127.0f), 127.0f);
    q[row * k + i] = static_cast<int8_t>(v);
  }
}

void launch_quant_int8(const half* w, int n, int k, int8_t* q, float* s, cudaStream_t st) {
  quant_int8_kernel<<<n, 256, 0, st>>>(w, k, q, s);
  MSW_LAUNCH_CHECK();
}

// One warp per (row, 128-group). Lane l owns k = 4l..4l+3 of the group.
// Packed word j of a row holds k = 8j..8j+7 with nibble position
// p(i) = (i >> 1) + 4 * (i & 1), so lop3(word >> 4i, 0x000F000F, 0x64006400)
// yields the fp16 pair (1024 + q[2i], 1024 + q[2i+1]).
__global__ void quant_w4_kernel(const half* w, int n, int k, uint32_t* packed, half* s) {
  const int lane = threadIdx.x & 31;
  const int groups = k / kW4Group;
  const long long item = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (item >= (long long)n * groups) return;
  const int row = int(item / groups), g = int(item % groups);
  const half* src = w + (size_t)row * k + (size_t)g * kW4Group + 4 * lane;
  float v[4];
  float amax = 0.0f;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    v[i] = __half2float(src[i]);
    amax = fmaxf(amax, fabsf(v[i]));
  }
  amax = warp_max(amax);
  const half sh = __float2half_rn((2.0f * amax) / 15.0f);
  const float sf = __half2float(sh);
  uint32_t word = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    int q = 8;
    if (sf > 0.0f) q = min(15, max(0, int(rintf(v[i] / sf)) + 8));
    const int idx = (lane & 1) * 4 + i;  // position of this k inside its 8-word
    const int pos = (idx >> 1) + 4 * (idx & 1);
    word |= uint32_t(q) << (4 * pos);
  }
  word |= __shfl_xor_sync(0xffffffffu, word, 1);
  if ((lane & 1) == 0) packed[(size_t)row * (k / 8) + (size_t)g * 16 + (lane >> 1)] = word;
  if (lane == 0) s[(size_t)row * groups + g] = sh;
}

void launch_quant_w4(const half* w, int n, int k, uint32_t* packed, half* s, cudaStream_t st) {
  const long long items = (long long)n * (k / kW4Group);
  quant_w4_kernel<<<ceil_div(items, 8), 256, 0, st>>>(w, n, k, packed, s);
  MSW_LAUNCH_CHECK();
}

__global__ void quant_awq4_kernel(const half* w, int n, int k, uint32_t* packed, half* s,
                                  uint8_t* zeros) {
  const int lane = threadIdx.x & 31;
  const int groups = k / kW4Group;
  const long long item = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (item >= (long long)n * groups) return;
  const int row = int(item / groups), g = int(item % groups);
  const half* src = w + (size_t)row * k + (size_t)g * kW4Group + 4 * lane;
  float v[4];
  float mx = -INFINITY, mn = INFINITY;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    v[i] = __half2float(src[i]);
    mx = fmaxf(mx, v[i]);
    mn = fminf(mn, v[i]);
  }
  mx = warp_max(mx);
  mn = -warp_max(-mn);
  const half sh = __float2half_rn(fmaxf(mx - mn, 1e-5f) / 15.0f);
  const float sf = __half2float(sh);
  const int z = int(fminf(fmaxf(-rintf(mn / sf), 0.0f), 15.0f));
  uint32_t word = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int q = min(15, max(0, int(rintf(v[i] / sf)) + z));
    const int idx = (lane & 1) * 4 + i;
    const int pos = (idx >> 1) + 4 * (idx & 1);
    word |= uint32_t(q) << (4 * pos);
  }
  word |= __shfl_xor_sync(0xffffffffu, word, 1);
  if ((lane & 1) == 0) packed[(size_t)row * (k / 8) + (size_t)g * 16 + (lane >> 1)] = word;
  if (lane == 0) {
    s[(size_t)row * groups + g] = sh;
    zeros[(size_t)row * groups + g] = uint8_t(z);
  }
}

void launch_quant_awq4(const half* w, int n, int k, uint32_t* packed, half* s, uint8_t* z,
                       cudaStream_t st) {
  const long long items = (long long)n * (k / kW4Group);
  quant_awq4_kernel<<<ceil_div(items, 8), 256, 0, st>>>(w, n, k, packed, s, z);
  MSW_LAUNCH_CHECK();
}

__global__ void unpack_w4_kernel(const uint32_t* packed, long long total, uint8_t* out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const uint32_t word = packed[i / 8];
    const int idx = int(i % 8);
    const int pos = (idx >> 1) + 4 * (idx & 1);
    out[i] = uint8_t((word >> (4 * pos)) & 0xF);
  }
}

void launch_unpack_w4(const uint32_t* packed, int n, int k, uint8_t* nibbles, cudaStream_t st) {
  const long long total = (long long)n * k;
  unpack_w4_kernel<<<std::min<long long>(ceil_div(total, 256), 4096), 256, 0, st>>>(packed, total,
                                                                                  nibbles);
  MSW_LAUNCH_CHECK();
}

// Successor lm_head: target row u = E[pred(u)];
// draft row u = [agree(p1)] E[p1] + [!agree(p2)] E[p2], p1 = pred(u), p2 = pred(p1).
__global__ void lm_head_kernel(const half* emb, const int* pred, const uint8_t* agree,
                               int is_draft, int H, half* out) {
  const int u = blockIdx.x;
  const int p1 = pred[u];
  const int p2 = pred[p1];
  const bool a1 = !is_draft || agree[p1];
  const bool a2 = is_draft && !agree[p2];
  for (int j = threadIdx.x; j < H; j += blockDim.x) {
    float r = 0.0f;
    if (a1) r = __fadd_rn(r, __half2float(emb[(size_t)p1 * H + j]));
    if (a2) r = __fadd_rn(r, __half2float(emb[(size_t)p2 * H + j]));
    out[(size_t)u * H + j] = __float2half_rn(r);
  }
}

void launch_lm_head(const half* emb, const int* pred, const uint8_t* agree, int is_draft, int V,
                    int H, half* out, cudaStream_t st) {
  lm_head_kernel<<<V, 256, 0, st>>>(emb, pred, agree, is_draft, H, out);
  MSW_LAUNCH_CHECK();
}

__global__ void interleave_kernel(const uint8_t* a, const uint8_t* b, int n, size_t row_bytes,
                                  uint8_t* out) {
  const size_t total = size_t(2) * n * row_bytes;
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < total;
       i += size_t(gridDim.x) * blockDim.x) {
    const size_t orow = i / row_bytes, off = i % row_bytes;
    const uint8_t* src = (orow & 1) ? b : a;
    out[i] = src[(orow >> 1) * row_bytes + off];
  }
}

void launch_interleave_rows(const void* a, const void* b, int n, size_t row_bytes, void* out,
                            cudaStream_t st) {
  interleave_kernel<<<kNumSMs * 16, 256, 0, st>>>(static_cast<const uint8_t*>(a),
                                                  static_cast<const uint8_t*>(b), n, row_bytes,
                                                  static_cast<uint8_t*>(out));
  MSW_LAUNCH_CHECK();
}

}  // namespace msw
