// The per-GPU mode executor behind include/msw_engine.h.
//
// All routable modes are resident at once (FP16, W8A8, W4 g128 weights of the
// target plus the FP16 draft), so a mode switch at a request boundary is a
// pointer switch. KV lives in a paged pool (16-token blocks) shared by all
// modes; prefix caching maps content-hashed full prompt blocks (keyed by
// weight format) onto already-computed physical blocks with refcounts and an
// LRU of idle cached blocks. Batch-1 decode replays one CUDA graph per
// (model, format) with the step state (token, position, slot, history) kept
// on the device, so a request's decode loop never synchronises with the host.
#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <list>
#include <map>
#include <memory>
#include <unordered_map>
#include <vector>

#include "kernels.cuh"
#include "msw_engine.h"

namespace msw {
namespace {

thread_local std::string g_last_error;

constexpr int kPrefillChunk = 2048;
constexpr int kChunkedPrefillTokens = 512;  // ChunkedPrefill screening mode
constexpr int kMaxLogitRows = 64;

int fmt_of_mode(int mode) {
  switch (mode) {
    case MSW_MODE_FP16:
    case MSW_MODE_SPECULATIVE:
    case MSW_MODE_CHUNKED_PREFILL:
    case MSW_MODE_CUDA_GRAPHS:
    case MSW_MODE_KV_COMPRESSION:
      return kFP16;
    case MSW_MODE_INT8:
    case MSW_MODE_INT8_CONT_BATCHING:
      return kINT8;
    case MSW_MODE_GPTQ4:
    case MSW_MODE_GPTQ_PREFIX_CACHING:
      return kW4;
    case MSW_MODE_AWQ4:
      return kSlotAWQ4;
    default:
      throw ConfigErr("unsupported mode id " + std::to_string(mode));
  }
}

int ceil_log2(long long x) {
  int l = 0;
  while ((1ll << l) < x) ++l;
  return l;
}
int floor_log2(long long x) {
  int l = 0;
  while ((2ll << l) <= x) ++l;
  return l;
}
int in_shift(long long k) { return (ceil_log2(k) + 1) / 2; }
int res_shift(int layers) { return floor_log2(layers) / 2; }

template <typename T>
T* dalloc(size_t count) {
  void* p = nullptr;
  MSW_CUDA(cudaMalloc(&p, std::max<size_t>(count, 1) * sizeof(T)));
  return static_cast<T*>(p);
}

// ---------------------------------------------------------------- block pool
class BlockPool {
 public:
  void init(int n) {
    n_ = n;
    ref_.assign(n, 0);
    key_.assign(n, 0);
    lru_pos_.assign(n, lru_.end());
    free_.clear();
    for (int b = n - 1; b >= 0; --b) free_.push_back(b);
  }
  int alloc() {
    int b;
    if (!free_.empty()) {
      b = free_.back();
      free_.pop_back();
    } else if (!lru_.empty()) {  // evict the least recently used idle cached block
      b = lru_.front();
      lru_.pop_front();
      lru_pos_[b] = lru_.end();
      cached_.erase(key_[b]);
      key_[b] = 0;
    } else {
      throw DataErr("KV pool exhausted");
    }
    ref_[b] = 1;
    return b;
  }
  int lookup(uint64_t key) {
    auto it = cached_.find(key);
    if (it == cached_.end()) return -1;
    const int b = it->second;
    if (ref_[b]++ == 0 && lru_pos_[b] != lru_.end()) {
      lru_.erase(lru_pos_[b]);
      lru_pos_[b] = lru_.end();
    }
    return b;
  }
  void publish(int b, uint64_t key) {
    if (key == 0 || cached_.count(key)) return;
    cached_[key] = b;
    key_[b] = key;
  }
  void release(int b) {
    if (--ref_[b] > 0) return;
    if (key_[b] != 0) {
      lru_.push_back(b);
      lru_pos_[b] = std::prev(lru_.end());
    } else {
      free_.push_back(b);
    }
  }
  void drop_cache() {
    for (int b : lru_) {
      lru_pos_[b] = lru_.end();
      cached_.erase(key_[b]);
      key_[b] = 0;
      free_.push_back(b);
    }
    lru_.clear();
    for (auto& kv : cached_) key_[kv.second] = 0;  // live blocks stay allocated, uncached
    cached_.clear();
  }
  int available() const { return int(free_.size() + lru_.size()); }

 private:
  int n_ = 0;
  std::vector<int> ref_;
  std::vector<uint64_t> key_;
  std::vector<int> free_;
  std::list<int> lru_;
  std::vector<std::list<int>::iterator> lru_pos_;
  std::unordered_map<uint64_t, int> cached_;
};

// ---------------------------------------------------------------- model
struct Layer {
  half* attn_norm = nullptr;
  half* ffn_norm = nullptr;
  LinearW qkv[kSlots], o[kSlots], gu[kSlots], down[kSlots];  // per weight slot
};

struct Model {
  msw_model_cfg c{};
  bool is_draft = false;
  bool fmt_on[kSlots] = {false, false, false, false};
  half* embed = nullptr;
  half* lm_head = nullptr;
  half* lm_head_tf = nullptr;  // decode (tile-fragment) copy
  half* final_norm = nullptr;
  float* inv_freq = nullptr;
  float2* rope = nullptr;  // [max_seq_len + 64][head_dim/2] (cos, sin)
  std::vector<Layer> layers;
  half* kc = nullptr;
  half* vc = nullptr;
  // KV-cache compression mode: FP8 E4M3 pool, same [layer][block][kv_head][16][D]
  // layout at one byte per element, its own block allocator
  uint8_t* kc8 = nullptr;
  uint8_t* vc8 = nullptr;
  BlockPool pool8;
  int* kvc_blocks = nullptr;  // device [2][max_blocks]: fp16 / fp8 block lists of a compress
  cudaGraphExec_t graph_kv8 = nullptr;
  int graph_kv8_nodes = 0;
  size_t kv_layer_elems = 0;
  int nblk = 0;
  int max_blocks = 0;  // block-table row stride
  int* block_table = nullptr;  // device [rows, max_blocks]
  int bt_rows = 0;
  int nsplit = 1;
  AttnShape ash{};
  BlockPool pool;
  std::vector<void*> allocations;
  cudaGraphExec_t graph[kSlots] = {nullptr, nullptr, nullptr, nullptr};
  int graph_nodes[kSlots] = {0, 0, 0, 0};

  size_t weight_bytes(int fmt) const {
    size_t b = size_t(c.vocab) * c.hidden * 2;  // fp16 lm_head in every mode
    for (const Layer& l : layers)
      b += l.qkv[fmt].bytes() + l.o[fmt].bytes() + l.gu[fmt].bytes() + l.down[fmt].bytes();
    return b;
  }
};

struct Scratch {
  int tmax = 0;
  float* h = nullptr;
  float* qkv = nullptr;
  half* q16 = nullptr;
  float* o = nullptr;
  float* act = nullptr;
  half* xh = nullptr;
  int8_t* xq = nullptr;
  float* xscale = nullptr;
  float* hsel = nullptr;
  float* logits = nullptr;
  float* part_o = nullptr;
  float* part_ml = nullptr;
  int* tok = nullptr;
  int* pos = nullptr;
  int* slot = nullptr;
  int* seq_of = nullptr;
  int* logit_rows = nullptr;
  unsigned long long* amax_ws = nullptr;  // argmax slots + counters [2 * kMaxLogitRows], self-resetting
  int* split_cnt = nullptr;  // attention split-merge counters [tokens, kv heads], self-resetting
  int* next = nullptr;
  int* step = nullptr;
  int* hist = nullptr;
  int* stage = nullptr;  // pinned host staging
  size_t stage_ints = 0;
  SpecState* spec = nullptr;  // speculative-decoding round state (device)
  int* spec_out = nullptr;    // emitted tokens of the running spec request
  int* cb_hbase = nullptr;    // continuous batching: per live row, history base
  int* cb_hist = nullptr;     // continuous batching: generated tokens [max_batch][max_seq_len]
};

}  // namespace
}  // namespace msw

struct msw_engine {
  int device = 0;
  msw_engine_cfg cfg{};
  cudaStream_t st = nullptr;
  msw::Model target, draft;
  msw::Scratch sc;
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
  long long launches = 0;
  std::vector<void*> owned;
  cudaGraphExec_t spec_graph = nullptr;  // WHILE(tokens to emit) { spec round }
  int spec_round_nodes = 0;
  std::map<int, std::pair<cudaGraphExec_t, int>> cb_graphs;  // live-batch size -> (step graph, nodes)
};

namespace msw {
namespace {

// ------------------------------------------------------------ weight build
void build_successor(const msw_engine_cfg& cfg, int V, std::vector<int>& pred,
                     std::vector<uint8_t>& agree) {
  std::vector<std::pair<uint64_t, int>> order(V);
  const uint64_t skey = mix64(cfg.weight_seed ^ kSuccSalt);
  for (int v = 0; v < V; ++v) order[v] = {mix64(skey + uint64_t(v)), v};
  std::sort(order.begin(), order.end());
  pred.assign(V, 0);
  for (int i = 0; i < V; ++i) pred[order[(i + 1) % V].second] = order[i].second;
  agree.assign(V, 0);
  const uint64_t akey = mix64(cfg.weight_seed ^ kAgreeSalt);
  for (int t = 0; t < V; ++t)
    agree[t] = int(mix64(akey + uint64_t(t)) % 1000ull) < cfg.draft_agree_permille ? 1 : 0;
}

template <typename T>
T* model_alloc(Model& m, size_t count) {
  T* p = dalloc<T>(count);
  m.allocations.push_back(p);
  return p;
}

LinearW make_linear(Model& m, int slot, const half* master, int n, int k, cudaStream_t st) {
  LinearW L;
  const int fmt = slot == kSlotAWQ4 ? kW4 : slot;  // AWQ4: W4 layout plus zero points
  L.fmt = fmt;
  L.n = n;
  L.k = k;
  if (fmt == kFP16) {
    half* w = model_alloc<half>(m, size_t(n) * k);
    MSW_CUDA(cudaMemcpyAsync(w, master, size_t(n) * k * 2, cudaMemcpyDeviceToDevice, st));
    L.w = w;
  } else if (fmt == kINT8) {
    int8_t* q = model_alloc<int8_t>(m, size_t(n) * k);
    float* s = model_alloc<float>(m, n);
    launch_quant_int8(master, n, k, q, s, st);
    L.w = q;
    L.s = s;
  } else if (slot == kSlotAWQ4) {
    uint32_t* q = model_alloc<uint32_t>(m, size_t(n) * k / 8);
    half* s = model_alloc<half>(m, size_t(n) * (k / kW4Group));
    uint8_t* z = model_alloc<uint8_t>(m, size_t(n) * (k / kW4Group));
    launch_quant_awq4(master, n, k, q, s, z, st);
    L.w = q;
    L.s = s;
    L.z = z;
  } else {
    uint32_t* q = model_alloc<uint32_t>(m, size_t(n) * k / 8);
    half* s = model_alloc<half>(m, size_t(n) * (k / kW4Group));
    launch_quant_w4(master, n, k, q, s, st);
    L.w = q;
    L.s = s;
  }
  // decode copy in tile-fragment order (prefill keeps the row-major copy for TMA)
  uint8_t* tf = model_alloc<uint8_t>(m, tf_bytes(fmt, n, k));
  launch_repack_tf(fmt, L.w, n, k, tf, st);
  L.w_tf = tf;
  return L;
}

void build_model(Model& m, const msw_model_cfg& c, bool is_draft, const msw_engine_cfg& cfg,
                 const std::vector<int>& pred, const std::vector<uint8_t>& agree, cudaStream_t st) {
  m.c = c;
  m.is_draft = is_draft;
  const int H = c.hidden, V = c.vocab, L = c.n_layers, D = c.head_dim;
  const int Hq = c.n_heads, Hk = c.n_kv_heads, F = c.ffn;
  if (H % 128 || F % 128 || (Hq * D) % 128 || Hq % Hk || (D != 64 && D != 128))
    throw ConfigErr("model shape: hidden/ffn/heads*head_dim must be multiples of 128, head_dim 64|128");
  const uint64_t base = is_draft ? kTidDraftBase : 0ull;
  const uint64_t seed = cfg.weight_seed;

  m.embed = model_alloc<half>(m, size_t(V) * H);
  launch_fill_fp16(m.embed, V, H, seed, base + kTidEmbed, 0, st);
  m.final_norm = model_alloc<half>(m, H);
  launch_fill_norm(m.final_norm, H, seed, base + kTidFinalNorm, st);
  {
    int* d_pred = dalloc<int>(V);
    uint8_t* d_agree = dalloc<uint8_t>(V);
    MSW_CUDA(cudaMemcpy(d_pred, pred.data(), sizeof(int) * V, cudaMemcpyHostToDevice));
    MSW_CUDA(cudaMemcpy(d_agree, agree.data(), V, cudaMemcpyHostToDevice));
    m.lm_head = model_alloc<half>(m, size_t(V) * H);
    launch_lm_head(m.embed, d_pred, d_agree, is_draft ? 1 : 0, V, H, m.lm_head, st);
    m.lm_head_tf = model_alloc<half>(m, size_t(V) * H);
    launch_repack_tf(kFP16, m.lm_head, V, H, m.lm_head_tf, st);
    MSW_CUDA(cudaStreamSynchronize(st));
    cudaFree(d_pred);
    cudaFree(d_agree);
  }

  // which formats this model needs resident
  const uint32_t mm = cfg.modes_mask;
  if (is_draft) {
    m.fmt_on[kFP16] = true;
  } else {
    m.fmt_on[kFP16] = mm & ((1u << MSW_MODE_FP16) | (1u << MSW_MODE_SPECULATIVE) |
                            (1u << MSW_MODE_CHUNKED_PREFILL) | (1u << MSW_MODE_CUDA_GRAPHS));
    m.fmt_on[kINT8] = mm & ((1u << MSW_MODE_INT8) | (1u << MSW_MODE_INT8_CONT_BATCHING));
    m.fmt_on[kW4] = mm & ((1u << MSW_MODE_GPTQ4) | (1u << MSW_MODE_GPTQ_PREFIX_CACHING));
    m.fmt_on[kSlotAWQ4] = mm & (1u << MSW_MODE_AWQ4);
    m.fmt_on[kFP16] = m.fmt_on[kFP16] || (mm & (1u << MSW_MODE_KV_COMPRESSION));
  }

  const size_t max_elems = std::max({size_t(Hq + 2 * Hk) * D * H, size_t(2) * F * H,
                                     size_t(H) * Hq * D, size_t(H) * F});
  half* master = dalloc<half>(max_elems);
  half* tmp_a = dalloc<half>(size_t(F) * H);
  half* tmp_b = dalloc<half>(size_t(F) * H);
  const int rs = res_shift(L);
  m.layers.resize(L);
  for (int l = 0; l < L; ++l) {
    Layer& ly = m.layers[l];
    ly.attn_norm = model_alloc<half>(m, H);
    ly.ffn_norm = model_alloc<half>(m, H);
    launch_fill_norm(ly.attn_norm, H, seed, base + tid_layer(l, kAttnNorm), st);
    launch_fill_norm(ly.ffn_norm, H, seed, base + tid_layer(l, kFfnNorm), st);
    auto each_fmt = [&](LinearW (&dst)[kSlots], int n, int k) {
      for (int f = 0; f < kSlots; ++f)
        if (m.fmt_on[f]) dst[f] = make_linear(m, f, master, n, k, st);
    };
    // qkv: rows [q (Hq*D); k (Hk*D); v (Hk*D)]
    launch_fill_fp16(master, size_t(Hq) * D, H, seed, base + tid_layer(l, kQ), in_shift(H), st);
    launch_fill_fp16(master + size_t(Hq) * D * H, size_t(Hk) * D, H, seed,
                     base + tid_layer(l, kK), in_shift(H), st);
    launch_fill_fp16(master + size_t(Hq + Hk) * D * H, size_t(Hk) * D, H, seed,
                     base + tid_layer(l, kV), in_shift(H), st);
    each_fmt(ly.qkv, (Hq + 2 * Hk) * D, H);
    launch_fill_fp16(master, H, size_t(Hq) * D, seed, base + tid_layer(l, kO),
                     in_shift(Hq * D) + rs, st);
    each_fmt(ly.o, H, Hq * D);
    // gate/up interleaved by row (2i = gate_i, 2i+1 = up_i)
    launch_fill_fp16(tmp_a, F, H, seed, base + tid_layer(l, kGate), in_shift(H), st);
    launch_fill_fp16(tmp_b, F, H, seed, base + tid_layer(l, kUp), in_shift(H), st);
    launch_interleave_rows(tmp_a, tmp_b, F, size_t(H) * 2, master, st);
    each_fmt(ly.gu, 2 * F, H);
    launch_fill_fp16(master, H, F, seed, base + tid_layer(l, kDown), in_shift(F) + rs, st);
    each_fmt(ly.down, H, F);
    MSW_CUDA(cudaStreamSynchronize(st));  // master is reused next layer
  }
  cudaFree(master);
  cudaFree(tmp_a);
  cudaFree(tmp_b);

  // llama3 rope inverse frequencies (transformers _compute_llama3_parameters)
  std::vector<float> inv(D / 2);
  for (int j = 0; j < D / 2; ++j) {
    double f = std::pow(double(c.rope_theta), -(2.0 * j) / double(D));
    if (c.rope_factor > 0.0f) {
      const double lo_wl = c.rope_orig_ctx / c.rope_low_freq_factor;
      const double hi_wl = c.rope_orig_ctx / c.rope_high_freq_factor;
      const double wl = 2.0 * 3.14159265358979323846 / f;
      if (wl > lo_wl) {
        f = f / c.rope_factor;
      } else if (wl >= hi_wl) {
        const double sm = (c.rope_orig_ctx / wl - c.rope_low_freq_factor) /
                          (c.rope_high_freq_factor - c.rope_low_freq_factor);
        f = (1.0 - sm) * f / c.rope_factor + sm * f;
      }
    }
    inv[j] = float(f);
  }
  m.inv_freq = model_alloc<float>(m, D / 2);
  MSW_CUDA(cudaMemcpy(m.inv_freq, inv.data(), sizeof(float) * inv.size(), cudaMemcpyHostToDevice));
  m.rope = model_alloc<float2>(m, size_t(cfg.max_seq_len + 64) * (D / 2));
  launch_rope_table(m.inv_freq, D, cfg.max_seq_len + 64, m.rope, st);

  // paged KV pool
  m.nblk = cfg.kv_blocks;
  m.kv_layer_elems = size_t(m.nblk) * Hk * kKvBlock * D;
  m.kc = model_alloc<half>(m, m.kv_layer_elems * L);
  m.vc = model_alloc<half>(m, m.kv_layer_elems * L);
  // finite contents everywhere: tensor-core attention reads whole 16-row
  // blocks, and 0 x NaN from never-written rows would poison P x V
  MSW_CUDA(cudaMemsetAsync(m.kc, 0, sizeof(half) * m.kv_layer_elems * L, st));
  MSW_CUDA(cudaMemsetAsync(m.vc, 0, sizeof(half) * m.kv_layer_elems * L, st));
  m.max_blocks = (cfg.max_seq_len + kKvBlock - 1) / kKvBlock + 2;
  m.bt_rows = is_draft ? 1 : std::max(1, cfg.max_batch);
  m.block_table = model_alloc<int>(m, size_t(m.bt_rows) * m.max_blocks);
  MSW_CUDA(cudaMemset(m.block_table, 0, sizeof(int) * size_t(m.bt_rows) * m.max_blocks));
  m.pool.init(m.nblk);
  if (!is_draft && (cfg.modes_mask & (1u << MSW_MODE_KV_COMPRESSION))) {
    m.kc8 = model_alloc<uint8_t>(m, m.kv_layer_elems * L);
    m.vc8 = model_alloc<uint8_t>(m, m.kv_layer_elems * L);
    MSW_CUDA(cudaMemsetAsync(m.kc8, 0, m.kv_layer_elems * L, st));
    MSW_CUDA(cudaMemsetAsync(m.vc8, 0, m.kv_layer_elems * L, st));
    m.pool8.init(m.nblk);
    m.kvc_blocks = model_alloc<int>(m, size_t(2) * m.max_blocks);
  }
  m.ash = AttnShape{Hq, Hk, D, m.max_blocks, m.nblk};
  // decode attention splits hold >= 256 positions (attention.cu kDecMinChunk):
  // no more splits than max_seq_len needs, so short-context engines do not
  // launch idle CTAs; and no more (token, kv head, split) CTAs than SMs, so
  // the 8-warp CTAs (139 KB of staging, one per SM) run in ONE wave (32
  // splits x 8 kv heads at 8K context ran as two)
  m.nsplit = std::max(1, std::min({32, kNumSMs / Hk, (cfg.max_seq_len + 255) / 256}));
}

void free_model(Model& m) {
  for (auto& g : m.graph)
    if (g) cudaGraphExecDestroy(g);
  if (m.graph_kv8) cudaGraphExecDestroy(m.graph_kv8);
  for (void* p : m.allocations) cudaFree(p);
  m.allocations.clear();
}

void alloc_scratch(msw_engine* e) {
  Scratch& s = e->sc;
  const msw_model_cfg& t = e->cfg.target;
  const msw_model_cfg& d = e->cfg.has_draft ? e->cfg.draft : e->cfg.target;
  const int T = std::max({kPrefillChunk, e->cfg.max_batch, e->cfg.spec_k + 1, 8});
  s.tmax = T;
  auto mx = [&](auto f) { return std::max(f(t), f(d)); };
  const size_t H = mx([](const msw_model_cfg& c) { return size_t(c.hidden); });
  const size_t QKV = mx([](const msw_model_cfg& c) {
    return size_t(c.n_heads + 2 * c.n_kv_heads) * c.head_dim;
  });
  const size_t QD = mx([](const msw_model_cfg& c) { return size_t(c.n_heads) * c.head_dim; });
  const size_t F = mx([](const msw_model_cfg& c) { return size_t(c.ffn); });
  const size_t V = mx([](const msw_model_cfg& c) { return size_t(c.vocab); });
  const size_t K = std::max({H, QD, F});
  const size_t HQ = mx([](const msw_model_cfg& c) { return size_t(c.n_heads); });
  const size_t D = mx([](const msw_model_cfg& c) { return size_t(c.head_dim); });
  const size_t tsplit = std::max<size_t>(kMaxLogitRows, e->cfg.spec_k + 1);
  s.h = dalloc<float>(T * H);
  s.qkv = dalloc<float>(T * QKV);
  s.q16 = dalloc<half>(T * QD);
  s.o = dalloc<float>(T * QD);
  s.act = dalloc<float>(T * F);
  s.xh = dalloc<half>(T * K);
  s.xq = dalloc<int8_t>(T * K);
  s.xscale = dalloc<float>(T);
  s.hsel = dalloc<float>(kMaxLogitRows * H);
  s.logits = dalloc<float>(kMaxLogitRows * V);
  s.part_o = dalloc<float>(tsplit * HQ * 32 * D);
  s.part_ml = dalloc<float>(tsplit * HQ * 32 * 2);
  s.tok = dalloc<int>(T);
  s.pos = dalloc<int>(T);
  s.slot = dalloc<int>(T);
  s.seq_of = dalloc<int>(T);
  s.logit_rows = dalloc<int>(kMaxLogitRows);
  MSW_CUDA(cudaMemset(s.logit_rows, 0, sizeof(int) * kMaxLogitRows));
  s.split_cnt = dalloc<int>(tsplit * 64);
  MSW_CUDA(cudaMemset(s.split_cnt, 0, sizeof(int) * tsplit * 64));
  s.next = dalloc<int>(kMaxLogitRows);
  s.amax_ws = dalloc<unsigned long long>(2 * kMaxLogitRows);
  MSW_CUDA(cudaMemset(s.amax_ws, 0, sizeof(unsigned long long) * 2 * kMaxLogitRows));
  s.step = dalloc<int>(1);
  s.hist = dalloc<int>(size_t(e->cfg.max_seq_len) + 64);
  s.cb_hbase = dalloc<int>(T);
  s.cb_hist = dalloc<int>(size_t(std::max(1, e->cfg.max_batch)) * e->cfg.max_seq_len);
  s.spec = dalloc<SpecState>(1);
  s.spec_out = dalloc<int>(size_t(e->cfg.max_seq_len) + 64);
  {
    SpecState init{};
    init.out = s.spec_out;
    MSW_CUDA(cudaMemcpy(s.spec, &init, sizeof(init), cudaMemcpyHostToDevice));
  }
  s.stage_ints = std::max<size_t>(size_t(T) * 6 + 256, sizeof(SpecState) / sizeof(int) + 8);
  MSW_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&s.stage), s.stage_ints * sizeof(int),
                         cudaHostAllocDefault));
  for (void* p : {(void*)s.h, (void*)s.qkv, (void*)s.q16, (void*)s.o, (void*)s.act, (void*)s.xh,
                  (void*)s.xq, (void*)s.xscale, (void*)s.hsel, (void*)s.logits, (void*)s.part_o,
                  (void*)s.part_ml, (void*)s.tok, (void*)s.pos, (void*)s.slot, (void*)s.seq_of,
                  (void*)s.logit_rows, (void*)s.split_cnt, (void*)s.next, (void*)s.amax_ws, (void*)s.step,
                  (void*)s.hist, (void*)s.spec, (void*)s.spec_out,
                  (void*)s.cb_hbase, (void*)s.cb_hist})
    e->owned.push_back(p);
}

// ------------------------------------------------------------ forward pass
// Runs T tokens (inputs already in sc.tok/pos/slot/seq_of) through model m in
// format fmt; logits + argmax for the n_logits rows listed in sc.logit_rows
// (rows == nullptr means rows 0..n_logits-1 == all T rows).
// Diagnostics build only (-DMSW_TRACE, libmsw_engine_trace.so):
// MSW_SKIP="attn,qkv,o,gu,down,head,argmax" drops those launches from the step
// (outputs become meaningless) to attribute in-graph step time per kernel
// class. The product library compiles this to a constant false.
#ifdef MSW_TRACE
bool diag_skip(const char* what) {
  static const char* env = std::getenv("MSW_SKIP");
  return env && std::strstr(env, what);
}
#else
constexpr bool diag_skip(const char*) { return false; }
#endif

void forward(msw_engine* e, Model& m, int fmt, int T, int n_logits, bool rows_identity,
             bool tokens_independent, bool one_seq = false, bool kv8 = false) {
  if (kv8 && !(tokens_independent && T == 1)) throw ConfigErr("FP8 KV cache: batch-1 decode steps only");
  Scratch& s = e->sc;
  cudaStream_t st = e->st;
  const msw_model_cfg& c = m.c;
  const int H = c.hidden, D = c.head_dim, Hq = c.n_heads, Hk = c.n_kv_heads, F = c.ffn;
  const float eps = c.rms_eps;
  const bool small = T <= kGemvMaxTokens;
  const int kfmt = fmt == kSlotAWQ4 ? kW4 : fmt;  // activation handling of the weight slot
  // attention splits: enough CTAs to fill the GPU, fewer as the token count grows
  int nsplit = 1;
  if (T <= kMaxLogitRows) nsplit = std::max(1, std::min(m.nsplit, kNumSMs / (T * Hk)));
  long long& n = e->launches;

  LinearW head;
  head.fmt = kFP16;
  head.n = c.vocab;
  head.k = H;
  head.w = m.lm_head;
  head.w_tf = m.lm_head_tf;
  launch_embed(m.embed, s.tok, T, H, s.h, st);
  ++n;
  for (int l = 0; l < c.n_layers; ++l) {
    const Layer& ly = m.layers[l];
    half* kc = m.kc + m.kv_layer_elems * l;
    half* vc = m.vc + m.kv_layer_elems * l;
    // attention block
    if (small) {
      if (!diag_skip("qkv"))
        launch_gemv(ly.qkv[fmt], kProNorm, kEpiStore, s.h, T, ly.attn_norm, eps, s.qkv, st, &ly.o[fmt]);
      ++n;
    } else {
      launch_prep_act(kfmt, s.h, T, H, ly.attn_norm, eps, s.xh, s.xq, s.xscale, st);
      launch_gemm(ly.qkv[fmt], kEpiStore, s.xh, s.xq, s.xscale, T, s.qkv, st);
      n += 2;
    }
    const bool run = !tokens_independent && one_seq && T <= kGemvMaxTokens;
    if (tokens_independent || run) {  // decode / CB / short runs: RoPE + KV append fused
      if (kv8)
        launch_attention_decode_kv8(s.qkv, m.rope, T, s.pos, s.slot, s.seq_of, m.block_table,
                                    m.kc8 + m.kv_layer_elems * l, m.vc8 + m.kv_layer_elems * l,
                                    m.ash, nsplit, s.part_o, s.part_ml, s.split_cnt, s.o, st, run);
      else if (!diag_skip("attn"))
        launch_attention_decode(s.qkv, m.rope, T, s.pos, s.slot, s.seq_of, m.block_table, kc, vc,
                                m.ash, nsplit, s.part_o, s.part_ml, s.split_cnt, s.o, st, run);
      n += 1;
    } else {
      launch_rope_append(s.qkv, T, s.pos, s.slot, m.rope, m.ash, s.q16, kc, vc, st);
      if (T > kMaxLogitRows) {
        launch_attention_prefill(s.q16, T, s.pos, s.seq_of, m.block_table, kc, vc, m.ash, s.o, st);
        n += 2;
      } else {
        launch_attention(s.q16, T, s.pos, s.seq_of, m.block_table, kc, vc, m.ash, nsplit,
                         s.part_o, s.part_ml, s.o, st);
        n += nsplit > 1 ? 3 : 2;
      }
    }
    if (small) {
      // each GEMV prefetches the head of the next one's weight stream into L2
      const LinearW* after_down = l + 1 < c.n_layers ? &m.layers[l + 1].qkv[fmt] : &head;
      if (!diag_skip("o,") && !diag_skip("oonly"))
        launch_gemv(ly.o[fmt], kProPlain, kEpiResid, s.o, T, nullptr, eps, s.h, st, &ly.gu[fmt]);
      if (!diag_skip("gu"))
        launch_gemv(ly.gu[fmt], kProNorm, kEpiSwiglu, s.h, T, ly.ffn_norm, eps, s.act, st, &ly.down[fmt]);
      if (!diag_skip("down"))
        launch_gemv(ly.down[fmt], kProPlain, kEpiResid, s.act, T, nullptr, eps, s.h, st, after_down);
      n += 3;
    } else {
      launch_prep_act(kfmt, s.o, T, Hq * D, nullptr, eps, s.xh, s.xq, s.xscale, st);
      launch_gemm(ly.o[fmt], kEpiResid, s.xh, s.xq, s.xscale, T, s.h, st);
      launch_prep_act(kfmt, s.h, T, H, ly.ffn_norm, eps, s.xh, s.xq, s.xscale, st);
      launch_gemm(ly.gu[fmt], kEpiSwiglu, s.xh, s.xq, s.xscale, T, s.act, st);
      launch_prep_act(kfmt, s.act, T, F, nullptr, eps, s.xh, s.xq, s.xscale, st);
      launch_gemm(ly.down[fmt], kEpiResid, s.xh, s.xq, s.xscale, T, s.h, st);
      n += 6;
    }
    (void)Hk;
  }
  // final norm + fp16 lm_head on the requested rows, then greedy argmax
  const float* hrows = s.h;
  if (!rows_identity) {
    launch_gather_rows(s.h, s.logit_rows, n_logits, H, s.hsel, st);
    hrows = s.hsel;
    ++n;
  }
  if (n_logits <= kGemvMaxTokens) {
    if (!diag_skip("head")) launch_gemv(head, kProNorm, kEpiStore, hrows, n_logits, m.final_norm, eps, s.logits, st);
    ++n;
  } else {
    launch_prep_act(kFP16, hrows, n_logits, H, m.final_norm, eps, s.xh, s.xq, s.xscale, st);
    launch_gemm(head, kEpiStore, s.xh, s.xq, s.xscale, n_logits, s.logits, st);
    n += 2;
  }
  if (!diag_skip("argmax")) launch_argmax(s.logits, n_logits, c.vocab, s.next, s.amax_ws, st);
  ++n;
}

// ------------------------------------------------------------ sequences
struct SeqBlocks {
  std::vector<int> blocks;
  int hit_tokens = 0;
  std::vector<uint64_t> keys;  // prefix keys of full prompt blocks (prefix caching)
};

uint64_t block_key(uint64_t prev, int fmt, const int32_t* toks) {
  uint64_t h = mix64(prev ^ (0xB10C0000ull + uint64_t(fmt)));
  for (int i = 0; i < kKvBlock; ++i) h = mix64(h ^ uint64_t(uint32_t(toks[i])));
  return h == 0 ? 1 : h;
}

// Maps n_positions KV slots for a sequence onto pool blocks; with prefix
// caching, leading full prompt blocks are looked up by content key.
SeqBlocks map_sequence(Model& m, int row, int n_positions, const int32_t* prompt, int plen,
                       bool prefix, int fmt, cudaStream_t st, int* stage) {
  SeqBlocks sb;
  const int nb = (n_positions + kKvBlock - 1) / kKvBlock;
  if (nb > m.max_blocks) throw DataErr("sequence longer than max_seq_len");
  int b = 0;
  if (prefix) {
    uint64_t key = 0x5EEDull;
    const int full = plen / kKvBlock;
    for (int i = 0; i < full; ++i) {
      key = block_key(key, fmt, prompt + size_t(i) * kKvBlock);
      sb.keys.push_back(key);
    }
    const int max_hit = (plen - 1) / kKvBlock;  // keep >= 1 prompt token to prefill
    for (; b < max_hit; ++b) {
      const int blk = m.pool.lookup(sb.keys[b]);
      if (blk < 0) break;
      sb.blocks.push_back(blk);
    }
    sb.hit_tokens = b * kKvBlock;
  }
  try {
    for (; b < nb; ++b) sb.blocks.push_back(m.pool.alloc());
  } catch (...) {
    for (int blk : sb.blocks) m.pool.release(blk);
    throw;
  }
  for (int i = 0; i < nb; ++i) stage[i] = sb.blocks[i];
  MSW_CUDA(cudaMemcpyAsync(m.block_table + size_t(row) * m.max_blocks, stage, sizeof(int) * nb,
                           cudaMemcpyHostToDevice, st));
  MSW_CUDA(cudaStreamSynchronize(st));
  return sb;
}

void publish_prefix(Model& m, const SeqBlocks& sb) {
  for (size_t i = sb.hit_tokens / kKvBlock; i < sb.keys.size(); ++i)
    m.pool.publish(sb.blocks[i], sb.keys[i]);
}

void release_sequence(Model& m, const SeqBlocks& sb) {
  for (int b : sb.blocks) m.pool.release(b);
}

// Prefill tokens [from, plen) of one sequence (block-table row `row`), in
// chunks; the last chunk yields logits/argmax for the last prompt token.
void prefill(msw_engine* e, Model& m, int fmt, int row, const int32_t* prompt, int from, int plen,
             const SeqBlocks& sb, int chunk = kPrefillChunk) {
  Scratch& s = e->sc;
  for (int c0 = from; c0 < plen; c0 += chunk) {
    const int T = std::min(chunk, plen - c0);
    int* st_tok = s.stage;
    int* st_pos = s.stage + T;
    int* st_slot = s.stage + 2 * T;
    int* st_seq = s.stage + 3 * T;
    for (int i = 0; i < T; ++i) {
      const int p = c0 + i;
      st_tok[i] = prompt[p];
      st_pos[i] = p;
      st_slot[i] = sb.blocks[p / kKvBlock] * kKvBlock + p % kKvBlock;
      st_seq[i] = row;
    }
    MSW_CUDA(cudaMemcpyAsync(s.tok, st_tok, sizeof(int) * T, cudaMemcpyHostToDevice, e->st));
    MSW_CUDA(cudaMemcpyAsync(s.pos, st_pos, sizeof(int) * T, cudaMemcpyHostToDevice, e->st));
    MSW_CUDA(cudaMemcpyAsync(s.slot, st_slot, sizeof(int) * T, cudaMemcpyHostToDevice, e->st));
    MSW_CUDA(cudaMemcpyAsync(s.seq_of, st_seq, sizeof(int) * T, cudaMemcpyHostToDevice, e->st));
    // every chunk's head runs on its last token (only the last chunk's result
    // is used; the row must be valid either way)
    if (T > 1) {
      int* st_rows = s.stage + 4 * T;
      st_rows[0] = T - 1;
      MSW_CUDA(cudaMemcpyAsync(s.logit_rows, st_rows, sizeof(int), cudaMemcpyHostToDevice, e->st));
    }
    forward(e, m, fmt, T, 1, /*rows_identity=*/T == 1, /*tokens_independent=*/T == 1,
            /*one_seq=*/true);
    MSW_CUDA(cudaStreamSynchronize(e->st));  // staging is reused by the next chunk
  }
}

// Packed prefill of several sequences (continuous-batching admission): the
// prompts of all admitted sequences are concatenated into chunks of up to
// kPrefillChunk tokens (ragged; every token carries its own seq_of / pos), so
// one GEMM per linear covers the whole cohort. A sequence may straddle chunks
// (attention reads the earlier chunk's K/V from the paged cache). The first
// generated token of sequence i lands in first_tok[i]; with logits_out[i]
// non-null its fp32 logits row is copied there.
void copy_logits_row(msw_engine* e, float* dst_host, int row);

struct PackSeq {
  int row;
  const int32_t* prompt;
  int plen;
  const SeqBlocks* sb;
};

void prefill_packed(msw_engine* e, Model& m, int fmt, const std::vector<PackSeq>& seqs,
                    int* first_tok, float* const* logits_out) {
  Scratch& s = e->sc;
  size_t i = 0;
  int p0 = 0;  // next prompt position of seqs[i]
  while (i < seqs.size()) {
    int T = 0, nl = 0;
    int* st_tok = s.stage;
    int* st_pos = s.stage + kPrefillChunk;
    int* st_slot = s.stage + 2 * kPrefillChunk;
    int* st_seq = s.stage + 3 * kPrefillChunk;
    int* st_rows = s.stage + 4 * kPrefillChunk;
    std::vector<int> owners;
    while (i < seqs.size() && T < kPrefillChunk && nl < kMaxLogitRows) {
      const PackSeq& q = seqs[i];
      const int take = std::min(q.plen - p0, kPrefillChunk - T);
      for (int j = 0; j < take; ++j) {
        const int p = p0 + j;
        st_tok[T + j] = q.prompt[p];
        st_pos[T + j] = p;
        st_slot[T + j] = q.sb->blocks[p / kKvBlock] * kKvBlock + p % kKvBlock;
        st_seq[T + j] = q.row;
      }
      T += take;
      p0 += take;
      if (p0 == q.plen) {
        st_rows[nl++] = T - 1;
        owners.push_back(int(i));
        ++i;
        p0 = 0;
      }
    }
    MSW_CUDA(cudaMemcpyAsync(s.tok, st_tok, sizeof(int) * T, cudaMemcpyHostToDevice, e->st));
    MSW_CUDA(cudaMemcpyAsync(s.pos, st_pos, sizeof(int) * T, cudaMemcpyHostToDevice, e->st));
    MSW_CUDA(cudaMemcpyAsync(s.slot, st_slot, sizeof(int) * T, cudaMemcpyHostToDevice, e->st));
    MSW_CUDA(cudaMemcpyAsync(s.seq_of, st_seq, sizeof(int) * T, cudaMemcpyHostToDevice, e->st));
    if (nl == 0) st_rows[0] = T - 1;  // no sequence ends here: head on a valid (unused) row
    MSW_CUDA(cudaMemcpyAsync(s.logit_rows, st_rows, sizeof(int) * std::max(nl, 1),
                             cudaMemcpyHostToDevice, e->st));
    const bool ident = nl == T;  // every token is some sequence's last
    forward(e, m, fmt, T, std::max(nl, 1), ident, false);
    int* got = s.stage + 4 * kPrefillChunk + kMaxLogitRows;
    if (nl > 0) {
      MSW_CUDA(cudaMemcpyAsync(got, s.next, sizeof(int) * nl, cudaMemcpyDeviceToHost, e->st));
      for (int j = 0; j < nl; ++j)
        if (logits_out[owners[j]]) copy_logits_row(e, logits_out[owners[j]], j);
    }
    MSW_CUDA(cudaStreamSynchronize(e->st));  // staging is reused by the next chunk
    for (int j = 0; j < nl; ++j) first_tok[owners[j]] = got[j];
  }
}

// One batch-1 decode step for model m / fmt, as a graph or eagerly.
void decode_step(msw_engine* e, Model& m, int fmt, bool use_graph, bool kv8 = false) {
  Scratch& s = e->sc;
  auto body = [&]() {
    forward(e, m, fmt, 1, 1, true, true, false, kv8);
    launch_advance(s.next, s.tok, s.pos, s.slot, s.step, s.hist, m.block_table, e->st);
    ++e->launches;
  };
  if (!use_graph) {
    body();
    return;
  }
  cudaGraphExec_t& gx = kv8 ? m.graph_kv8 : m.graph[fmt];
  int& gn = kv8 ? m.graph_kv8_nodes : m.graph_nodes[fmt];
  if (!gx) {
    const long long before = e->launches;
    cudaGraph_t g;
    MSW_CUDA(cudaStreamBeginCapture(e->st, cudaStreamCaptureModeThreadLocal));
    try {
      body();
    } catch (...) {
      cudaStreamEndCapture(e->st, &g);
      throw;
    }
    MSW_CUDA(cudaStreamEndCapture(e->st, &g));
    MSW_CUDA(cudaGraphInstantiate(&gx, g, 0));
    cudaGraphDestroy(g);
    gn = int(e->launches - before);
    e->launches = before;
  }
  MSW_CUDA(cudaGraphLaunch(gx, e->st));
  e->launches += gn;
}

// Sets the batch-1 decode state so the next decode_step processes `tok_src`
// (device int) at position pos; history[step0 ..] continues.
void start_decode(msw_engine* e, Model& m, const int* next_src, int pos_before, int step0) {
  Scratch& s = e->sc;
  int* st = s.stage + s.stage_ints - 8;
  st[0] = pos_before;
  st[1] = step0;
  MSW_CUDA(cudaMemcpyAsync(s.pos, &st[0], sizeof(int), cudaMemcpyHostToDevice, e->st));
  MSW_CUDA(cudaMemcpyAsync(s.step, &st[1], sizeof(int), cudaMemcpyHostToDevice, e->st));
  // advance: history[step0] = next, tok = next, pos = pos_before + 1, slot
  launch_advance(next_src, s.tok, s.pos, s.slot, s.step, s.hist, m.block_table, e->st);
  ++e->launches;
}

double now_ms() {
  return std::chrono::duration<double, std::milli>(
             std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

void check_request(msw_engine* e, const msw_request& r, int extra) {
  if (r.prompt_len < 1 || r.max_new_tokens < 1) throw DataErr("prompt_len and max_new_tokens must be >= 1");
  if (r.prompt_ids == nullptr) throw DataErr("prompt_ids is NULL");
  if (r.prompt_len + r.max_new_tokens + extra > e->cfg.max_seq_len)
    throw DataErr("request exceeds max_seq_len");
  for (int i = 0; i < r.prompt_len; ++i)
    if (r.prompt_ids[i] < 0 || r.prompt_ids[i] >= e->cfg.target.vocab)
      throw DataErr("token id out of range");
}

void copy_logits_row(msw_engine* e, float* dst_host, int row) {
  MSW_CUDA(cudaMemcpyAsync(dst_host, e->sc.logits + size_t(row) * e->cfg.target.vocab,
                           sizeof(float) * e->cfg.target.vocab, cudaMemcpyDeviceToHost, e->st));
}

// ---------------------------------------------------------------- modes
void run_single(msw_engine* e, const msw_request& r, msw_result& res) {
  const int fmt = fmt_of_mode(r.mode);
  Model& m = e->target;
  if (!m.fmt_on[fmt]) throw ConfigErr("mode not resident in this engine");
  check_request(e, r, 1);
  const double t0 = now_ms();
  const bool prefix = r.mode == MSW_MODE_GPTQ_PREFIX_CACHING;
  const int n_new = r.max_new_tokens;
  SeqBlocks sb = map_sequence(m, 0, r.prompt_len + n_new, r.prompt_ids, r.prompt_len, prefix, fmt,
                              e->st, e->sc.stage);
  const bool want_logits = res.logits != nullptr;
  // CudaGraphs screening mode: graph-replayed decode even when the engine was
  // configured eager (cfg.use_graphs = 0); ChunkedPrefill: 512-token prefill chunks
  const bool graphs = (e->cfg.use_graphs || r.mode == MSW_MODE_CUDA_GRAPHS) && !want_logits;
  try {
    MSW_CUDA(cudaEventRecord(e->ev[0], e->st));
    prefill(e, m, fmt, 0, r.prompt_ids, sb.hit_tokens, r.prompt_len, sb,
            r.mode == MSW_MODE_CHUNKED_PREFILL ? kChunkedPrefillTokens : kPrefillChunk);
    if (want_logits) copy_logits_row(e, res.logits, 0);
    start_decode(e, m, e->sc.next, r.prompt_len - 1, 0);
    MSW_CUDA(cudaEventRecord(e->ev[1], e->st));
    for (int i = 1; i < n_new; ++i) {
      decode_step(e, m, fmt, graphs);
      if (want_logits) copy_logits_row(e, res.logits + size_t(i) * m.c.vocab, 0);
    }
    MSW_CUDA(cudaEventRecord(e->ev[2], e->st));
    MSW_CUDA(cudaMemcpyAsync(res.out_ids, e->sc.hist, sizeof(int) * n_new, cudaMemcpyDeviceToHost,
                             e->st));
    MSW_CUDA(cudaStreamSynchronize(e->st));
  } catch (...) {
    release_sequence(m, sb);
    throw;
  }
  if (prefix) publish_prefix(m, sb);
  release_sequence(m, sb);
  float a = 0, b = 0;
  MSW_CUDA(cudaEventElapsedTime(&a, e->ev[0], e->ev[1]));
  MSW_CUDA(cudaEventElapsedTime(&b, e->ev[1], e->ev[2]));
  res.prefill_ms = a;
  res.decode_ms = b;
  res.n_out = n_new;
  res.prefix_hit_tokens = sb.hit_tokens;
  res.total_ms = now_ms() - t0;
}

// KV-cache compression (screening mode, reference domain.hpp:81): FP16
// weights; the prompt is prefilled on the fp16 cache (full-precision prefill
// attention), its K / V are then converted to FP8 E4M3 blocks of a separate
// pool and the fp16 blocks are released, so the request holds its context at
// one byte per element for the whole decode; each decode step appends E4M3
// K / V and attends over the E4M3 cache (attn_decode_kernel<..., KV8>).
void run_kvc(msw_engine* e, const msw_request& r, msw_result& res) {
  Model& m = e->target;
  if (!m.kc8 || !m.fmt_on[kFP16]) throw ConfigErr("mode not resident in this engine");
  check_request(e, r, 1);
  Scratch& s = e->sc;
  const double t0 = now_ms();
  const int plen = r.prompt_len, n_new = r.max_new_tokens;
  SeqBlocks s16 = map_sequence(m, 0, plen, r.prompt_ids, plen, false, kFP16, e->st, s.stage);
  std::vector<int> b8;
  const bool want_logits = res.logits != nullptr;
  const bool graphs = e->cfg.use_graphs && !want_logits;
  bool released16 = false;
  try {
    const int nb8 = (plen + n_new + kKvBlock - 1) / kKvBlock;
    if (nb8 > m.max_blocks) throw DataErr("sequence longer than max_seq_len");
    for (int i = 0; i < nb8; ++i) b8.push_back(m.pool8.alloc());
    MSW_CUDA(cudaEventRecord(e->ev[0], e->st));
    prefill(e, m, kFP16, 0, r.prompt_ids, 0, plen, s16);
    if (want_logits) copy_logits_row(e, res.logits, 0);
    // block lists for the conversion, then the row points at the E4M3 blocks
    const int nb16 = int(s16.blocks.size());
    int* stg = s.stage;
    for (int i = 0; i < nb16; ++i) stg[i] = s16.blocks[i];
    for (int i = 0; i < nb8; ++i) stg[m.max_blocks + i] = b8[i];
    MSW_CUDA(cudaMemcpyAsync(m.kvc_blocks, stg, sizeof(int) * (m.max_blocks + nb8),
                             cudaMemcpyHostToDevice, e->st));
    MSW_CUDA(cudaMemcpyAsync(m.block_table, stg + m.max_blocks, sizeof(int) * nb8,
                             cudaMemcpyHostToDevice, e->st));
    launch_kv_compress(m.kc, m.vc, m.kc8, m.vc8, m.kv_layer_elems, m.c.n_layers, m.kvc_blocks,
                       m.kvc_blocks + m.max_blocks, plen, m.c.n_kv_heads, m.c.head_dim, e->st);
    ++e->launches;
    // stream order: anything that reuses these blocks runs after the conversion
    release_sequence(m, s16);
    released16 = true;
    start_decode(e, m, s.next, plen - 1, 0);
    MSW_CUDA(cudaEventRecord(e->ev[1], e->st));
    for (int i = 1; i < n_new; ++i) {
      decode_step(e, m, kFP16, graphs, /*kv8=*/true);
      if (want_logits) copy_logits_row(e, res.logits + size_t(i) * m.c.vocab, 0);
    }
    MSW_CUDA(cudaEventRecord(e->ev[2], e->st));
    MSW_CUDA(cudaMemcpyAsync(res.out_ids, s.hist, sizeof(int) * n_new, cudaMemcpyDeviceToHost,
                             e->st));
    MSW_CUDA(cudaStreamSynchronize(e->st));
  } catch (...) {
    cudaStreamSynchronize(e->st);
    if (!released16) release_sequence(m, s16);
    for (int b : b8) m.pool8.release(b);
    throw;
  }
  for (int b : b8) m.pool8.release(b);
  float a = 0, b = 0;
  MSW_CUDA(cudaEventElapsedTime(&a, e->ev[0], e->ev[1]));
  MSW_CUDA(cudaEventElapsedTime(&b, e->ev[1], e->ev[2]));
  res.prefill_ms = a;
  res.decode_ms = b;
  res.n_out = n_new;
  res.total_ms = now_ms() - t0;
}

// Speculative decoding: FP16 target + FP16 draft, k greedy proposals, one
// batched verify of k+1 tokens; emitted tokens are the target's greedy tokens.
// Everything after the two prefills runs on the device: one round is the
// draft's T=2 step (re-running position n-2 so the round shape is fixed), its
// k-1 T=1 steps, the target's (k+1)-token verify and the accept kernel, which
// commits the tokens to the device state and sets the condition of the CUDA
// graph WHILE node that repeats the round. A request's whole decode is one
// graph launch with no host synchronisation; the host reads the tokens and
// counters once at the end.
void spec_round(msw_engine* e, cudaGraphConditionalHandle cond, bool use_cond) {
  Scratch& s = e->sc;
  Model& dr = e->draft;
  Model& tg = e->target;
  const int k = e->cfg.spec_k;
  cudaStream_t st = e->st;
  launch_spec_draft_setup(s.spec, s.tok, s.pos, s.slot, s.seq_of, s.logit_rows, dr.block_table, st);
  forward(e, dr, kFP16, 2, 1, /*rows_identity=*/false, /*tokens_independent=*/false,
          /*one_seq=*/true);
  for (int i = 1; i < k; ++i) {
    launch_spec_draft_next(s.spec, i, s.next, s.tok, s.pos, s.slot, s.seq_of, dr.block_table, st);
    forward(e, dr, kFP16, 1, 1, true, true);
  }
  launch_spec_verify_setup(s.spec, k, s.next, s.tok, s.pos, s.slot, s.seq_of, tg.block_table, st);
  forward(e, tg, kFP16, k + 1, k + 1, true, false, /*one_seq=*/true);
  launch_spec_accept(s.spec, k, s.next, s.logits, tg.c.vocab, cond, use_cond, st);
  e->launches += 4 + k;
}

void build_spec_graph(msw_engine* e) {
  cudaGraph_t g;
  MSW_CUDA(cudaGraphCreate(&g, 0));
  try {
    cudaGraphConditionalHandle h;
    MSW_CUDA(cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault));
    cudaGraphNodeParams p{};
    p.type = cudaGraphNodeTypeConditional;
    p.conditional.handle = h;
    p.conditional.type = cudaGraphCondTypeWhile;
    p.conditional.size = 1;
    cudaGraphNode_t node;
    MSW_CUDA(cudaGraphAddNode(&node, g, nullptr, 0, &p));
    cudaGraph_t body = p.conditional.phGraph_out[0];
    const long long before = e->launches;
    MSW_CUDA(cudaStreamBeginCaptureToGraph(e->st, body, nullptr, nullptr, 0,
                                           cudaStreamCaptureModeThreadLocal));
    try {
      spec_round(e, h, true);
    } catch (...) {
      cudaGraph_t dummy;
      cudaStreamEndCapture(e->st, &dummy);
      throw;
    }
    MSW_CUDA(cudaStreamEndCapture(e->st, &body));
    e->spec_round_nodes = int(e->launches - before);
    e->launches = before;
    MSW_CUDA(cudaGraphInstantiate(&e->spec_graph, g, 0));
  } catch (...) {
    cudaGraphDestroy(g);
    throw;
  }
  cudaGraphDestroy(g);
}

void run_spec(msw_engine* e, const msw_request& r, msw_result& res) {
  if (!e->cfg.has_draft) throw ConfigErr("speculative decoding needs a draft model");
  Model& tg = e->target;
  Model& dr = e->draft;
  if (!tg.fmt_on[kFP16]) throw ConfigErr("speculative decoding needs the FP16 target");
  const int k = e->cfg.spec_k;
  if (k < 1 || k + 1 > kGemvMaxTokens || k > kSpecMaxK) throw ConfigErr("spec_k must be in [1, 5]");
  check_request(e, r, k + 2);
  Scratch& s = e->sc;
  const int plen = r.prompt_len, n_new = r.max_new_tokens, V = tg.c.vocab;
  const double t0 = now_ms();
  const int npos = plen + n_new + k + 2;
  SeqBlocks tb = map_sequence(tg, 0, npos, r.prompt_ids, plen, false, kFP16, e->st, s.stage);
  SeqBlocks db;
  try {
    db = map_sequence(dr, 0, npos, r.prompt_ids, plen, false, kFP16, e->st, s.stage);
  } catch (...) {
    release_sequence(tg, tb);
    throw;
  }
  const bool graphs = e->cfg.use_graphs != 0;
  float* lg_dev = nullptr;
  SpecState fin{};
  float prefill_ms = 0, decode_ms = 0;
  try {
    if (res.logits) lg_dev = dalloc<float>(size_t(n_new) * V);
    if (graphs && !e->spec_graph) build_spec_graph(e);
    MSW_CUDA(cudaEventRecord(e->ev[0], e->st));
    prefill(e, dr, kFP16, 0, r.prompt_ids, 0, plen, db);
    prefill(e, tg, kFP16, 0, r.prompt_ids, 0, plen, tb);
    launch_spec_init(s.spec, s.next, plen, n_new, r.prompt_ids[plen - 1], lg_dev, e->st);
    if (lg_dev)
      MSW_CUDA(cudaMemcpyAsync(lg_dev, s.logits, sizeof(float) * V, cudaMemcpyDeviceToDevice, e->st));
    e->launches += 1;
    MSW_CUDA(cudaEventRecord(e->ev[1], e->st));
    if (n_new > 1) {
      if (graphs) {
        MSW_CUDA(cudaGraphLaunch(e->spec_graph, e->st));
      } else {
        int* emitted = s.stage;
        do {
          spec_round(e, 0, false);
          MSW_CUDA(cudaMemcpyAsync(emitted, &s.spec->emitted, sizeof(int), cudaMemcpyDeviceToHost, e->st));
          MSW_CUDA(cudaStreamSynchronize(e->st));
        } while (*emitted < n_new);
      }
    }
    MSW_CUDA(cudaEventRecord(e->ev[2], e->st));
    MSW_CUDA(cudaMemcpyAsync(res.out_ids, s.spec_out, sizeof(int) * n_new, cudaMemcpyDeviceToHost, e->st));
    MSW_CUDA(cudaMemcpyAsync(s.stage, s.spec, sizeof(SpecState), cudaMemcpyDeviceToHost, e->st));
    if (lg_dev)
      MSW_CUDA(cudaMemcpyAsync(res.logits, lg_dev, sizeof(float) * size_t(n_new) * V,
                               cudaMemcpyDeviceToHost, e->st));
    MSW_CUDA(cudaStreamSynchronize(e->st));
    std::memcpy(&fin, s.stage, sizeof(SpecState));
    MSW_CUDA(cudaEventElapsedTime(&prefill_ms, e->ev[0], e->ev[1]));
    MSW_CUDA(cudaEventElapsedTime(&decode_ms, e->ev[1], e->ev[2]));
  } catch (...) {
    if (lg_dev) cudaFree(lg_dev);
    release_sequence(tg, tb);
    release_sequence(dr, db);
    throw;
  }
  if (lg_dev) cudaFree(lg_dev);
  release_sequence(tg, tb);
  release_sequence(dr, db);
  if (graphs) e->launches += (long long)fin.rounds * e->spec_round_nodes;
  res.n_out = n_new;
  res.prefill_ms = prefill_ms;
  res.decode_ms = decode_ms;
  res.spec_rounds = fin.rounds;
  res.spec_proposed = fin.proposed;
  res.spec_accepted = fin.accepted;
  res.total_ms = now_ms() - t0;
}

// INT8 + continuous batching: iteration-level scheduling of a co-scheduled
// cohort. Up to max_batch live sequences; each engine step decodes one token
// for every live sequence (ragged positions, one block-table row each);
// finished sequences retire and queued ones are admitted (prefilled, packed)
// before the next step. Per-request latency = its admission to its last token.
//
// The step state (input token, position, KV slot, row, history base of every
// live sequence) stays on the device and the step's own cb_advance kernel
// moves it forward, so between scheduling events (a retirement, which frees a
// row and KV blocks for admission) the host issues the steps back to back —
// one CUDA graph per live-batch size T — and synchronises only at the event.
// The host knows when the next event is: min over live sequences of the
// tokens they still have to generate.
void cb_step_body(msw_engine* e, Model& m, int T) {
  Scratch& s = e->sc;
  forward(e, m, kINT8, T, T, true, true);
  launch_cb_advance(s.next, T, s.tok, s.pos, s.slot, s.seq_of, s.cb_hbase, s.cb_hist,
                    m.block_table, m.max_blocks, e->st);
  ++e->launches;
}

// The step graph of a live-batch size T (captured once per engine).
std::map<int, std::pair<cudaGraphExec_t, int>>::iterator cb_graph(msw_engine* e, Model& m, int T) {
  auto body = [&]() { cb_step_body(e, m, T); };
  auto it = e->cb_graphs.find(T);
  if (it == e->cb_graphs.end()) {
    const long long before = e->launches;
    cudaGraph_t g;
    MSW_CUDA(cudaStreamBeginCapture(e->st, cudaStreamCaptureModeThreadLocal));
    try {
      body();
    } catch (...) {
      cudaStreamEndCapture(e->st, &g);
      throw;
    }
    MSW_CUDA(cudaStreamEndCapture(e->st, &g));
    cudaGraphExec_t x;
    const cudaError_t rc = cudaGraphInstantiate(&x, g, 0);
    cudaGraphDestroy(g);
    MSW_CUDA(rc);
    it = e->cb_graphs.emplace(T, std::make_pair(x, int(e->launches - before))).first;
    e->launches = before;
  }
  return it;
}

void cb_step(msw_engine* e, Model& m, int T, bool use_graph) {
  if (!use_graph) {
    cb_step_body(e, m, T);
    return;
  }
  auto it = cb_graph(e, m, T);
  MSW_CUDA(cudaGraphLaunch(it->second.first, e->st));
  e->launches += it->second.second;
}

void run_cb(msw_engine* e, const msw_request* reqs, int n, msw_result* res) {
  Model& m = e->target;
  const int fmt = kINT8;
  if (!m.fmt_on[fmt]) throw ConfigErr("INT8 weights not resident");
  const int maxb = std::min(e->cfg.max_batch, std::min(m.bt_rows, kMaxLogitRows));
  for (int i = 0; i < n; ++i) {
    if (reqs[i].mode != MSW_MODE_INT8_CONT_BATCHING) throw ConfigErr("run_batch: mode must be int8_continuous_batching");
    check_request(e, reqs[i], 1);
  }
  Scratch& s = e->sc;
  const int hstride = e->cfg.max_seq_len;  // device history ints per batch row
  const int V = m.c.vocab;
  const bool graphs = e->cfg.use_graphs != 0;
  struct Live {
    int req;
    int row;
    int generated;
    int last_tok;
    SeqBlocks sb;
    double t_admit;
  };
  // the step graphs of every live-batch size are captured once per engine,
  // before its first cohort (as serving engines capture their batch-size
  // buckets at start-up): a ragged cohort shrinks through many sizes, and a
  // capture + instantiate inside the step loop costs milliseconds of host time
  if (graphs)
    for (int T = 1; T <= maxb; ++T) cb_graph(e, m, T);
  std::vector<Live> live;
  std::vector<int> free_rows;
  for (int r = maxb - 1; r >= 0; --r) free_rows.push_back(r);
  int next_req = 0;
  auto retire = [&](Live& L) {
    msw_result& rr = res[L.req];
    if (L.generated > 1)
      MSW_CUDA(cudaMemcpy(rr.out_ids + 1, s.cb_hist + size_t(L.row) * hstride + 1,
                          sizeof(int) * (L.generated - 1), cudaMemcpyDeviceToHost));
    release_sequence(m, L.sb);
    free_rows.push_back(L.row);
    rr.n_out = L.generated;
    rr.total_ms = now_ms() - L.t_admit;
    rr.decode_ms = rr.total_ms - rr.prefill_ms;
  };
  try {
    while (next_req < n || !live.empty()) {
      // admission: map every request that fits, then prefill them packed
      std::vector<Live> adm;
      while (next_req < n && !free_rows.empty()) {
        const msw_request& r = reqs[next_req];
        // KV admission: a sequence is admitted only when the pool holds all of
        // its blocks (prompt + max_new); otherwise wait for live sequences to
        // retire. Only a request that cannot fit an empty pool is an error.
        const int need = (r.prompt_len + r.max_new_tokens + kKvBlock - 1) / kKvBlock;
        if (need > m.pool.available()) {
          if (live.empty() && adm.empty())
            throw DataErr("request needs more KV blocks than the pool holds");
          break;
        }
        Live L;
        L.req = next_req;
        L.row = free_rows.back();
        L.generated = 0;
        L.t_admit = now_ms();
        try {
          L.sb = map_sequence(m, L.row, r.prompt_len + r.max_new_tokens, r.prompt_ids,
                              r.prompt_len, false, fmt, e->st, s.stage);
        } catch (...) {
          for (Live& A : adm) release_sequence(m, A.sb);
          throw;
        }
        free_rows.pop_back();
        adm.push_back(std::move(L));
        ++next_req;
      }
      if (!adm.empty()) {
        const double tp = now_ms();
        std::vector<PackSeq> ps;
        std::vector<float*> lg;
        std::vector<int> first(adm.size());
        for (const Live& L : adm) {
          const msw_request& r = reqs[L.req];
          ps.push_back({L.row, r.prompt_ids, r.prompt_len, &L.sb});
          lg.push_back(res[L.req].logits);
        }
        try {
          prefill_packed(e, m, fmt, ps, first.data(), lg.data());
        } catch (...) {
          for (Live& L : adm) release_sequence(m, L.sb);
          throw;
        }
        const double tdone = now_ms();
        for (size_t j = 0; j < adm.size(); ++j) {
          Live& L = adm[j];
          msw_result& rr = res[L.req];
          L.last_tok = first[j];
          rr.out_ids[0] = L.last_tok;
          L.generated = 1;
          rr.prefill_ms = tdone - tp;
          if (L.generated >= reqs[L.req].max_new_tokens) {
            retire(L);
          } else {
            live.push_back(std::move(L));
          }
        }
      }
      if (live.empty()) continue;
      // load the device step state of the live set (after any admission the
      // packed prefill has reused these scratch arrays)
      const int T = int(live.size());
      int steps = 1 << 30;
      for (int i = 0; i < T; ++i) {
        const Live& L = live[i];
        const msw_request& r = reqs[L.req];
        const int p = r.prompt_len + L.generated - 1;
        s.stage[i] = L.last_tok;
        s.stage[T + i] = p;
        s.stage[2 * T + i] = L.sb.blocks[p / kKvBlock] * kKvBlock + p % kKvBlock;
        s.stage[3 * T + i] = L.row;
        s.stage[4 * T + i] = L.row * hstride - r.prompt_len + 1;  // hist index of the output = hbase + p
        steps = std::min(steps, r.max_new_tokens - L.generated);
      }
      MSW_CUDA(cudaMemcpyAsync(s.tok, s.stage, sizeof(int) * T, cudaMemcpyHostToDevice, e->st));
      MSW_CUDA(cudaMemcpyAsync(s.pos, s.stage + T, sizeof(int) * T, cudaMemcpyHostToDevice, e->st));
      MSW_CUDA(cudaMemcpyAsync(s.slot, s.stage + 2 * T, sizeof(int) * T, cudaMemcpyHostToDevice, e->st));
      MSW_CUDA(cudaMemcpyAsync(s.seq_of, s.stage + 3 * T, sizeof(int) * T, cudaMemcpyHostToDevice, e->st));
      MSW_CUDA(cudaMemcpyAsync(s.cb_hbase, s.stage + 4 * T, sizeof(int) * T, cudaMemcpyHostToDevice, e->st));
      // steps until the next retirement, back to back on the device
      for (int k = 0; k < steps; ++k) {
        cb_step(e, m, T, graphs);
        for (int i = 0; i < T; ++i) {
          msw_result& rr = res[live[i].req];
          if (rr.logits) copy_logits_row(e, rr.logits + size_t(live[i].generated + k) * V, i);
        }
      }
      MSW_CUDA(cudaMemcpyAsync(s.stage + 5 * T, s.tok, sizeof(int) * T, cudaMemcpyDeviceToHost, e->st));
      MSW_CUDA(cudaStreamSynchronize(e->st));
      std::vector<Live> still;
      for (int i = 0; i < T; ++i) {
        Live& L = live[i];
        L.generated += steps;
        L.last_tok = s.stage[5 * T + i];
        if (L.generated >= reqs[L.req].max_new_tokens) {
          retire(L);
        } else {
          still.push_back(std::move(L));
        }
      }
      live.swap(still);
    }
  } catch (...) {
    for (Live& L : live) release_sequence(m, L.sb);
    throw;
  }
}

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const ConfigErr& ex) {
    g_last_error = ex.what();
    return 2;
  } catch (const DataErr& ex) {
    g_last_error = ex.what();
    return 3;
  } catch (const std::exception& ex) {
    g_last_error = ex.what();
    return 1;
  } catch (...) {
    g_last_error = "unknown error";
    return 1;
  }
}

}  // namespace
}  // namespace msw

using namespace msw;

extern "C" {

int msw_engine_create(int device, const msw_engine_cfg* cfg, msw_engine** out) {
  return guarded([&] {
    if (!cfg || !out) throw ConfigErr("NULL argument");
    *out = nullptr;
    if (cfg->kv_blocks < 4 || cfg->max_seq_len < 16 || cfg->max_batch < 1)
      throw ConfigErr("kv_blocks/max_seq_len/max_batch too small");
    if (cfg->has_draft && cfg->draft.vocab != cfg->target.vocab)
      throw ConfigErr("draft and target must share the vocabulary");
    MSW_CUDA(cudaSetDevice(device));
    auto e = std::make_unique<msw_engine>();
    e->device = device;
    e->cfg = *cfg;
    if (e->cfg.max_batch > kMaxLogitRows) e->cfg.max_batch = kMaxLogitRows;
    MSW_CUDA(cudaStreamCreateWithFlags(&e->st, cudaStreamNonBlocking));
    for (auto& ev : e->ev) MSW_CUDA(cudaEventCreate(&ev));
    std::vector<int> pred;
    std::vector<uint8_t> agree;
    build_successor(e->cfg, cfg->target.vocab, pred, agree);
    build_model(e->target, cfg->target, false, e->cfg, pred, agree, e->st);
    if (cfg->has_draft) build_model(e->draft, cfg->draft, true, e->cfg, pred, agree, e->st);
    alloc_scratch(e.get());
    MSW_CUDA(cudaStreamSynchronize(e->st));
    *out = e.release();
  });
}

int msw_engine_run(msw_engine* e, const msw_request* req, msw_result* res) {
  return guarded([&] {
    if (!e || !req || !res || !res->out_ids) throw ConfigErr("NULL argument");
    MSW_CUDA(cudaSetDevice(e->device));
    res->n_out = 0;
    res->spec_rounds = res->spec_proposed = res->spec_accepted = 0;
    res->prefix_hit_tokens = 0;
    const long long before = e->launches;
    if (req->mode == MSW_MODE_SPECULATIVE) {
      run_spec(e, *req, *res);
    } else if (req->mode == MSW_MODE_INT8_CONT_BATCHING) {
      run_cb(e, req, 1, res);
    } else if (req->mode == MSW_MODE_KV_COMPRESSION) {
      run_kvc(e, *req, *res);
    } else {
      run_single(e, *req, *res);
    }
    res->kernel_launches = int(e->launches - before);
  });
}

int msw_engine_run_batch(msw_engine* e, const msw_request* reqs, int32_t n, msw_result* res) {
  return guarded([&] {
    if (!e || !reqs || !res || n < 1) throw ConfigErr("bad arguments");
    MSW_CUDA(cudaSetDevice(e->device));
    for (int i = 0; i < n; ++i) {
      if (!res[i].out_ids) throw ConfigErr("NULL out_ids");
      res[i].n_out = 0;
      res[i].spec_rounds = res[i].spec_proposed = res[i].spec_accepted = 0;
      res[i].prefix_hit_tokens = 0;
    }
    const long long before = e->launches;
    run_cb(e, reqs, n, res);
    for (int i = 0; i < n; ++i) res[i].kernel_launches = int(e->launches - before);
  });
}

void msw_engine_destroy(msw_engine* e) {
  if (!e) return;
  cudaSetDevice(e->device);
  cudaStreamSynchronize(e->st);
  if (e->spec_graph) cudaGraphExecDestroy(e->spec_graph);
  for (auto& kv : e->cb_graphs) cudaGraphExecDestroy(kv.second.first);
  free_model(e->target);
  free_model(e->draft);
  for (void* p : e->owned) cudaFree(p);
  if (e->sc.stage) cudaFreeHost(e->sc.stage);
  for (auto& ev : e->ev)
    if (ev) cudaEventDestroy(ev);
  if (e->st) cudaStreamDestroy(e->st);
  delete e;
}

const char* msw_last_error(void) { return g_last_error.c_str(); }

int msw_engine_weight_bytes(msw_engine* e, int32_t mode, int64_t* bytes) {
  return guarded([&] {
    if (!e || !bytes) throw ConfigErr("NULL argument");
    const int fmt = fmt_of_mode(mode);
    if (!e->target.fmt_on[fmt]) throw ConfigErr("mode not resident");
    *bytes = int64_t(e->target.weight_bytes(fmt));
  });
}

int msw_engine_memory_bytes(msw_engine* e, int32_t mode, int32_t tokens, int64_t* bytes) {
  return guarded([&] {
    if (!e || !bytes) throw ConfigErr("NULL argument");
    if (tokens < 0) throw DataErr("tokens must be >= 0");
    const int fmt = fmt_of_mode(mode);
    if (!e->target.fmt_on[fmt]) throw ConfigErr("mode not resident");
    auto kv_pos = [](const Model& m) {
      return int64_t(2) * m.c.n_layers * m.c.n_kv_heads * m.c.head_dim * 2;  // K + V fp16
    };
    // KV-cache compression holds the request's context at one byte per element
    const int64_t kv = mode == MSW_MODE_KV_COMPRESSION ? kv_pos(e->target) / 2 : kv_pos(e->target);
    int64_t b = int64_t(e->target.weight_bytes(fmt)) + int64_t(tokens) * kv;
    if (mode == MSW_MODE_SPECULATIVE) {
      if (!e->cfg.has_draft) throw ConfigErr("speculative decoding needs a draft model");
      b += int64_t(e->draft.weight_bytes(kFP16)) + int64_t(tokens) * kv_pos(e->draft);
    }
    *bytes = b;
  });
}

int msw_fp8_e4m3_roundtrip(const uint16_t* x, int64_t n, uint8_t* q, uint16_t* y, void* stream) {
  return guarded([&] {
    if (n % 2) throw DataErr("msw_fp8_e4m3_roundtrip: n must be even");
    launch_fp8_roundtrip(reinterpret_cast<const half*>(x), n, q, reinterpret_cast<half*>(y),
                         static_cast<cudaStream_t>(stream));
  });
}

int msw_engine_reset_prefix_cache(msw_engine* e) {
  return guarded([&] {
    if (!e) throw ConfigErr("NULL argument");
    e->target.pool.drop_cache();
  });
}

}  // extern "C"

namespace {
// Test entry shared by msw_linear and msw_linear_i8_raw: the production
// dispatch (decode GEMV on the tile-fragment layout for t <= 6, prep_act +
// tcgen05 GEMM otherwise) on row-major weights, with temporary buffers.
void run_linear_entry(int32_t wtype, const void* w, const void* scales, int32_t n, int32_t k,
                      const float* x, int32_t t, float* y, int epi, cudaStream_t st,
                      const uint8_t* zeros = nullptr) {
  LinearW W;
  W.fmt = wtype;
  W.n = n;
  W.k = k;
  W.w = w;
  W.s = scales;
  W.z = zeros;
  if (t <= kGemvMaxTokens) {
    // weights arrive row-major; build the decode layout first
    uint8_t* tf = dalloc<uint8_t>(tf_bytes(wtype, n, k));
    launch_repack_tf(wtype, w, n, k, tf, st);
    // the GEMV's producer streams weights BEFORE griddepcontrol.wait (PDL), so
    // freshly repacked weights must be complete before it launches
    MSW_CUDA(cudaStreamSynchronize(st));
    W.w_tf = tf;
    launch_gemv(W, kProPlain, epi, x, t, nullptr, 1e-5f, y, st);
    MSW_CUDA(cudaStreamSynchronize(st));
    cudaFree(tf);
  } else {
    half* xh = dalloc<half>(size_t(t) * k);
    int8_t* xq = dalloc<int8_t>(size_t(t) * k);
    float* xs = dalloc<float>(t);
    launch_prep_act(wtype, x, t, k, nullptr, 1e-5f, xh, xq, xs, st);
    launch_gemm(W, epi, xh, xq, xs, t, y, st);
    MSW_CUDA(cudaStreamSynchronize(st));
    cudaFree(xh);
    cudaFree(xq);
    cudaFree(xs);
  }
}
}  // namespace

extern "C" {

int msw_linear(int32_t wtype, const void* w, const void* scales, int32_t n, int32_t k,
               const float* x, int32_t t, float* y, void* stream) {
  return guarded([&] {
    run_linear_entry(wtype, w, scales, n, k, x, t, y, kEpiStore, static_cast<cudaStream_t>(stream));
  });
}

int msw_linear_i8_raw(const int8_t* w, int32_t n, int32_t k, const float* x, int32_t t,
                      int32_t* acc, void* stream) {
  return guarded([&] {
    // the kernels stage / read the per-row scales in every epilogue (the raw
    // one ignores them): give them a valid array
    float* ones = dalloc<float>(size_t(n));
    std::vector<float> h(size_t(n), 1.0f);
    try {
      MSW_CUDA(cudaMemcpy(ones, h.data(), sizeof(float) * h.size(), cudaMemcpyHostToDevice));
      run_linear_entry(kINT8, w, ones, n, k, x, t, reinterpret_cast<float*>(acc), kEpiRaw,
                       static_cast<cudaStream_t>(stream));
    } catch (...) {
      cudaFree(ones);
      throw;
    }
    cudaFree(ones);
  });
}

int msw_linear_decode(int32_t wtype, const void* w_tf, const void* scales, int32_t n, int32_t k,
                      const float* x, int32_t t, float* y, void* stream) {
  return guarded([&] {
    LinearW W;
    W.fmt = wtype;
    W.n = n;
    W.k = k;
    W.s = scales;
    W.w_tf = w_tf;
    launch_gemv(W, kProPlain, kEpiStore, x, t, nullptr, 1e-5f, y, static_cast<cudaStream_t>(stream));
  });
}

int msw_repack_decode(int32_t wtype, const void* w, int32_t n, int32_t k, void* out, void* stream) {
  return guarded([&] { launch_repack_tf(wtype, w, n, k, out, static_cast<cudaStream_t>(stream)); });
}

int msw_gemv_i8_acc(const int8_t* w, const int8_t* x, int32_t n, int32_t k, int32_t* acc,
                    void* stream) {
  return guarded([&] { launch_gemv_i8_acc(w, x, n, k, acc, static_cast<cudaStream_t>(stream)); });
}

int msw_fill_fp16(uint16_t* dst, int64_t rows, int64_t cols, uint64_t seed, uint64_t tensor_id,
                  int32_t scale_log2, void* stream) {
  return guarded([&] {
    launch_fill_fp16(reinterpret_cast<half*>(dst), rows, cols, seed, tensor_id, scale_log2,
                     static_cast<cudaStream_t>(stream));
  });
}

int msw_quant_int8_rows(const uint16_t* w, int32_t n, int32_t k, int8_t* q, float* scales,
                        void* stream) {
  return guarded([&] {
    launch_quant_int8(reinterpret_cast<const half*>(w), n, k, q, scales,
                      static_cast<cudaStream_t>(stream));
  });
}

int msw_linear_awq4(const void* w, const void* scales, const uint8_t* zeros, int32_t n, int32_t k,
                    const float* x, int32_t t, float* y, void* stream) {
  return guarded([&] {
    if (!zeros) throw ConfigErr("msw_linear_awq4: zero points required");
    run_linear_entry(kW4, w, scales, n, k, x, t, y, kEpiStore, static_cast<cudaStream_t>(stream),
                     zeros);
  });
}

int msw_quant_awq4_rows(const uint16_t* w, int32_t n, int32_t k, uint8_t* packed, uint16_t* scales,
                        uint8_t* zeros, void* stream) {
  return guarded([&] {
    launch_quant_awq4(reinterpret_cast<const half*>(w), n, k, reinterpret_cast<uint32_t*>(packed),
                      reinterpret_cast<half*>(scales), zeros, static_cast<cudaStream_t>(stream));
  });
}

int msw_quant_w4_rows(const uint16_t* w, int32_t n, int32_t k, uint8_t* packed, uint16_t* scales,
                      void* stream) {
  return guarded([&] {
    launch_quant_w4(reinterpret_cast<const half*>(w), n, k, reinterpret_cast<uint32_t*>(packed),
                    reinterpret_cast<half*>(scales), static_cast<cudaStream_t>(stream));
  });
}

int msw_attention_decode(const float* qkv, const void* rope, int32_t T, const int32_t* pos,
                         const int32_t* slot, const int32_t* seq_of, const int32_t* block_table,
                         int32_t max_blocks, uint16_t* kc, uint16_t* vc, int32_t n_heads,
                         int32_t n_kv_heads, int32_t head_dim, int32_t nsplit, float* o,
                         void* stream) {
  return guarded([&] {
    if (T < 1 || nsplit < 1 || nsplit > 64 || n_kv_heads < 1 || n_heads % n_kv_heads)
      throw ConfigErr("msw_attention_decode: bad shape");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const size_t parts = size_t(T) * n_heads * nsplit;
    float* part_o = dalloc<float>(parts * head_dim);
    float* part_ml = dalloc<float>(parts * 2);
    int* cnt = dalloc<int>(size_t(T) * n_kv_heads);
    try {
      MSW_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int) * size_t(T) * n_kv_heads, st));
      const AttnShape a{n_heads, n_kv_heads, head_dim, max_blocks};
      launch_attention_decode(qkv, static_cast<const float2*>(rope), T, pos, slot, seq_of,
                              block_table, reinterpret_cast<half*>(kc), reinterpret_cast<half*>(vc),
                              a, nsplit, part_o, part_ml, cnt, o, st);
      MSW_CUDA(cudaStreamSynchronize(st));
    } catch (...) {
      cudaFree(part_o);
      cudaFree(part_ml);
      cudaFree(cnt);
      throw;
    }
    cudaFree(part_o);
    cudaFree(part_ml);
    cudaFree(cnt);
  });
}

int msw_device_sync(void) {
  return guarded([&] { MSW_CUDA(cudaDeviceSynchronize()); });
}

int msw_device_pci_bus_id(int32_t device, char* buf, int32_t len) {
  return guarded([&] {
    if (!buf || len < 13) throw ConfigErr("msw_device_pci_bus_id: buffer too small");
    MSW_CUDA(cudaDeviceGetPCIBusId(buf, len, device));
  });
}

}  // extern "C"
