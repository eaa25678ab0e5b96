// K1 — paged KV pool: deterministic host block allocator, device block table,
// coalesced 16-byte commit / copy kernels, and the fused RoPE + commit epilogue
// of the QKV projection.
//
// Replaces the reference's integer KV accounting (`engine.py:259,285,313,335,366`),
// the evict-to-prefix rule (`engine.py:380-384`) and slot release
// (`engine.py:385,397`). Allocation policy: block size 16, LIFO
// free list initialised so that pops yield 0,1,2,...; reserve grows a slot to
// ceil(len/16) blocks; truncate frees from the tail, so the next pop reuses the
// lowest freed logical block first. oracle/kv_alloc.py restates this policy.
#include <cstdarg>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include "../../include/stb200.h"
#include "common.cuh"
#include "pool.cuh"
#include "rope.cuh"

namespace stb {

static thread_local std::string g_err;
static int64_t g_launches = 0;

void set_error(const std::string& msg) { g_err = msg; }
int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}
void count_launch(int n) { __atomic_fetch_add(&g_launches, (int64_t)n, __ATOMIC_RELAXED); }
bool pdl_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("STB200_PDL");
    on = (e && e[0] == '0') ? 0 : 1;
  }
  return on == 1;
}

}  // namespace stb

using namespace stb;


static void table_set(stb_kv_pool* p, int slot, int idx, int32_t value) {
  int64_t flat = (int64_t)slot * p->max_bps + idx;
  p->table[flat] = value;
  p->updates.push_back((int32_t)flat);
  p->updates.push_back(value);
}

__global__ void apply_updates_kernel(const int32_t* __restrict__ upd, int n, int32_t* __restrict__ table) {
  pdl_wait();
  pdl_launch();
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) table[upd[2 * i]] = upd[2 * i + 1];
}

// 16-byte vector scatter of K and V rows into their pages.
// thread -> (token, which of K/V, 16B chunk of the n_kv*d_head row)
__global__ void kv_commit_kernel(const __nv_bfloat16* __restrict__ k, const __nv_bfloat16* __restrict__ v, int64_t ld,
                                 const int32_t* __restrict__ slot_of, const int32_t* __restrict__ pos_of, int n,
                                 const int32_t* __restrict__ table, int max_bps, __nv_bfloat16* __restrict__ kpages,
                                 __nv_bfloat16* __restrict__ vpages, int n_kv, int d_head) {
  pdl_wait();
  pdl_launch();
  const int chunks = n_kv * d_head / 8;  // 8 bf16 per 16 bytes
  int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t total = (int64_t)n * 2 * chunks;
  if (gid >= total) return;
  int c = gid % chunks;
  int which = (gid / chunks) % 2;
  int t = gid / (2 * chunks);
  int pos = pos_of[t];
  int blk = table[(int64_t)slot_of[t] * max_bps + (pos >> 4)];
  int h = (c * 8) / d_head, dd = (c * 8) % d_head;
  int64_t dst = (((int64_t)blk * n_kv + h) * 16 + (pos & 15)) * d_head + kv_phys_chunk(pos & 15, dd / 8) * 8;
  const __nv_bfloat16* src = (which ? v : k) + (int64_t)t * ld + c * 8;
  __nv_bfloat16* pages = which ? vpages : kpages;
  *reinterpret_cast<uint4*>(pages + dst) = *reinterpret_cast<const uint4*>(src);
}

__global__ void kv_copy_blocks_kernel(__nv_bfloat16* __restrict__ pages, const int32_t* __restrict__ src,
                                      const int32_t* __restrict__ dst, int n, int64_t block_elems, int64_t half_elems,
                                      int layers) {
  pdl_wait();
  pdl_launch();
  // grid.y = block pair, grid.z = layer*2 + {K,V}; threads stride the block in 16B vectors
  int pair = blockIdx.y;
  int lz = blockIdx.z;
  int64_t base = (int64_t)lz * half_elems;
  const uint4* s = reinterpret_cast<const uint4*>(pages + base + (int64_t)src[pair] * block_elems);
  uint4* d = reinterpret_cast<uint4*>(pages + base + (int64_t)dst[pair] * block_elems);
  int64_t nvec = block_elems / 8;
  for (int64_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nvec; i += (int64_t)gridDim.x * blockDim.x) d[i] = s[i];
}

// Fused QKV epilogue: (optional per-head RMSNorm of q and k — Qwen3 qk-norm), rotate q
// and k (rotate-half RoPE), write q as bf16, commit k and v into the pool pages.
// thread -> (token, head among n_q + 2*n_kv, group of 8 rotation pairs); every store is 16
// bytes (rope.cuh).
__global__ void qkv_rope_commit_kernel(float* __restrict__ qkv, __nv_bfloat16* __restrict__ q_out,
                                       const int32_t* __restrict__ slot_of, const int32_t* __restrict__ pos_of, int n,
                                       int n_q, int n_kv, int d_head, const float* __restrict__ inv_freq,
                                       const int32_t* __restrict__ table, int max_bps,
                                       __nv_bfloat16* __restrict__ kpages, __nv_bfloat16* __restrict__ vpages,
                                       int clear_rows, const __nv_bfloat16* __restrict__ q_norm,
                                       const __nv_bfloat16* __restrict__ k_norm, float eps,
                                       const float* __restrict__ bias, float rope_scale) {
  pdl_wait();
  pdl_launch();
  rope_commit_elem((int64_t)blockIdx.x * blockDim.x + threadIdx.x, qkv, q_out, slot_of, pos_of, n, n_q, n_kv, d_head,
                   inv_freq, table, max_bps, kpages, vpages, clear_rows, q_norm, k_norm, eps, bias, rope_scale);
}

// ------------------------------------------------------------------- C ABI
// inverse frequencies are a pure function of (theta, d_head): one cached device table per pair
const float* stb_rope_inv_freq(float rope_theta, int d_head) {
  static std::mutex mu;
  static std::vector<std::pair<std::pair<float, int>, float*>> cache;
  std::lock_guard<std::mutex> g(mu);
  for (auto& e : cache)
    if (e.first.first == rope_theta && e.first.second == d_head) return e.second;
  const int half = d_head / 2;
  std::vector<float> h(half);
  for (int i = 0; i < half; ++i) h[i] = (float)(1.0 / pow((double)rope_theta, (2.0 * i) / d_head));
  float* inv = nullptr;
  if (cudaMalloc(&inv, half * sizeof(float)) != cudaSuccess) return nullptr;
  cudaMemcpy(inv, h.data(), half * sizeof(float), cudaMemcpyHostToDevice);
  cache.push_back({{rope_theta, d_head}, inv});
  return inv;
}

extern "C" {

const char* stb_last_error(void) { return g_err.c_str(); }
int stb_version(void) { return 1; }
int64_t stb_launch_count(void) { return __atomic_load_n(&g_launches, __ATOMIC_RELAXED); }

int stb_kv_pool_create(int device, int layers, int n_kv, int d_head, int block_size, int num_blocks, int max_slots,
                       int max_blocks_per_slot, stb_kv_pool** out) {
  if (!out || layers < 1 || n_kv < 1 || num_blocks < 1 || max_slots < 1 || max_blocks_per_slot < 1)
    return fail(STB_EINVAL, "kv_pool_create: bad geometry");
  if (block_size != 16) return fail(STB_EINVAL, "kv_pool_create: block_size must be 16");
  if (d_head % 8 != 0 || d_head > 256) return fail(STB_EINVAL, "kv_pool_create: d_head must be a multiple of 8 <= 256");
  if (cudaSetDevice(device) != cudaSuccess) return fail(STB_ECUDA, "kv_pool_create: cudaSetDevice(%d)", device);
  auto* p = new stb_kv_pool();
  p->device = device;
  p->layers = layers;
  p->n_kv = n_kv;
  p->d_head = d_head;
  p->bs = block_size;
  p->num_blocks = num_blocks;
  p->max_slots = max_slots;
  p->max_bps = max_blocks_per_slot;
  p->block_elems = (int64_t)n_kv * block_size * d_head;
  p->half_elems = (int64_t)num_blocks * p->block_elems;
  size_t bytes = (size_t)layers * 2 * p->half_elems * sizeof(__nv_bfloat16);
  if (cudaMalloc(&p->pages, bytes) != cudaSuccess) {
    delete p;
    cudaGetLastError();
    return fail(STB_ENOMEM, "kv_pool_create: cannot allocate %zu bytes of pages", bytes);
  }
  // zeroed once so rows never written (page tails) are finite for masked P*V
  cudaMemset(p->pages, 0, bytes);
  size_t tbytes = (size_t)max_slots * max_blocks_per_slot * sizeof(int32_t);
  if (cudaMalloc(&p->dev_table, tbytes) != cudaSuccess || cudaMemset(p->dev_table, 0, tbytes) != cudaSuccess) {
    cudaFree(p->pages);
    delete p;
    cudaGetLastError();
    return fail(STB_ENOMEM, "kv_pool_create: cannot allocate block table");
  }
  for (int b = num_blocks - 1; b >= 0; --b) p->free_list.push_back(b);
  p->blocks.resize(max_slots);
  p->len.assign(max_slots, 0);
  p->table.assign((size_t)max_slots * max_blocks_per_slot, 0);
  for (int i = 0; i < 2; ++i) cudaEventCreateWithFlags(&p->done[i], cudaEventDisableTiming);
  *out = p;
  return STB_OK;
}

int stb_kv_pool_destroy(stb_kv_pool* p) {
  if (!p) return STB_OK;
  cudaDeviceSynchronize();
  cudaFree(p->pages);
  cudaFree(p->dev_table);
  for (int i = 0; i < 2; ++i) {
    if (p->staging[i]) cudaFreeHost(p->staging[i]);
    if (p->dev_updates[i]) cudaFree(p->dev_updates[i]);
    if (p->done[i]) cudaEventDestroy(p->done[i]);
  }
  delete p;
  return STB_OK;
}

static int check_slot(const stb_kv_pool* p, int slot) {
  if (!p) return fail(STB_EINVAL, "null pool");
  if (slot < 0 || slot >= p->max_slots) return fail(STB_EINVAL, "slot %d out of range [0,%d)", slot, p->max_slots);
  return STB_OK;
}

int stb_kv_reserve(stb_kv_pool* p, int slot, int new_len) {
  if (int rc = check_slot(p, slot)) return rc;
  if (new_len < 0) return fail(STB_EINVAL, "reserve: negative length");
  int need = (new_len + p->bs - 1) / p->bs;
  if (need > p->max_bps) return fail(STB_ECAPACITY, "reserve: %d blocks exceed the %d-block row", need, p->max_bps);
  auto& bl = p->blocks[slot];
  int extra = need - (int)bl.size();
  if (extra > (int)p->free_list.size())
    return fail(STB_ECAPACITY, "reserve: need %d free blocks, %zu left", extra, p->free_list.size());
  while ((int)bl.size() < need) {
    int32_t b = p->free_list.back();
    p->free_list.pop_back();
    table_set(p, slot, (int)bl.size(), b);
    bl.push_back(b);
  }
  if (new_len > p->len[slot]) p->len[slot] = new_len;
  return STB_OK;
}

int stb_kv_truncate(stb_kv_pool* p, int slot, int new_len) {
  if (int rc = check_slot(p, slot)) return rc;
  if (new_len < 0) return fail(STB_EINVAL, "truncate: negative length");
  int keep = (new_len + p->bs - 1) / p->bs;
  auto& bl = p->blocks[slot];
  while ((int)bl.size() > keep) {
    p->free_list.push_back(bl.back());
    bl.pop_back();
  }
  if (new_len < p->len[slot]) p->len[slot] = new_len;
  return STB_OK;
}

int stb_kv_release(stb_kv_pool* p, int slot) {
  int rc = stb_kv_truncate(p, slot, 0);
  if (rc == STB_OK) p->len[slot] = 0;
  return rc;
}

int stb_pool_geometry(const stb_kv_pool* p, int* n_kv, int* d_head) {
  if (!p) return fail(STB_EINVAL, "null pool");
  *n_kv = p->n_kv;
  *d_head = p->d_head;
  return STB_OK;
}

int stb_kv_free_blocks(const stb_kv_pool* p) { return p ? (int)p->free_list.size() : fail(STB_EINVAL, "null pool"); }

int stb_kv_slot_len(const stb_kv_pool* p, int slot) {
  if (int rc = check_slot(p, slot)) return rc;
  return p->len[slot];
}

int stb_kv_slot_blocks(const stb_kv_pool* p, int slot, int32_t* out, int cap) {
  if (int rc = check_slot(p, slot)) return rc;
  const auto& bl = p->blocks[slot];
  int n = (int)bl.size();
  if (out) memcpy(out, bl.data(), sizeof(int32_t) * (size_t)(n < cap ? n : cap));
  return n;
}

int stb_kv_sync(stb_kv_pool* p, void* stream) {
  if (!p) return fail(STB_EINVAL, "null pool");
  int64_t n = (int64_t)p->updates.size();
  if (n == 0) return STB_OK;
  cudaStream_t st = (cudaStream_t)stream;
  int i = p->flip;
  p->flip ^= 1;
  cudaEventSynchronize(p->done[i]);  // the copy that last used this staging buffer has landed
  if (n > p->cap[i]) {
    if (p->staging[i]) cudaFreeHost(p->staging[i]);
    if (p->dev_updates[i]) cudaFree(p->dev_updates[i]);
    int64_t c = n * 2 > 4096 ? n * 2 : 4096;
    if (cudaMallocHost(&p->staging[i], c * sizeof(int32_t)) != cudaSuccess ||
        cudaMalloc(&p->dev_updates[i], c * sizeof(int32_t)) != cudaSuccess)
      return fail(STB_ENOMEM, "kv_sync: staging allocation failed");
    p->cap[i] = c;
  }
  memcpy(p->staging[i], p->updates.data(), n * sizeof(int32_t));
  p->updates.clear();
  cudaMemcpyAsync(p->dev_updates[i], p->staging[i], n * sizeof(int32_t), cudaMemcpyHostToDevice, st);
  int pairs = (int)(n / 2);
  launch_k(apply_updates_kernel, dim3((pairs + 255) / 256), dim3(256), 0, st, p->dev_updates[i], pairs, p->dev_table);
  cudaEventRecord(p->done[i], st);
  STB_CHECK_LAUNCH("kv_sync");
  return STB_OK;
}

int stb_kv_layer_ptrs(const stb_kv_pool* p, int layer, void** k_pages, void** v_pages) {
  if (!p || layer < 0 || layer >= p->layers) return fail(STB_EINVAL, "kv_layer_ptrs: bad layer");
  __nv_bfloat16* base = p->pages + (int64_t)layer * 2 * p->half_elems;
  if (k_pages) *k_pages = base;
  if (v_pages) *v_pages = base + p->half_elems;
  return STB_OK;
}

int stb_kv_block_table(const stb_kv_pool* p, int32_t** dev_table, int* row_stride) {
  if (!p) return fail(STB_EINVAL, "null pool");
  if (dev_table) *dev_table = p->dev_table;
  if (row_stride) *row_stride = p->max_bps;
  return STB_OK;
}

int stb_kv_commit(stb_kv_pool* p, int layer, const void* k, const void* v, int64_t ld, const int32_t* slot_of,
                  const int32_t* pos_of, int n, void* stream) {
  if (!p || layer < 0 || layer >= p->layers) return fail(STB_EINVAL, "kv_commit: bad layer");
  if (n <= 0) return STB_OK;
  if (ld % 8 != 0) return fail(STB_EINVAL, "kv_commit: row stride must be a multiple of 8 elements");
  void *kp, *vp;
  stb_kv_layer_ptrs(p, layer, &kp, &vp);
  int64_t total = (int64_t)n * 2 * (p->n_kv * p->d_head / 8);
  int threads = 256;
  launch_k(kv_commit_kernel, dim3((unsigned)((total + threads - 1) / threads)), dim3(threads), 0, (cudaStream_t)stream, 
      (const __nv_bfloat16*)k, (const __nv_bfloat16*)v, ld, slot_of, pos_of, n, p->dev_table, p->max_bps,
      (__nv_bfloat16*)kp, (__nv_bfloat16*)vp, p->n_kv, p->d_head);
  STB_CHECK_LAUNCH("kv_commit");
  return STB_OK;
}

int stb_kv_copy_blocks(stb_kv_pool* p, const int32_t* src, const int32_t* dst, int n, void* stream) {
  if (!p) return fail(STB_EINVAL, "null pool");
  if (n <= 0) return STB_OK;
  if (n > 65535) return fail(STB_EINVAL, "kv_copy_blocks: at most 65535 pairs per call");
  dim3 grid(4, n, p->layers * 2);
  launch_k(kv_copy_blocks_kernel, dim3(grid), dim3(256), 0, (cudaStream_t)stream, p->pages, src, dst, n, p->block_elems, p->half_elems,
                                                                 p->layers);
  STB_CHECK_LAUNCH("kv_copy_blocks");
  return STB_OK;
}

static int rope_commit(stb_kv_pool* p, int layer, float* qkv, void* q_out, const int32_t* slot_of,
                       const int32_t* pos_of, int n, int n_q, float rope_theta, const void* q_norm, const void* k_norm,
                       float eps, int clear_rows, const float* inv_freq, float rope_scale, const float* bias,
                       void* stream) {
  if ((q_norm == nullptr) != (k_norm == nullptr)) return fail(STB_EINVAL, "qkv_rope_commit: q_norm and k_norm go together");
  if (!p || layer < 0 || layer >= p->layers) return fail(STB_EINVAL, "qkv_rope_commit: bad layer");
  if (n <= 0) return STB_OK;
  const float* inv = inv_freq ? inv_freq : stb_rope_inv_freq(rope_theta, p->d_head);
  if (!inv) return fail(STB_ENOMEM, "qkv_rope_commit: inv_freq");
  void *kp, *vp;
  stb_kv_layer_ptrs(p, layer, &kp, &vp);
  if (p->d_head % 16 != 0) return fail(STB_EINVAL, "qkv_rope_commit: d_head must be a multiple of 16");
  int64_t total = (int64_t)n * (n_q + 2 * p->n_kv) * (p->d_head / 16);
  int threads = 256;
  launch_k(qkv_rope_commit_kernel, dim3((unsigned)((total + threads - 1) / threads)), dim3(threads), 0, (cudaStream_t)stream, 
      qkv, (__nv_bfloat16*)q_out, slot_of, pos_of, n, n_q, p->n_kv, p->d_head, inv, p->dev_table, p->max_bps,
      (__nv_bfloat16*)kp, (__nv_bfloat16*)vp, clear_rows, (const __nv_bfloat16*)q_norm,
      (const __nv_bfloat16*)k_norm, eps, bias, rope_scale);
  STB_CHECK_LAUNCH("qkv_rope_commit");
  return STB_OK;
}

int stb_qkv_norm_rope_commit(stb_kv_pool* p, int layer, float* qkv, void* q_out, const int32_t* slot_of,
                             const int32_t* pos_of, int n, int n_q, float rope_theta, const void* q_norm,
                             const void* k_norm, float eps, int clear_rows, void* stream) {
  return rope_commit(p, layer, qkv, q_out, slot_of, pos_of, n, n_q, rope_theta, q_norm, k_norm, eps, clear_rows,
                     nullptr, 1.f, nullptr, stream);
}

int stb_qkv_rope_commit_ex(stb_kv_pool* p, int layer, float* qkv, void* q_out, const int32_t* slot_of,
                           const int32_t* pos_of, int n, int n_q, float rope_theta, const float* inv_freq,
                           float rope_scale, const float* bias, int clear_rows, void* stream) {
  return rope_commit(p, layer, qkv, q_out, slot_of, pos_of, n, n_q, rope_theta, nullptr, nullptr, 0.f, clear_rows,
                     inv_freq, rope_scale, bias, stream);
}

int stb_qkv_rope_commit(stb_kv_pool* p, int layer, float* qkv, void* q_out, const int32_t* slot_of,
                        const int32_t* pos_of, int n, int n_q, float rope_theta, int clear_rows, void* stream) {
  return stb_qkv_norm_rope_commit(p, layer, qkv, q_out, slot_of, pos_of, n, n_q, rope_theta, nullptr, nullptr, 0.f,
                                  clear_rows, stream);
}

}  // extern "C"
