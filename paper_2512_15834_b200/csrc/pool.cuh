// Internal definition of the paged KV pool handle (opaque in include/stb200.h).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

struct stb_kv_pool {
  int device, layers, n_kv, d_head, bs, num_blocks, max_slots, max_bps;
  __nv_bfloat16* pages = nullptr;   // [layers][2][num_blocks][n_kv][bs][d_head]
  int64_t block_elems = 0;          // n_kv * bs * d_head
  int64_t half_elems = 0;           // num_blocks * block_elems (K -> V)
  std::vector<int32_t> free_list;   // stack: back() is the next block handed out
  std::vector<std::vector<int32_t>> blocks;
  std::vector<int> len;             // reserved logical length per slot
  std::vector<int32_t> table;       // host mirror [max_slots][max_bps]
  int32_t* dev_table = nullptr;
  // pending device-table updates: (flat index, value) pairs, double-buffered staging
  std::vector<int32_t> updates;
  int32_t* staging[2] = {nullptr, nullptr};
  int32_t* dev_updates[2] = {nullptr, nullptr};
  int64_t cap[2] = {0, 0};
  cudaEvent_t done[2] = {nullptr, nullptr};
  int flip = 0;
};


// Pages are stored pre-swizzled: within each 128-byte half-row of a [16][d_head] page,
// logical 16-byte chunk c of token row r sits at chunk (c ^ r) & 7. That is exactly the
// layout TMA SWIZZLE_128B / the ldmatrix XOR swizzle produce in shared memory, so a
// page is moved HBM -> smem with plain bulk copies (no per-lane swizzle, no tensor-map
// swizzle) and consumed in place.
__host__ __device__ __forceinline__ int kv_phys_chunk(int row, int c) { return (c & ~7) | ((c ^ row) & 7); }

// RoPE inverse frequencies 1/theta^(2i/d_head) (fp32 from a float64 pow), one cached device
// table per (theta, d_head) — shared by the rope/commit kernel and the fused QKV epilogue
const float* stb_rope_inv_freq(float rope_theta, int d_head);
extern "C" int stb_pool_geometry(const stb_kv_pool* p, int* n_kv, int* d_head);
extern "C" int stb_kv_layer_ptrs(const stb_kv_pool* pool, int layer, void** k_pages, void** v_pages);
// K2 tensor-core path (attn_prefill_tc.cu), dispatched from stb_attn_prefill
// active_hint: (query-tile pair, kv head, run) units that hold queries (0: assume the full grid)
int stb_attn_prefill_tc(const stb_kv_pool* pool, int layer, const void* q, void* out, const int32_t* slots,
                        const int32_t* q_start, const int32_t* ctx, int S, int T, int n_q, float scale, int max_q,
                        int active_hint, int window, const float* sinks, void* stream);
