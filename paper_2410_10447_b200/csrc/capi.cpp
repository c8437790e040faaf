// capi.cpp — host implementation of the C-ABI in include/mdr.h.
//
// Validation mirrors the reference's exceptions (thrown before any work):
//   BlockConfig simblock.cpp:10-19, reduce4 reduce.cpp:81-83,
//   baseline_block_reduce reduce.cpp:138-147, reduce7 reduce.cpp:192-196,
//   lga_run docking.cpp:395-397, adadelta_step docking.cpp:285-293.
// SyncStats are the reference's model counters for the chosen method
// (reduce.cpp:86-110, 149-162; docking.cpp:215-220) so the drop-in API
// returns the values reference callers expect; real device behaviour is
// measured by ncu (profiles/).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <limits>
#include <string>
#include <vector>

#include <chrono>
#include <cstdlib>

#include "dock_launch.h"
#include "mdr.h"
#include "mdr_shared.h"

using namespace mdr;

struct mdr_dev_instance;
struct mdr_lga_batch;

// One cached docking setup for the host-buffer lga_run path: the device
// ligand and the instantiated CUDA graph are reused while the shapes,
// settings and method match (contents are re-uploaded every call).
struct LgaCache {
  int na = -1, ns = -1, nr = -1, method = -1, pair = -1, accum = -1, wpb = -1, R = -1;
  mdr_lga_settings s{};
  mdr_dev_instance* di = nullptr;
  mdr_lga_batch* b = nullptr;
};

struct mdr_ctx {
  int device = 0;
  cudaStream_t own = nullptr;
  cudaStream_t stream = nullptr;
  // Default pair arithmetic: FP64 with FMA + one reciprocal per pair.  Its
  // float outputs matched the reference bit for bit on every measured
  // evaluation and local search and on 380 of 400 paired LGA runs
  // (profiles/r1_parity_scale.json); MDR_PAIR_FP64 keeps the reference's
  // exact double operation order with correctly rounded trig (399 of 400).
  int pair = MDR_PAIR_FP64_FAST;
  int wpb = 2;        // warps per CTA of the warp-per-pose kernels
  int cta_warps = 0;  // 0: warp per pose (fastest measured); >0: CTA-per-pose LS
  int exact = 0;      // analytic mode: exact per-group torsion gradient (mdr_ctx_set_exact_torsion)
  int chunking = 1;   // FP64-fast: chunked site mapping for small ligands (MDR_CHUNKING=0 disables)
  int chunk_len = 0;  // > 0: pin the chunk length (MDR_CHUNK_LEN, timing only)
  int ls_pair = 1;    // warp-pair Lamarckian searches (MDR_LS_PAIR=0 disables)
  int tc05 = 1;       // TcuSplit batched reductions on tcgen05 where they win (MDR_TC05=0 disables)
  int ls_warps = 3;   // LGA Lamarckian search form (MDR_LS_WARPS): 3 = ls_multi.cu leaders + shared item-warp pool,
                      // 2 = ls_multi.cu leader + helper warp, 1 = one warp, 0 = legacy pair kernel
  int ls_chunk_len = 0;  // > 0: pin the search's chunk length (MDR_LS_CHUNK_LEN, timing only)
  int ls_group = 0;      // > 0: pin the search's atoms per item (MDR_LS_GROUP: 1 or 3)

  std::string err;
  uint64_t launches = 0;
  LgaCache lga;
};

struct mdr_dev_instance {
  LigandView view{};
  void* block = nullptr;  // one device allocation holding every array
  int n_atoms = 0, n_sites = 0, n_rot = 0;
  // grid-map scoring mode (mdr_instance_set_grid)
  bool grid = false;
  GridView gview{};
  FlexView flex{};
  void* flex_block = nullptr;
};

struct mdr_dev_grid {
  GridView view{};
  float* maps = nullptr;
};

namespace {

thread_local std::string t_err;

int fail(mdr_ctx* ctx, int code, const std::string& msg) {
  t_err = msg;
  if (ctx) ctx->err = msg;
  return code;
}

int cuda_fail(mdr_ctx* ctx, cudaError_t e, const char* where) {
  return fail(ctx, MDR_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

#define CK(expr)                                            \
  do {                                                      \
    cudaError_t _e = (expr);                                \
    if (_e != cudaSuccess) return cuda_fail(ctx, _e, #expr); \
  } while (0)

bool legal_block(int threads, int method) {
  const int lo = method == MDR_METHOD_TCU ? 64 : 32;
  return threads >= lo && threads <= 1024 && threads % 32 == 0;
}

int check_partition(mdr_ctx* ctx, int partition, int method) {
  if (method < 0 || method > 2) return fail(ctx, MDR_ERR_INVALID, "unknown reduce method");
  if (!legal_block(partition, method))
    return fail(ctx, MDR_ERR_BLOCK_SIZE,
                std::string(method == MDR_METHOD_TCU ? "tcu" : "baseline") +
                    " blocks support multiples of 32 in [" + (method == MDR_METHOD_TCU ? "64" : "32") +
                    ", 1024], got " + std::to_string(partition));
  return MDR_OK;
}

// ---------------------------------------------------------- model counters
void st_zero(mdr_sync_stats* s) { std::memset(s, 0, sizeof *s); }
void st_add(mdr_sync_stats* a, const mdr_sync_stats& b, uint64_t k = 1) {
  a->block_syncs += k * b.block_syncs;
  a->warp_shuffles += k * b.warp_shuffles;
  a->atomic_adds += k * b.atomic_adds;
  a->memory_fences += k * b.memory_fences;
  a->mma_ops += k * b.mma_ops;
  a->shared_mem_bytes += k * b.shared_mem_bytes;
  a->precision_conversions += k * b.precision_conversions;
}
mdr_sync_stats block_stats(int threads) {  // reduce.cpp:149-162
  mdr_sync_stats s;
  st_zero(&s);
  s.block_syncs = 3;
  s.memory_fences = 2;
  s.shared_mem_bytes = 4;
  s.atomic_adds = (uint64_t)(threads / 32);
  s.warp_shuffles = 160ull * (uint64_t)(threads / 32);
  return s;
}
mdr_sync_stats reduce4_stats(int n, int accum) {  // reduce.cpp:84-110
  mdr_sync_stats s;
  st_zero(&s);
  const uint64_t chunks = (uint64_t)((n + 63) / 64);
  s.block_syncs = 2;
  s.shared_mem_bytes = chunks * 64 * 4 * 2;
  s.precision_conversions = 4ull * (uint64_t)n + (accum == MDR_ACCUM_HALF ? 4u : 256u);
  s.mma_ops = chunks + 1;
  return s;
}
// TcuSplit (new method): counts of the in-warp implementation per reduction
// of n records with `comps` components: tf32 hi/lo conversions, one
// m16n8k8 per 8 source lanes, a 1 KiB staging buffer, broadcast shuffles.
mdr_sync_stats split_stats(int n, int comps) {
  mdr_sync_stats s;
  st_zero(&s);
  const uint64_t groups = (uint64_t)((n + 31) / 32);
  s.mma_ops = 4 * groups;
  s.shared_mem_bytes = 1024;
  s.precision_conversions = 2ull * (uint64_t)comps * (uint64_t)n;
  s.warp_shuffles = 32ull * (uint64_t)comps;
  return s;
}
mdr_sync_stats reduce7_stats(int n, int method, int accum) {
  mdr_sync_stats s;
  st_zero(&s);
  if (method == MDR_METHOD_BASELINE) {
    st_add(&s, block_stats(n), 7);
  } else if (method == MDR_METHOD_TCU) {
    st_add(&s, reduce4_stats(n, accum), 2);
  } else {
    s = split_stats(n, 7);
  }
  return s;
}

template <class T>
struct DevBuf {
  T* p = nullptr;
  cudaStream_t s = nullptr;
  cudaError_t alloc(size_t n, cudaStream_t st) {
    s = st;
    if (n == 0) n = 1;
    return cudaMallocAsync(reinterpret_cast<void**>(&p), n * sizeof(T), st);
  }
  ~DevBuf() {
    if (p) cudaFreeAsync(p, s);
  }
};

cudaStream_t S(mdr_ctx* c) { return c->stream; }

// The CTA-per-pose local search is used for the fast pair modes; the
// bit-faithful FP64 mode keeps the warp-per-pose kernels (sites summed in
// the reference's order).
int cta_warps_for(const mdr_ctx* c) { return c->pair == MDR_PAIR_FP64 || c->exact ? 0 : c->cta_warps; }

// The analytic-mode ligand view a launch uses: the instance's arrays plus the
// context's torsion-gradient mode.
// Site chunking of the FP64-fast warp-per-pose evaluation (mdr_device.cuh
// score_sums): lane per atom leaves 32 - n_atoms lanes idle in the site loop
// of a small ligand, so the sites are split into chunks of `len` (a multiple
// of the kernel's ILP batch MDR_PV_CHUNK, so no chunk runs a scalar tail
// unless n_sites itself is ragged) and the n_atoms x n_chunks (atom, chunk)
// items spread over the 32 lanes.  len minimises the per-lane cost
// rounds x (len + 4 sites' worth of staging and shorter ILP), with at most
// kMaxChunkItems items; 1 chunk keeps lane per atom.  C3 (20 atoms x 64
// sites) measured: lane per atom 145.8, len 8 / 16 / 24 / 32 -> 148.0 /
// 146.3 / 150.4 / 130.0 M evals/s; the model picks 24.  When the LGA's
// searches run on a warp pair (`pair_lanes`: more than 32 items go to the
// 64 lanes of lga_ls_pair_kernel) the rounds are counted over 64 lanes with
// no staging term, ties to the shorter chunk: C3 measured len 8 / 16 / 24 /
// 32 -> 170.6 / 162.8 / 165.2 / 142.0 M, the model picks 8.  `force_len` > 0
// pins len (timing).
void pick_chunks(int na, int ns, int search_lanes, int force_len, int& n_chunks, int& chunk_len) {
  constexpr int kBatch = 8;  // MDR_PV_CHUNK
  n_chunks = 1;
  chunk_len = ns;
  long best = (long)((na + 31) / 32) * ns;
  for (int len = kBatch; len < ns; len += kBatch) {
    const int n = (ns + len - 1) / len;
    if (na * n > kMaxChunkItems) continue;
    const int lanes = search_lanes > 32 && na * n > 32 ? search_lanes : 32;
    const long cost = (long)((na * n + lanes - 1) / lanes) * (len + (lanes > 32 ? 0 : 4));
    if (force_len > 0 ? len == force_len : cost < best) {
      best = cost;
      n_chunks = n;
      chunk_len = len;
      if (force_len > 0) break;
    }
  }
}

// Items of the two-warp LGA search (ls_multi.cu): (chunk of len sites,
// group of G atoms) over 64 lanes; the critical path is rounds x G x len
// pair terms per lane, G = 1 preferred on ties.  C3 (20 atoms x 64 sites):
// G = 1, len 8 -> 160 items, 3 rounds x 8; G = 3, len 8 -> 56 items, 1
// round x 24: equal path and a third of the site loads, but measured
// 200.3 vs 179.9 M evals/s (G = 3 holds 6 pair terms in flight per lane at
// 128 registers, G = 1 eight; profiles/r2_ls_multi_ab.json).  Up to 512
// (atom, chunk) items (C4 analytic, 100 atoms x 64 sites: 4 chunks of 16,
// 54.6 M evals/s against 51.3 M with the warp-per-pose kernels' 256-item
// limit, 2 chunks of 32).
void pick_search_items(int na, int ns, int force_len, int force_group, int& n_chunks, int& chunk_len, int& group) {
  constexpr int kBatch = 8;
  n_chunks = 1;
  chunk_len = ns;
  group = 1;
  if (force_len > 0) {  // timing / test override (MDR_LS_CHUNK_LEN, MDR_LS_GROUP): any length, 1-3 atoms per item
    const int n = (ns + force_len - 1) / force_len;
    if (n > 1 && na * n <= kMaxChunkItemsForced && na * n > 32) {
      n_chunks = n;
      chunk_len = force_len;
      group = force_group >= 1 && force_group <= 3 ? force_group : 1;
    }
    return;
  }
  long best = (long)((na + 31) / 32) * ns;
  for (int G : {1, 3}) {
    if (force_group > 0 && G != force_group) continue;
    for (int len = kBatch; len < ns; len += kBatch) {
      const int n = (ns + len - 1) / len;
      if (na * n > kMaxChunkItemsForced || na * n <= 32) continue;  // the search's own part buffers
      const int items = (na + G - 1) / G * n;
      const long cost = (long)((items + 63) / 64) * G * len;
      if (cost < best) {
        best = cost;
        n_chunks = n;
        chunk_len = len;
        group = G;
      }
    }
  }
}

LigandView launch_view(const mdr_ctx* c, const mdr_dev_instance* di) {
  LigandView L = di->view;
  L.exact_torsion = c->exact;
  L.n_chunks = 1;
  L.chunk_len = L.n_sites;
  L.ls_pair = c->ls_pair;
  L.ls_warps = c->ls_warps;
  L.ls_n_chunks = 1;
  L.ls_chunk_len = L.n_sites;
  // the warp-per-pose kernels (score, init, offspring, one-warp search,
  // polish) spread chunk items over 32 lanes; the LGA's multi-warp search
  // over the 64 lanes of its warp pair (ls_multi.cu or the legacy kernel)
  const bool multi = c->ls_pair && c->ls_warps != 1 && !c->exact && c->wpb <= 7 && c->cta_warps == 0;
  const int search_lanes = multi ? 64 : 32;
  L.ls_group = 1;
  if (c->pair == MDR_PAIR_FP64_FAST && c->chunking) {
    pick_chunks(L.n_atoms, L.n_sites, 32, c->chunk_len, L.n_chunks, L.chunk_len);
    const int force = c->ls_chunk_len > 0 ? c->ls_chunk_len : c->chunk_len;
    if (multi && c->ls_warps >= 2)
      pick_search_items(L.n_atoms, L.n_sites, force, c->ls_group, L.ls_n_chunks, L.ls_chunk_len, L.ls_group);
    else
      pick_chunks(L.n_atoms, L.n_sites, search_lanes, force, L.ls_n_chunks, L.ls_chunk_len);
  }
  return L;
}

int check_exact(mdr_ctx* ctx, const mdr_dev_instance* di) {
  if (ctx->exact && !di->grid && di->n_atoms > kMaxExactAtoms)
    return fail(ctx, MDR_ERR_SIZE, "exact-torsion mode supports at most " + std::to_string(kMaxExactAtoms) + " atoms");
  return MDR_OK;
}


}  // namespace

extern "C" {

const char* mdr_version(void) { return "mdr-b200 0.1.0 (sm_100a)"; }

int mdr_phase_prof(uint64_t* out16, int reset) {
  if (!out16) return fail(nullptr, MDR_ERR_INVALID, "null argument");
  unsigned long long v[16];
  if (!phase_prof_read(v, reset != 0))
    return fail(nullptr, MDR_ERR_INVALID, "not a phase-profiling build (-DMDR_PHASE_PROF=1)");
  for (int k = 0; k < 16; ++k) out16[k] = v[k];
  return MDR_OK;
}

int mdr_phase_prof_sm(uint32_t* out256, int reset) {
  if (!out256) return fail(nullptr, MDR_ERR_INVALID, "null argument");
  unsigned v[256];
  unsigned gv[256];
  if (!sm_searches_read(v, reset != 0) || !sm_grid_read(gv, reset != 0))
    return fail(nullptr, MDR_ERR_INVALID, "not a phase-profiling build (-DMDR_PHASE_PROF=1)");
  for (int k = 0; k < 256; ++k) out256[k] = v[k] + gv[k];  // analytic two-warp search + grid-mode search
  return MDR_OK;
}

mdr_ctx* mdr_ctx_create(int device) {
  if (cudaSetDevice(device) != cudaSuccess) return nullptr;
  mdr_ctx* c = new mdr_ctx;
  c->device = device;
  if (cudaStreamCreateWithFlags(&c->own, cudaStreamNonBlocking) != cudaSuccess) {
    delete c;
    return nullptr;
  }
  c->stream = c->own;
  if (const char* v = std::getenv("MDR_CHUNKING")) c->chunking = std::atoi(v) != 0;  // A/B timing knobs
  if (const char* v = std::getenv("MDR_CHUNK_LEN")) c->chunk_len = std::atoi(v);
  if (const char* v = std::getenv("MDR_LS_PAIR")) c->ls_pair = std::atoi(v) != 0;
  if (const char* v = std::getenv("MDR_TC05")) c->tc05 = std::atoi(v) != 0;
  if (const char* v = std::getenv("MDR_LS_WARPS")) c->ls_warps = std::atoi(v);
  if (const char* v = std::getenv("MDR_LS_CHUNK_LEN")) c->ls_chunk_len = std::atoi(v);
  if (const char* v = std::getenv("MDR_LS_GROUP")) c->ls_group = std::atoi(v);
  return c;
}

void mdr_ctx_destroy(mdr_ctx* c) {
  if (!c) return;
  cudaStreamSynchronize(c->stream);
  mdr_lga_batch_destroy(c, c->lga.b);
  mdr_instance_free(c, c->lga.di);
  cudaStreamDestroy(c->own);
  delete c;
}

int mdr_ctx_set_stream(mdr_ctx* c, void* s) {
  if (!c) return MDR_ERR_INVALID;
  c->stream = s ? static_cast<cudaStream_t>(s) : c->own;
  return MDR_OK;
}
void* mdr_ctx_stream(mdr_ctx* c) { return c ? c->stream : nullptr; }

int mdr_ctx_set_pair_precision(mdr_ctx* c, int p) {
  if (!c || p < MDR_PAIR_FP64 || p > MDR_PAIR_FP64_FAST) return fail(c, MDR_ERR_INVALID, "bad pair precision");
  c->pair = p;
  return MDR_OK;
}

int mdr_ctx_set_cta_warps(mdr_ctx* c, int w) {
  if (!c || w < 0 || w > 16) return fail(c, MDR_ERR_INVALID, "CTA warps must be 0..16 (0 = warp per pose)");
  c->cta_warps = w;
  return MDR_OK;
}

int mdr_ctx_set_ls_warps(mdr_ctx* c, int w) {
  if (!c || w < 0 || w > 3)
    return fail(c, MDR_ERR_INVALID, "search form must be 0..3 (3 = item-warp pool, 2 = helper, 1 = one warp, 0 = legacy pair)");
  c->ls_warps = w;
  c->ls_pair = w != 1;
  return MDR_OK;
}

int mdr_search_chunking(int pair, int na, int ns, int warps, int* n_chunks, int* chunk_len, int* atoms_per_item) {
  if (!n_chunks || !chunk_len || na < 0 || ns < 0 || warps < 1 || warps > 3 || pair < MDR_PAIR_FP64 ||
      pair > MDR_PAIR_FP64_FAST)
    return fail(nullptr, MDR_ERR_INVALID, "bad argument");
  *n_chunks = 1;
  *chunk_len = ns;
  int group = 1;
  if (pair == MDR_PAIR_FP64_FAST) {
    if (warps >= 2)
      pick_search_items(na, ns, 0, 0, *n_chunks, *chunk_len, group);
    else
      pick_chunks(na, ns, 32, 0, *n_chunks, *chunk_len);
  }
  if (atoms_per_item) *atoms_per_item = group;
  return MDR_OK;
}

int mdr_site_chunking(int pair, int na, int ns, int* n_chunks, int* chunk_len) {
  if (!n_chunks || !chunk_len || na < 0 || ns < 0 || pair < MDR_PAIR_FP64 || pair > MDR_PAIR_FP64_FAST)
    return fail(nullptr, MDR_ERR_INVALID, "bad argument");
  *n_chunks = 1;
  *chunk_len = ns;
  if (pair == MDR_PAIR_FP64_FAST) pick_chunks(na, ns, 32, 0, *n_chunks, *chunk_len);
  return MDR_OK;
}

int mdr_ctx_set_exact_torsion(mdr_ctx* c, int on) {
  if (!c || (on != 0 && on != 1)) return fail(c, MDR_ERR_INVALID, "exact torsion flag must be 0 or 1");
  c->exact = on;
  return MDR_OK;
}

int mdr_ctx_set_warps_per_block(mdr_ctx* c, int wpb) {
  if (!c || wpb < 1 || wpb > 16) return fail(c, MDR_ERR_INVALID, "warps per block must be 1..16");
  c->wpb = wpb;
  return MDR_OK;
}

const char* mdr_last_error(mdr_ctx* c) { return c ? c->err.c_str() : t_err.c_str(); }
uint64_t mdr_ctx_launch_count(mdr_ctx* c) { return c ? c->launches : 0; }
int mdr_ctx_synchronize(mdr_ctx* ctx) {
  CK(cudaStreamSynchronize(ctx->stream));
  return MDR_OK;
}

// ---------------------------------------------------------------- L0
int mdr_f32_to_half_batch(mdr_ctx* ctx, const float* in, size_t n, uint16_t* out) {
  if (!ctx || (n && (!in || !out))) return fail(ctx, MDR_ERR_INVALID, "null argument");
  if (n == 0) return MDR_OK;
  DevBuf<float> di;
  DevBuf<uint16_t> dout;
  CK(di.alloc(n, S(ctx)));
  CK(dout.alloc(n, S(ctx)));
  CK(cudaMemcpyAsync(di.p, in, n * 4, cudaMemcpyHostToDevice, S(ctx)));
  CK(launch_f32_to_half(di.p, n, dout.p, S(ctx)));
  ctx->launches++;
  CK(cudaMemcpyAsync(out, dout.p, n * 2, cudaMemcpyDeviceToHost, S(ctx)));
  CK(cudaStreamSynchronize(S(ctx)));
  return MDR_OK;
}

int mdr_half_to_f32_batch(mdr_ctx* ctx, const uint16_t* in, size_t n, float* out) {
  if (!ctx || (n && (!in || !out))) return fail(ctx, MDR_ERR_INVALID, "null argument");
  if (n == 0) return MDR_OK;
  DevBuf<uint16_t> di;
  DevBuf<float> dout;
  CK(di.alloc(n, S(ctx)));
  CK(dout.alloc(n, S(ctx)));
  CK(cudaMemcpyAsync(di.p, in, n * 2, cudaMemcpyHostToDevice, S(ctx)));
  CK(launch_half_to_f32(di.p, n, dout.p, S(ctx)));
  ctx->launches++;
  CK(cudaMemcpyAsync(out, dout.p, n * 4, cudaMemcpyDeviceToHost, S(ctx)));
  CK(cudaStreamSynchronize(S(ctx)));
  return MDR_OK;
}

int mdr_mma_batch(mdr_ctx* ctx, const uint16_t* a, const uint16_t* b, const float* c, int n_tiles, int accum,
                  float* d) {
  if (!ctx || n_tiles < 0 || (n_tiles && (!a || !b || !c || !d))) return fail(ctx, MDR_ERR_INVALID, "bad argument");
  if (n_tiles == 0) return MDR_OK;
  const size_t n = (size_t)n_tiles * 256;
  DevBuf<uint16_t> da, db;
  DevBuf<float> dc, dd;
  CK(da.alloc(n, S(ctx)));
  CK(db.alloc(n, S(ctx)));
  CK(dc.alloc(n, S(ctx)));
  CK(dd.alloc(n, S(ctx)));
  CK(cudaMemcpyAsync(da.p, a, n * 2, cudaMemcpyHostToDevice, S(ctx)));
  CK(cudaMemcpyAsync(db.p, b, n * 2, cudaMemcpyHostToDevice, S(ctx)));
  CK(cudaMemcpyAsync(dc.p, c, n * 4, cudaMemcpyHostToDevice, S(ctx)));
  CK(launch_mma16(da.p, db.p, dc.p, n_tiles, accum == MDR_ACCUM_HALF, dd.p, S(ctx)));
  ctx->launches++;
  CK(cudaMemcpyAsync(d, dd.p, n * 4, cudaMemcpyDeviceToHost, S(ctx)));
  CK(cudaStreamSynchronize(S(ctx)));
  return MDR_OK;
}

// ---------------------------------------------------------------- L1
int mdr_warp_reduce_batch(mdr_ctx* ctx, const float* lanes, int n_red, float* out, mdr_sync_stats* st) {
  if (!ctx || n_red < 0 || (n_red && (!lanes || !out))) return fail(ctx, MDR_ERR_INVALID, "bad argument");
  if (st) {
    st_zero(st);
    st->warp_shuffles = 160;
  }
  if (n_red == 0) return MDR_OK;
  DevBuf<float> di, dout;
  CK(di.alloc((size_t)n_red * 32, S(ctx)));
  CK(dout.alloc(n_red, S(ctx)));
  CK(cudaMemcpyAsync(di.p, lanes, (size_t)n_red * 32 * 4, cudaMemcpyHostToDevice, S(ctx)));
  CK(launch_warp_reduce(di.p, n_red, dout.p, S(ctx)));
  ctx->launches++;
  CK(cudaMemcpyAsync(out, dout.p, (size_t)n_red * 4, cudaMemcpyDeviceToHost, S(ctx)));
  CK(cudaStreamSynchronize(S(ctx)));
  return MDR_OK;
}

int mdr_block_reduce_batch(mdr_ctx* ctx, const float* values, int threads, int n_red, float* out,
                           mdr_sync_stats* st) {
  if (!ctx || n_red < 0 || (n_red && (!values || !out))) return fail(ctx, MDR_ERR_INVALID, "bad argument");
  if (!legal_block(threads, MDR_METHOD_BASELINE))
    return fail(ctx, MDR_ERR_BLOCK_SIZE,
                "baseline_block_reduce supports multiples of 32 in [32, 1024], got " + std::to_string(threads));
  if (st) *st = block_stats(threads);
  if (n_red == 0) return MDR_OK;
  const size_t n = (size_t)n_red * threads;
  DevBuf<float> di, dout;
  CK(di.alloc(n, S(ctx)));
  CK(dout.alloc(n_red, S(ctx)));
  CK(cudaMemcpyAsync(di.p, values, n * 4, cudaMemcpyHostToDevice, S(ctx)));
  CK(launch_block_reduce(di.p, threads, n_red, dout.p, S(ctx)));
  ctx->launches++;
  CK(cudaMemcpyAsync(out, dout.p, (size_t)n_red * 4, cudaMemcpyDeviceToHost, S(ctx)));
  CK(cudaStreamSynchronize(S(ctx)));
  return MDR_OK;
}

// TcuSplit batches on the tcgen05 contraction (K2t, tc05_reduce.cu): many
// reductions of a multiple of 32 records, at least kTc05MinRed of them (one
// 32-reduction tile per CTA on every SM).  Elsewhere the warp-per-reduction
// mma.sync kernels run.  Both are fp32-accurate (tf32 hi/lo split).
constexpr int kTc05MinRed = 148 * 32;
static bool use_tc05(const mdr_ctx* ctx, int method, int n, int n_red) {
  return ctx->tc05 && method == MDR_METHOD_TCU_SPLIT && n % 32 == 0 && n >= 32 && n_red >= kTc05MinRed;
}

static int reduce4_check(mdr_ctx* ctx, int n, int method, int accum, mdr_sync_stats* st) {
  if (method < 0 || method > 2) return fail(ctx, MDR_ERR_INVALID, "unknown reduce method");
  if (n < 1) return fail(ctx, MDR_ERR_SIZE, "reduce4 requires at least one vector");
  if (method == MDR_METHOD_BASELINE && !legal_block(n, method))
    return fail(ctx, MDR_ERR_BLOCK_SIZE, "baseline blocks support multiples of 32 in [32, 1024], got " +
                                             std::to_string(n));
  if (st) {
    if (method == MDR_METHOD_TCU) {
      *st = reduce4_stats(n, accum);
    } else if (method == MDR_METHOD_BASELINE) {
      st_zero(st);
      st_add(st, block_stats(n), 4);
    } else {
      *st = split_stats(n, 4);
    }
  }
  return MDR_OK;
}

static cudaError_t enqueue_reduce4(mdr_ctx* ctx, const float* d_in, int n, int n_red, int method, int accum,
                                   float* d_out) {
  if (use_tc05(ctx, method, n, n_red)) return launch_reduce4_tc05(d_in, n, n_red, d_out, 3, S(ctx));
  return launch_reduce4(d_in, n, n_red, method, accum == MDR_ACCUM_HALF, d_out, S(ctx));
}

int mdr_reduce4_batch(mdr_ctx* ctx, const float* vecs, int n, int n_red, int method, int accum, float* out,
                      mdr_sync_stats* st) {
  if (!ctx || n_red < 0 || (n_red && (!vecs || !out))) return fail(ctx, MDR_ERR_INVALID, "bad argument");
  if (int rc = reduce4_check(ctx, n, method, accum, st)) return rc;
  if (n_red == 0) return MDR_OK;
  const size_t cnt = (size_t)n_red * n * 4;
  DevBuf<float> di, dout;
  CK(di.alloc(cnt, S(ctx)));
  CK(dout.alloc((size_t)n_red * 4, S(ctx)));
  CK(cudaMemcpyAsync(di.p, vecs, cnt * 4, cudaMemcpyHostToDevice, S(ctx)));
  CK(enqueue_reduce4(ctx, di.p, n, n_red, method, accum, dout.p));
  ctx->launches++;
  CK(cudaMemcpyAsync(out, dout.p, (size_t)n_red * 16, cudaMemcpyDeviceToHost, S(ctx)));
  CK(cudaStreamSynchronize(S(ctx)));
  return MDR_OK;
}

int mdr_reduce4_dev(mdr_ctx* ctx, const float* d_vecs, int n, int n_red, int method, int accum, float* d_out) {
  if (!ctx || n_red < 0 || (n_red && (!d_vecs || !d_out))) return fail(ctx, MDR_ERR_INVALID, "bad argument");
  if (int rc = reduce4_check(ctx, n, method, accum, nullptr)) return rc;
  if (n_red == 0) return MDR_OK;
  CK(enqueue_reduce4(ctx, d_vecs, n, n_red, method, accum, d_out));
  ctx->launches++;
  return MDR_OK;
}

static int reduce7_check(mdr_ctx* ctx, int n, int method, int accum, mdr_sync_stats* st) {
  if (method < 0 || method > 2) return fail(ctx, MDR_ERR_INVALID, "unknown reduce method");
  if (method == MDR_METHOD_BASELINE && !legal_block(n, method))
    return fail(ctx, MDR_ERR_BLOCK_SIZE, "baseline_block_reduce supports multiples of 32 in [32, 1024], got " +
                                             std::to_string(n));
  if (method == MDR_METHOD_TCU && n < 64)
    return fail(ctx, MDR_ERR_BLOCK_SIZE,
                "tcu reduce7 needs at least 64 records (a full 16x16 tile), got " + std::to_string(n));
  if (method == MDR_METHOD_TCU_SPLIT && n < 1) return fail(ctx, MDR_ERR_SIZE, "reduce7 needs records");
  if (st) *st = reduce7_stats(n, method, accum);
  return MDR_OK;
}

static cudaError_t enqueue_reduce7(mdr_ctx* ctx, const float* d_in, int n, int n_red, int method, int accum,
                                   float* d_out) {
  if (use_tc05(ctx, method, n, n_red)) return launch_reduce7_tc05(d_in, n, n_red, d_out, 3, S(ctx));
  return launch_reduce7(d_in, n, n_red, method, accum == MDR_ACCUM_HALF, d_out, S(ctx));
}

int mdr_reduce7_batch(mdr_ctx* ctx, const float* recs, int n, int n_red, int method, int accum, float* out,
                      mdr_sync_stats* st) {
  if (!ctx || n_red < 0 || (n_red && (!recs || !out))) return fail(ctx, MDR_ERR_INVALID, "bad argument");
  if (int rc = reduce7_check(ctx, n, method, accum, st)) return rc;
  if (n_red == 0) return MDR_OK;
  const size_t cnt = (size_t)n_red * n * 7;
  DevBuf<float> di, dout;
  CK(di.alloc(cnt, S(ctx)));
  CK(dout.alloc((size_t)n_red * 7, S(ctx)));
  CK(cudaMemcpyAsync(di.p, recs, cnt * 4, cudaMemcpyHostToDevice, S(ctx)));
  CK(enqueue_reduce7(ctx, di.p, n, n_red, method, accum, dout.p));
  ctx->launches++;
  CK(cudaMemcpyAsync(out, dout.p, (size_t)n_red * 28, cudaMemcpyDeviceToHost, S(ctx)));
  CK(cudaStreamSynchronize(S(ctx)));
  return MDR_OK;
}

int mdr_reduce7_dev(mdr_ctx* ctx, const float* d_recs, int n, int n_red, int method, int accum, float* d_out) {
  if (!ctx || n_red < 0 || (n_red && (!d_recs || !d_out))) return fail(ctx, MDR_ERR_INVALID, "bad argument");
  if (int rc = reduce7_check(ctx, n, method, accum, nullptr)) return rc;
  if (n_red == 0) return MDR_OK;
  CK(enqueue_reduce7(ctx, d_recs, n, n_red, method, accum, d_out));
  ctx->launches++;
  return MDR_OK;
}

int mdr_ctx_set_tc05(mdr_ctx* ctx, int on) {
  if (!ctx) return MDR_ERR_INVALID;
  ctx->tc05 = on != 0;
  return MDR_OK;
}

int mdr_reduce_uses_tc05(mdr_ctx* ctx, int method, int n, int n_red) {
  return ctx && use_tc05(ctx, method, n, n_red) ? 1 : 0;
}

// Self test of the branch-free libdevice sincos (mdr_device.cuh sincos_fast).
int mdr_selftest_sincos(mdr_ctx* ctx, uint64_t seed, int64_t n, uint64_t* mismatches) {
  if (!ctx || !mismatches || n < 0) return fail(ctx, MDR_ERR_INVALID, "bad argument");
  DevBuf<unsigned long long> d;
  CK(d.alloc(1, S(ctx)));
  CK(cudaMemsetAsync(d.p, 0, sizeof(unsigned long long), S(ctx)));
  CK(launch_sincos_selftest(seed, (long long)n, d.p, S(ctx)));
  ctx->launches++;
  unsigned long long h = 0;
  CK(cudaMemcpyAsync(&h, d.p, sizeof h, cudaMemcpyDeviceToHost, S(ctx)));
  CK(cudaStreamSynchronize(S(ctx)));
  *mismatches = h;
  return MDR_OK;
}

// Self test of the branch-free FP64 square root of the LGA search (ls_multi.cu).
int mdr_selftest_dsqrt(mdr_ctx* ctx, uint64_t seed, int64_t n, uint64_t* mismatches) {
  if (!ctx || !mismatches || n < 0) return fail(ctx, MDR_ERR_INVALID, "bad argument");
  DevBuf<unsigned long long> d;
  CK(d.alloc(1, S(ctx)));
  CK(cudaMemsetAsync(d.p, 0, sizeof(unsigned long long), S(ctx)));
  CK(launch_dsqrt_selftest(seed, (long long)n, d.p, S(ctx)));
  ctx->launches++;
  unsigned long long h = 0;
  CK(cudaMemcpyAsync(&h, d.p, sizeof h, cudaMemcpyDeviceToHost, S(ctx)));
  CK(cudaStreamSynchronize(S(ctx)));
  *mismatches = h;
  return MDR_OK;
}

// Self test of the branch-free FP64 division used by the strict pair loop:
// number of bit mismatches against IEEE div.rn.f64 over n operand pairs.
int mdr_selftest_ddiv(mdr_ctx* ctx, uint64_t seed, int64_t n, uint64_t* mismatches) {
  if (!ctx || !mismatches || n < 0) return fail(ctx, MDR_ERR_INVALID, "bad argument");
  DevBuf<unsigned long long> d;
  CK(d.alloc(1, S(ctx)));
  CK(cudaMemsetAsync(d.p, 0, sizeof(unsigned long long), S(ctx)));
  CK(launch_ddiv_selftest(seed, (long long)n, d.p, S(ctx)));
  ctx->launches++;
  unsigned long long h = 0;
  CK(cudaMemcpyAsync(&h, d.p, sizeof h, cudaMemcpyDeviceToHost, S(ctx)));
  CK(cudaStreamSynchronize(S(ctx)));
  *mismatches = h;
  return MDR_OK;
}

// C2 microbench: one block-level float4 reduce-and-broadcast per thread
// block (see bench_reduce.cu for the kernel roster).
int mdr_crmath_values(mdr_ctx* ctx, int64_t i0, int n, double* out) {
  if (!ctx || n < 0 || (n && !out)) return fail(ctx, MDR_ERR_INVALID, "bad argument");
  if (n == 0) return MDR_OK;
  DevBuf<double> d;
  CK(d.alloc((size_t)8 * n, S(ctx)));
  CK(launch_crmath_probe((long long)i0, n, d.p, S(ctx)));
  ctx->launches++;
  CK(cudaMemcpyAsync(out, d.p, sizeof(double) * 8 * n, cudaMemcpyDeviceToHost, S(ctx)));
  CK(cudaStreamSynchronize(S(ctx)));
  return MDR_OK;
}

int mdr_selftest_crmath(mdr_ctx* ctx, int64_t n, uint64_t* mismatches) {
  if (!ctx || n < 0 || !mismatches) return fail(ctx, MDR_ERR_INVALID, "bad argument");
  std::memset(mismatches, 0, sizeof(uint64_t) * 8);
  const int chunk = 1 << 20;
  DevBuf<double> d;
  CK(d.alloc((size_t)8 * chunk, S(ctx)));
  std::vector<double> h((size_t)8 * chunk);
  auto u64 = [](uint64_t nn) {  // RngStream draw with key 0 (rng.cpp:34-37)
    uint64_t z = nn * 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
  };
  const double pi = 3.14159265358979323846;
  for (int64_t i0 = 0; i0 < n; i0 += chunk) {
    const int m = (int)std::min<int64_t>(chunk, n - i0);
    CK(launch_crmath_probe(i0, m, d.p, S(ctx)));
    CK(cudaMemcpyAsync(h.data(), d.p, sizeof(double) * 8 * m, cudaMemcpyDeviceToHost, S(ctx)));
    CK(cudaStreamSynchronize(S(ctx)));
    for (int t = 0; t < m; ++t) {
      const uint64_t i = (uint64_t)(i0 + t);
      const double a = -pi + 2.0 * pi * ((double)(u64(4 * i + 1) >> 11) * 0x1p-53);
      const double u1 = (double)((u64(4 * i + 2) >> 11) + 1) * 0x1p-53;
      const double z = 2.0 * pi * ((double)(u64(4 * i + 3) >> 11) * 0x1p-53);
      const double want[4] = {std::sin(a), std::cos(a), std::log(u1), std::cos(z)};
      const double* o = &h[(size_t)8 * t];
      for (int k = 0; k < 4; ++k) {
        mismatches[k] += o[k] != want[k];
        mismatches[4 + k] += o[4 + k] != want[k];
      }
    }
  }
  ctx->launches += (uint64_t)((n + chunk - 1) / chunk);
  return MDR_OK;
}

int mdr_reduce_bench_chain_cycles_dev(mdr_ctx* ctx, int kernel, int block, const float* d_in, int n_red,
                                      int chain_steps, float* d_out, int64_t* d_cycles) {
  if (!ctx || !d_in || !d_out || !d_cycles || n_red <= 0 || chain_steps <= 0 || kernel < 0 || kernel >= 7)
    return fail(ctx, MDR_ERR_INVALID, "bad argument (chain-mode kernels 0..6)");
  if (block < 64 || block > 1024 || block % 64)
    return fail(ctx, MDR_ERR_BLOCK_SIZE, "bench blocks are multiples of 64 in [64, 1024]");
  if (n_red % chain_steps) return fail(ctx, MDR_ERR_SIZE, "n_red must be a multiple of steps");
  CK(launch_reduce_bench(kernel, block, d_in, n_red, chain_steps, d_out, 0, ctx->stream,
                         reinterpret_cast<long long*>(d_cycles)));
  ctx->launches++;
  return MDR_OK;
}

int mdr_reduce_bench_kernels(void) { return kReduceBenchKernels; }
const char* mdr_reduce_bench_kernel_name(int k) { return reduce_bench_name(k); }

int mdr_reduce_bench_dev(mdr_ctx* ctx, int kernel, int block, const float* d_in, int n_red, int chain_steps,
                         float* d_out) {
  if (!ctx || !d_in || !d_out || n_red <= 0 || kernel < 0 || kernel >= kReduceBenchKernels)
    return fail(ctx, MDR_ERR_INVALID, "bad argument");
  if (block < 64 || block > 1024 || block % 64)
    return fail(ctx, MDR_ERR_BLOCK_SIZE, "bench blocks are multiples of 64 in [64, 1024]");
  if (chain_steps > 0 && n_red % chain_steps) return fail(ctx, MDR_ERR_SIZE, "n_red must be a multiple of steps");
  if (kernel == 7 || kernel == 8) {  // tcgen05 batched: streaming only (32 reductions per contraction)
    if (chain_steps > 0) return fail(ctx, MDR_ERR_INVALID, "the tcgen05 batched kernels have no chain mode");
    if (kernel == 7)
      CK(launch_reduce4_tc05(d_in, block, n_red, d_out, 3, ctx->stream));
    else
      CK(launch_reduce4_tc05_tma(d_in, block, n_red, d_out, ctx->stream));
  } else {
    CK(launch_reduce_bench(kernel, block, d_in, n_red, chain_steps, d_out, 2048 / block, ctx->stream));
  }
  ctx->launches++;
  return MDR_OK;
}

// ---------------------------------------------------------------- ligand
static void torsion_axis_host(int k, double* out) {  // docking.cpp:181-189 (glibc, like the reference)
  constexpr double kGolden = 2.399963229728653;
  const double az = kGolden * k + 0.3;
  const double zc = 0.5 + 0.35 * std::sin(0.9 * k + 0.4);
  const double v[3] = {0.8 * std::cos(az), 0.8 * std::sin(az), zc};
  const double n = std::sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]);
  out[0] = v[0] / n;
  out[1] = v[1] / n;
  out[2] = v[2] / n;
}

static int check_instance(mdr_ctx* ctx, const mdr_instance* in) {
  if (!in || !in->atom_xyzw || !in->atom_torsion || !in->site_xyzdd)
    return fail(ctx, MDR_ERR_INVALID, "null instance");
  if (in->n_atoms < 1 || in->n_sites < 1) return fail(ctx, MDR_ERR_SIZE, "instance needs atoms and sites");
  if (in->n_rot < 0 || in->n_rot > kMaxRot)
    return fail(ctx, MDR_ERR_SIZE, "n_rot must be in [0, " + std::to_string(kMaxRot) + "] on the device path");
  if (in->n_sites > kMaxSites || in->n_atoms > kMaxAtoms)
    return fail(ctx, MDR_ERR_SIZE, "instance exceeds the device limits (sites <= 2048, atoms <= 4096)");
  for (int i = 0; i < in->n_atoms; ++i)
    if (in->atom_torsion[i] >= in->n_rot || in->atom_torsion[i] < -1)
      return fail(ctx, MDR_ERR_SIZE, "atom references a torsion outside [0, n_rot)");
  return MDR_OK;
}

// random_genotype's box (docking.cpp:362-374): site bounding box +- (max d0 + 1).
static void genotype_box(const mdr_instance* in, double box[6]) {
  double lo[3] = {std::numeric_limits<double>::max(), std::numeric_limits<double>::max(),
                  std::numeric_limits<double>::max()};
  double hi[3] = {std::numeric_limits<double>::lowest(), std::numeric_limits<double>::lowest(),
                  std::numeric_limits<double>::lowest()};
  double max_d0 = 0.0;
  for (int j = 0; j < in->n_sites; ++j) {
    const double* s = in->site_xyzdd + 5 * j;
    for (int a = 0; a < 3; ++a) {
      lo[a] = std::min(lo[a], s[a]);
      hi[a] = std::max(hi[a], s[a]);
    }
    max_d0 = std::max(max_d0, s[4]);
  }
  const double margin = max_d0 + 1.0;
  for (int a = 0; a < 3; ++a) {
    box[a] = lo[a] - margin;
    box[3 + a] = hi[a] + margin;
  }
}

// Device layout of one ligand: a single allocation
//   sites | atoms | torsion axes | torsion ids | fp32 sites | fp32 consts | box
namespace {
struct InstLayout {
  size_t o_sites, o_atoms, o_tax, o_tors, o_sf, o_sf2, o_box, total;
  explicit InstLayout(int na, int ns, int nr) {
    auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
    o_sites = 0;
    o_atoms = o_sites + al(sizeof(SiteD) * ns);
    o_tax = o_atoms + al(sizeof(double4) * na);
    o_tors = o_tax + al(sizeof(double) * 3 * (size_t)std::max(nr, 1));
    o_sf = o_tors + al(sizeof(int) * na);
    o_sf2 = o_sf + al(sizeof(float4) * ns);
    o_box = o_sf2 + al(sizeof(float2) * ns);
    total = o_box + al(sizeof(double) * 6);
  }
};

// Host-side preparation + async copy of a ligand into an existing block of
// the same shape.  The pair-loop constants and the random_genotype box are
// computed here in the reference's evaluation order (docking.cpp:114-116,
// 362-374); torsion axes with glibc like torsion_axis (docking.cpp:181-189).
int write_instance(mdr_ctx* ctx, mdr_dev_instance* di, const mdr_instance* in) {
  const int na = in->n_atoms, ns = in->n_sites, nr = in->n_rot;
  const InstLayout lay(na, ns, nr);
  std::vector<SiteD> sites(ns);
  std::vector<float4> sf(ns);
  std::vector<float2> sf2(ns);
  double lo[3] = {std::numeric_limits<double>::max(), std::numeric_limits<double>::max(),
                  std::numeric_limits<double>::max()};
  double hi[3] = {std::numeric_limits<double>::lowest(), std::numeric_limits<double>::lowest(),
                  std::numeric_limits<double>::lowest()};
  double max_d0 = 0.0;
  for (int j = 0; j < ns; ++j) {
    const double* s = in->site_xyzdd + 5 * j;
    const double d0 = s[4];
    SiteD& o = sites[j];
    o.x = s[0];
    o.y = s[1];
    o.z = s[2];
    o.depth = s[3];
    o.c2 = 0.5625 * d0 * d0;  // docking.cpp:114
    o.num = d0 * d0 + o.c2;   // docking.cpp:116
    sf[j] = {(float)s[0], (float)s[1], (float)s[2], (float)s[3]};
    sf2[j] = {(float)o.c2, (float)o.num};
    for (int a = 0; a < 3; ++a) {
      lo[a] = std::min(lo[a], s[a]);
      hi[a] = std::max(hi[a], s[a]);
    }
    max_d0 = std::max(max_d0, d0);
  }
  std::vector<double> taxes(3 * (size_t)std::max(nr, 1), 0.0);
  for (int k = 0; k < nr; ++k) torsion_axis_host(k, &taxes[3 * k]);
  const double margin = max_d0 + 1.0;  // random_genotype docking.cpp:374
  double box[6];
  for (int a = 0; a < 3; ++a) {
    box[a] = lo[a] - margin;
    box[3 + a] = hi[a] + margin;
  }
  char* b = static_cast<char*>(di->block);
  cudaStream_t s = ctx->stream;
  CK(cudaMemcpyAsync(b + lay.o_sites, sites.data(), sizeof(SiteD) * ns, cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(b + lay.o_atoms, in->atom_xyzw, sizeof(double) * 4 * na, cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(b + lay.o_tax, taxes.data(), sizeof(double) * taxes.size(), cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(b + lay.o_tors, in->atom_torsion, sizeof(int) * na, cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(b + lay.o_sf, sf.data(), sizeof(float4) * ns, cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(b + lay.o_sf2, sf2.data(), sizeof(float2) * ns, cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(b + lay.o_box, box, sizeof(box), cudaMemcpyHostToDevice, s));
  CK(cudaStreamSynchronize(s));  // host staging vectors die at return
  return MDR_OK;
}
}  // namespace

mdr_dev_instance* mdr_instance_upload(mdr_ctx* ctx, const mdr_instance* in) {
  if (!ctx || check_instance(ctx, in) != MDR_OK) return nullptr;
  const int na = in->n_atoms, ns = in->n_sites, nr = in->n_rot;
  const InstLayout lay(na, ns, nr);
  mdr_dev_instance* di = new mdr_dev_instance;
  if (cudaMalloc(&di->block, lay.total) != cudaSuccess) {
    fail(ctx, MDR_ERR_CUDA, "cudaMalloc failed for instance");
    delete di;
    return nullptr;
  }
  if (write_instance(ctx, di, in) != MDR_OK) {
    cudaFree(di->block);
    delete di;
    return nullptr;
  }
  char* b = static_cast<char*>(di->block);
  LigandView& L = di->view;
  L.n_atoms = na;
  L.n_sites = ns;
  L.n_rot = nr;
  L.sites = reinterpret_cast<const SiteD*>(b + lay.o_sites);
  L.atoms = reinterpret_cast<const double4*>(b + lay.o_atoms);
  L.taxes = reinterpret_cast<const double*>(b + lay.o_tax);
  L.tors = reinterpret_cast<const int*>(b + lay.o_tors);
  L.sites_f = reinterpret_cast<const float4*>(b + lay.o_sf);
  L.sites_f2 = reinterpret_cast<const float2*>(b + lay.o_sf2);
  L.box = reinterpret_cast<const double*>(b + lay.o_box);
  di->n_atoms = na;
  di->n_sites = ns;
  di->n_rot = nr;
  return di;
}

void mdr_instance_free(mdr_ctx* ctx, mdr_dev_instance* di) {
  if (!di) return;
  if (ctx) cudaStreamSynchronize(ctx->stream);
  cudaFree(di->block);
  if (di->flex_block) cudaFree(di->flex_block);
  delete di;
}

struct InstanceGuard {
  mdr_ctx* ctx;
  mdr_dev_instance* di;
  ~InstanceGuard() { mdr_instance_free(ctx, di); }
};

// Grid kernels run the strict FP64 path (the oracle's arithmetic and order,
// grid.cu grid_eval_strict) when the context's pair precision is
// MDR_PAIR_FP64, the FP32 path with the requested reduction otherwise.
static int grid_method(const mdr_ctx* ctx, int method) {
  return ctx->pair == MDR_PAIR_FP64 ? kGridStrictMethod : method;
}

// Grid mode runs one CTA of `partition` threads per pose: thread d owns
// genotype dimension d, so the block must cover the genotype.
static int check_grid_block(mdr_ctx* ctx, const mdr_dev_instance* di, int partition) {
  if (partition < 6 + di->n_rot)
    return fail(ctx, MDR_ERR_BLOCK_SIZE, "grid mode needs partition >= 6 + n_rot (one thread per dimension)");
  if (grid_smem_for(di->view, di->flex, partition, grid_method(ctx, MDR_METHOD_BASELINE)) > 227 * 1024)
    return fail(ctx, MDR_ERR_SIZE, "grid-mode ligand does not fit in shared memory");
  return MDR_OK;
}

// ---------------------------------------------------------------- L2
static mdr_sync_stats score_stats(int method, int accum, int partition) {
  return reduce7_stats(partition, method, accum);
}

int mdr_score_dev(mdr_ctx* ctx, const mdr_dev_instance* di, const double* g, int n, int method, int accum,
                  int partition, float* e, float* grad, float* tq) {
  if (!ctx || !di) return fail(ctx, MDR_ERR_INVALID, "null argument");
  if (int rc = check_partition(ctx, partition, method)) return rc;
  if (di->grid) {
    if (int rc = check_grid_block(ctx, di, partition)) return rc;
    if (n <= 0) return MDR_OK;
    CK(launch_grid_score(di->view, di->gview, di->flex, g, n, grid_method(ctx, method), partition, e, grad, tq,
                         ctx->stream));
    ctx->launches++;
    return MDR_OK;
  }
  if (int rc = check_exact(ctx, di)) return rc;
  if (n <= 0) return MDR_OK;
  CK(launch_score(launch_view(ctx, di), g, n, method, ctx->pair, partition, accum == MDR_ACCUM_HALF, e, grad, tq, ctx->stream,
                  ctx->wpb));
  ctx->launches++;
  return MDR_OK;
}

int mdr_score_batch(mdr_ctx* ctx, const mdr_instance* inst, const double* genos, int n, int method, int accum,
                    int partition, float* energy, float* gradient, float* torque, mdr_sync_stats* st) {
  if (!ctx || n < 0 || (n && (!genos || !energy || !gradient || !torque)))
    return fail(ctx, MDR_ERR_INVALID, "bad argument");
  if (int rc = check_instance(ctx, inst)) return rc;
  if (int rc = check_partition(ctx, partition, method)) return rc;
  if (st) *st = score_stats(method, accum, partition);
  if (n == 0) return MDR_OK;
  InstanceGuard ig{ctx, mdr_instance_upload(ctx, inst)};
  if (!ig.di) return MDR_ERR_CUDA;
  const int dim = 6 + inst->n_rot;
  DevBuf<double> dg;
  DevBuf<float> de, dgr, dt;
  CK(dg.alloc((size_t)n * dim, S(ctx)));
  CK(de.alloc(n, S(ctx)));
  CK(dgr.alloc((size_t)n * dim, S(ctx)));
  CK(dt.alloc((size_t)n * 3, S(ctx)));
  CK(cudaMemcpyAsync(dg.p, genos, sizeof(double) * n * dim, cudaMemcpyHostToDevice, S(ctx)));
  if (int rc = mdr_score_dev(ctx, ig.di, dg.p, n, method, accum, partition, de.p, dgr.p, dt.p)) return rc;
  CK(cudaMemcpyAsync(energy, de.p, sizeof(float) * n, cudaMemcpyDeviceToHost, S(ctx)));
  CK(cudaMemcpyAsync(gradient, dgr.p, sizeof(float) * n * dim, cudaMemcpyDeviceToHost, S(ctx)));
  CK(cudaMemcpyAsync(torque, dt.p, sizeof(float) * n * 3, cudaMemcpyDeviceToHost, S(ctx)));
  CK(cudaStreamSynchronize(S(ctx)));
  return MDR_OK;
}

int mdr_score_reference_batch(mdr_ctx* ctx, const mdr_instance* inst, const double* genos, int n, double* energy,
                              double* gradient, double* torque) {
  if (!ctx || n < 0 || (n && (!genos || !energy || !gradient || !torque)))
    return fail(ctx, MDR_ERR_INVALID, "bad argument");
  if (int rc = check_instance(ctx, inst)) return rc;
  if (n == 0) return MDR_OK;
  InstanceGuard ig{ctx, mdr_instance_upload(ctx, inst)};
  if (!ig.di) return MDR_ERR_CUDA;
  const int dim = 6 + inst->n_rot;
  DevBuf<double> dg, de, dgr, dt;
  CK(dg.alloc((size_t)n * dim, S(ctx)));
  CK(de.alloc(n, S(ctx)));
  CK(dgr.alloc((size_t)n * dim, S(ctx)));
  CK(dt.alloc((size_t)n * 3, S(ctx)));
  CK(cudaMemcpyAsync(dg.p, genos, sizeof(double) * n * dim, cudaMemcpyHostToDevice, S(ctx)));
  CK(launch_score_reference(ig.di->view, dg.p, n, de.p, dgr.p, dt.p, S(ctx), ctx->wpb));
  ctx->launches++;
  CK(cudaMemcpyAsync(energy, de.p, sizeof(double) * n, cudaMemcpyDeviceToHost, S(ctx)));
  CK(cudaMemcpyAsync(gradient, dgr.p, sizeof(double) * n * dim, cudaMemcpyDeviceToHost, S(ctx)));
  CK(cudaMemcpyAsync(torque, dt.p, sizeof(double) * n * 3, cudaMemcpyDeviceToHost, S(ctx)));
  CK(cudaStreamSynchronize(S(ctx)));
  return MDR_OK;
}

// ---------------------------------------------------------------- L3
int mdr_adadelta_step_batch(mdr_ctx* ctx, int dim, int n, double rho, double eps, double* sq_g, double* sq_u,
                            double* geno, const double* grad) {
  if (!ctx || dim < 6 || dim > kMaxDim || n < 0 || (n && (!sq_g || !sq_u || !geno || !grad)))
    return fail(ctx, MDR_ERR_SIZE, "adadelta_step: state/gradient dimensions do not match genotype");
  if (n == 0) return MDR_OK;
  const size_t cnt = (size_t)n * dim;
  // NumericDomainError is raised before any state changes (docking.cpp:289-293)
  for (size_t i = 0; i < cnt; ++i)
    if (!std::isfinite(grad[i])) return fail(ctx, MDR_ERR_NUMERIC_DOMAIN, "adadelta_step: non-finite gradient component");
  DevBuf<double> a, b, g, gr;
  DevBuf<int> stt;
  CK(a.alloc(cnt, S(ctx)));
  CK(b.alloc(cnt, S(ctx)));
  CK(g.alloc(cnt, S(ctx)));
  CK(gr.alloc(cnt, S(ctx)));
  CK(stt.alloc(n, S(ctx)));
  CK(cudaMemsetAsync(stt.p, 0, sizeof(int) * n, S(ctx)));
  CK(cudaMemcpyAsync(a.p, sq_g, cnt * 8, cudaMemcpyHostToDevice, S(ctx)));
  CK(cudaMemcpyAsync(b.p, sq_u, cnt * 8, cudaMemcpyHostToDevice, S(ctx)));
  CK(cudaMemcpyAsync(g.p, geno, cnt * 8, cudaMemcpyHostToDevice, S(ctx)));
  CK(cudaMemcpyAsync(gr.p, grad, cnt * 8, cudaMemcpyHostToDevice, S(ctx)));
  CK(launch_adadelta(dim, n, rho, eps, a.p, b.p, g.p, gr.p, stt.p, S(ctx)));
  ctx->launches++;
  CK(cudaMemcpyAsync(sq_g, a.p, cnt * 8, cudaMemcpyDeviceToHost, S(ctx)));
  CK(cudaMemcpyAsync(sq_u, b.p, cnt * 8, cudaMemcpyDeviceToHost, S(ctx)));
  CK(cudaMemcpyAsync(geno, g.p, cnt * 8, cudaMemcpyDeviceToHost, S(ctx)));
  CK(cudaStreamSynchronize(S(ctx)));
  return MDR_OK;
}

int mdr_local_search_dev(mdr_ctx* ctx, const mdr_dev_instance* di, const double* starts, int n, int max_iters,
                         double tol, int method, int accum, int partition, double* og, double* oe, int32_t* oit,
                         int32_t* ocv, int32_t* status) {
  if (!ctx || !di || max_iters < 0) return fail(ctx, MDR_ERR_INVALID, "bad argument");
  if (int rc = check_partition(ctx, partition, method)) return rc;
  if (di->grid) {
    if (int rc = check_grid_block(ctx, di, partition)) return rc;
    if (n <= 0) return MDR_OK;
    CK(launch_grid_local_search(di->view, di->gview, di->flex, starts, n, max_iters, tol, grid_method(ctx, method),
                                partition, og, oe,
                                oit, ocv, status, ctx->stream));
    ctx->launches++;
    return MDR_OK;
  }
  if (int rc = check_exact(ctx, di)) return rc;
  if (n <= 0) return MDR_OK;
  CK(launch_local_search(launch_view(ctx, di), starts, n, max_iters, tol, method, ctx->pair, partition, accum == MDR_ACCUM_HALF,
                         og, oe, oit, ocv, status, ctx->stream, ctx->wpb, cta_warps_for(ctx)));
  ctx->launches++;
  return MDR_OK;
}

int mdr_local_search_batch(mdr_ctx* ctx, const mdr_instance* inst, const double* starts, int n, int max_iters,
                           double tol, int method, int accum, int partition, double* out_g, double* out_e,
                           int32_t* out_it, int32_t* out_cv, mdr_sync_stats* st) {
  if (!ctx || n < 0 || max_iters < 0 || (n && (!starts || !out_g || !out_e || !out_it || !out_cv)))
    return fail(ctx, MDR_ERR_INVALID, "bad argument");
  if (int rc = check_instance(ctx, inst)) return rc;
  if (int rc = check_partition(ctx, partition, method)) return rc;
  if (n == 0) return MDR_OK;
  InstanceGuard ig{ctx, mdr_instance_upload(ctx, inst)};
  if (!ig.di) return MDR_ERR_CUDA;
  const int dim = 6 + inst->n_rot;
  DevBuf<double> ds, dg, de;
  DevBuf<int> dit, dcv, dst;
  CK(ds.alloc((size_t)n * dim, S(ctx)));
  CK(dg.alloc((size_t)n * dim, S(ctx)));
  CK(de.alloc(n, S(ctx)));
  CK(dit.alloc(n, S(ctx)));
  CK(dcv.alloc(n, S(ctx)));
  CK(dst.alloc(n, S(ctx)));
  CK(cudaMemsetAsync(dst.p, 0, sizeof(int) * n, S(ctx)));
  CK(cudaMemcpyAsync(ds.p, starts, sizeof(double) * n * dim, cudaMemcpyHostToDevice, S(ctx)));
  if (int rc = mdr_local_search_dev(ctx, ig.di, ds.p, n, max_iters, tol, method, accum, partition, dg.p, de.p, dit.p,
                                    dcv.p, dst.p))
    return rc;
  std::vector<int> status(n);
  CK(cudaMemcpyAsync(out_g, dg.p, sizeof(double) * n * dim, cudaMemcpyDeviceToHost, S(ctx)));
  CK(cudaMemcpyAsync(out_e, de.p, sizeof(double) * n, cudaMemcpyDeviceToHost, S(ctx)));
  CK(cudaMemcpyAsync(out_it, dit.p, sizeof(int) * n, cudaMemcpyDeviceToHost, S(ctx)));
  CK(cudaMemcpyAsync(out_cv, dcv.p, sizeof(int) * n, cudaMemcpyDeviceToHost, S(ctx)));
  CK(cudaMemcpyAsync(status.data(), dst.p, sizeof(int) * n, cudaMemcpyDeviceToHost, S(ctx)));
  CK(cudaStreamSynchronize(S(ctx)));
  for (int i = 0; i < n; ++i)
    if (status[i] != MDR_OK) return fail(ctx, status[i], "adadelta_step: non-finite gradient component");
  if (st) {
    const mdr_sync_stats one = score_stats(method, accum, partition);
    for (int i = 0; i < n; ++i) {
      st_zero(&st[i]);
      st_add(&st[i], one, (uint64_t)out_it[i] + 1);
    }
  }
  return MDR_OK;
}

// ---------------------------------------------------------------- LGA
void mdr_lga_defaults(mdr_lga_settings* s) {  // docking.hpp:106-115
  s->population_size = 36;
  s->generations = 20;
  s->max_evaluations = 100000;
  s->ls_fraction = 0.25;
  s->ls_max_iters = 150;
  s->partition = 64;
  s->ls_convergence_tol = 1e-4;
  s->mutation_sigma = 0.3;
}

static int ls_count_of(const mdr_lga_settings* s) {  // docking.cpp:424-426
  const int off = s->population_size - 1;
  return std::clamp(static_cast<int>(std::ceil(s->ls_fraction * off)), 0, off);
}

int mdr_lga_max_records(const mdr_lga_settings* s) { return s->generations * ls_count_of(s) + 1; }

struct mdr_lga_batch {
  LgaDev D{};
  LigandView L{};
  int method = 0, pair = 0, accum = 0;
  void* block = nullptr;
  uint64_t* seeds = nullptr;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  cudaStream_t captured_on = nullptr;
  int launches = 0;
  int cta_warps = 0;
  mdr_lga_settings settings{};
  bool grid = false;
  GridView G{};
  GridLigands GL{};    // device tables (one ligand, or a screen batch)
  void* gl_block = nullptr;
  size_t gsm = 0;      // dynamic shared memory of the grid kernels
  int gmethod = 0;     // grid kernels' method (kGridStrictMethod: strict FP64 path)
};

static uint64_t mix64_host(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

static uint64_t label_hash(const char* label) {  // mix64(fnv1a64(label)), rng.cpp:11-32
  uint64_t h = 0xcbf29ce484222325ull;
  for (const unsigned char* p = reinterpret_cast<const unsigned char*>(label); *p; ++p) h = (h ^ *p) * 0x100000001b3ull;
  return mix64_host(h);
}

int mdr_fill_uniform_dev(mdr_ctx* ctx, uint64_t seed, const char* label, int64_t n, float* d_out) {
  if (!ctx || !label || n < 0 || (n && !d_out)) return fail(ctx, MDR_ERR_INVALID, "bad argument");
  CK(launch_fill_uniform(mix64_host(seed ^ label_hash(label)), (long long)n, d_out, S(ctx)));  // rng.cpp:31-32
  ctx->launches++;
  return MDR_OK;
}

static int check_lga(mdr_ctx* ctx, int method, const mdr_lga_settings* s) {
  if (!s) return fail(ctx, MDR_ERR_INVALID, "null settings");
  if (s->population_size < 2) return fail(ctx, MDR_ERR_SIZE, "lga_run needs a population of at least 2");
  if (s->generations < 0 || s->ls_max_iters < 0) return fail(ctx, MDR_ERR_INVALID, "negative generations/iters");
  return check_partition(ctx, s->partition, method);
}

// Device state of R runs with genotype stride `dim` (zero-initialised).
static mdr_lga_batch* lga_batch_alloc(mdr_ctx* ctx, int method, int accum, const mdr_lga_settings* s, int R,
                                      int dim) {
  mdr_lga_batch* b = new mdr_lga_batch;
  b->method = method;
  b->pair = ctx->pair;
  b->accum = accum;
  b->settings = *s;
  LgaDev& D = b->D;
  D.R = R;
  D.P = s->population_size;
  D.dim = dim;
  D.off = D.P - 1;
  D.L = ls_count_of(s);
  D.gens = s->generations;
  D.ls_iters = s->ls_max_iters;
  D.maxrec = mdr_lga_max_records(s);
  D.partition = s->partition;
  D.half_mode = accum == MDR_ACCUM_HALF;
  D.max_evals = s->max_evaluations;
  D.tol = s->ls_convergence_tol;
  D.sigma = s->mutation_sigma;
  D.label_hash = label_hash("lga");
  const size_t dm = D.dim, P = D.P, L = std::max(D.L, 1), Rr = R;
  auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
  size_t off = 0;
  std::vector<std::pair<void**, size_t>> parts;
  double *pop0, *pop1, *pe0, *pe1;
  parts.push_back({(void**)&pop0, sizeof(double) * Rr * P * dm});
  parts.push_back({(void**)&pop1, sizeof(double) * Rr * P * dm});
  parts.push_back({(void**)&pe0, sizeof(double) * Rr * P});
  parts.push_back({(void**)&pe1, sizeof(double) * Rr * P});
  parts.push_back({(void**)&D.cur, sizeof(int) * Rr});
  parts.push_back({(void**)&D.lsg, sizeof(double) * Rr * L * dm});
  parts.push_back({(void**)&D.lse, sizeof(double) * Rr * L});
  parts.push_back({(void**)&D.lsit, sizeof(int) * Rr * L});
  parts.push_back({(void**)&D.lscv, sizeof(int) * Rr * L});
  parts.push_back({(void**)&D.lstarget, sizeof(int) * Rr * L});
  parts.push_back({(void**)&D.best_e, sizeof(double) * Rr});
  parts.push_back({(void**)&D.best_g, sizeof(double) * Rr * dm});
  parts.push_back({(void**)&D.evals, sizeof(long long) * Rr});
  parts.push_back({(void**)&D.active, sizeof(int) * Rr});
  parts.push_back({(void**)&D.nrec, sizeof(int) * Rr});
  parts.push_back({(void**)&D.recs, sizeof(mdr_ls_record) * Rr * D.maxrec});
  parts.push_back({(void**)&D.conv, sizeof(int) * Rr});
  parts.push_back({(void**)&D.status, sizeof(int) * Rr});
  parts.push_back({(void**)&D.ls_next, sizeof(int) * (size_t)(D.gens + 1)});
  parts.push_back({(void**)&D.ls_done, sizeof(int) * Rr});
  parts.push_back({(void**)&b->seeds, sizeof(uint64_t) * Rr});
  for (auto& p : parts) off += al(p.second);
  if (cudaMalloc(&b->block, off) != cudaSuccess || cudaMemset(b->block, 0, off) != cudaSuccess) {
    fail(ctx, MDR_ERR_CUDA, "cudaMalloc failed for LGA batch");
    if (b->block) cudaFree(b->block);
    delete b;
    return nullptr;
  }
  off = 0;
  for (auto& p : parts) {
    *p.first = static_cast<char*>(b->block) + off;
    off += al(p.second);
  }
  D.pop[0] = pop0;
  D.pop[1] = pop1;
  D.pope[0] = pe0;
  D.pope[1] = pe1;
  D.seeds = b->seeds;
  return b;
}

static void lga_batch_release(mdr_lga_batch* b) {
  if (b->exec) cudaGraphExecDestroy(b->exec);
  if (b->graph) cudaGraphDestroy(b->graph);
  if (b->gl_block) cudaFree(b->gl_block);
  cudaFree(b->block);
  delete b;
}

// Enqueue the whole docking of a batch on stream s (graph capture or a
// profiling replay with events).
static cudaError_t lga_batch_enqueue(mdr_lga_batch* b, cudaStream_t s, int wpb, int* launches,
                                     cudaEvent_t* ev = nullptr) {
  if (b->grid) return launch_grid_lga(b->GL, b->gsm, b->G, b->D, b->gmethod, b->D.partition, s, launches, ev);
  return launch_lga(b->L, b->D, b->method, b->pair, s, wpb, b->cta_warps, launches, ev);
}

mdr_lga_batch* mdr_lga_batch_create(mdr_ctx* ctx, const mdr_dev_instance* di, int method, int accum,
                                    const mdr_lga_settings* s, int R) {
  if (!ctx || !di || R <= 0) {
    fail(ctx, MDR_ERR_INVALID, "bad argument");
    return nullptr;
  }
  if (check_lga(ctx, method, s)) return nullptr;
  if (di->grid && check_grid_block(ctx, di, s->partition)) return nullptr;
  if (check_exact(ctx, di)) return nullptr;
  mdr_lga_batch* b = lga_batch_alloc(ctx, method, accum, s, R, 6 + di->n_rot);
  if (!b) return nullptr;
  b->L = di->grid ? di->view : launch_view(ctx, di);
  b->cta_warps = cta_warps_for(ctx);
  b->grid = di->grid;
  cudaError_t e = cudaSuccess;
  if (b->grid) {
    b->G = di->gview;
    e = cudaMalloc(&b->gl_block, 256 + sizeof(FlexView));
    if (e == cudaSuccess) e = cudaMemcpy(b->gl_block, &di->view, sizeof(LigandView), cudaMemcpyHostToDevice);
    if (e == cudaSuccess)
      e = cudaMemcpy(static_cast<char*>(b->gl_block) + 256, &di->flex, sizeof(FlexView), cudaMemcpyHostToDevice);
    b->GL.L = static_cast<const LigandView*>(b->gl_block);
    b->GL.F = reinterpret_cast<const FlexView*>(static_cast<char*>(b->gl_block) + 256);
    b->GL.run_lig = nullptr;
    b->gmethod = grid_method(ctx, method);
    b->gsm = grid_smem_for(di->view, di->flex, s->partition, b->gmethod);
    if (e == cudaSuccess) e = prepare_grid_lga(b->gsm, b->gmethod);
  } else {
    e = prepare_lga(b->L, method, b->pair, ctx->wpb, b->cta_warps);
  }
  // capture the whole docking (init, gens x {offspring, LS, finalize}, polish)
  // into one CUDA graph, replayed per call
  cudaStream_t cs = nullptr;
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal);
  if (e == cudaSuccess) {
    e = lga_batch_enqueue(b, cs, ctx->wpb, &b->launches);
    cudaGraph_t g = nullptr;
    const cudaError_t e2 = cudaStreamEndCapture(cs, &g);
    if (e == cudaSuccess) e = e2;
    b->graph = g;
    if (e == cudaSuccess) e = cudaGraphInstantiate(&b->exec, g, 0);
  }
  if (cs) cudaStreamDestroy(cs);
  if (e != cudaSuccess) {
    cuda_fail(ctx, e, "LGA graph capture");
    lga_batch_release(b);
    return nullptr;
  }
  return b;
}

void mdr_lga_batch_destroy(mdr_ctx* ctx, mdr_lga_batch* b) {
  if (!b) return;
  if (ctx) cudaStreamSynchronize(ctx->stream);
  lga_batch_release(b);
}

int mdr_lga_batch_run_dev(mdr_ctx* ctx, mdr_lga_batch* b, const uint64_t* d_seeds) {
  if (!ctx || !b || !d_seeds) return fail(ctx, MDR_ERR_INVALID, "bad argument");
  CK(cudaMemcpyAsync(b->seeds, d_seeds, sizeof(uint64_t) * b->D.R, cudaMemcpyDeviceToDevice, ctx->stream));
  CK(cudaGraphLaunch(b->exec, ctx->stream));
  ctx->launches += (uint64_t)b->launches;
  return MDR_OK;
}

int mdr_lga_batch_profile_dev(mdr_ctx* ctx, mdr_lga_batch* b, const uint64_t* d_seeds, float* ls_ms,
                              float* step_ms, int64_t* ls_evals) {
  if (!ctx || !b || !d_seeds) return fail(ctx, MDR_ERR_INVALID, "bad argument");
  const LgaDev& D = b->D;
  const int ne = 2 * D.gens + 4;
  std::vector<cudaEvent_t> ev(ne);
  for (auto& e : ev) CK(cudaEventCreate(&e));
  CK(cudaMemcpyAsync(b->seeds, d_seeds, sizeof(uint64_t) * D.R, cudaMemcpyDeviceToDevice, ctx->stream));
  int launches = 0;
  CK(lga_batch_enqueue(b, ctx->stream, ctx->wpb, &launches, ev.data()));
  ctx->launches += (uint64_t)launches;
  CK(cudaStreamSynchronize(ctx->stream));
  float tot = 0.f, t = 0.f;
  for (int g = 0; g <= D.gens; ++g) {
    CK(cudaEventElapsedTime(&t, ev[2 * g], ev[2 * g + 1]));
    tot += t;
  }
  CK(cudaEventElapsedTime(&t, ev[2 * D.gens + 2], ev[2 * D.gens + 3]));
  for (auto& e : ev) cudaEventDestroy(e);
  if (ls_ms) *ls_ms = tot;
  if (step_ms) *step_ms = t;
  if (ls_evals) {
    std::vector<mdr_ls_record> recs((size_t)D.R * D.maxrec);
    std::vector<int> nrec(D.R);
    CK(cudaMemcpy(recs.data(), D.recs, sizeof(mdr_ls_record) * recs.size(), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(nrec.data(), D.nrec, sizeof(int) * D.R, cudaMemcpyDeviceToHost));
    int64_t s = 0;
    for (int r = 0; r < D.R; ++r)
      for (int k = 0; k < std::min(nrec[r], D.maxrec); ++k) s += recs[(size_t)r * D.maxrec + k].iterations + 1;
    *ls_evals = s;
  }
  return MDR_OK;
}

int mdr_lga_batch_total_evals_dev(mdr_ctx* ctx, mdr_lga_batch* b, int64_t* d_total) {
  if (!ctx || !b || !d_total) return fail(ctx, MDR_ERR_INVALID, "bad argument");
  CK(launch_lga_total(b->D, reinterpret_cast<long long*>(d_total), ctx->stream));
  ctx->launches++;
  return MDR_OK;
}

int mdr_lga_batch_download(mdr_ctx* ctx, mdr_lga_batch* b, double* best_e, double* best_g, int64_t* evals,
                           int32_t* conv, int32_t* n_records, mdr_ls_record* records, mdr_sync_stats* total) {
  if (!ctx || !b) return fail(ctx, MDR_ERR_INVALID, "bad argument");
  const LgaDev& D = b->D;
  std::vector<int> status(D.R);
  if (best_e) CK(cudaMemcpyAsync(best_e, D.best_e, sizeof(double) * D.R, cudaMemcpyDeviceToHost, ctx->stream));
  if (best_g)
    CK(cudaMemcpyAsync(best_g, D.best_g, sizeof(double) * D.R * D.dim, cudaMemcpyDeviceToHost, ctx->stream));
  std::vector<long long> ev(D.R);
  CK(cudaMemcpyAsync(ev.data(), D.evals, sizeof(long long) * D.R, cudaMemcpyDeviceToHost, ctx->stream));
  if (conv) CK(cudaMemcpyAsync(conv, D.conv, sizeof(int) * D.R, cudaMemcpyDeviceToHost, ctx->stream));
  if (n_records) CK(cudaMemcpyAsync(n_records, D.nrec, sizeof(int) * D.R, cudaMemcpyDeviceToHost, ctx->stream));
  if (records)
    CK(cudaMemcpyAsync(records, D.recs, sizeof(mdr_ls_record) * D.R * D.maxrec, cudaMemcpyDeviceToHost,
                       ctx->stream));
  CK(cudaMemcpyAsync(status.data(), D.status, sizeof(int) * D.R, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  for (int r = 0; r < D.R; ++r) {
    if (evals) evals[r] = ev[r];
    if (total) {
      st_zero(&total[r]);
      st_add(&total[r], score_stats(b->method, b->accum, D.partition), (uint64_t)ev[r]);
    }
  }
  for (int r = 0; r < D.R; ++r)
    if (status[r] != MDR_OK) return fail(ctx, status[r], "adadelta_step: non-finite gradient component");
  return MDR_OK;
}

int mdr_lga_run_batch(mdr_ctx* ctx, const mdr_instance* inst, int method, int accum, const mdr_lga_settings* s,
                      const uint64_t* seeds, int n_runs, double* best_e, double* best_g, int64_t* evals,
                      int32_t* conv, int32_t* n_records, mdr_ls_record* records, mdr_sync_stats* total) {
  if (!ctx || n_runs < 0 || (n_runs && !seeds)) return fail(ctx, MDR_ERR_INVALID, "bad argument");
  if (int rc = check_instance(ctx, inst)) return rc;
  if (int rc = check_lga(ctx, method, s)) return rc;
  if (n_runs == 0) return MDR_OK;
  LgaCache& c = ctx->lga;
  const bool hit = c.b && c.b->cta_warps == cta_warps_for(ctx) && c.b->L.exact_torsion == ctx->exact && c.b->L.ls_warps == ctx->ls_warps && c.b->L.ls_pair == ctx->ls_pair && c.na == inst->n_atoms && c.ns == inst->n_sites && c.nr == inst->n_rot &&
                   c.method == method && c.pair == ctx->pair && c.accum == accum && c.wpb == ctx->wpb &&
                   c.R == n_runs && std::memcmp(&c.s, s, sizeof *s) == 0;
  if (hit) {
    if (int rc = write_instance(ctx, c.di, inst)) return rc;
  } else {
    mdr_lga_batch_destroy(ctx, c.b);
    mdr_instance_free(ctx, c.di);
    c = LgaCache{};
    c.di = mdr_instance_upload(ctx, inst);
    if (!c.di) return MDR_ERR_CUDA;
    c.b = mdr_lga_batch_create(ctx, c.di, method, accum, s, n_runs);
    if (!c.b) return MDR_ERR_CUDA;
    c.na = inst->n_atoms;
    c.ns = inst->n_sites;
    c.nr = inst->n_rot;
    c.method = method;
    c.pair = ctx->pair;
    c.accum = accum;
    c.wpb = ctx->wpb;
    c.R = n_runs;
    c.s = *s;
  }
  mdr_lga_batch* b = c.b;
  CK(cudaMemcpyAsync(b->seeds, seeds, sizeof(uint64_t) * n_runs, cudaMemcpyHostToDevice, S(ctx)));
  CK(cudaGraphLaunch(b->exec, S(ctx)));
  ctx->launches += (uint64_t)b->launches;
  return mdr_lga_batch_download(ctx, b, best_e, best_g, evals, conv, n_records, records, total);
}

// ---------------------------------------------------------------- grid mode
static int check_grid_shape(mdr_ctx* ctx, const mdr_grid* g) {
  if (!g) return fail(ctx, MDR_ERR_INVALID, "null grid");
  if (g->nx < 2 || g->ny < 2 || g->nz < 2 || g->n_types < 1 || !(g->spacing > 0.0))
    return fail(ctx, MDR_ERR_SIZE, "grid needs >= 2 points per axis, >= 1 type map and spacing > 0");
  if ((long long)g->nx * g->ny * g->nz > (1ll << 31) / (g->n_types + 2))
    return fail(ctx, MDR_ERR_SIZE, "grid too large");
  return MDR_OK;
}

static mdr_dev_grid* grid_alloc(mdr_ctx* ctx, const mdr_grid* g) {
  mdr_dev_grid* d = new mdr_dev_grid;
  GridView& v = d->view;
  v.nx = g->nx;
  v.ny = g->ny;
  v.nz = g->nz;
  v.n_types = g->n_types;
  v.ox = g->origin[0];
  v.oy = g->origin[1];
  v.oz = g->origin[2];
  v.h = g->spacing;
  v.inv_h = 1.0 / g->spacing;
  v.stride = (long long)g->nx * g->ny * g->nz;
  if (cudaMalloc(&d->maps, sizeof(float) * (size_t)v.stride * (g->n_types + 2)) != cudaSuccess) {
    fail(ctx, MDR_ERR_CUDA, "cudaMalloc failed for grid maps");
    delete d;
    return nullptr;
  }
  v.maps = d->maps;
  return d;
}

mdr_dev_grid* mdr_grid_upload(mdr_ctx* ctx, const mdr_grid* g) {
  if (!ctx || check_grid_shape(ctx, g)) return nullptr;
  if (!g->maps) {
    fail(ctx, MDR_ERR_INVALID, "null maps");
    return nullptr;
  }
  mdr_dev_grid* d = grid_alloc(ctx, g);
  if (!d) return nullptr;
  const size_t bytes = sizeof(float) * (size_t)d->view.stride * (g->n_types + 2);
  if (cudaMemcpyAsync(d->maps, g->maps, bytes, cudaMemcpyHostToDevice, ctx->stream) != cudaSuccess ||
      cudaStreamSynchronize(ctx->stream) != cudaSuccess) {
    fail(ctx, MDR_ERR_CUDA, "grid upload failed");
    mdr_grid_free(ctx, d);
    return nullptr;
  }
  return d;
}

mdr_dev_grid* mdr_grid_build(mdr_ctx* ctx, const mdr_instance* sites, const mdr_receptor_fields* f,
                             const mdr_grid* shape) {
  if (!ctx || check_grid_shape(ctx, shape)) return nullptr;
  if (!sites || !f || !sites->site_xyzdd || sites->n_sites < 1 || !f->site_charge || !f->site_volume ||
      !f->type_depth_scale || !f->type_dist_scale || !(f->desolv_sigma > 0.0)) {
    fail(ctx, MDR_ERR_INVALID, "bad receptor fields");
    return nullptr;
  }
  mdr_dev_grid* d = grid_alloc(ctx, shape);
  if (!d) return nullptr;
  const int ns = sites->n_sites, nt = shape->n_types;
  double* buf = nullptr;
  const size_t nd = 5 * (size_t)ns + 2 * (size_t)ns + 2 * (size_t)nt;
  cudaError_t e = cudaMallocAsync(&buf, sizeof(double) * nd, ctx->stream);
  std::vector<double> h(nd);
  std::memcpy(h.data(), sites->site_xyzdd, sizeof(double) * 5 * ns);
  std::memcpy(h.data() + 5 * ns, f->site_charge, sizeof(double) * ns);
  std::memcpy(h.data() + 6 * ns, f->site_volume, sizeof(double) * ns);
  std::memcpy(h.data() + 7 * ns, f->type_depth_scale, sizeof(double) * nt);
  std::memcpy(h.data() + 7 * ns + nt, f->type_dist_scale, sizeof(double) * nt);
  if (e == cudaSuccess) e = cudaMemcpyAsync(buf, h.data(), sizeof(double) * nd, cudaMemcpyHostToDevice, ctx->stream);
  if (e == cudaSuccess)
    e = launch_grid_build(d->view, buf, ns, buf + 5 * ns, buf + 6 * ns, buf + 7 * ns, buf + 7 * ns + nt,
                          f->elec_scale, f->desolv_sigma, d->maps, ctx->stream);
  if (e == cudaSuccess) ctx->launches++;
  if (buf) cudaFreeAsync(buf, ctx->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
  if (e != cudaSuccess) {
    cuda_fail(ctx, e, "mdr_grid_build");
    mdr_grid_free(ctx, d);
    return nullptr;
  }
  return d;
}

int mdr_grid_download(mdr_ctx* ctx, const mdr_dev_grid* d, float* maps) {
  if (!ctx || !d || !maps) return fail(ctx, MDR_ERR_INVALID, "bad argument");
  CK(cudaMemcpyAsync(maps, d->maps, sizeof(float) * (size_t)d->view.stride * (d->view.n_types + 2),
                     cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return MDR_OK;
}

void mdr_grid_free(mdr_ctx* ctx, mdr_dev_grid* d) {
  if (!d) return;
  if (ctx) cudaStreamSynchronize(ctx->stream);
  cudaFree(d->maps);
  delete d;
}

// Host preparation of the grid-mode chemistry (FlexView): per-atom
// {radius, sqrt(epsilon), q, k_e q} and the torsion-group CSR.
static int prep_flex(mdr_ctx* ctx, int na, int nr, const int* tors, const mdr_ligand_params* p, int n_types,
                     std::vector<int>& type, std::vector<float4>& chem, std::vector<int>& off,
                     std::vector<int>& members, std::vector<double4>* chem64 = nullptr) {
  if (!p || !p->atom_type || !p->atom_charge || !p->atom_radius || !p->atom_epsilon)
    return fail(ctx, MDR_ERR_INVALID, "null ligand parameters");
  type.assign(na, 0);
  chem.assign(na, float4{});
  for (int i = 0; i < na; ++i) {
    if (p->atom_type[i] < 0 || p->atom_type[i] >= n_types)
      return fail(ctx, MDR_ERR_SIZE, "atom type outside [0, n_types)");
    if (!(p->atom_epsilon[i] >= 0.0) || !std::isfinite(p->atom_charge[i]) || !std::isfinite(p->atom_radius[i]))
      return fail(ctx, MDR_ERR_NUMERIC_DOMAIN, "non-finite or negative ligand parameter");
    type[i] = p->atom_type[i];
    chem[i] = make_float4((float)p->atom_radius[i], (float)std::sqrt(p->atom_epsilon[i]), (float)p->atom_charge[i],
                          (float)(p->elec_scale * p->atom_charge[i]));
    if (chem64) {
      if (i == 0) chem64->assign(na, double4{});
      (*chem64)[i] = make_double4(p->atom_radius[i], p->atom_epsilon[i], p->atom_charge[i], 0.0);
    }
  }
  off.assign(nr + 1, 0);
  members.clear();
  for (int k = 0; k < nr; ++k) {
    off[k] = (int)members.size();
    for (int i = 0; i < na; ++i)
      if (tors[i] == k) members.push_back(i);
  }
  off[nr] = (int)members.size();
  return MDR_OK;
}

int mdr_instance_set_grid(mdr_ctx* ctx, mdr_dev_instance* di, const mdr_dev_grid* g, const mdr_ligand_params* p) {
  if (!ctx || !di) return fail(ctx, MDR_ERR_INVALID, "bad argument");
  if (!g) {
    di->grid = false;
    return MDR_OK;
  }
  const int na = di->n_atoms, nr = di->n_rot;
  std::vector<int> tors(na), type, off, members;
  std::vector<float4> chem;
  std::vector<double4> chem64;
  CK(cudaMemcpy(tors.data(), di->view.tors, sizeof(int) * na, cudaMemcpyDeviceToHost));
  if (int rc = prep_flex(ctx, na, nr, tors.data(), p, g->view.n_types, type, chem, off, members, &chem64)) return rc;
  const int nta = (int)members.size();
  auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
  const size_t o_type = 0, o_chem = al(sizeof(int) * na), o_off = o_chem + al(sizeof(float4) * na),
               o_mem = o_off + al(sizeof(int) * (nr + 1)), o_c64 = o_mem + al(sizeof(int) * std::max(nta, 1)),
               total = o_c64 + al(sizeof(double4) * std::max(na, 1));
  if (di->flex_block) {
    CK(cudaStreamSynchronize(ctx->stream));
    cudaFree(di->flex_block);
    di->flex_block = nullptr;
  }
  CK(cudaMalloc(&di->flex_block, total));
  char* b = static_cast<char*>(di->flex_block);
  CK(cudaMemcpy(b + o_type, type.data(), sizeof(int) * na, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(b + o_chem, chem.data(), sizeof(float4) * na, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(b + o_off, off.data(), sizeof(int) * (nr + 1), cudaMemcpyHostToDevice));
  if (nta) CK(cudaMemcpy(b + o_mem, members.data(), sizeof(int) * nta, cudaMemcpyHostToDevice));
  if (na) CK(cudaMemcpy(b + o_c64, chem64.data(), sizeof(double4) * na, cudaMemcpyHostToDevice));
  FlexView& F = di->flex;
  F.chem64 = reinterpret_cast<const double4*>(b + o_c64);
  F.elec_scale = p->elec_scale;
  F.type = reinterpret_cast<const int*>(b + o_type);
  F.chem = reinterpret_cast<const float4*>(b + o_chem);
  F.grp_off = reinterpret_cast<const int*>(b + o_off);
  F.grp_atoms = reinterpret_cast<const int*>(b + o_mem);
  F.n_tors_atoms = nta;
  F.intra = p->intra != 0;
  di->gview = g->view;
  di->grid = true;
  return MDR_OK;
}

namespace {
struct GridLigand {  // a per-call device ligand switched to grid mode
  mdr_ctx* ctx;
  mdr_dev_instance* di = nullptr;
  ~GridLigand() { mdr_instance_free(ctx, di); }
};
int grid_ligand(mdr_ctx* ctx, GridLigand& gl, const mdr_dev_grid* g, const mdr_instance* inst,
                const mdr_ligand_params* p) {
  if (!g) return fail(ctx, MDR_ERR_INVALID, "null grid");
  if (int rc = check_instance(ctx, inst)) return rc;
  gl.di = mdr_instance_upload(ctx, inst);
  if (!gl.di) return MDR_ERR_CUDA;
  return mdr_instance_set_grid(ctx, gl.di, g, p);
}
}  // namespace

int mdr_grid_score_batch(mdr_ctx* ctx, const mdr_dev_grid* g, const mdr_instance* inst, const mdr_ligand_params* p,
                         const double* genos, int n, int method, int partition, float* energy, float* gradient,
                         float* torque) {
  if (!ctx || n < 0 || (n && (!genos || !energy || !gradient || !torque)))
    return fail(ctx, MDR_ERR_INVALID, "bad argument");
  GridLigand gl{ctx};
  if (int rc = grid_ligand(ctx, gl, g, inst, p)) return rc;
  if (int rc = check_partition(ctx, partition, method)) return rc;
  if (int rc = check_grid_block(ctx, gl.di, partition)) return rc;
  if (n == 0) return MDR_OK;
  const int dim = 6 + inst->n_rot;
  DevBuf<double> dg;
  DevBuf<float> de, dgr, dt;
  CK(dg.alloc((size_t)n * dim, S(ctx)));
  CK(de.alloc(n, S(ctx)));
  CK(dgr.alloc((size_t)n * dim, S(ctx)));
  CK(dt.alloc((size_t)n * 3, S(ctx)));
  CK(cudaMemcpyAsync(dg.p, genos, sizeof(double) * n * dim, cudaMemcpyHostToDevice, S(ctx)));
  if (int rc = mdr_score_dev(ctx, gl.di, dg.p, n, method, MDR_ACCUM_SINGLE, partition, de.p, dgr.p, dt.p)) return rc;
  CK(cudaMemcpyAsync(energy, de.p, sizeof(float) * n, cudaMemcpyDeviceToHost, S(ctx)));
  CK(cudaMemcpyAsync(gradient, dgr.p, sizeof(float) * n * dim, cudaMemcpyDeviceToHost, S(ctx)));
  CK(cudaMemcpyAsync(torque, dt.p, sizeof(float) * n * 3, cudaMemcpyDeviceToHost, S(ctx)));
  CK(cudaStreamSynchronize(S(ctx)));
  return MDR_OK;
}

int mdr_grid_local_search_batch(mdr_ctx* ctx, const mdr_dev_grid* g, const mdr_instance* inst,
                                const mdr_ligand_params* p, const double* starts, int n, int max_iters, double tol,
                                int method, int partition, double* out_g, double* out_e, int32_t* out_it,
                                int32_t* out_cv) {
  if (!ctx || n < 0 || max_iters < 0 || (n && (!starts || !out_g || !out_e || !out_it || !out_cv)))
    return fail(ctx, MDR_ERR_INVALID, "bad argument");
  GridLigand gl{ctx};
  if (int rc = grid_ligand(ctx, gl, g, inst, p)) return rc;
  if (int rc = check_partition(ctx, partition, method)) return rc;
  if (int rc = check_grid_block(ctx, gl.di, partition)) return rc;
  if (n == 0) return MDR_OK;
  const int dim = 6 + inst->n_rot;
  DevBuf<double> ds, dg, de;
  DevBuf<int> dit, dcv, dst;
  CK(ds.alloc((size_t)n * dim, S(ctx)));
  CK(dg.alloc((size_t)n * dim, S(ctx)));
  CK(de.alloc(n, S(ctx)));
  CK(dit.alloc(n, S(ctx)));
  CK(dcv.alloc(n, S(ctx)));
  CK(dst.alloc(n, S(ctx)));
  CK(cudaMemsetAsync(dst.p, 0, sizeof(int) * n, S(ctx)));
  CK(cudaMemcpyAsync(ds.p, starts, sizeof(double) * n * dim, cudaMemcpyHostToDevice, S(ctx)));
  if (int rc = mdr_local_search_dev(ctx, gl.di, ds.p, n, max_iters, tol, method, MDR_ACCUM_SINGLE, partition, dg.p,
                                    de.p, dit.p, dcv.p, dst.p))
    return rc;
  std::vector<int> status(n);
  CK(cudaMemcpyAsync(out_g, dg.p, sizeof(double) * n * dim, cudaMemcpyDeviceToHost, S(ctx)));
  CK(cudaMemcpyAsync(out_e, de.p, sizeof(double) * n, cudaMemcpyDeviceToHost, S(ctx)));
  CK(cudaMemcpyAsync(out_it, dit.p, sizeof(int) * n, cudaMemcpyDeviceToHost, S(ctx)));
  CK(cudaMemcpyAsync(out_cv, dcv.p, sizeof(int) * n, cudaMemcpyDeviceToHost, S(ctx)));
  CK(cudaMemcpyAsync(status.data(), dst.p, sizeof(int) * n, cudaMemcpyDeviceToHost, S(ctx)));
  CK(cudaStreamSynchronize(S(ctx)));
  for (int i = 0; i < n; ++i)
    if (status[i] != MDR_OK) return fail(ctx, status[i], "adadelta_step: non-finite gradient component");
  return MDR_OK;
}

int mdr_grid_lga_run_batch(mdr_ctx* ctx, const mdr_dev_grid* g, const mdr_instance* inst,
                           const mdr_ligand_params* p, int method, const mdr_lga_settings* s, const uint64_t* seeds,
                           int n_runs, double* best_e, double* best_g, int64_t* evals, int32_t* conv,
                           int32_t* n_records, mdr_ls_record* records) {
  if (!ctx || n_runs < 0 || (n_runs && !seeds)) return fail(ctx, MDR_ERR_INVALID, "bad argument");
  GridLigand gl{ctx};
  if (int rc = grid_ligand(ctx, gl, g, inst, p)) return rc;
  if (int rc = check_lga(ctx, method, s)) return rc;
  if (n_runs == 0) return MDR_OK;
  mdr_lga_batch* b = mdr_lga_batch_create(ctx, gl.di, method, MDR_ACCUM_SINGLE, s, n_runs);
  if (!b) return MDR_ERR_CUDA;
  int rc = MDR_OK;
  if (cudaMemcpyAsync(b->seeds, seeds, sizeof(uint64_t) * n_runs, cudaMemcpyHostToDevice, S(ctx)) != cudaSuccess ||
      cudaGraphLaunch(b->exec, S(ctx)) != cudaSuccess)
    rc = fail(ctx, MDR_ERR_CUDA, "grid LGA launch failed");
  if (rc == MDR_OK) {
    ctx->launches += (uint64_t)b->launches;
    rc = mdr_lga_batch_download(ctx, b, best_e, best_g, evals, conv, n_records, records, nullptr);
  }
  mdr_lga_batch_destroy(ctx, b);
  return rc;
}

// ---------------------------------------------------------------- screen
int mdr_grid_screen_batch(mdr_ctx* ctx, const mdr_dev_grid* g, const mdr_instance* ligs,
                          const mdr_ligand_params* params, int n_lig, int runs, int method, const mdr_lga_settings* s,
                          const uint64_t* seeds, double tol, double* best_e, double* best_g, int64_t* evals,
                          int32_t* conv, int32_t* cluster_of, double* rmsd, int32_t* n_clusters) {
  if (!ctx || !g || !ligs || !params || n_lig < 0 || runs < 0 || (n_lig && runs && !seeds))
    return fail(ctx, MDR_ERR_INVALID, "bad argument");
  if (int rc = check_lga(ctx, method, s)) return rc;
  if (n_lig == 0 || runs == 0) return MDR_OK;
  const int T = s->partition;
  static const bool timing = std::getenv("MDR_SCREEN_TIMING") != nullptr;  // host-pack / total split (stderr)
  const auto t_start = std::chrono::steady_clock::now();
  // ---- validate and pack every ligand into one host image of the device block
  struct Lay {
    size_t atoms, taxes, box, tors, type, chem, off, mem;
    int na, nr, nta;
  };
  std::vector<Lay> lay(n_lig);
  std::vector<char> img;
  auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
  auto put = [&](const void* src, size_t bytes, size_t reserve = 0) {  // reserve >= bytes of zeros
    const size_t o = img.size();
    img.resize(o + al(std::max(bytes, reserve)), 0);
    if (bytes) std::memcpy(img.data() + o, src, bytes);
    return o;
  };
  int max_dim = 6, max_na = 1;
  size_t max_smem = 0;
  for (int j = 0; j < n_lig; ++j) {
    const mdr_instance* in = &ligs[j];
    if (int rc = check_instance(ctx, in)) return rc;
    Lay& L = lay[j];
    L.na = in->n_atoms;
    L.nr = in->n_rot;
    if (T < 6 + L.nr) return fail(ctx, MDR_ERR_BLOCK_SIZE, "grid mode needs partition >= 6 + n_rot (one thread per dimension)");
    std::vector<int> type, off, members;
    std::vector<float4> chem;
    if (int rc = prep_flex(ctx, L.na, L.nr, in->atom_torsion, &params[j], g->view.n_types, type, chem, off, members))
      return rc;
    L.nta = (int)members.size();
    const size_t sm = grid_smem_for(L.na, L.nr, L.nta, T);  // screening: the FP32 grid path
    if (sm > 227 * 1024) return fail(ctx, MDR_ERR_SIZE, "grid-mode ligand does not fit in shared memory");
    max_smem = std::max(max_smem, sm);
    max_dim = std::max(max_dim, 6 + L.nr);
    max_na = std::max(max_na, L.na);
    std::vector<double> taxes(3 * (size_t)std::max(L.nr, 1), 0.0);
    for (int k = 0; k < L.nr; ++k) torsion_axis_host(k, &taxes[3 * k]);
    double box[6];
    genotype_box(in, box);
    L.atoms = put(in->atom_xyzw, sizeof(double) * 4 * L.na);
    L.taxes = put(taxes.data(), sizeof(double) * taxes.size());
    L.box = put(box, sizeof box);
    L.tors = put(in->atom_torsion, sizeof(int) * L.na);
    L.type = put(type.data(), sizeof(int) * L.na);
    L.chem = put(chem.data(), sizeof(float4) * L.na);
    L.off = put(off.data(), sizeof(int) * (L.nr + 1));
    L.mem = put(members.data(), sizeof(int) * L.nta, sizeof(int));
  }
  const int R = n_lig * runs;
  const size_t o_views = img.size();
  img.resize(o_views + al(sizeof(LigandView) * n_lig) + al(sizeof(FlexView) * n_lig) + al(sizeof(int) * R) +
                 al(sizeof(int) * (n_lig + 1)) + al(sizeof(int) * n_lig),
             0);
  const size_t o_flex = o_views + al(sizeof(LigandView) * n_lig), o_rl = o_flex + al(sizeof(FlexView) * n_lig),
               o_seg = o_rl + al(sizeof(int) * R), o_segna = o_seg + al(sizeof(int) * (n_lig + 1));
  mdr_lga_batch* b = lga_batch_alloc(ctx, method, MDR_ACCUM_SINGLE, s, R, max_dim);
  if (!b) return MDR_ERR_CUDA;
  struct Release {
    mdr_ctx* ctx;
    mdr_lga_batch* b;
    ~Release() { mdr_lga_batch_destroy(ctx, b); }
  } rel{ctx, b};
  CK(cudaMalloc(&b->gl_block, img.size()));
  char* base = static_cast<char*>(b->gl_block);
  {
    LigandView* lv = reinterpret_cast<LigandView*>(img.data() + o_views);
    FlexView* fv = reinterpret_cast<FlexView*>(img.data() + o_flex);
    int* rl = reinterpret_cast<int*>(img.data() + o_rl);
    int* seg = reinterpret_cast<int*>(img.data() + o_seg);
    int* segna = reinterpret_cast<int*>(img.data() + o_segna);
    for (int j = 0; j < n_lig; ++j) {
      const Lay& L = lay[j];
      LigandView v{};
      v.n_atoms = L.na;
      v.n_sites = 0;
      v.n_rot = L.nr;
      v.atoms = reinterpret_cast<const double4*>(base + L.atoms);
      v.taxes = reinterpret_cast<const double*>(base + L.taxes);
      v.tors = reinterpret_cast<const int*>(base + L.tors);
      v.box = reinterpret_cast<const double*>(base + L.box);
      lv[j] = v;
      FlexView f{};
      f.type = reinterpret_cast<const int*>(base + L.type);
      f.chem = reinterpret_cast<const float4*>(base + L.chem);
      f.grp_off = reinterpret_cast<const int*>(base + L.off);
      f.grp_atoms = reinterpret_cast<const int*>(base + L.mem);
      f.n_tors_atoms = L.nta;
      f.intra = params[j].intra != 0;
      fv[j] = f;
      for (int k = 0; k < runs; ++k) rl[j * runs + k] = j;
      seg[j] = j * runs;
      segna[j] = L.na;
    }
    seg[n_lig] = R;
  }
  const auto t_packed = std::chrono::steady_clock::now();
  CK(cudaMemcpyAsync(base, img.data(), img.size(), cudaMemcpyHostToDevice, S(ctx)));
  b->grid = true;
  b->G = g->view;
  b->GL.L = reinterpret_cast<const LigandView*>(base + o_views);
  b->GL.F = reinterpret_cast<const FlexView*>(base + o_flex);
  b->GL.run_lig = reinterpret_cast<const int*>(base + o_rl);
  b->gsm = max_smem;
  b->gmethod = method;  // screening runs the FP32 grid path
  CK(prepare_grid_lga(b->gsm, method));
  CK(cudaMemcpyAsync(b->seeds, seeds, sizeof(uint64_t) * R, cudaMemcpyHostToDevice, S(ctx)));
  int launches = 0;
  CK(lga_batch_enqueue(b, S(ctx), ctx->wpb, &launches));
  ctx->launches += (uint64_t)launches;
  // ---- per-ligand clustering of the best poses (one CTA per ligand)
  DevBuf<double> xyz, dr;
  DevBuf<int> dc, dn, order, sd;
  if (cluster_of || rmsd || n_clusters) {
    CK(xyz.alloc((size_t)R * 3 * max_na, S(ctx)));
    CK(dr.alloc(R, S(ctx)));
    CK(dc.alloc(R, S(ctx)));
    CK(dn.alloc(n_lig, S(ctx)));
    CK(order.alloc(R, S(ctx)));
    CK(sd.alloc(R, S(ctx)));
    CK(launch_pose_coords(b->GL.L, b->GL.run_lig, b->D.best_g, b->D.dim, R, 3ll * max_na, xyz.p, S(ctx)));
    CK(launch_cluster(xyz.p, 3ll * max_na, b->D.best_e, reinterpret_cast<const int*>(base + o_seg),
                      reinterpret_cast<const int*>(base + o_segna), n_lig, max_na, tol, dc.p, dr.p, dn.p, order.p,
                      sd.p, S(ctx)));
    ctx->launches += 2;
  }
  // ---- results
  std::vector<double> bg((size_t)R * b->D.dim);
  std::vector<int> status(R);
  std::vector<long long> ev(R);
  if (best_e) CK(cudaMemcpyAsync(best_e, b->D.best_e, sizeof(double) * R, cudaMemcpyDeviceToHost, S(ctx)));
  if (best_g) CK(cudaMemcpyAsync(bg.data(), b->D.best_g, sizeof(double) * bg.size(), cudaMemcpyDeviceToHost, S(ctx)));
  CK(cudaMemcpyAsync(ev.data(), b->D.evals, sizeof(long long) * R, cudaMemcpyDeviceToHost, S(ctx)));
  if (conv) CK(cudaMemcpyAsync(conv, b->D.conv, sizeof(int) * R, cudaMemcpyDeviceToHost, S(ctx)));
  CK(cudaMemcpyAsync(status.data(), b->D.status, sizeof(int) * R, cudaMemcpyDeviceToHost, S(ctx)));
  if (cluster_of) CK(cudaMemcpyAsync(cluster_of, dc.p, sizeof(int) * R, cudaMemcpyDeviceToHost, S(ctx)));
  if (rmsd) CK(cudaMemcpyAsync(rmsd, dr.p, sizeof(double) * R, cudaMemcpyDeviceToHost, S(ctx)));
  if (n_clusters) CK(cudaMemcpyAsync(n_clusters, dn.p, sizeof(int) * n_lig, cudaMemcpyDeviceToHost, S(ctx)));
  CK(cudaStreamSynchronize(S(ctx)));
  if (evals)
    for (int r = 0; r < R; ++r) evals[r] = ev[r];
  if (best_g) {
    size_t o = 0;
    for (int j = 0; j < n_lig; ++j) {
      const int dim = 6 + lay[j].nr;
      for (int k = 0; k < runs; ++k, o += dim)
        std::memcpy(best_g + o, bg.data() + (size_t)(j * runs + k) * b->D.dim, sizeof(double) * dim);
    }
  }
  if (timing) {
    const auto t_end = std::chrono::steady_clock::now();
    std::fprintf(stderr, "mdr_grid_screen_batch: %d ligands, host pack %.1f ms, total %.1f ms\n", n_lig,
                 std::chrono::duration<double, std::milli>(t_packed - t_start).count(),
                 std::chrono::duration<double, std::milli>(t_end - t_start).count());
  }
  for (int r = 0; r < R; ++r)
    if (status[r] != MDR_OK) return fail(ctx, status[r], "adadelta_step: non-finite gradient component");
  return MDR_OK;
}

// ---------------------------------------------------------------- clustering
int mdr_cluster_segments_dev(mdr_ctx* ctx, const mdr_dev_instance* di, const double* genos, const double* energy,
                             const int32_t* seg_off, int n_seg, int n_total, double tol, int32_t* cluster_of,
                             double* rmsd, int32_t* n_clusters) {
  if (!ctx || !di || n_seg < 0 || n_total < 0 || !(tol >= 0.0)) return fail(ctx, MDR_ERR_INVALID, "bad argument");
  if (n_seg == 0 || n_total == 0) return MDR_OK;
  DevBuf<double> xyz;
  DevBuf<int> order, seeds;
  DevBuf<LigandView> lv;
  CK(xyz.alloc((size_t)n_total * 3 * di->n_atoms, S(ctx)));
  CK(order.alloc(n_total, S(ctx)));
  CK(seeds.alloc(n_total, S(ctx)));
  CK(lv.alloc(1, S(ctx)));
  CK(cudaMemcpyAsync(lv.p, &di->view, sizeof(LigandView), cudaMemcpyHostToDevice, S(ctx)));
  const long long xs = 3ll * di->n_atoms;
  CK(launch_pose_coords(lv.p, nullptr, genos, 6 + di->n_rot, n_total, xs, xyz.p, S(ctx)));
  CK(launch_cluster(xyz.p, xs, energy, seg_off, nullptr, n_seg, di->n_atoms, tol, cluster_of, rmsd, n_clusters,
                    order.p, seeds.p, S(ctx)));
  CK(cudaStreamSynchronize(S(ctx)));  // the staged view dies at return
  ctx->launches += 2;
  return MDR_OK;
}

int mdr_pose_coords_batch(mdr_ctx* ctx, const mdr_instance* inst, const double* genos, int n, double* xyz) {
  if (!ctx || n < 0 || (n && (!genos || !xyz))) return fail(ctx, MDR_ERR_INVALID, "bad argument");
  if (int rc = check_instance(ctx, inst)) return rc;
  if (n == 0) return MDR_OK;
  InstanceGuard ig{ctx, mdr_instance_upload(ctx, inst)};
  if (!ig.di) return MDR_ERR_CUDA;
  const int dim = 6 + inst->n_rot;
  DevBuf<double> dg, dx;
  CK(dg.alloc((size_t)n * dim, S(ctx)));
  CK(dx.alloc((size_t)n * 3 * inst->n_atoms, S(ctx)));
  CK(cudaMemcpyAsync(dg.p, genos, sizeof(double) * n * dim, cudaMemcpyHostToDevice, S(ctx)));
  DevBuf<LigandView> lv;
  CK(lv.alloc(1, S(ctx)));
  CK(cudaMemcpyAsync(lv.p, &ig.di->view, sizeof(LigandView), cudaMemcpyHostToDevice, S(ctx)));
  CK(launch_pose_coords(lv.p, nullptr, dg.p, dim, n, 3ll * inst->n_atoms, dx.p, S(ctx)));
  ctx->launches++;
  CK(cudaMemcpyAsync(xyz, dx.p, sizeof(double) * n * 3 * inst->n_atoms, cudaMemcpyDeviceToHost, S(ctx)));
  CK(cudaStreamSynchronize(S(ctx)));
  return MDR_OK;
}

int mdr_cluster_poses(mdr_ctx* ctx, const mdr_instance* inst, const double* genos, const double* energies, int n,
                      double tol, int32_t* cluster_of, double* rmsd, int32_t* n_clusters) {
  if (!ctx || n < 0 || !n_clusters || (n && (!genos || !energies || !cluster_of))) 
    return fail(ctx, MDR_ERR_INVALID, "bad argument");
  if (!(tol >= 0.0)) return fail(ctx, MDR_ERR_INVALID, "rmsd tolerance must be >= 0");
  if (int rc = check_instance(ctx, inst)) return rc;
  *n_clusters = 0;
  if (n == 0) return MDR_OK;
  InstanceGuard ig{ctx, mdr_instance_upload(ctx, inst)};
  if (!ig.di) return MDR_ERR_CUDA;
  const int dim = 6 + inst->n_rot;
  DevBuf<double> dg, de, dr;
  DevBuf<int> dc, dn, doff;
  CK(dg.alloc((size_t)n * dim, S(ctx)));
  CK(de.alloc(n, S(ctx)));
  CK(dr.alloc(n, S(ctx)));
  CK(dc.alloc(n, S(ctx)));
  CK(dn.alloc(1, S(ctx)));
  CK(doff.alloc(2, S(ctx)));
  const int off[2] = {0, n};
  CK(cudaMemcpyAsync(dg.p, genos, sizeof(double) * n * dim, cudaMemcpyHostToDevice, S(ctx)));
  CK(cudaMemcpyAsync(de.p, energies, sizeof(double) * n, cudaMemcpyHostToDevice, S(ctx)));
  CK(cudaMemcpyAsync(doff.p, off, sizeof off, cudaMemcpyHostToDevice, S(ctx)));
  if (int rc = mdr_cluster_segments_dev(ctx, ig.di, dg.p, de.p, doff.p, 1, n, tol, dc.p, dr.p, dn.p)) return rc;
  CK(cudaMemcpyAsync(cluster_of, dc.p, sizeof(int) * n, cudaMemcpyDeviceToHost, S(ctx)));
  if (rmsd) CK(cudaMemcpyAsync(rmsd, dr.p, sizeof(double) * n, cudaMemcpyDeviceToHost, S(ctx)));
  CK(cudaMemcpyAsync(n_clusters, dn.p, sizeof(int), cudaMemcpyDeviceToHost, S(ctx)));
  CK(cudaStreamSynchronize(S(ctx)));
  return MDR_OK;
}

int mdr_lga_batch_cluster(mdr_ctx* ctx, mdr_lga_batch* b, double tol, int32_t* cluster_of, double* rmsd,
                          int32_t* n_clusters) {
  if (!ctx || !b || !cluster_of || !n_clusters) return fail(ctx, MDR_ERR_INVALID, "bad argument");
  const LgaDev& D = b->D;
  mdr_dev_instance view;  // the batch's ligand (LigandView copy; nothing owned)
  view.view = b->L;
  view.n_atoms = b->L.n_atoms;
  view.n_rot = b->L.n_rot;
  DevBuf<double> dr;
  DevBuf<int> dc, dn, doff;
  CK(dr.alloc(D.R, S(ctx)));
  CK(dc.alloc(D.R, S(ctx)));
  CK(dn.alloc(1, S(ctx)));
  CK(doff.alloc(2, S(ctx)));
  const int off[2] = {0, D.R};
  CK(cudaMemcpyAsync(doff.p, off, sizeof off, cudaMemcpyHostToDevice, S(ctx)));
  int rc = mdr_cluster_segments_dev(ctx, &view, D.best_g, D.best_e, doff.p, 1, D.R, tol, dc.p, dr.p, dn.p);
  view.block = nullptr;
  if (rc) return rc;
  CK(cudaMemcpyAsync(cluster_of, dc.p, sizeof(int) * D.R, cudaMemcpyDeviceToHost, S(ctx)));
  if (rmsd) CK(cudaMemcpyAsync(rmsd, dr.p, sizeof(double) * D.R, cudaMemcpyDeviceToHost, S(ctx)));
  CK(cudaMemcpyAsync(n_clusters, dn.p, sizeof(int), cudaMemcpyDeviceToHost, S(ctx)));
  CK(cudaStreamSynchronize(S(ctx)));
  return MDR_OK;
}

}  // extern "C"
