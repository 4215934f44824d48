// capi.cu -- the C ABI of libdsr.so (include/dsr.h): host layout, heap
// lifecycle, do-all orchestration, audit / statistics kernels.
#include <cstdio>
#include <cstring>
#include <cuda.h>   // driver types for entry points resolved at run time (no libcuda link dependency)
#include <new>
#include "dsr_host.h"
#include "dsr_doall.cuh"

#ifndef DSR_BUILD_INFO
#define DSR_BUILD_INFO "sm_100a"
#endif

#include <nvtx3/nvToolsExt.h>   // header-only NVTX: no-ops unless a profiler is attached
#include <algorithm>
#include <mutex>
#include <vector>
#include <unordered_map>

namespace dsr {
std::atomic<unsigned long long> g_launches{0};

int resident_ctas(const void* kernel, int threads) {
  static std::mutex mu;
  static std::unordered_map<const void*, int> cache;
  std::lock_guard<std::mutex> lock(mu);
  auto key = (const void*)((const char*)kernel + threads);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  int nb = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kernel, threads, 0) != cudaSuccess || nb < 1) nb = 1;
  cache[key] = nb;
  return nb;
}
}
using namespace dsr;

struct dsr_heap {
  dsr_layout L;
  dsr_type_desc types[DSR_MAX_TYPES];
  DevHeap dev;
  int device;
  int sms;
  // host-input staging (dsr_mb_new_args.in_host): two device buffers used
  // alternately, filled on a copy stream; `used` = the last kernel reading it
  void* stage[2] = {nullptr, nullptr};
  size_t stage_cap[2] = {0, 0};
  cudaEvent_t ready[2] = {nullptr, nullptr}, used[2] = {nullptr, nullptr};
  cudaStream_t cstream = nullptr;
  int stage_next = 0;
  ~dsr_heap() {
    for (int k = 0; k < 2; ++k) {
      if (stage[k]) cudaFree(stage[k]);
      if (ready[k]) cudaEventDestroy(ready[k]);
      if (used[k]) cudaEventDestroy(used[k]);
    }
    if (cstream) cudaStreamDestroy(cstream);
  }
};

#define CUDA_TRY(x)                                         \
  do {                                                      \
    cudaError_t e_ = (x);                                   \
    if (e_ != cudaSuccess) {                                \
      fprintf(stderr, "[dsr] %s: %s\n", #x, cudaGetErrorString(e_)); \
      return DSR_ERR_CUDA;                                  \
    }                                                       \
  } while (0)

// control page (4 KiB) + warp block-hint table: H hardware-warp slots x 8 types
// x u32, H = pow2floor(heap_bytes / 64 KiB) clamped to [64, 16384] (R-LAYOUT)
static uint64_t hint_slots(uint64_t heap_bytes) {
  uint64_t h = 64;
  while (h * 2 <= (heap_bytes >> 16) && h < 16384) h *= 2;
  return h;
}
static uint64_t ctrl_bytes(uint64_t heap_bytes) { return 4096 + hint_slots(heap_bytes) * 8 * 4; }
static uint64_t align_up(uint64_t x, uint64_t a) { return (x + a - 1) / a * a; }

// ---------------------------------------------------------------- layout
// Reading R-LAYOUT.  Regions, each 256-B aligned:
// control page (4 KiB) | data M*block_bytes | alloc_bm M*8 | iter_bm M*8 |
// type M*1 | R M*4 | (1 + 2*ntypes) hierarchical bitmaps of bitmap_words u64.
static void shape(uint64_t n, uint32_t* nlev, uint64_t* lw, uint64_t* tot) {
  uint32_t l = 0;
  uint64_t t = 0;
  for (;;) {
    uint64_t w = (n + 63) / 64;
    if (!w) w = 1;
    lw[l++] = w;
    t += w;
    if (n <= 64) break;
    n = w;
  }
  *nlev = l;
  *tot = t;
}
static uint64_t place(dsr_layout* L, uint64_t M, uint64_t heap_bytes) {
  uint64_t off = ctrl_bytes(heap_bytes);
  L->M = M;
  L->off_data = off;     off = align_up(off + M * L->block_bytes, 256);
  L->off_alloc_bm = off; off = align_up(off + M * 8, 256);
  L->off_iter_bm = off;  off = align_up(off + M * 8, 256);
  L->off_type = off;     off = align_up(off + M, 256);
  L->off_R = off;        off = align_up(off + M * 4, 256);
  uint64_t tot = 0;
  shape(M ? M : 1, &L->nlevels, L->level_words, &tot);
  L->bitmap_words = align_up(tot, 32);
  L->off_bitmaps = off;
  off += (1 + 2 * (uint64_t)L->ntypes) * L->bitmap_words * 8;
  L->total_bytes = off;
  return off;
}

extern "C" dsr_status dsr_layout_compute(const dsr_type_desc* types, uint32_t ntypes, uint64_t heap_bytes,
                                         dsr_layout* L) {
  if (!types || !L || ntypes < 1 || ntypes > DSR_MAX_TYPES) return DSR_ERR_INVALID;
  memset(L, 0, sizeof(*L));
  L->ntypes = ntypes;
  uint64_t sz[DSR_MAX_TYPES], smallest = ~0ull;
  for (uint32_t t = 0; t < ntypes; ++t) {
    const dsr_type_desc& d = types[t];
    if (d.num_fields < 1 || d.num_fields > DSR_MAX_FIELDS) return DSR_ERR_INVALID;
    if (d.parent) {                                           // inherited fields first
      if (d.parent > t) return DSR_ERR_INVALID;               // the base is declared earlier
      const dsr_type_desc& b = types[d.parent - 1];
      if (b.num_fields > d.num_fields) return DSR_ERR_INVALID;
      for (uint32_t f = 0; f < b.num_fields; ++f)
        if (b.field_bytes[f] != d.field_bytes[f]) return DSR_ERR_INVALID;
    }
    sz[t] = 0;
    for (uint32_t f = 0; f < d.num_fields; ++f) {
      const uint32_t b = d.field_bytes[f];
      if (b != 1 && b != 2 && b != 4 && b != 8 && b != 16) return DSR_ERR_INVALID;
      sz[t] += b;
    }
    if (sz[t] < smallest) smallest = sz[t];
  }
  uint64_t data = 0;
  for (uint32_t t = 0; t < ntypes; ++t) {
    const uint64_t cap = (64 * smallest) / sz[t];
    if (cap == 0) return DSR_ERR_INVALID;                     // > 64x the smallest type
    L->cap[t] = (uint32_t)cap;
    uint64_t end = 0;
    for (uint32_t f = 0; f < types[t].num_fields; ++f) {
      const uint64_t bytes = cap * types[t].field_bytes[f];
      const uint64_t off = align_up(end, 16);                // columns packed, 16-B aligned (R-LAYOUT)
      L->col_off[t][f] = (uint32_t)off;
      end = off + bytes;
    }
    if (end > data) data = end;
  }
  L->block_bytes = (uint32_t)align_up(data, 128);
  uint64_t lo = 0, hi = heap_bytes / L->block_bytes + 1;
  if (hi > 0xFFFFFFFFull) hi = 0xFFFFFFFFull;
  while (lo < hi) {
    const uint64_t mid = lo + (hi - lo + 1) / 2;
    if (place(L, mid, heap_bytes) <= heap_bytes) lo = mid; else hi = mid - 1;
  }
  if (lo == 0) return DSR_ERR_INVALID;
  place(L, lo, heap_bytes);
  return DSR_OK;
}

// ---------------------------------------------------------------- init kernels
// free bitmap: bits < size_l set on every level, everything else 0
__global__ void k_init_free(DevBitmap b, uint64_t nbits) {
  uint64_t size = nbits;
  for (uint32_t l = 0; l < b.nlevels; ++l) {
    const uint64_t words = (size + 63) / 64;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < words;
         i += (uint64_t)gridDim.x * blockDim.x) {
      const uint64_t lo = i * 64;
      const uint64_t nb = size - lo >= 64 ? 64 : size - lo;
      b.lvl[l][i] = nb == 64 ? ~0ull : ((1ull << nb) - 1ull);
    }
    size = words;
  }
}

#ifdef DSR_DEBUG
#define DSR_BUILD_KIND " debug"
#elif defined(DSR_FAULT)
#define DSR_BUILD_KIND " fault"
#else
#define DSR_BUILD_KIND ""
#endif
static dsr_status heap_init(dsr_heap* h, cudaStream_t st) {
  const dsr_layout& L = h->L;
  uint8_t* base = h->dev.data - L.off_data;
  CUDA_TRY(cudaMemsetAsync(base, 0, 4096, st));
  CUDA_TRY(cudaMemsetAsync(base + 4096, 0xFF, (h->dev.hint_mask + 1) * 8 * 4, st));   // warp hints: none
  CUDA_TRY(cudaMemsetAsync(base + L.off_alloc_bm, 0xFF, L.M * 8, st));     // invalidated == uninitialised
  CUDA_TRY(cudaMemsetAsync(base + L.off_type, 0, L.M, st));
  CUDA_TRY(cudaMemsetAsync(base + L.off_bitmaps, 0, (1 + 2 * (uint64_t)L.ntypes) * L.bitmap_words * 8, st));
  k_init_free<<<64, 256, 0, st>>>(h->dev.freebm, L.M);
  count_launch();
  CUDA_TRY(cudaGetLastError());
  return DSR_OK;
}

static void fill_bitmap(DevBitmap* b, uint64_t* words, const dsr_layout& L) {
  uint64_t off = 0;
  for (uint32_t l = 0; l < DSR_MAX_LEVELS; ++l) b->lvl[l] = nullptr;
  for (uint32_t l = 0; l < L.nlevels; ++l) {
    b->lvl[l] = words + off;
    off += L.level_words[l];
  }
  b->nlevels = L.nlevels;
  b->nbits = L.M;
}
static void fill_bitmaps(DevHeap& d, const dsr_layout& L, uint64_t* bm) {
  fill_bitmap(&d.freebm, bm, L);
  d.freebm.err = &d.ctrl[CTRL_ERR];
  for (uint32_t t = 0; t < L.ntypes; ++t) {
    fill_bitmap(&d.allocbm[t], bm + (1 + 2 * t) * L.bitmap_words, L);
    fill_bitmap(&d.activebm[t], bm + (2 + 2 * t) * L.bitmap_words, L);
    d.allocbm[t].err = d.activebm[t].err = &d.ctrl[CTRL_ERR];
  }
}

static void apply_cfg(dsr_heap* h, const dsr_config* cfg) {
  h->dev.r_attempts = (cfg && cfg->active_retries) ? cfg->active_retries : 5;   // r = 5
  h->dev.flags = cfg ? cfg->flags : 0u;
  h->dev.seed = cfg ? cfg->seed : 0x5eedull;
}

extern "C" dsr_status dsr_heap_create(const dsr_type_desc* types, uint32_t ntypes, void* dev_buf, uint64_t heap_bytes,
                                      const dsr_config* cfg, void* stream, dsr_heap** out) {
  if (!out || !dev_buf || ((uintptr_t)dev_buf & 255)) return DSR_ERR_INVALID;
  *out = nullptr;
  dsr_layout L;
  dsr_status s = dsr_layout_compute(types, ntypes, heap_bytes, &L);
  if (s != DSR_OK) return s;
  if (cfg && cfg->max_blocks && cfg->max_blocks < L.M) place(&L, cfg->max_blocks, heap_bytes);   // fewer blocks fit
  if (L.nlevels > DSR_MAX_LEVELS) return DSR_ERR_INVALID;
  dsr_heap* h = new (std::nothrow) dsr_heap;
  if (!h) return DSR_ERR_INVALID;
  memset(h, 0, sizeof(*h));
  h->L = L;
  memcpy(h->types, types, sizeof(dsr_type_desc) * ntypes);
  if (cudaGetDevice(&h->device) != cudaSuccess ||
      cudaDeviceGetAttribute(&h->sms, cudaDevAttrMultiProcessorCount, h->device) != cudaSuccess) {
    delete h;
    return DSR_ERR_CUDA;
  }
  uint8_t* base = (uint8_t*)dev_buf;
  DevHeap& d = h->dev;
  d.data = base + L.off_data;
  d.alloc_bm = (uint64_t*)(base + L.off_alloc_bm);
  d.iter_bm = (uint64_t*)(base + L.off_iter_bm);
  d.type = base + L.off_type;
  d.R = (uint32_t*)(base + L.off_R);
  d.ctrl = (ull*)base;
  d.hints = (uint32_t*)(base + 4096);
  d.hint_mask = (uint32_t)hint_slots(heap_bytes) - 1;
  d.sms = (uint32_t)h->sms;
  d.M = (uint32_t)L.M;
  d.block_bytes = L.block_bytes;
  d.ntypes = ntypes;
  fill_bitmaps(d, L, (uint64_t*)(base + L.off_bitmaps));
  for (uint32_t t = 0; t < ntypes; ++t) {
    DevType& ty = d.types[t];
    ty.cap = L.cap[t];
    ty.nfields = types[t].num_fields;
    ty.parent = types[t].parent;
    ty.valid = ty.cap == 64 ? ~0ull : ((1ull << ty.cap) - 1ull);
    ty.pad = ~ty.valid;
    for (uint32_t f = 0; f < ty.nfields; ++f) {
      ty.fsize[f] = types[t].field_bytes[f];
      ty.col_off[f] = L.col_off[t][f];
    }
  }
  apply_cfg(h, cfg);
  s = heap_init(h, (cudaStream_t)stream);
  if (s != DSR_OK) { delete h; return s; }
  *out = h;
  return DSR_OK;
}

extern "C" dsr_status dsr_heap_reset(dsr_heap* h, void* stream) {
  if (!h) return DSR_ERR_INVALID;
  return heap_init(h, (cudaStream_t)stream);
}
extern "C" dsr_status dsr_heap_destroy(dsr_heap* h) {
  if (!h) return DSR_ERR_INVALID;
  delete h;
  return DSR_OK;
}
extern "C" dsr_status dsr_heap_layout(const dsr_heap* h, dsr_layout* out) {
  if (!h || !out) return DSR_ERR_INVALID;
  *out = h->L;
  return DSR_OK;
}
extern "C" dsr_status dsr_heap_configure(dsr_heap* h, const dsr_config* cfg) {
  if (!h) return DSR_ERR_INVALID;
  apply_cfg(h, cfg);
  return DSR_OK;
}

static LaunchCtx ctx(dsr_heap* h, void* stream) {
  LaunchCtx c;
  c.h = h->dev;
  c.st = (cudaStream_t)stream;
  c.sms = h->sms;
  c.grid = h->sms * 8;   // 8 x 256 threads = 2048 resident threads per SM
  return c;
}

// do-all prologue grid: one warp per half level-1 container of the block
// bitmaps (2048 blocks), at most one wave of resident CTAs (k_compact strides)
static int compact_grid(const dsr_heap* h) {
  const uint64_t items = 2 * (((h->L.M + 63) / 64 + 63) / 64);       // halves of level-1 containers
  const uint64_t ctas = (items + kCompactThreads / 32 - 1) / (kCompactThreads / 32);
  const uint64_t cap = (uint64_t)h->sms * (uint64_t)resident_ctas((const void*)k_compact, kCompactThreads);
  return (int)(ctas < 1 ? 1 : (ctas < cap ? ctas : cap));
}

// ---------------------------------------------------------------- operations
static bool method_info(uint32_t method_id, MethodInfo* mi) {
  return mb_method_info(method_id, mi) || gol_method_info(method_id, mi) || wt_method_info(method_id, mi) ||
         nb_method_info(method_id, mi);
}

extern "C" dsr_status dsr_doall_prologue(dsr_heap* h, uint32_t type, uint32_t method_id, void* stream) {
  nvtxRangePushA("dsr doall_prologue");
  struct Pop { ~Pop() { nvtxRangePop(); } } pop_;
  if (!h || type >= h->L.ntypes) return DSR_ERR_INVALID;
  MethodInfo mi;
  if (!method_info(method_id, &mi)) return DSR_ERR_UNSUPPORTED;
  if (mi.snapshot == 4) return DSR_OK;             // the method enumerates its objects itself (no block list)
  cudaStream_t st = (cudaStream_t)stream;
  // R := compact(allocated[T]) (+ iteration-bitmap snapshot when the method may allocate)
  CUDA_TRY(cudaMemsetAsync(&h->dev.ctrl[CTRL_RCOUNT], 0, 8, st));
  k_compact<<<compact_grid(h), kCompactThreads, 0, st>>>(h->dev, type, mi.snapshot);
  count_launch();
  CUDA_TRY(cudaGetLastError());
  return DSR_OK;
}

static dsr_status doall_body(dsr_heap* h, uint32_t type, uint32_t method_id, const void* args, size_t args_bytes,
                             void* stream, int rk) {
  if (!h || type >= h->L.ntypes) return DSR_ERR_INVALID;
  MethodInfo mi;
  if (!method_info(method_id, &mi)) return DSR_ERR_UNSUPPORTED;
  if (mi.args_bytes && (args_bytes != mi.args_bytes || !args)) return DSR_ERR_INVALID;
  static const uint64_t zero_args[16] = {0};
  if (!mi.args_bytes) args = zero_args;
  LaunchCtx c = ctx(h, stream);
  c.rk = rk;
  bool ok = mb_method_launch(method_id, c, type, mi.snapshot, args) ||
            gol_method_launch(method_id, c, type, mi.snapshot, args) ||
            wt_method_launch(method_id, c, type, mi.snapshot, args) ||
            nb_method_launch(method_id, c, type, mi.snapshot, args);
  if (!ok) return DSR_ERR_INVALID;
  CUDA_TRY(cudaGetLastError());
  return DSR_OK;
}

extern "C" dsr_status dsr_doall_body(dsr_heap* h, uint32_t type, uint32_t method_id, const void* args,
                                     size_t args_bytes, void* stream) {
  nvtxRangePushA("dsr doall_body");
  struct Pop { ~Pop() { nvtxRangePop(); } } pop_;
  return doall_body(h, type, method_id, args, args_bytes, stream, -1);
}

// T and its subtypes, in type order (subtypes are declared after their base)
static uint32_t subtree(const dsr_heap* h, uint32_t type, uint32_t* out) {
  uint32_t n = 0;
  for (uint32_t t = 0; t < h->L.ntypes; ++t) {
    uint32_t u = t;
    for (int k = 0; k <= DSR_MAX_TYPES; ++k) {
      if (u == type) { out[n++] = t; break; }
      if (!h->types[u].parent) break;
      u = h->types[u].parent - 1;
    }
  }
  return n;
}

// NVTX range per do-all / user-kernel launch (name = operation, type, id),
// so nsys / ncu timelines show each pass of a step
struct NvtxRange {
  explicit NvtxRange(const char* what, uint32_t type, uint32_t id) {
    char name[64];
    snprintf(name, sizeof(name), "dsr %s T%u #%u", what, type, id);
    nvtxRangePushA(name);
  }
  ~NvtxRange() { nvtxRangePop(); }
};

extern "C" dsr_status dsr_parallel_do(dsr_heap* h, uint32_t type, uint32_t method_id, const void* args,
                                      size_t args_bytes, void* stream) {
  NvtxRange nv("parallel_do", type, method_id);
  MethodInfo mi;
  if (!h || type >= h->L.ntypes) return DSR_ERR_INVALID;
  if (!method_info(method_id, &mi)) return DSR_ERR_UNSUPPORTED;
  if (mi.args_bytes && (args_bytes != mi.args_bytes || !args)) return DSR_ERR_INVALID;
  uint32_t sub[DSR_MAX_TYPES];
  const uint32_t ns = subtree(h, type, sub);
  if (ns == 1) {
    dsr_status s = dsr_doall_prologue(h, type, method_id, stream);
    if (s != DSR_OK) return s;
    return dsr_doall_body(h, type, method_id, args, args_bytes, stream);
  }
  // Subtypes: one body per type, but every type's snapshot and block
  // range of R are taken before the first body runs, so objects a body
  // creates -- of any type of the subtree -- are not visited by this pass.
  cudaStream_t st = (cudaStream_t)stream;
  CUDA_TRY(cudaMemsetAsync(&h->dev.ctrl[CTRL_RCOUNT], 0, 8, st));
  CUDA_TRY(cudaMemsetAsync(&h->dev.ctrl[CTRL_RBEG], 0, 8, st));
  for (uint32_t k = 0; k < ns; ++k) {
    k_compact<<<compact_grid(h), kCompactThreads, 0, st>>>(h->dev, sub[k], mi.snapshot);
    count_launch();
    CUDA_TRY(cudaMemcpyAsync(&h->dev.ctrl[CTRL_RBEG + k + 1], &h->dev.ctrl[CTRL_RCOUNT], 8, cudaMemcpyDeviceToDevice,
                             st));
  }
  CUDA_TRY(cudaGetLastError());
  for (uint32_t k = 0; k < ns; ++k) {
    dsr_status s = doall_body(h, sub[k], method_id, args, args_bytes, stream, (int)k);
    if (s != DSR_OK) return s;
  }
  return DSR_OK;
}

extern "C" dsr_status dsr_parallel_new(dsr_heap* h, uint32_t type, uint64_t n, uint32_t ctor_id, const void* args,
                                       size_t args_bytes, void* stream) {
  NvtxRange nv("parallel_new", type, ctor_id);
  if (!h || type >= h->L.ntypes) return DSR_ERR_INVALID;
  if (n == 0) return DSR_OK;
  LaunchCtx c = ctx(h, stream);
  int ok = 1;
  bool known = wt_ctor_launch(ctor_id, c, type, n, args, args_bytes, &ok) ||
               nb_ctor_launch(ctor_id, c, type, n, args, args_bytes, &ok);
  if (!known) return DSR_ERR_UNSUPPORTED;
  if (!ok) return DSR_ERR_INVALID;
  CUDA_TRY(cudaGetLastError());
  return DSR_OK;
}

// dsr_mb_new_args.in_host: stage the caller's host array into a device buffer
// on the heap's copy stream; `launch_stream` waits for it (see dsr.h)
static dsr_status stage_host_input(dsr_heap* h, uint64_t n, dsr_mb_new_args* a, cudaStream_t st) {
  const size_t bytes = (size_t)64 * ((n + 3) / 4);
  const int k = h->stage_next;
  h->stage_next ^= 1;
  if (!h->cstream) {
    CUDA_TRY(cudaStreamCreateWithFlags(&h->cstream, cudaStreamNonBlocking));
    for (int j = 0; j < 2; ++j) {
      CUDA_TRY(cudaEventCreateWithFlags(&h->ready[j], cudaEventDisableTiming));
      CUDA_TRY(cudaEventCreateWithFlags(&h->used[j], cudaEventDisableTiming));
    }
  }
  if (h->stage_cap[k] < bytes) {                      // grow (first use): wait for the buffer's last reader
    CUDA_TRY(cudaEventSynchronize(h->used[k]));
    if (h->stage[k]) CUDA_TRY(cudaFree(h->stage[k]));
    h->stage[k] = nullptr;
    h->stage_cap[k] = 0;
    CUDA_TRY(cudaMalloc(&h->stage[k], bytes));
    h->stage_cap[k] = bytes;
  }
  CUDA_TRY(cudaStreamWaitEvent(h->cstream, h->used[k], 0));
  CUDA_TRY(cudaMemcpyAsync(h->stage[k], a->in, bytes, cudaMemcpyHostToDevice, h->cstream));
  CUDA_TRY(cudaEventRecord(h->ready[k], h->cstream));
  CUDA_TRY(cudaStreamWaitEvent(st, h->ready[k], 0));
  a->in = (const uint32_t*)h->stage[k];
  a->in_host = 0;
  return DSR_OK;
}

extern "C" dsr_status dsr_launch(dsr_heap* h, uint32_t kernel_id, uint64_t n, const void* args, size_t args_bytes,
                                 void* stream) {
  NvtxRange nv("launch", 0, kernel_id);
  if (!h || !args) return DSR_ERR_INVALID;
  if (n == 0) return DSR_OK;
  LaunchCtx c = ctx(h, stream);
  int ok = 1;
  dsr_mb_new_args staged;
  int stage_slot = -1;
  if ((kernel_id == DSR_K_MB_NEW || kernel_id == DSR_K_MB_NEW_BULK) && args_bytes == sizeof(dsr_mb_new_args) &&
      ((const dsr_mb_new_args*)args)->in && ((const dsr_mb_new_args*)args)->in_host) {
    staged = *(const dsr_mb_new_args*)args;
    if (staged.t0 & 3) return DSR_ERR_INVALID;
    stage_slot = h->stage_next;
    dsr_status s = stage_host_input(h, n, &staged, c.st);
    if (s != DSR_OK) return s;
    args = &staged;
  }
  bool known = mb_kernel_launch(kernel_id, c, n, args, args_bytes, &ok) ||
               gol_kernel_launch(kernel_id, c, n, args, args_bytes, &ok) ||
               wt_kernel_launch(kernel_id, c, n, args, args_bytes, &ok) ||
               nb_kernel_launch(kernel_id, c, n, args, args_bytes, &ok);
  if (!known) return DSR_ERR_UNSUPPORTED;
  if (!ok) return DSR_ERR_INVALID;
  CUDA_TRY(cudaGetLastError());
  if (stage_slot >= 0) CUDA_TRY(cudaEventRecord(h->used[stage_slot], c.st));   // the staging buffer's reader
  return DSR_OK;
}

// ---------------------------------------------------------------- bulk slow path / trim
__global__ void __launch_bounds__(256) k_reserve_blocks(DevHeap h, uint32_t T, uint64_t nblocks) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nblocks; i += stride) {
    int64_t bid = -1;
    // a FAIL of clear() can be spurious while other threads clear bits of the
    // same containers (transient level inconsistency): retry; give up
    // only when the top-level word of the free bitmap is 0 (heap exhausted)
    for (uint32_t k = 0; bid < 0 && k < 64; ++k) {
      bid = bm_clear_any(h, h.freebm, i * 0x9E3779B97F4A7C15ull + 1, (uint64_t)k << 8);   // rotated per thread
      if (bid < 0 && ld_relaxed(h.freebm.lvl[h.freebm.nlevels - 1]) == 0) return;
    }
    if (bid < 0) return;
    init_block(h, T, (uint32_t)bid);
    bm_set(h.allocbm[T], (uint64_t)bid);
    bm_set(h.activebm[T], (uint64_t)bid);
    stat_add(h, ST_INITS, 1);
  }
}

__global__ void __launch_bounds__(256) k_trim(DevHeap h, uint32_t T) {
  const DevBitmap& ab = h.allocbm[T];
  const uint64_t nwords = ((uint64_t)h.M + 63) / 64;
  const uint64_t pad = h.types[T].pad;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nwords; i += (uint64_t)gridDim.x * blockDim.x) {
    if (ab.nlevels > 1 && !((ab.lvl[1][i >> 6] >> (i & 63)) & 1ull)) continue;
    uint64_t w = ab.lvl[0][i];
    while (w) {
      const uint32_t b = (uint32_t)(i * 64 + __ffsll((long long)w) - 1);
      w &= w - 1;
      if (h.alloc_bm[b] != pad) continue;                  // holds objects
      uint32_t t;
      if (block_invalidate(h, b, &t)) {                    // quiescent: succeeds for an empty block (t == T)
        bm_clear(h.activebm[T], b);
        bm_clear(h.allocbm[T], b);
        bm_set(h.freebm, b);
        stat_add(h, ST_BFREES, 1);
      }
    }
  }
}

extern "C" dsr_status dsr_reserve_blocks(dsr_heap* h, uint32_t type, uint64_t nblocks, void* stream) {
  if (!h || type >= h->L.ntypes) return DSR_ERR_INVALID;
  if (nblocks == 0) return DSR_OK;
  LaunchCtx c = ctx(h, stream);
  k_reserve_blocks<<<grid_for(c, nblocks, k_reserve_blocks), 256, 0, c.st>>>(h->dev, type, nblocks);
  count_launch();
  CUDA_TRY(cudaGetLastError());
  return DSR_OK;
}

extern "C" dsr_status dsr_trim(dsr_heap* h, uint32_t type, void* stream) {
  if (!h || type >= h->L.ntypes) return DSR_ERR_INVALID;
  LaunchCtx c = ctx(h, stream);
  k_trim<<<h->sms * 4, 256, 0, c.st>>>(h->dev, type);
  count_launch();
  CUDA_TRY(cudaGetLastError());
  return DSR_OK;
}

// ---------------------------------------------------------------- live count / stats
__global__ void k_live(DevHeap h, uint32_t T, unsigned long long* out) {
  const DevBitmap& ab = h.allocbm[T];
  const uint64_t nwords = ((uint64_t)h.M + 63) / 64;
  unsigned long long acc = 0;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nwords; i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t w = ab.lvl[0][i];
    while (w) {
      const uint32_t b = (uint32_t)(i * 64 + __ffsll((long long)w) - 1);
      w &= w - 1;
      acc += __popcll(h.alloc_bm[b] & h.types[T].valid);
    }
  }
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0 && acc) atomicAdd(out, acc);
}

extern "C" dsr_status dsr_live_count(dsr_heap* h, uint32_t type, uint64_t* dev_out, void* stream) {
  if (!h || !dev_out || type >= h->L.ntypes) return DSR_ERR_INVALID;
  cudaStream_t st = (cudaStream_t)stream;
  CUDA_TRY(cudaMemsetAsync(dev_out, 0, 8, st));
  k_live<<<h->sms * 4, 256, 0, st>>>(h->dev, type, (unsigned long long*)dev_out);
  count_launch();
  CUDA_TRY(cudaGetLastError());
  return DSR_OK;
}

extern "C" dsr_status dsr_live_count_sync(dsr_heap* h, uint32_t type, uint64_t* host_out, void* stream) {
  if (!h || !host_out || type >= h->L.ntypes) return DSR_ERR_INVALID;
  uint64_t* scratch = (uint64_t*)&h->dev.ctrl[CTRL_SCRATCH];
  dsr_status s = dsr_live_count(h, type, scratch, stream);
  if (s != DSR_OK) return s;
  CUDA_TRY(cudaMemcpyAsync(host_out, scratch, 8, cudaMemcpyDeviceToHost, (cudaStream_t)stream));
  CUDA_TRY(cudaStreamSynchronize((cudaStream_t)stream));
  return DSR_OK;
}

extern "C" dsr_status dsr_poll_error(dsr_heap* h, void* stream) {
  if (!h) return DSR_ERR_INVALID;
  unsigned long long e = 0;
  cudaStream_t st = (cudaStream_t)stream;
  CUDA_TRY(cudaMemcpyAsync(&e, &h->dev.ctrl[CTRL_ERR], 8, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaMemsetAsync(&h->dev.ctrl[CTRL_ERR], 0, 8, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  if (e & ERRB_OOM) return DSR_ERR_OOM;
  if (e & ERRB_BUDGET) return DSR_ERR_RETRY_BUDGET;
  if (e & ERRB_BOUNDS) return DSR_ERR_INVARIANT;
  return DSR_OK;
}

// ---------------------------------------------------------------- quiescent audit
__device__ __forceinline__ bool bget(const DevBitmap& b, uint64_t pos) { return (b.lvl[0][pos >> 6] >> (pos & 63)) & 1; }

__global__ void k_audit_blocks(DevHeap h, unsigned long long* fails) {
  unsigned long long bad = 0;
  for (uint64_t b = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; b < h.M; b += (uint64_t)gridDim.x * blockDim.x) {
    const bool fr = bget(h.freebm, b);
    int owners = fr ? 1 : 0;
    const uint64_t w = h.alloc_bm[b];
    for (uint32_t t = 0; t < h.ntypes; ++t) {
      const bool al = bget(h.allocbm[t], b), ac = bget(h.activebm[t], b);
      if (ac && !al) ++bad;                                   // active ⊆ allocated
      if (!al) continue;
      ++owners;
      const DevType& ty = h.types[t];
      if (h.type[b] != t + 1) ++bad;                          // block type id
      if ((w | ty.valid) != ~0ull) ++bad;                     // padding bits set
      if ((w & ty.valid) == 0) ++bad;                         // allocated blocks are non-empty
      if (ac != (w != ~0ull)) ++bad;                          // active iff non-full
    }
    if (owners != 1) ++bad;                                   // free ⊎ allocated[.] partition [0, M)
    if (fr && w != ~0ull) ++bad;                              // free blocks are invalidated
  }
  if (bad) atomicAdd(fails, bad);
}

// hierarchy consistency b^{l+1}_i = OR(C^l_i) (Def. P:1115) and no bit >= size
__global__ void k_audit_bitmap(DevBitmap b, unsigned long long* fails) {
  unsigned long long bad = 0;
  uint64_t size = b.nbits;
  for (uint32_t l = 0; l < b.nlevels; ++l) {
    const uint64_t words = (size + 63) / 64;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < words; i += (uint64_t)gridDim.x * blockDim.x) {
      const uint64_t w = b.lvl[l][i];
      const uint64_t lo = i * 64;
      const uint64_t nb = size - lo >= 64 ? 64 : size - lo;
      if (nb < 64 && (w >> nb)) ++bad;
      if (l + 1 < b.nlevels) {
        const bool up = (b.lvl[l + 1][i >> 6] >> (i & 63)) & 1;
        if (up != (w != 0)) ++bad;
      }
    }
    size = words;
  }
  if (bad) atomicAdd(fails, bad);
}

extern "C" dsr_status dsr_check_invariants(dsr_heap* h, void* stream, uint64_t* failures_out) {
  if (!h) return DSR_ERR_INVALID;
  cudaStream_t st = (cudaStream_t)stream;
  unsigned long long* f = &h->dev.ctrl[CTRL_AUDIT];
  CUDA_TRY(cudaMemsetAsync(f, 0, 8, st));
  k_audit_blocks<<<h->sms * 4, 256, 0, st>>>(h->dev, f);
  k_audit_bitmap<<<h->sms, 256, 0, st>>>(h->dev.freebm, f);
  count_launch(2);
  for (uint32_t t = 0; t < h->L.ntypes; ++t) {
    k_audit_bitmap<<<h->sms, 256, 0, st>>>(h->dev.allocbm[t], f);
    k_audit_bitmap<<<h->sms, 256, 0, st>>>(h->dev.activebm[t], f);
    count_launch(2);
  }
  unsigned long long hf = 0;
  CUDA_TRY(cudaMemcpyAsync(&hf, f, 8, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  if (failures_out) *failures_out = hf;
  return hf ? DSR_ERR_INVARIANT : DSR_OK;
}

// ---------------------------------------------------------------- fragmentation
__global__ void k_frag(DevHeap h, unsigned long long* acc /* [t*3 + {used, slots, blocks}] */) {
  for (uint32_t t = 0; t < h.ntypes; ++t) {
    const uint64_t nwords = ((uint64_t)h.M + 63) / 64;
    unsigned long long used = 0, blocks = 0;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nwords; i += (uint64_t)gridDim.x * blockDim.x) {
      uint64_t w = h.allocbm[t].lvl[0][i];
      while (w) {
        const uint32_t b = (uint32_t)(i * 64 + __ffsll((long long)w) - 1);
        w &= w - 1;
        used += __popcll(h.alloc_bm[b] & h.types[t].valid);
        ++blocks;
      }
    }
    for (int o = 16; o; o >>= 1) {
      used += __shfl_xor_sync(0xffffffffu, used, o);
      blocks += __shfl_xor_sync(0xffffffffu, blocks, o);
    }
    if ((threadIdx.x & 31) == 0 && blocks) {
      atomicAdd(acc + 3 * t + 0, used);
      atomicAdd(acc + 3 * t + 2, blocks);
    }
  }
}

extern "C" dsr_status dsr_fragmentation(dsr_heap* h, double* out, uint64_t* blocks_per_type, void* stream) {
  if (!h || !out) return DSR_ERR_INVALID;
  cudaStream_t st = (cudaStream_t)stream;
  unsigned long long* acc = &h->dev.ctrl[CTRL_AUDIT + 1];
  CUDA_TRY(cudaMemsetAsync(acc, 0, 8 * 3 * DSR_MAX_TYPES, st));
  k_frag<<<h->sms * 4, 256, 0, st>>>(h->dev, acc);
  count_launch();
  unsigned long long hv[3 * DSR_MAX_TYPES];
  CUDA_TRY(cudaMemcpyAsync(hv, acc, sizeof(hv), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  double unused = 0, slots = 0;
  for (uint32_t t = 0; t < h->L.ntypes; ++t) {
    const double s = (double)hv[3 * t + 2] * h->L.cap[t];
    slots += s;
    unused += s - (double)hv[3 * t];
    if (blocks_per_type) blocks_per_type[t] = hv[3 * t + 2];
  }
  *out = slots > 0 ? unused / slots : 0.0;     // 0 without blocks (reading C36)
  return DSR_OK;
}

extern "C" dsr_status dsr_stats(dsr_heap* h, dsr_counters* out, void* stream) {
  if (!h || !out) return DSR_ERR_INVALID;
  unsigned long long v[ST_N];
  cudaStream_t st = (cudaStream_t)stream;
  CUDA_TRY(cudaMemcpyAsync(v, &h->dev.ctrl[CTRL_STATS], sizeof(v), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  out->allocs = v[ST_ALLOCS];
  out->frees = v[ST_FREES];
  out->block_inits = v[ST_INITS];
  out->block_frees = v[ST_BFREES];
  out->rollbacks = v[ST_ROLLBACKS];
  out->invalidate_fail = v[ST_INVFAIL];
  out->reserve_retries = v[ST_RESRETRY];
  out->oom = v[ST_OOM];
  out->requests = v[ST_REQ];
  out->finds = v[ST_FIND];
  out->find_fails = v[ST_FINDFAIL];
  out->reserve_zero = v[ST_RESZERO];
  out->cyc_find = v[ST_CYC_FIND];
  out->cyc_slow = v[ST_CYC_SLOW];
  out->cyc_reserve = v[ST_CYC_RES];
  out->cyc_request = v[ST_CYC_REQ];
  out->hint_zero = v[ST_HINTZERO];
  return DSR_OK;
}
extern "C" dsr_status dsr_stats_reset(dsr_heap* h, void* stream) {
  if (!h) return DSR_ERR_INVALID;
  CUDA_TRY(cudaMemsetAsync(&h->dev.ctrl[CTRL_STATS], 0, 8 * ST_N, (cudaStream_t)stream));
  return DSR_OK;
}

extern "C" dsr_status dsr_copy_state(dsr_heap* h, uint32_t what, uint32_t type, void* host_out, size_t cap,
                                     size_t* used, void* stream) {
  if (!h || !host_out) return DSR_ERR_INVALID;
  cudaStream_t st = (cudaStream_t)stream;
  const void* src = nullptr;
  size_t n = 0;
  uint64_t lw = 0;
  for (uint32_t l = 0; l < h->L.nlevels; ++l) lw += h->L.level_words[l];
  switch (what) {
    case 0: src = h->dev.alloc_bm; n = h->L.M * 8; break;
    case 1: src = h->dev.type; n = h->L.M; break;
    case 2: src = h->dev.freebm.lvl[0]; n = lw * 8; break;
    case 3: if (type >= h->L.ntypes) return DSR_ERR_INVALID; src = h->dev.allocbm[type].lvl[0]; n = lw * 8; break;
    case 4: if (type >= h->L.ntypes) return DSR_ERR_INVALID; src = h->dev.activebm[type].lvl[0]; n = lw * 8; break;
    case 5: src = h->dev.R; n = h->L.M * 4; break;
    default: return DSR_ERR_INVALID;
  }
  if (cap < n + (what == 5 ? 8 : 0)) return DSR_ERR_INVALID;
  CUDA_TRY(cudaMemcpyAsync(host_out, src, n, cudaMemcpyDeviceToHost, st));
  if (what == 5) CUDA_TRY(cudaMemcpyAsync((uint8_t*)host_out + n, &h->dev.ctrl[CTRL_RCOUNT], 8, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  if (used) *used = n + (what == 5 ? 8 : 0);
  return DSR_OK;
}

// ---------------------------------------------------------------- canonical dump, device view
__global__ void k_dump_records(DevHeap h, uint32_t T, uint32_t rb, uint8_t* out, unsigned long long* cursor) {
  const uint32_t r = ld_relaxed_u32((const uint32_t*)&h.ctrl[CTRL_RCOUNT]);
  const uint32_t N = h.types[T].cap;
  const uint64_t total = (uint64_t)r * N;
  for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t b = h.R[e / N], s = (uint32_t)(e % N);
    if (!((h.alloc_bm[b] >> s) & 1ull)) continue;
    uint8_t* rec = out + atomicAdd(cursor, 1ull) * rb;
    for (uint32_t f = 0, o = 0; f < h.types[T].nfields; ++f) {
      const uint32_t sz = h.types[T].fsize[f];
      const uint8_t* src = h.data + (size_t)b * h.block_bytes + h.types[T].col_off[f] + (size_t)s * sz;
      for (uint32_t k = 0; k < sz; ++k) rec[o + k] = src[k];
      o += sz;
    }
  }
}

extern "C" dsr_status dsr_canonical_dump(dsr_heap* h, uint32_t type, void* host_buf, size_t cap, size_t* used,
                                         void* stream) {
  if (!h || type >= h->L.ntypes || !used) return DSR_ERR_INVALID;
  cudaStream_t st = (cudaStream_t)stream;
  uint64_t live = 0;
  dsr_status s = dsr_live_count_sync(h, type, &live, stream);
  if (s != DSR_OK) return s;
  uint32_t rb = 0;
  for (uint32_t f = 0; f < h->types[type].num_fields; ++f) rb += h->types[type].field_bytes[f];
  *used = (size_t)live * rb;
  if (!host_buf || cap < *used) return DSR_ERR_INVALID;
  if (live == 0) return DSR_OK;
  uint8_t* d = nullptr;
  // the record cursor gets its own 8-B aligned word after the records (record
  // sizes such as 5, 12 or 17 B leave live * rb unaligned)
  const size_t cur_off = align_up(*used, 8);
  CUDA_TRY(cudaMallocAsync((void**)&d, cur_off + 8, st));
  unsigned long long* cursor = (unsigned long long*)(d + cur_off);
  CUDA_TRY(cudaMemsetAsync(cursor, 0, 8, st));
  CUDA_TRY(cudaMemsetAsync(&h->dev.ctrl[CTRL_RCOUNT], 0, 8, st));
  k_compact<<<compact_grid(h), kCompactThreads, 0, st>>>(h->dev, type, 0);
  k_dump_records<<<h->sms * 8, 256, 0, st>>>(h->dev, type, rb, d, cursor);
  count_launch(2);
  std::vector<uint8_t> tmp(*used);
  CUDA_TRY(cudaMemcpyAsync(tmp.data(), d, *used, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaFreeAsync(d, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  std::vector<uint64_t> idx(live);
  for (uint64_t i = 0; i < live; ++i) idx[i] = i;
  const uint8_t* base = tmp.data();
  std::sort(idx.begin(), idx.end(),
            [&](uint64_t a, uint64_t b) { return memcmp(base + a * rb, base + b * rb, rb) < 0; });
  for (uint64_t i = 0; i < live; ++i) memcpy((uint8_t*)host_buf + i * rb, base + idx[i] * rb, rb);
  return DSR_OK;
}

extern "C" size_t dsr_device_view_bytes(void) { return sizeof(DevHeap); }
extern "C" dsr_status dsr_device_view(const dsr_heap* h, void* out, size_t out_bytes) {
  if (!h || !out || out_bytes != sizeof(DevHeap)) return DSR_ERR_INVALID;
  memcpy(out, &h->dev, sizeof(DevHeap));
  return DSR_OK;
}

// ---- atomic-throughput probe (the allocator's roofline denominator)
static __global__ void __launch_bounds__(256) k_probe_atom(unsigned long long* buf, uint64_t words, uint32_t mode,
                                                           uint32_t iters, unsigned long long* sink) {
  const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  uint64_t x = t * 0x9E3779B97F4A7C15ull + 1, acc = 0;
  for (uint32_t i = 0; i < iters; ++i) {
    x ^= x >> 29; x *= 0xBF58476D1CE4E5B9ull;                  // next hashed address
    const uint64_t w = mode ? 0 : (x >> 20) % words;
    acc += atomicOr(buf + w, 1ull << (t & 63));                 // RMW with return (ATOMG)
  }
  if (acc == 0x5EED5EED5EED5EEDull) *sink = acc;                 // keeps the results live
}

extern "C" dsr_status dsr_ipc_handle(void* dev_ptr, void* handle_out, uint64_t* offset_out) {
  if (!dev_ptr || !handle_out || !offset_out) return DSR_ERR_INVALID;
  // the handle names the whole cudaMalloc block (a caching allocator such as
  // torch's hands out pieces of larger blocks): report dev_ptr's offset in it
  typedef CUresult (*RangeFn)(CUdeviceptr*, size_t*, CUdeviceptr);
  static RangeFn range = nullptr;
  if (!range) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn)
      return DSR_ERR_CUDA;
    range = (RangeFn)fn;
  }
  CUdeviceptr base = 0;
  size_t size = 0;
  if (range(&base, &size, (CUdeviceptr)dev_ptr) != CUDA_SUCCESS) return DSR_ERR_CUDA;
  cudaIpcMemHandle_t hd;
  if (cudaIpcGetMemHandle(&hd, (void*)base) != cudaSuccess) return DSR_ERR_CUDA;
  static_assert(sizeof(hd) == 64, "CUDA IPC handles are 64 bytes");
  memcpy(handle_out, &hd, sizeof(hd));
  *offset_out = (uint64_t)((CUdeviceptr)dev_ptr - base);
  return DSR_OK;
}
extern "C" dsr_status dsr_ipc_open(const void* handle, void** dev_ptr_out) {
  if (!handle || !dev_ptr_out) return DSR_ERR_INVALID;
  cudaIpcMemHandle_t hd;
  memcpy(&hd, handle, sizeof(hd));
  if (cudaIpcOpenMemHandle(dev_ptr_out, hd, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) return DSR_ERR_CUDA;
  return DSR_OK;
}
extern "C" dsr_status dsr_ipc_close(void* dev_ptr) {
  if (!dev_ptr) return DSR_ERR_INVALID;
  return cudaIpcCloseMemHandle(dev_ptr) == cudaSuccess ? DSR_OK : DSR_ERR_CUDA;
}

extern "C" dsr_status dsr_probe_atomics(void* dev_buf, uint64_t bytes, uint32_t mode, uint32_t iters,
                                        uint64_t* ops_out, void* stream) {
  if (!dev_buf || bytes < 16 || iters == 0 || mode > 1 || !ops_out) return DSR_ERR_INVALID;
  int dev = 0, sms = 0, per = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_probe_atom, 256, 0));
  const uint64_t words = bytes / 8 - 1;                          // the last word is the sink
  unsigned long long* buf = (unsigned long long*)dev_buf;
  const int grid = sms * per;
  k_probe_atom<<<grid, 256, 0, (cudaStream_t)stream>>>(buf, words, mode, iters, buf + words);
  count_launch();
  CUDA_TRY(cudaGetLastError());
  *ops_out = (uint64_t)grid * 256 * iters;
  return DSR_OK;
}

extern "C" uint64_t dsr_kernel_launches(void) { return g_launches.load(); }

extern "C" const char* dsr_status_str(dsr_status s) {
  switch (s) {
    case DSR_OK: return "DSR_OK";
    case DSR_ERR_INVALID: return "DSR_ERR_INVALID";
    case DSR_ERR_OOM: return "DSR_ERR_OOM";
    case DSR_ERR_CUDA: return "DSR_ERR_CUDA";
    case DSR_ERR_RETRY_BUDGET: return "DSR_ERR_RETRY_BUDGET";
    case DSR_ERR_INVARIANT: return "DSR_ERR_INVARIANT";
    case DSR_ERR_UNSUPPORTED: return "DSR_ERR_UNSUPPORTED";
  }
  return "DSR_ERR_?";
}
extern "C" const char* dsr_build_info(void) { return DSR_BUILD_INFO DSR_BUILD_KIND; }
