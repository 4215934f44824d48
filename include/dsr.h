/*
 * dsr.h -- C ABI of the B200-native DynaSOAr hot path (libdsr.so).
 *
 * DynaSOAr (Springer & Masuhara, arXiv 1810.11765; "P:n" = PAPER.md line n)
 * is an object allocator with five operations:
 *   parallel_do<T, &T::f>(args)   run f on every object of T existing at launch
 *   parallel_new<T>(n, args)      construct n objects; constructor i gets id i
 *   new(d_allocator) T(args)      device-side allocation
 *   destroy(d_allocator, p)       device-side deallocation
 *   device_do<T, &T::f>(args)     sequential for-each inside one thread
 * Types and methods are fixed at compile time ("The types ... must be
 * specified at compile time"), so methods and constructors are selected by id
 * from tables compiled into the library (DSR_M_* / DSR_C_* / DSR_K_* below).
 *
 * Conventions for every entry point:
 *   - returns dsr_status; DSR_ERR_INVALID is returned before any launch when
 *     an argument is out of range; DSR_ERR_CUDA when a CUDA call fails.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default
 *     stream).  Calls are stream-ordered and asynchronous unless their name
 *     ends in _sync or they are documented as synchronising.
 *   - "device pointer" arguments must point into device memory of the
 *     current device; "host pointer" arguments into host memory.
 *   - Device-side OOM / retry-budget exhaustion never aborts a kernel: the
 *     operation yields a null handle and ORs a bit into the heap's sticky
 *     error word, reported by the next synchronising call (dsr_poll_error,
 *     *_sync, dsr_check_invariants, dsr_fragmentation, dsr_stats).
 *   - One host thread per heap; calls on one heap are ordered by one stream.
 */
#ifndef DSR_H
#define DSR_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  DSR_OK = 0,
  DSR_ERR_INVALID = 1,       /* bad argument, detected on the host before launch */
  DSR_ERR_OOM = 2,           /* device-side: free block bitmap exhausted (reading R-OOM) */
  DSR_ERR_CUDA = 3,          /* a CUDA runtime call failed */
  DSR_ERR_RETRY_BUDGET = 4,  /* debug builds (-DDSR_DEBUG): illegal use detected -- a bitmap spin exceeded its
                                bound or a destroy named a slot that is not allocated (Alg. 7
                                precondition); release builds deadlock there, as the paper does */
  DSR_ERR_INVARIANT = 5,     /* dsr_check_invariants found violations */
  DSR_ERR_UNSUPPORTED = 6    /* id not compiled into this library */
} dsr_status;

/* Object handle ("fake pointer", Fig. 5; Listing 2):
 *   bits  0-5  slot in block          (mask 0x3F)
 *   bits  6-49 block index            (mask 0x3FFFFFFFFFFC0; reading R-BID: an index, not an address)
 *   bits 50-55 block capacity N_T - 1 (mask 0xFC000000000000; reading R-CAP)
 *   bits 56-63 type id (1-based; 0 = null / free block, reading R-TYPEID)
 * 0 is the null handle. */
typedef uint64_t dsr_handle;

#define DSR_MAX_TYPES 8
#define DSR_MAX_FIELDS 16
#define DSR_MAX_LEVELS 6

/* One object type: its fields in declaration order (inherited fields first,
 * P:293).  field_bytes[f] in {1, 2, 4, 8, 16}.  parent: 0 = no base type;
 * k = the type derives from type k - 1, which must be declared earlier and
 * whose fields must be this type's first fields (the inherited SOA columns
 * precede the newly introduced ones).  A base field f is then column f
 * of every subtype, addressed through any handle with the capacity of the
 * handle's runtime type (handle bits 50-55). */
typedef struct {
  uint32_t num_fields;
  uint32_t field_bytes[DSR_MAX_FIELDS];
  uint32_t parent;
} dsr_type_desc;

/* Heap layout in the caller's device buffer.  All
 * offsets are bytes from the buffer start.  Computed by dsr_layout_compute. */
typedef struct {
  uint32_t ntypes;
  uint32_t cap[DSR_MAX_TYPES];                     /* N_T = floor(64 size(T_s)/size(T)) */
  uint32_t col_off[DSR_MAX_TYPES][DSR_MAX_FIELDS]; /* SOA column offsets inside a block */
  uint32_t block_bytes;                            /* data bytes per block, multiple of 128 */
  uint64_t M;                                      /* number of blocks */
  uint32_t nlevels;                                /* levels of each M-bit hierarchical bitmap */
  uint64_t level_words[8];                         /* u64 containers per level */
  uint64_t off_data, off_alloc_bm, off_iter_bm, off_type, off_R, off_bitmaps;
  uint64_t bitmap_words;                           /* u64 words reserved per hierarchical bitmap */
  uint64_t total_bytes;                            /* bytes of the buffer used (<= heap_bytes) */
} dsr_layout;

/* dsr_config.flags */
#define DSR_F_NO_ROTATE   0x1u  /* plain ffs instead of rotated search ("NoShift") */
#define DSR_F_NO_COALESCE 0x2u  /* one reservation per thread ("NoCoal") */
#define DSR_F_STATS       0x4u  /* maintain device counters (dsr_stats) */
#define DSR_F_SPIN_ON_OOM 0x8u  /* paper behaviour: loop forever on OOM */
#define DSR_F_NO_HINT     0x10u /* no per-warp block hint: every request searches active[T] (paper-exact, replay) */
#define DSR_F_CTA_NEW     0x20u /* bulk constructors use CTA-level instead of warp-level request coalescing (microbench new kernel only) */
#define DSR_F_HOME_ROT    0x40u /* ablation: SM-affine rotation (searches start in the SM's range of level-1 containers) */
#define DSR_F_SLOT_ROTATE 0x80u /* paper: also rotate a block's object bitmap before choosing its free slots; off by default */
#define DSR_F_SCALAR_DOALL 0x100u /* ablation: one thread per object in methods that also have a quad-mapped (vectorised) body */
#define DSR_F_QUAD_FREE   0x200u /* ablation: microbench free passes as quad-mapped do-alls (lanes of a block combine their masks) instead of block-mapped (one lane per block) */
#define DSR_F_BULK_DENSE  0x400u /* warp-cooperative new (R-BULK): one failed lookup attempt per round instead of per failed lane -- fills partially free blocks longer (lower fragmentation, slower) */

typedef struct {
  uint32_t active_retries;   /* r: try_find_set attempts before the slow path (Fig. 11); 0 -> 5 */
  uint32_t flags;            /* DSR_F_* */
  uint64_t seed;             /* rotation seed */
  uint64_t max_blocks;       /* dsr_heap_create only: 0 = as many blocks as fit in the buffer, else
                                M = min(that, max_blocks) ("M is determined at compile time") */
} dsr_config;

typedef struct {
  uint64_t allocs;           /* successful new */
  uint64_t frees;            /* successful destroy */
  uint64_t block_inits;      /* slow-path initialize_block (Alg. 8) */
  uint64_t block_frees;      /* successful invalidate -> free.set (Alg. 2 l.7-11) */
  uint64_t rollbacks;        /* type-changed reservations rolled back (Alg. 1 l.14) */
  uint64_t invalidate_fail;  /* failed / rolled-back invalidations (Alg. 9 l.8) */
  uint64_t reserve_retries;  /* reservations that lost every selected bit (Alg. 6 loop) */
  uint64_t oom;              /* OOM events */
  /* profiling (DSR_F_STATS in a library built with -DDSR_PROFILE, else 0):
   * leader requests, active lookups, failed lookups,
   * zero-slot reservations, and SM cycles summed over leaders spent in the
   * lookup, the slow path, the reservation (+ FULL handling), whole requests */
  uint64_t requests, finds, find_fails, reserve_zero, cyc_find, cyc_slow, cyc_reserve, cyc_request;
  uint64_t hint_zero;        /* zero-slot reservations on the warp's hinted block (part of reserve_zero) */
} dsr_counters;

typedef struct dsr_heap dsr_heap;   /* opaque, host side, owned by the library */

/* ---------------------------------------------------------------- layout
 * Pure host computation of the heap layout for `ntypes` types in a buffer of
 * heap_bytes (P:286 M equal-size blocks; P:305-313 capacity; column
 * alignment reading R-LAYOUT).  Errors: ntypes not in [1, 8], a field size
 * not in {1,2,4,8,16}, a type > 64x the smallest, heap too small. */
dsr_status dsr_layout_compute(const dsr_type_desc* types, uint32_t ntypes, uint64_t heap_bytes,
                              dsr_layout* out);

/* ---------------------------------------------------------------- heap
 * Create a heap in the caller-owned device buffer dev_buf (heap_bytes
 * bytes, 256-byte aligned, must outlive the heap; e.g. a torch uint8 CUDA
 * tensor).  Launches the init kernel on `stream`: free = all 1 for bits < M
 * (P:350), allocated/active = 0, every object bitmap all 1
 * ("invalidated" == "uninitialized").  cfg may be NULL (defaults).
 * The returned heap object is owned by the library until dsr_heap_destroy. */
dsr_status dsr_heap_create(const dsr_type_desc* types, uint32_t ntypes, void* dev_buf, uint64_t heap_bytes,
                           const dsr_config* cfg, void* stream, dsr_heap** out);
/* Re-run the init kernel (all objects dropped).  Stream-ordered. */
dsr_status dsr_heap_reset(dsr_heap* h, void* stream);
/* Free the host object; never frees dev_buf. */
dsr_status dsr_heap_destroy(dsr_heap* h);
/* Copy the layout (host). */
dsr_status dsr_heap_layout(const dsr_heap* h, dsr_layout* out);
/* Change r / flags / seed for subsequent launches. */
dsr_status dsr_heap_configure(dsr_heap* h, const dsr_config* cfg);

/* ---------------------------------------------------------------- operations
 * parallel_new<T>(n, args): constructor `ctor_id` runs for ids
 * 0..n-1; objects are allocated with warp-aggregated device new.  args
 * (args_bytes bytes, host memory) is copied into kernel parameter space; its
 * struct type is fixed by ctor_id (see the DSR_C_* list). */
dsr_status dsr_parallel_new(dsr_heap* h, uint32_t type, uint64_t n, uint32_t ctor_id, const void* args,
                            size_t args_bytes, void* stream);

/* parallel_do<T, method>(args): snapshot the iteration bitmaps
 * (P:291), compact allocated[T] into the block list R with warp ballots and
 * prefix sums, then run `method_id` on every object of
 * T and of T's subtypes that exists at launch -- one body kernel per type, in
 * type order (P:123 footnote); the block lists of all of them are built
 * before the first body runs.  Objects created during the pass are not visited.
 * The method may allocate any type, destroy objects of other types, and
 * destroy only `this` among T.  No host synchronisation. */
dsr_status dsr_parallel_do(dsr_heap* h, uint32_t type, uint32_t method_id, const void* args, size_t args_bytes,
                           void* stream);

/* The two halves of dsr_parallel_do, for callers that time them apart or
 * reuse one block list R for several passes over a type whose set of blocks
 * cannot change in between (e.g. a static Cell grid): the prologue builds R
 * (and the snapshot if `method_id` may allocate); the body runs the method
 * over the current R.  dsr_parallel_do == prologue + body. */
dsr_status dsr_doall_prologue(dsr_heap* h, uint32_t type, uint32_t method_id, void* stream);
dsr_status dsr_doall_body(dsr_heap* h, uint32_t type, uint32_t method_id, const void* args, size_t args_bytes,
                          void* stream);

/* Bulk slow path ahead of time: initialise up to `nblocks` empty blocks of
 * `type` (free.clear -> initialize_block -> allocated.set -> active.set, the
 * slow path of Alg. 1) in one parallel kernel, so that a following
 * burst of device new finds active blocks on the fast path.  Fewer blocks are
 * initialised if the free bitmap runs out (no error).  Stream-ordered. */
dsr_status dsr_reserve_blocks(dsr_heap* h, uint32_t type, uint64_t nblocks, void* stream);
/* Quiescent: return every allocated block of `type` that holds no object to
 * the free bitmap (invalidate, active.clear, allocated.clear, free.set; Alg. 2
 * l.7-11).  Used after dsr_reserve_blocks.  Stream-ordered. */
dsr_status dsr_trim(dsr_heap* h, uint32_t type, void* stream);

/* Launch a compiled user kernel `kernel_id` over n logical threads that may
 * call device new/destroy -- e.g. the microbenchmark's allocation
 * kernel or the Linux Scalability kernels.  args as above. */
dsr_status dsr_launch(dsr_heap* h, uint32_t kernel_id, uint64_t n, const void* args, size_t args_bytes,
                      void* stream);

/* Number of live objects of `type` = sum over allocated[T] of used slots,
 * written as one u64 to dev_out (device pointer).  Stream-ordered. */
dsr_status dsr_live_count(dsr_heap* h, uint32_t type, uint64_t* dev_out, void* stream);
/* Same, synchronising, into host memory. */
dsr_status dsr_live_count_sync(dsr_heap* h, uint32_t type, uint64_t* host_out, void* stream);

/* Synchronise `stream`; return and clear the sticky device error
 * (DSR_ERR_OOM / DSR_ERR_RETRY_BUDGET; in a -DDSR_DEBUG build also
 * DSR_ERR_INVARIANT for an object access that failed its bounds check) or
 * DSR_OK. */
dsr_status dsr_poll_error(dsr_heap* h, void* stream);

/* Quiescent audit (synchronising): hierarchy consistency of every bitmap
 * (Definition), free/allocated partition of [0, M), active ⊆
 * allocated, active iff non-full, block type ids, padding bits
 * (P:978), no empty allocated block.  *failures_out (host, may be NULL) gets
 * the number of violations; returns DSR_ERR_INVARIANT if any. */
dsr_status dsr_check_invariants(dsr_heap* h, void* stream, uint64_t* failures_out);

/* Fragmentation F over all allocated blocks (synchronising), and the
 * number of allocated blocks per type (host array of ntypes, may be NULL). */
dsr_status dsr_fragmentation(dsr_heap* h, double* out, uint64_t* blocks_per_type, void* stream);

/* Device counters (synchronising; zero unless DSR_F_STATS). */
dsr_status dsr_stats(dsr_heap* h, dsr_counters* out, void* stream);
dsr_status dsr_stats_reset(dsr_heap* h, void* stream);

/* Copy raw heap state to host memory for parity tests (synchronising):
 * what = 0: alloc_bm[M] (u64); 1: type[M] (u8); 2: words of the free bitmap;
 * 3: words of allocated[type]; 4: words of active[type]; 5: R[M] (u32) and
 * the R count.  Bitmap words are level 0 first, then level 1, ...
 * (layout.level_words).  *used gets the bytes written. */
dsr_status dsr_copy_state(dsr_heap* h, uint32_t what, uint32_t type, void* host_out, size_t cap, size_t* used,
                          void* stream);

/* Canonical dump of the live objects of `type` (synchronising; SURVEY c.8):
 * each live object as one packed record -- its fields in declaration order,
 * field_bytes[f] bytes each (little endian), no padding -- with the records
 * sorted lexicographically by their bytes, so the dump does not depend on
 * placement (which block and slot an object got).  host_buf gets the
 * records if cap is large enough; *used = live x record bytes either way
 * (DSR_ERR_INVALID when cap < *used).  Rebuilds the do-all block list R. */
dsr_status dsr_canonical_dump(dsr_heap* h, uint32_t type, void* host_buf, size_t cap, size_t* used, void* stream);

/* The device-side heap descriptor: a POD that kernels take by value.  User
 * kernels compiled outside this library against the device header
 * paper_1810_11765_b200/csrc/dsr_device.cuh call dsr::dsr_new,
 * dsr::dsr_destroy and dsr::field_ptr on it like the library's own kernels
 * (new / destroy from GPU code), and every host call of this
 * header keeps working on the same heap.  out (host) receives the view;
 * out_bytes must equal dsr_device_view_bytes(). */
size_t dsr_device_view_bytes(void);
dsr_status dsr_device_view(const dsr_heap* h, void* out, size_t out_bytes);

/* Roofline denominator for the allocator's atomics ("allocs/s
 * ... as a fraction of the measured atomic peak").  Launches one persistent
 * grid in which every thread issues `iters` 64-bit atomicOr WITH return value
 * (the allocator's RMW form, atom.global.or.b64) on the u64 words of dev_buf
 * (bytes, device, caller-owned, contents overwritten):
 *   mode 0  hashed, independent addresses over the buffer (size it to fit L2
 *           for the L2 atomic-ALU peak: every bitmap word the allocator
 *           touches is L2-resident)
 *   mode 1  every thread on word 0 (same-address serialisation)
 * *ops_out (host) receives the number of atomics issued; time the call with
 * events on `stream`.  DSR_ERR_INVALID if bytes < 8 or iters == 0. */
/* CUDA IPC for the peer-memory exchanges: export the device
 * allocation that contains dev_ptr as a 64-byte handle (handle_out, host) and
 * dev_ptr's byte offset in it (*offset_out, host; caching allocators such as
 * torch's hand out pieces of larger blocks), open another process's handle
 * into this one (*dev_ptr_out: the block's base, usable by kernels on the
 * current device -- over NVLink when the memory lives on a peer GPU; add the
 * offset), and close it.  DSR_ERR_CUDA when the driver refuses (e.g. no P2P
 * path between the GPUs). */
dsr_status dsr_ipc_handle(void* dev_ptr, void* handle_out, uint64_t* offset_out);
dsr_status dsr_ipc_open(const void* handle, void** dev_ptr_out);
dsr_status dsr_ipc_close(void* dev_ptr);

dsr_status dsr_probe_atomics(void* dev_buf, uint64_t bytes, uint32_t mode, uint32_t iters, uint64_t* ops_out,
                             void* stream);

/* Number of kernels this library launched since load (host counter). */
uint64_t dsr_kernel_launches(void);
const char* dsr_status_str(dsr_status s);
/* Library build string: "sm_100a <git/date>". */
const char* dsr_build_info(void);

/* ================================================================ ids
 * Method ids (dsr_parallel_do), constructor ids (dsr_parallel_new) and user
 * kernel ids (dsr_launch) compiled into this library, with their argument
 * structs (copied by value).  Device pointers inside args are device memory.
 */

/* ---- allocator microbenchmark (BASELINE configs[4], SURVEY c.4) ----
 * types: 0 = A{3 x u32}, 1 = B{4 x u32}, 2 = C{6 x u32} */
/* thread t -> new [A,A,B,C][(t0+t)&3].  in == NULL: field k of thread t's
 * object = low32(key(seed, 0, MB_FIELD, 16t + k)) computed on the device.
 * in != NULL (t0 % 4 == 0): the field values come from the caller, packed per
 * 4 threads as 16 u32 = {A: 3, A: 3, B: 4, C: 6 fields}, i.e. thread t0 + i
 * reads in[16 (i / 4) + {0, 3, 6, 10}[i % 4] + k]; ceil(n / 4) groups.
 *   in_host == 0: `in` is a device pointer.
 *   in_host != 0: `in` is a HOST pointer (pinned for asynchronous copies).
 *     dsr_launch copies it into one of two heap-owned device staging buffers
 *     on the heap's own copy stream (waiting until the kernel that last read
 *     that buffer has finished) and makes `stream` wait for the copy, so the
 *     copy of one launch overlaps the work already queued on `stream`.  The
 *     host buffer must stay valid until the copy completes (stream-ordered:
 *     synchronise `stream` before reusing it). */
typedef struct { uint64_t seed; uint64_t t0; const uint32_t* in; uint32_t in_host; uint32_t pad_; } dsr_mb_new_args;
typedef struct { uint64_t* out3; } dsr_mb_reduce_args;           /* out3[0..2] += (count, sum, xor) */
enum {
  DSR_K_MB_NEW = 1,          /* args dsr_mb_new_args; fields k = low32(key(seed,0,MB_FIELD,16t+k)) or from `in` */
  /* The same objects and fields, allocated with warp-cooperative bulk requests
   * (reading R-BULK): a warp takes 3072 consecutive t and reserves
   * all objects of one type of them with one request -- fresh blocks up to 64
   * per free-bitmap atomic, or free slots of active blocks found by 32
   * parallel rotated searches (P:649-654 generalised to many slots).  Which
   * object lands in which slot differs; every object and field value is the
   * same as DSR_K_MB_NEW's. */
  DSR_K_MB_NEW_BULK = 8,
  DSR_M_MB_REDUCE = 1,       /* args dsr_mb_reduce_args (no allocation: reads the allocation bitmap) */
  DSR_M_MB_FREE_ODD = 2,     /* args none: destroy(this) if field0 & 1 */
  DSR_M_MB_FREE_ALL = 3      /* args none: destroy(this) */
};

/* ---- Linux Scalability ----
 * one type of 64 B (16 x u32); thread t allocates n objects, stored to
 * handles[t*n + i]; the free kernel destroys them. */
typedef struct { uint64_t* handles; uint32_t per_thread; uint32_t type; } dsr_ls_args;
enum { DSR_K_LS_ALLOC = 2, DSR_K_LS_FREE = 3 };

/* ---- single-thread replay / torture (test kernels) ---- */
typedef struct {
  const uint32_t* ops;       /* pairs (op, arg): op 0 = new type arg, op 1 = destroy handle of op #arg */
  uint64_t nops;
  uint64_t* handles_out;     /* one per op (0 for destroy) */
} dsr_replay_args;
typedef struct {
  uint64_t seed;
  uint32_t iters;            /* alloc/free rounds per thread */
  uint32_t keep;             /* 1: keep the survivors; 0: free everything at the end */
  uint64_t* ledger;          /* per thread up to 8 live handles at the end (0 = none) */
  uint64_t* errors;          /* canary mismatches */
} dsr_torture_args;
enum { DSR_K_REPLAY = 4, DSR_K_TORTURE = 5 };
typedef struct { uint64_t* out; uint64_t* count; } dsr_collect_args;   /* out[atomic++] = this */
enum { DSR_M_COLLECT = 4 };    /* any type: append every visited handle */

/* ---- inheritance test kernels ----
 * Types of a hierarchy whose root has fields {u32 id, u32 acc} (every
 * subtype inherits them as fields 0 and 1; further fields f >= 2 are the
 * subtype's own, each set to (id * (f + 1)) truncated to its size). */
typedef struct {
  uint64_t* handles;             /* K_INH_NEW: handles[i] = the new object of thread i */
  uint32_t ntypes;               /* K_INH_NEW: thread i creates type i % ntypes */
  uint32_t spawn_id0;            /* M_INH_SPAWN: id offset of the spawned objects */
  unsigned long long* out;       /* M_INH_SUM: out[2T] += 1, out[2T+1] += acc + own fields; M_INH_SPAWN: out[0] += 1 */
  uint64_t* vals;                /* K_INH_READ: vals[i] = acc | is_a(handles[i], k) << (32 + k) */
} dsr_inh_args;
enum {
  DSR_K_INH_NEW = 6, DSR_K_INH_READ = 7,
  DSR_M_INH_BUMP = 5,            /* acc = 3 acc + id, through the inherited columns */
  DSR_M_INH_SUM = 6,             /* per runtime type: count and checksum */
  DSR_M_INH_SPAWN = 7            /* out[0] += 1; new object of the next type (i % ntypes + 1) */
};

/* ---- Game of Life (BASELINE configs[0]/[3], reading R-GOL) ----
 * types: 0 = Alive{cell u32, is_new u8, action u8}, 1 = Candidate{cell u32, action u8}
 * cell: device array of W*H handles (0 = empty). */
typedef struct {
  uint64_t* cell; uint32_t W, H; const uint8_t* alive0; uint32_t* dump;
  /* Row-sharded mode (ghost = 1): the grid arrays have H + 2 rows,
   * rows 0 and H + 1 are ghost copies of the neighbour shards' boundary rows
   * (no wrap in y; the torus closes through the exchange).  halo: 4 x W bytes
   * (bit 0 next-alive, bit 1 new-alive): [0] my row 1 (to the shard above),
   * [1] my row H (to the shard below), [2] received for ghost row 0, [3] for
   * ghost row H + 1. */
  uint32_t ghost; uint8_t* halo;
  /* Optional alive-bit mirror (variant; NULL = off): 1 bit per cell (ghost rows
   * included), row pitch ceil(W / 32) u32 words, zeroed by the caller before
   * DSR_K_GOL_INIT_ALIVE.  Kept equal to "the cell holds an Alive" at every
   * pass boundary (set on spawn, cleared on death, ghost rows from the halo);
   * the prepare passes then count neighbours from it instead of loading 8
   * handles (SURVEY D4 "state-grid mirror" design knob). */
  uint32_t* bits;
  /* Peer-memory halo exchange ("fused pack + send"; peer_up =
   * NULL: off).  peer_up / peer_down: the halo buffers of the shards above and
   * below, mapped into this process (dsr_ipc_open over NVLink / NVSwitch when
   * they live on other GPUs; plain device pointers when they are other shards
   * on this GPU; my own buffer when P = 1).  halo is then
   * DSR_GOL_PEER_HALO_BYTES(W) bytes: received masks double-buffered by the
   * parity of `gen` -- segment 2 + 2 (gen & 1) from the shard above, 3 + 2 (gen & 1)
   * from the shard below -- and at DSR_GOL_PEER_FLAGS(W) two u32 flags (from
   * above, from below) that the neighbours set to gen + 1 (system-scope
   * release) after writing generation gen's masks.  gen: the generation. */
  uint8_t* peer_up;
  uint8_t* peer_down;
  uint32_t gen;
} dsr_gol_args;
#define DSR_GOL_PEER_FLAGS(W) ((6u * (W) + 15u) & ~15u)
#define DSR_GOL_PEER_HALO_BYTES(W) (DSR_GOL_PEER_FLAGS(W) + 16u)
enum {
  DSR_K_GOL_INIT_ALIVE = 10,     /* n = W*H (W*(H+2) sharded); Alive(c) for alive0[c] (+ ghost cells) */
  DSR_K_GOL_INIT_CAND = 11,      /* n as above; Candidate(c) for dead c with >= 1 alive neighbour */
  DSR_K_GOL_HALO_PACK = 12,      /* n = W: after pass 3, masks of the boundary rows into halo[0], halo[1] */
  DSR_K_GOL_HALO_APPLY = 13,     /* n = W: before pass 4, ghost rows from halo[2], halo[3]; Candidates on
                                    empty boundary cells next to a remote new Alive (owner computes).
                                    Peer mode: waits until both flags reach gen + 1, reads the gen-parity slots */
  DSR_K_GOL_HALO_PUSH = 14,      /* n = W, peer mode only: after pass 3, the masks of my row 1 / row H written
                                    straight into the halo buffers of the shards above / below (one kernel,
                                    no staging, no collective), then their flags := gen + 1 */
  DSR_M_GOL_CAND_PREPARE = 10,   /* type 1 */
  DSR_M_GOL_ALIVE_PREPARE = 11,  /* type 0 */
  DSR_M_GOL_CAND_UPDATE = 12,    /* type 1 (allocates Alive) */
  DSR_M_GOL_ALIVE_UPDATE = 13,   /* type 0 (allocates Candidate) */
  DSR_M_GOL_DUMP = 14,           /* any type: dump[cell] = kind | is_new << 8 | action << 16 */
  /* The same four methods as cell-tiled do-alls: the objects of the type are
   * enumerated through the cell grid (each sits in exactly one cell) instead
   * of the block list, so no prologue runs; prepare passes stage (8+2) x
   * (128+2) tiles of handles in shared memory, update passes visit cells in
   * row-major order so a warp's new objects come from neighbouring cells.
   * Results are those of the block-list passes.  Not with `bits`. */
  DSR_M_GOL_CAND_PREPARE_TILED = 15, DSR_M_GOL_ALIVE_PREPARE_TILED = 16,
  DSR_M_GOL_CAND_UPDATE_TILED = 17, DSR_M_GOL_ALIVE_UPDATE_TILED = 18
};

/* ---- Wa-Tor (BASELINE configs[1], reading R-WATOR) ----
 * types: 0 = Fish{cell, target, egg: u32}, 1 = Shark{cell, target, egg, energy: u32},
 *        2 = Cell{id u32, agent u64, req[5] u8}
 * cells: device array of W*H Cell handles (filled by DSR_C_WT_CELL). */
typedef struct {
  uint64_t* cells;
  uint32_t W, H;
  uint32_t FB, SB, SS;
  uint64_t seed;
  uint32_t step;
  const uint8_t* kind0; const uint32_t* egg0; const uint32_t* energy0;   /* init only */
  uint32_t* out_kind; uint32_t* out_egg; uint32_t* out_energy;           /* dump only */
  unsigned long long* counters;   /* [0] fish born, [1] sharks born, [2] eaten, [3] starved */
  /* Row-sharded mode (ghost = 1): this shard owns global rows
   * y0 .. y0+H-1 of a W x Hg torus; the cell arrays have H + 2 rows, rows 0 and
   * H + 1 are ghost cells mirroring the neighbour shards' boundary rows (their
   * agent field holds a type-only handle, never dereferenced).  Keys use global
   * cell ids.  halo: DSR_WT_HALO_BYTES(W) bytes, each segment [side][W] with
   * side 0 = my row 1 / ghost row 0 (the shard above), side 1 = my row H /
   * ghost row H + 1 (the shard below); "out" segments go to the neighbour,
   * "in" segments are the neighbour's "out" of the opposite side:
   *   req  (u8)        requests into the neighbour's boundary cells
   *   grant (u8)       decisions for the neighbour's boundary agents
   *   occ  (u8)        agent kind (0 none, 1 fish, 2 shark) of my boundary rows
   *   mig  (3 x u32)   migrating agents {kind, egg, energy} (kind 0 = none) */
  uint32_t ghost, y0, Hg;
  uint8_t* halo;
  /* If non-NULL, the step number is read from this device word instead of
   * `step` (so one captured CUDA graph of a step can be replayed while the
   * caller advances the word on the device). */
  const uint32_t* step_dev;
} dsr_wator_args;
#define DSR_WT_HALO_REQ_OUT(W)   0u
#define DSR_WT_HALO_REQ_IN(W)    (2u * (W))
#define DSR_WT_HALO_GRANT_OUT(W) (4u * (W))
#define DSR_WT_HALO_GRANT_IN(W)  (6u * (W))
#define DSR_WT_HALO_OCC_OUT(W)   (8u * (W))
#define DSR_WT_HALO_OCC_IN(W)    (10u * (W))
#define DSR_WT_HALO_MIG_OUT(W)   ((12u * (W) + 15u) & ~15u)
#define DSR_WT_HALO_MIG_IN(W)    (DSR_WT_HALO_MIG_OUT(W) + 24u * (W))
#define DSR_WT_HALO_BYTES(W)     (DSR_WT_HALO_MIG_IN(W) + 24u * (W))
enum {
  DSR_C_WT_CELL = 20,            /* parallel_new<Cell>(W*H) (W*(H+2) sharded): cells[i] = this */
  DSR_K_WT_INIT_AGENTS = 21,     /* n = W*H (W*(H+2)): Fish/Shark from kind0/egg0/energy0 (+ ghost kinds) */
  /* sharded mode, n = W each, in step order around the exchanges of each half step:
   * prepare -> REQ_PACK | exchange req | REQ_APPLY -> decide | exchange grant | GRANT_APPLY
   * -> update | exchange mig | MIG_APPLY -> OCC_PACK | exchange occ | OCC_APPLY */
  DSR_K_WT_HALO_REQ_PACK = 22,   /* ghost cells' incoming requests -> req out; clears grant/mig out */
  DSR_K_WT_HALO_REQ_APPLY = 23,  /* req in -> my boundary cells' req[0] (row 1) / req[2] (row H) */
  DSR_K_WT_HALO_GRANT_APPLY = 24,/* grant in -> target of my boundary agents := the ghost cell */
  DSR_K_WT_HALO_MIG_APPLY = 25,  /* mig in -> new agents on my boundary cells (a shark eats a fish there) */
  DSR_K_WT_HALO_OCC_PACK = 26,   /* my boundary rows' agent kinds -> occ out */
  DSR_K_WT_HALO_OCC_APPLY = 27,  /* occ in -> ghost cells' agent kinds */
  DSR_M_WT_CELL_PREPARE = 20, DSR_M_WT_FISH_PREPARE = 21, DSR_M_WT_CELL_DECIDE_FISH = 22,
  DSR_M_WT_FISH_UPDATE = 23, DSR_M_WT_SHARK_PREPARE = 24, DSR_M_WT_CELL_DECIDE_SHARK = 25,
  DSR_M_WT_SHARK_UPDATE = 26, DSR_M_WT_DUMP = 27
};

/* ---- N-body with collisions (BASELINE configs[2], reading R-NBODY) ----
 * type 0 = Body{x, y, vx, vy, fx, fy, m: f32; id, target, incoming: u32; merged: u8}
 * Id-indexed device arrays of length n_total shared by all passes (on every
 * rank of a multi-GPU run; the rank owns ids [id_lo, id_hi)):
 *   S[4*id + {0,1,2,3}] = (x, y, m, 0) snapshot (m = 0: dead id)
 *   V[2*id + {0,1}]     = (vx, vy) snapshot
 *   target[id], incoming[id] (u32, 0xFFFFFFFF = NONE), shandle[id] (local handles only) */
typedef struct {
  float* S;
  float* V;
  uint32_t* target;
  uint32_t* incoming;
  uint64_t* shandle;
  const float *x0, *y0, *vx0, *vy0, *m0;  /* init only: id_hi - id_lo bodies */
  float G, dt, eps, R;
  uint32_t n_total, id_lo, id_hi;
  float* out;                         /* dump: 6 floats per id (x, y, vx, vy, m, alive) */
  float* scratch;                     /* all-pairs partials: >= 2 * ceil(n_total/4096) * (id_hi - id_lo) floats */
  float* live;                        /* the all-pairs passes' live list (device, caller-owned, scratch):
                                         >= 4 * n_total + ceil(n_total/4096) floats; each 4096-id chunk of S
                                         compacted to its bodies with m > 0 (x, y, m, id bits), ascending id */
  /* Peer-memory all-gathers (npeers = 0: off, the caller
   * all-gathers S, V and target itself).  The snapshot pass writes each of
   * this rank's bodies into S / V here AND into every peer's S / V (the
   * peers' buffers of the same epoch parity, mapped into this process:
   * dsr_ipc_open over NVLink, or other shards' buffers on this GPU), and
   * DSR_K_NB_CLEAR_SNAPSHOT clears this rank's rows in all of them; after
   * the snapshot DSR_K_NB_SIGNAL sets flag slot `rank` of every peer's
   * `flags` to epoch + 1 (system-scope release); DSR_M_NB_FORCE and
   * DSR_M_NB_PREPARE_MERGE first make the stream wait (cuStreamWaitValue32)
   * until every other slot of this rank's flags[0 .. world) reached
   * epoch + 1.  target: after prepare_merge, DSR_K_NB_PUSH_TARGET writes this
   * rank's rows of target into every peer's target and sets their slot
   * world + rank to step + 1; DSR_K_NB_CLAIM waits for slots world .. 2 world.
   * The caller alternates S / V by epoch parity and target by step parity
   * (two buffers each), which makes the exchanges safe without a barrier. */
  uint32_t npeers;                    /* number of other ranks (<= 7) */
  uint32_t rank, world;               /* this rank; ranks in the group (peer i = rank (rank + 1 + i) % world) */
  uint32_t epoch;                     /* snapshot epoch (2 per step); for the target exchange: step */
  uint32_t* flags;                    /* this rank's flags: 2 * world u32 (device) */
  float* peer_S[7];
  float* peer_V[7];
  uint32_t* peer_target[7];
  uint32_t* peer_flags[7];
} dsr_nbody_args;
enum {
  DSR_C_NB_BODY = 30,            /* parallel_new<Body>(id_hi - id_lo): body i gets id id_lo + i */
  DSR_M_NB_SNAPSHOT = 30,        /* S[id], V[id] = own state; shandle[id] = this */
  DSR_M_NB_FORCE = 31,           /* compute_force for own ids: tiled all-pairs over S (device_do) */
  DSR_M_NB_MOVE = 32,
  DSR_M_NB_PREPARE_MERGE = 33,   /* target[id] for own ids over S */
  DSR_M_NB_CLAIM = 34,           /* over ALL ids (redundant per rank): incoming[target[i]] = min i */
  DSR_M_NB_ABSORB = 35,
  DSR_M_NB_DELETE_MERGED = 36,   /* destroy(this) iff incoming[target] == id and target[target] == NONE */
  DSR_M_NB_DUMP = 37,
  DSR_K_NB_CLEAR_SNAPSHOT = 30,  /* n = n_total: S.m = 0, shandle = 0, target = incoming = NONE
                                    (peer mode: this rank's rows of S in every peer too) */
  DSR_K_NB_CLAIM = 31,           /* n = n_total: the claim pass over the (gathered) target array
                                    (peer mode: waits for the peers' target rows first) */
  DSR_K_NB_SIGNAL = 32,          /* n = n_total, peer mode: the snapshot's rows are in every peer: set their flags */
  DSR_K_NB_PUSH_TARGET = 33      /* n = n_total, peer mode: this rank's target rows into every peer + their flags */
};

/* ---- Static-allocation baseline of Wa-Tor ----
 * "Baselines (SOA/AOS) are application variants without any dynamic memory
 * allocation ... In category (3), classes are merged with the underlying
 * static cell data structure".  The Wa-Tor rules, keys and
 * request / decide protocol of the object version (reading R-WATOR) on
 * cell-indexed SOA device arrays, no heap: its results equal the object
 * version's and the oracle's (or_wator_dense) bit for bit, so its time prices
 * DynaSOAr's dynamic allocation on the same GPU.
 *   kind[c]   u8   0 empty, 1 fish, 2 shark        (in/out, W*H)
 *   egg[c]    u32  breeding counter                (in/out, W*H; 0 on empty cells)
 *   energy[c] u32  shark energy                    (in/out, W*H; 0 unless shark)
 *   target[c] u32  scratch, W*H, all 0xFFFFFFFF before the first call (the call leaves it so)
 *   req       u8   scratch, W*H rounded up to a multiple of 4 bytes, 4-byte aligned,
 *                  all zero before the first call (the call leaves it so)
 *   counters  u64[4] or NULL: += fish born, sharks born, fish eaten, sharks starved
 * All pointers are caller-owned device memory; the call only enqueues work.
 * Torus W x H, W, H >= 3, W*H < 2^32.  DSR_ERR_INVALID on a bad argument. */
typedef struct {
  uint32_t W, H;
  uint32_t FB, SB, SS;
  uint32_t step;                  /* step number of the first step (RNG key) */
  uint64_t seed;
  uint8_t* kind; uint32_t* egg; uint32_t* energy;
  uint32_t* target; uint8_t* req;
  unsigned long long* counters;
} dsr_wator_static_args;
/* `steps` consecutive Wa-Tor steps (6 kernels each: prepare / decide / update
 * for fish, then sharks) on `stream` (cudaStream_t as void*, NULL = default). */
dsr_status dsr_wator_static_step(const dsr_wator_static_args* args, uint32_t steps, void* stream);

/* ---- Static-allocation baseline of N-body ----
 * The six passes of reading R-NBODY on id-indexed SOA device arrays, no heap:
 *   S[4*id + {0,1,2,3}] = (x, y, m, 0)  (in/out; m = 0: dead id)
 *   V[2*id + {0,1}]     = (vx, vy)      (in/out)
 *   target, incoming    u32[n] scratch
 *   scratch             f32, >= 2 * ceil(n / 4096) * n (all-pairs partials)
 * The all-pairs passes are the heap version's kernels over S; the per-body
 * passes repeat its operations in its order, so the state after any number of
 * steps equals the heap version's (dsr_nbody_args runs) bit for bit.
 * Caller-owned device memory; enqueues work on `stream` only. */
typedef struct {
  float* S; float* V; uint32_t* target; uint32_t* incoming; float* scratch;
  float G, dt, eps, R;
  uint32_t n;
  uint32_t merges;      /* 0: App2 N-Body (force + move only) */
  float* live;          /* live list scratch, as dsr_nbody_args.live */
} dsr_nbody_static_args;
dsr_status dsr_nbody_static_step(const dsr_nbody_static_args* args, uint32_t steps, void* stream);

/* ---- Static-allocation baseline of Game of Life (NEXT-4) ----
 * B3/S23 on a W x H torus of u8 cells (0 dead, 1 alive): `cur` and `next`
 * (device, W*H bytes each, caller-owned) are swapped every step; after the
 * call the state is in `cur` (odd step counts end with one device copy).
 * One kernel per generation, (8 + 2) x (128 + 2) cell tiles in shared memory.
 * Equals the object version's alive map (and textbook Life) every step. */
typedef struct { uint32_t W, H; uint8_t* cur; uint8_t* next; } dsr_gol_static_args;
dsr_status dsr_gol_static_step(const dsr_gol_static_args* args, uint32_t steps, void* stream);

#ifdef __cplusplus
}
#endif
#endif
