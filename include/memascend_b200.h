/*
 * memascend_b200.h — C ABI of the B200-native MemAscend optimizer hot path.
 *
 * libmemascend_b200.so exports exactly the functions below (plain pointers,
 * sizes and status codes; no C++ or torch types).  It replaces, on sm_100a,
 * the reference's CPU hot path in /root/reference/proj:
 *
 *   fused_overflow_check   proj/include/memascend/overflow.hpp:56-62, proj/src/overflow.cpp:73-145
 *   adam_step_fp32         proj/include/memascend/optimizer.hpp:48-50, proj/src/optimizer.cpp:103-109
 *   adam_step_bf16         proj/include/memascend/optimizer.hpp:54-57, proj/src/optimizer.cpp:111-118
 *   fp16/bf16 cast-back    proj/include/memascend/halfprec.hpp:25-74, proj/src/simulator.cpp:461-467
 *   LossScaler + step loop proj/include/memascend/optimizer.hpp:19-35, proj/src/simulator.cpp:427-492
 *   PinnedAllocator        proj/src/pinned.cpp:98-148 ("registered" becomes cudaHostRegister)
 *   pseudo_gradient etc.   proj/include/memascend/simulator.hpp:23-42 (synthetic workload)
 *
 * The drop-in C++ API (headers under include/memascend/, namespace memascend) is a
 * thin layer over these entry points; INTEGRATION.md shows the ctypes / C++
 * bindings a maintainer adds.
 *
 * Conventions
 *  - Every function returns 0 (MA_OK) or a status.  Statuses 1..17 are
 *    1 + memascend::ErrorCode (proj/include/memascend/error.hpp:9-27) so the
 *    C++ layer rethrows memascend::Error with the same code; MA_ERR_CUDA and
 *    MA_ERR_NO_DEVICE extend it.  ma_last_error() describes the last failure
 *    on the calling thread.
 *  - "_async" functions take a cudaStream_t (as void*) and return once the
 *    work is enqueued; their pointers must be device-accessible (device
 *    memory, or host memory registered through ma_host_register /
 *    cudaHostRegister).  The functions without the suffix are synchronous
 *    like the reference: they accept device, registered-host or pageable-host
 *    pointers and return with results visible on the host.
 *  - Element kinds: MA_DT_F32 / MA_DT_BF16 / MA_DT_F16 (MA_DT_NONE = absent).
 *  - There is no CPU fallback: without a CUDA device every compute entry
 *    point fails with MA_ERR_NO_DEVICE.
 */
#ifndef MEMASCEND_B200_H
#define MEMASCEND_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MA_ABI_VERSION 1

#if defined(__GNUC__)
#define MA_API __attribute__((visibility("default")))
#else
#define MA_API
#endif

enum ma_status {
    MA_OK = 0,
    MA_ERR_INVALID_ARGUMENT = 1, /* ErrorCode::invalid_argument */
    MA_ERR_OUT_OF_MEMORY = 2,
    MA_ERR_OVERFLOW = 3,
    MA_ERR_LIFECYCLE = 4,
    MA_ERR_UNKNOWN_REGION = 5,
    MA_ERR_POOL_EXHAUSTED = 6,
    MA_ERR_SIZE_VIOLATION = 7,
    MA_ERR_ALREADY_CHECKED_OUT = 8,
    MA_ERR_NOT_FOUND = 9,
    MA_ERR_STORAGE_FULL = 10,
    MA_ERR_DEVICE_ERROR = 11,
    MA_ERR_CAPABILITY = 12,
    MA_ERR_IO_ERROR = 13,
    MA_ERR_ALIGNMENT = 14,
    MA_ERR_BUSY = 15,
    MA_ERR_UNCALIBRATED = 16,
    MA_ERR_BAD_CONFIG = 17,
    MA_ERR_CUDA = 100,      /* a CUDA runtime call failed */
    MA_ERR_NO_DEVICE = 101, /* no usable sm_100 device: there is no CPU fallback */
    MA_ERR_NCCL = 102       /* an NCCL call failed (or libnccl.so.2 is not loadable) */
};

enum ma_dtype { MA_DT_F32 = 0, MA_DT_BF16 = 1, MA_DT_F16 = 2, MA_DT_NONE = 3 };

/* AdamHyper, proj/include/memascend/optimizer.hpp:9-15 */
typedef struct ma_adam_hyper {
    float lr;
    float beta1;
    float beta2;
    float eps;
    float weight_decay;
} ma_adam_hyper;

/* ------------------------------------------------------------------ */
/* library / device                                                   */
MA_API const char* ma_last_error(void);
MA_API int ma_abi_version(void);
/* Current device ordinal, SM count and compute capability. */
MA_API int ma_device_info(int* device, int* sm_count, int* cc_major, int* cc_minor);

/* ------------------------------------------------------------------ */
/* K1 — fused overflow check (overflow.cpp:73-145).
 * ORs "all exponent bits set" over n elements of kind g_dtype into *d_flag
 * (device uint32, NOT cleared here: accumulate several buffers into one flag
 * and clear it yourself).  d_first_index (device uint64 initialised to
 * UINT64_MAX, may be NULL) receives atomicMin of the offending indices. */
MA_API int ma_overflow_check_async(const void* grads, uint64_t n, int g_dtype, uint32_t* d_flag,
                            uint64_t* d_first_index, void* stream);

/* Synchronous form with the reference's OverflowResult semantics. */
MA_API int ma_overflow_check(const void* grads, uint64_t n, int g_dtype, int track_first_index,
                      int* overflow, uint64_t* first_index);

/* ------------------------------------------------------------------ */
/* K2 — fused unscale + Adam/AdamW + cast-back (optimizer.cpp:26-44,
 * 103-109; halfprec.hpp:25-74).  p, m, v fp32 in place; g of kind g_dtype;
 * w_out (kind w_dtype, or MA_DT_NONE) receives the rounded working weights.
 * bc1/bc2 = 1 - powf(beta, t) are computed on the host with glibc powf
 * exactly as optimizer.cpp:20-24.  If d_skip_flag != NULL and *d_skip_flag
 * != 0 when the kernel runs, nothing is touched (the skip step). */
MA_API int ma_adam_step_async(float* p, float* m, float* v, const void* g, int g_dtype, uint64_t n,
                       uint64_t t, const ma_adam_hyper* h, float loss_scale, void* w_out,
                       int w_dtype, const uint32_t* d_skip_flag, void* stream);

/* Synchronous, any memory (device / registered host / pageable host). */
MA_API int ma_adam_step(float* p, float* m, float* v, const void* g, int g_dtype, uint64_t n,
                 uint64_t t, const ma_adam_hyper* h, float loss_scale, void* w_out, int w_dtype);

/* K3 — bf16 optimizer state (optimizer.cpp:83-93,111-118), synchronous. */
MA_API int ma_adam_step_bf16(uint16_t* p, uint16_t* m, uint16_t* v, const float* g, uint64_t n,
                      uint64_t t, const ma_adam_hyper* h, float loss_scale);

/* ------------------------------------------------------------------ */
/* Step driver: the composition of simulator.cpp:427-492 with the loss
 * scaler kept on the device, so a whole step (check -> optional cross-rank
 * OR -> update -> scaler) is enqueued without a host round trip.
 *
 *   per step:  ma_stepper_check_async(...)   for every gradient buffer
 *              [allreduce(max) of *ma_stepper_flag(s) across ranks]
 *              ma_stepper_apply_async(...)   for every sub-group
 *              ma_stepper_finish_async(...)  scaler + counters, re-arms
 *
 * t (the Adam step) counts APPLIED updates, not steps
 * (simulator.cpp:360,444,456).  bc1/bc2 come from a host-computed glibc-powf
 * table indexed on the device by t. */
typedef struct ma_stepper ma_stepper;

typedef struct ma_subgroup {
    float* p;         /* fp32 master */
    float* m;         /* fp32 momentum */
    float* v;         /* fp32 variance */
    const void* g;    /* scaled gradients, stepper g_dtype */
    void* w;          /* working weights, stepper w_dtype (NULL if MA_DT_NONE) */
    uint64_t n;
} ma_subgroup;

typedef struct ma_step_state {
    float scale;           /* LossScaler::scale after the last finished step */
    uint32_t clean_steps;  /* LossScaler::clean_steps */
    uint64_t updates;      /* applied updates (Adam t of the last update) */
    uint64_t steps;        /* finished steps */
    uint32_t last_overflow;
    uint32_t growth_interval;
} ma_step_state;

/* d_state: optional caller-owned device buffer of MA_STEPPER_STATE_BYTES
 * (e.g. a framework tensor, so the flag can be all-reduced in place); NULL
 * lets the library allocate it.  Layout: uint32 flag at byte 0, float scale
 * at byte 8 (see ma_stepper_flag / ma_stepper_scale). */
#define MA_STEPPER_STATE_BYTES 64
MA_API int ma_stepper_create(const ma_adam_hyper* h, float init_scale, uint32_t growth_interval,
                      int g_dtype, int w_dtype, void* d_state, ma_stepper** out);
MA_API int ma_stepper_destroy(ma_stepper* s);
MA_API int ma_stepper_check_async(ma_stepper* s, const void* g, uint64_t n, void* stream);
/* Host-buffer ingest: copies the step's gradients from PINNED host memory
 * into dev_g on copy_stream in chunk_elems pieces and runs K1 on each piece
 * on `stream` as soon as it lands, so the check overlaps the PCIe transfer
 * (the staged H2D of PAPER.md §4.4 / north-star item (1)). */
MA_API int ma_stepper_check_host_async(ma_stepper* s, const void* host_g, void* dev_g, uint64_t n,
                                       uint64_t chunk_elems, void* stream, void* copy_stream);
/* The same check, with the update of every sub-group whose gradients have
 * landed started at once while the flag is still clear (its p/m/v/w first
 * copied to `backup`, device memory of backup_bytes; sub-groups in order
 * while it has room, at most 96, their g tiling dev_g contiguously), so the
 * update overlaps the PCIe transfer.  Complete the step with
 * ma_stepper_apply_spec_async (same groups; after any flag exchange), which
 * updates the rest and, when the step's flag is set, restores the
 * speculated sub-groups from their backups — bit for bit the plain
 * check -> apply result either way — then ma_stepper_finish_async. */
MA_API int ma_stepper_check_host_spec_async(ma_stepper* s, const void* host_g, void* dev_g,
                                            uint64_t n, uint64_t chunk_elems,
                                            const ma_subgroup* groups, uint32_t count,
                                            void* backup, uint64_t backup_bytes, void* stream,
                                            void* copy_stream);
MA_API int ma_stepper_apply_spec_async(ma_stepper* s, const ma_subgroup* groups, uint32_t count,
                                       void* stream);
/* Cross-rank skip decision fused into K1 (replaces the all-reduce(max) of
 * the flag).  Each rank creates an exchange object, publishes its 64-byte
 * CUDA IPC handle, and opens everybody's handles (rank order); then, per
 * step, the LAST check of the step goes through ma_stepper_check_xchg_async:
 * K1's last CTA writes this rank's flag into every peer's slot over NVLink
 * (peer memory mapped with CUDA IPC), waits for all peers' slots of this
 * step, and leaves the OR in the local flag, so the following apply skips or
 * updates identically on every rank.  All ranks must call it the same number
 * of times.  A peer that does not arrive within MA_PEER_TIMEOUT_S seconds
 * (environment, default 300) is FATAL for the whole job, never a local skip:
 * the waiting rank posts a poison value into every peer's slots and traps
 * (its CUDA context reports cudaErrorLaunchFailure / MA_ERR_CUDA from then
 * on), and every rank that reads the poison traps as well — ranks cannot
 * diverge (one skipping while another updates).  ma_xchg_error reports 1
 * only while the context is still usable (i.e. never after a trap). */
#define MA_IPC_HANDLE_BYTES 64
typedef struct ma_xchg ma_xchg;
MA_API int ma_xchg_create(int world, int rank, ma_xchg** out, void* ipc_handle_out);
MA_API int ma_xchg_open(ma_xchg* x, const void* all_handles);
MA_API int ma_xchg_error(ma_xchg* x, int* timed_out);
MA_API int ma_xchg_destroy(ma_xchg* x);
MA_API int ma_stepper_check_xchg_async(ma_stepper* s, const void* g, uint64_t n, ma_xchg* x,
                                       void* stream);

/* Producer-side fused check: dst[i] = src[i] * scale
 * stored in the stepper's gradient kind — the scaled copy into the flat
 * buffer of simulator.cpp:401-405, with the device-resident loss scale — and
 * the overflow test applied to the stored values in the same pass (sets the
 * step's flag).  Replaces ma_stepper_check_async for buffers produced this
 * way: the gradients are read once per step instead of twice. */
MA_API int ma_stepper_ingest_async(ma_stepper* s, const void* src, int src_dtype, void* dst,
                                   uint64_t n, void* stream);
/* Reduce-scatter epilogue form of the producer-side check (SURVEY §8(f)
 * row 2, "the NCCL reduce-scatter epilogue"; K4): dst[i] = post_scale *
 * (srcs[0][i] + srcs[1][i] + ... ) summed in fp32 in source order, NaN stored
 * as the canonical quiet NaN, written in the stepper's gradient kind, with
 * the overflow test of overflow.hpp:46-51 applied to the stored values (sets
 * the step's flag).  srcs are any device-loadable pointers (local buffers or
 * peer memory); the caller orders their production before this call. */
MA_API int ma_stepper_reduce_check_async(ma_stepper* s, const void* const* srcs, int nsrc,
                                         int src_dtype, uint64_t n, float post_scale, void* dst,
                                         void* stream);
/* Multi-process form over NVLink peer memory.  Every rank shares its
 * full-length gradient buffer (n_total elements of dtype) once: ma_rs_create
 * returns a MA_RS_HANDLE_BYTES record, the records of all ranks are gathered
 * in rank order (any host channel) and passed to ma_rs_open.  Per step,
 * ma_stepper_reduce_scatter_async reduces elements [base, base+n) of all
 * ranks' buffers into dst: a one-warp entry barrier (all ranks' gradients are
 * complete), then K4 reading every peer over NVLink, whose last CTA is the
 * exit barrier (nobody overwrites gradients still being read) and the OR of
 * all ranks' flags — the stepper's flag is the global skip decision when the
 * call completes, with no separate collective.  A peer missing for
 * MA_PEER_TIMEOUT_S seconds stops the job (poison + trap on every rank, as
 * for ma_stepper_check_xchg_async): no rank overwrites gradients a peer may
 * still read, and no rank's decision differs from another's. */
typedef struct ma_rs ma_rs;
#define MA_RS_HANDLE_BYTES 192
MA_API int ma_rs_create(int world, int rank, const void* grads, uint64_t n_total, int dtype,
                        ma_rs** out, void* handle_out);
MA_API int ma_rs_open(ma_rs* r, const void* all_handles);
MA_API int ma_rs_error(ma_rs* r, int* timed_out);
MA_API int ma_rs_destroy(ma_rs* r);
MA_API int ma_stepper_reduce_scatter_async(ma_stepper* s, ma_rs* r, uint64_t base, uint64_t n,
                                           float post_scale, void* dst, void* stream);
/* Update fused with the weight all-gather (the collective that follows the
 * optimizer step in ZeRO data parallelism: every rank needs every partition's
 * new working weights for the next forward).  `ag` is an ma_rs created over
 * each rank's FULL-LENGTH working-weight buffer (dtype = the stepper's
 * w_dtype) and opened with all ranks' records.  groups[k].w must lie inside
 * this rank's buffer; K2 stores every updated working weight into this
 * rank's buffer AND, over NVLink through the IPC mappings, at the same offset
 * into every peer's buffer — no separate all-gather pass, the peer stores
 * overlap the HBM-bound update.  An entry barrier (all ranks are done with
 * the previous weights) and an exit barrier (all pushes complete) bracket it;
 * a skipped step stores nothing anywhere.  At most 8 ranks. */
MA_API int ma_stepper_apply_allgather_async(ma_stepper* s, const ma_subgroup* groups,
                                            uint32_t count, ma_rs* ag, void* stream);
/* Device uint32 holding this step's overflow flag (for the cross-rank OR). */
MA_API uint32_t* ma_stepper_flag(ma_stepper* s);
/* Device float holding the current loss scale (gradient producers read it). */
MA_API float* ma_stepper_scale(ma_stepper* s);
MA_API int ma_stepper_apply_async(ma_stepper* s, const ma_subgroup* groups, uint32_t count,
                           void* stream);
/* Pure-bf16 optimizer mode (OptimPrecision::pure_bf16, optimizer.cpp:83-93,
 * simulator.cpp:470-486): p (the bf16 weights themselves), m and v are bf16
 * arrays updated in place by K3; g is the stepper's gradient kind. */
typedef struct ma_subgroup_bf16 {
    uint16_t* p;
    uint16_t* m;
    uint16_t* v;
    const void* g;
    uint64_t n;
} ma_subgroup_bf16;
MA_API int ma_stepper_apply_bf16_async(ma_stepper* s, const ma_subgroup_bf16* groups,
                                       uint32_t count, void* stream);
/* The speculative host-gradient check / decision (see
 * ma_stepper_check_host_spec_async) in the pure-bf16 mode: K3 on bf16
 * weights / m / v, which are what the backup holds. */
MA_API int ma_stepper_check_host_spec_bf16_async(ma_stepper* s, const void* host_g, void* dev_g,
                                                 uint64_t n, uint64_t chunk_elems,
                                                 const ma_subgroup_bf16* groups, uint32_t count,
                                                 void* backup, uint64_t backup_bytes,
                                                 void* stream, void* copy_stream);
MA_API int ma_stepper_apply_spec_bf16_async(ma_stepper* s, const ma_subgroup_bf16* groups,
                                            uint32_t count, void* stream);

/* Streamed update (configs 4/5: state offloaded to the pinned host pool).
 * groups[k].p/m/v live in registered host memory, .g/.w on the device.
 * Sub-group slices are staged through `slots` (2..16) device slots of
 * slot_elems fp32 x {p, m, v} (d_staging, 3 * slots * slot_elems floats):
 * H2D on h2d_stream, K2 on stream, D2H on d2h_stream, slot reuse ordered by
 * events, so the copy-in of slice k+1 and the write-back of k-1 overlap the
 * update of k (§4.4 double buffering).  Reads this step's flag
 * first (one 4-byte readback): a skipped step moves no state (*skipped = 1).
 * Returns with the work enqueued; `stream` is ordered after the last
 * write-back. */
MA_API int ma_stepper_apply_streamed(ma_stepper* s, const ma_subgroup* groups, uint32_t count,
                                     float* d_staging, uint64_t slot_elems, uint32_t slots,
                                     void* stream, void* h2d_stream, void* d2h_stream,
                                     int* skipped);
MA_API int ma_stepper_finish_async(ma_stepper* s, void* stream);
/* Synchronises the stepper's last stream and reads the scaler state. */
MA_API int ma_stepper_state(ma_stepper* s, ma_step_state* out);
/* Per-step log (overflow flag, scale after the step) of the most recent
 * min(count, 65536) steps, oldest first. */
MA_API int ma_stepper_history(ma_stepper* s, uint8_t* overflow, float* scale_after, uint64_t cap,
                       uint64_t* count);

/* Resume a run (checkpoint/restart): the Adam step count
 * (OptimizerState::step_t, optimizer.hpp:60-66) and the LossScaler's scale
 * and clean_steps (optimizer.hpp:19-35) of a saved run.  Synchronous.  The
 * next applied update uses t = updates + 1, exactly as the reference's
 * adam_step (optimizer.cpp:120-124) continues from a restored step_t. */
MA_API int ma_stepper_set_state(ma_stepper* s, float scale, uint32_t clean_steps,
                                uint64_t updates);

/* CUDA graph of a step chain: between graph_begin and graph_end every
 * *_async call on `stream` (a non-default stream) is captured instead of
 * executed — e.g. check -> ma_stepper_allreduce_flag_async -> apply ->
 * finish; ma_graph_launch then replays the whole chain with one launch.
 * Loss scale, skip flag and t live on the device, so one graph serves every
 * later step; `reserve_steps` sizes the bias-correction table the graph
 * holds (a launch beyond it fails with MA_ERR_LIFECYCLE: capture again).
 * The peer-memory collectives (check_xchg, reduce_scatter,
 * apply_allgather) keep their epoch on the device and replay correctly too.
 * Calls that synchronise with the host (apply_streamed / apply_swapped,
 * state, set_state) cannot be captured. */
typedef struct ma_graph ma_graph;
MA_API int ma_stepper_graph_begin(ma_stepper* s, uint64_t reserve_steps, void* stream);
MA_API int ma_stepper_graph_end(ma_stepper* s, void* stream, ma_graph** out);
MA_API int ma_graph_launch(ma_graph* g, void* stream);
MA_API int ma_graph_destroy(ma_graph* g);

/* ------------------------------------------------------------------ */
/* NCCL communicator (SURVEY §8(b) `ma_init(device, ncclUniqueId*, rank,
 * world)` / `ma_flag_allreduce_max`): the cross-rank OR of the skip flag as
 * one ncclAllReduce(max) of the uint32 flag on the compute stream, so every
 * rank makes the reference's single global decision (simulator.cpp:431-440).
 * Rank 0 creates the id (ma_comm_unique_id), every rank receives it over any
 * host channel and calls ma_comm_create on its own device (current CUDA
 * device).  libnccl.so.2 is resolved at run time (the copy torch already
 * loaded, else the system's); without it these return MA_ERR_NCCL. */
#define MA_NCCL_ID_BYTES 128
typedef struct ma_comm ma_comm;
MA_API int ma_comm_unique_id(void* id_out);
MA_API int ma_comm_create(const void* nccl_unique_id, int world, int rank, ma_comm** out);
MA_API int ma_comm_destroy(ma_comm* c);
MA_API int ma_comm_info(ma_comm* c, int* world, int* rank, int* nccl_version);
/* In-place ncclAllReduce(max) of `count` device uint32 values on `stream`. */
MA_API int ma_comm_allreduce_max_u32(ma_comm* c, uint32_t* d_buf, uint64_t count, void* stream);
/* The step's skip decision across ranks: all-reduce(max) of *ma_stepper_flag(s). */
MA_API int ma_stepper_allreduce_flag_async(ma_stepper* s, ma_comm* c, void* stream);

/* ------------------------------------------------------------------ */
/* Synthetic workload generators, bit-exact with simulator.hpp:23-42.
 * Element i of the buffer is global element (base + i). */
MA_API int ma_gen_seeded_weights_async(float* p, void* w, int w_dtype, uint64_t n, uint64_t base,
                                uint64_t seed, void* stream);
/* g[i] = cast(pseudo_gradient(seed, step, base+i, widen(w[i])) * scale);
 * scale is read from d_scale when non-NULL (e.g. ma_stepper_scale). */
MA_API int ma_gen_pseudo_grads_async(void* g, int g_dtype, const void* w, int w_dtype, uint64_t n,
                              uint64_t base, uint64_t seed, uint64_t step,
                              const float* d_scale, float scale, void* stream);
/* Plants one raw bit pattern (32-bit for F32, low 16 bits otherwise). */
MA_API int ma_plant_bits_async(void* buf, int dtype, uint64_t index, uint32_t bits, void* stream);

/* ------------------------------------------------------------------ */
/* Host memory (PinnedAllocator, pinned.cpp:98-148): page-lock an existing
 * allocation for DMA and device access (cudaHostRegisterPortable|Mapped). */
MA_API int ma_host_register(void* ptr, uint64_t bytes);
MA_API int ma_host_unregister(void* ptr);
/* 1 if ptr is device memory, 2 registered/pinned host, 0 pageable host. */
MA_API int ma_pointer_kind(const void* ptr, int* kind);
/* NUMA placement (multi-socket hosts, e.g. 8 x B200 on two sockets): the
 * node of the current device's PCIe root (-1 if unknown), and the node
 * backing a host address (-1 if unknown).  ma_host_register first prefers
 * the device's node for the region's pages (mbind, moving pages already
 * touched) unless MA_NUMA_BIND=0 — best effort, a no-op on one-node hosts. */
MA_API int ma_device_numa_node(int* node);
/* The same placement alone, for memory about to be first touched (call it
 * before filling a fresh allocation; ma_host_register would move the pages). */
MA_API int ma_host_place(void* ptr, uint64_t bytes);
MA_API int ma_host_numa_node(const void* ptr, int* node);

/* ------------------------------------------------------------------ */
/* Swap store (DirectIoEngine, proj/include/memascend/direct_io.hpp:23-180,
 * proj/src/direct_io.cpp): key-addressed tensors on raw or file-backed
 * devices opened with O_DIRECT, payloads padded to 4096 and striped in equal
 * granule counts across the devices, space claimed once per key (growth
 * abandons the old extents), a per-key busy guard (MA_ERR_BUSY), a JSON
 * manifest.  Host-side by design (north star item 4): these entry points do
 * file I/O only and need no GPU.  Backends: MA_IO_SYNC (pread/pwrite),
 * MA_IO_POSIX_AIO (lio_listio, the reference's), MA_IO_URING (new: one
 * io_uring per worker, queue_depth requests in flight across tasks);
 * MA_IO_AUTO picks io_uring when the kernel allows it, else POSIX AIO
 * (env MEMASCEND_IO_BACKEND=sync|aio|uring overrides). */
typedef struct ma_swap ma_swap;
typedef struct ma_swap_op ma_swap_op;
enum ma_io_backend { MA_IO_AUTO = 0, MA_IO_SYNC = 1, MA_IO_POSIX_AIO = 2, MA_IO_URING = 3 };
typedef struct ma_swap_device {
    const char* path;
    uint64_t capacity_bytes; /* positive multiple of 4096 */
    int kind;                /* 0 raw_block, 1 file_backed_virtual */
} ma_swap_device;
typedef struct ma_swap_config {
    uint32_t workers;     /* >= 1 (reference default 2) */
    uint32_t queue_depth; /* requests in flight per worker (reference default 8) */
    int backend;          /* ma_io_backend */
    int cache_bypass;     /* open with O_DIRECT */
    const char* manifest_path; /* NULL/"" = volatile table */
} ma_swap_config;
typedef struct ma_swap_extent {
    uint32_t device_index;
    uint64_t device_offset;
    uint64_t length;
} ma_swap_extent;
typedef struct ma_swap_stats {
    uint64_t bytes_written, bytes_read, write_requests, read_requests, submitted_ios,
        abandoned_bytes;
} ma_swap_stats;
typedef void (*ma_io_trace_fn)(void* user, uint32_t device, uint64_t offset, uint64_t length,
                               int write);
MA_API int ma_swap_create(const ma_swap_device* devs, uint32_t ndev, const ma_swap_config* cfg,
                          ma_swap** out);
MA_API int ma_swap_destroy(ma_swap* s); /* saves the manifest when configured */
/* allocate_extents: *count = number of extents (at most cap copied to out). */
MA_API int ma_swap_allocate(ma_swap* s, const char* key, uint64_t logical_bytes,
                            ma_swap_extent* out, uint32_t cap, uint32_t* count);
/* src/dst must be 4096-aligned and cover the padded length.  The _async
 * forms return an op to pass to ma_swap_wait (which frees it); the key stays
 * busy until then. */
MA_API int ma_swap_write(ma_swap* s, const char* key, const void* src, uint64_t src_bytes,
                         uint64_t logical_bytes);
MA_API int ma_swap_read(ma_swap* s, const char* key, void* dst, uint64_t dst_bytes,
                        uint64_t* logical_bytes);
MA_API int ma_swap_write_async(ma_swap* s, const char* key, const void* src, uint64_t src_bytes,
                               uint64_t logical_bytes, ma_swap_op** op);
MA_API int ma_swap_read_async(ma_swap* s, const char* key, void* dst, uint64_t dst_bytes,
                              ma_swap_op** op);
MA_API int ma_swap_wait(ma_swap_op* op, uint64_t* logical_bytes);
MA_API int ma_swap_contains(ma_swap* s, const char* key, int* out);
MA_API int ma_swap_location(ma_swap* s, const char* key, uint64_t* logical, uint64_t* padded,
                            ma_swap_extent* out, uint32_t cap, uint32_t* count);
/* All keys, sorted, NUL-separated; *needed = bytes required. */
MA_API int ma_swap_keys(ma_swap* s, char* buf, uint64_t cap, uint64_t* needed);
MA_API int ma_swap_get_stats(ma_swap* s, ma_swap_stats* out);
MA_API int ma_swap_info(ma_swap* s, int* backend, uint64_t* total_capacity,
                        uint32_t* device_count);
MA_API int ma_swap_set_trace(ma_swap* s, ma_io_trace_fn fn, void* user);
MA_API int ma_swap_save_manifest(ma_swap* s);
/* dir/vdev<i>.img, i < count, each `bytes` long (preallocated). */
MA_API int ma_swap_create_virtual_devices(const char* dir, uint32_t count, uint64_t bytes);
MA_API int ma_swap_uring_available(void);
/* SharedCursor (direct_io.hpp:69-92): per-device next-free offsets; with a
 * path the counters live in that file under flock (cross-process). */
typedef struct ma_cursor ma_cursor;
MA_API int ma_cursor_open(uint32_t devices, const char* path, ma_cursor** out);
MA_API int ma_cursor_close(ma_cursor* c);
MA_API int ma_cursor_advance(ma_cursor* c, uint32_t device, uint64_t bytes, uint64_t* old);
MA_API int ma_cursor_position(ma_cursor* c, uint32_t device, uint64_t* pos);
MA_API int ma_cursor_restore(ma_cursor* c, uint32_t device, uint64_t pos);

/* Swapped update (config 5: state on NVMe, simulator.cpp:453-469's
 * read master/m/v -> adam_step_fp32 -> write back, as a pipeline).  For a
 * group with keys, its fp32 master/m/v live in the swap store under
 * key_p/key_m/key_v (n <= slot_elems); for a group with NULL keys they live
 * in registered host memory at p/m/v (the DRAM tier).  g/w are on the
 * device.  Swapped groups are read into one of host_slots registered host
 * slots (h_staging, 4096-aligned, host_slots x 3 x align4096(4*slot_elems)
 * bytes) up to host_slots-1 groups ahead, copied into one of dev_slots
 * device slots (d_staging, dev_slots x 3 x slot_elems floats), updated by K2
 * on `stream`, copied back and written to the store by a writer thread
 * while later groups are read and updated.  A skipped step moves nothing
 * (*skipped = 1).  Returns when every swapped group is back in the store;
 * host-resident write-backs are ordered before `stream`. */
typedef struct ma_swap_group {
    const char* key_p;
    const char* key_m;
    const char* key_v;
    float* p;
    float* m;
    float* v;
    const void* g;
    void* w;
    uint64_t n;
} ma_swap_group;
MA_API int ma_stepper_apply_swapped(ma_stepper* s, ma_swap* e, const ma_swap_group* groups,
                                    uint32_t count, void* h_staging, uint32_t host_slots,
                                    float* d_staging, uint32_t dev_slots, uint64_t slot_elems,
                                    void* stream, void* h2d_stream, void* d2h_stream,
                                    int* skipped);
/* Pure-bf16 form (OptimPrecision::pure_bf16; simulator.cpp:470-486 swaps the
 * bf16 m/v under "m.<g>"/"v.<g>" with 2-byte elements): per group the bf16
 * momentum/variance come from the store (key_m/key_v) or the registered DRAM
 * tier (m/v), the bf16 weights p stay on the device and are updated in place
 * by K3.  Host slots are host_slots x 2 x align4096(2 * slot_elems) bytes,
 * device slots dev_slots x 2 x slot_elems bf16; slot_elems a multiple of 8.
 * 4 B per swapped parameter each way instead of 12. */
typedef struct ma_swap_group_bf16 {
    const char* key_m;
    const char* key_v;
    uint16_t* m;
    uint16_t* v;
    uint16_t* p;
    const void* g;
    uint64_t n;
} ma_swap_group_bf16;
MA_API int ma_stepper_apply_swapped_bf16(ma_stepper* s, ma_swap* e,
                                         const ma_swap_group_bf16* groups, uint32_t count,
                                         void* h_staging, uint32_t host_slots, void* d_staging,
                                         uint32_t dev_slots, uint64_t slot_elems, void* stream,
                                         void* h2d_stream, void* d2h_stream, int* skipped);

/* ------------------------------------------------------------------ */
/* Device-side adaptive pool + weight prefetch.
 * PAPER.md §4.2: the adaptive buffer pool "extends naturally to GDS-based
 * offloading, which necessitates similar buffer management on the GPU".
 * ma_dpool is that pool in HBM: one cudaMalloc'd backing carved into
 * exact-fit slot classes (pool.cpp:22-68 planning: stride = payload rounded
 * to 4096, classes laid out back to back); a tensor takes the tightest class
 * whose payload fits (pool.cpp:111-131).  ma_prefetcher is the layer-wise
 * parameter swapper of simulator.cpp:367-425 moved onto the GPU: tensors
 * submitted in order are read from the swap store into registered host
 * slots (store workers), copied into device slots on the prefetcher's copy
 * stream and handed out by acquire (the consumer's stream waits on the
 * copy's event; no host sync), and a slot returns to the pool at release
 * (reuse ordered after the consumer's work by an event).  Prefetch depth is
 * bounded by the device slots (the pool's in-flight blocks) and by
 * host_slots. */
typedef struct ma_dpool ma_dpool;
typedef struct ma_dpool_stats {
    uint64_t capacity_bytes;  /* sum of slot payloads (pool_capacity) */
    uint64_t backing_bytes;   /* HBM reserved (4096-rounded strides) */
    uint64_t peak_live_bytes; /* largest sum of checked-out payloads */
    uint64_t live_bytes;
    uint64_t checkout_count;
    uint64_t checkin_count;
} ma_dpool_stats;
MA_API int ma_dpool_create(const uint64_t* slot_payload_bytes, const uint32_t* slot_counts,
                           uint32_t nclasses, ma_dpool** out);
MA_API int ma_dpool_destroy(ma_dpool* p);
MA_API int ma_dpool_get_stats(ma_dpool* p, ma_dpool_stats* out);

typedef struct ma_prefetcher ma_prefetcher;
/* h_staging: registered host memory, 4096-aligned, host_slots x h_slot_bytes
 * (h_slot_bytes a multiple of 4096 covering the largest padded tensor). */
MA_API int ma_prefetcher_create(ma_swap* store, ma_dpool* pool, void* h_staging,
                                uint64_t h_slot_bytes, uint32_t host_slots, ma_prefetcher** out);
/* Queue `key` (a tensor in the store) for prefetch; keys are served in order. */
MA_API int ma_prefetch_submit(ma_prefetcher* f, const char* key);
/* Blocks until `key`'s copy is enqueued, makes `stream` wait for it and
 * returns its device address and logical length. */
MA_API int ma_prefetch_acquire(ma_prefetcher* f, const char* key, void* stream, void** dptr,
                               uint64_t* bytes);
/* Returns `key`'s device slot; its next user waits for `stream`'s work so far. */
MA_API int ma_prefetch_release(ma_prefetcher* f, const char* key, void* stream);
MA_API int ma_prefetcher_destroy(ma_prefetcher* f);

/* ------------------------------------------------------------------ */
/* Verification hooks (used by tests/; they run the product device code). */
/* FNV-1a-64 of every 2^block_log2 consecutive fp32->kind conversions over
 * all 2^32 inputs, through the same device cast K2 uses; out_host has
 * 2^(32-block_log2) entries. */
MA_API int ma_debug_cast_sweep(int kind, int block_log2, uint64_t* out_host);
/* Number of 32-bit (kind F32) or 16-bit patterns where K1's predicate
 * disagrees with !isfinite(); exhaustive. */
MA_API int ma_debug_mask_sweep(int kind, uint64_t* mismatches);
/* Verification of the hoisted-guard Adam fast path against the IEEE
 * intrinsics (see ma_device.cuh): mode 0 square root over every admitted
 * input, mode 1 division by each of `divisors` (bias corrections) over all
 * significands at eight exponents, mode 2 `samples` random (m_hat, den)
 * divisions.  Returns the number of bitwise mismatches and of inputs checked. */
MA_API int ma_debug_fast_sweep(int mode, const float* divisors, uint32_t ndiv, uint64_t samples,
                               uint64_t seed, uint64_t* mismatches, uint64_t* checked);

#ifdef __cplusplus
}
#endif

#endif /* MEMASCEND_B200_H */
