// Kernel declarations and launch-parameter blocks shared by kernels.cu and
// capi.cu.  Parameter blocks are passed by value (kernel parameter space).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "ma_device.cuh"

namespace ma {

constexpr int kK1Threads = 256;
constexpr int kK1Unroll = 8;  // 8 x 16 B in flight per thread per batch (A/B: MA_K1_UNROLL=4)
constexpr int kK2Threads = 256;
constexpr int kMaxSegs = 96;  // sub-groups per K2 launch (8.5 KB of kernel parameters)

// Cross-rank flag exchange over peer memory (NVLink P2P through CUDA IPC
// mappings), fused into K1's last CTA.  slots[bank][r] on every rank holds
// rank r's (epoch << 1 | flag) for epochs of parity `bank`; two banks make it
// impossible for a rank that runs one step ahead to overwrite a value a slower
// rank has not read yet.
constexpr int kMaxRanks = 64;

struct XchgDev {
    unsigned long long* peer_slots[kMaxRanks];  // rank r's slot array, mapped here
    unsigned long long* my_slots;               // this rank's slot array [2][world]
    unsigned int* counter;                      // K1 CTAs finished (last CTA exchanges)
    unsigned int* error;                        // set before a fatal timeout / poison trap
    unsigned long long* epoch;                  // exchanges completed (device-side, so a
                                                // captured graph replays correctly)
    uint32_t world;
    uint32_t rank;
    unsigned long long timeout_ns;              // MA_PEER_TIMEOUT_S (default 300 s)
};

// Posted into every peer's slots by a rank that gives up on an exchange: a
// value no epoch can take (epochs are < 2^63).  Whoever reads it traps too.
constexpr unsigned long long kXchgPoison = ~0ull;

struct K1Args {
    const uint4* body;      // 16-byte aligned vector body
    const void* raw;        // element 0 (for the unaligned head/tail)
    uint64_t n;             // elements
    uint64_t head;          // elements before `body`
    uint64_t nvec;          // uint4 vectors in the body
    uint64_t index_base;    // added to reported indices (chunked host scans)
    uint32_t* flag;
    uint64_t* first;        // kTrack only
    int kind;
    uint32_t elem_bytes;
    int early_exit;
    const XchgDev* xchg;    // non-null: exchange the flag with all ranks at the end
    uint64_t keep_from;     // vectors from here on are loaded with an L2 evict_last
                            // policy (the tail K2 reads last; nvec = none)
};

struct Seg {
    float* p;
    float* m;
    float* v;
    const void* g;
    void* w;
    uint64_t n;
    uint64_t head;        // scalar elements before the co-aligned body
    uint64_t nvec;        // VEC-element vectors in the body
    uint64_t tile_begin;  // first tile of this sub-group in the launch
    uint64_t tile_end;
    uint32_t vector_ok;
};

struct SegTable {
    Seg seg[kMaxSegs];
    uint32_t count;
    uint64_t total_tiles;
};

// Fused weight all-gather (ma_stepper_apply_allgather_async): K2 also
// stores each rank's updated working weights into every peer's full-length
// weight buffer over NVLink (CUDA IPC mappings); delta[r] is the byte offset
// from a local working-weight address to the same element in peer r's buffer.
constexpr int kMaxAgPeers = 7;  // one NVSwitch box: 8 ranks
struct PeerW {
    long long delta[kMaxAgPeers];
    uint32_t n;
};

struct AdamArgs {
    AdamConsts c;
    // explicit step (ma_adam_step*): used when st == nullptr
    float scale, bc1, bc2;
    const uint32_t* skip;    // optional skip flag
    const StepDev* st;       // optional device-resident scaler
    // (st != nullptr: the step scalars are read from st, precomputed by
    //  k_step_prepare / k_step_finish from the bias-correction table)
    PeerW peers;             // fused all-gather targets (launch_k2_allgather only)
    // 128-byte gradient lines the preceding stepper check left under an L2
    // evict_last policy: the update returns them to normal
    // priority so they do not outlive the step in L2
    const char* demote;
    uint64_t demote_lines;
};

// Host-side launchers (defined next to the kernels in kernels.cu so every
// template instantiation lives in one translation unit).
// oneshot: grid = ceil(nvec / (kK1Threads * kK1Unroll)) CTAs, one block of
// vectors each (production); otherwise the persistent grid-stride form (A/B)
void launch_k1(const K1Args& a, bool track, int unroll, bool oneshot, unsigned grid,
               cudaStream_t st);
// K2 variants (MA_K2_VARIANT, A/B record in DESIGN.md): persistent grid-stride
// 0 thread-contiguous VEC=8, 1 thread-contiguous VEC=4, 2 warp-contiguous
// U=2, 3 U=1 + prefetch, 4 U=2 + prefetch, 5 U=4, 6/9 forced occupancy,
// 7/8 load cache hints, 10/11 TMA bulk-copy ring, 12 approximate-math probe;
// one tile per CTA: 13 U=2, 14 U=4, 15 U=1; **20 = 14 launched as a
// programmatic dependent of K1 (production)**, 21 = 20 with the tile's loads
// before griddepcontrol.wait, 22 = 14 with the tiles back to front.  Dtype
// pairs other than (bf16, bf16) only carry kK2DefaultVariant.
constexpr int kK2DefaultVariant = 20;
int k2_effective_variant(int gk, int wk, int variant);
void k2_variant_shape(int variant, int* vec, int* tile_vectors, bool* stream);
// one tile per CTA: grid = total_tiles + trailing CTAs for the scalar remainder
bool k2_variant_oneshot(int variant);
int k2_blocks_per_sm(int gk, int wk, int variant);
// K2 (production one-shot shape) with the fused weight all-gather
void launch_k2_allgather(int gk, int wk, const SegTable& tab, const AdamArgs& a, unsigned grid,
                         cudaStream_t st);
void launch_k2(int gk, int wk, int variant, const SegTable& tab, const AdamArgs& a, unsigned grid,
               cudaStream_t st);
// K3 (bf16 state): Seg p/m/v point at uint16 arrays; one tile of
// kK3Slots x 256 slots of 4 elements per CTA, trailing CTAs for remainders.
constexpr int kK3Slots = 4;
int k3_slots(int gk, int variant);
// elements per vector (slot) of the K3 variant: 4, or 8 for A/B variants 4/5
int k3_vec(int gk, int variant);
int k3_tiles_per_cta(int gk, int variant);
int k3_blocks_per_sm(int gk, int variant);
void launch_k3(int gk, int variant, const SegTable& tab, const AdamArgs& a, unsigned grid,
               cudaStream_t st);
// K4: gradient reduce-scatter with the overflow check in its epilogue
// (SURVEY §8(f) row 2).  dst[i] = post_scale * sum_r src[r][i] (fp32, rank
// order), stored in the stepper's gradient kind, non-finite test on the
// stored value.  8-element units; one tile of rs_units(src kind) x 256 units
// per CTA, trailing CTAs for the scalar head/tail (or the whole range when the
// sources and dst cannot be co-aligned).
constexpr int rs_units(int sk) { return sk == kF32 ? 2 : 4; }
struct RsArgs {
    const void* src[kMaxRanks];  // each source at the element `head` is measured from
    void* dst;
    uint64_t n;
    uint64_t head;   // scalar elements before the 16-byte-aligned body
    uint64_t nvec;   // 8-element units in the body
    uint64_t tiles;  // CTAs of the vector body
    uint32_t nsrc;
    float post_scale;
    uint32_t* flag;
    const XchgDev* xchg;  // non-null: exit barrier + flag OR fused into the last CTA
};
void launch_reduce_check(int sk, int dk, const RsArgs& a, unsigned grid, cudaStream_t st);
// units per thread the launch for (source kind, source count) uses (host tile size)
int rs_units_for(int sk, uint32_t nsrc);
// all ranks meet at the exchange object's next epoch (one warp; peers'
// slots over NVLink); a peer missing for MA_PEER_TIMEOUT_S stops every rank
void launch_peer_barrier(const XchgDev* x, cudaStream_t st);
// bc_table holds (1-b1^t, 1-b2^t) for t = bc_first, bc_first + 1, ...
void launch_step_finish(StepDev* st, StepLog* log, const float2* bc_table, uint64_t bc_first,
                        const AdamConsts& c, cudaStream_t s);
void launch_step_prepare(StepDev* st, const float2* bc_table, uint64_t bc_first,
                         const AdamConsts& c, cudaStream_t s);
void launch_gen_weights(int wk, float* p, uint16_t* w, uint64_t n, uint64_t base, uint64_t seed,
                        unsigned grid, cudaStream_t st);
void launch_gen_grads(int gk, int wk, void* g, const uint16_t* w, uint64_t n, uint64_t base,
                      uint64_t seed, uint64_t step, const float* d_scale, float scale,
                      unsigned grid, cudaStream_t st);
void launch_plant(void* buf, int dtype, uint64_t index, uint32_t bits, cudaStream_t st);
// Speculative update during the host-gradient transfer
// (ma_stepper_check_host_spec_async): after a sub-group's speculative K2,
// marker = value if this step's flag is still clear (the applied sub-groups
// are then exactly the first `marker` speculated ones); at the end of the
// step, when the (exchanged) flag is set, the backups of those sub-groups
// are copied back, and the marker is re-armed either way.
constexpr int kMaxSpecCopies = 384;  // 96 sub-groups x (p, m, v, w) (12 KB of kernel parameters)
struct SpecCopy {
    const void* src;
    void* dst;
    uint64_t bytes;
    uint32_t group;  // index among the speculated sub-groups
};
struct SpecRestore {
    SpecCopy c[kMaxSpecCopies];
    uint32_t count;
};
void launch_spec_mark(const StepDev* st, uint32_t* marker, uint32_t value, cudaStream_t s);
void launch_spec_restore(const SpecRestore& r, const StepDev* st, uint32_t* marker, unsigned grid,
                         cudaStream_t s);
// producer-side check: one tile of ingest_units(sk) x 256 eight-element
// units per CTA over [head, head + 8 * nvec), trailing CTAs for the rest
struct IngestArgs {
    const void* src;
    void* dst;
    uint64_t n, head, nvec, tiles;
    const float* d_scale;
    uint32_t* flag;
};
int ingest_units(int sk);
void launch_ingest(int sk, int dk, const IngestArgs& a, unsigned grid, cudaStream_t st);
void launch_cast_sweep(int kind, int log2, uint64_t* out, uint64_t nblocks);
void launch_mask_sweep(int kind, unsigned long long* mismatches, unsigned grid);
void launch_fast_sweep(int mode, const float* divs, uint64_t count, uint64_t seed,
                       unsigned long long* bad, unsigned grid);

}  // namespace ma
