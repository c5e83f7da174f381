// Kernel declarations and launch-parameter blocks shared by kernels.cu and
// capi.cu.  Parameter blocks are passed by value (kernel parameter space).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "ma_device.cuh"

namespace ma {

constexpr int kK1Threads = 256;
constexpr int kK1Unroll = 4;  // 4 x 16 B in flight per thread per batch
constexpr int kK2Threads = 256;
constexpr int kMaxSegs = 96;  // sub-groups per K2 launch (8.5 KB of kernel parameters)

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

struct AdamArgs {
    AdamConsts c;
    // explicit step (ma_adam_step*): used when st == nullptr
    float scale, bc1, bc2;
    const uint32_t* skip;    // optional skip flag
    const StepDev* st;       // optional device-resident scaler
    const float2* bc_table;  // (1-b1^t, 1-b2^t) for t = 1.. when st != nullptr
};

template <bool kTrack>
__global__ void k1_overflow(K1Args a);

template <int GK, int WK, int VEC>
__global__ void k2_adam(SegTable tab, AdamArgs a);

__global__ void k3_adam_bf16(uint16_t* p, uint16_t* m, uint16_t* v, const float* g, uint64_t n,
                             AdamArgs a);

__global__ void k_step_finish(StepDev* st, StepLog* log);

template <int WK>
__global__ void k_gen_weights(float* p, uint16_t* w, uint64_t n, uint64_t base, uint64_t seed);

template <int GK, int WK>
__global__ void k_gen_grads(void* g, const uint16_t* w, uint64_t n, uint64_t base, uint64_t seed,
                            uint64_t step, const float* d_scale, float scale);

__global__ void k_plant(void* buf, int dtype, uint64_t index, uint32_t bits);

template <int K>
__global__ void k_cast_sweep(int log2, uint64_t* out, uint64_t nblocks);

__global__ void k_mask_sweep(int kind, unsigned long long* mismatches);

}  // namespace ma
