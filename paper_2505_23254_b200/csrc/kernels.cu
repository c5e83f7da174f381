// sm_100a kernels of the MemAscend optimizer hot path.
//
//   K1  k1_overflow        fused overflow check   (proj/src/overflow.cpp:45-145)
//   K2  k2_adam            unscale + AdamW + cast (proj/src/optimizer.cpp:26-44,103-109,
//                                                  proj/src/simulator.cpp:461-467)
//   K3  k3_adam_bf16       bf16-state Adam        (proj/src/optimizer.cpp:83-93,111-118)
//       k_step_finish      LossScaler + counters  (optimizer.hpp:19-35, simulator.cpp:438-491)
//       k_gen_*            synthetic workload     (simulator.hpp:23-42)
//
// All three are HBM-streaming kernels (no data reuse, no tensor-core work):
// 128-bit coalesced loads/stores, persistent grid-stride launches sized to
// the SM count, streaming cache hints (.cs = evict-first) so 10^2 GB of
// one-touch state does not thrash L2.
#include "kernels.cuh"

#include <cstdlib>
#include <type_traits>
#include <utility>

namespace ma {

// Programmatic dependent launch (sm_90+): a kernel launched with
// cudaLaunchAttributeProgrammaticStreamSerialization may start once every
// CTA of the previous kernel has executed launch_dependents (or exited);
// griddepcontrol.wait then blocks until that kernel has completed and its
// writes are visible.  Both are no-ops without a programmatic dependency.
__device__ __forceinline__ void pdl_trigger() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// K1's kept gradient tail back to normal L2 priority (applypriority only
// re-tags a line that is present; it neither evicts nor moves data), spread
// over the grid's first threads.  Measured without it: an L2-resident
// workload right after the step ran 12-17% slower
// (tools/l2_pollution_probe.py).
__device__ __forceinline__ void demote_kept(const char* base, uint64_t lines) {
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < lines;
         i += stride) {
        asm volatile("applypriority.global.L2::evict_normal [%0], 128;" ::"l"(base + i * 128)
                     : "memory");
    }
}

// ============================================================== K1
// One pass over the raw bits; each thread ORs (w & MASK) + INC over its
// 16-byte vectors, one warp vote at the end, one plain store of 1 by the
// first lane of any warp that saw a non-finite lane (idempotent, no atomics).
// Early exit (ScanConfig::early_exit, overflow.cpp:88-114): warps poll the
// flag once per unrolled batch and stop once any CTA has set it.
// ---- fused cross-rank exchange (last CTA of K1, warp 0) -------------------
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// Every rank's K1 ends here: the last CTA to finish publishes this rank's
// flag into slot [epoch & 1][rank] of every peer (remote stores over
// NVLink), then waits for all peers' entries of this epoch in its own slots
// and replaces the local flag by the OR — the all-reduce(max) of the skip
// decision without a separate collective launch.
//
// Failure is FATAL and shared, never a local decision: a rank whose peers do
// not all arrive within timeout_ns (MA_PEER_TIMEOUT_S, default 300 s, wall
// clock from %globaltimer) posts kXchgPoison into every peer's slots, sets
// its error word and traps; a rank that reads a poisoned slot does the same.
// No rank can therefore skip while another updates: a rank either completes
// the exchange with every peer's value or dies, and a peer that completed
// the exchange just before the poison landed dies at the next exchange —
// the job stops loudly instead of continuing with diverged optimizer state.
__device__ __forceinline__ unsigned long long global_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __noinline__ void xchg_abort(const XchgDev& x, unsigned lane) {
    for (uint32_t r = lane; r < x.world; r += 32) {
        st_release_sys(x.peer_slots[r] + x.rank, kXchgPoison);
        st_release_sys(x.peer_slots[r] + x.world + x.rank, kXchgPoison);
    }
    if (lane == 0) atomicExch(x.error, 1u);
    __threadfence_system();
    __trap();
}

// One warp: publish (epoch << 1 | local) to every rank, wait for every
// rank's value of this epoch; returns the OR of the flags.
__device__ uint32_t xchg_post_wait(const XchgDev& x, unsigned long long epoch, uint32_t local,
                                   unsigned lane) {
    const unsigned long long bank = epoch & 1ull;
    const unsigned long long val = (epoch << 1) | local;
    __threadfence_system();  // everything this rank wrote before is visible to the peers
    for (uint32_t r = lane; r < x.world; r += 32) {
        st_release_sys(x.peer_slots[r] + bank * x.world + x.rank, val);
    }
    uint32_t any = 0, failed = 0;
    const unsigned long long start = global_ns();
    for (uint32_t r = lane; r < x.world && !failed; r += 32) {
        for (;;) {
            const unsigned long long v = ld_acquire_sys(x.my_slots + bank * x.world + r);
            if (v == kXchgPoison) {
                failed = 1;
                break;
            }
            if ((v >> 1) == epoch) {
                any |= static_cast<uint32_t>(v & 1ull);
                break;
            }
            if (global_ns() - start > x.timeout_ns) {
                failed = 1;
                break;
            }
        }
    }
    if (__any_sync(0xFFFFFFFFu, failed != 0u)) xchg_abort(x, lane);
    return __any_sync(0xFFFFFFFFu, any != 0u);
}

// The exchange object's next epoch, read by lane 0 (the previous exchange on
// this object completed earlier in stream order) and broadcast to the warp;
// commit_epoch records it once every peer's value has been seen.
__device__ __forceinline__ unsigned long long next_epoch(const XchgDev& x, unsigned lane) {
    unsigned long long e = 0;
    if (lane == 0) e = *reinterpret_cast<volatile unsigned long long*>(x.epoch) + 1ull;
    return __shfl_sync(0xFFFFFFFFu, e, 0);
}
__device__ __forceinline__ void commit_epoch(const XchgDev& x, unsigned long long e,
                                             unsigned lane) {
    if (lane == 0) *reinterpret_cast<volatile unsigned long long*>(x.epoch) = e;
}

__device__ void exchange_epilogue(const XchgDev* xp, uint32_t* flag, unsigned lane) {
    __shared__ uint32_t is_last;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        is_last = atomicAdd(xp->counter, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!is_last || threadIdx.x >= 32) return;
    const XchgDev& x = *xp;
    __threadfence();
    const uint32_t local = *reinterpret_cast<volatile uint32_t*>(flag) != 0u;
    const unsigned long long epoch = next_epoch(x, lane);
    const uint32_t any = xchg_post_wait(x, epoch, local, lane);
    commit_epoch(x, epoch, lane);
    if (lane == 0) {
        *flag = any ? 1u : 0u;
        *x.counter = 0u;  // re-arm for the next launch (all CTAs have arrived)
        __threadfence();
    }
}

__device__ __forceinline__ void k1_exchange_epilogue(const K1Args& a, unsigned lane) {
    exchange_epilogue(a.xchg, a.flag, lane);
}

// Entry / exit barrier of the peer-memory collectives (same fatal rule).
__global__ void k_peer_barrier(const XchgDev* xp) {
    const unsigned lane = threadIdx.x & 31u;
    const unsigned long long epoch = next_epoch(*xp, lane);
    xchg_post_wait(*xp, epoch, 0u, lane);
    commit_epoch(*xp, epoch, lane);
}

// One-shot K1 (production): CTA b scans the U * 256 consecutive 16-byte
// vectors [b * U * 256, (b + 1) * U * 256) — all U loads in flight before
// the OR — and exits, so the block scheduler sweeps the buffer front to back
// (6.9 vs 6.2 TB/s for the grid-stride form, tools/layout_probe.cu).  A CTA
// that starts after the flag is already set skips its loads (the reference's
// cooperative early exit); with an exchange it still takes part in it.
// K1 load flavour for the vectors from keep_from on (the buffer's last
// MA_K1_KEEP_MB of a stepper check — an A/B option, default 0 = off;
// keep_from = nvec otherwise): 1 = L2 evict_last policy — those gradients
// stay in L2 while K2 streams p/m/v through it with evict-first accesses and
// K2's last tiles read them from L2; the update then demotes them
// (demote_kept).  2 = default caching for the tail.  Why it is off:
// DESIGN.md §3.5.
template <int LDK>
__device__ __forceinline__ uint4 k1_load(const uint4* p, uint64_t pol) {
    if constexpr (LDK == 0) return __ldcs(p);
    if constexpr (LDK == 2) return *p;  // default (evict_normal) caching
    uint4 r;
    asm volatile("ld.global.L2::cache_hint.v4.u32 {%0, %1, %2, %3}, [%4], %5;"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p), "l"(pol));
    return r;
}

template <bool kTrack, int U, int LDK = 0>
__global__ void __launch_bounds__(kK1Threads) k1_oneshot(K1Args a) {
    pdl_trigger();  // K2 (PDL launch) may be scheduled during K1's last wave
    const ScanWord sw = scan_word(a.kind);
    const unsigned lane = threadIdx.x & 31u;
    const uint32_t per_vec = 16u / a.elem_bytes;
    const uint64_t first = static_cast<uint64_t>(blockIdx.x) * U * blockDim.x + threadIdx.x;
    uint32_t acc = 0;
    const bool skip = !kTrack && a.early_exit && *reinterpret_cast<volatile uint32_t*>(a.flag) != 0u;
    if (!skip) {
        uint64_t pol = 0;
        if constexpr (LDK == 1) {
            asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
        }
        uint4 q[U];
        // only the CTAs that reach the kept tail take the per-vector test
        const bool keep = LDK != 0 && first - threadIdx.x + U * blockDim.x > a.keep_from;
        if (keep) {
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const uint64_t i = first + static_cast<uint64_t>(u) * blockDim.x;
                q[u] = i >= a.nvec ? make_uint4(0, 0, 0, 0)
                       : i >= a.keep_from ? k1_load<LDK>(a.body + i, pol) : __ldcs(a.body + i);
            }
        } else {
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const uint64_t i = first + static_cast<uint64_t>(u) * blockDim.x;
                q[u] = i < a.nvec ? __ldcs(a.body + i) : make_uint4(0, 0, 0, 0);
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            acc |= ((q[u].x & sw.mask) + sw.inc) | ((q[u].y & sw.mask) + sw.inc) |
                   ((q[u].z & sw.mask) + sw.inc) | ((q[u].w & sw.mask) + sw.inc);
        }
        if (kTrack && (acc & sw.top)) {
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const uint64_t i = first + static_cast<uint64_t>(u) * blockDim.x;
                if (i >= a.nvec) continue;
                const uint32_t w4[4] = {q[u].x, q[u].y, q[u].z, q[u].w};
                for (uint32_t e = 0; e < per_vec; ++e) {
                    const uint32_t word = w4[(e * a.elem_bytes) >> 2];
                    const uint32_t bits =
                        a.elem_bytes == 4 ? word : (word >> (16 * (e & 1u))) & 0xFFFFu;
                    if (elem_non_finite(bits, a.kind)) {
                        atomicMin(reinterpret_cast<unsigned long long*>(a.first),
                                  static_cast<unsigned long long>(a.index_base + a.head +
                                                                  i * per_vec + e));
                        break;
                    }
                }
            }
        }
    }
    if (blockIdx.x == 0) {  // unaligned head / tail elements
        const uint64_t tail_begin = a.head + a.nvec * per_vec;
        const uint64_t extra = a.head + (a.n - tail_begin);
        for (uint64_t k = threadIdx.x; k < extra; k += blockDim.x) {
            const uint64_t e = k < a.head ? k : tail_begin + (k - a.head);
            const uint32_t bits = a.elem_bytes == 4 ? reinterpret_cast<const uint32_t*>(a.raw)[e]
                                                    : reinterpret_cast<const uint16_t*>(a.raw)[e];
            if (elem_non_finite(bits, a.kind)) {
                acc |= sw.top;
                if (kTrack) {
                    atomicMin(reinterpret_cast<unsigned long long*>(a.first),
                              static_cast<unsigned long long>(a.index_base + e));
                }
            }
        }
    }
    if (__any_sync(0xFFFFFFFFu, (acc & sw.top) != 0u) && lane == 0) {
        *a.flag = 1u;
        if (a.xchg) __threadfence();
    }
    if (a.xchg) k1_exchange_epilogue(a, lane);
}

template <bool kTrack, int kK1Unroll>
__global__ void __launch_bounds__(kK1Threads) k1_overflow(K1Args a) {
    const ScanWord sw = scan_word(a.kind);
    const uint64_t tid = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    const unsigned lane = threadIdx.x & 31u;
    const uint32_t per_vec = 16u / a.elem_bytes;  // elements per uint4
    uint32_t acc = 0;

    // The trip count is warp-uniform (tested on the warp's first lane) so the
    // early-exit shuffle below is always executed by all 32 lanes.
    for (uint64_t base = tid; base - lane < a.nvec; base += stride * kK1Unroll) {
        uint4 q[kK1Unroll];
#pragma unroll
        for (int u = 0; u < kK1Unroll; ++u) {
            const uint64_t i = base + u * stride;
            q[u] = i < a.nvec ? __ldcs(a.body + i) : make_uint4(0, 0, 0, 0);
        }
        uint32_t batch = 0;
#pragma unroll
        for (int u = 0; u < kK1Unroll; ++u) {
            batch |= ((q[u].x & sw.mask) + sw.inc) | ((q[u].y & sw.mask) + sw.inc) |
                     ((q[u].z & sw.mask) + sw.inc) | ((q[u].w & sw.mask) + sw.inc);
        }
        if (kTrack && (batch & sw.top)) {
            // exact lowest offending index within this thread's vectors
#pragma unroll
            for (int u = 0; u < kK1Unroll; ++u) {
                const uint64_t i = base + u * stride;
                if (i >= a.nvec) continue;
                const uint32_t w4[4] = {q[u].x, q[u].y, q[u].z, q[u].w};
                for (uint32_t e = 0; e < per_vec; ++e) {
                    const uint32_t word = w4[(e * a.elem_bytes) >> 2];
                    const uint32_t bits =
                        a.elem_bytes == 4 ? word : (word >> (16 * (e & 1u))) & 0xFFFFu;
                    if (elem_non_finite(bits, a.kind)) {
                        atomicMin(reinterpret_cast<unsigned long long*>(a.first),
                                  static_cast<unsigned long long>(a.index_base + a.head +
                                                                  i * per_vec + e));
                        break;
                    }
                }
            }
        }
        acc |= batch;
        if (!kTrack && a.early_exit) {
            uint32_t seen = 0;
            if (lane == 0) seen = *reinterpret_cast<volatile uint32_t*>(a.flag);
            if (__shfl_sync(0xFFFFFFFFu, seen, 0) != 0) break;
        }
    }
    // unaligned head / tail elements (fewer than 16 bytes each) on CTA 0
    if (blockIdx.x == 0) {
        const uint64_t tail_begin = a.head + a.nvec * per_vec;
        const uint64_t extra = a.head + (a.n - tail_begin);
        for (uint64_t k = threadIdx.x; k < extra; k += blockDim.x) {
            const uint64_t e = k < a.head ? k : tail_begin + (k - a.head);
            const uint32_t bits = a.elem_bytes == 4
                                      ? reinterpret_cast<const uint32_t*>(a.raw)[e]
                                      : reinterpret_cast<const uint16_t*>(a.raw)[e];
            if (elem_non_finite(bits, a.kind)) {
                acc |= sw.top;
                if (kTrack) {
                    atomicMin(reinterpret_cast<unsigned long long*>(a.first),
                              static_cast<unsigned long long>(a.index_base + e));
                }
            }
        }
    }
    if (__any_sync(0xFFFFFFFFu, (acc & sw.top) != 0u) && lane == 0) {
        *a.flag = 1u;
        if (a.xchg) __threadfence();
    }
    if (a.xchg) k1_exchange_epilogue(a, lane);
}


// ============================================================== K2
// Per-step scalars of an explicit step (scale, bc1, bc2 from the host).
__device__ __forceinline__ void scalars_from(float scale, float bc1, float bc2,
                                             const AdamConsts& c, StepScalars& s) {
    s.scale = scale;
    s.bc1 = bc1;
    s.bc2 = bc2;
    s.scale_pow2 = exact_reciprocal(s.scale, &s.inv_scale);
    s.fast = s.scale_pow2 && fast_step_ok(s.bc1, s.bc2, c.eps, c.lr, c.lr_wd);
    s.y1 = s.fast ? rcp_refined(s.bc1) : 0.0f;
    s.y2 = s.fast ? rcp_refined(s.bc2) : 0.0f;
}

__device__ __forceinline__ bool resolve_step(const AdamArgs& a, StepScalars& s) {
    if (a.st != nullptr) {
        // device-resident scaler: the flag, the scale and the precomputed
        // scalars of t = updates + 1 in three independent loads (the skip
        // flag of a stepper launch is always st->flag)
        const uint4 h = *reinterpret_cast<const uint4*>(a.st);
        const float4 q = *reinterpret_cast<const float4*>(&a.st->inv_scale);
        const uint2 r = *reinterpret_cast<const uint2*>(&a.st->y2);
        if (h.x != 0u) return false;
        s.scale = __uint_as_float(h.z);
        s.inv_scale = q.x;
        s.bc1 = q.y;
        s.bc2 = q.z;
        s.y1 = q.w;
        s.y2 = __uint_as_float(r.x);
        s.scale_pow2 = (r.y & 1u) != 0u;
        s.fast = (r.y & 2u) != 0u;
        return true;
    }
    if (a.skip != nullptr && *a.skip != 0u) return false;
    scalars_from(a.scale, a.bc1, a.bc2, a.c, s);
    return true;
}

// vector of VEC fp32 lanes through float4 (VEC = 4 or 8)
template <int VEC>
__device__ __forceinline__ void ld_f32(const float* p, float (&x)[VEC]) {
    const float4* q = reinterpret_cast<const float4*>(p);
#pragma unroll
    for (int k = 0; k < VEC / 4; ++k) {
        const float4 t = __ldcs(q + k);
        x[4 * k + 0] = t.x;
        x[4 * k + 1] = t.y;
        x[4 * k + 2] = t.z;
        x[4 * k + 3] = t.w;
    }
}

template <int VEC>
__device__ __forceinline__ void st_f32(float* p, const float (&x)[VEC]) {
    float4* q = reinterpret_cast<float4*>(p);
#pragma unroll
    for (int k = 0; k < VEC / 4; ++k) {
        __stcs(q + k, make_float4(x[4 * k + 0], x[4 * k + 1], x[4 * k + 2], x[4 * k + 3]));
    }
}

// VEC 16-bit lanes: VEC=8 -> one uint4, VEC=4 -> one uint2
template <int VEC>
__device__ __forceinline__ void ld_u16(const uint16_t* p, uint32_t (&h)[VEC]) {
    if constexpr (VEC == 8) {
        const uint4 t = __ldcs(reinterpret_cast<const uint4*>(p));
        const uint32_t w[4] = {t.x, t.y, t.z, t.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            h[2 * k] = w[k] & 0xFFFFu;
            h[2 * k + 1] = w[k] >> 16;
        }
    } else {
        const uint2 t = __ldcs(reinterpret_cast<const uint2*>(p));
        h[0] = t.x & 0xFFFFu;
        h[1] = t.x >> 16;
        h[2] = t.y & 0xFFFFu;
        h[3] = t.y >> 16;
    }
}

template <int VEC>
__device__ __forceinline__ void st_u16(uint16_t* p, const uint32_t (&h)[VEC]) {
    if constexpr (VEC == 8) {
        __stcs(reinterpret_cast<uint4*>(p),
               make_uint4(h[0] | (h[1] << 16), h[2] | (h[3] << 16), h[4] | (h[5] << 16),
                          h[6] | (h[7] << 16)));
    } else {
        __stcs(reinterpret_cast<uint2*>(p), make_uint2(h[0] | (h[1] << 16), h[2] | (h[3] << 16)));
    }
}

template <int GK>
__device__ __forceinline__ float load_grad1(const void* g, uint64_t e) {
    if constexpr (GK == kF32) return reinterpret_cast<const float*>(g)[e];
    return widen<GK>(reinterpret_cast<const uint16_t*>(g)[e]);
}

// working-weight stores; with AG also into every peer's weight buffer
// (fully unrolled over the peer slots so the deltas stay kernel parameters)
template <int AG, typename T>
__device__ __forceinline__ void store_w(T* dst, T val, const PeerW& pw) {
    if constexpr (sizeof(T) >= 8) {
        __stcs(dst, val);
    } else {
        *dst = val;
    }
    if constexpr (AG != 0) {
#pragma unroll
        for (int r = 0; r < kMaxAgPeers; ++r)
            if (r < static_cast<int>(pw.n))
                *reinterpret_cast<T*>(reinterpret_cast<char*>(dst) + pw.delta[r]) = val;
    }
}

__device__ __constant__ PeerW kNoPeers = {};

template <int GK, int WK, int AG = 0>
__device__ __forceinline__ void adam_scalar(const Seg& sg, uint64_t e, const AdamConsts& c,
                                            const StepScalars& s, const PeerW& pw = kNoPeers) {
    float p = sg.p[e], m = sg.m[e], v = sg.v[e];
    adam_any(p, m, v, load_grad1<GK>(sg.g, e), c, s);
    sg.p[e] = p;
    sg.m[e] = m;
    sg.v[e] = v;
    if constexpr (WK != kNone)
        store_w<AG>(reinterpret_cast<uint16_t*>(sg.w) + e, narrow<WK>(p), pw);
}

template <int GK, int WK, int VEC>
__device__ __forceinline__ void adam_vector(const Seg& sg, uint64_t e, const AdamConsts& c,
                                            const StepScalars& s) {
    float p[VEC], m[VEC], v[VEC], g[VEC];
    ld_f32<VEC>(sg.p + e, p);
    ld_f32<VEC>(sg.m + e, m);
    ld_f32<VEC>(sg.v + e, v);
    if constexpr (GK == kF32) {
        ld_f32<VEC>(reinterpret_cast<const float*>(sg.g) + e, g);
    } else {
        uint32_t h[VEC];
        ld_u16<VEC>(reinterpret_cast<const uint16_t*>(sg.g) + e, h);
#pragma unroll
        for (int k = 0; k < VEC; ++k) g[k] = widen<GK>(h[k]);
    }
#pragma unroll
    for (int k = 0; k < VEC; ++k) adam_elem(p[k], m[k], v[k], g[k], c, s);
    st_f32<VEC>(sg.p + e, p);
    st_f32<VEC>(sg.m + e, m);
    st_f32<VEC>(sg.v + e, v);
    if constexpr (WK != kNone) {
        uint32_t w[VEC];
#pragma unroll
        for (int k = 0; k < VEC; ++k) w[k] = narrow<WK>(p[k]);
        st_u16<VEC>(reinterpret_cast<uint16_t*>(sg.w) + e, w);
    }
}

// Persistent grid-stride walk over the tiles of up to kMaxSegs sub-groups.
// A tile is kK2Threads vectors of VEC elements.  Tile 0 of a vectorised
// sub-group also handles its unaligned head and its tail scalar-wise; a
// sub-group whose pointers cannot be co-aligned runs scalar tiles.
template <int GK, int WK, int VEC>
__global__ void __launch_bounds__(kK2Threads) k2_adam(SegTable tab, AdamArgs a) {
    StepScalars s;
    if (!resolve_step(a, s)) return;  // skipped step: no state touched
    const AdamConsts c = a.c;
    uint32_t si = 0;
    for (uint64_t tile = blockIdx.x; tile < tab.total_tiles; tile += gridDim.x) {
        while (tile >= tab.seg[si].tile_end) ++si;  // tiles are visited in increasing order
        const Seg& sg = tab.seg[si];
        const uint64_t lt = tile - sg.tile_begin;
        if (sg.vector_ok) {
            const uint64_t j = lt * kK2Threads + threadIdx.x;
            if (j < sg.nvec) adam_vector<GK, WK, VEC>(sg, sg.head + j * VEC, c, s);
            if (lt == 0) {
                const uint64_t tail_begin = sg.head + sg.nvec * VEC;
                const uint64_t extra = sg.head + (sg.n - tail_begin);
                for (uint64_t k = threadIdx.x; k < extra; k += kK2Threads) {
                    adam_scalar<GK, WK>(sg, k < sg.head ? k : tail_begin + (k - sg.head), c, s);
                }
            }
        } else {
            const uint64_t e0 = lt * static_cast<uint64_t>(kK2Threads) * VEC;
#pragma unroll
            for (int r = 0; r < VEC; ++r) {
                const uint64_t e = e0 + static_cast<uint64_t>(r) * kK2Threads + threadIdx.x;
                if (e < sg.n) adam_scalar<GK, WK>(sg, e, c, s);
            }
        }
    }
}

// -------------------------------------------------------------- K2 streaming
// Warp-contiguous variant: a "slot" is 4 consecutive elements (one float4 of
// p, m, v; 8 B of 16-bit grads / working weights); the 32 lanes of a warp
// take 32 consecutive slots, so every load/store instruction covers 512 B
// (or 256 B) of contiguous memory in whole 32-B sectors.  A CTA tile is
// U * 256 slots; with PF the next tile's loads are issued before the current
// tile is computed, so HBM keeps streaming while the ALUs run the
// division/sqrt sequences.
struct Slot4 {
    float4 p, m, v;
    uint4 g;  // f32: four floats; 16-bit kinds: halves packed in .x/.y
};

// Load flavours (A/B): 0 = ld.global.cs (evict-first), 1 = default caching,
// 2 = ld.global.L1::no_allocate.L2::256B (L2 sector prefetch hint).
template <int LD>
__device__ __forceinline__ float4 ld4(const float4* p) {
    if constexpr (LD == 0 || LD == 3) return __ldcs(p);
    if constexpr (LD == 1) return *p;
    float4 r;
    asm("ld.global.L1::no_allocate.L2::256B.v4.f32 {%0, %1, %2, %3}, [%4];"
        : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p));
    return r;
}

template <int LD>
__device__ __forceinline__ uint2 ld2(const uint2* p) {
    if constexpr (LD == 0 || LD == 3) return __ldcs(p);
    if constexpr (LD == 1) return *p;
    uint2 r;
    asm("ld.global.L1::no_allocate.L2::256B.v2.u32 {%0, %1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p));
    return r;
}

template <int GK, int LD = 0>
__device__ __forceinline__ void load_slot(const Seg& sg, uint64_t e, Slot4& s) {
    s.p = ld4<LD>(reinterpret_cast<const float4*>(sg.p + e));
    s.m = ld4<LD>(reinterpret_cast<const float4*>(sg.m + e));
    s.v = ld4<LD>(reinterpret_cast<const float4*>(sg.v + e));
    if constexpr (GK == kF32) {
        const float4 t = ld4<LD>(reinterpret_cast<const float4*>(reinterpret_cast<const float*>(sg.g) + e));
        s.g = make_uint4(__float_as_uint(t.x), __float_as_uint(t.y), __float_as_uint(t.z),
                         __float_as_uint(t.w));
    } else {
        const uint2 t = ld2<LD>(reinterpret_cast<const uint2*>(reinterpret_cast<const uint16_t*>(sg.g) + e));
        s.g.x = t.x;
        s.g.y = t.y;
    }
}

// The exact path of one 4-element slot, kept OUT OF LINE: a slot lands here
// only when an element leaves the fast path's guarded ranges (zero or tiny
// moments, non-finite values, a non-power-of-two loss scale), and inlined
// into every slot of a tile it multiplied the kernels' code (15k SASS lines
// for K3) and competed with the fast path for registers.
struct Exact4 {
    float4 p, m, v;
};
template <int ORD>
__device__ __noinline__ Exact4 adam_exact4(float4 p, float4 m, float4 v, float4 g,
                                           const AdamConsts c, const StepScalars s) {
    adam_any<ORD>(p.x, m.x, v.x, g.x, c, s);
    adam_any<ORD>(p.y, m.y, v.y, g.y, c, s);
    adam_any<ORD>(p.z, m.z, v.z, g.z, c, s);
    adam_any<ORD>(p.w, m.w, v.w, g.w, c, s);
    return Exact4{p, m, v};
}

// MATH: 0 = production (hoisted-guard fast path, exact fallback), 1 = probe
// (approximate div/sqrt, never production), 2 = exact intrinsics only (A/B)
template <int GK, int WK, int MATH = 0, int AG = 0>
__device__ __forceinline__ void update_slot(const Seg& sg, uint64_t e, Slot4& s,
                                            const AdamConsts& c, const StepScalars& sc,
                                            const PeerW& pw = kNoPeers) {
    float g0, g1, g2, g3;
    if constexpr (GK == kF32) {
        g0 = __uint_as_float(s.g.x);
        g1 = __uint_as_float(s.g.y);
        g2 = __uint_as_float(s.g.z);
        g3 = __uint_as_float(s.g.w);
    } else {
        g0 = widen<GK>(s.g.x & 0xFFFFu);
        g1 = widen<GK>(s.g.x >> 16);
        g2 = widen<GK>(s.g.y & 0xFFFFu);
        g3 = widen<GK>(s.g.y >> 16);
    }
    if constexpr (MATH == 1) {
        adam_elem_probe(s.p.x, s.m.x, s.v.x, g0, c, sc);
        adam_elem_probe(s.p.y, s.m.y, s.v.y, g1, c, sc);
        adam_elem_probe(s.p.z, s.m.z, s.v.z, g2, c, sc);
        adam_elem_probe(s.p.w, s.m.w, s.v.w, g3, c, sc);
    } else if constexpr (MATH == 2) {
        adam_elem(s.p.x, s.m.x, s.v.x, g0, c, sc);
        adam_elem(s.p.y, s.m.y, s.v.y, g1, c, sc);
        adam_elem(s.p.z, s.m.z, s.v.z, g2, c, sc);
        adam_elem(s.p.w, s.m.w, s.v.w, g3, c, sc);
    } else {
        float p[4] = {s.p.x, s.p.y, s.p.z, s.p.w};
        float m[4] = {s.m.x, s.m.y, s.m.z, s.m.w};
        float v[4] = {s.v.x, s.v.y, s.v.z, s.v.w};
        const float g[4] = {g0, g1, g2, g3};
        if (sc.fast && adam_fast<4>(p, m, v, g, c, sc)) {
            // no output of a fast slot is NaN: plain pair conversions
            __stcs(reinterpret_cast<float4*>(sg.p + e), make_float4(p[0], p[1], p[2], p[3]));
            __stcs(reinterpret_cast<float4*>(sg.m + e), make_float4(m[0], m[1], m[2], m[3]));
            __stcs(reinterpret_cast<float4*>(sg.v + e), make_float4(v[0], v[1], v[2], v[3]));
            if constexpr (WK != kNone) {
                store_w<AG>(reinterpret_cast<uint2*>(reinterpret_cast<uint16_t*>(sg.w) + e),
                            make_uint2(narrow2_num<WK>(p[0], p[1]), narrow2_num<WK>(p[2], p[3])),
                            pw);
            }
            return;
        }
        const Exact4 r = adam_exact4<kOrdFp32>(s.p, s.m, s.v, make_float4(g0, g1, g2, g3), c, sc);
        s.p = r.p;
        s.m = r.m;
        s.v = r.v;
    }
    __stcs(reinterpret_cast<float4*>(sg.p + e), s.p);
    __stcs(reinterpret_cast<float4*>(sg.m + e), s.m);
    __stcs(reinterpret_cast<float4*>(sg.v + e), s.v);
    if constexpr (WK != kNone) {
        const uint32_t lo = narrow2<WK>(s.p.x, s.p.y);
        const uint32_t hi = narrow2<WK>(s.p.z, s.p.w);
        store_w<AG>(reinterpret_cast<uint2*>(reinterpret_cast<uint16_t*>(sg.w) + e),
                    make_uint2(lo, hi), pw);
    }
}

// The fast half of update_slot for the deferred K2 (A/B variant 19): true
// and stored when the slot passes the guard (incl. the cold second chance),
// false — nothing stored — otherwise; the caller lists the slot for the
// CTA's deferred phase (k2_oneshot DEFER).
template <int GK, int WK>
__device__ __forceinline__ bool update_slot_fast(const Seg& sg, uint64_t e, const Slot4& s,
                                                 const AdamConsts& c, const StepScalars& sc) {
    if (!sc.fast) return false;
    float g[4];
    if constexpr (GK == kF32) {
        g[0] = __uint_as_float(s.g.x); g[1] = __uint_as_float(s.g.y);
        g[2] = __uint_as_float(s.g.z); g[3] = __uint_as_float(s.g.w);
    } else {
        g[0] = widen<GK>(s.g.x & 0xFFFFu); g[1] = widen<GK>(s.g.x >> 16);
        g[2] = widen<GK>(s.g.y & 0xFFFFu); g[3] = widen<GK>(s.g.y >> 16);
    }
    float p[4] = {s.p.x, s.p.y, s.p.z, s.p.w};
    float m[4] = {s.m.x, s.m.y, s.m.z, s.m.w};
    float v[4] = {s.v.x, s.v.y, s.v.z, s.v.w};
    if (!adam_fast<4>(p, m, v, g, c, sc)) return false;
    __stcs(reinterpret_cast<float4*>(sg.p + e), make_float4(p[0], p[1], p[2], p[3]));
    __stcs(reinterpret_cast<float4*>(sg.m + e), make_float4(m[0], m[1], m[2], m[3]));
    __stcs(reinterpret_cast<float4*>(sg.v + e), make_float4(v[0], v[1], v[2], v[3]));
    if constexpr (WK != kNone) {
        __stcs(reinterpret_cast<uint2*>(reinterpret_cast<uint16_t*>(sg.w) + e),
               make_uint2(narrow2_num<WK>(p[0], p[1]), narrow2_num<WK>(p[2], p[3])));
    }
    return true;
}

template <int GK, int U, int LD = 0>
__device__ __forceinline__ void load_tile(const Seg& sg, uint64_t lt, Slot4 (&t)[U]) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const uint64_t j = lt * (U * kK2Threads) + u * kK2Threads + threadIdx.x;
        if (j < sg.nvec) load_slot<GK, LD>(sg, sg.head + 4 * j, t[u]);
    }
}

template <int GK, int WK, int U, int MATH = 0>
__device__ __forceinline__ void update_tile(const Seg& sg, uint64_t lt, Slot4 (&t)[U],
                                            const AdamConsts& c, const StepScalars& sc) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const uint64_t j = lt * (U * kK2Threads) + u * kK2Threads + threadIdx.x;
        if (j < sg.nvec) update_slot<GK, WK, MATH>(sg, sg.head + 4 * j, t[u], c, sc);
    }
}

template <int GK, int WK, int U, bool PF, int MINB = 1, int LD = 0>
__global__ void __launch_bounds__(kK2Threads, MINB) k2_stream(SegTable tab, AdamArgs a) {
    StepScalars sc;
    if (!resolve_step(a, sc)) return;  // skipped step: no state touched
    const AdamConsts c = a.c;
    uint64_t t = blockIdx.x;
    if (t < tab.total_tiles) {
        uint32_t si = 0;
        while (t >= tab.seg[si].tile_end) ++si;
        Slot4 cur[U];
        load_tile<GK, U, LD>(tab.seg[si], t - tab.seg[si].tile_begin, cur);
        for (;;) {
            const uint64_t tn = t + gridDim.x;
            const bool more = tn < tab.total_tiles;
            uint32_t sn = si;
            if (more) {
                while (tn >= tab.seg[sn].tile_end) ++sn;
            }
            if constexpr (PF) {
                Slot4 nxt[U];
                if (more) load_tile<GK, U, LD>(tab.seg[sn], tn - tab.seg[sn].tile_begin, nxt);
                update_tile<GK, WK, U, LD == 3 ? 1 : 0>(tab.seg[si], t - tab.seg[si].tile_begin, cur, c, sc);
                if (!more) break;
#pragma unroll
                for (int u = 0; u < U; ++u) cur[u] = nxt[u];
            } else {
                update_tile<GK, WK, U, LD == 3 ? 1 : 0>(tab.seg[si], t - tab.seg[si].tile_begin, cur, c, sc);
                if (!more) break;
                load_tile<GK, U, LD>(tab.seg[sn], tn - tab.seg[sn].tile_begin, cur);
            }
            t = tn;
            si = sn;
        }
    }
    // scalar remainder: unaligned heads/tails, and whole sub-groups whose
    // pointers cannot be co-aligned (rare; spread over the grid)
    const uint64_t gtid = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    const uint64_t gsize = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint32_t k = 0; k < tab.count; ++k) {
        const Seg& sg = tab.seg[k];
        if (sg.vector_ok) {
            if (blockIdx.x != k % gridDim.x) continue;
            const uint64_t tail_begin = sg.head + sg.nvec * 4;
            const uint64_t extra = sg.head + (sg.n - tail_begin);
            for (uint64_t q = threadIdx.x; q < extra; q += blockDim.x) {
                adam_scalar<GK, WK>(sg, q < sg.head ? q : tail_begin + (q - sg.head), c, sc);
            }
        } else {
            for (uint64_t e = gtid; e < sg.n; e += gsize) adam_scalar<GK, WK>(sg, e, c, sc);
        }
    }
}


// -------------------------------------------------------------- K2 one-shot
// Same slots and arithmetic as k2_stream, but ONE tile per CTA on a grid of
// total_tiles (+ a few trailing CTAs for the scalar remainder): the hardware
// block scheduler then walks the address space monotonically, which keeps
// the set of DRAM rows in use compact.  Measured (tools/layout_probe.cu): the
// 5-stream pattern moves 6.9 TB/s this way against 6.0-6.1 TB/s with a
// persistent grid-stride loop.
__device__ __forceinline__ uint32_t seg_of_tile(const SegTable& tab, uint64_t t) {
    // last segment whose first tile is <= t (zero-tile segments share their
    // successor's tile_begin, so they are never selected for a real tile)
    uint32_t lo = 0, hi = tab.count;
    while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (tab.seg[mid].tile_begin <= t) lo = mid; else hi = mid;
    }
    return lo;
}

// PDL (programmatic dependent launch, A/B variants 20/21): 1 = launched
// while the previous kernel (K1) drains, griddepcontrol.wait before anything
// else; 2 = the tile's p/m/v/g loads are issued before the wait (only the
// stores and the skip decision depend on K1; the launch must follow a kernel
// that writes none of p/m/v/g).
template <int GK, int WK, int U, int MATH = 0, int MINB = 1, int AG = 0, bool DEFER = false,
          int PDL = 0, bool REV = false>
__global__ void __launch_bounds__(kK2Threads, MINB) k2_oneshot(SegTable tab, AdamArgs a) {
    static_assert(!DEFER || (AG == 0 && MATH == 0), "deferred slots: plain K2 only");
    static_assert(PDL == 0 || (AG == 0 && !DEFER), "PDL: plain K2 only");
    StepScalars sc;
    if constexpr (PDL != 0) pdl_trigger();
    if constexpr (PDL == 1) pdl_wait();
    if constexpr (PDL != 2) {
        if (a.demote_lines) demote_kept(a.demote, a.demote_lines);
    }
    // REV (A/B): tiles back to front, so the first tiles read the gradients
    // K1 touched last (still in L2)
    const uint64_t t = REV && blockIdx.x < tab.total_tiles ? tab.total_tiles - 1 - blockIdx.x
                                                           : blockIdx.x;
    if constexpr (PDL == 2) {
        if (t >= tab.total_tiles) pdl_wait();
    }
    if (PDL != 2 || t >= tab.total_tiles) {
        if (!resolve_step(a, sc)) return;
    }
    const AdamConsts c = a.c;
    __shared__ uint32_t dlist[DEFER ? U * kK2Threads : 1];
    __shared__ uint32_t dn;
    if constexpr (DEFER) {
        if (threadIdx.x == 0) dn = 0;
        __syncthreads();
    }
    if (t < tab.total_tiles) {
        const Seg& sg = tab.seg[seg_of_tile(tab, t)];
        const uint64_t lt = t - sg.tile_begin;
        // this thread's slot-0 element; slot u is u * 1024 elements further,
        // so every access below is base register + compile-time offset
        const uint64_t j0 = lt * (U * kK2Threads) + threadIdx.x;
        const uint64_t e0 = sg.head + 4 * j0;
        Seg loc;
        loc.p = sg.p + e0;
        loc.m = sg.m + e0;
        loc.v = sg.v + e0;
        loc.g = static_cast<const uint8_t*>(sg.g) + e0 * (GK == kF32 ? 4 : 2);
        loc.w = WK == kNone ? nullptr : static_cast<void*>(static_cast<uint16_t*>(sg.w) + e0);
        const uint64_t nv = sg.nvec;
        const bool full = (lt + 1) * (U * kK2Threads) <= nv;
        Slot4 cur[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (full || j0 + u * kK2Threads < nv) load_slot<GK>(loc, 4 * u * kK2Threads, cur[u]);
        }
        if constexpr (PDL == 2) {
            pdl_wait();
            if (!resolve_step(a, sc)) return;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (full || j0 + u * kK2Threads < nv) {
                if constexpr (DEFER) {
                    if (!update_slot_fast<GK, WK>(loc, 4 * u * kK2Threads, cur[u], c, sc))
                        dlist[atomicAdd(&dn, 1u)] = u * kK2Threads + threadIdx.x;
                } else {
                    update_slot<GK, WK, MATH, AG>(loc, 4 * u * kK2Threads, cur[u], c, sc, a.peers);
                }
            }
        }
        if constexpr (DEFER) {
            // listed slots: one per thread, element by element (adam_any)
            __syncthreads();
            const uint32_t nd = dn;
            if (nd == 0) return;
            const Seg& sd = tab.seg[seg_of_tile(tab, t)];
            const uint64_t b0 = sd.head + 4 * ((t - sd.tile_begin) * (U * kK2Threads));
            for (uint32_t d = threadIdx.x; d < nd; d += kK2Threads) {
                const uint64_t e = b0 + 4ull * dlist[d];
                float4 p4 = __ldcs(reinterpret_cast<const float4*>(sd.p + e));
                float4 m4 = __ldcs(reinterpret_cast<const float4*>(sd.m + e));
                float4 v4 = __ldcs(reinterpret_cast<const float4*>(sd.v + e));
                float g[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) g[k] = load_grad1<GK>(sd.g, e + k);
                adam_any(p4.x, m4.x, v4.x, g[0], c, sc);
                adam_any(p4.y, m4.y, v4.y, g[1], c, sc);
                adam_any(p4.z, m4.z, v4.z, g[2], c, sc);
                adam_any(p4.w, m4.w, v4.w, g[3], c, sc);
                __stcs(reinterpret_cast<float4*>(sd.p + e), p4);
                __stcs(reinterpret_cast<float4*>(sd.m + e), m4);
                __stcs(reinterpret_cast<float4*>(sd.v + e), v4);
                if constexpr (WK != kNone) {
                    __stcs(reinterpret_cast<uint2*>(reinterpret_cast<uint16_t*>(sd.w) + e),
                           make_uint2(narrow2<WK>(p4.x, p4.y), narrow2<WK>(p4.z, p4.w)));
                }
            }
            return;
        }
        // peer stores reach system scope before the exit barrier's release
        if constexpr (AG != 0) __threadfence_system();
        return;
    }
    // trailing CTAs: unaligned heads/tails and non-co-alignable sub-groups
    const uint64_t q = t - tab.total_tiles;
    const uint64_t nq = gridDim.x - tab.total_tiles;
    for (uint32_t k = 0; k < tab.count; ++k) {
        const Seg& sg = tab.seg[k];
        if (sg.vector_ok) {
            if (q != k % nq) continue;
            const uint64_t tail_begin = sg.head + sg.nvec * 4;
            const uint64_t extra = sg.head + (sg.n - tail_begin);
            for (uint64_t i = threadIdx.x; i < extra; i += blockDim.x) {
                adam_scalar<GK, WK, AG>(sg, i < sg.head ? i : tail_begin + (i - sg.head), c, sc,
                                        a.peers);
            }
        } else {
            for (uint64_t e = q * blockDim.x + threadIdx.x; e < sg.n; e += nq * blockDim.x) {
                adam_scalar<GK, WK, AG>(sg, e, c, sc, a.peers);
            }
        }
    }
    if constexpr (AG != 0) __threadfence_system();
}

// -------------------------------------------------------------- K2 TMA
// Bulk-copy pipeline variant (A/B variant 10): one producer thread streams
// each 1024-element tile's p, m, v and g into a kStages-deep shared-memory
// ring with cp.async.bulk (TMA, completion on an mbarrier); four consumer
// warps wait on the stage's full barrier, update from shared memory and store
// p/m/v/w straight to global with coalesced 128-bit stores, then release the
// stage.  Loads are thereby decoupled from the division/sqrt work.
constexpr int kTmaTile = 1024;        // elements per tile (multiple of 8 => 16-B bulk sizes)
constexpr int kTmaStages = 6;
constexpr int kTmaConsumers = 128;    // 4 warps; warp 4 is the producer
constexpr int kTmaThreads = kTmaConsumers + 32;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("{ .reg .b64 st; mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1; }"
                 ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("{ .reg .b64 st; mbarrier.arrive.shared::cta.b64 st, [%0]; }"
                 ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    uint32_t done = 0;
    do {
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; "
                     "selp.u32 %0, 1, 0, p; }"
                     : "=r"(done) : "r"(smem_u32(bar)), "r"(parity) : "memory");
    } while (!done);
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

// elements of the 1024-element tile starting at e0 that lie in the body
__device__ __forceinline__ uint32_t tile_count(const Seg& sg, uint64_t e0) {
    const uint64_t left = sg.head + sg.nvec * 8 - e0;
    return static_cast<uint32_t>(left < kTmaTile ? left : kTmaTile);
}

template <int GK>
constexpr uint32_t tma_stage_bytes() {
    return kTmaTile * (12u + (GK == kF32 ? 4u : 2u));
}

template <int GK, int WK, int NC = kTmaConsumers>
__global__ void __launch_bounds__(NC + 32, 2) k2_tma(SegTable tab, AdamArgs a) {
    StepScalars sc;
    if (!resolve_step(a, sc)) return;
    const AdamConsts c = a.c;
    constexpr uint32_t kGB = GK == kF32 ? 4u : 2u;
    constexpr uint32_t kStage = tma_stage_bytes<GK>();
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + kTmaStages * kStage);
    uint64_t* empty = full + kTmaStages;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kTmaStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], NC / 32);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int warp = threadIdx.x >> 5;
    if (warp == NC / 32) {
        // ---------------- producer
        if ((threadIdx.x & 31) == 0) {
            uint32_t si = 0, it = 0;
            for (uint64_t t = blockIdx.x; t < tab.total_tiles; t += gridDim.x, ++it) {
                while (t >= tab.seg[si].tile_end) ++si;
                const Seg& sg = tab.seg[si];
                const uint64_t e0 = sg.head + (t - sg.tile_begin) * kTmaTile;
                const uint32_t cnt = static_cast<uint32_t>(
                    tile_count(sg, e0));
                const uint32_t s = it % kTmaStages;
                mbar_wait(&empty[s], ((it / kTmaStages) & 1u) ^ 1u);
                unsigned char* st = smem + s * kStage;
                mbar_expect_tx(&full[s], cnt * (12u + kGB));
                bulk_g2s(st, sg.p + e0, cnt * 4u, &full[s]);
                bulk_g2s(st + kTmaTile * 4, sg.m + e0, cnt * 4u, &full[s]);
                bulk_g2s(st + kTmaTile * 8, sg.v + e0, cnt * 4u, &full[s]);
                bulk_g2s(st + kTmaTile * 12, static_cast<const unsigned char*>(sg.g) + e0 * kGB,
                         cnt * kGB, &full[s]);
            }
        }
    } else {
        // ---------------- consumers: 8 elements per thread per tile
        uint32_t si = 0, it = 0;
        for (uint64_t t = blockIdx.x; t < tab.total_tiles; t += gridDim.x, ++it) {
            while (t >= tab.seg[si].tile_end) ++si;
            const Seg& sg = tab.seg[si];
            const uint64_t e0 = sg.head + (t - sg.tile_begin) * kTmaTile;
            const uint32_t cnt = static_cast<uint32_t>(
                tile_count(sg, e0));
            const uint32_t s = it % kTmaStages;
            mbar_wait(&full[s], (it / kTmaStages) & 1u);
            const unsigned char* st = smem + s * kStage;
#pragma unroll
            for (int half = 0; half < kTmaTile / (4 * NC); ++half) {
                const uint32_t q = half * (4 * NC) + 4u * threadIdx.x;  // element in tile
                if (q < cnt) {
                    Slot4 sl;
                    sl.p = *reinterpret_cast<const float4*>(st + 4 * q);
                    sl.m = *reinterpret_cast<const float4*>(st + kTmaTile * 4 + 4 * q);
                    sl.v = *reinterpret_cast<const float4*>(st + kTmaTile * 8 + 4 * q);
                    if constexpr (GK == kF32) {
                        sl.g = *reinterpret_cast<const uint4*>(st + kTmaTile * 12 + 4 * q);
                    } else {
                        const uint2 gg = *reinterpret_cast<const uint2*>(st + kTmaTile * 12 + 2 * q);
                        sl.g.x = gg.x;
                        sl.g.y = gg.y;
                    }
                    update_slot<GK, WK>(sg, e0 + q, sl, c, sc);
                }
            }
            __syncwarp();
            if ((threadIdx.x & 31) == 0) mbar_arrive(&empty[s]);
        }
    }
    // scalar remainder (heads, tails < 8 elements, unaligned sub-groups)
    const uint64_t gtid = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    const uint64_t gsize = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint32_t k = 0; k < tab.count; ++k) {
        const Seg& sg = tab.seg[k];
        if (sg.vector_ok) {
            if (blockIdx.x != k % gridDim.x) continue;
            const uint64_t tail_begin = sg.head + sg.nvec * 8;
            const uint64_t extra = sg.head + (sg.n - tail_begin);
            for (uint64_t q = threadIdx.x; q < extra; q += blockDim.x) {
                adam_scalar<GK, WK>(sg, q < sg.head ? q : tail_begin + (q - sg.head), c, sc);
            }
        } else {
            for (uint64_t e = gtid; e < sg.n; e += gsize) adam_scalar<GK, WK>(sg, e, c, sc);
        }
    }
}

// ============================================================== K3
// Pure-bf16 mode (Bf16Access, optimizer.cpp:83-93; simulator.cpp:470-486):
// the weights ARE the bf16 parameters, m and v are bf16; every quantity is
// widened, updated in fp32 with K2's arithmetic and rounded back with the
// reference's bf16 rounding.  12 B/param of state traffic (the paper's 58%
// I/O cut) + the gradient.  Same warp-contiguous 4-element slots as K2; the
// Seg's p/m/v point at uint16 arrays.
template <int GK>
__device__ __forceinline__ void bf16_state_scalar(const Seg& sg, uint64_t e, const AdamConsts& c,
                                                  const StepScalars& s) {
    uint16_t* P = reinterpret_cast<uint16_t*>(sg.p);
    uint16_t* M = reinterpret_cast<uint16_t*>(sg.m);
    uint16_t* V = reinterpret_cast<uint16_t*>(sg.v);
    float p = widen_bf16(P[e]), m = widen_bf16(M[e]), v = widen_bf16(V[e]);
    adam_any<kOrdBf16>(p, m, v, load_grad1<GK>(sg.g, e), c, s);
    P[e] = narrow<kBF16>(p);
    M[e] = narrow<kBF16>(m);
    V[e] = narrow<kBF16>(v);
}

__device__ __forceinline__ uint2 pack_bf16x4(float a, float b, float c, float d) {
    return make_uint2(narrow2<kBF16>(a, b), narrow2<kBF16>(c, d));
}

// One 4-element slot of bf16 state: 3 x 8 B of p/m/v and 8 B (bf16/f16) or
// 16 B (f32) of gradient.  A tile's slots are all loaded before the first
// store (stores could alias later loads, so the compiler would otherwise
// keep one slot in flight per thread).
struct Slot3 {
    uint2 p, m, v;
    uint4 g;
};

template <int GK>
__device__ __forceinline__ void bf16_state_load(const uint16_t* P, const uint16_t* M,
                                                const uint16_t* V, const void* G, Slot3& q) {
    q.p = __ldcs(reinterpret_cast<const uint2*>(P));
    q.m = __ldcs(reinterpret_cast<const uint2*>(M));
    q.v = __ldcs(reinterpret_cast<const uint2*>(V));
    if constexpr (GK == kF32) {
        q.g = __ldcs(reinterpret_cast<const uint4*>(G));
    } else {
        const uint2 t = __ldcs(reinterpret_cast<const uint2*>(G));
        q.g = make_uint4(t.x, t.y, 0u, 0u);
    }
}

template <bool NUM>
__device__ __forceinline__ uint2 pack4(const float (&x)[4]) {
    if constexpr (NUM) return make_uint2(narrow2_num<kBF16>(x[0], x[1]), narrow2_num<kBF16>(x[2], x[3]));
    return make_uint2(narrow2<kBF16>(x[0], x[1]), narrow2<kBF16>(x[2], x[3]));
}

// P/M/V/G point at this thread's element of slot 0; slot u is u * 1024
// elements further (compile-time offsets folded into the memory instructions).
template <int GK>
__device__ __forceinline__ void bf16_state_update(uint16_t* P, uint16_t* M, uint16_t* V,
                                                  const Slot3& q, const AdamConsts& c,
                                                  const StepScalars& s) {
    float g[4];
    if constexpr (GK == kF32) {
        g[0] = __uint_as_float(q.g.x); g[1] = __uint_as_float(q.g.y);
        g[2] = __uint_as_float(q.g.z); g[3] = __uint_as_float(q.g.w);
    } else {
        g[0] = widen<GK>(q.g.x & 0xFFFFu); g[1] = widen<GK>(q.g.x >> 16);
        g[2] = widen<GK>(q.g.y & 0xFFFFu); g[3] = widen<GK>(q.g.y >> 16);
    }
    float p[4] = {widen_bf16(q.p.x & 0xFFFFu), widen_bf16(q.p.x >> 16), widen_bf16(q.p.y & 0xFFFFu),
                  widen_bf16(q.p.y >> 16)};
    float m[4] = {widen_bf16(q.m.x & 0xFFFFu), widen_bf16(q.m.x >> 16), widen_bf16(q.m.y & 0xFFFFu),
                  widen_bf16(q.m.y >> 16)};
    float v[4] = {widen_bf16(q.v.x & 0xFFFFu), widen_bf16(q.v.x >> 16), widen_bf16(q.v.y & 0xFFFFu),
                  widen_bf16(q.v.y >> 16)};
    if (s.fast && adam_fast<4>(p, m, v, g, c, s)) {
        __stcs(reinterpret_cast<uint2*>(P), pack4<true>(p));
        __stcs(reinterpret_cast<uint2*>(M), pack4<true>(m));
        __stcs(reinterpret_cast<uint2*>(V), pack4<true>(v));
        return;
    }
    const Exact4 r = adam_exact4<kOrdBf16>(make_float4(p[0], p[1], p[2], p[3]),
                                           make_float4(m[0], m[1], m[2], m[3]),
                                           make_float4(v[0], v[1], v[2], v[3]),
                                           make_float4(g[0], g[1], g[2], g[3]), c, s);
    p[0] = r.p.x; p[1] = r.p.y; p[2] = r.p.z; p[3] = r.p.w;
    m[0] = r.m.x; m[1] = r.m.y; m[2] = r.m.z; m[3] = r.m.w;
    v[0] = r.v.x; v[1] = r.v.y; v[2] = r.v.z; v[3] = r.v.w;
    __stcs(reinterpret_cast<uint2*>(P), pack4<false>(p));
    __stcs(reinterpret_cast<uint2*>(M), pack4<false>(m));
    __stcs(reinterpret_cast<uint2*>(V), pack4<false>(v));
}

template <int GK, int U = kK3Slots, int MINB = 1>
__global__ void __launch_bounds__(kK2Threads, MINB) k3_adam_bf16(SegTable tab, AdamArgs a) {
    StepScalars sc;
    if (!resolve_step(a, sc)) return;
    const AdamConsts c = a.c;
    // one tile per CTA (same one-shot grid as K2), then trailing CTAs
    const uint64_t t = blockIdx.x;
    if (t < tab.total_tiles) {
        const Seg& sg = tab.seg[seg_of_tile(tab, t)];
        const uint64_t lt = t - sg.tile_begin;
        const uint64_t j0 = lt * (U * kK2Threads) + threadIdx.x;
        const uint64_t e0 = sg.head + 4 * j0;
        uint16_t* P = reinterpret_cast<uint16_t*>(sg.p) + e0;
        uint16_t* M = reinterpret_cast<uint16_t*>(sg.m) + e0;
        uint16_t* V = reinterpret_cast<uint16_t*>(sg.v) + e0;
        const uint8_t* G = static_cast<const uint8_t*>(sg.g) + e0 * (GK == kF32 ? 4 : 2);
        const uint64_t nv = sg.nvec;
        const bool full = (lt + 1) * (U * kK2Threads) <= nv;
        Slot3 q[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (full || j0 + u * kK2Threads < nv) {
                const int o = 4 * u * kK2Threads;
                bf16_state_load<GK>(P + o, M + o, V + o, G + o * (GK == kF32 ? 4 : 2), q[u]);
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (full || j0 + u * kK2Threads < nv) {
                const int o = 4 * u * kK2Threads;
                bf16_state_update<GK>(P + o, M + o, V + o, q[u], c, sc);
            }
        }
        return;
    }
    const uint64_t q0 = t - tab.total_tiles;
    const uint64_t nq = gridDim.x - tab.total_tiles;
    for (uint32_t k = 0; k < tab.count; ++k) {
        const Seg& sg = tab.seg[k];
        if (sg.vector_ok) {
            if (q0 != k % nq) continue;
            const uint64_t tail_begin = sg.head + sg.nvec * 4;
            const uint64_t extra = sg.head + (sg.n - tail_begin);
            for (uint64_t q = threadIdx.x; q < extra; q += blockDim.x) {
                bf16_state_scalar<GK>(sg, q < sg.head ? q : tail_begin + (q - sg.head), c, sc);
            }
        } else {
            for (uint64_t e = q0 * blockDim.x + threadIdx.x; e < sg.n; e += nq * blockDim.x) {
                bf16_state_scalar<GK>(sg, e, c, sc);
            }
        }
    }
}

// K3 with 8-element slots (A/B variants 4/5): one 16-byte access per thread
// for each of p, m, v and a bf16 gradient slot (two for fp32 gradients),
// half the memory instructions of the 4-element slots; the arithmetic and
// its order are unchanged (adam_fast<8> / adam_elem per element).
struct Slot8 {
    uint4 p, m, v;
    uint4 g[2];
};

__device__ __forceinline__ void unpack8(const uint4& q, float (&x)[8]) {
    x[0] = widen_bf16(q.x & 0xFFFFu); x[1] = widen_bf16(q.x >> 16);
    x[2] = widen_bf16(q.y & 0xFFFFu); x[3] = widen_bf16(q.y >> 16);
    x[4] = widen_bf16(q.z & 0xFFFFu); x[5] = widen_bf16(q.z >> 16);
    x[6] = widen_bf16(q.w & 0xFFFFu); x[7] = widen_bf16(q.w >> 16);
}

template <bool NUM>
__device__ __forceinline__ uint4 pack8(const float (&x)[8]) {
    if constexpr (NUM)
        return make_uint4(narrow2_num<kBF16>(x[0], x[1]), narrow2_num<kBF16>(x[2], x[3]),
                          narrow2_num<kBF16>(x[4], x[5]), narrow2_num<kBF16>(x[6], x[7]));
    return make_uint4(narrow2<kBF16>(x[0], x[1]), narrow2<kBF16>(x[2], x[3]),
                      narrow2<kBF16>(x[4], x[5]), narrow2<kBF16>(x[6], x[7]));
}

template <int GK, int U, int MINB>
__global__ void __launch_bounds__(kK2Threads, MINB) k3_adam_bf16_v8(SegTable tab, AdamArgs a) {
    StepScalars sc;
    if (!resolve_step(a, sc)) return;
    const AdamConsts c = a.c;
    constexpr uint32_t kGB = GK == kF32 ? 4u : 2u;
    const uint64_t t = blockIdx.x;
    if (t < tab.total_tiles) {
        const Seg& sg = tab.seg[seg_of_tile(tab, t)];
        const uint64_t lt = t - sg.tile_begin;
        const uint64_t j0 = lt * (U * kK2Threads) + threadIdx.x;
        const uint64_t e0 = sg.head + 8 * j0;
        uint16_t* P = reinterpret_cast<uint16_t*>(sg.p) + e0;
        uint16_t* M = reinterpret_cast<uint16_t*>(sg.m) + e0;
        uint16_t* V = reinterpret_cast<uint16_t*>(sg.v) + e0;
        const uint8_t* G = static_cast<const uint8_t*>(sg.g) + e0 * kGB;
        const uint64_t nv = sg.nvec;
        const bool full = (lt + 1) * (U * kK2Threads) <= nv;
        Slot8 q[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (full || j0 + u * kK2Threads < nv) {
                const int o = 8 * u * kK2Threads;
                q[u].p = __ldcs(reinterpret_cast<const uint4*>(P + o));
                q[u].m = __ldcs(reinterpret_cast<const uint4*>(M + o));
                q[u].v = __ldcs(reinterpret_cast<const uint4*>(V + o));
                q[u].g[0] = __ldcs(reinterpret_cast<const uint4*>(G + o * kGB));
                if constexpr (GK == kF32) q[u].g[1] = __ldcs(reinterpret_cast<const uint4*>(G + o * kGB) + 1);
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (full || j0 + u * kK2Threads < nv) {
                const int o = 8 * u * kK2Threads;
                float g[8], p[8], m[8], v[8];
                if constexpr (GK == kF32) {
                    const uint32_t w[8] = {q[u].g[0].x, q[u].g[0].y, q[u].g[0].z, q[u].g[0].w,
                                           q[u].g[1].x, q[u].g[1].y, q[u].g[1].z, q[u].g[1].w};
#pragma unroll
                    for (int k = 0; k < 8; ++k) g[k] = __uint_as_float(w[k]);
                } else {
                    const uint32_t w[4] = {q[u].g[0].x, q[u].g[0].y, q[u].g[0].z, q[u].g[0].w};
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        g[2 * k] = widen<GK>(w[k] & 0xFFFFu);
                        g[2 * k + 1] = widen<GK>(w[k] >> 16);
                    }
                }
                unpack8(q[u].p, p);
                unpack8(q[u].m, m);
                unpack8(q[u].v, v);
                if (sc.fast && adam_fast<8>(p, m, v, g, c, sc)) {
                    __stcs(reinterpret_cast<uint4*>(P + o), pack8<true>(p));
                    __stcs(reinterpret_cast<uint4*>(M + o), pack8<true>(m));
                    __stcs(reinterpret_cast<uint4*>(V + o), pack8<true>(v));
                } else {
#pragma unroll
                    for (int k = 0; k < 8; ++k) adam_elem<kOrdBf16>(p[k], m[k], v[k], g[k], c, sc);
                    __stcs(reinterpret_cast<uint4*>(P + o), pack8<false>(p));
                    __stcs(reinterpret_cast<uint4*>(M + o), pack8<false>(m));
                    __stcs(reinterpret_cast<uint4*>(V + o), pack8<false>(v));
                }
            }
        }
        return;
    }
    const uint64_t q0 = t - tab.total_tiles;
    const uint64_t nq = gridDim.x - tab.total_tiles;
    for (uint32_t k = 0; k < tab.count; ++k) {
        const Seg& sg = tab.seg[k];
        if (sg.vector_ok) {
            if (q0 != k % nq) continue;
            const uint64_t tail_begin = sg.head + sg.nvec * 8;
            const uint64_t extra = sg.head + (sg.n - tail_begin);
            for (uint64_t q = threadIdx.x; q < extra; q += blockDim.x) {
                bf16_state_scalar<GK>(sg, q < sg.head ? q : tail_begin + (q - sg.head), c, sc);
            }
        } else {
            for (uint64_t e = q0 * blockDim.x + threadIdx.x; e < sg.n; e += nq * blockDim.x) {
                bf16_state_scalar<GK>(sg, e, c, sc);
            }
        }
    }
}

// -------------------------------------------------------------- K3 v2
// Issue-slot economy for the pure-bf16 update (K3 moves half K2's bytes per
// parameter, so at the same bandwidth it must retire twice the parameters
// per second: it was instruction-bound at ~56 issued instructions per
// parameter).  Changes against k3_adam_bf16, arithmetic unchanged:
//  * 8-element slots: one 16-byte access per tensor and slot (7 memory
//    instructions per 8 parameters instead of per 4);
//  * bf16 widening straight from the packed words (shift / mask), narrowing
//    by pair conversion (F2FP) — no unpacked intermediate arrays;
//  * the admission guard as floating-point compares on |M|, V and |p|
//    (ordered compares also reject NaN), accumulated in one predicate per
//    slot: the same admitted set as fast_m_ok / fast_v_ok / fast_p_ok;
//  * a slot that fails the guard takes the out-of-line exact path on its
//    raw words (adam_exact8_bf16), so the fast path's registers hold nothing
//    for it.
template <int GK>
struct K3Raw {
    uint4 p, m, v;
    uint4 g[GK == kF32 ? 2 : 1];
};

template <int GK>
__device__ __forceinline__ float k3_grad(const K3Raw<GK>& r, int k) {
    if constexpr (GK == kF32) {
        const uint4& q = r.g[k >> 2];
        return __uint_as_float((k & 3) == 0 ? q.x : (k & 3) == 1 ? q.y : (k & 3) == 2 ? q.z : q.w);
    } else {
        const uint4& q = r.g[0];
        const uint32_t w = (k >> 1) == 0 ? q.x : (k >> 1) == 1 ? q.y : (k >> 1) == 2 ? q.z : q.w;
        if constexpr (GK == kBF16) return (k & 1) ? __uint_as_float(w & 0xFFFF0000u) : __uint_as_float(w << 16);
        return widen_f16((k & 1) ? (w >> 16) : (w & 0xFFFFu));
    }
}

__device__ __forceinline__ float bf16_lane(const uint4& q, int k) {
    const uint32_t w = (k >> 1) == 0 ? q.x : (k >> 1) == 1 ? q.y : (k >> 1) == 2 ? q.z : q.w;
    return (k & 1) ? __uint_as_float(w & 0xFFFF0000u) : __uint_as_float(w << 16);
}

template <int GK>
__device__ __noinline__ void adam_exact8_bf16(K3Raw<GK> r, uint4* out, const AdamConsts c,
                                              const StepScalars s) {
    float p[8], m[8], v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        p[k] = bf16_lane(r.p, k);
        m[k] = bf16_lane(r.m, k);
        v[k] = bf16_lane(r.v, k);
        adam_any<kOrdBf16>(p[k], m[k], v[k], k3_grad<GK>(r, k), c, s);
    }
    out[0] = make_uint4(narrow2<kBF16>(p[0], p[1]), narrow2<kBF16>(p[2], p[3]),
                        narrow2<kBF16>(p[4], p[5]), narrow2<kBF16>(p[6], p[7]));
    out[1] = make_uint4(narrow2<kBF16>(m[0], m[1]), narrow2<kBF16>(m[2], m[3]),
                        narrow2<kBF16>(m[4], m[5]), narrow2<kBF16>(m[6], m[7]));
    out[2] = make_uint4(narrow2<kBF16>(v[0], v[1]), narrow2<kBF16>(v[2], v[3]),
                        narrow2<kBF16>(v[4], v[5]), narrow2<kBF16>(v[6], v[7]));
}

// One 8-element slot through the fast path; false when any element leaves
// the guarded ranges (then nothing is produced).
// NaN-propagating 3-input min / max (FMNMX3.NAN, sm_100): a NaN anywhere
// makes the result NaN, which every ordered compare below rejects.
__device__ __forceinline__ float min3n(float a, float b, float c) {
    float r;
    asm("min.NaN.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
    return r;
}
__device__ __forceinline__ float max3n(float a, float b, float c) {
    float r;
    asm("max.NaN.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
    return r;
}

// GUARD: 0 = five compares per element, 1 = the same ranges tested once per
// slot on NaN-propagating min / max reductions (FMNMX3.NAN).
// EARLY (GUARD 1 only): the guard is evaluated on M, V, p before the
// division / square-root sequences, and a warp whose active lanes all fail
// it returns at once (cold rows, non-finite blocks: the deferred phase
// recomputes those slots anyway); a warp with any admitted lane computes as
// before.
template <int GK, int GUARD = 0, bool EARLY = false>
__device__ __forceinline__ bool k3_fast8(const K3Raw<GK>& r, uint4& po, uint4& mo, uint4& vo,
                                         const AdamConsts& c, const StepScalars& s) {
    static_assert(!EARLY || GUARD != 0, "early reject: reduction guard only");
    float P[8], M[8], V[8], AM[8], AP[8];
    bool ok = true;
    if constexpr (EARLY) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const float m = bf16_lane(r.m, k), v = bf16_lane(r.v, k);
            const float g = __fmul_rn(k3_grad<GK>(r, k), s.inv_scale);
            M[k] = __fadd_rn(__fmul_rn(c.beta1, m), __fmul_rn(c.one_minus_b1, g));
            V[k] = __fadd_rn(__fmul_rn(c.beta2, v), __fmul_rn(c.one_minus_b2, __fmul_rn(g, g)));
            AM[k] = fabsf(M[k]);
            AP[k] = fabsf(bf16_lane(r.p, k));
        }
        const float mn_m = min3n(min3n(AM[0], AM[1], AM[2]), min3n(AM[3], AM[4], AM[5]),
                                 min3n(AM[6], AM[7], AM[7]));
        const float mx_m = max3n(max3n(AM[0], AM[1], AM[2]), max3n(AM[3], AM[4], AM[5]),
                                 max3n(AM[6], AM[7], AM[7]));
        const float mn_v = min3n(min3n(V[0], V[1], V[2]), min3n(V[3], V[4], V[5]),
                                 min3n(V[6], V[7], V[7]));
        const float mx_v = max3n(max3n(V[0], V[1], V[2]), max3n(V[3], V[4], V[5]),
                                 max3n(V[6], V[7], V[7]));
        const float mx_p = max3n(max3n(AP[0], AP[1], AP[2]), max3n(AP[3], AP[4], AP[5]),
                                 max3n(AP[6], AP[7], AP[7]));
        ok = (mn_m >= 0x1p-50f) & (mx_m < 0x1p51f) & (mn_v >= 0x1p-96f) & (mx_v < 0x1p80f) &
             (mx_p < __uint_as_float(0x7F800000u));
        if (!__any_sync(__activemask(), ok)) return false;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const float p = bf16_lane(r.p, k);
            const float mh = div_by(M[k], s.bc1, s.y1);
            const float vh = div_by(V[k], s.bc2, s.y2);
            const float den = __fadd_rn(sqrt_fast(vh), c.eps);
            const float upd = __fmul_rn(c.lr, div_by(mh, den, rcp_refined(den)));
            P[k] = __fsub_rn(__fsub_rn(p, upd), __fmul_rn(c.lr_wd, p));
        }
        po = make_uint4(narrow2_num<kBF16>(P[0], P[1]), narrow2_num<kBF16>(P[2], P[3]),
                        narrow2_num<kBF16>(P[4], P[5]), narrow2_num<kBF16>(P[6], P[7]));
        mo = make_uint4(narrow2_num<kBF16>(M[0], M[1]), narrow2_num<kBF16>(M[2], M[3]),
                        narrow2_num<kBF16>(M[4], M[5]), narrow2_num<kBF16>(M[6], M[7]));
        vo = make_uint4(narrow2_num<kBF16>(V[0], V[1]), narrow2_num<kBF16>(V[2], V[3]),
                        narrow2_num<kBF16>(V[4], V[5]), narrow2_num<kBF16>(V[6], V[7]));
        return ok;
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const float p = bf16_lane(r.p, k), m = bf16_lane(r.m, k), v = bf16_lane(r.v, k);
        const float g = __fmul_rn(k3_grad<GK>(r, k), s.inv_scale);
        M[k] = __fadd_rn(__fmul_rn(c.beta1, m), __fmul_rn(c.one_minus_b1, g));
        V[k] = __fadd_rn(__fmul_rn(c.beta2, v), __fmul_rn(c.one_minus_b2, __fmul_rn(g, g)));
        const float am = fabsf(M[k]);
        if constexpr (GUARD == 0) {
            ok &= (am >= 0x1p-50f) & (am < 0x1p51f) & (V[k] >= 0x1p-96f) & (V[k] < 0x1p80f) &
                  (fabsf(p) < __uint_as_float(0x7F800000u));
        } else {
            AM[k] = am;
            AP[k] = fabsf(p);
        }
        const float mh = div_by(M[k], s.bc1, s.y1);
        const float vh = div_by(V[k], s.bc2, s.y2);
        const float den = __fadd_rn(sqrt_fast(vh), c.eps);
        const float upd = __fmul_rn(c.lr, div_by(mh, den, rcp_refined(den)));
        P[k] = __fsub_rn(__fsub_rn(p, upd), __fmul_rn(c.lr_wd, p));
    }
    po = make_uint4(narrow2_num<kBF16>(P[0], P[1]), narrow2_num<kBF16>(P[2], P[3]),
                    narrow2_num<kBF16>(P[4], P[5]), narrow2_num<kBF16>(P[6], P[7]));
    mo = make_uint4(narrow2_num<kBF16>(M[0], M[1]), narrow2_num<kBF16>(M[2], M[3]),
                    narrow2_num<kBF16>(M[4], M[5]), narrow2_num<kBF16>(M[6], M[7]));
    vo = make_uint4(narrow2_num<kBF16>(V[0], V[1]), narrow2_num<kBF16>(V[2], V[3]),
                    narrow2_num<kBF16>(V[4], V[5]), narrow2_num<kBF16>(V[6], V[7]));
    if constexpr (GUARD != 0) {
        const float mn_m = min3n(min3n(AM[0], AM[1], AM[2]), min3n(AM[3], AM[4], AM[5]),
                                 min3n(AM[6], AM[7], AM[7]));
        const float mx_m = max3n(max3n(AM[0], AM[1], AM[2]), max3n(AM[3], AM[4], AM[5]),
                                 max3n(AM[6], AM[7], AM[7]));
        const float mn_v = min3n(min3n(V[0], V[1], V[2]), min3n(V[3], V[4], V[5]),
                                 min3n(V[6], V[7], V[7]));
        const float mx_v = max3n(max3n(V[0], V[1], V[2]), max3n(V[3], V[4], V[5]),
                                 max3n(V[6], V[7], V[7]));
        const float mx_p = max3n(max3n(AP[0], AP[1], AP[2]), max3n(AP[3], AP[4], AP[5]),
                                 max3n(AP[6], AP[7], AP[7]));
        ok = (mn_m >= 0x1p-50f) & (mx_m < 0x1p51f) & (mn_v >= 0x1p-96f) & (mx_v < 0x1p80f) &
             (mx_p < __uint_as_float(0x7F800000u));
    }
    return ok;
}


// NOT an optimizer: the same loads / stores / grid with a trivial update
// (A/B variant 16, MA_K3_VARIANT=16) — the access pattern's own ceiling.
template <int GK>
__device__ __forceinline__ void k3_probe8(const K3Raw<GK>& r, uint4& po, uint4& mo, uint4& vo) {
    float P[8], M[8], V[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const float d = __fmul_rn(k3_grad<GK>(r, k), 1e-9f);
        P[k] = __fadd_rn(bf16_lane(r.p, k), d);
        M[k] = __fadd_rn(bf16_lane(r.m, k), d);
        V[k] = __fadd_rn(bf16_lane(r.v, k), d);
    }
    po = make_uint4(narrow2_num<kBF16>(P[0], P[1]), narrow2_num<kBF16>(P[2], P[3]),
                    narrow2_num<kBF16>(P[4], P[5]), narrow2_num<kBF16>(P[6], P[7]));
    mo = make_uint4(narrow2_num<kBF16>(M[0], M[1]), narrow2_num<kBF16>(M[2], M[3]),
                    narrow2_num<kBF16>(M[4], M[5]), narrow2_num<kBF16>(M[6], M[7]));
    vo = make_uint4(narrow2_num<kBF16>(V[0], V[1]), narrow2_num<kBF16>(V[2], V[3]),
                    narrow2_num<kBF16>(V[4], V[5]), narrow2_num<kBF16>(V[6], V[7]));
}

// TPC consecutive tiles per CTA (one after the other): the per-CTA set-up
// (step scalars, segment lookup, ...) is paid once per TPC tiles.
// DEFER: a slot that fails the fast guard is not computed in the hot loop
// (no call there); its index goes to a shared-memory list and, after the
// tile, all threads of the CTA process the listed slots element by element
// (adam_any: fast, cold second chance, else the full exact sequence) — no
// SIMT divergence, and cold or non-finite slots cost their own work only.
// COLD (with DEFER), bit 0: k3_fast8's early warp-uniform reject; bit 1: a
// listed slot whose eight elements all take the M == 0 shortcut of
// cold_elem (m = g = 0: an untouched row) is finished in one vector step
// instead of eight adam_any calls; bit 2: the vector second chance (the
// fast, M == 0 and scaled routes over the slot, all-M == 0 slots without
// the sequences) before the per-element path.
template <int GK, int U, int MINB, bool PROBE = false, int GUARD = 0, int TPC = 1,
          bool DEFER = false, int COLD = 0>
__global__ void __launch_bounds__(kK2Threads, MINB) k3_v2(SegTable tab, AdamArgs a) {
    static_assert(!DEFER || TPC == 1, "deferred slots: one tile per CTA");
    // programmatic dependent of K1 (production launch, §3.5): nothing is read
    // before the previous grid has completed (no-ops on a plain launch)
    pdl_trigger();
    pdl_wait();
    if (a.demote_lines) demote_kept(a.demote, a.demote_lines);
    StepScalars sc;
    if (!resolve_step(a, sc)) return;
    const AdamConsts c = a.c;
    constexpr uint32_t kGB = GK == kF32 ? 4u : 2u;
    const uint64_t main_ctas = (tab.total_tiles + TPC - 1) / TPC;
    __shared__ uint32_t dlist[DEFER ? U * kK2Threads : 1];
    __shared__ uint32_t dn;
    if constexpr (DEFER) {
        if (threadIdx.x == 0) dn = 0;
        __syncthreads();
    }
    if (blockIdx.x < main_ctas) {
#pragma unroll 1
    for (int it = 0; it < TPC; ++it) {
        const uint64_t t = static_cast<uint64_t>(blockIdx.x) * TPC + it;
        if (t >= tab.total_tiles) break;
        const Seg& sg = tab.seg[seg_of_tile(tab, t)];
        const uint64_t lt = t - sg.tile_begin;
        const uint64_t j0 = lt * (U * kK2Threads) + threadIdx.x;
        const uint64_t e0 = sg.head + 8 * j0;
        uint4* P = reinterpret_cast<uint4*>(reinterpret_cast<uint16_t*>(sg.p) + e0);
        uint4* M = reinterpret_cast<uint4*>(reinterpret_cast<uint16_t*>(sg.m) + e0);
        uint4* V = reinterpret_cast<uint4*>(reinterpret_cast<uint16_t*>(sg.v) + e0);
        const uint4* G = reinterpret_cast<const uint4*>(static_cast<const uint8_t*>(sg.g) + e0 * kGB);
        const uint64_t nv = sg.nvec;
        const bool full = (lt + 1) * (U * kK2Threads) <= nv;
        constexpr int kS = kK2Threads;  // uint4 stride between a thread's slots
        K3Raw<GK> q[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (full || j0 + u * kK2Threads < nv) {
                q[u].p = __ldcs(P + u * kS);
                q[u].m = __ldcs(M + u * kS);
                q[u].v = __ldcs(V + u * kS);
                q[u].g[0] = __ldcs(G + u * kS * (kGB / 2));
                if constexpr (GK == kF32) q[u].g[1] = __ldcs(G + u * kS * 2 + 1);
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (full || j0 + u * kK2Threads < nv) {
                uint4 po, mo, vo;
                if constexpr (PROBE) {
                    k3_probe8<GK>(q[u], po, mo, vo);
                } else if (!(sc.fast && k3_fast8<GK, GUARD, (COLD & 1) != 0>(q[u], po, mo, vo, c, sc))) {
                    if constexpr (DEFER) {
                        dlist[atomicAdd(&dn, 1u)] = u * kK2Threads + threadIdx.x;
                        continue;
                    } else {
                        // includes cold slots: adam_exact8_bf16 -> adam_any (fast,
                        // cold second chance, else the full exact sequence)
                        uint4 out[3];
                        adam_exact8_bf16<GK>(q[u], out, c, sc);
                        po = out[0];
                        mo = out[1];
                        vo = out[2];
                    }
                }
                __stcs(P + u * kS, po);
                __stcs(M + u * kS, mo);
                __stcs(V + u * kS, vo);
            }
        }
        if constexpr (DEFER) {
            // one listed slot per thread, 16-byte accesses as in the hot loop
            __syncthreads();
            const uint32_t nd = dn;
            if (nd == 0) continue;
            // the tile's slot 0, recomputed here so no pointer stays live
            // through the hot loop for this rare phase
            const Seg& sd = tab.seg[seg_of_tile(tab, t)];
            const uint64_t b0 = sd.head + 8 * ((t - sd.tile_begin) * (U * kK2Threads));
            uint4* P0 = reinterpret_cast<uint4*>(reinterpret_cast<uint16_t*>(sd.p) + b0);
            uint4* M0 = reinterpret_cast<uint4*>(reinterpret_cast<uint16_t*>(sd.m) + b0);
            uint4* V0 = reinterpret_cast<uint4*>(reinterpret_cast<uint16_t*>(sd.v) + b0);
            const uint4* G0 = reinterpret_cast<const uint4*>(static_cast<const uint8_t*>(sd.g) + b0 * kGB);
            // split drain (COLD bit 3, A/B variant 27): two threads per
            // listed slot, four elements (8-byte accesses) each, so a tile
            // with a few listed slots ends after half the serial tail; the
            // M == 0 route per half (helps scattered cold
            // slots, costs dense cold tiles; also when chosen at run time by
            // the list length)
            if constexpr ((COLD & 8) != 0) {
                for (uint32_t d2 = threadIdx.x; d2 < 2 * nd; d2 += kK2Threads) {
                    const uint32_t sl = dlist[d2 >> 1];
                    const uint32_t hf = d2 & 1u;
                    uint2* Ph = reinterpret_cast<uint2*>(P0 + sl) + hf;
                    uint2* Mh = reinterpret_cast<uint2*>(M0 + sl) + hf;
                    uint2* Vh = reinterpret_cast<uint2*>(V0 + sl) + hf;
                    const uint2 rp = __ldcs(Ph), rm = __ldcs(Mh), rv = __ldcs(Vh);
                    float gq[4];
                    if constexpr (GK == kF32) {
                        const uint4 t4 = __ldcs(G0 + sl * 2 + hf);
                        gq[0] = __uint_as_float(t4.x);
                        gq[1] = __uint_as_float(t4.y);
                        gq[2] = __uint_as_float(t4.z);
                        gq[3] = __uint_as_float(t4.w);
                    } else {
                        const uint2 t2 = __ldcs(reinterpret_cast<const uint2*>(G0 + sl) + hf);
                        const uint32_t gw[2] = {t2.x, t2.y};
#pragma unroll
                        for (int k = 0; k < 4; ++k) {
                            const uint32_t hb = (k & 1) ? (gw[k >> 1] >> 16) : (gw[k >> 1] & 0xFFFFu);
                            gq[k] = GK == kBF16 ? __uint_as_float(hb << 16) : widen_f16(hb);
                        }
                    }
                    const uint32_t pw[2] = {rp.x, rp.y}, mw[2] = {rm.x, rm.y}, vw[2] = {rv.x, rv.y};
                    auto lane16 = [](const uint32_t (&w)[2], int k) {
                        return __uint_as_float((k & 1) ? (w[k >> 1] & 0xFFFF0000u) : (w[k >> 1] << 16));
                    };
                    float P[4], M[4], V[4];
                    bool cold = sc.fast;
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const float p = lane16(pw, k);
                        const float g = __fmul_rn(gq[k], sc.inv_scale);
                        M[k] = __fadd_rn(__fmul_rn(c.beta1, lane16(mw, k)), __fmul_rn(c.one_minus_b1, g));
                        V[k] = __fadd_rn(__fmul_rn(c.beta2, lane16(vw, k)),
                                         __fmul_rn(c.one_minus_b2, __fmul_rn(g, g)));
                        cold &= (M[k] == 0.0f) & (V[k] >= 0.0f) & fast_p_ok(p);
                        P[k] = __fsub_rn(__fsub_rn(p, __fmul_rn(c.lr, M[k])), __fmul_rn(c.lr_wd, p));
                    }
                    if (!cold) {
#pragma unroll
                        for (int k = 0; k < 4; ++k) {
                            P[k] = lane16(pw, k);
                            M[k] = lane16(mw, k);
                            V[k] = lane16(vw, k);
                            adam_any<kOrdBf16>(P[k], M[k], V[k], gq[k], c, sc);
                        }
                    }
                    __stcs(Ph, make_uint2(narrow2<kBF16>(P[0], P[1]), narrow2<kBF16>(P[2], P[3])));
                    __stcs(Mh, make_uint2(narrow2<kBF16>(M[0], M[1]), narrow2<kBF16>(M[2], M[3])));
                    __stcs(Vh, make_uint2(narrow2<kBF16>(V[0], V[1]), narrow2<kBF16>(V[2], V[3])));
                }
                continue;
            }
            for (uint32_t d = threadIdx.x; d < nd; d += kK2Threads) {
                const uint32_t sl = dlist[d];
                K3Raw<GK> r;
                r.p = __ldcs(P0 + sl);
                r.m = __ldcs(M0 + sl);
                r.v = __ldcs(V0 + sl);
                r.g[0] = __ldcs(G0 + sl * (kGB / 2));
                if constexpr (GK == kF32) r.g[1] = __ldcs(G0 + sl * 2 + 1);
                uint32_t wp[4], wm[4], wv[4];
                if constexpr ((COLD & 2) != 0) {
                    // all eight cold (M == 0, V >= 0, p finite): cold_elem's
                    // first route, P = (p - lr * M) - lr_wd * p; the test
                    // first, then the pairs recomputed (no 24 live floats)
                    bool cold = sc.fast;
#pragma unroll
                    for (int k = 0; k < 8; ++k) {
                        const float g = __fmul_rn(k3_grad<GK>(r, k), sc.inv_scale);
                        const float M = __fadd_rn(__fmul_rn(c.beta1, bf16_lane(r.m, k)),
                                                  __fmul_rn(c.one_minus_b1, g));
                        const float V = __fadd_rn(__fmul_rn(c.beta2, bf16_lane(r.v, k)),
                                                  __fmul_rn(c.one_minus_b2, __fmul_rn(g, g)));
                        cold &= (M == 0.0f) & (V >= 0.0f) & fast_p_ok(bf16_lane(r.p, k));
                    }
                    if (cold) {
#pragma unroll
                        for (int k = 0; k < 8; k += 2) {
                            float P[2], M[2], V[2];
#pragma unroll
                            for (int h = 0; h < 2; ++h) {
                                const float p = bf16_lane(r.p, k + h);
                                const float g = __fmul_rn(k3_grad<GK>(r, k + h), sc.inv_scale);
                                M[h] = __fadd_rn(__fmul_rn(c.beta1, bf16_lane(r.m, k + h)),
                                                 __fmul_rn(c.one_minus_b1, g));
                                V[h] = __fadd_rn(__fmul_rn(c.beta2, bf16_lane(r.v, k + h)),
                                                 __fmul_rn(c.one_minus_b2, __fmul_rn(g, g)));
                                P[h] = __fsub_rn(__fsub_rn(p, __fmul_rn(c.lr, M[h])),
                                                 __fmul_rn(c.lr_wd, p));
                            }
                            wp[k >> 1] = narrow2<kBF16>(P[0], P[1]);
                            wm[k >> 1] = narrow2<kBF16>(M[0], M[1]);
                            wv[k >> 1] = narrow2<kBF16>(V[0], V[1]);
                        }
                        __stcs(P0 + sl, make_uint4(wp[0], wp[1], wp[2], wp[3]));
                        __stcs(M0 + sl, make_uint4(wm[0], wm[1], wm[2], wm[3]));
                        __stcs(V0 + sl, make_uint4(wv[0], wv[1], wv[2], wv[3]));
                        continue;
                    }
                }
                if constexpr ((COLD & 4) != 0) {
                    // the vector second chance: every element takes one of
                    // adam_any's non-IEEE routes — the fast sequences, the
                    // M == 0 shortcut or the 2^64-scaled sequences for
                    // |M| in [2^-100, 2^-50) (cold_elem) — packed pair by
                    // pair; any element outside them sends the whole slot
                    // to the per-element path below.  A slot that is all
                    // M == 0 (an untouched row) skips the sequences.
                    bool ok = sc.fast;
                    // on the raw bits (no values to keep): m = g = +-0 gives
                    // M = +-0 exactly, and v >= 0 then gives V >= 0
                    uint32_t zm = (r.m.x | r.m.y | r.m.z | r.m.w) & 0x7FFF7FFFu;
                    if constexpr (GK == kF32) {
                        zm |= (r.g[0].x | r.g[0].y | r.g[0].z | r.g[0].w | r.g[1].x | r.g[1].y |
                               r.g[1].z | r.g[1].w) & 0x7FFFFFFFu;
                    } else {
                        zm |= (r.g[0].x | r.g[0].y | r.g[0].z | r.g[0].w) & 0x7FFF7FFFu;  // bf16 / fp16 +-0
                    }
                    bool allzero = ok && zm == 0u;
#pragma unroll
                    for (int k = 0; k < 8; ++k) {
                        allzero &= (bf16_lane(r.v, k) >= 0.0f) & fast_p_ok(bf16_lane(r.p, k));
                    }
#pragma unroll
                    for (int k = 0; k < 8; k += 2) {
                        if (!ok) break;  // also keeps the pairs' live ranges apart
                        float P[2], M[2], V[2];
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            const float p = bf16_lane(r.p, k + h);
                            const float g = __fmul_rn(k3_grad<GK>(r, k + h), sc.inv_scale);
                            M[h] = __fadd_rn(__fmul_rn(c.beta1, bf16_lane(r.m, k + h)),
                                             __fmul_rn(c.one_minus_b1, g));
                            V[h] = __fadd_rn(__fmul_rn(c.beta2, bf16_lane(r.v, k + h)),
                                             __fmul_rn(c.one_minus_b2, __fmul_rn(g, g)));
                            float q = M[h];  // the M == 0 route
                            if (!allzero) {
                                const float am = fabsf(M[h]);
                                const bool vok = fast_v_ok(V[h]);
                                const bool fastr = fast_m_ok(M[h]) & vok;
                                const bool zero = (M[h] == 0.0f) & (V[h] >= 0.0f);
                                const bool scaled = (am >= 0x1p-100f) & (am < 0x1p-50f) & vok;
                                const float ms = scaled ? __fmul_rn(M[h], 0x1p64f) : M[h];
                                const float mh = div_by(ms, sc.bc1, sc.y1);
                                // M == 0: q = M for any positive den; V = 1 keeps it finite
                                const float vh = div_by(zero ? 1.0f : V[h], sc.bc2, sc.y2);
                                const float den = __fadd_rn(sqrt_fast(vh), c.eps);
                                const float qs = div_by(mh, den, rcp_refined(den));
                                q = zero ? M[h] : scaled ? __fmul_rn(qs, 0x1p-64f) : qs;
                                ok &= fast_p_ok(p) &
                                      (fastr | zero | (scaled & (fabsf(qs) >= 0x1p-61f)));
                            }
                            P[h] = __fsub_rn(__fsub_rn(p, __fmul_rn(c.lr, q)),
                                             __fmul_rn(c.lr_wd, p));
                        }
                        wp[k >> 1] = narrow2<kBF16>(P[0], P[1]);
                        wm[k >> 1] = narrow2<kBF16>(M[0], M[1]);
                        wv[k >> 1] = narrow2<kBF16>(V[0], V[1]);
                    }
                    if (ok) {
                        __stcs(P0 + sl, make_uint4(wp[0], wp[1], wp[2], wp[3]));
                        __stcs(M0 + sl, make_uint4(wm[0], wm[1], wm[2], wm[3]));
                        __stcs(V0 + sl, make_uint4(wv[0], wv[1], wv[2], wv[3]));
                        continue;
                    }
                }
#pragma unroll
                for (int k = 0; k < 8; k += 2) {
                    float p2[2], m2[2], v2[2];
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        p2[h] = bf16_lane(r.p, k + h);
                        m2[h] = bf16_lane(r.m, k + h);
                        v2[h] = bf16_lane(r.v, k + h);
                        adam_any<kOrdBf16>(p2[h], m2[h], v2[h], k3_grad<GK>(r, k + h), c, sc);
                    }
                    wp[k >> 1] = narrow2<kBF16>(p2[0], p2[1]);
                    wm[k >> 1] = narrow2<kBF16>(m2[0], m2[1]);
                    wv[k >> 1] = narrow2<kBF16>(v2[0], v2[1]);
                }
                __stcs(P0 + sl, make_uint4(wp[0], wp[1], wp[2], wp[3]));
                __stcs(M0 + sl, make_uint4(wm[0], wm[1], wm[2], wm[3]));
                __stcs(V0 + sl, make_uint4(wv[0], wv[1], wv[2], wv[3]));
            }
        }
    }
        return;
    }
    const uint64_t q0 = blockIdx.x - main_ctas;
    const uint64_t nq = gridDim.x - main_ctas;
    for (uint32_t k = 0; k < tab.count; ++k) {
        const Seg& sg = tab.seg[k];
        if (sg.vector_ok) {
            if (q0 != k % nq) continue;
            const uint64_t tail_begin = sg.head + sg.nvec * 8;
            const uint64_t extra = sg.head + (sg.n - tail_begin);
            for (uint64_t i = threadIdx.x; i < extra; i += blockDim.x) {
                bf16_state_scalar<GK>(sg, i < sg.head ? i : tail_begin + (i - sg.head), c, sc);
            }
        } else {
            for (uint64_t e = q0 * blockDim.x + threadIdx.x; e < sg.n; e += nq * blockDim.x) {
                bf16_state_scalar<GK>(sg, e, c, sc);
            }
        }
    }
}

// ============================================================== step finish
// The next update's scalars (t = updates + 1, current scale) into StepDev.
__device__ void step_prepare(StepDev* st, const float2* bc_table, unsigned long long bc_first,
                             const AdamConsts c) {
    const float2 bc = bc_table[st->updates + 1ull - bc_first];  // t = updates + 1
    StepScalars s;
    scalars_from(st->scale, bc.x, bc.y, c, s);
    st->inv_scale = s.scale_pow2 ? s.inv_scale : 0.0f;
    st->bc1 = s.bc1;
    st->bc2 = s.bc2;
    st->y1 = s.y1;
    st->y2 = s.y2;
    st->mode = (s.scale_pow2 ? 1u : 0u) | (s.fast ? 2u : 0u);
}

__global__ void k_step_prepare(StepDev* st, const float2* bc_table, unsigned long long bc_first,
                               const AdamConsts c) {
    if (threadIdx.x == 0 && blockIdx.x == 0) step_prepare(st, bc_table, bc_first, c);
}

// LossScaler::on_overflow / on_clean_step (optimizer.hpp:24-34) and the
// update counter (simulator.cpp:438-444,491); re-arms the flag and prepares
// the next update's scalars.
__global__ void k_step_finish(StepDev* st, StepLog* log, const float2* bc_table,
                              unsigned long long bc_first, const AdamConsts c) {
    pdl_wait();
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    const uint32_t of = st->flag != 0u;
    if (of) {
        st->scale = st->scale * 0.5f;
        st->clean_steps = 0;
    } else {
        st->updates += 1ull;
        st->clean_steps += 1u;
        if (st->clean_steps >= st->growth_interval) {
            st->scale = st->scale * 2.0f;
            st->clean_steps = 0;
        }
    }
    log[st->steps % kHistory] = StepLog{st->scale, of};
    st->steps += 1ull;
    st->last_overflow = of;
    st->flag = 0u;
    step_prepare(st, bc_table, bc_first, c);
}

// ============================================================== generators
template <int WK>
__global__ void k_gen_weights(float* __restrict__ p, uint16_t* __restrict__ w, uint64_t n,
                              uint64_t base, uint64_t seed) {
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
         i += stride) {
        const float x = seeded_weight(seed, base + i);
        if (p) p[i] = x;
        if constexpr (WK != kNone) w[i] = narrow<WK>(x);
    }
}

template <int GK, int WK>
__global__ void k_gen_grads(void* __restrict__ g, const uint16_t* __restrict__ w, uint64_t n,
                            uint64_t base, uint64_t seed, uint64_t step, const float* d_scale,
                            float scale) {
    const float sc = d_scale ? *d_scale : scale;
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
         i += stride) {
        const float gs = __fmul_rn(pseudo_gradient(seed, step, base + i, widen<WK>(w[i])), sc);
        if constexpr (GK == kF32) {
            reinterpret_cast<float*>(g)[i] = gs;
        } else {
            reinterpret_cast<uint16_t*>(g)[i] = narrow<GK>(gs);
        }
    }
}

// Producer-side fused check: the scaled store into the
// flat gradient buffer that simulator.cpp:401-405 performs
// (flat[i] = g * scale), with K1's exponent test applied to the stored value
// in the same pass — the optimizer step then needs no separate K1 read.
// ============================================================== K4
// Reduce-scatter epilogue check (the order and NaN rule
// are those of oracle ora_reduce_check).  Sources are this rank's partition
// on every rank, read over NVLink through CUDA IPC mappings (or any pointers
// the device can load); each element is read once from each rank, summed in
// rank order in fp32, scaled, stored once and tested once — the K1 pass over
// the flat buffer disappears.  Streaming 128-bit loads; peers are read in
// rank order, two ranks' units in flight together (rs_units(SK) 16- or
// 32-byte units per thread per rank).
// Raw (still packed) unit: the loads of two ranks stay in flight in 2 x U
// uint4 registers (16-bit kinds) and are widened as they are added.
template <int K>
struct RsRaw {
    uint4 q[K == kF32 ? 2 : 1];
};

template <int K>
__device__ __forceinline__ RsRaw<K> rs_raw(const void* base, uint64_t j) {
    RsRaw<K> r;
    if constexpr (K == kF32) {
        const uint4* s = reinterpret_cast<const uint4*>(base) + 2 * j;
        r.q[0] = __ldcs(s);
        r.q[1] = __ldcs(s + 1);
    } else {
        r.q[0] = __ldcs(reinterpret_cast<const uint4*>(base) + j);
    }
    return r;
}

template <int K>
__device__ __forceinline__ float rs_elem(const RsRaw<K>& r, int k) {
    if constexpr (K == kF32) {
        const uint4& q = r.q[k >> 2];
        const uint32_t w = (k & 3) == 0 ? q.x : (k & 3) == 1 ? q.y : (k & 3) == 2 ? q.z : q.w;
        return __uint_as_float(w);
    } else {
        const uint4& q = r.q[0];
        const uint32_t w = (k >> 1) == 0 ? q.x : (k >> 1) == 1 ? q.y : (k >> 1) == 2 ? q.z : q.w;
        return widen<K>((k & 1) ? (w >> 16) : (w & 0xFFFFu));
    }
}

template <int K>
__device__ __forceinline__ float rs_load1(const void* base, uint64_t e) {
    return K == kF32 ? reinterpret_cast<const float*>(base)[e]
                     : widen<K>(reinterpret_cast<const uint16_t*>(base)[e]);
}

__device__ __forceinline__ float rs_finish(float acc, float post_scale) {
    if (post_scale != 1.0f) acc = __fmul_rn(acc, post_scale);
    return isnan(acc) ? __uint_as_float(0x7FC00000u) : acc;
}

// store 8 results; returns the OR of (word & MASK) + INC over the stored words
template <int K>
__device__ __forceinline__ uint32_t rs_store8(void* base, uint64_t j, const float (&x)[8]) {
    const ScanWord sw = scan_word(K);
    if constexpr (K == kF32) {
        float4* d = reinterpret_cast<float4*>(base) + 2 * j;
        __stcs(d, make_float4(x[0], x[1], x[2], x[3]));
        __stcs(d + 1, make_float4(x[4], x[5], x[6], x[7]));
        uint32_t acc = 0;
#pragma unroll
        for (int k = 0; k < 8; ++k) acc |= (__float_as_uint(x[k]) & sw.mask) + sw.inc;
        return acc;
    } else {
        uint32_t w[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            w[k] = narrow2<K>(x[2 * k], x[2 * k + 1]);
        }
        __stcs(reinterpret_cast<uint4*>(base) + j, make_uint4(w[0], w[1], w[2], w[3]));
        return ((w[0] & sw.mask) + sw.inc) | ((w[1] & sw.mask) + sw.inc) |
               ((w[2] & sw.mask) + sw.inc) | ((w[3] & sw.mask) + sw.inc);
    }
}

// rs_store8 without the per-pair NaN branch (pair conversions only): the
// stored words carry the GPU's canonical NaN; callers re-store a unit whose
// check bits show a non-finite value with the defined NaN rule.
template <int K>
__device__ __forceinline__ uint32_t rs_store8_num(void* base, uint64_t j, const float (&x)[8]) {
    const ScanWord sw = scan_word(K);
    if constexpr (K == kF32) {
        return rs_store8<K>(base, j, x);
    } else {
        uint32_t w[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) w[k] = narrow2_num<K>(x[2 * k], x[2 * k + 1]);
        __stcs(reinterpret_cast<uint4*>(base) + j, make_uint4(w[0], w[1], w[2], w[3]));
        return ((w[0] & sw.mask) + sw.inc) | ((w[1] & sw.mask) + sw.inc) |
               ((w[2] & sw.mask) + sw.inc) | ((w[3] & sw.mask) + sw.inc);
    }
}

// Producer-side check: dst = cast(src * scale) with the
// overflow test on the stored values.  One tile of U x 256 eight-element
// units per CTA, 16-byte accesses (src and dst co-aligned at element
// `head`), trailing CTAs for the scalar head/tail.  Per element exactly the
// arithmetic of the reference store (simulator.cpp:401-405): fp32 multiply,
// then the cast.
template <int SK, int DK, int U>
__global__ void __launch_bounds__(256) k_ingest(IngestArgs a) {
    const float sc = *a.d_scale;
    constexpr uint32_t kSB = SK == kF32 ? 4 : 2, kDB = DK == kF32 ? 4 : 2;
    const uint32_t top = scan_word(DK).top;
    uint32_t acc_bits = 0;
    bool bad = false;
    if (blockIdx.x < a.tiles) {
        const uint64_t j0 = static_cast<uint64_t>(blockIdx.x) * U * blockDim.x + threadIdx.x;
        const uint8_t* sb = static_cast<const uint8_t*>(a.src) + a.head * kSB;
        uint8_t* db = static_cast<uint8_t*>(a.dst) + a.head * kDB;
        RsRaw<SK> x[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t j = j0 + static_cast<uint64_t>(u) * blockDim.x;
            if (j < a.nvec) x[u] = rs_raw<SK>(sb, j);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t j = j0 + static_cast<uint64_t>(u) * blockDim.x;
            if (j >= a.nvec) continue;
            float y[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) y[k] = __fmul_rn(rs_elem<SK>(x[u], k), sc);
            const uint32_t unit = rs_store8<DK>(db, j, y);
            if ((unit & top) != 0u) {
                // a non-finite unit (rare): store it again with the x86 NaN
                // of `g * scale` (simulator.cpp:404) — the gradient's payload,
                // quieted — instead of the GPU's canonical NaN
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const float xk = rs_elem<SK>(x[u], k);
                    y[k] = x86(y[k], xk, sc);
                }
                rs_store8<DK>(db, j, y);
            }
            acc_bits |= unit;
        }
    } else {
        const uint64_t q0 = blockIdx.x - a.tiles, nq = gridDim.x - a.tiles;
        const uint64_t tail_begin = a.head + a.nvec * 8;
        const uint64_t extra = a.head + (a.n - tail_begin);
        for (uint64_t k = q0 * blockDim.x + threadIdx.x; k < extra; k += nq * blockDim.x) {
            const uint64_t i = k < a.head ? k : tail_begin + (k - a.head);
            const float xs = rs_load1<SK>(a.src, i);
            const float gs = x86(__fmul_rn(xs, sc), xs, sc);
            if constexpr (DK == kF32) {
                reinterpret_cast<float*>(a.dst)[i] = gs;
                bad |= elem_non_finite(__float_as_uint(gs), kF32);
            } else {
                const uint16_t h = narrow<DK>(gs);
                reinterpret_cast<uint16_t*>(a.dst)[i] = h;
                bad |= elem_non_finite(h, DK);
            }
        }
    }
    if (__any_sync(0xFFFFFFFFu, bad || (acc_bits & top) != 0u) && (threadIdx.x & 31u) == 0)
        *a.flag = 1u;
}

int ingest_units(int sk) { return sk == kF32 ? 2 : 4; }

void launch_ingest(int sk, int dk, const IngestArgs& a, unsigned grid, cudaStream_t st) {
#define MA_ING(S, D)                                                                   \
    if (sk == S && dk == D) {                                                          \
        k_ingest<S, D, (S == kF32 ? 2 : 4)><<<grid, 256, 0, st>>>(a);                 \
        return;                                                                        \
    }
    MA_ING(kF32, kF32) MA_ING(kF32, kBF16) MA_ING(kF32, kF16)
    MA_ING(kBF16, kF32) MA_ING(kBF16, kBF16) MA_ING(kBF16, kF16)
    MA_ING(kF16, kF32) MA_ING(kF16, kBF16) MA_ING(kF16, kF16)
#undef MA_ING
}

template <int SK, int DK>
__device__ __forceinline__ bool rs_scalar(const RsArgs& a, uint64_t e) {
    float acc = rs_load1<SK>(a.src[0], e);
    for (uint32_t r = 1; r < a.nsrc; ++r) acc = __fadd_rn(acc, rs_load1<SK>(a.src[r], e));
    acc = rs_finish(acc, a.post_scale);
    if constexpr (DK == kF32) {
        reinterpret_cast<float*>(a.dst)[e] = acc;
        return elem_non_finite(__float_as_uint(acc), kF32);
    } else {
        const uint16_t h = narrow<DK>(acc);
        reinterpret_cast<uint16_t*>(a.dst)[e] = h;
        return elem_non_finite(h, DK);
    }
}

// ONE = 1: the single-source specialisation (world 1, or a scaled copy with
// the check): no second-source registers, so 6 CTAs fit per SM instead of 3.
// HALF = 1: half the units per thread (many sources: more CTAs instead of
// more loads per thread; the host sizes tiles with rs_units_for)
template <int SK, int DK, int ONE = 0, int HALF = 0>
__global__ void __launch_bounds__(256, ONE ? 6 : HALF ? 5 : 3) k4_reduce_check(RsArgs a) {
    constexpr int U = HALF ? (rs_units(SK) > 1 ? rs_units(SK) / 2 : 1) : rs_units(SK);
    constexpr uint32_t kSrcBytes = SK == kF32 ? 4 : 2, kDstBytes = DK == kF32 ? 4 : 2;
    const unsigned lane = threadIdx.x & 31u;
    const uint32_t top = scan_word(DK).top;
    uint32_t acc_bits = 0;
    bool bad = false;
    if (blockIdx.x < a.tiles) {
        const uint64_t j0 = static_cast<uint64_t>(blockIdx.x) * U * blockDim.x + threadIdx.x;
        const bool full = j0 + (U - 1) * static_cast<uint64_t>(blockDim.x) < a.nvec;
        float acc[U][8];
        uint32_t r;
        {
            // sources 0 and 1 together: acc = src0 (+ src1), the same
            // roundings as starting from src0 and adding src1
            const uint8_t* b0 = static_cast<const uint8_t*>(a.src[0]) + a.head * kSrcBytes;
            const uint8_t* b1 = static_cast<const uint8_t*>(a.src[a.nsrc > 1 ? 1 : 0]) + a.head * kSrcBytes;
            if constexpr (ONE != 0) {
                RsRaw<SK> x[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const uint64_t j = j0 + static_cast<uint64_t>(u) * blockDim.x;
                    if (full || j < a.nvec) x[u] = rs_raw<SK>(b0, j);
                }
#pragma unroll
                for (int u = 0; u < U; ++u) {
#pragma unroll
                    for (int k = 0; k < 8; ++k) acc[u][k] = rs_elem<SK>(x[u], k);
                }
                r = 1;
            } else {
            RsRaw<SK> x[U], y[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const uint64_t j = j0 + static_cast<uint64_t>(u) * blockDim.x;
                if (full || j < a.nvec) {
                    x[u] = rs_raw<SK>(b0, j);
                    if (a.nsrc > 1) y[u] = rs_raw<SK>(b1, j);
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    acc[u][k] = a.nsrc > 1 ? __fadd_rn(rs_elem<SK>(x[u], k), rs_elem<SK>(y[u], k))
                                           : rs_elem<SK>(x[u], k);
                }
            }
            r = a.nsrc > 1 ? 2 : 1;
            }
        }
        for (; ONE == 0 && r + 1 < a.nsrc; r += 2) {
            const uint8_t* b0 = static_cast<const uint8_t*>(a.src[r]) + a.head * kSrcBytes;
            const uint8_t* b1 = static_cast<const uint8_t*>(a.src[r + 1]) + a.head * kSrcBytes;
            RsRaw<SK> x[U], y[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const uint64_t j = j0 + static_cast<uint64_t>(u) * blockDim.x;
                if (full || j < a.nvec) {
                    x[u] = rs_raw<SK>(b0, j);
                    y[u] = rs_raw<SK>(b1, j);
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    acc[u][k] = __fadd_rn(__fadd_rn(acc[u][k], rs_elem<SK>(x[u], k)), rs_elem<SK>(y[u], k));
                }
            }
        }
        if (ONE == 0 && r < a.nsrc) {
            const uint8_t* b0 = static_cast<const uint8_t*>(a.src[r]) + a.head * kSrcBytes;
            RsRaw<SK> x[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const uint64_t j = j0 + static_cast<uint64_t>(u) * blockDim.x;
                if (full || j < a.nvec) x[u] = rs_raw<SK>(b0, j);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
#pragma unroll
                for (int k = 0; k < 8; ++k) acc[u][k] = __fadd_rn(acc[u][k], rs_elem<SK>(x[u], k));
            }
        }
        uint8_t* dbody = static_cast<uint8_t*>(a.dst) + a.head * kDstBytes;
        const bool scaled = a.post_scale != 1.0f;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t j = j0 + static_cast<uint64_t>(u) * blockDim.x;
            if (j >= a.nvec) continue;
            float y[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) y[k] = scaled ? __fmul_rn(acc[u][k], a.post_scale) : acc[u][k];
            const uint32_t unit = rs_store8_num<DK>(dbody, j, y);
            if ((unit & top) != 0u) {
                // a non-finite unit (rare): the defined canonical NaN
#pragma unroll
                for (int k = 0; k < 8; ++k) y[k] = rs_finish(acc[u][k], a.post_scale);
                rs_store8<DK>(dbody, j, y);
            }
            acc_bits |= unit;
        }
    } else {
        // trailing CTAs: the scalar head and tail (everything when nvec == 0)
        const uint64_t q0 = blockIdx.x - a.tiles, nq = gridDim.x - a.tiles;
        const uint64_t tail_begin = a.head + a.nvec * 8;
        const uint64_t extra = a.head + (a.n - tail_begin);
        for (uint64_t k = q0 * blockDim.x + threadIdx.x; k < extra; k += nq * blockDim.x) {
            bad |= rs_scalar<SK, DK>(a, k < a.head ? k : tail_begin + (k - a.head));
        }
    }
    if (__any_sync(0xFFFFFFFFu, bad || (acc_bits & top) != 0u) && lane == 0) {
        *a.flag = 1u;
        if (a.xchg) __threadfence();
    }
    if (a.xchg) exchange_epilogue(a.xchg, a.flag, lane);
}

// MA_K4_SINGLE=0 (A/B only) keeps single-source launches on the general kernel
bool k4_single() {
    static const bool on = [] {
        const char* e = std::getenv("MA_K4_SINGLE");
        return !(e && e[0] == '0');
    }();
    return on;
}

// Half the units per thread (and 5 CTAs/SM instead of 3) from
// MA_K4_HALF_MIN sources on (default 2: 2 sources 0.935 -> 0.971 of the copy
// peak, 4 sources 0.88 -> 1.01, 8 sources 0.93 -> 1.02; A/B:
// MA_K4_HALF_MIN=0 disables it)
bool rs_half(int sk, uint32_t nsrc) {
    static const uint32_t from = [] {
        const char* e = std::getenv("MA_K4_HALF_MIN");
        const int v = e ? std::atoi(e) : 2;
        return v <= 0 ? 0xFFFFFFFFu : static_cast<uint32_t>(v);
    }();
    return nsrc >= from && nsrc >= 2 && sk != kF32;
}

int rs_units_for(int sk, uint32_t nsrc) {
    return rs_half(sk, nsrc) ? rs_units(sk) / 2 : rs_units(sk);
}

void launch_reduce_check(int sk, int dk, const RsArgs& a, unsigned grid, cudaStream_t st) {
#define MA_RS(S, D)                                                 \
    if (sk == S && dk == D) {                                       \
        if (a.nsrc == 1 && k4_single())                             \
            k4_reduce_check<S, D, 1><<<grid, 256, 0, st>>>(a);      \
        else if (rs_half(S, a.nsrc))                                \
            k4_reduce_check<S, D, 0, 1><<<grid, 256, 0, st>>>(a);   \
        else                                                        \
            k4_reduce_check<S, D><<<grid, 256, 0, st>>>(a);         \
        return;                                                     \
    }
    MA_RS(kF32, kF32) MA_RS(kF32, kBF16) MA_RS(kF32, kF16)
    MA_RS(kBF16, kF32) MA_RS(kBF16, kBF16) MA_RS(kBF16, kF16)
    MA_RS(kF16, kF32) MA_RS(kF16, kBF16) MA_RS(kF16, kF16)
#undef MA_RS
}

void launch_peer_barrier(const XchgDev* x, cudaStream_t st) {
    k_peer_barrier<<<1, 32, 0, st>>>(x);
}

__global__ void k_plant(void* buf, int dtype, uint64_t index, uint32_t bits) {
    if (dtype == kF32) {
        reinterpret_cast<uint32_t*>(buf)[index] = bits;
    } else {
        reinterpret_cast<uint16_t*>(buf)[index] = static_cast<uint16_t>(bits);
    }
}

// ============================================================== verification
// FNV-1a-64 over each 2^log2 block of fp32->kind conversions (one thread per
// block), through the same narrow<>() K2 uses.
template <int K>
__global__ void k_cast_sweep(int log2, uint64_t* out, uint64_t nblocks) {
    const uint64_t b = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (b >= nblocks) return;
    uint64_t h = 1469598103934665603ull;
    const uint64_t len = 1ull << log2;
    bool lanes_agree = true;
    for (uint64_t k = 0; k < len; k += 2) {
        // consecutive patterns through the pair conversion, and again with the
        // lanes swapped, so every input is checked in both lanes
        const float x0 = __uint_as_float(static_cast<uint32_t>((b << log2) + k));
        const float x1 = __uint_as_float(static_cast<uint32_t>((b << log2) + k + 1));
        const uint32_t w = narrow2<K>(x0, x1);
        const uint32_t sw = narrow2<K>(x1, x0);
        lanes_agree &= sw == ((w >> 16) | (w << 16));
        for (int e = 0; e < 2; ++e) {
            const uint32_t r = (w >> (16 * e)) & 0xFFFFu;
            h = (h ^ (r & 0xFFu)) * 1099511628211ull;
            h = (h ^ (r >> 8)) * 1099511628211ull;
        }
    }
    out[b] = lanes_agree ? h : ~h;
}

// Equality of the hoisted-guard fast path (ma_device.cuh) with the IEEE
// intrinsics over the ranges adam_fast admits:
//  mode 0: sqrt_fast(x) == __fsqrt_rn(x) for EVERY x in [2^-96, 2^96];
//  mode 1: div_by(a, d, rcp_refined(d)) == __fdiv_rn(a, d) for every divisor
//          in `divs` and all 2^24 signed significands of a at eight exponents
//          spanning the admitted range (a power-of-two factor is exact in both);
//  mode 2: `count` seeded random pairs, |a| in [2^-50, 2^66], d in
//          [2^-40, 2^49] (the mh / den division).
__global__ void k_fast_sweep(int mode, const float* divs, uint64_t count, uint64_t seed,
                             unsigned long long* bad) {
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    unsigned long long nbad = 0;
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < count;
         i += stride) {
        if (mode == 0) {
            const float x = __uint_as_float(0x0F800000u + static_cast<uint32_t>(i));
            nbad += __float_as_uint(sqrt_fast(x)) != __float_as_uint(__fsqrt_rn(x));
        } else if (mode == 1) {
            constexpr uint32_t kExp[8] = {31, 32, 77, 126, 127, 176, 177, 205};
            const float d = divs[i >> 27];
            const uint32_t r = static_cast<uint32_t>(i & ((1ull << 27) - 1));
            const uint32_t bits = ((r & (1u << 23)) << 8) | (kExp[r >> 24] << 23) | (r & 0x7FFFFFu);
            const float a = __uint_as_float(bits);
            nbad += __float_as_uint(div_by(a, d, rcp_refined(d))) != __float_as_uint(__fdiv_rn(a, d));
        } else {
            const uint64_t h1 = splitmix64(seed ^ (2 * i)), h2 = splitmix64(seed ^ (2 * i + 1));
            const uint32_t ea = 77 + static_cast<uint32_t>((h1 >> 32) % 117);  // 2^-50 .. 2^66
            const uint32_t ed = 87 + static_cast<uint32_t>((h2 >> 32) % 90);   // 2^-40 .. 2^49
            const float a = __uint_as_float((static_cast<uint32_t>(h1 >> 31) & 0x80000000u) |
                                            (ea << 23) | (static_cast<uint32_t>(h1) & 0x7FFFFFu));
            const float d = __uint_as_float((ed << 23) | (static_cast<uint32_t>(h2) & 0x7FFFFFu));
            nbad += __float_as_uint(div_by(a, d, rcp_refined(d))) != __float_as_uint(__fdiv_rn(a, d));
        }
    }
    if (nbad) atomicAdd(bad, nbad);
}

void launch_fast_sweep(int mode, const float* divs, uint64_t count, uint64_t seed,
                       unsigned long long* bad, unsigned grid) {
    k_fast_sweep<<<grid, 256>>>(mode, divs, count, seed, bad);
}

// K1's word test applied to every pattern vs the IEEE classification.
__global__ void k_mask_sweep(int kind, unsigned long long* mismatches) {
    const ScanWord sw = scan_word(kind);
    const uint64_t total = kind == kF32 ? (1ull << 32) : (1ull << 16);
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    unsigned long long bad = 0;
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < total;
         i += stride) {
        const uint32_t bits = static_cast<uint32_t>(i);
        bool nonfinite;
        uint32_t word;
        if (kind == kF32) {
            nonfinite = !isfinite(__uint_as_float(bits));
            word = bits;
        } else if (kind == kBF16) {
            nonfinite = !isfinite(widen_bf16(bits));
            word = bits << 16;  // test it in the upper lane; lower lane 0 (finite)
        } else {
            nonfinite = !isfinite(widen_f16(bits));
            word = bits << 16;
        }
        const bool vec = (((word & sw.mask) + sw.inc) & sw.top) != 0u;
        const bool scalar = elem_non_finite(bits, kind);
        bad += (vec != nonfinite) + (scalar != nonfinite);
    }
    if (bad) atomicAdd(mismatches, bad);
}

// ============================================================== speculation
__global__ void k_spec_mark(const StepDev* st, uint32_t* marker, uint32_t value) {
    if (threadIdx.x == 0 && blockIdx.x == 0 &&
        *reinterpret_cast<const volatile uint32_t*>(&st->flag) == 0u)
        *marker = value;
}

// Copies back the backups of the first *marker speculated sub-groups when
// the step's flag is set; the last CTA to finish re-arms the marker.
__global__ void __launch_bounds__(256) k_spec_restore(SpecRestore r, const StepDev* st,
                                                      uint32_t* marker) {
    const uint32_t applied = *reinterpret_cast<const volatile uint32_t*>(marker);
    if (st->flag != 0u) {
        const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
        for (uint32_t k = 0; k < r.count; ++k) {
            if (r.c[k].group >= applied) continue;
            const uint64_t first = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
            if (((reinterpret_cast<uintptr_t>(r.c[k].src) | reinterpret_cast<uintptr_t>(r.c[k].dst) |
                  r.c[k].bytes) & 15u) == 0) {
                const uint4* src = static_cast<const uint4*>(r.c[k].src);
                uint4* dst = static_cast<uint4*>(r.c[k].dst);
                for (uint64_t i = first; i < r.c[k].bytes / 16; i += stride) __stcs(dst + i, __ldcs(src + i));
            } else {  // a misaligned view (rare): byte by byte
                const uint8_t* src = static_cast<const uint8_t*>(r.c[k].src);
                uint8_t* dst = static_cast<uint8_t*>(r.c[k].dst);
                for (uint64_t i = first; i < r.c[k].bytes; i += stride) dst[i] = src[i];
            }
        }
    }
    __shared__ bool last;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        last = atomicAdd(marker + 1, 1u) == gridDim.x - 1;  // marker[1]: CTA counter
    }
    __syncthreads();
    if (last && threadIdx.x == 0) {
        marker[0] = 0u;
        marker[1] = 0u;
    }
}

// ============================================================== launchers
void launch_spec_mark(const StepDev* st, uint32_t* marker, uint32_t value, cudaStream_t s) {
    k_spec_mark<<<1, 32, 0, s>>>(st, marker, value);
}

void launch_spec_restore(const SpecRestore& r, const StepDev* st, uint32_t* marker, unsigned grid,
                         cudaStream_t s) {
    k_spec_restore<<<grid, 256, 0, s>>>(r, st, marker);
}

// Launch as a programmatic dependent of the previous kernel in the stream
// (the kernel must pdl_wait() before consuming that kernel's results).
template <typename... P, typename... A>
void launch_pdl(void (*fn)(P...), unsigned grid, unsigned block, cudaStream_t st, A&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, fn, std::forward<A>(args)...);
}

int k1_ldk() {
    static const int v = [] {
        const char* e = std::getenv("MA_K1_LDK");  // A/B only
        return e ? std::atoi(e) : 1;
    }();
    return v;
}

// MA_PDL=0 turns every programmatic launch into a plain one (the kernels'
// griddepcontrol instructions are then no-ops); MA_PDL_FINISH / MA_PDL_K3 =
// 0 do it for the scaler / K3 alone (A/B).
bool pdl_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("MA_PDL");
        return !(e && e[0] == '0');
    }();
    return on;
}

bool pdl_finish() {
    static const bool on = [] {
        const char* e = std::getenv("MA_PDL_FINISH");  // A/B only (0 = plain launch)
        return !(e && e[0] == '0');
    }();
    return on && pdl_enabled();
}

void launch_k1(const K1Args& a, bool track, int unroll, bool oneshot, unsigned grid,
               cudaStream_t st) {
    if (oneshot) {
        if (track) {
            k1_oneshot<true, kK1Unroll><<<grid, kK1Threads, 0, st>>>(a);
        } else if (k1_ldk() == 0 || a.keep_from >= a.nvec) {
            k1_oneshot<false, kK1Unroll, 0><<<grid, kK1Threads, 0, st>>>(a);
        } else if (k1_ldk() == 2) {
            k1_oneshot<false, kK1Unroll, 2><<<grid, kK1Threads, 0, st>>>(a);
        } else {
            k1_oneshot<false, kK1Unroll, 1><<<grid, kK1Threads, 0, st>>>(a);
        }
        return;
    }
    if (track) {
        k1_overflow<true, 4><<<grid, kK1Threads, 0, st>>>(a);
    } else if (unroll == 8) {
        k1_overflow<false, 8><<<grid, kK1Threads, 0, st>>>(a);
    } else {
        k1_overflow<false, 4><<<grid, kK1Threads, 0, st>>>(a);
    }
}

namespace {

// K2 variants (see kernels.cuh: k2_variant_shape).  Every dtype pair gets the
// production variant; the bench pair (bf16 grads, bf16 weights) additionally
// carries the alternatives used for the A/B measurements in DESIGN.md.
template <int GK, int WK, int V>
struct K2Kernel;
template <int GK, int WK> struct K2Kernel<GK, WK, 0> { static constexpr auto fn = k2_adam<GK, WK, 8>; };
template <int GK, int WK> struct K2Kernel<GK, WK, 1> { static constexpr auto fn = k2_adam<GK, WK, 4>; };
template <int GK, int WK> struct K2Kernel<GK, WK, 2> { static constexpr auto fn = k2_stream<GK, WK, 2, false>; };
template <int GK, int WK> struct K2Kernel<GK, WK, 3> { static constexpr auto fn = k2_stream<GK, WK, 1, true>; };
template <int GK, int WK> struct K2Kernel<GK, WK, 4> { static constexpr auto fn = k2_stream<GK, WK, 2, true>; };
template <int GK, int WK> struct K2Kernel<GK, WK, 5> { static constexpr auto fn = k2_stream<GK, WK, 4, false>; };
template <int GK, int WK> struct K2Kernel<GK, WK, 6> { static constexpr auto fn = k2_stream<GK, WK, 2, false, 5, 0>; };
template <int GK, int WK> struct K2Kernel<GK, WK, 7> { static constexpr auto fn = k2_stream<GK, WK, 2, false, 1, 1>; };
template <int GK, int WK> struct K2Kernel<GK, WK, 8> { static constexpr auto fn = k2_stream<GK, WK, 2, false, 1, 2>; };
template <int GK, int WK> struct K2Kernel<GK, WK, 9> { static constexpr auto fn = k2_stream<GK, WK, 2, false, 6, 0>; };
// 12: PROBE ONLY (approximate div/sqrt, not bit-exact) — bounds the cost of the IEEE sequences
template <int GK, int WK> struct K2Kernel<GK, WK, 12> { static constexpr auto fn = k2_stream<GK, WK, 2, false, 1, 3>; };
// 13-15: one tile per CTA (k2_oneshot) with U = 2, 4, 1 slots per thread
template <int GK, int WK> struct K2Kernel<GK, WK, 13> { static constexpr auto fn = k2_oneshot<GK, WK, 2>; };
template <int GK, int WK> struct K2Kernel<GK, WK, 14> { static constexpr auto fn = k2_oneshot<GK, WK, 4>; };
template <int GK, int WK> struct K2Kernel<GK, WK, 15> { static constexpr auto fn = k2_oneshot<GK, WK, 1>; };
// 16: PROBE ONLY — variant 14 with approximate div/sqrt (power/instruction headroom)
template <int GK, int WK> struct K2Kernel<GK, WK, 16> { static constexpr auto fn = k2_oneshot<GK, WK, 4, 1>; };
// 17: variant 14 held to 3 CTAs/SM (<= 80 registers); 18: variant 14 with the
// exact intrinsics only (no hoisted-guard fast path) — the previous production
template <int GK, int WK> struct K2Kernel<GK, WK, 17> { static constexpr auto fn = k2_oneshot<GK, WK, 4, 0, 3>; };
template <int GK, int WK> struct K2Kernel<GK, WK, 18> { static constexpr auto fn = k2_oneshot<GK, WK, 4, 2>; };
// 19: variant 14 with rejected slots deferred to the CTA's list (no call in the hot loop)
template <int GK, int WK> struct K2Kernel<GK, WK, 19> { static constexpr auto fn = k2_oneshot<GK, WK, 4, 0, 1, 0, true>; };
// 20 / 21: variant 14 launched as a programmatic dependent of K1 (wait first /
// the tile's loads issued before the wait)
template <int GK, int WK> struct K2Kernel<GK, WK, 20> { static constexpr auto fn = k2_oneshot<GK, WK, 4, 0, 1, 0, false, 1>; };
template <int GK, int WK> struct K2Kernel<GK, WK, 21> { static constexpr auto fn = k2_oneshot<GK, WK, 4, 0, 1, 0, false, 2>; };
// 22: variant 14 with the tiles in reverse order (L2 reuse of K1's last gradients)
template <int GK, int WK> struct K2Kernel<GK, WK, 22> { static constexpr auto fn = k2_oneshot<GK, WK, 4, 0, 1, 0, false, 0, true>; };

template <int GK, int WK, int V>
int k2_occupancy() {
    static const int b = [] {
        int x = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&x, K2Kernel<GK, WK, V>::fn, kK2Threads, 0);
        return x > 0 ? x : 1;
    }();
    return b;
}

template <int GK, int WK, typename F>
void k2_variants(int variant, F&& f) {
    if constexpr (GK == kBF16 && WK == kBF16) {
        switch (variant) {
            case 0: f(std::integral_constant<int, 0>{}); return;
            case 1: f(std::integral_constant<int, 1>{}); return;
            case 2: f(std::integral_constant<int, 2>{}); return;
            case 3: f(std::integral_constant<int, 3>{}); return;
            case 4: f(std::integral_constant<int, 4>{}); return;
            case 5: f(std::integral_constant<int, 5>{}); return;
            case 6: f(std::integral_constant<int, 6>{}); return;
            case 7: f(std::integral_constant<int, 7>{}); return;
            case 8: f(std::integral_constant<int, 8>{}); return;
            case 9: f(std::integral_constant<int, 9>{}); return;
            case 12: f(std::integral_constant<int, 12>{}); return;
            case 13: f(std::integral_constant<int, 13>{}); return;
            case 14: f(std::integral_constant<int, 14>{}); return;
            case 15: f(std::integral_constant<int, 15>{}); return;
            case 16: f(std::integral_constant<int, 16>{}); return;
            case 17: f(std::integral_constant<int, 17>{}); return;
            case 18: f(std::integral_constant<int, 18>{}); return;
            case 19: f(std::integral_constant<int, 19>{}); return;
            case 20: f(std::integral_constant<int, 20>{}); return;
            case 21: f(std::integral_constant<int, 21>{}); return;
            case 22: f(std::integral_constant<int, 22>{}); return;
            default: break;
        }
    }
    f(std::integral_constant<int, kK2DefaultVariant>{});
}

template <typename F>
void k2_dispatch(int gk, int wk, int variant, F&& f) {
#define MA_K2_CASE(G, W)                                                          \
    if (gk == G && wk == W) {                                                     \
        k2_variants<G, W>(variant, [&](auto V) { f(std::integral_constant<int, G>{}, \
                                                   std::integral_constant<int, W>{}, V); }); \
        return;                                                                   \
    }
    MA_K2_CASE(kF32, kNone) MA_K2_CASE(kF32, kBF16) MA_K2_CASE(kF32, kF16)
    MA_K2_CASE(kBF16, kNone) MA_K2_CASE(kBF16, kBF16) MA_K2_CASE(kBF16, kF16)
    MA_K2_CASE(kF16, kNone) MA_K2_CASE(kF16, kBF16) MA_K2_CASE(kF16, kF16)
#undef MA_K2_CASE
}

}  // namespace

namespace {

constexpr int kTmaVariant = 10;     // 128 consumer threads per CTA
constexpr int kTmaVariantWide = 11; // 256 consumer threads per CTA

size_t tma_smem_bytes() {
    return static_cast<size_t>(kTmaStages) * tma_stage_bytes<kBF16>() + 2 * kTmaStages * 8;
}

template <int NC>
int tma_blocks_per_sm() {
    static const int b = [] {
        cudaFuncSetAttribute(k2_tma<kBF16, kBF16, NC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(tma_smem_bytes()));
        int x = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&x, k2_tma<kBF16, kBF16, NC>, NC + 32,
                                                      tma_smem_bytes());
        return x > 0 ? x : 1;
    }();
    return b;
}

bool is_tma(int variant) { return variant == kTmaVariant || variant == kTmaVariantWide; }

}  // namespace

int k2_effective_variant(int gk, int wk, int variant) {
    if (is_tma(variant) && gk == kBF16 && wk == kBF16) return variant;
    int v = kK2DefaultVariant;
    k2_dispatch(gk, wk, variant, [&](auto, auto, auto V) { v = decltype(V)::value; });
    return v;
}

bool k2_variant_oneshot(int variant) { return variant >= 13 && variant <= 22; }

void k2_variant_shape(int variant, int* vec, int* tile_vectors, bool* stream) {
    if (is_tma(variant)) {
        *vec = 8;
        *tile_vectors = kTmaTile / 8;
        *stream = true;
        return;
    }
    if (k2_variant_oneshot(variant)) {
        *vec = 4;
        *tile_vectors = (variant == 13 ? 2 : variant == 15 ? 1 : 4) * kK2Threads;
        *stream = true;
        return;
    }
    static const int kVec[10] = {8, 4, 4, 4, 4, 4, 4, 4, 4, 4};
    static const int kTile[10] = {kK2Threads, kK2Threads, 2 * kK2Threads, kK2Threads,
                                  2 * kK2Threads, 4 * kK2Threads, 2 * kK2Threads, 2 * kK2Threads,
                                  2 * kK2Threads, 2 * kK2Threads};
    const int v = variant >= 0 && variant < 10 ? variant : 2;  // 12 = variant 2's shape
    *vec = kVec[v];
    *tile_vectors = kTile[v];
    *stream = v >= 2;
}

int k2_blocks_per_sm(int gk, int wk, int variant) {
    if (variant == kTmaVariant) return tma_blocks_per_sm<128>();
    if (variant == kTmaVariantWide) return tma_blocks_per_sm<256>();
    int b = 1;
    k2_dispatch(gk, wk, variant, [&](auto G, auto W, auto V) {
        b = k2_occupancy<decltype(G)::value, decltype(W)::value, decltype(V)::value>();
    });
    return b;
}

void launch_k2(int gk, int wk, int variant, const SegTable& tab, const AdamArgs& a, unsigned grid,
               cudaStream_t st) {
    if (variant == kTmaVariant) {
        tma_blocks_per_sm<128>();  // sets the dynamic shared-memory attribute once
        k2_tma<kBF16, kBF16, 128><<<grid, 160, tma_smem_bytes(), st>>>(tab, a);
        return;
    }
    if (variant == kTmaVariantWide) {
        tma_blocks_per_sm<256>();
        k2_tma<kBF16, kBF16, 256><<<grid, 288, tma_smem_bytes(), st>>>(tab, a);
        return;
    }
    k2_dispatch(gk, wk, variant, [&](auto G, auto W, auto V) {
        constexpr int v = decltype(V)::value;
        auto fn = K2Kernel<decltype(G)::value, decltype(W)::value, v>::fn;
        if constexpr (v == 20 || v == 21) {
            if (pdl_enabled()) {
                launch_pdl(fn, grid, kK2Threads, st, tab, a);
            } else {
                fn<<<grid, kK2Threads, 0, st>>>(tab, a);
            }
        } else {
            fn<<<grid, kK2Threads, 0, st>>>(tab, a);
        }
    });
}

void launch_k2_allgather(int gk, int wk, const SegTable& tab, const AdamArgs& a, unsigned grid,
                         cudaStream_t st) {
#define MA_AG(G, W)                                                                    \
    if (gk == G && wk == W) {                                                          \
        k2_oneshot<G, W, 4, 0, 1, 1><<<grid, kK2Threads, 0, st>>>(tab, a);             \
        return;                                                                        \
    }
    MA_AG(kF32, kBF16) MA_AG(kF32, kF16) MA_AG(kBF16, kBF16) MA_AG(kBF16, kF16)
    MA_AG(kF16, kBF16) MA_AG(kF16, kF16)
#undef MA_AG
}

// K3 A/B (MA_K3_VARIANT), fractions of the copy peak at 268 M
// params, bf16 g.  0 = production: k3_v2, two 8-element slots per thread at
// 4 CTA/SM, the admission guard on NaN-propagating min / max reductions,
// slots that fail it deferred to a shared-memory list and computed after the
// tile (no call in the hot loop; 1.00).  17 = the same with the exact path
// called from the hot loop (0.98), 9 = 17 with five compares per element
// (0.975), 10 = 9 at 3 CTA/SM (0.95), 11 = one slot at 4 (0.87), 12 = four
// slots at 2 (0.96), 13 = two slots unbounded (0.80), 14 = one slot at 6
// (0.87), 18 = 17 at 3 CTA/SM (0.95), 19 / 20 = 17 with 2 / 4 tiles per CTA
// (0.93), 16 = access-pattern probe, no Adam (1.01: the ceiling).  Round-1
// kernels (k3_adam_bf16, 4-element slots): 15 = 4 slots at 4 CTA/SM (the
// round-1 production, 0.94 before / 0.89 after the x86-NaN exact path), 1 =
// 4 slots unbounded (0.90), 2 = 2 slots at 4 (0.84), 3 = 8 slots (0.89),
// 4/5 = 8-element slots at 4 / unbounded (0.90 / 0.80), 6 = 2 slots at 5
// (0.86), 7 = 3 slots at 4 (0.91), 8 = 4 slots at 5 (0.88).  Cold routes
// (round 2 final; production = 21 = COLD 3): 24 = the deferred kernel without
// them (100% cold rows 0.57 -> 0.84, 20% 0.88 -> 0.97), 22 = only the
// vectorised M == 0 route of the deferred phase, 23 = only the early
// warp-uniform reject (slower: 0.94 on live state).
int k3_slots(int gk, int variant) {
    if (gk != kBF16) return 2;  // k3_v2<GK, 2, 4>
    switch (variant) {
        case 0: case 2: case 4: case 5: case 6: case 9: case 10: case 13: return 2;
        case 3: return 8;
        case 7: return 3;
        case 11: case 14: return 1;
        case 1: case 8: case 12: case 15: return 4;
        default: return 2;
    }
}

int k3_tiles_per_cta(int gk, int variant) {
    if (gk != kBF16) return 1;
    return variant == 19 ? 2 : variant == 20 ? 4 : 1;
}

int k3_vec(int gk, int variant) {
    if (gk != kBF16) return 8;
    return (variant >= 1 && variant <= 3) || (variant >= 6 && variant <= 8) || variant == 15 ? 4 : 8;
}

template <typename F>
void k3_dispatch(int gk, int variant, F&& f) {
    if (gk == kF32) return f(k3_v2<kF32, 2, 4, false, 1, 1, true, 3>);
    if (gk == kF16) return f(k3_v2<kF16, 2, 4, false, 1, 1, true, 0>);  // COLD 3 spills here
    switch (variant) {
        case 1: return f(k3_adam_bf16<kBF16, 4, 1>);
        case 2: return f(k3_adam_bf16<kBF16, 2, 4>);
        case 3: return f(k3_adam_bf16<kBF16, 8, 1>);
        case 4: return f(k3_adam_bf16_v8<kBF16, 2, 4>);
        case 5: return f(k3_adam_bf16_v8<kBF16, 2, 1>);
        case 6: return f(k3_adam_bf16<kBF16, 2, 5>);
        case 7: return f(k3_adam_bf16<kBF16, 3, 4>);
        case 8: return f(k3_adam_bf16<kBF16, 4, 5>);
        case 10: return f(k3_v2<kBF16, 2, 3>);
        case 11: return f(k3_v2<kBF16, 1, 4>);
        case 12: return f(k3_v2<kBF16, 4, 2>);
        case 13: return f(k3_v2<kBF16, 2, 1>);
        case 14: return f(k3_v2<kBF16, 1, 6>);
        case 15: return f(k3_adam_bf16<kBF16, 4, 4>);
        case 9: return f(k3_v2<kBF16, 2, 4>);
        case 16: return f(k3_v2<kBF16, 2, 4, true>);
        case 18: return f(k3_v2<kBF16, 2, 3, false, 1>);
        case 19: return f(k3_v2<kBF16, 2, 4, false, 1, 2>);
        case 17: return f(k3_v2<kBF16, 2, 4, false, 1>);
        case 20: return f(k3_v2<kBF16, 2, 4, false, 1, 4>);
        case 21: return f(k3_v2<kBF16, 2, 4, false, 1, 1, true, 3>);
        case 22: return f(k3_v2<kBF16, 2, 4, false, 1, 1, true, 2>);
        case 23: return f(k3_v2<kBF16, 2, 4, false, 1, 1, true, 1>);
        case 24: return f(k3_v2<kBF16, 2, 4, false, 1, 1, true, 0>);  // production until the cold routes
        case 25: return f(k3_v2<kBF16, 2, 4, false, 1, 1, true, 5>);  // early reject + vector second chance
        case 27: return f(k3_v2<kBF16, 2, 4, false, 1, 1, true, 9>);  // early reject + split drain
        default: return f(k3_v2<kBF16, 2, 4, false, 1, 1, true, 3>);
    }
}

int k3_blocks_per_sm(int gk, int variant) {
    int x = 0;
    k3_dispatch(gk, variant, [&](auto fn) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&x, fn, kK2Threads, 0);
    });
    return x > 0 ? x : 1;
}

void launch_k3(int gk, int variant, const SegTable& tab, const AdamArgs& a, unsigned grid,
               cudaStream_t st) {
    // the production k3_v2 waits on entry: launched as a programmatic
    // dependent (MA_PDL_K3=0: plain launch, A/B); the older A/B kernels do not
    static const bool pdl = [] {
        const char* e = std::getenv("MA_PDL_K3");
        return !(e && e[0] == '0') && pdl_enabled();
    }();
    const bool production = gk != kBF16 || variant == 0 || variant >= 21;
    k3_dispatch(gk, variant, [&](auto fn) {
        if (pdl && production) {
            launch_pdl(fn, grid, kK2Threads, st, tab, a);
        } else {
            fn<<<grid, kK2Threads, 0, st>>>(tab, a);
        }
    });
}

void launch_step_finish(StepDev* st, StepLog* log, const float2* bc_table, uint64_t bc_first,
                        const AdamConsts& c, cudaStream_t s) {
    if (pdl_finish()) {
        launch_pdl(k_step_finish, 1, 32, s, st, log, bc_table, static_cast<unsigned long long>(bc_first), c);
    } else {
        k_step_finish<<<1, 32, 0, s>>>(st, log, bc_table, bc_first, c);
    }
}

void launch_step_prepare(StepDev* st, const float2* bc_table, uint64_t bc_first,
                         const AdamConsts& c, cudaStream_t s) {
    k_step_prepare<<<1, 32, 0, s>>>(st, bc_table, bc_first, c);
}

void launch_gen_weights(int wk, float* p, uint16_t* w, uint64_t n, uint64_t base, uint64_t seed,
                        unsigned grid, cudaStream_t st) {
    if (wk == kBF16) {
        k_gen_weights<kBF16><<<grid, 256, 0, st>>>(p, w, n, base, seed);
    } else if (wk == kF16) {
        k_gen_weights<kF16><<<grid, 256, 0, st>>>(p, w, n, base, seed);
    } else {
        k_gen_weights<kNone><<<grid, 256, 0, st>>>(p, nullptr, n, base, seed);
    }
}

void launch_gen_grads(int gk, int wk, void* g, const uint16_t* w, uint64_t n, uint64_t base,
                      uint64_t seed, uint64_t step, const float* d_scale, float scale,
                      unsigned grid, cudaStream_t st) {
#define MA_GEN(G, W)                                                                       \
    if (gk == G && wk == W) {                                                              \
        k_gen_grads<G, W><<<grid, 256, 0, st>>>(g, w, n, base, seed, step, d_scale, scale); \
        return;                                                                            \
    }
    MA_GEN(kF32, kBF16) MA_GEN(kF32, kF16) MA_GEN(kBF16, kBF16) MA_GEN(kBF16, kF16)
    MA_GEN(kF16, kBF16) MA_GEN(kF16, kF16)
#undef MA_GEN
}

void launch_plant(void* buf, int dtype, uint64_t index, uint32_t bits, cudaStream_t st) {
    k_plant<<<1, 1, 0, st>>>(buf, dtype, index, bits);
}

void launch_cast_sweep(int kind, int log2, uint64_t* out, uint64_t nblocks) {
    const unsigned grid = static_cast<unsigned>((nblocks + 63) / 64);
    if (kind == kBF16) {
        k_cast_sweep<kBF16><<<grid, 64>>>(log2, out, nblocks);
    } else {
        k_cast_sweep<kF16><<<grid, 64>>>(log2, out, nblocks);
    }
}

void launch_mask_sweep(int kind, unsigned long long* mismatches, unsigned grid) {
    k_mask_sweep<<<grid, 256>>>(kind, mismatches);
}

}  // namespace ma
