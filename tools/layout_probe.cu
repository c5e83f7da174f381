// Layout probe (measurement tool, not part of the library): does the
// optimizer's 5-stream access pattern (p, m, v fp32 read+write, g bf16 read,
// w bf16 write) reach the copy bandwidth, and would a blocked p/m/v layout
// (p, m, v of the same 1024 elements adjacent) do better than separate
// arrays?  No Adam arithmetic: this bounds what layout alone can buy.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o layout_probe tools/layout_probe.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

constexpr int kThreads = 256;
constexpr int kBlock = 1024;  // elements per p/m/v block in the blocked layout

template <bool BLOCKED>
__global__ void __launch_bounds__(kThreads) probe(float* __restrict__ state, float* __restrict__ p,
                                                  float* __restrict__ m, float* __restrict__ v,
                                                  const uint16_t* __restrict__ g, uint16_t* __restrict__ w,
                                                  uint64_t nslots) {
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t j = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; j < nslots;
         j += stride) {
        const uint64_t e = 4 * j;
        float4 *P, *M, *V;
        if (BLOCKED) {
            const uint64_t blk = e / kBlock, off = e % kBlock;
            float* base = state + blk * 3 * kBlock;
            P = reinterpret_cast<float4*>(base + off);
            M = reinterpret_cast<float4*>(base + kBlock + off);
            V = reinterpret_cast<float4*>(base + 2 * kBlock + off);
        } else {
            P = reinterpret_cast<float4*>(p + e);
            M = reinterpret_cast<float4*>(m + e);
            V = reinterpret_cast<float4*>(v + e);
        }
        float4 a = __ldcs(P), b = __ldcs(M), c = __ldcs(V);
        const uint2 gg = __ldcs(reinterpret_cast<const uint2*>(g + e));
        const float d = __uint_as_float(gg.x << 16) * 1e-9f;
        a.x += d; a.y += d; a.z += d; a.w += d;
        b.x += d; b.y += d; b.z += d; b.w += d;
        c.x += d; c.y += d; c.z += d; c.w += d;
        __stcs(P, a);
        __stcs(M, b);
        __stcs(V, c);
        __stcs(reinterpret_cast<uint2*>(w + e),
               make_uint2((__float_as_uint(a.x) >> 16) | (__float_as_uint(a.y) & 0xFFFF0000u),
                          (__float_as_uint(a.z) >> 16) | (__float_as_uint(a.w) & 0xFFFF0000u)));
    }
}

__global__ void copy(const float4* __restrict__ a, float4* __restrict__ b, uint64_t n4) {
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n4; i += stride)
        __stcs(b + i, __ldcs(a + i));
}

// one-shot grid: each CTA owns U * blockDim consecutive vectors, loads all U
// before storing (the shape of torch's vectorized elementwise kernels)
template <int U, bool CS>
__global__ void copy_oneshot(const float4* __restrict__ a, float4* __restrict__ b, uint64_t n4) {
    const uint64_t base = blockIdx.x * static_cast<uint64_t>(blockDim.x) * U + threadIdx.x;
    float4 r[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const uint64_t i = base + u * blockDim.x;
        if (i < n4) r[u] = CS ? __ldcs(a + i) : a[i];
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const uint64_t i = base + u * blockDim.x;
        if (i < n4) {
            if (CS) __stcs(b + i, r[u]); else b[i] = r[u];
        }
    }
}

// 5-stream pattern on a one-shot grid, U slots per thread
template <int U>
__global__ void __launch_bounds__(kThreads) probe_oneshot(float* __restrict__ p, float* __restrict__ m,
                                                          float* __restrict__ v,
                                                          const uint16_t* __restrict__ g,
                                                          uint16_t* __restrict__ w, uint64_t nslots) {
    const uint64_t base = blockIdx.x * static_cast<uint64_t>(blockDim.x) * U + threadIdx.x;
    float4 a[U], b[U], c[U];
    uint2 gg[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const uint64_t j = base + u * blockDim.x;
        if (j < nslots) {
            a[u] = __ldcs(reinterpret_cast<const float4*>(p) + j);
            b[u] = __ldcs(reinterpret_cast<const float4*>(m) + j);
            c[u] = __ldcs(reinterpret_cast<const float4*>(v) + j);
            gg[u] = __ldcs(reinterpret_cast<const uint2*>(g) + j);
        }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const uint64_t j = base + u * blockDim.x;
        if (j < nslots) {
            const float d = __uint_as_float(gg[u].x << 16) * 1e-9f;
            a[u].x += d; b[u].y += d; c[u].z += d;
            __stcs(reinterpret_cast<float4*>(p) + j, a[u]);
            __stcs(reinterpret_cast<float4*>(m) + j, b[u]);
            __stcs(reinterpret_cast<float4*>(v) + j, c[u]);
            __stcs(reinterpret_cast<uint2*>(w) + j,
                   make_uint2(__float_as_uint(a[u].x) >> 16, __float_as_uint(a[u].z) >> 16));
        }
    }
}

// 256-bit global accesses (sm_100: LDG.E.256 / STG.E.256)
struct F8 {
    float x[8];
};
__device__ __forceinline__ F8 ld256(const float* p) {
    F8 r;
    asm volatile("ld.global.cs.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(r.x[0]), "=f"(r.x[1]), "=f"(r.x[2]), "=f"(r.x[3]), "=f"(r.x[4]),
                   "=f"(r.x[5]), "=f"(r.x[6]), "=f"(r.x[7])
                 : "l"(p));
    return r;
}
__device__ __forceinline__ void st256(float* p, const F8& r) {
    asm volatile("st.global.cs.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "f"(r.x[0]),
                 "f"(r.x[1]), "f"(r.x[2]), "f"(r.x[3]), "f"(r.x[4]), "f"(r.x[5]), "f"(r.x[6]),
                 "f"(r.x[7])
                 : "memory");
}

template <int U>
__global__ void copy_oneshot256(const float* __restrict__ a, float* __restrict__ b, uint64_t n8) {
    const uint64_t base = blockIdx.x * static_cast<uint64_t>(blockDim.x) * U + threadIdx.x;
    F8 r[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const uint64_t i = base + u * blockDim.x;
        if (i < n8) r[u] = ld256(a + 8 * i);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const uint64_t i = base + u * blockDim.x;
        if (i < n8) st256(b + 8 * i, r[u]);
    }
}

// the 5-stream pattern with 8-element slots: p/m/v by 32-byte accesses,
// g/w by 16-byte ones
template <int U>
__global__ void __launch_bounds__(kThreads) probe_oneshot256(float* __restrict__ p,
                                                             float* __restrict__ m,
                                                             float* __restrict__ v,
                                                             const uint16_t* __restrict__ g,
                                                             uint16_t* __restrict__ w,
                                                             uint64_t nslots8) {
    const uint64_t base = blockIdx.x * static_cast<uint64_t>(blockDim.x) * U + threadIdx.x;
    F8 a[U], b[U], c[U];
    uint4 gg[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const uint64_t j = base + u * blockDim.x;
        if (j < nslots8) {
            a[u] = ld256(p + 8 * j);
            b[u] = ld256(m + 8 * j);
            c[u] = ld256(v + 8 * j);
            gg[u] = __ldcs(reinterpret_cast<const uint4*>(g) + j);
        }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const uint64_t j = base + u * blockDim.x;
        if (j < nslots8) {
            const float d = __uint_as_float(gg[u].x << 16) * 1e-9f;
            a[u].x[0] += d; b[u].x[1] += d; c[u].x[2] += d;
            st256(p + 8 * j, a[u]);
            st256(m + 8 * j, b[u]);
            st256(v + 8 * j, c[u]);
            __stcs(reinterpret_cast<uint4*>(w) + j,
                   make_uint4(__float_as_uint(a[u].x[0]) >> 16, __float_as_uint(a[u].x[2]) >> 16,
                              __float_as_uint(a[u].x[4]) >> 16, __float_as_uint(a[u].x[6]) >> 16));
        }
    }
}

int main() {
    const uint64_t n = 1ull << 31;  // 2 Gi elements: 56 GiB of traffic per pass
    float *state, *p, *m, *v;
    uint16_t *g, *w;
    cudaMalloc(&state, 3 * n * 4);
    cudaMalloc(&p, n * 4);
    cudaMalloc(&m, n * 4);
    cudaMalloc(&v, n * 4);
    cudaMalloc(&g, n * 2);
    cudaMalloc(&w, n * 2);
    cudaMemset(state, 0, 3 * n * 4);
    cudaMemset(p, 0, n * 4);
    cudaMemset(m, 0, n * 4);
    cudaMemset(v, 0, n * 4);
    cudaMemset(g, 0, n * 2);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto time = [&](auto&& launch, double bytes, const char* name) {
        for (int i = 0; i < 2; ++i) launch();
        cudaEventRecord(a);
        const int reps = 5;
        for (int i = 0; i < reps; ++i) launch();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        printf("%-34s %8.1f GB/s  (%s)\n", name, bytes * reps / (ms / 1e3) / 1e9,
               cudaGetErrorString(cudaGetLastError()));
    };
    const uint64_t nslots = n / 4;
    for (int per_sm : {4, 8}) {
        const unsigned grid = sms * per_sm;
        char nm[64];
        snprintf(nm, sizeof nm, "SoA 5-stream (grid %d/SM)", per_sm);
        time([&] { probe<false><<<grid, kThreads>>>(state, p, m, v, g, w, nslots); }, 28.0 * n, nm);
        snprintf(nm, sizeof nm, "blocked p/m/v (grid %d/SM)", per_sm);
        time([&] { probe<true><<<grid, kThreads>>>(state, p, m, v, g, w, nslots); }, 28.0 * n, nm);
    }
    time([&] { copy<<<sms * 8, kThreads>>>(reinterpret_cast<float4*>(p),
                                            reinterpret_cast<float4*>(m), n / 4); },
         8.0 * n, "plain copy (read+write)");
    const uint64_t n4 = n / 4;
    time([&] { copy_oneshot<4, true><<<(n4 + 1023) / 1024, 256>>>(reinterpret_cast<float4*>(p),
                                                                  reinterpret_cast<float4*>(m), n4); },
         8.0 * n, "one-shot copy U4 .cs");
    time([&] { copy_oneshot<4, false><<<(n4 + 1023) / 1024, 256>>>(reinterpret_cast<float4*>(p),
                                                                   reinterpret_cast<float4*>(m), n4); },
         8.0 * n, "one-shot copy U4 default");
    time([&] { copy_oneshot<8, true><<<(n4 + 2047) / 2048, 256>>>(reinterpret_cast<float4*>(p),
                                                                  reinterpret_cast<float4*>(m), n4); },
         8.0 * n, "one-shot copy U8 .cs");
    time([&] { copy_oneshot<1, true><<<(n4 + 255) / 256, 256>>>(reinterpret_cast<float4*>(p),
                                                                reinterpret_cast<float4*>(m), n4); },
         8.0 * n, "one-shot copy U1 .cs");
    time([&] { probe_oneshot<1><<<(nslots + 255) / 256, kThreads>>>(p, m, v, g, w, nslots); },
         28.0 * n, "one-shot 5-stream U1");
    time([&] { probe_oneshot<2><<<(nslots + 511) / 512, kThreads>>>(p, m, v, g, w, nslots); },
         28.0 * n, "one-shot 5-stream U2");
    time([&] { probe_oneshot<4><<<(nslots + 1023) / 1024, kThreads>>>(p, m, v, g, w, nslots); },
         28.0 * n, "one-shot 5-stream U4");
    const uint64_t n8 = n / 8;
    time([&] { copy_oneshot256<2><<<(n8 + 511) / 512, 256>>>(p, m, n8); }, 8.0 * n,
         "one-shot copy 256-bit U2");
    time([&] { copy_oneshot256<4><<<(n8 + 1023) / 1024, 256>>>(p, m, n8); }, 8.0 * n,
         "one-shot copy 256-bit U4");
    time([&] { probe_oneshot256<1><<<(n8 + 255) / 256, kThreads>>>(p, m, v, g, w, n8); },
         28.0 * n, "one-shot 5-stream 256-bit U1");
    time([&] { probe_oneshot256<2><<<(n8 + 511) / 512, kThreads>>>(p, m, v, g, w, n8); },
         28.0 * n, "one-shot 5-stream 256-bit U2");
    time([&] { probe_oneshot256<4><<<(n8 + 1023) / 1024, kThreads>>>(p, m, v, g, w, n8); },
         28.0 * n, "one-shot 5-stream 256-bit U4");
    return 0;
}
