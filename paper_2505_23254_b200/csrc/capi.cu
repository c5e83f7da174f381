// Host side of the C ABI declared in include/memascend_b200.h.
//
// Launch planning, memory classification (device / registered host /
// pageable host), the staging path for pageable spans, and the device-
// resident step driver.  Every entry point converts failures to a status
// code plus a thread-local message; nothing here falls back to the CPU.
#include <cuda.h>
#include <cuda_runtime.h>
#include <sys/syscall.h>
#include <unistd.h>

#include <algorithm>
#include <cctype>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstddef>
#include <cstring>
#include <fstream>
#include <mutex>
#include <condition_variable>
#include <deque>
#include <functional>
#include <string>
#include <thread>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "kernels.cuh"
#include "memascend_b200.h"
#include "swap.hpp"

namespace {

thread_local std::string g_err;

// NVTX range per entry point (header-only NVTX v3: free unless a tool such as
// nsys / ncu --nvtx attaches), SURVEY.md §5 "tracing".
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};

struct Status {
    int code;
};

[[noreturn]] void fail(int code, const std::string& msg) {
    g_err = msg;
    throw Status{code};
}

void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) {
        cudaGetLastError();
        fail(e == cudaErrorMemoryAllocation ? MA_ERR_OUT_OF_MEMORY : MA_ERR_CUDA,
             std::string(what) + ": " + cudaGetErrorString(e));
    }
}

#define CK(call) cuda_check((call), #call)

template <typename F>
int guarded(F&& fn) {
    try {
        fn();
        return MA_OK;
    } catch (const Status& s) {
        return s.code;
    } catch (const ma::swp::Failure& f) {
        g_err = f.msg;
        return f.code;
    } catch (const std::exception& e) {
        g_err = e.what();
        return MA_ERR_DEVICE_ERROR;
    }
}

struct DeviceInfo {
    int device = -1;
    int sms = 0;
    int major = 0;
    int minor = 0;
};

DeviceInfo device_info() {
    int count = 0;
    const cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count == 0) {
        cudaGetLastError();
        fail(MA_ERR_NO_DEVICE,
             "no CUDA device visible: the memascend B200 path has no CPU fallback");
    }
    DeviceInfo d;
    CK(cudaGetDevice(&d.device));
    static std::mutex mu;
    static std::vector<DeviceInfo> cache(64);
    std::lock_guard<std::mutex> lock(mu);
    DeviceInfo& c = cache[static_cast<size_t>(d.device) % cache.size()];
    if (c.device != d.device) {
        CK(cudaDeviceGetAttribute(&d.sms, cudaDevAttrMultiProcessorCount, d.device));
        CK(cudaDeviceGetAttribute(&d.major, cudaDevAttrComputeCapabilityMajor, d.device));
        CK(cudaDeviceGetAttribute(&d.minor, cudaDevAttrComputeCapabilityMinor, d.device));
        if (d.major != 10) {
            fail(MA_ERR_CAPABILITY, "device " + std::to_string(d.device) + " is sm_" +
                                        std::to_string(d.major * 10 + d.minor) +
                                        "; this build targets sm_100a (B200) only");
        }
        c = d;
    }
    return c;
}

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

int elem_bytes(int dt) { return dt == MA_DT_F32 ? 4 : 2; }

void check_grad_dtype(int dt) {
    if (dt != MA_DT_F32 && dt != MA_DT_BF16 && dt != MA_DT_F16)
        fail(MA_ERR_INVALID_ARGUMENT, "gradient dtype must be F32, BF16 or F16");
}

void check_w_dtype(int dt) {
    if (dt != MA_DT_NONE && dt != MA_DT_BF16 && dt != MA_DT_F16)
        fail(MA_ERR_INVALID_ARGUMENT, "working-weight dtype must be BF16, F16 or NONE");
}

// 0 pageable host, 1 device/managed, 2 registered host; *dev gets the
// device-accessible alias.
int classify(const void* p, const void** dev) {
    *dev = p;
    if (p == nullptr) return 1;
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    switch (at.type) {
        case cudaMemoryTypeDevice:
        case cudaMemoryTypeManaged:
            return 1;
        case cudaMemoryTypeHost:
            *dev = at.devicePointer ? at.devicePointer : p;
            return 2;
        default:
            return 0;
    }
}

// ------------------------------------------------------------ scratch
// Grow-only device scratch + a library stream for the synchronous entry
// points (pageable staging, result flags).
struct Scratch {
    std::mutex mu;
    void* dev = nullptr;
    size_t bytes = 0;
    cudaStream_t stream = nullptr;
    int device = -1;

    void* get(size_t need) {
        if (need > bytes) {
            if (dev) CK(cudaFree(dev));
            dev = nullptr;
            bytes = 0;
            CK(cudaMalloc(&dev, need));
            bytes = need;
        }
        return dev;
    }
    cudaStream_t strm() {
        if (!stream) CK(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
        return stream;
    }
};

Scratch& scratch() {
    static Scratch s[16];
    int d = 0;
    cudaGetDevice(&d);
    return s[d % 16];
}

// ------------------------------------------------------------ NUMA
// Host memory the GPU streams from (gradients, the state pool, staging
// slots) belongs on the NUMA node of the GPU's PCIe root: on a two-socket
// 8 x B200 box the other socket's memory reaches the GPU through the
// inter-socket link at a fraction of the PCIe rate.  The node comes from
// sysfs; pages are preferred there (and already-touched ones moved) with
// mbind before cudaHostRegister pins them.  Best effort: one-node hosts,
// containers without mbind, and MA_NUMA_BIND=0 leave the placement alone.
int current_device_numa_node() {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return -1;
    char bus[32] = {0};
    if (cudaDeviceGetPCIBusId(bus, sizeof bus, dev) != cudaSuccess) return -1;
    std::string id(bus);
    for (char& ch : id) ch = static_cast<char>(std::tolower(static_cast<unsigned char>(ch)));
    std::ifstream f("/sys/bus/pci/devices/" + id + "/numa_node");
    int node = -1;
    if (!(f >> node)) return -1;
    return node;
}

int host_numa_nodes() {
    std::ifstream f("/sys/devices/system/node/possible");  // e.g. "0-1"
    std::string s;
    if (!(f >> s)) return 1;
    const auto dash = s.find('-');
    return dash == std::string::npos ? 1 : std::atoi(s.c_str() + dash + 1) + 1;
}

void numa_place_for_device(void* ptr, uint64_t bytes) {
    if (const char* e = std::getenv("MA_NUMA_BIND"); e && e[0] == '0') return;
    static const int nodes = host_numa_nodes();
    if (nodes < 2) return;
    const int node = current_device_numa_node();
    if (node < 0 || node >= 1024) return;
    const uintptr_t page = 4096;
    const uintptr_t lo = reinterpret_cast<uintptr_t>(ptr) & ~(page - 1);
    const uintptr_t hi = (reinterpret_cast<uintptr_t>(ptr) + bytes + page - 1) & ~(page - 1);
    unsigned long mask[16] = {0};
    mask[node / 64] |= 1ul << (node % 64);
    // MPOL_PREFERRED (1), MPOL_MF_MOVE (2): errors are ignored (best effort)
    ::syscall(SYS_mbind, lo, hi - lo, 1ul, mask, 1024ul, 2ul);
}

// ------------------------------------------------------------ K1 launch
// keep_tail: a stepper check whose gradients K2 reads next — with
// MA_K1_KEEP_MB > 0 (A/B; default 0 = off) the buffer's last
// MA_K1_KEEP_MB are loaded under an L2 evict_last policy so K2's last tiles
// find them in L2 (kernels.cu k1_load).
// kept_lo / kept_lines (keep_tail only): the 128-byte lines now under
// evict_last, for the update to demote (ma::AdamArgs::demote).
void launch_k1(const void* data, uint64_t n, int dt, uint32_t* flag, uint64_t* first,
               uint64_t index_base, bool early_exit, cudaStream_t st,
               const ma::XchgDev* xchg = nullptr, bool keep_tail = false,
               const char** kept_lo = nullptr, uint64_t* kept_lines = nullptr) {
    if (n == 0 && !xchg) return;  // an empty rank still takes part in the exchange
    const DeviceInfo d = device_info();
    const uint32_t es = static_cast<uint32_t>(elem_bytes(dt));
    const uintptr_t addr = reinterpret_cast<uintptr_t>(data);
    if (addr % es) fail(MA_ERR_ALIGNMENT, "gradient buffer is not element-aligned");
    ma::K1Args a{};
    a.xchg = xchg;
    a.raw = data;
    a.n = n;
    a.head = std::min<uint64_t>(((16 - (addr & 15)) & 15) / es, n);
    a.nvec = (n - a.head) * es / 16;
    a.body = reinterpret_cast<const uint4*>(addr + a.head * es);
    a.index_base = index_base;
    a.flag = flag;
    a.first = first;
    a.kind = dt;
    a.elem_bytes = es;
    a.early_exit = early_exit ? 1 : 0;
    static const uint64_t keep_vecs = [] {
        const char* e = std::getenv("MA_K1_KEEP_MB");  // A/B only
        return (e ? std::strtoull(e, nullptr, 10) : 0ull) << 16;  // MiB / 16 B (default off)
    }();
    a.keep_from = keep_tail ? a.nvec - std::min<uint64_t>(a.nvec, keep_vecs) : a.nvec;
    if (kept_lo && kept_lines) {
        if (a.keep_from < a.nvec) {
            const uintptr_t lo = reinterpret_cast<uintptr_t>(a.body + a.keep_from) & ~uintptr_t(127);
            const uintptr_t hi = (reinterpret_cast<uintptr_t>(a.body + a.nvec) + 127) & ~uintptr_t(127);
            *kept_lo = reinterpret_cast<const char*>(lo);
            *kept_lines = (hi - lo) / 128;
        } else {
            *kept_lo = nullptr;
            *kept_lines = 0;
        }
    }
    // MA_K1_UNROLL / MA_K1_CTAS_PER_SM: A/B knobs (defaults 4 and 8)
    static const int unroll = [] {
        const char* e = std::getenv("MA_K1_UNROLL");
        return e ? (std::atoi(e) == 4 ? 4 : 8) : ma::kK1Unroll;
    }();
    static const int ctas = [] {
        const char* e = std::getenv("MA_K1_CTAS_PER_SM");
        const int v = e ? std::atoi(e) : 8;
        return v > 0 && v <= 32 ? v : 8;
    }();
    // MA_K1_GRIDSTRIDE=1 selects the persistent grid-stride form (A/B only)
    static const bool gridstride = [] {
        const char* e = std::getenv("MA_K1_GRIDSTRIDE");
        return e && std::atoi(e) == 1;
    }();
    const uint64_t per_cta =
        static_cast<uint64_t>(ma::kK1Threads) * (gridstride ? unroll : ma::kK1Unroll);
    const uint64_t want = std::max<uint64_t>(1, (a.nvec + per_cta - 1) / per_cta);
    if (!gridstride && want > 0x7FFFFFFFull) fail(MA_ERR_INVALID_ARGUMENT, "gradient buffer too large");
    const uint64_t grid =
        gridstride ? std::min<uint64_t>(want, static_cast<uint64_t>(d.sms) * ctas) : want;
    ma::launch_k1(a, first != nullptr, unroll, !gridstride, static_cast<unsigned>(grid), st);
    CK(cudaGetLastError());
}

// ------------------------------------------------------------ K2 planning
// MA_K2_VARIANT selects an alternative K2 schedule (A/B measurements only;
// see kernels.cuh).  Unset = the production variant.
int k2_variant() {
    static const int v = [] {
        const char* e = std::getenv("MA_K2_VARIANT");
        return e ? std::atoi(e) : ma::kK2DefaultVariant;
    }();
    return v;
}

bool aligned(const void* p, uint64_t h, uint32_t es, uint32_t need) {
    return p == nullptr || ((reinterpret_cast<uintptr_t>(p) + h * es) % need) == 0;
}

// Co-aligns the five streams of one sub-group: `head` scalar elements, then
// nvec vectors of `vec` elements whose p/m/v start on 16 B and whose 16-bit
// (or fp32) grads and working weights start on their vector width.
ma::Seg plan_seg(const ma_subgroup& g, int gdt, int wdt, int vec, int tile_vectors, bool stream,
                 uint64_t tile_begin, uint32_t state_es = 4) {
    ma::Seg s{};
    s.p = g.p;
    s.m = g.m;
    s.v = g.v;
    s.g = g.g;
    s.w = wdt == MA_DT_NONE ? nullptr : g.w;
    s.n = g.n;
    const uint32_t ges = static_cast<uint32_t>(elem_bytes(gdt));
    const uint32_t gneed = ges * static_cast<uint32_t>(vec) >= 16 ? 16u : ges * vec;
    const uint32_t wneed = 2u * static_cast<uint32_t>(vec) >= 16 ? 16u : 2u * vec;
    const uint32_t sneed = state_es * static_cast<uint32_t>(vec) >= 16 ? 16u : state_es * vec;
    s.vector_ok = 0;
    for (uint64_t h = 0; h < static_cast<uint64_t>(vec) && h <= g.n; ++h) {
        if (aligned(g.p, h, state_es, sneed) && aligned(g.m, h, state_es, sneed) &&
            aligned(g.v, h, state_es, sneed) && aligned(g.g, h, ges, gneed) &&
            aligned(s.w, h, 2, wneed)) {
            s.vector_ok = 1;
            s.head = h;
            break;
        }
    }
    uint64_t tiles;
    if (s.vector_ok) {
        s.nvec = (g.n - s.head) / vec;
        tiles = (s.nvec + tile_vectors - 1) / tile_vectors;
        if (!stream) tiles = std::max<uint64_t>(1, tiles);  // tile 0 carries head/tail
    } else {
        s.nvec = 0;
        // stream variants run unaligned sub-groups in their grid-wide scalar pass
        tiles = stream ? 0 : (g.n + static_cast<uint64_t>(tile_vectors) * vec - 1) /
                                 (static_cast<uint64_t>(tile_vectors) * vec);
    }
    s.tile_begin = tile_begin;
    s.tile_end = tile_begin + tiles;
    return s;
}

// One CTA per tile, then trailing CTAs for heads/tails and unaligned
// sub-groups (at least one whenever any remainder exists).
uint64_t oneshot_grid(const ma::SegTable& tab, int vec, uint64_t scalar_elems, uint64_t cap) {
    bool remainder = scalar_elems > 0;
    for (uint32_t k = 0; k < tab.count && !remainder; ++k) {
        const ma::Seg& sg = tab.seg[k];
        remainder = sg.head > 0 || sg.head + sg.nvec * vec != sg.n;
    }
    const uint64_t trailing =
        remainder ? std::max<uint64_t>(1, std::min<uint64_t>(cap, (scalar_elems + 255) / 256)) : 0;
    const uint64_t grid = std::max<uint64_t>(1, tab.total_tiles + trailing);
    if (grid > 0x7FFFFFFFull) fail(MA_ERR_INVALID_ARGUMENT, "sub-group table too large for one launch");
    return grid;
}

void launch_k2(const ma_subgroup* groups, uint32_t count, int gdt, int wdt, const ma::AdamArgs& a,
               cudaStream_t st, bool allgather = false) {
    const DeviceInfo d = device_info();
    // the fused all-gather runs in the production one-shot tile shape (U = 4)
    const int variant = allgather ? ma::kK2DefaultVariant
                                  : ma::k2_effective_variant(gdt, wdt, k2_variant());
    int vec, tile_vectors;
    bool stream;
    ma::k2_variant_shape(variant, &vec, &tile_vectors, &stream);
    const uint64_t cap = static_cast<uint64_t>(d.sms) * ma::k2_blocks_per_sm(gdt, wdt, variant);
    for (uint32_t first = 0; first < count; first += ma::kMaxSegs) {
        ma::SegTable tab{};
        uint64_t tiles = 0;
        uint64_t scalar_elems = 0;
        const uint32_t last = std::min<uint32_t>(count, first + ma::kMaxSegs);
        for (uint32_t k = first; k < last; ++k) {
            if (groups[k].n == 0) continue;
            if (!groups[k].p || !groups[k].m || !groups[k].v || !groups[k].g)
                fail(MA_ERR_INVALID_ARGUMENT, "sub-group with a null state/grad pointer");
            if (wdt != MA_DT_NONE && !groups[k].w)
                fail(MA_ERR_INVALID_ARGUMENT, "sub-group without a working-weight buffer");
            ma::Seg& sg = tab.seg[tab.count];
            sg = plan_seg(groups[k], gdt, wdt, vec, tile_vectors, stream, tiles);
            tiles = sg.tile_end;
            scalar_elems += sg.vector_ok ? 0 : sg.n;
            tab.count += 1;
        }
        if (tab.count == 0) continue;
        tab.total_tiles = tiles;
        uint64_t grid;
        if (ma::k2_variant_oneshot(variant)) {
            grid = oneshot_grid(tab, vec, scalar_elems, cap);
        } else {
            grid = std::min<uint64_t>(tiles, cap);
            if (stream && scalar_elems > 0) {
                grid = std::max<uint64_t>(grid, std::min<uint64_t>(cap, (scalar_elems + 255) / 256));
            }
            grid = std::max<uint64_t>(grid, 1);
        }
        if (allgather)
            ma::launch_k2_allgather(gdt, wdt, tab, a, static_cast<unsigned>(grid), st);
        else
            ma::launch_k2(gdt, wdt, variant, tab, a, static_cast<unsigned>(grid), st);
        CK(cudaGetLastError());
    }
}

// K3: pure-bf16 state; groups' p/m/v point at uint16 (bf16) arrays.
void launch_k3(const ma_subgroup* groups, uint32_t count, int gdt, const ma::AdamArgs& a,
               cudaStream_t st) {
    const DeviceInfo d = device_info();
    static const int variant = [] {
        const char* e = std::getenv("MA_K3_VARIANT");  // A/B only
        return e ? std::atoi(e) : 0;
    }();
    const int kVec = ma::k3_vec(gdt, variant);
    const int kTile = ma::k3_slots(gdt, variant) * ma::kK2Threads;
    const uint64_t cap = static_cast<uint64_t>(d.sms) * ma::k3_blocks_per_sm(gdt, variant);
    for (uint32_t first = 0; first < count; first += ma::kMaxSegs) {
        ma::SegTable tab{};
        uint64_t tiles = 0, scalar_elems = 0;
        const uint32_t last = std::min<uint32_t>(count, first + ma::kMaxSegs);
        for (uint32_t k = first; k < last; ++k) {
            if (groups[k].n == 0) continue;
            if (!groups[k].p || !groups[k].m || !groups[k].v || !groups[k].g)
                fail(MA_ERR_INVALID_ARGUMENT, "sub-group with a null state/grad pointer");
            ma::Seg& sg = tab.seg[tab.count];
            sg = plan_seg(groups[k], gdt, MA_DT_NONE, kVec, kTile, true, tiles, 2);
            tiles = sg.tile_end;
            scalar_elems += sg.vector_ok ? 0 : sg.n;
            tab.count += 1;
        }
        if (tab.count == 0) continue;
        tab.total_tiles = tiles;
        // one CTA per TPC tiles (kernels.cu k3_v2), then the trailing CTAs
        const uint64_t tpc = static_cast<uint64_t>(ma::k3_tiles_per_cta(gdt, variant));
        const uint64_t grid = oneshot_grid(tab, kVec, scalar_elems, cap) - tab.total_tiles +
                              (tab.total_tiles + tpc - 1) / tpc;
        ma::launch_k3(gdt, variant, tab, a, static_cast<unsigned>(std::max<uint64_t>(grid, 1)), st);
        CK(cudaGetLastError());
    }
}

// optimizer.cpp:20-24 on the host: glibc powf, float exponent.
void bias_corrections(uint64_t t, float b1, float b2, float* bc1, float* bc2) {
    const float tf = static_cast<float>(t);
    *bc1 = 1.0f - std::pow(b1, tf);
    *bc2 = 1.0f - std::pow(b2, tf);
}

ma::AdamConsts make_consts(const ma_adam_hyper* h) {
    if (!h) fail(MA_ERR_INVALID_ARGUMENT, "null hyper-parameters");
    ma::AdamConsts c{};
    c.lr = h->lr;
    c.beta1 = h->beta1;
    c.beta2 = h->beta2;
    c.eps = h->eps;
    // (1.0f - beta) and lr * wd as the reference evaluates them (fp32)
    volatile float one = 1.0f;
    c.one_minus_b1 = one - h->beta1;
    c.one_minus_b2 = one - h->beta2;
    volatile float lr = h->lr;
    c.lr_wd = lr * h->weight_decay;
    return c;
}

ma::AdamArgs explicit_args(const ma_adam_hyper* h, uint64_t t, float scale, const uint32_t* skip) {
    if (t == 0) fail(MA_ERR_INVALID_ARGUMENT, "adam step count t must be >= 1");
    ma::AdamArgs a{};
    a.c = make_consts(h);
    a.scale = scale;
    bias_corrections(t, h->beta1, h->beta2, &a.bc1, &a.bc2);
    a.skip = skip;
    return a;
}

}  // namespace

// ====================================================================== C ABI
struct ma_stepper {
    ma::AdamConsts c{};
    ma_adam_hyper h{};
    int g_dtype = MA_DT_BF16;
    int w_dtype = MA_DT_BF16;
    ma::StepDev* d_st = nullptr;
    ma::StepLog* d_log = nullptr;
    float2* d_bc = nullptr;  // bias corrections of t = bc_first .. bc_first + bc_cap - 1
    uint64_t bc_cap = 0;
    uint64_t bc_first = 1;
    uint64_t issued = 0;  // finish calls enqueued since creation / the last set_state
    uint64_t t_base = 0;  // updates at creation / the last set_state (resumed runs)
    cudaStream_t last = nullptr;
    int device = 0;
    bool owns_state = true;
    bool capturing = false;        // between ma_stepper_graph_begin / _end
    const char* kept_lo = nullptr; // gradient lines the last check kept in L2,
    uint64_t kept_lines = 0;       // demoted by the next update (stepper_args)
    // speculative updates of the pending host-gradient check
    // (ma_stepper_check_host_spec_async -> ma_stepper_apply_spec_async)
    uint32_t* d_spec = nullptr;             // [marker, CTA counter]
    std::vector<ma_subgroup> spec_groups;   // the speculated sub-groups, in order
    ma::SpecRestore spec_restore{};
    uint64_t capture_issued = 0;
    std::vector<float2*> retired;  // superseded bias tables (graphs may hold them)
    std::vector<cudaEvent_t> events;

    cudaEvent_t event(uint64_t i) {
        while (events.size() <= i) {
            cudaEvent_t e;
            CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            events.push_back(e);
        }
        return events[i];
    }
    ~ma_stepper() {
        for (cudaEvent_t e : events) cudaEventDestroy(e);
    }
};

namespace {

// AdamArgs of a stepper update
ma::AdamArgs stepper_args(ma_stepper* s) {
    ma::AdamArgs a{};
    a.c = s->c;
    a.skip = &s->d_st->flag;
    a.st = s->d_st;
    // the first update after a check demotes the lines that check kept
    a.demote = s->kept_lo;
    a.demote_lines = s->kept_lines;
    s->kept_lines = 0;
    return a;
}

// The bias-correction table is a window of t values: finish / prepare read
// the entry of t = updates + 1, and the host only bounds `updates` (it is
// t_base + the number of applied steps, and skips are decided on the
// device): t_base <= updates <= t_base + issued.  The window must cover
// [t_base + 1, last_t]; when it does not, the actual updates is read back
// (one synchronisation, every ~65536 steps) and a fresh window starts
// there, so the table's size never depends on how far training has gone
// (a run resumed at t = 10^9 holds the same 0.5 MB as a fresh one).
void stepper_cover_bc(ma_stepper* s, uint64_t last_t) {
    if (s->d_bc && s->bc_first <= s->t_base + 1 && last_t < s->bc_first + s->bc_cap) return;
    if (s->capturing)
        fail(MA_ERR_LIFECYCLE, "bias-correction window exhausted during graph capture");
    CK(cudaDeviceSynchronize());  // `updates` below is final
    unsigned long long updates = 0;
    CK(cudaMemcpy(&updates, &s->d_st->updates, sizeof updates, cudaMemcpyDeviceToHost));
    // exact now: issued keeps counting the finishes after t_base
    const uint64_t applied = updates - std::min<uint64_t>(updates, s->t_base);
    s->issued -= std::min<uint64_t>(s->issued, applied);
    last_t = std::max<uint64_t>(last_t, updates + 2);
    s->t_base = updates;
    const uint64_t first = updates + 1;
    const uint64_t cap = (last_t - first + 1) + 65536;
    std::vector<float2> host(cap);
    for (uint64_t k = 0; k < cap; ++k)
        bias_corrections(first + k, s->h.beta1, s->h.beta2, &host[k].x, &host[k].y);
    float2* fresh = nullptr;
    CK(cudaMalloc(&fresh, cap * sizeof(float2)));
    CK(cudaMemcpy(fresh, host.data(), cap * sizeof(float2), cudaMemcpyHostToDevice));
    // captured graphs may still read the old window: retired, not freed,
    // until the stepper is destroyed
    if (s->d_bc) s->retired.push_back(s->d_bc);
    s->d_bc = fresh;
    s->bc_first = first;
    s->bc_cap = cap;
}

}  // namespace

namespace ma {
void set_error(const std::string& msg) { g_err = msg; }
}  // namespace ma

extern "C" {

const char* ma_last_error(void) { return g_err.c_str(); }

int ma_abi_version(void) { return MA_ABI_VERSION; }

int ma_device_info(int* device, int* sm_count, int* cc_major, int* cc_minor) {
    return guarded([&] {
        const DeviceInfo d = device_info();
        if (device) *device = d.device;
        if (sm_count) *sm_count = d.sms;
        if (cc_major) *cc_major = d.major;
        if (cc_minor) *cc_minor = d.minor;
    });
}

int ma_overflow_check_async(const void* grads, uint64_t n, int g_dtype, uint32_t* d_flag,
                            uint64_t* d_first_index, void* stream) {
    NvtxRange nvtx_range("ma_overflow_check_async");
    return guarded([&] {
        check_grad_dtype(g_dtype);
        if (!d_flag) fail(MA_ERR_INVALID_ARGUMENT, "null flag pointer");
        if (n && !grads) fail(MA_ERR_INVALID_ARGUMENT, "null gradient pointer");
        launch_k1(grads, n, g_dtype, d_flag, d_first_index, 0, d_first_index == nullptr,
                  as_stream(stream));
    });
}

int ma_overflow_check(const void* grads, uint64_t n, int g_dtype, int track_first_index,
                      int* overflow, uint64_t* first_index) {
    NvtxRange nvtx_range("ma_overflow_check");
    return guarded([&] {
        check_grad_dtype(g_dtype);
        if (!overflow) fail(MA_ERR_INVALID_ARGUMENT, "null result pointer");
        *overflow = 0;
        if (first_index) *first_index = UINT64_MAX;
        if (n == 0) return;  // overflow.cpp:77-79
        if (!grads) fail(MA_ERR_INVALID_ARGUMENT, "null gradient pointer");
        device_info();
        Scratch& sc = scratch();
        CK(cudaDeviceSynchronize());  // synchronous API: operands see all prior device work
        std::lock_guard<std::mutex> lock(sc.mu);
        const uint64_t es = elem_bytes(g_dtype);
        const void* dev = nullptr;
        const int kind = classify(grads, &dev);
        const uint64_t chunk = kind == 0 ? (64ull << 20) / es : n;  // 64 MiB staging chunks
        const size_t need = 256 + (kind == 0 ? chunk * es : 0);
        uint8_t* base = static_cast<uint8_t*>(sc.get(need));
        uint32_t* d_flag = reinterpret_cast<uint32_t*>(base);
        uint64_t* d_first = reinterpret_cast<uint64_t*>(base + 64);
        cudaStream_t st = sc.strm();
        CK(cudaMemsetAsync(d_flag, 0, 4, st));
        CK(cudaMemsetAsync(d_first, 0xFF, 8, st));
        for (uint64_t off = 0; off < n; off += chunk) {
            const uint64_t len = std::min(chunk, n - off);
            const void* src;
            if (kind == 0) {
                CK(cudaMemcpyAsync(base + 256, static_cast<const uint8_t*>(grads) + off * es,
                                   len * es, cudaMemcpyHostToDevice, st));
                src = base + 256;
            } else {
                src = static_cast<const uint8_t*>(dev) + off * es;
            }
            launch_k1(src, len, g_dtype, d_flag, track_first_index ? d_first : nullptr, off,
                      !track_first_index, st);
        }
        uint32_t flag = 0;
        uint64_t first = UINT64_MAX;
        CK(cudaMemcpyAsync(&flag, d_flag, 4, cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(&first, d_first, 8, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        *overflow = flag ? 1 : 0;
        if (first_index && track_first_index && flag) *first_index = first;
    });
}

int ma_adam_step_async(float* p, float* m, float* v, const void* g, int g_dtype, uint64_t n,
                       uint64_t t, const ma_adam_hyper* h, float loss_scale, void* w_out,
                       int w_dtype, const uint32_t* d_skip_flag, void* stream) {
    NvtxRange nvtx_range("ma_adam_step_async");
    return guarded([&] {
        check_grad_dtype(g_dtype);
        check_w_dtype(w_dtype);
        const ma::AdamArgs a = explicit_args(h, t, loss_scale, d_skip_flag);
        ma_subgroup grp{p, m, v, g, w_out, n};
        launch_k2(&grp, 1, g_dtype, w_dtype, a, as_stream(stream));
    });
}

int ma_adam_step(float* p, float* m, float* v, const void* g, int g_dtype, uint64_t n,
                 uint64_t t, const ma_adam_hyper* h, float loss_scale, void* w_out, int w_dtype) {
    NvtxRange nvtx_range("ma_adam_step");
    return guarded([&] {
        check_grad_dtype(g_dtype);
        check_w_dtype(w_dtype);
        const ma::AdamArgs a = explicit_args(h, t, loss_scale, nullptr);
        if (n == 0) return;
        device_info();
        Scratch& sc = scratch();
        CK(cudaDeviceSynchronize());  // synchronous API: operands see all prior device work
        std::lock_guard<std::mutex> lock(sc.mu);
        cudaStream_t st = sc.strm();
        const uint64_t ges = elem_bytes(g_dtype);
        void* ptrs[5] = {p, m, v, const_cast<void*>(g), w_dtype == MA_DT_NONE ? nullptr : w_out};
        const uint64_t esz[5] = {4, 4, 4, ges, 2};
        const void* dev[5];
        int kinds[5];
        bool any_pageable = false;
        for (int k = 0; k < 5; ++k) {
            kinds[k] = classify(ptrs[k], &dev[k]);
            any_pageable |= kinds[k] == 0;
        }
        if (!any_pageable) {
            ma_subgroup grp{const_cast<float*>(static_cast<const float*>(dev[0])),
                            const_cast<float*>(static_cast<const float*>(dev[1])),
                            const_cast<float*>(static_cast<const float*>(dev[2])), dev[3],
                            const_cast<void*>(dev[4]), n};
            launch_k2(&grp, 1, g_dtype, w_dtype, a, st);
            CK(cudaStreamSynchronize(st));
            return;
        }
        // stage pageable spans through device scratch in 16 Mi-element chunks
        const uint64_t chunk = std::min<uint64_t>(n, 16ull << 20);
        uint64_t offs[5], total = 0;
        for (int k = 0; k < 5; ++k) {
            offs[k] = total;
            if (kinds[k] == 0 && ptrs[k]) total += (chunk * esz[k] + 255) / 256 * 256;
        }
        uint8_t* base = static_cast<uint8_t*>(sc.get(std::max<uint64_t>(total, 256)));
        for (uint64_t off = 0; off < n; off += chunk) {
            const uint64_t len = std::min(chunk, n - off);
            void* cur[5];
            for (int k = 0; k < 5; ++k) {
                if (!ptrs[k]) {
                    cur[k] = nullptr;
                } else if (kinds[k] == 0) {
                    cur[k] = base + offs[k];
                    if (k < 4) {  // inputs: p, m, v, g
                        CK(cudaMemcpyAsync(cur[k], static_cast<uint8_t*>(ptrs[k]) + off * esz[k],
                                           len * esz[k], cudaMemcpyHostToDevice, st));
                    }
                } else {
                    cur[k] = const_cast<uint8_t*>(static_cast<const uint8_t*>(dev[k])) + off * esz[k];
                }
            }
            ma_subgroup grp{static_cast<float*>(cur[0]), static_cast<float*>(cur[1]),
                            static_cast<float*>(cur[2]), cur[3], cur[4], len};
            launch_k2(&grp, 1, g_dtype, w_dtype, a, st);
            for (int k : {0, 1, 2, 4}) {  // outputs: p, m, v, w
                if (ptrs[k] && kinds[k] == 0) {
                    CK(cudaMemcpyAsync(static_cast<uint8_t*>(ptrs[k]) + off * esz[k], cur[k],
                                       len * esz[k], cudaMemcpyDeviceToHost, st));
                }
            }
            CK(cudaStreamSynchronize(st));
        }
    });
}

int ma_adam_step_bf16(uint16_t* p, uint16_t* m, uint16_t* v, const float* g, uint64_t n,
                      uint64_t t, const ma_adam_hyper* h, float loss_scale) {
    NvtxRange nvtx_range("ma_adam_step_bf16");
    return guarded([&] {
        const ma::AdamArgs a = explicit_args(h, t, loss_scale, nullptr);
        if (n == 0) return;
        const DeviceInfo d = device_info();
        Scratch& sc = scratch();
        CK(cudaDeviceSynchronize());  // synchronous API: operands see all prior device work
        std::lock_guard<std::mutex> lock(sc.mu);
        cudaStream_t st = sc.strm();
        const void* dp;
        const void* dm;
        const void* dv;
        const void* dg;
        const int kp = classify(p, &dp), km = classify(m, &dm), kv = classify(v, &dv),
                  kg = classify(g, &dg);
        // K3 is the "next" row: stage everything that is not device-accessible
        const uint64_t r16 = (2 * n + 255) / 256 * 256;  // 256-B aligned staging regions
        const uint64_t bytes = 3 * r16 + 4 * n;
        uint8_t* base = static_cast<uint8_t*>(sc.get(bytes));
        uint16_t* sp = kp ? const_cast<uint16_t*>(static_cast<const uint16_t*>(dp))
                          : reinterpret_cast<uint16_t*>(base);
        uint16_t* sm = km ? const_cast<uint16_t*>(static_cast<const uint16_t*>(dm))
                          : reinterpret_cast<uint16_t*>(base + r16);
        uint16_t* sv = kv ? const_cast<uint16_t*>(static_cast<const uint16_t*>(dv))
                          : reinterpret_cast<uint16_t*>(base + 2 * r16);
        const float* sg = kg ? static_cast<const float*>(dg) : reinterpret_cast<float*>(base + 3 * r16);
        if (!kp) CK(cudaMemcpyAsync(sp, p, 2 * n, cudaMemcpyHostToDevice, st));
        if (!km) CK(cudaMemcpyAsync(sm, m, 2 * n, cudaMemcpyHostToDevice, st));
        if (!kv) CK(cudaMemcpyAsync(sv, v, 2 * n, cudaMemcpyHostToDevice, st));
        if (!kg) CK(cudaMemcpyAsync(const_cast<float*>(sg), g, 4 * n, cudaMemcpyHostToDevice, st));
        (void)d;
        ma_subgroup grp{reinterpret_cast<float*>(sp), reinterpret_cast<float*>(sm),
                        reinterpret_cast<float*>(sv), sg, nullptr, n};
        launch_k3(&grp, 1, MA_DT_F32, a, st);
        if (!kp) CK(cudaMemcpyAsync(p, sp, 2 * n, cudaMemcpyDeviceToHost, st));
        if (!km) CK(cudaMemcpyAsync(m, sm, 2 * n, cudaMemcpyDeviceToHost, st));
        if (!kv) CK(cudaMemcpyAsync(v, sv, 2 * n, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
    });
}

// ------------------------------------------------------------ stepper
int ma_stepper_create(const ma_adam_hyper* h, float init_scale, uint32_t growth_interval,
                      int g_dtype, int w_dtype, void* d_state, ma_stepper** out) {
    return guarded([&] {
        check_grad_dtype(g_dtype);
        check_w_dtype(w_dtype);
        if (!out) fail(MA_ERR_INVALID_ARGUMENT, "null output pointer");
        if (!(init_scale > 0.0f)) fail(MA_ERR_INVALID_ARGUMENT, "loss scale must be > 0");
        if (growth_interval == 0) fail(MA_ERR_INVALID_ARGUMENT, "growth_interval must be >= 1");
        const DeviceInfo d = device_info();
        auto* s = new ma_stepper();
        try {
            s->h = *h;
            s->c = make_consts(h);
            s->g_dtype = g_dtype;
            s->w_dtype = w_dtype;
            s->device = d.device;
            static_assert(sizeof(ma::StepDev) <= MA_STEPPER_STATE_BYTES, "state layout");
            static_assert(offsetof(ma::StepDev, scale) == 8, "scale offset");
            if (d_state) {
                if (reinterpret_cast<uintptr_t>(d_state) % 8)
                    fail(MA_ERR_ALIGNMENT, "stepper state must be 8-byte aligned");
                s->d_st = static_cast<ma::StepDev*>(d_state);
                s->owns_state = false;
            } else {
                CK(cudaMalloc(&s->d_st, sizeof(ma::StepDev)));
            }
            CK(cudaMalloc(&s->d_log, sizeof(ma::StepLog) * ma::kHistory));
            ma::StepDev init{};
            init.scale = init_scale;
            init.growth_interval = growth_interval;
            CK(cudaMemcpy(s->d_st, &init, sizeof init, cudaMemcpyHostToDevice));
            CK(cudaMemset(s->d_log, 0, sizeof(ma::StepLog) * ma::kHistory));
            stepper_cover_bc(s, 2);
            ma::launch_step_prepare(s->d_st, s->d_bc, s->bc_first, s->c, nullptr);
            CK(cudaGetLastError());
            CK(cudaDeviceSynchronize());
        } catch (...) {
            if (s->d_st && s->owns_state) cudaFree(s->d_st);
            if (s->d_log) cudaFree(s->d_log);
            if (s->d_bc) cudaFree(s->d_bc);
            delete s;
            throw;
        }
        *out = s;
    });
}

int ma_stepper_destroy(ma_stepper* s) {
    return guarded([&] {
        if (!s) return;
        cudaDeviceSynchronize();
        if (s->owns_state) cudaFree(s->d_st);
        cudaFree(s->d_spec);
        cudaFree(s->d_log);
        cudaFree(s->d_bc);
        for (float2* t : s->retired) cudaFree(t);
        delete s;
    });
}

int ma_stepper_check_async(ma_stepper* s, const void* g, uint64_t n, void* stream) {
    NvtxRange nvtx_range("ma_stepper_check_async");
    return guarded([&] {
        if (!s) fail(MA_ERR_INVALID_ARGUMENT, "null stepper");
        if (n && !g) fail(MA_ERR_INVALID_ARGUMENT, "null gradient pointer");
        launch_k1(g, n, s->g_dtype, &s->d_st->flag, nullptr, 0, true, as_stream(stream), nullptr,
                  true, &s->kept_lo, &s->kept_lines);
        s->last = as_stream(stream);
    });
}

int ma_stepper_check_host_async(ma_stepper* s, const void* host_g, void* dev_g, uint64_t n,
                                uint64_t chunk_elems, void* stream, void* copy_stream) {
    NvtxRange nvtx_range("ma_stepper_check_host_async");
    return guarded([&] {
        if (!s) fail(MA_ERR_INVALID_ARGUMENT, "null stepper");
        if (n == 0) return;
        if (!host_g || !dev_g) fail(MA_ERR_INVALID_ARGUMENT, "null gradient pointer");
        const void* alias;
        if (classify(host_g, &alias) != 2)
            fail(MA_ERR_INVALID_ARGUMENT, "host gradients must be pinned (registered) memory");
        if (chunk_elems == 0) chunk_elems = 64ull << 20;
        const uint64_t es = elem_bytes(s->g_dtype);
        cudaStream_t cs = as_stream(copy_stream);
        cudaStream_t st = as_stream(stream);
        // the copy stream must not overwrite dev_g before earlier work on it retired
        cudaEvent_t ready = s->event(0);
        CK(cudaEventRecord(ready, st));
        CK(cudaStreamWaitEvent(cs, ready, 0));
        uint64_t k = 0;
        for (uint64_t off = 0; off < n; off += chunk_elems, ++k) {
            const uint64_t len = std::min(chunk_elems, n - off);
            CK(cudaMemcpyAsync(static_cast<uint8_t*>(dev_g) + off * es,
                               static_cast<const uint8_t*>(host_g) + off * es, len * es,
                               cudaMemcpyHostToDevice, cs));
            cudaEvent_t landed = s->event(1 + k);
            CK(cudaEventRecord(landed, cs));
            CK(cudaStreamWaitEvent(st, landed, 0));
            launch_k1(static_cast<uint8_t*>(dev_g) + off * es, len, s->g_dtype, &s->d_st->flag,
                      nullptr, 0, true, st, nullptr, off + len == n,
                      off + len == n ? &s->kept_lo : nullptr, &s->kept_lines);
        }
        s->last = st;
    });
}

// Speculative update while the host gradients stream in.  The reference
// decides a step on the whole flat buffer first (simulator.cpp:431-440); on
// the host-buffer path that decision waits for the last PCIe chunk, and the
// update would follow the transfer instead of overlapping it.  Here each
// sub-group whose gradients have all landed (and passed K1) while the flag
// is still clear is updated at once — after copying its p/m/v/w to `backup`
// — and the step's final decision is applied in ma_stepper_apply_spec_async:
// a clear flag keeps the updates, a set one copies the backups back.  The
// bits equal the plain check -> apply path either way (an update is a pure
// function of the old state, and a skip leaves the old state); only the
// HBM traffic of the speculated groups grows (the backup copy), which the
// PCIe transfer hides.  Sub-groups are speculated in order while `backup`
// has room (and at most 96); their g must tile dev_g contiguously, else
// nothing is speculated.
}  // extern "C"

namespace {

// Shared by the fp32-state (K2) and pure-bf16 (K3) forms.  bf16: groups'
// p/m/v are uint16 arrays (as ma_stepper_apply_bf16_async passes them) and
// there are no working weights.
void check_host_spec(ma_stepper* s, const void* host_g, void* dev_g, uint64_t n,
                     uint64_t chunk_elems, const ma_subgroup* groups, uint32_t count, bool bf16,
                     void* backup, uint64_t backup_bytes, void* stream, void* copy_stream) {
    if (!s) fail(MA_ERR_INVALID_ARGUMENT, "null stepper");
    if (!s->spec_groups.empty())
        fail(MA_ERR_LIFECYCLE, "speculative step pending: call ma_stepper_apply_spec_async");
    if (count && !groups) fail(MA_ERR_INVALID_ARGUMENT, "null sub-group list");
    if (n == 0) return;
    if (!host_g || !dev_g) fail(MA_ERR_INVALID_ARGUMENT, "null gradient pointer");
    const void* alias;
    if (classify(host_g, &alias) != 2)
        fail(MA_ERR_INVALID_ARGUMENT, "host gradients must be pinned (registered) memory");
    if (chunk_elems == 0) chunk_elems = 64ull << 20;
    const uint64_t es = elem_bytes(s->g_dtype);
    const uint64_t state_es = bf16 ? 2 : 4;
    const int ntens = bf16 || s->w_dtype == MA_DT_NONE ? 3 : 4;
    auto al = [](uint64_t b) { return (b + 255) & ~uint64_t(255); };
    // plan: the leading sub-groups that tile dev_g and fit the backup
    std::vector<uint64_t> ends, boff;
    {
        uint64_t cum = 0, used = 0;
        bool tiles = true;
        for (uint32_t k = 0; k < count && tiles; ++k) {
            tiles = groups[k].g == static_cast<const uint8_t*>(dev_g) + cum * es;
            cum += groups[k].n;
        }
        tiles = tiles && cum == n;
        cum = 0;
        for (uint32_t k = 0; tiles && backup && k < count && k < ma::kMaxSpecCopies / 4; ++k) {
            const uint64_t gn = groups[k].n;
            const uint64_t need = 3 * al(gn * state_es) + (ntens == 4 ? al(gn * 2) : 0);
            if (used + need > backup_bytes) break;
            boff.push_back(used);
            used += need;
            cum += gn;
            ends.push_back(cum);
        }
    }
    if (!ends.empty() && !s->d_spec) {
        CK(cudaMalloc(&s->d_spec, 2 * sizeof(uint32_t)));
        CK(cudaMemset(s->d_spec, 0, 2 * sizeof(uint32_t)));
    }
    cudaStream_t cs = as_stream(copy_stream);
    cudaStream_t st = as_stream(stream);
    cudaEvent_t ready = s->event(0);
    CK(cudaEventRecord(ready, st));
    CK(cudaStreamWaitEvent(cs, ready, 0));
    ma::SpecRestore rs{};
    std::vector<ma_subgroup> spec;
    size_t next = 0;  // next sub-group to speculate
    uint64_t k = 0;
    for (uint64_t off = 0; off < n; off += chunk_elems, ++k) {
        const uint64_t len = std::min(chunk_elems, n - off);
        CK(cudaMemcpyAsync(static_cast<uint8_t*>(dev_g) + off * es,
                           static_cast<const uint8_t*>(host_g) + off * es, len * es,
                           cudaMemcpyHostToDevice, cs));
        cudaEvent_t landed = s->event(1 + k);
        CK(cudaEventRecord(landed, cs));
        CK(cudaStreamWaitEvent(st, landed, 0));
        launch_k1(static_cast<uint8_t*>(dev_g) + off * es, len, s->g_dtype, &s->d_st->flag,
                  nullptr, 0, true, st, nullptr, off + len == n,
                  off + len == n ? &s->kept_lo : nullptr, &s->kept_lines);
        while (next < ends.size() && ends[next] <= off + len) {
            const ma_subgroup& g = groups[next];
            const uint64_t gn = g.n;
            void* src[4] = {g.p, g.m, g.v, g.w};
            const uint64_t bytes[4] = {gn * state_es, gn * state_es, gn * state_es, gn * 2};
            char* dst = static_cast<char*>(backup) + boff[next];
            for (int t = 0; t < ntens; ++t) {
                CK(cudaMemcpyAsync(dst, src[t], bytes[t], cudaMemcpyDeviceToDevice, st));
                rs.c[rs.count++] = ma::SpecCopy{dst, src[t], bytes[t], static_cast<uint32_t>(next)};
                dst += al(bytes[t]);
            }
            if (bf16)
                launch_k3(&g, 1, s->g_dtype, stepper_args(s), st);
            else
                launch_k2(&g, 1, s->g_dtype, s->w_dtype, stepper_args(s), st);
            ma::launch_spec_mark(s->d_st, s->d_spec, static_cast<uint32_t>(next + 1), st);
            CK(cudaGetLastError());
            spec.push_back(g);
            ++next;
        }
    }
    s->spec_groups = std::move(spec);
    s->spec_restore = rs;
    s->last = st;
}

void apply_spec(ma_stepper* s, const ma_subgroup* groups, uint32_t count, bool bf16,
                void* stream) {
    if (!s) fail(MA_ERR_INVALID_ARGUMENT, "null stepper");
    if (count && !groups) fail(MA_ERR_INVALID_ARGUMENT, "null sub-group list");
    const uint32_t S = static_cast<uint32_t>(s->spec_groups.size());
    if (S > count) fail(MA_ERR_INVALID_ARGUMENT, "fewer sub-groups than were speculated");
    for (uint32_t k = 0; k < S; ++k) {
        const ma_subgroup& a = groups[k];
        const ma_subgroup& b = s->spec_groups[k];
        if (a.p != b.p || a.m != b.m || a.v != b.v || a.g != b.g || a.w != b.w || a.n != b.n)
            fail(MA_ERR_INVALID_ARGUMENT, "sub-groups differ from the speculative check's");
    }
    cudaStream_t st = as_stream(stream);
    if (count > S) {
        if (bf16)
            launch_k3(groups + S, count - S, s->g_dtype, stepper_args(s), st);
        else
            launch_k2(groups + S, count - S, s->g_dtype, s->w_dtype, stepper_args(s), st);
    }
    if (S) {
        const DeviceInfo d = device_info();
        ma::launch_spec_restore(s->spec_restore, s->d_st, s->d_spec,
                                static_cast<unsigned>(d.sms) * 4, st);
        CK(cudaGetLastError());
    }
    s->spec_groups.clear();
    s->spec_restore.count = 0;
    s->last = st;
}

std::vector<ma_subgroup> as_subgroups(const ma_subgroup_bf16* groups, uint32_t count) {
    std::vector<ma_subgroup> gs(count);
    for (uint32_t k = 0; k < count; ++k)
        gs[k] = ma_subgroup{reinterpret_cast<float*>(groups[k].p),
                            reinterpret_cast<float*>(groups[k].m),
                            reinterpret_cast<float*>(groups[k].v), groups[k].g, nullptr,
                            groups[k].n};
    return gs;
}

}  // namespace

extern "C" {

// Speculative update while the host gradients stream in.  The reference
// decides a step on the whole flat buffer first (simulator.cpp:431-440); on
// the host-buffer path that decision waits for the last PCIe chunk, and the
// update would follow the transfer instead of overlapping it.  Here each
// sub-group whose gradients have all landed (and passed K1) while the flag
// is still clear is updated at once — after copying its state to `backup`
// — and the step's final decision is applied in ma_stepper_apply_spec_async:
// a clear flag keeps the updates, a set one copies the backups back.  The
// bits equal the plain check -> apply path either way (an update is a pure
// function of the old state, and a skip leaves the old state); only the
// HBM traffic of the speculated groups grows (the backup copy), which the
// PCIe transfer hides.  Sub-groups are speculated in order while `backup`
// has room (and at most 96); their g must tile dev_g contiguously, else
// nothing is speculated.
int ma_stepper_check_host_spec_async(ma_stepper* s, const void* host_g, void* dev_g, uint64_t n,
                                     uint64_t chunk_elems, const ma_subgroup* groups,
                                     uint32_t count, void* backup, uint64_t backup_bytes,
                                     void* stream, void* copy_stream) {
    NvtxRange nvtx_range("ma_stepper_check_host_spec_async");
    return guarded([&] {
        check_host_spec(s, host_g, dev_g, n, chunk_elems, groups, count, false, backup,
                        backup_bytes, stream, copy_stream);
    });
}

// The step's decision for a speculative check: sub-groups that were not
// speculated are updated now (K2 reads the — possibly exchanged — flag);
// when the flag is set, the speculated ones get their backups back.  groups
// / count as given to the check.  ma_stepper_finish_async follows as usual.
int ma_stepper_apply_spec_async(ma_stepper* s, const ma_subgroup* groups, uint32_t count,
                                void* stream) {
    NvtxRange nvtx_range("ma_stepper_apply_spec_async");
    return guarded([&] { apply_spec(s, groups, count, false, stream); });
}

// The pure-bf16 forms (K3; bf16 weights / m / v backed up).
int ma_stepper_check_host_spec_bf16_async(ma_stepper* s, const void* host_g, void* dev_g,
                                          uint64_t n, uint64_t chunk_elems,
                                          const ma_subgroup_bf16* groups, uint32_t count,
                                          void* backup, uint64_t backup_bytes, void* stream,
                                          void* copy_stream) {
    NvtxRange nvtx_range("ma_stepper_check_host_spec_bf16_async");
    return guarded([&] {
        if (count && !groups) fail(MA_ERR_INVALID_ARGUMENT, "null sub-group list");
        const std::vector<ma_subgroup> gs = as_subgroups(groups, count);
        check_host_spec(s, host_g, dev_g, n, chunk_elems, gs.data(), count, true, backup,
                        backup_bytes, stream, copy_stream);
    });
}

int ma_stepper_apply_spec_bf16_async(ma_stepper* s, const ma_subgroup_bf16* groups,
                                     uint32_t count, void* stream) {
    NvtxRange nvtx_range("ma_stepper_apply_spec_bf16_async");
    return guarded([&] {
        if (count && !groups) fail(MA_ERR_INVALID_ARGUMENT, "null sub-group list");
        const std::vector<ma_subgroup> gs = as_subgroups(groups, count);
        apply_spec(s, gs.data(), count, true, stream);
    });
}

}  // extern "C"

// ------------------------------------------------------------ peer exchange
struct ma_xchg {
    int world = 1;
    int rank = 0;
    unsigned long long* slots = nullptr;  // [2][world], shared with peers via CUDA IPC
    unsigned int* local = nullptr;        // [0] CTA counter, [1] error, [2..3] epoch (u64)
    ma::XchgDev* d_desc = nullptr;
    std::vector<void*> opened;
    bool ready = false;
};

namespace {

ma_xchg* xchg_new(int world, int rank, void* ipc_handle_out) {
    if (world < 1 || world > ma::kMaxRanks || rank < 0 || rank >= world)
        fail(MA_ERR_INVALID_ARGUMENT, "bad world/rank for the peer exchange");
    static_assert(sizeof(cudaIpcMemHandle_t) <= MA_IPC_HANDLE_BYTES, "ipc handle size");
    device_info();
    auto* x = new ma_xchg();
    try {
        x->world = world;
        x->rank = rank;
        CK(cudaMalloc(&x->slots, 2 * static_cast<size_t>(world) * sizeof(unsigned long long)));
        CK(cudaMemset(x->slots, 0, 2 * static_cast<size_t>(world) * sizeof(unsigned long long)));
        CK(cudaMalloc(&x->local, 4 * sizeof(unsigned int)));  // counter, error, epoch (u64)
        CK(cudaMemset(x->local, 0, 4 * sizeof(unsigned int)));
        CK(cudaMalloc(&x->d_desc, sizeof(ma::XchgDev)));
        cudaIpcMemHandle_t h;
        CK(cudaIpcGetMemHandle(&h, x->slots));
        std::memset(ipc_handle_out, 0, MA_IPC_HANDLE_BYTES);
        std::memcpy(ipc_handle_out, &h, sizeof h);
        CK(cudaDeviceSynchronize());  // zeroed slots before any peer can write them
    } catch (...) {
        if (x->slots) cudaFree(x->slots);
        if (x->local) cudaFree(x->local);
        if (x->d_desc) cudaFree(x->d_desc);
        delete x;
        throw;
    }
    return x;
}

// How long a rank waits for its peers inside an exchange / barrier before
// the whole job is stopped (poison + trap, kernels.cu xchg_post_wait):
// MA_PEER_TIMEOUT_S seconds (fractional allowed), default 300.
unsigned long long peer_timeout_ns() {
    double secs = 300.0;
    if (const char* e = std::getenv("MA_PEER_TIMEOUT_S")) {
        char* end = nullptr;
        const double v = std::strtod(e, &end);
        if (end == e || !(v > 0.0) || v > 1e6)
            fail(MA_ERR_INVALID_ARGUMENT, "MA_PEER_TIMEOUT_S must be a positive number of seconds");
        secs = v;
    }
    return static_cast<unsigned long long>(secs * 1e9);
}

// all_handles: world records of `stride` bytes, the slot handle first in each
void xchg_open_impl(ma_xchg* x, const void* all_handles, size_t stride) {
    if (x->ready) fail(MA_ERR_LIFECYCLE, "peer exchange already opened");
    ma::XchgDev desc{};
    desc.world = static_cast<uint32_t>(x->world);
    desc.rank = static_cast<uint32_t>(x->rank);
    desc.my_slots = x->slots;
    desc.counter = x->local;
    desc.error = x->local + 1;
    desc.epoch = reinterpret_cast<unsigned long long*>(x->local + 2);
    desc.timeout_ns = peer_timeout_ns();
    for (int r = 0; r < x->world; ++r) {
        if (r == x->rank) {
            desc.peer_slots[r] = x->slots;
            continue;
        }
        cudaIpcMemHandle_t h;
        std::memcpy(&h, static_cast<const unsigned char*>(all_handles) + r * stride, sizeof h);
        void* p = nullptr;
        CK(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
        x->opened.push_back(p);
        desc.peer_slots[r] = static_cast<unsigned long long*>(p);
    }
    CK(cudaMemcpy(x->d_desc, &desc, sizeof desc, cudaMemcpyHostToDevice));
    x->ready = true;
}

void xchg_free(ma_xchg* x) {
    if (!x) return;
    cudaDeviceSynchronize();
    for (void* p : x->opened) cudaIpcCloseMemHandle(p);
    cudaFree(x->slots);
    cudaFree(x->local);
    cudaFree(x->d_desc);
    delete x;
}

bool xchg_timed_out(const ma_xchg* x) {
    unsigned int e = 0;
    CK(cudaMemcpy(&e, x->local + 1, sizeof e, cudaMemcpyDeviceToHost));
    return e != 0;
}

}  // namespace

extern "C" {

int ma_xchg_create(int world, int rank, ma_xchg** out, void* ipc_handle_out) {
    return guarded([&] {
        if (!out || !ipc_handle_out) fail(MA_ERR_INVALID_ARGUMENT, "null output");
        *out = xchg_new(world, rank, ipc_handle_out);
    });
}

int ma_xchg_open(ma_xchg* x, const void* all_handles) {
    return guarded([&] {
        if (!x || !all_handles) fail(MA_ERR_INVALID_ARGUMENT, "null argument");
        xchg_open_impl(x, all_handles, MA_IPC_HANDLE_BYTES);
    });
}

int ma_xchg_error(ma_xchg* x, int* timed_out) {
    return guarded([&] {
        if (!x || !timed_out) fail(MA_ERR_INVALID_ARGUMENT, "null argument");
        *timed_out = xchg_timed_out(x) ? 1 : 0;
    });
}

int ma_xchg_destroy(ma_xchg* x) {
    return guarded([&] { xchg_free(x); });
}

int ma_stepper_check_xchg_async(ma_stepper* s, const void* g, uint64_t n, ma_xchg* x,
                                void* stream) {
    NvtxRange nvtx_range("ma_stepper_check_xchg_async");
    return guarded([&] {
        if (!s || !x) fail(MA_ERR_INVALID_ARGUMENT, "null stepper / exchange");
        if (!x->ready) fail(MA_ERR_LIFECYCLE, "peer exchange not opened (ma_xchg_open)");
        if (n && !g) fail(MA_ERR_INVALID_ARGUMENT, "null gradient pointer");
        alignas(16) static const uint32_t dummy[4] = {0, 0, 0, 0};  // never read (n == 0)
        launch_k1(n ? g : &dummy, n, s->g_dtype, &s->d_st->flag, nullptr, 0, true,
                  as_stream(stream), x->d_desc, true, &s->kept_lo, &s->kept_lines);
        s->last = as_stream(stream);
    });
}

int ma_stepper_ingest_async(ma_stepper* s, const void* src, int src_dtype, void* dst, uint64_t n,
                            void* stream) {
    NvtxRange nvtx_range("ma_stepper_ingest_async");
    return guarded([&] {
        if (!s) fail(MA_ERR_INVALID_ARGUMENT, "null stepper");
        check_grad_dtype(src_dtype);
        if (n == 0) return;
        if (!src || !dst) fail(MA_ERR_INVALID_ARGUMENT, "null gradient pointer");
        const DeviceInfo d = device_info();
        ma::IngestArgs a{};
        a.src = src;
        a.dst = dst;
        a.n = n;
        a.d_scale = &s->d_st->scale;
        a.flag = &s->d_st->flag;
        const uint32_t es = elem_bytes(src_dtype), ed = elem_bytes(s->g_dtype);
        for (uint64_t h = 0; n >= 8 && h < 8; ++h) {  // co-align src and dst on 16 bytes
            if ((reinterpret_cast<uintptr_t>(src) + h * es) % 16 == 0 &&
                (reinterpret_cast<uintptr_t>(dst) + h * ed) % 16 == 0) {
                a.head = h;
                a.nvec = (n - h) / 8;
                break;
            }
        }
        const uint64_t tile = static_cast<uint64_t>(ma::ingest_units(src_dtype)) * 256;
        a.tiles = (a.nvec + tile - 1) / tile;
        const uint64_t rem = n - a.nvec * 8;
        const uint64_t cap = static_cast<uint64_t>(d.sms) * 8;
        const uint64_t trailing =
            rem ? std::max<uint64_t>(1, std::min<uint64_t>(cap, (rem + 255) / 256)) : 0;
        const uint64_t grid = std::max<uint64_t>(1, a.tiles + trailing);
        if (grid > 0x7FFFFFFFull) fail(MA_ERR_INVALID_ARGUMENT, "buffer too large for one launch");
        ma::launch_ingest(src_dtype, s->g_dtype, a, static_cast<unsigned>(grid), as_stream(stream));
        CK(cudaGetLastError());
        s->last = as_stream(stream);
    });
}

uint32_t* ma_stepper_flag(ma_stepper* s) { return s ? &s->d_st->flag : nullptr; }

float* ma_stepper_scale(ma_stepper* s) { return s ? &s->d_st->scale : nullptr; }

int ma_stepper_apply_async(ma_stepper* s, const ma_subgroup* groups, uint32_t count,
                           void* stream) {
    NvtxRange nvtx_range("ma_stepper_apply_async");
    return guarded([&] {
        if (!s) fail(MA_ERR_INVALID_ARGUMENT, "null stepper");
        if (count && !groups) fail(MA_ERR_INVALID_ARGUMENT, "null sub-group list");
        const ma::AdamArgs a = stepper_args(s);
        launch_k2(groups, count, s->g_dtype, s->w_dtype, a, as_stream(stream));
        s->last = as_stream(stream);
    });
}

int ma_stepper_apply_bf16_async(ma_stepper* s, const ma_subgroup_bf16* groups, uint32_t count,
                                void* stream) {
    NvtxRange nvtx_range("ma_stepper_apply_bf16_async");
    return guarded([&] {
        if (!s) fail(MA_ERR_INVALID_ARGUMENT, "null stepper");
        if (count && !groups) fail(MA_ERR_INVALID_ARGUMENT, "null sub-group list");
        const ma::AdamArgs a = stepper_args(s);
        std::vector<ma_subgroup> gs(count);
        for (uint32_t k = 0; k < count; ++k) {
            gs[k] = ma_subgroup{reinterpret_cast<float*>(groups[k].p),
                                reinterpret_cast<float*>(groups[k].m),
                                reinterpret_cast<float*>(groups[k].v), groups[k].g, nullptr,
                                groups[k].n};
        }
        launch_k3(gs.data(), count, s->g_dtype, a, as_stream(stream));
        s->last = as_stream(stream);
    });
}

}  // extern "C"

namespace {

// The swapped pipeline shared by the fp32 (K2) and pure-bf16 (K3) forms.
// Each group moves `ntens` tensors of `esize`-byte elements: from the swap
// store (keys) through a registered host slot, or from the registered DRAM
// tier (host pointers), into a device slot; `launch` runs the update on the
// compute stream over the device slot's tensors; everything flows back the
// same way.
struct SwapPlan {
    uint32_t count = 0;
    int ntens = 3;
    uint64_t esize = 4;
    std::function<const char*(uint32_t, int)> key;  // nullptr: DRAM tier
    std::function<char*(uint32_t, int)> host;       // DRAM-tier tensor base
    std::function<uint64_t(uint32_t)> n;
    std::function<void(uint32_t, uint64_t, uint64_t, char* const*, cudaStream_t)> launch;
};

void run_swapped(ma_stepper* s, ma_swap* e, const SwapPlan& plan, void* h_staging,
                 uint32_t host_slots, void* d_staging, uint32_t dev_slots, uint64_t slot_elems,
                 void* stream, void* h2d_stream, void* d2h_stream, int* skipped) {
    if (!s) fail(MA_ERR_INVALID_ARGUMENT, "null stepper");
    if (!d_staging || slot_elems == 0 || dev_slots < 2 || dev_slots > 16)
        fail(MA_ERR_INVALID_ARGUMENT, "device staging needs 2..16 slots of slot_elems > 0");
    const int T = plan.ntens;
    const uint64_t E = plan.esize;
    if (slot_elems % (16 / E))  // 16-byte aligned device slot tensors
        fail(MA_ERR_ALIGNMENT, "slot_elems must be a multiple of " + std::to_string(16 / E));
    const uint64_t tb = (slot_elems * E + ma::swp::kGranule - 1) / ma::swp::kGranule *
                        ma::swp::kGranule;  // one tensor in a host slot
    uint32_t n_swapped = 0;
    for (uint32_t k = 0; k < plan.count; ++k) {
        int keys = 0;
        for (int t = 0; t < T; ++t) keys += plan.key(k, t) ? 1 : 0;
        if (keys && keys != T)
            fail(MA_ERR_INVALID_ARGUMENT, "a swapped group needs a key for every state tensor");
        if (keys && plan.n(k) > slot_elems)
            fail(MA_ERR_SIZE_VIOLATION, "swapped group " + std::to_string(k) + " has " +
                                            std::to_string(plan.n(k)) + " elements > slot_elems");
        if (!keys && plan.n(k))
            for (int t = 0; t < T; ++t)
                if (!plan.host(k, t))
                    fail(MA_ERR_INVALID_ARGUMENT, "host-resident group without its state tensors");
        n_swapped += keys && plan.n(k) ? 1 : 0;
    }
    if (n_swapped) {
        if (!e) fail(MA_ERR_INVALID_ARGUMENT, "swapped groups need a swap store");
        if (!h_staging || host_slots < 2)
            fail(MA_ERR_INVALID_ARGUMENT, "swapped groups need >= 2 host slots");
        if (reinterpret_cast<uintptr_t>(h_staging) % ma::swp::kGranule)
            fail(MA_ERR_ALIGNMENT, "host staging must be 4096-aligned");
        const void* alias;
        if (classify(h_staging, &alias) != 2)
            fail(MA_ERR_INVALID_ARGUMENT,
                 "host staging must be registered host memory (ma_host_register)");
    }
    cudaStream_t cs = as_stream(stream);
    cudaStream_t hs = as_stream(h2d_stream);
    cudaStream_t ds = as_stream(d2h_stream);
    // a skipped step reads and writes no optimizer state (simulator.cpp:438-441)
    uint32_t flag = 0;
    CK(cudaMemcpyAsync(&flag, &s->d_st->flag, 4, cudaMemcpyDeviceToHost, cs));
    CK(cudaStreamSynchronize(cs));
    if (skipped) *skipped = flag ? 1 : 0;
    s->last = cs;
    if (flag) return;
    int dev = 0;
    CK(cudaGetDevice(&dev));
    ma::swp::Engine* engp = e ? e->e : nullptr;
    char* hbase = static_cast<char*>(h_staging);
    char* dbase = static_cast<char*>(d_staging);
    auto hslot_ptr = [&](uint32_t h, int t) { return hbase + (static_cast<uint64_t>(T) * h + t) * tb; };
    auto dslot_ptr = [&](uint32_t d, int t) {
        return dbase + (static_cast<uint64_t>(T) * d + t) * slot_elems * E;
    };
    // events: [0] entry, [1 + 3*d + {0 h2d, 1 update, 2 d2h}] device slots,
    // [1 + 3*dev_slots + h] host slot's D2H — all created here: the writer
    // thread must not touch s->events
    s->event(3 * dev_slots + host_slots);
    const std::vector<cudaEvent_t> evs(s->events.begin(),
                                       s->events.begin() + 1 + 3 * dev_slots + host_slots);
    cudaEvent_t entry = evs[0];
    auto dev_ev = [&](uint32_t d, int kind) { return evs[1 + 3 * d + kind]; };
    auto host_ev = [&](uint32_t h) { return evs[1 + 3 * dev_slots + h]; };
    CK(cudaEventRecord(entry, cs));
    CK(cudaStreamWaitEvent(hs, entry, 0));

    // writer thread: waits for a host slot's D2H, writes the group's state
    // back to the store, frees the slot
    struct WB {
        uint32_t group, hslot;
    };
    std::mutex mu;
    std::condition_variable cv;
    std::deque<WB> wq;
    std::vector<char> hfree(host_slots, 1);
    bool closing = false;
    int werr_code = 0;
    std::string werr;
    std::thread writer([&] {
        cudaSetDevice(dev);
        for (;;) {
            WB wb;
            {
                std::unique_lock<std::mutex> lock(mu);
                cv.wait(lock, [&] { return closing || !wq.empty(); });
                if (wq.empty()) return;
                wb = wq.front();
                wq.pop_front();
            }
            int code = 0;
            std::string msg;
            NvtxRange wr("ma_swapped_writeback");
            const cudaError_t ce = cudaEventSynchronize(host_ev(wb.hslot));
            if (ce != cudaSuccess) {
                code = MA_ERR_CUDA;
                msg = std::string("cudaEventSynchronize: ") + cudaGetErrorString(ce);
            } else {
                std::vector<ma::swp::Op*> ops(T, nullptr);
                for (int t = 0; t < T; ++t) {
                    try {
                        ops[t] = engp->submit_write(plan.key(wb.group, t), hslot_ptr(wb.hslot, t),
                                                  tb, plan.n(wb.group) * E);
                    } catch (const ma::swp::Failure& f) {
                        if (!code) code = f.code, msg = f.msg;
                    }
                }
                for (int t = 0; t < T; ++t) {
                    if (!ops[t]) continue;
                    try {
                        engp->wait(ops[t]);
                    } catch (const ma::swp::Failure& f) {
                        if (!code) code = f.code, msg = f.msg;
                    }
                }
            }
            std::lock_guard<std::mutex> lock(mu);
            if (code && !werr_code) werr_code = code, werr = msg;
            hfree[wb.hslot] = 1;
            cv.notify_all();
        }
    });

    // reads: swapped groups in order, each into a free host slot
    std::vector<uint32_t> swapped;
    for (uint32_t k = 0; k < plan.count; ++k)
        if (plan.key(k, 0) && plan.n(k)) swapped.push_back(k);  // empty groups move nothing
    struct Pending {
        uint32_t hslot = 0;
        std::vector<ma::swp::Op*> ops;
    };
    std::vector<Pending> pend(plan.count);
    size_t next_read = 0;
    auto claim_slot = [&](bool block) -> int {
        std::unique_lock<std::mutex> lock(mu);
        for (;;) {
            if (werr_code) return -2;
            for (uint32_t h = 0; h < host_slots; ++h)
                if (hfree[h]) {
                    hfree[h] = 0;
                    return static_cast<int>(h);
                }
            if (!block) return -1;
            cv.wait(lock);
        }
    };
    auto submit_reads = [&](uint32_t k, uint32_t h) {
        pend[k].hslot = h;
        pend[k].ops.assign(T, nullptr);
        for (int t = 0; t < T; ++t)
            pend[k].ops[t] = engp->submit_read(plan.key(k, t), hslot_ptr(h, t), tb);
    };
    auto drain_reads = [&] {  // error path: never leave I/O into the slots in flight
        for (auto& p : pend)
            for (auto*& op : p.ops)
                if (op) {
                    try {
                        engp->wait(op);
                    } catch (const ma::swp::Failure&) {
                    }
                    op = nullptr;
                }
    };
    auto stop_writer = [&] {
        {
            std::lock_guard<std::mutex> lock(mu);
            closing = true;
        }
        cv.notify_all();
        writer.join();
    };
    try {
        std::vector<bool> dused(dev_slots, false);
        uint64_t chunk_no = 0;
        for (uint32_t k = 0; k < plan.count; ++k) {
            if (plan.n(k) == 0) continue;
            const bool keyed = plan.key(k, 0) != nullptr;
            // keep the read-ahead full: block only for this group's own slot
            while (next_read < swapped.size()) {
                const bool mine = swapped[next_read] == k;
                const int h = claim_slot(mine);
                if (h == -2) fail(werr_code, werr);
                if (h < 0) break;
                submit_reads(swapped[next_read], static_cast<uint32_t>(h));
                ++next_read;
            }
            if (keyed) {
                for (auto*& op : pend[k].ops) {
                    ma::swp::Op* o = op;
                    op = nullptr;
                    engp->wait(o);
                }
            }
            const uint64_t n = plan.n(k);
            for (uint64_t off = 0; off < n; off += slot_elems, ++chunk_no) {
                const uint64_t len = std::min(slot_elems, n - off);
                const uint32_t d = static_cast<uint32_t>(chunk_no % dev_slots);
                char* dp[3];
                char* hp[3];
                for (int t = 0; t < T; ++t) {
                    dp[t] = dslot_ptr(d, t);
                    hp[t] = keyed ? hslot_ptr(pend[k].hslot, t) : plan.host(k, t) + off * E;
                }
                if (dused[d]) CK(cudaStreamWaitEvent(hs, dev_ev(d, 2), 0));
                for (int t = 0; t < T; ++t)
                    CK(cudaMemcpyAsync(dp[t], hp[t], len * E, cudaMemcpyHostToDevice, hs));
                CK(cudaEventRecord(dev_ev(d, 0), hs));
                CK(cudaStreamWaitEvent(cs, dev_ev(d, 0), 0));
                plan.launch(k, off, len, dp, cs);
                CK(cudaEventRecord(dev_ev(d, 1), cs));
                CK(cudaStreamWaitEvent(ds, dev_ev(d, 1), 0));
                for (int t = 0; t < T; ++t)
                    CK(cudaMemcpyAsync(hp[t], dp[t], len * E, cudaMemcpyDeviceToHost, ds));
                CK(cudaEventRecord(dev_ev(d, 2), ds));
                dused[d] = true;
            }
            if (keyed) {
                CK(cudaEventRecord(host_ev(pend[k].hslot), ds));
                std::lock_guard<std::mutex> lock(mu);
                wq.push_back(WB{k, pend[k].hslot});
                cv.notify_all();
            }
        }
        for (uint32_t d = 0; d < dev_slots; ++d)
            if (dused[d]) CK(cudaStreamWaitEvent(cs, dev_ev(d, 2), 0));
    } catch (...) {
        drain_reads();
        stop_writer();
        throw;
    }
    stop_writer();
    if (werr_code) fail(werr_code, werr);
}

}  // namespace

extern "C" {

int ma_stepper_apply_swapped(ma_stepper* s, ma_swap* e, const ma_swap_group* groups,
                             uint32_t count, void* h_staging, uint32_t host_slots,
                             float* d_staging, uint32_t dev_slots, uint64_t slot_elems,
                             void* stream, void* h2d_stream, void* d2h_stream, int* skipped) {
    NvtxRange nvtx_range("ma_stepper_apply_swapped");
    return guarded([&] {
        if (count && !groups) fail(MA_ERR_INVALID_ARGUMENT, "null sub-group list");
        SwapPlan plan;
        plan.count = count;
        plan.ntens = 3;
        plan.esize = 4;
        plan.key = [&](uint32_t k, int t) {
            return t == 0 ? groups[k].key_p : t == 1 ? groups[k].key_m : groups[k].key_v;
        };
        plan.host = [&](uint32_t k, int t) {
            return reinterpret_cast<char*>(t == 0 ? groups[k].p : t == 1 ? groups[k].m : groups[k].v);
        };
        plan.n = [&](uint32_t k) { return groups[k].n; };
        const int gdt = s ? s->g_dtype : 0, wdt = s ? s->w_dtype : 0;
        const uint64_t ges = elem_bytes(gdt);
        plan.launch = [&](uint32_t k, uint64_t off, uint64_t len, char* const* d, cudaStream_t st) {
            const ma_swap_group& gr = groups[k];
            ma_subgroup part{reinterpret_cast<float*>(d[0]), reinterpret_cast<float*>(d[1]),
                             reinterpret_cast<float*>(d[2]),
                             static_cast<const uint8_t*>(gr.g) + off * ges,
                             gr.w ? static_cast<uint8_t*>(gr.w) + off * 2 : nullptr, len};
            launch_k2(&part, 1, gdt, wdt, stepper_args(s), st);
        };
        run_swapped(s, e, plan, h_staging, host_slots, d_staging, dev_slots, slot_elems, stream,
                    h2d_stream, d2h_stream, skipped);
    });
}

int ma_stepper_apply_swapped_bf16(ma_stepper* s, ma_swap* e, const ma_swap_group_bf16* groups,
                                  uint32_t count, void* h_staging, uint32_t host_slots,
                                  void* d_staging, uint32_t dev_slots, uint64_t slot_elems,
                                  void* stream, void* h2d_stream, void* d2h_stream,
                                  int* skipped) {
    NvtxRange nvtx_range("ma_stepper_apply_swapped_bf16");
    return guarded([&] {
        if (count && !groups) fail(MA_ERR_INVALID_ARGUMENT, "null sub-group list");
        for (uint32_t k = 0; k < count; ++k)
            if (groups[k].n && !groups[k].p)
                fail(MA_ERR_INVALID_ARGUMENT, "pure-bf16 groups need their device weights");
        SwapPlan plan;
        plan.count = count;
        plan.ntens = 2;
        plan.esize = 2;
        plan.key = [&](uint32_t k, int t) { return t == 0 ? groups[k].key_m : groups[k].key_v; };
        plan.host = [&](uint32_t k, int t) {
            return reinterpret_cast<char*>(t == 0 ? groups[k].m : groups[k].v);
        };
        plan.n = [&](uint32_t k) { return groups[k].n; };
        const int gdt = s ? s->g_dtype : 0;
        const uint64_t ges = elem_bytes(gdt);
        plan.launch = [&](uint32_t k, uint64_t off, uint64_t len, char* const* d, cudaStream_t st) {
            const ma_swap_group_bf16& gr = groups[k];
            ma_subgroup part{reinterpret_cast<float*>(gr.p + off), reinterpret_cast<float*>(d[0]),
                             reinterpret_cast<float*>(d[1]),
                             static_cast<const uint8_t*>(gr.g) + off * ges, nullptr, len};
            launch_k3(&part, 1, gdt, stepper_args(s), st);
        };
        run_swapped(s, e, plan, h_staging, host_slots, d_staging, dev_slots, slot_elems, stream,
                    h2d_stream, d2h_stream, skipped);
    });
}

// configs[3]: every group's state in registered host memory — the swapped
// pipeline with no store (no host slots, no I/O), slices of slot_elems.
int ma_stepper_apply_streamed(ma_stepper* s, const ma_subgroup* groups, uint32_t count,
                              float* d_staging, uint64_t slot_elems, uint32_t slots,
                              void* stream, void* h2d_stream, void* d2h_stream,
                              int* skipped) {
    NvtxRange nvtx_range("ma_stepper_apply_streamed");
    return guarded([&] {
        if (count && !groups) fail(MA_ERR_INVALID_ARGUMENT, "null sub-group list");
        if (!d_staging || slot_elems == 0 || slots < 2 || slots > 16)
            fail(MA_ERR_INVALID_ARGUMENT, "staging needs 2..16 slots of slot_elems > 0");
        SwapPlan plan;
        plan.count = count;
        plan.ntens = 3;
        plan.esize = 4;
        plan.key = [](uint32_t, int) -> const char* { return nullptr; };
        plan.host = [&](uint32_t k, int t) {
            return reinterpret_cast<char*>(t == 0 ? groups[k].p : t == 1 ? groups[k].m : groups[k].v);
        };
        plan.n = [&](uint32_t k) { return groups[k].n; };
        const int gdt = s ? s->g_dtype : 0, wdt = s ? s->w_dtype : 0;
        const uint64_t ges = elem_bytes(gdt);
        plan.launch = [&](uint32_t k, uint64_t off, uint64_t len, char* const* d, cudaStream_t st) {
            const ma_subgroup& gr = groups[k];
            ma_subgroup part{reinterpret_cast<float*>(d[0]), reinterpret_cast<float*>(d[1]),
                             reinterpret_cast<float*>(d[2]),
                             static_cast<const uint8_t*>(gr.g) + off * ges,
                             gr.w ? static_cast<uint8_t*>(gr.w) + off * 2 : nullptr, len};
            launch_k2(&part, 1, gdt, wdt, stepper_args(s), st);
        };
        run_swapped(s, nullptr, plan, nullptr, 0, d_staging, slots, slot_elems, stream,
                    h2d_stream, d2h_stream, skipped);
    });
}

int ma_stepper_finish_async(ma_stepper* s, void* stream) {
    NvtxRange nvtx_range("ma_stepper_finish_async");
    return guarded([&] {
        if (!s) fail(MA_ERR_INVALID_ARGUMENT, "null stepper");
        stepper_cover_bc(s, s->t_base + s->issued + 2);  // the next update's scalars
        ma::launch_step_finish(s->d_st, s->d_log, s->d_bc, s->bc_first, s->c,
                               as_stream(stream));
        CK(cudaGetLastError());
        s->issued += 1;
        s->last = as_stream(stream);
    });
}

int ma_stepper_state(ma_stepper* s, ma_step_state* out) {
    return guarded([&] {
        if (!s || !out) fail(MA_ERR_INVALID_ARGUMENT, "null argument");
        CK(cudaStreamSynchronize(s->last));
        ma::StepDev st{};
        CK(cudaMemcpy(&st, s->d_st, sizeof st, cudaMemcpyDeviceToHost));
        out->scale = st.scale;
        out->clean_steps = st.clean_steps;
        out->updates = st.updates;
        out->steps = st.steps;
        out->last_overflow = st.last_overflow;
        out->growth_interval = st.growth_interval;
    });
}

// Resume: OptimizerState::step_t and LossScaler::{scale, clean_steps}
// (optimizer.hpp:19-35,60-66) restored into the device-resident step state.
int ma_stepper_set_state(ma_stepper* s, float scale, uint32_t clean_steps, uint64_t updates) {
    return guarded([&] {
        if (!s) fail(MA_ERR_INVALID_ARGUMENT, "null stepper");
        if (s->capturing) fail(MA_ERR_LIFECYCLE, "set_state during graph capture");
        if (!(scale > 0.0f)) fail(MA_ERR_INVALID_ARGUMENT, "loss scale must be > 0");
        CK(cudaDeviceSynchronize());  // no step in flight reads the state
        ma::StepDev st{};
        CK(cudaMemcpy(&st, s->d_st, sizeof st, cudaMemcpyDeviceToHost));
        if (clean_steps >= st.growth_interval)
            fail(MA_ERR_INVALID_ARGUMENT, "clean_steps must be < growth_interval");
        st.flag = 0;
        st.scale = scale;
        st.clean_steps = clean_steps;
        st.updates = updates;
        CK(cudaMemcpy(s->d_st, &st, sizeof st, cudaMemcpyHostToDevice));
        s->t_base = updates;
        s->issued = 0;
        stepper_cover_bc(s, updates + 2);
        ma::launch_step_prepare(s->d_st, s->d_bc, s->bc_first, s->c, nullptr);
        CK(cudaGetLastError());
        CK(cudaDeviceSynchronize());
    });
}

int ma_stepper_history(ma_stepper* s, uint8_t* overflow, float* scale_after, uint64_t cap,
                       uint64_t* count) {
    return guarded([&] {
        if (!s || !count) fail(MA_ERR_INVALID_ARGUMENT, "null argument");
        CK(cudaStreamSynchronize(s->last));
        ma::StepDev st{};
        CK(cudaMemcpy(&st, s->d_st, sizeof st, cudaMemcpyDeviceToHost));
        std::vector<ma::StepLog> log(ma::kHistory);
        CK(cudaMemcpy(log.data(), s->d_log, sizeof(ma::StepLog) * ma::kHistory,
                      cudaMemcpyDeviceToHost));
        const uint64_t avail = std::min<uint64_t>(st.steps, ma::kHistory);
        const uint64_t k = std::min<uint64_t>(avail, cap);
        const uint64_t first = st.steps - k;
        for (uint64_t i = 0; i < k; ++i) {
            const ma::StepLog& e = log[(first + i) % ma::kHistory];
            if (overflow) overflow[i] = static_cast<uint8_t>(e.overflow);
            if (scale_after) scale_after[i] = e.scale_after;
        }
        *count = k;
    });
}

// ------------------------------------------------------------ generators
int ma_gen_seeded_weights_async(float* p, void* w, int w_dtype, uint64_t n, uint64_t base,
                                uint64_t seed, void* stream) {
    return guarded([&] {
        check_w_dtype(w_dtype);
        if (n == 0) return;
        const DeviceInfo d = device_info();
        const unsigned grid = static_cast<unsigned>(
            std::min<uint64_t>((n + 255) / 256, static_cast<uint64_t>(d.sms) * 16));
        auto* w16 = static_cast<uint16_t*>(w);
        cudaStream_t st = as_stream(stream);
        ma::launch_gen_weights(w ? w_dtype : MA_DT_NONE, p, w16, n, base, seed, grid, st);
        CK(cudaGetLastError());
    });
}

int ma_gen_pseudo_grads_async(void* g, int g_dtype, const void* w, int w_dtype, uint64_t n,
                              uint64_t base, uint64_t seed, uint64_t step, const float* d_scale,
                              float scale, void* stream) {
    return guarded([&] {
        check_grad_dtype(g_dtype);
        if (w_dtype != MA_DT_BF16 && w_dtype != MA_DT_F16)
            fail(MA_ERR_INVALID_ARGUMENT, "working weights must be BF16 or F16");
        if (n == 0) return;
        const DeviceInfo d = device_info();
        const unsigned grid = static_cast<unsigned>(
            std::min<uint64_t>((n + 255) / 256, static_cast<uint64_t>(d.sms) * 16));
        const auto* w16 = static_cast<const uint16_t*>(w);
        cudaStream_t st = as_stream(stream);
ma::launch_gen_grads(g_dtype, w_dtype, g, w16, n, base, seed, step, d_scale, scale, grid, st);
        CK(cudaGetLastError());
    });
}

int ma_plant_bits_async(void* buf, int dtype, uint64_t index, uint32_t bits, void* stream) {
    return guarded([&] {
        check_grad_dtype(dtype);
        device_info();
        ma::launch_plant(buf, dtype, index, bits, as_stream(stream));
        CK(cudaGetLastError());
    });
}

// ------------------------------------------------------------ host memory
int ma_host_register(void* ptr, uint64_t bytes) {
    return guarded([&] {
        if (!ptr || bytes == 0) fail(MA_ERR_INVALID_ARGUMENT, "empty host region");
        device_info();
        numa_place_for_device(ptr, bytes);  // before pinning: pages can still move
        CK(cudaHostRegister(ptr, bytes, cudaHostRegisterPortable | cudaHostRegisterMapped));
    });
}

int ma_host_place(void* ptr, uint64_t bytes) {
    return guarded([&] {
        if (!ptr || bytes == 0) fail(MA_ERR_INVALID_ARGUMENT, "empty host region");
        numa_place_for_device(ptr, bytes);
    });
}

int ma_device_numa_node(int* node) {
    return guarded([&] {
        if (!node) fail(MA_ERR_INVALID_ARGUMENT, "null output");
        device_info();
        *node = current_device_numa_node();
    });
}

int ma_host_numa_node(const void* ptr, int* node) {
    return guarded([&] {
        if (!ptr || !node) fail(MA_ERR_INVALID_ARGUMENT, "null argument");
        int n = -1;
        // get_mempolicy(MPOL_F_NODE | MPOL_F_ADDR): the node backing the page
        if (::syscall(SYS_get_mempolicy, &n, nullptr, 0ul, const_cast<void*>(ptr), 3ul) != 0)
            n = -1;
        *node = n;
    });
}

int ma_host_unregister(void* ptr) {
    return guarded([&] {
        if (!ptr) fail(MA_ERR_INVALID_ARGUMENT, "null host region");
        device_info();
        const cudaError_t e = cudaHostUnregister(ptr);
        if (e == cudaErrorHostMemoryNotRegistered) {
            cudaGetLastError();
            fail(MA_ERR_UNKNOWN_REGION, "host region was never registered");
        }
        CK(e);
    });
}

int ma_pointer_kind(const void* ptr, int* kind) {
    return guarded([&] {
        if (!kind) fail(MA_ERR_INVALID_ARGUMENT, "null output");
        device_info();
        const void* dev;
        const int k = classify(ptr, &dev);
        *kind = k;
    });
}

// ------------------------------------------------------------ verification
int ma_debug_cast_sweep(int kind, int block_log2, uint64_t* out_host) {
    return guarded([&] {
        if (kind != MA_DT_BF16 && kind != MA_DT_F16)
            fail(MA_ERR_INVALID_ARGUMENT, "cast sweep kind must be BF16 or F16");
        if (block_log2 < 8 || block_log2 > 24) fail(MA_ERR_INVALID_ARGUMENT, "block_log2 in [8, 24]");
        device_info();
        const uint64_t nb = 1ull << (32 - block_log2);
        uint64_t* d = nullptr;
        CK(cudaMalloc(&d, nb * 8));
        ma::launch_cast_sweep(kind, block_log2, d, nb);
        const cudaError_t e = cudaGetLastError();
        const cudaError_t e2 = cudaMemcpy(out_host, d, nb * 8, cudaMemcpyDeviceToHost);
        cudaFree(d);
        CK(e);
        CK(e2);
    });
}

int ma_debug_fast_sweep(int mode, const float* divisors, uint32_t ndiv, uint64_t samples,
                        uint64_t seed, uint64_t* mismatches, uint64_t* checked) {
    return guarded([&] {
        if (!mismatches || !checked) fail(MA_ERR_INVALID_ARGUMENT, "null output");
        if (mode < 0 || mode > 2) fail(MA_ERR_INVALID_ARGUMENT, "mode must be 0, 1 or 2");
        if (mode == 1 && (!divisors || ndiv == 0)) fail(MA_ERR_INVALID_ARGUMENT, "no divisors");
        const DeviceInfo dv = device_info();
        const uint64_t count = mode == 0 ? 0x60000001ull
                               : mode == 1 ? static_cast<uint64_t>(ndiv) << 27
                                           : samples;
        unsigned long long* d = nullptr;
        float* dd = nullptr;
        CK(cudaMalloc(&d, 8));
        CK(cudaMemset(d, 0, 8));
        if (mode == 1) {
            CK(cudaMalloc(&dd, ndiv * sizeof(float)));
            CK(cudaMemcpy(dd, divisors, ndiv * sizeof(float), cudaMemcpyHostToDevice));
        }
        ma::launch_fast_sweep(mode, dd, count, seed, d, static_cast<unsigned>(dv.sms * 16));
        const cudaError_t e = cudaGetLastError();
        unsigned long long h = 0;
        const cudaError_t e2 = cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
        cudaFree(d);
        if (dd) cudaFree(dd);
        CK(e);
        CK(e2);
        *mismatches = h;
        *checked = count;
    });
}

int ma_debug_mask_sweep(int kind, uint64_t* mismatches) {
    return guarded([&] {
        check_grad_dtype(kind);
        const DeviceInfo dv = device_info();
        unsigned long long* d = nullptr;
        CK(cudaMalloc(&d, 8));
        CK(cudaMemset(d, 0, 8));
        ma::launch_mask_sweep(kind, d, static_cast<unsigned>(dv.sms * 8));
        const cudaError_t e = cudaGetLastError();
        unsigned long long h = 0;
        const cudaError_t e2 = cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
        cudaFree(d);
        CK(e);
        CK(e2);
        *mismatches = h;
    });
}

}  // extern "C"

// ------------------------------------------------------------ reduce-scatter
// K4 host side: the gradient reduce-scatter with the overflow check in its
// epilogue.  ma_rs shares this rank's full gradient
// buffer with every peer through CUDA IPC (the allocation handle plus the
// offset of the buffer inside it) and owns an exchange slot set for the two
// barriers of a step.
struct ma_rs {
    ma_xchg* x = nullptr;
    int dtype = MA_DT_BF16;
    uint64_t n_total = 0;
    std::vector<const void*> grads;  // [world]: this rank's buffer, peers' mappings
    std::vector<void*> opened;
    bool ready = false;
};

namespace {

constexpr uint32_t kRsMagic = 0x4D415253u;  // "MARS"

struct RsHandle {
    unsigned char slots[MA_IPC_HANDLE_BYTES];
    unsigned char grads[MA_IPC_HANDLE_BYTES];
    uint64_t offset;
    uint64_t n_total;
    int32_t dtype, rank, world;
    uint32_t magic;
};
static_assert(sizeof(RsHandle) <= MA_RS_HANDLE_BYTES, "reduce-scatter handle size");

// Base of the device allocation holding p (IPC handles name allocations).
const void* allocation_base(const void* p) {
    using Fn = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
    static Fn fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q{};
        void* f = nullptr;
        CK(cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q));
        if (q != cudaDriverEntryPointSuccess || !f) fail(MA_ERR_CUDA, "cuMemGetAddressRange unavailable");
        fn = reinterpret_cast<Fn>(f);
    }
    CUdeviceptr base = 0;
    size_t size = 0;
    if (fn(&base, &size, reinterpret_cast<CUdeviceptr>(p)) != CUDA_SUCCESS)
        fail(MA_ERR_INVALID_ARGUMENT, "gradient buffer is not device memory");
    return reinterpret_cast<const void*>(base);
}

uint32_t dtype_bytes(int dt) { return dt == MA_DT_F32 ? 4u : 2u; }

void launch_reduce(ma_stepper* s, const void* const* srcs, int nsrc, int sdt, uint64_t n,
                   float post_scale, void* dst, const ma::XchgDev* xd, cudaStream_t st) {
    if (n == 0 && !xd) return;
    const DeviceInfo d = device_info();
    ma::RsArgs a{};
    const uint32_t es = dtype_bytes(sdt), ed = dtype_bytes(s->g_dtype);
    for (int r = 0; r < nsrc; ++r) a.src[r] = srcs[r];
    a.nsrc = static_cast<uint32_t>(nsrc);
    a.dst = dst;
    a.n = n;
    a.post_scale = post_scale;
    a.flag = &s->d_st->flag;
    a.xchg = xd;
    // co-align every source and dst on 16 bytes at the same element
    for (uint64_t h = 0; n >= 8 && h < 8; ++h) {
        bool ok = (reinterpret_cast<uintptr_t>(dst) + h * ed) % 16 == 0;
        for (int r = 0; r < nsrc && ok; ++r)
            ok = (reinterpret_cast<uintptr_t>(srcs[r]) + h * es) % 16 == 0;
        if (ok) {
            a.head = h;
            a.nvec = (n - h) / 8;
            break;
        }
    }
    const uint64_t tile = static_cast<uint64_t>(ma::rs_units_for(sdt, a.nsrc)) * 256;
    a.tiles = (a.nvec + tile - 1) / tile;
    const uint64_t rem = n - a.nvec * 8;
    const uint64_t cap = static_cast<uint64_t>(d.sms) * 8;
    const uint64_t trailing = rem ? std::max<uint64_t>(1, std::min<uint64_t>(cap, (rem + 255) / 256)) : 0;
    const uint64_t grid = std::max<uint64_t>(1, a.tiles + trailing);
    if (grid > 0x7FFFFFFFull) fail(MA_ERR_INVALID_ARGUMENT, "partition too large for one launch");
    ma::launch_reduce_check(sdt, s->g_dtype, a, static_cast<unsigned>(grid), st);
    CK(cudaGetLastError());
}

}  // namespace

extern "C" {

int ma_stepper_reduce_check_async(ma_stepper* s, const void* const* srcs, int nsrc, int src_dtype,
                                  uint64_t n, float post_scale, void* dst, void* stream) {
    NvtxRange nvtx_range("ma_stepper_reduce_check_async");
    return guarded([&] {
        if (!s) fail(MA_ERR_INVALID_ARGUMENT, "null stepper");
        check_grad_dtype(src_dtype);
        if (nsrc < 1 || nsrc > ma::kMaxRanks) fail(MA_ERR_INVALID_ARGUMENT, "nsrc out of range");
        if (n == 0) return;
        if (!srcs || !dst) fail(MA_ERR_INVALID_ARGUMENT, "null source list / destination");
        for (int r = 0; r < nsrc; ++r)
            if (!srcs[r]) fail(MA_ERR_INVALID_ARGUMENT, "null source pointer");
        launch_reduce(s, srcs, nsrc, src_dtype, n, post_scale, dst, nullptr, as_stream(stream));
        s->last = as_stream(stream);
    });
}

int ma_rs_create(int world, int rank, const void* grads, uint64_t n_total, int dtype, ma_rs** out,
                 void* handle_out) {
    return guarded([&] {
        if (!out || !handle_out) fail(MA_ERR_INVALID_ARGUMENT, "null output");
        check_grad_dtype(dtype);
        if (!grads || n_total == 0) fail(MA_ERR_INVALID_ARGUMENT, "empty gradient buffer");
        RsHandle h{};
        ma_xchg* x = xchg_new(world, rank, h.slots);
        auto* r = new ma_rs();
        try {
            r->x = x;
            r->dtype = dtype;
            r->n_total = n_total;
            const void* base = allocation_base(grads);
            cudaIpcMemHandle_t gh;
            CK(cudaIpcGetMemHandle(&gh, const_cast<void*>(base)));
            std::memcpy(h.grads, &gh, sizeof gh);
            h.offset = static_cast<uint64_t>(static_cast<const uint8_t*>(grads) -
                                             static_cast<const uint8_t*>(base));
            h.n_total = n_total;
            h.dtype = dtype;
            h.rank = rank;
            h.world = world;
            h.magic = kRsMagic;
            r->grads.assign(world, nullptr);
            r->grads[rank] = grads;
        } catch (...) {
            xchg_free(x);
            delete r;
            throw;
        }
        std::memset(handle_out, 0, MA_RS_HANDLE_BYTES);
        std::memcpy(handle_out, &h, sizeof h);
        *out = r;
    });
}

int ma_rs_open(ma_rs* r, const void* all_handles) {
    return guarded([&] {
        if (!r || !all_handles) fail(MA_ERR_INVALID_ARGUMENT, "null argument");
        if (r->ready) fail(MA_ERR_LIFECYCLE, "reduce-scatter already opened");
        const int world = r->x->world;
        const auto* blob = static_cast<const unsigned char*>(all_handles);
        for (int k = 0; k < world; ++k) {
            RsHandle h;
            std::memcpy(&h, blob + static_cast<size_t>(k) * MA_RS_HANDLE_BYTES, sizeof h);
            if (h.magic != kRsMagic || h.rank != k || h.world != world)
                fail(MA_ERR_INVALID_ARGUMENT, "handle list is not in rank order / not ma_rs handles");
            if (h.n_total != r->n_total || h.dtype != r->dtype)
                fail(MA_ERR_INVALID_ARGUMENT, "ranks disagree on the gradient length or dtype");
        }
        for (int k = 0; k < world; ++k) {
            if (k == r->x->rank) continue;
            RsHandle h;
            std::memcpy(&h, blob + static_cast<size_t>(k) * MA_RS_HANDLE_BYTES, sizeof h);
            cudaIpcMemHandle_t gh;
            std::memcpy(&gh, h.grads, sizeof gh);
            void* p = nullptr;
            CK(cudaIpcOpenMemHandle(&p, gh, cudaIpcMemLazyEnablePeerAccess));
            r->opened.push_back(p);
            r->grads[k] = static_cast<const uint8_t*>(p) + h.offset;
        }
        xchg_open_impl(r->x, all_handles, MA_RS_HANDLE_BYTES);
        r->ready = true;
    });
}

int ma_rs_error(ma_rs* r, int* timed_out) {
    return guarded([&] {
        if (!r || !timed_out) fail(MA_ERR_INVALID_ARGUMENT, "null argument");
        *timed_out = xchg_timed_out(r->x) ? 1 : 0;
    });
}

int ma_rs_destroy(ma_rs* r) {
    return guarded([&] {
        if (!r) return;
        cudaDeviceSynchronize();
        for (void* p : r->opened) cudaIpcCloseMemHandle(p);
        xchg_free(r->x);
        delete r;
    });
}

int ma_stepper_reduce_scatter_async(ma_stepper* s, ma_rs* r, uint64_t base, uint64_t n,
                                    float post_scale, void* dst, void* stream) {
    NvtxRange nvtx_range("ma_stepper_reduce_scatter_async");
    return guarded([&] {
        if (!s || !r) fail(MA_ERR_INVALID_ARGUMENT, "null stepper / reduce-scatter");
        if (!r->ready) fail(MA_ERR_LIFECYCLE, "reduce-scatter not opened (ma_rs_open)");
        if (base > r->n_total || n > r->n_total - base)
            fail(MA_ERR_INVALID_ARGUMENT, "partition outside the gradient buffer");
        if (n && !dst) fail(MA_ERR_INVALID_ARGUMENT, "null destination");
        const cudaStream_t st = as_stream(stream);
        const int world = r->x->world;
        const uint32_t es = dtype_bytes(r->dtype);
        std::vector<const void*> srcs(world);
        for (int k = 0; k < world; ++k) srcs[k] = static_cast<const uint8_t*>(r->grads[k]) + base * es;
        // entry: every rank's gradients are complete before anyone reads them
        ma::launch_peer_barrier(r->x->d_desc, st);
        CK(cudaGetLastError());
        // K4, whose last CTA is the exit barrier (no rank overwrites its
        // gradients while a peer still reads them) and the flag OR
        alignas(16) static const uint32_t dummy[4] = {0, 0, 0, 0};  // never written (n == 0)
        launch_reduce(s, srcs.data(), world, r->dtype, n, post_scale, n ? dst : const_cast<uint32_t*>(dummy),
                      r->x->d_desc, st);
        s->last = st;
    });
}

int ma_stepper_apply_allgather_async(ma_stepper* s, const ma_subgroup* groups, uint32_t count,
                                     ma_rs* ag, void* stream) {
    NvtxRange nvtx_range("ma_stepper_apply_allgather_async");
    return guarded([&] {
        if (!s || !ag) fail(MA_ERR_INVALID_ARGUMENT, "null stepper / peer weight set");
        if (count && !groups) fail(MA_ERR_INVALID_ARGUMENT, "null sub-group list");
        if (!ag->ready) fail(MA_ERR_LIFECYCLE, "peer weight set not opened (ma_rs_open)");
        if (s->w_dtype == MA_DT_NONE || ag->dtype != s->w_dtype)
            fail(MA_ERR_INVALID_ARGUMENT,
                 "the peer buffers must hold the stepper's working-weight kind");
        const int world = ag->x->world, rank = ag->x->rank;
        if (world - 1 > ma::kMaxAgPeers)
            fail(MA_ERR_INVALID_ARGUMENT, "the fused all-gather spans at most 8 ranks");
        const char* local = static_cast<const char*>(ag->grads[rank]);
        const char* local_end = local + ag->n_total * 2;
        for (uint32_t k = 0; k < count; ++k) {
            if (groups[k].n == 0) continue;
            const char* w = static_cast<const char*>(groups[k].w);
            if (!w || w < local || w + groups[k].n * 2 > local_end)
                fail(MA_ERR_INVALID_ARGUMENT, "sub-group " + std::to_string(k) +
                                                  "'s working weights are not inside this "
                                                  "rank's shared weight buffer");
        }
        const cudaStream_t st = as_stream(stream);
        ma::AdamArgs a = stepper_args(s);
        for (int k = 0; k < world; ++k)
            if (k != rank)
                a.peers.delta[a.peers.n++] =
                    static_cast<long long>(static_cast<const char*>(ag->grads[k]) - local);
        // entry: every rank is done with its copy of the previous weights
        // (a rank missing here forces this rank's skip, like the exchange)
        ma::launch_peer_barrier(ag->x->d_desc, st);
        CK(cudaGetLastError());
        launch_k2(groups, count, s->g_dtype, s->w_dtype, a, st, /*allgather=*/true);
        // exit: every rank's pushes into every buffer are complete
        ma::launch_peer_barrier(ag->x->d_desc, st);
        CK(cudaGetLastError());
        s->last = st;
    });
}

}  // extern "C"

// ------------------------------------------------------------ CUDA graphs
// A captured step chain (check -> [flag all-reduce] -> apply -> finish, any
// sequence of *_async calls on one stream) replayed with one launch.  The
// kernels read the loss scale, the skip flag and t on the device, so one
// graph serves every later step; the only host-side state is the count of
// finish calls (t's upper bound for the bias-correction table baked into the
// graph, which begin() sizes for `reserve_steps` replays of one step).
struct ma_graph {
    ma_stepper* s = nullptr;
    cudaGraphExec_t exec = nullptr;
    uint64_t finishes = 0;  // finish calls per replay
    uint64_t bc_first = 0;  // the window of bias corrections the graph's kernels read
    uint64_t bc_cap = 0;
};

extern "C" {

int ma_stepper_graph_begin(ma_stepper* s, uint64_t reserve_steps, void* stream) {
    return guarded([&] {
        if (!s) fail(MA_ERR_INVALID_ARGUMENT, "null stepper");
        if (!stream) fail(MA_ERR_INVALID_ARGUMENT, "graph capture needs a non-default stream");
        if (s->capturing) fail(MA_ERR_LIFECYCLE, "graph capture already in progress");
        stepper_cover_bc(s, s->t_base + s->issued + reserve_steps + 2);
        CK(cudaStreamBeginCapture(as_stream(stream), cudaStreamCaptureModeThreadLocal));
        s->capturing = true;
        s->capture_issued = s->issued;
    });
}

int ma_stepper_graph_end(ma_stepper* s, void* stream, ma_graph** out) {
    return guarded([&] {
        if (!s || !out) fail(MA_ERR_INVALID_ARGUMENT, "null argument");
        if (!s->capturing) fail(MA_ERR_LIFECYCLE, "no graph capture in progress");
        cudaGraph_t graph = nullptr;
        const cudaError_t e = cudaStreamEndCapture(as_stream(stream), &graph);
        s->capturing = false;
        const uint64_t finishes = s->issued - s->capture_issued;
        s->issued = s->capture_issued;  // nothing executed yet
        cuda_check(e, "cudaStreamEndCapture");
        auto* g = new ma_graph();
        g->s = s;
        g->finishes = finishes;
        g->bc_first = s->bc_first;
        g->bc_cap = s->bc_cap;
        const cudaError_t ie = cudaGraphInstantiate(&g->exec, graph, 0);
        cudaGraphDestroy(graph);
        if (ie != cudaSuccess) {
            delete g;
            cuda_check(ie, "cudaGraphInstantiate");
        }
        *out = g;
    });
}

int ma_graph_launch(ma_graph* g, void* stream) {
    return guarded([&] {
        if (!g) fail(MA_ERR_INVALID_ARGUMENT, "null graph");
        ma_stepper* s = g->s;
        if (s->t_base + 1 < g->bc_first ||
            s->t_base + s->issued + g->finishes + 1 >= g->bc_first + g->bc_cap)
            fail(MA_ERR_LIFECYCLE, "graph's bias-correction window exhausted: capture again");
        CK(cudaGraphLaunch(g->exec, as_stream(stream)));
        s->issued += g->finishes;
        s->last = as_stream(stream);
    });
}

int ma_graph_destroy(ma_graph* g) {
    return guarded([&] {
        if (!g) return;
        if (g->exec) cudaGraphExecDestroy(g->exec);
        delete g;
    });
}

}  // extern "C"
