// ORACLE — TEST INFRASTRUCTURE ONLY.
//
// extern "C" shim over the UNMODIFIED reference library, compiled from the
// sources where they lie under /root/reference/proj (oracle/Makefile) into
// oracle/_ref/libmemascend_ref.so.  Loaded via ctypes by tests/ (to pin the
// restatement in memascend_oracle.c) and by bench.py's reference arm /
// cpu_baseline leg (the reference's own CPU path, timed on the host cores).
#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <span>
#include <string>
#include <thread>
#include <vector>

#include "memascend/direct_io.hpp"
#include "memascend/error.hpp"
#include "memascend/halfprec.hpp"
#include "memascend/model.hpp"
#include "memascend/optimizer.hpp"
#include "memascend/overflow.hpp"
#include "memascend/simulator.hpp"

using namespace memascend;

namespace {

thread_local std::string g_last_error;

template <typename F>
int guarded(F&& fn) {
    try {
        fn();
        return 0;
    } catch (const Error& e) {
        g_last_error = e.what();
        return 1 + static_cast<int>(e.code());
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return 1000;
    }
}

AdamHyper to_hyper(const float* h) {
    AdamHyper a;
    a.lr = h[0];
    a.beta1 = h[1];
    a.beta2 = h[2];
    a.eps = h[3];
    a.weight_decay = h[4];
    return a;
}

// Splits [0, n) into `workers` contiguous slices run on std::threads.
template <typename F>
void parallel_slices(std::uint64_t n, std::uint32_t workers, F&& body) {
    if (workers <= 1 || n < 4096) {
        body(0, n);
        return;
    }
    const std::uint64_t per = (n + workers - 1) / workers;
    std::vector<std::thread> th;
    for (std::uint32_t w = 0; w < workers; ++w) {
        const std::uint64_t b = w * per;
        const std::uint64_t e = std::min(n, b + per);
        if (b >= e) break;
        th.emplace_back([&body, b, e] { body(b, e); });
    }
    for (auto& t : th) t.join();
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_last_error.c_str(); }

// proj/src/overflow.cpp:73-145
int ref_fused_overflow_check(const float* data, std::uint64_t n, std::uint32_t workers,
                             std::uint64_t chunk_bytes, int early_exit, int track,
                             int* overflow, std::uint64_t* first) {
    return guarded([&] {
        ScanConfig cfg;
        cfg.worker_count = workers;
        cfg.chunk_bytes = chunk_bytes;
        cfg.early_exit = early_exit != 0;
        cfg.track_first_index = track != 0;
        const auto r = fused_overflow_check(std::span<const float>(data, n), cfg);
        *overflow = r.overflow ? 1 : 0;
        if (first) *first = r.first_offending_index.value_or(UINT64_MAX);
    });
}

// proj/src/overflow.cpp:147-199
int ref_naive_overflow_check(const float* data, std::uint64_t n, int* overflow,
                             std::uint64_t* peak_extra) {
    return guarded([&] {
        MemoryMeter meter;
        const auto r = naive_overflow_check(std::span<const float>(data, n), meter);
        *overflow = r.overflow ? 1 : 0;
        *peak_extra = r.peak_extra_bytes;
    });
}

// proj/src/optimizer.cpp:103-109; hyper = {lr, beta1, beta2, eps, wd}
int ref_adam_step_fp32(float* p, float* m, float* v, const float* g, std::uint64_t n,
                       std::uint64_t t, const float* hyper, float scale, std::uint32_t workers) {
    return guarded([&] {
        adam_step_fp32({p, n}, {m, n}, {v, n}, {g, n}, t, to_hyper(hyper), scale, workers);
    });
}

// proj/src/optimizer.cpp:111-118
int ref_adam_step_bf16(std::uint16_t* p, std::uint16_t* m, std::uint16_t* v, const float* g,
                       std::uint64_t n, std::uint64_t t, const float* hyper, float scale,
                       std::uint32_t workers) {
    return guarded([&] {
        adam_step_bf16({p, n}, {m, n}, {v, n}, {g, n}, t, to_hyper(hyper), scale, workers);
    });
}

std::uint16_t ref_fp16_from_float(float f) { return fp16_from_float(f); }
std::uint16_t ref_bf16_from_float(float f) { return bf16_from_float(f); }
float ref_fp16_to_float(std::uint16_t h) { return fp16_to_float(h); }
float ref_bf16_to_float(std::uint16_t h) { return bf16_to_float(h); }

// kind 1 = bf16, 2 = fp16 (memascend_oracle.h numbering)
void ref_cast_sweep_checksums(int kind, int block_log2, std::uint64_t* out, int threads) {
    const std::uint64_t nblocks = 1ull << (32 - block_log2);
    const std::uint64_t bs = 1ull << block_log2;
    std::atomic<std::uint64_t> next{0};
    auto worker = [&] {
        for (;;) {
            const std::uint64_t b = next.fetch_add(1);
            if (b >= nblocks) return;
            std::uint64_t h = 1469598103934665603ull;
            for (std::uint64_t k = 0; k < bs; ++k) {
                const float f = bits_float(static_cast<std::uint32_t>(b * bs + k));
                const std::uint16_t r = kind == 1 ? bf16_from_float(f) : fp16_from_float(f);
                const auto* c = reinterpret_cast<const unsigned char*>(&r);
                h = (h ^ c[0]) * 1099511628211ull;
                h = (h ^ c[1]) * 1099511628211ull;
            }
            out[b] = h;
        }
    };
    std::vector<std::thread> th;
    for (int t = 1; t < threads; ++t) th.emplace_back(worker);
    worker();
    for (auto& t : th) t.join();
}

float ref_pseudo_gradient(std::uint64_t seed, std::uint64_t step, std::uint64_t index, float w) {
    return pseudo_gradient(seed, step, index, w);
}
float ref_seeded_weight(std::uint64_t seed, std::uint64_t index) {
    return seeded_weight(seed, index);
}

std::uint64_t ref_preset_elements(const char* name, std::uint64_t ranks) {
    std::uint64_t n = 0;
    guarded([&] {
        auto spec = preset(name);
        for (const auto& t : enumerate_offload_tensors(spec, ranks)) n += t.rows * t.cols;
    });
    return n;
}

// proj/src/simulator.cpp:243-535 (run_training) on a preset.
// digest_out: 17 chars.  overflow_steps: capacity `cap`.
int ref_run_training(const char* preset_name, std::uint64_t steps, std::uint64_t seed,
                     int pure_bf16, std::int64_t fault_step, std::uint64_t fault_index,
                     std::uint32_t fault_bits, char* digest_out, float* final_scale,
                     std::uint64_t* overflow_steps, std::uint64_t cap, std::uint64_t* n_overflow) {
    return guarded([&] {
        SimConfig cfg;
        cfg.model = preset(preset_name);
        cfg.steps = steps;
        cfg.seed = seed;
        cfg.device_bytes = 32ull << 20;
        cfg.precision = pure_bf16 ? OptimPrecision::pure_bf16 : OptimPrecision::mixed_fp16_fp32master;
        if (fault_step >= 0) {
            cfg.fault = FaultInjection{static_cast<std::uint64_t>(fault_step), fault_index, fault_bits};
        }
        const auto rep = run_training(cfg);
        std::memcpy(digest_out, rep.master_digest.c_str(), 17);
        *final_scale = rep.final_scale;
        *n_overflow = rep.overflow_steps.size();
        for (std::uint64_t i = 0; i < rep.overflow_steps.size() && i < cap; ++i) {
            overflow_steps[i] = rep.overflow_steps[i];
        }
    });
}

// The reference's composed clean-step hot path on one partition, the way
// run_training drives it (simulator.cpp:431-469): one fused check over the
// whole flat fp32 buffer, then per sub-group adam_step_fp32 followed by the
// working-weight refresh.  The cast loop is serial in the reference; here it
// is split across `workers` threads so the CPU baseline is not penalised.
// w_kind: 1 = bf16, 2 = fp16.  Returns wall seconds in *seconds.
int ref_bench_step(const float* g, float* p, float* m, float* v, std::uint16_t* w, int w_kind,
                   std::uint64_t n, std::uint64_t subgroup, std::uint64_t t, const float* hyper,
                   float scale, std::uint32_t workers, int* overflow, double* seconds) {
    return guarded([&] {
        const auto t0 = std::chrono::steady_clock::now();
        ScanConfig cfg;
        cfg.worker_count = workers;
        const bool of = fused_overflow_check(std::span<const float>(g, n), cfg).overflow;
        *overflow = of ? 1 : 0;
        if (!of) {
            const AdamHyper h = to_hyper(hyper);
            for (std::uint64_t off = 0; off < n; off += subgroup) {
                const std::uint64_t len = std::min(subgroup, n - off);
                adam_step_fp32({p + off, len}, {m + off, len}, {v + off, len}, {g + off, len}, t,
                               h, scale, workers);
                parallel_slices(len, workers, [&](std::uint64_t b, std::uint64_t e) {
                    for (std::uint64_t k = b; k < e; ++k) {
                        w[off + k] = w_kind == 1 ? bf16_from_float(p[off + k])
                                                 : fp16_from_float(p[off + k]);
                    }
                });
            }
        }
        *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    });
}

// The reference's swapped optimizer step (configs[4]; simulator.cpp:453-469,
// mixed branch): per group read master/m/v from its DirectIoEngine,
// adam_step_fp32, write master/m/v back, refresh the working weights.  The
// store lives in `dir` (file-backed virtual devices, O_DIRECT); `groups`
// groups of `group_elems` are initialised (seeded weights, zero moments) and
// then `warmup + steps` steps run with fixed gradients.  workers > 1 splits
// Adam and the cast (the reference's simulator passes workers = 1).
// *seconds = median wall seconds per step; *io_bytes = bytes moved per step.
int ref_swap_bench(const char* dir, std::uint32_t devices, std::uint64_t group_elems,
                   std::uint32_t groups, std::uint32_t steps, std::uint32_t warmup,
                   const float* g, const float* hyper, float scale, std::uint32_t workers,
                   std::uint32_t io_workers, double* seconds, double* io_bytes) {
    return guarded([&] {
        const std::uint64_t tbytes = (group_elems * 4 + 4095) / 4096 * 4096;
        const std::uint64_t per_dev =
            ((3 * tbytes * groups) / devices + (16u << 20)) / 4096 * 4096;
        auto devset = DirectIoEngine::create_virtual_devices(dir, devices, per_dev);
        EngineConfig cfg;
        cfg.workers = io_workers;
        DirectIoEngine engine(devset, cfg);
        auto alloc = [&](std::uint64_t b) {
            return static_cast<float*>(std::aligned_alloc(4096, b));
        };
        float* master = alloc(tbytes);
        float* m = alloc(tbytes);
        float* v = alloc(tbytes);
        std::vector<std::uint16_t> w16(group_elems);
        auto bytes = [&](float* p) { return std::span<std::byte>(reinterpret_cast<std::byte*>(p), tbytes); };
        for (std::uint32_t k = 0; k < groups; ++k) {
            for (std::uint64_t i = 0; i < group_elems; ++i)
                master[i] = seeded_weight(1, k * group_elems + i);
            std::memset(m, 0, tbytes);
            engine.write_tensor("master.g" + std::to_string(k), bytes(master), group_elems * 4);
            engine.write_tensor("m.g" + std::to_string(k), bytes(m), group_elems * 4);
            engine.write_tensor("v.g" + std::to_string(k), bytes(m), group_elems * 4);
        }
        const AdamHyper h = to_hyper(hyper);
        std::vector<double> times;
        const auto io0 = engine.stats();
        for (std::uint32_t s = 0; s < warmup + steps; ++s) {
            const auto t0 = std::chrono::steady_clock::now();
            for (std::uint32_t k = 0; k < groups; ++k) {
                const std::string id = "g" + std::to_string(k);
                engine.read_tensor("m." + id, bytes(m));
                engine.read_tensor("v." + id, bytes(v));
                engine.read_tensor("master." + id, bytes(master));
                adam_step_fp32({master, group_elems}, {m, group_elems}, {v, group_elems},
                               {g + k * group_elems, group_elems}, s + 1, h, scale, workers);
                engine.write_tensor("master." + id, bytes(master), group_elems * 4);
                engine.write_tensor("m." + id, bytes(m), group_elems * 4);
                engine.write_tensor("v." + id, bytes(v), group_elems * 4);
                parallel_slices(group_elems, workers, [&](std::uint64_t b, std::uint64_t e) {
                    for (std::uint64_t i = b; i < e; ++i) w16[i] = bf16_from_float(master[i]);
                });
            }
            if (s >= warmup)
                times.push_back(
                    std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
        }
        const auto io1 = engine.stats();
        std::sort(times.begin(), times.end());
        *seconds = times[times.size() / 2];
        *io_bytes = static_cast<double>((io1.bytes_read - io0.bytes_read) +
                                        (io1.bytes_written - io0.bytes_written)) /
                    (warmup + steps);
        std::free(master);
        std::free(m);
        std::free(v);
    });
}

}  // extern "C"
