// bench-pool: the pool capacity / fragmentation report of the reference's CLI
// (proj/tools/memascend_cli.cpp:186-268), over this
// library's drop-in Pool (registered host backing) and — when a GPU is
// present — its device-side DevicePool (HBM backing, same class plan).
//
//   g++ -std=c++20 -O2 -Iinclude tools/bench_pool.cpp -o bench_pool \
//       -Lpaper_2505_23254_b200/lib -lmemascend -lmemascend_b200 \
//       -Wl,-rpath,$PWD/paper_2505_23254_b200/lib
//   ./bench_pool <preset|model.json> [inflight=1] [max_backing_gib=3]
//
// Rows per mode (monolithic, adaptive): capacity_bytes, and either a live
// replay of the trainer's prefetch/hold pattern (backing, peak live,
// fragmentation, checkouts, blocked ms) or, above the backing budget, the
// analytic peak-live prediction — the reference's rules.  Device rows report
// the HBM a DevicePool of the same plan reserves.  Built with
// -DMA_REFERENCE_BUILD against the reference's own library (oracle/Makefile,
// test infrastructure) it prints the reference's host rows, which
// tests/test_swap.py compares with ours.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#ifndef MA_REFERENCE_BUILD
#include "memascend/device_pool.hpp"
#endif
#include "memascend/error.hpp"
#include "memascend/model.hpp"
#include "memascend/pool.hpp"

using namespace memascend;

int main(int argc, char** argv) {
    if (argc < 2) {
        std::fprintf(stderr, "usage: %s <preset|model.json> [inflight] [max_backing_gib]\n", argv[0]);
        return 2;
    }
    const std::string ref = argv[1];
    const std::uint64_t inflight = argc > 2 ? std::strtoull(argv[2], nullptr, 10) : 1;  // CLI defaults
    const double max_gib = argc > 3 ? std::atof(argv[3]) : 3.0;
    try {
        ModelSpec spec;
        bool is_preset = false;
        for (const auto& p : preset_names()) is_preset |= p == ref;
        spec = is_preset ? preset(ref) : load_model_spec(ref);
        const auto inv = enumerate_offload_tensors(spec, 1);
        std::printf("{\"cmd\": \"bench-pool\", \"model\": \"%s\", \"inflight_blocks\": %llu, \"rows\": [",
                    spec.name.c_str(), (unsigned long long)inflight);
        bool first = true;
        for (PoolMode mode : {PoolMode::monolithic, PoolMode::adaptive}) {
            const char* name = mode == PoolMode::monolithic ? "monolithic" : "adaptive";
            const std::uint64_t cap = pool_capacity(inv, mode, inflight);
            std::printf("%s\n  {\"mode\": \"%s\", \"tier\": \"host\", \"capacity_bytes\": %llu", first ? "" : ",",
                        name, (unsigned long long)cap);
            first = false;
            bool replayed = false;
            if (static_cast<double>(cap) / (1ull << 30) <= max_gib) try {
                PoolConfig cfg;
                cfg.mode = mode;
                cfg.inflight_blocks = inflight;
                Pool pool(inv, cfg);
                std::vector<BufferHandle> step_held, block_held;
                std::string current;
                for (const auto& t : inv) {
                    auto h = pool.checkout(t.name, tensor_bytes(t));
                    if (!is_per_layer_role(t.role)) {
                        step_held.push_back(h);
                        continue;
                    }
                    const std::string group = t.name.substr(0, t.name.find('.'));
                    if (group != current && !block_held.empty()) {
                        for (auto& b : block_held) pool.checkin(b);
                        block_held.clear();
                    }
                    current = group;
                    block_held.push_back(h);
                }
                for (auto& b : block_held) pool.checkin(b);
                for (auto& b : step_held) pool.checkin(b);
                const PoolStats st = pool.stats();
                std::printf(", \"replayed\": true, \"backing_bytes\": %llu, \"peak_live_bytes\": %llu, "
                            "\"fragmentation\": %.6f, \"checkout_count\": %llu, \"blocked_ms\": %.3f}",
                            (unsigned long long)st.backing_bytes, (unsigned long long)st.peak_live_bytes,
                            fragmentation(st.capacity_bytes, st.peak_live_bytes),
                            (unsigned long long)st.checkout_count,
                            std::chrono::duration<double, std::milli>(st.blocked_time).count());
                replayed = true;
            } catch (const Error& e) {
                if (e.code() != ErrorCode::pool_exhausted) throw;
                // the hold pattern needs >= 2 blocks in flight in this mode
                std::printf(", \"replay_error\": \"pool-exhausted\"");
            }
            if (!replayed) {
                // analytic: every slot holding an exact payload at the deepest point
                std::uint64_t peak = 0;
                if (mode == PoolMode::adaptive) {
                    peak = cap;
                } else {
                    std::uint64_t per_block = 0, layers = 0;
                    for (const auto& t : inv) {
                        if (!is_per_layer_role(t.role)) peak += tensor_bytes(t);
                        if (t.name.rfind("layer0.", 0) == 0) per_block += tensor_bytes(t);
                        if (t.name.rfind("layer", 0) == 0)
                            layers = std::max<std::uint64_t>(
                                layers, std::stoull(t.name.substr(5, t.name.find('.') - 5)) + 1);
                    }
                    peak += per_block * std::min<std::uint64_t>(inflight, layers);
                }
                std::printf(", \"replayed\": false, \"peak_live_bytes\": %llu, \"fragmentation\": %.6f}",
                            (unsigned long long)peak, fragmentation(cap, peak));
            }
#ifndef MA_REFERENCE_BUILD
            // the same plan in HBM (needs a GPU; skipped without one)
            try {
                DevicePool dp(inv, mode, inflight);
                const PoolStats ds = dp.stats();
                std::printf(",\n  {\"mode\": \"%s\", \"tier\": \"device\", \"capacity_bytes\": %llu, "
                            "\"backing_bytes\": %llu}",
                            name, (unsigned long long)ds.capacity_bytes,
                            (unsigned long long)ds.backing_bytes);
            } catch (const Error& e) {
                if (e.code() != ErrorCode::device_error && e.code() != ErrorCode::out_of_memory) throw;
            }
#endif
        }
        std::printf("\n]}\n");
    } catch (const std::exception& e) {
        std::fprintf(stderr, "bench-pool: %s\n", e.what());
        return 1;
    }
    return 0;
}
