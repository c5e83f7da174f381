// bench-overflow: the reference CLI's fused-vs-staged overflow check report
// (proj/tools/memascend_cli.cpp:272-285, a caller of the hot path listed in
// SURVEY §8(b)), over memascend::bench_overflow.  Built against the
// reference's library (oracle/_ref/bench_overflow_ref: its CPU fused scan)
// and against ours (oracle/_ref/bench_overflow_ours: K1 on the B200 over the
// registered GradFlatBuffer) — the same CSV, so the two can be compared on
// the GPU box's own host.
//
//   ./bench_overflow [sizes=1000000,4000000,10000000] [workers=nproc] [repeats=5]
#include <cstdio>
#include <cstdlib>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "memascend/overflow.hpp"

using namespace memascend;

int main(int argc, char** argv) {
    std::vector<std::uint64_t> sizes{1000000, 4000000, 10000000};
    if (argc > 1) {
        sizes.clear();
        std::stringstream ss(argv[1]);
        std::string item;
        while (std::getline(ss, item, ',')) sizes.push_back(std::strtoull(item.c_str(), nullptr, 10));
    }
    ScanConfig cfg;
    cfg.worker_count = argc > 2 ? static_cast<std::uint32_t>(std::atoi(argv[2]))
                                : std::max(1u, std::thread::hardware_concurrency());
    const int repeats = argc > 3 ? std::atoi(argv[3]) : 5;
    try {
        const auto rows = bench_overflow(sizes, cfg, repeats);
        std::printf("size,fused_ns,naive_ns,naive_peak_extra_bytes,speedup\n");
        for (const auto& r : rows)
            std::printf("%llu,%llu,%llu,%llu,%g\n", (unsigned long long)r.elements,
                        (unsigned long long)r.fused_ns, (unsigned long long)r.naive_ns,
                        (unsigned long long)r.naive_peak_extra_bytes, r.speedup);
    } catch (const std::exception& e) {
        std::fprintf(stderr, "bench-overflow: %s\n", e.what());
        return 1;
    }
    return 0;
}
