// bench-io: the reference CLI's storage report (proj/tools/memascend_cli.cpp:
// 288-360): DirectIoEngine vs the one-file-per-tensor FsBaselineStore, median
// write/read times per payload size.  Built against the reference's library
// (oracle/_ref/bench_io_ref: its pread/pwrite / POSIX-AIO engine) and against
// ours (oracle/_ref/bench_io_ours: the io_uring engine via auto_probe) — the
// same CSV, so the engines can be compared on one box's disk.
//
//   ./bench_io [sizes=4096,65536,1048576,8388608] [workers=2] [queue_depth=8]
//              [repeats=5] [devices=2] [vdev_mib=1024]
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <filesystem>
#include <sstream>
#include <string>
#include <vector>

#include <unistd.h>

#include "memascend/direct_io.hpp"
#include "memascend/pinned.hpp"

using namespace memascend;

int main(int argc, char** argv) {
    std::vector<std::uint64_t> sizes{4096, 65536, 1 << 20, 8 << 20};
    if (argc > 1) {
        sizes.clear();
        std::stringstream ss(argv[1]);
        std::string it;
        while (std::getline(ss, it, ',')) sizes.push_back(std::strtoull(it.c_str(), nullptr, 10));
    }
    EngineConfig ecfg;
    ecfg.workers = argc > 2 ? std::atoi(argv[2]) : 2;
    ecfg.queue_depth = argc > 3 ? std::atoi(argv[3]) : 8;
    const int repeats = argc > 4 ? std::atoi(argv[4]) : 5;
    const std::uint32_t devices = argc > 5 ? std::atoi(argv[5]) : 2;
    std::uint64_t vdev = (argc > 6 ? std::strtoull(argv[6], nullptr, 10) : 1024) << 20;
    for (auto s : sizes) vdev = std::max<std::uint64_t>(vdev, (2 * s / devices + (8 << 20)) / 4096 * 4096);
    const auto scratch = std::filesystem::temp_directory_path() /
                         ("memascend-bench-io-" + std::to_string(::getpid()));
    try {
        auto devset = DirectIoEngine::create_virtual_devices((scratch / "dev").string(), devices, vdev);
        DirectIoEngine engine(devset, ecfg);
        FsBaselineStore fs((scratch / "fs").string());
        auto& alloc = PinnedAllocator::global();
        std::printf("size,direct_write_ns,fs_write_ns,direct_read_ns,fs_read_ns,write_speedup,"
                    "direct_write_gbs,direct_read_gbs\n");
        for (const std::uint64_t size : sizes) {
            auto payload = alloc.allocate(size, {AllocPolicyKind::alignment_free});
            auto dst = alloc.allocate(size, {AllocPolicyKind::alignment_free});
            auto span = payload.bytes();
            for (std::uint64_t i = 0; i < size; ++i) span[i] = static_cast<std::byte>(i * 31 + 7);
            auto median = [&](auto&& fn) {
                std::vector<std::uint64_t> ns;
                for (int r = 0; r < repeats; ++r) {
                    const auto t0 = std::chrono::steady_clock::now();
                    fn();
                    ns.push_back(std::chrono::duration_cast<std::chrono::nanoseconds>(
                                     std::chrono::steady_clock::now() - t0)
                                     .count());
                }
                std::sort(ns.begin(), ns.end());
                return ns[ns.size() / 2];
            };
            const std::string key = "bench-" + std::to_string(size);
            engine.write_tensor(key, payload.bytes(), size);  // extents claimed once
            fs.write(key, payload.bytes(), size);
            const auto dw = median([&] { engine.write_tensor(key, payload.bytes(), size); });
            const auto fw = median([&] { fs.write(key, payload.bytes(), size); });
            const auto dr = median([&] { engine.read_tensor(key, dst.bytes()); });
            const auto fr = median([&] { fs.read(key, dst.bytes()); });
            std::printf("%llu,%llu,%llu,%llu,%llu,%g,%.3f,%.3f\n", (unsigned long long)size,
                        (unsigned long long)dw, (unsigned long long)fw, (unsigned long long)dr,
                        (unsigned long long)fr, dw ? static_cast<double>(fw) / dw : 0.0,
                        size / static_cast<double>(dw), size / static_cast<double>(dr));
            alloc.release(payload);
            alloc.release(dst);
        }
    } catch (const std::exception& e) {
        std::fprintf(stderr, "bench-io: %s\n", e.what());
        std::error_code ec;
        std::filesystem::remove_all(scratch, ec);
        return 1;
    }
    std::error_code ec;
    std::filesystem::remove_all(scratch, ec);
    return 0;
}
