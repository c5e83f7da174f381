// C++ check of include/memascend/device_pool.hpp on the B200 (built and run by
// tests/test_gpu_prefetch.py): the reference's own model inventory drives the
// HBM pool's class plan, and a toy model's weights stream store -> HBM
// through WeightPrefetcher in consumption order with the prefetch/hold
// pattern of simulator.cpp:367-425, compared byte for byte.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "memascend/device_pool.hpp"
#include "memascend/direct_io.hpp"
#include "memascend/model.hpp"
#include "memascend/pool.hpp"

using namespace memascend;

static int fails = 0;
#define EXPECT(c)                                                      \
    do {                                                               \
        if (!(c)) {                                                    \
            std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #c);    \
            ++fails;                                                   \
        }                                                              \
    } while (0)

int main(int argc, char** argv) {
    const std::string dir = argc > 1 ? argv[1] : "/tmp/ma_dpool_check";
    try {
        // 1. class plan = the reference Pool's, for a real inventory
        const auto inv8b = enumerate_offload_tensors(preset("llama3.1-8b"), 1);
        for (PoolMode mode : {PoolMode::adaptive, PoolMode::monolithic}) {
            DevicePool dp(inv8b, mode, 2);
            const PoolStats s = dp.stats();
            EXPECT(s.capacity_bytes == pool_capacity(inv8b, mode, 2));
            EXPECT(s.live_bytes == 0 && s.checkout_count == 0);
            std::printf("llama3.1-8b %s: %zu classes, capacity %llu, backing %llu\n",
                        mode == PoolMode::adaptive ? "adaptive" : "monolithic", dp.classes().size(),
                        (unsigned long long)s.capacity_bytes, (unsigned long long)s.backing_bytes);
        }
        // 2. stream a toy model's tensors through the pipeline
        const auto inv = enumerate_offload_tensors(preset("toy-dense"), 1);
        auto devs = DirectIoEngine::create_virtual_devices(dir, 2, 16 << 20);
        DirectIoEngine store(devs, {});
        std::vector<std::vector<unsigned char>> data;
        std::uint64_t biggest = 0;
        for (size_t k = 0; k < inv.size(); ++k) {
            const std::uint64_t nb = tensor_bytes(inv[k]);
            biggest = std::max(biggest, nb);
            const std::uint64_t padded = (nb + 4095) / 4096 * 4096;
            auto* buf = static_cast<unsigned char*>(std::aligned_alloc(4096, padded));
            data.emplace_back(nb);
            for (std::uint64_t i = 0; i < nb; ++i) data[k][i] = buf[i] = static_cast<unsigned char>(k * 131 + i * 7);
            store.write_tensor(inv[k].name, {reinterpret_cast<std::byte*>(buf), padded}, nb);
            std::free(buf);
        }
        DevicePool pool(inv, PoolMode::adaptive, 1);
        WeightPrefetcher pf(store, pool, 2, biggest);
        for (const auto& t : inv) pf.submit(t.name);
        cudaStream_t st;
        cudaStreamCreate(&st);
        // the trainer's hold pattern (simulator.cpp:384-401): a block's
        // tensors are checked in once the whole block has been consumed
        std::map<std::string, size_t> block_size;
        for (const auto& t : inv)
            if (is_per_layer_role(t.role)) block_size[t.name.substr(0, t.name.find('.'))] += 1;
        std::vector<std::string> held, step_held;
        for (size_t k = 0; k < inv.size(); ++k) {
            const auto& t = inv[k];
            std::uint64_t nb = 0;
            void* d = pf.acquire(t.name, st, &nb);
            EXPECT(nb == data[k].size());
            std::vector<unsigned char> back(nb);
            cudaMemcpyAsync(back.data(), d, nb, cudaMemcpyDeviceToHost, st);
            cudaStreamSynchronize(st);
            EXPECT(std::memcmp(back.data(), data[k].data(), nb) == 0);
            if (!is_per_layer_role(t.role)) {
                step_held.push_back(t.name);
                continue;
            }
            held.push_back(t.name);
            if (held.size() == block_size[t.name.substr(0, t.name.find('.'))]) {
                for (auto& h : held) pf.release(h, st);
                held.clear();
            }
        }
        for (auto& h : held) pf.release(h, st);
        for (auto& h : step_held) pf.release(h, st);
        cudaStreamSynchronize(st);
        const PoolStats s = pool.stats();
        EXPECT(s.checkout_count == inv.size() && s.checkin_count == inv.size());
        EXPECT(s.live_bytes == 0);
        EXPECT(s.peak_live_bytes <= s.capacity_bytes);
        std::printf("toy-dense: %zu tensors streamed, peak live %llu of %llu\n", inv.size(),
                    (unsigned long long)s.peak_live_bytes, (unsigned long long)s.capacity_bytes);
        cudaStreamDestroy(st);
    } catch (const std::exception& e) {
        std::printf("FAIL exception: %s\n", e.what());
        return 1;
    }
    std::printf("%s\n", fails ? "FAILED" : "ok");
    return fails ? 1 : 0;
}
