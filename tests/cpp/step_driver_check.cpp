// C++ check of include/memascend/step_driver.hpp on the B200 (built and run by
// tests/test_gpu_prefetch.py): the reference's configs workload case
// cfg_bf16_n100003 (tests/golden/workload.json) through memascend::StepDriver
// — generators from the C ABI, K1 -> K2 -> scaler per step — once over
// HBM-resident sub-groups and once with every sub-group's state in a
// DirectIoEngine store (apply_swapped).  Further modes, same golden digests:
//   nccl    the cross-rank decision through the library's NCCL communicator
//           (world 1: Communicator + StepDriver::exchange between K1 and K2);
//   graph   check -> exchange -> apply -> finish captured once into a CUDA
//           graph and replayed every step (gradients produced outside it);
//   resume  three steps, then a NEW StepDriver built from the saved
//           LossScaler and step_t continues the run (checkpoint/restart).
// Prints the final FNV-1a digests of p/m/v/w, the scale and t; the test
// compares them with the golden values.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "memascend/direct_io.hpp"
#include "memascend/step_driver.hpp"

using namespace memascend;

static std::uint64_t fnv(const void* p, size_t n) {
    std::uint64_t h = 1469598103934665603ull;
    const auto* b = static_cast<const unsigned char*>(p);
    for (size_t i = 0; i < n; ++i) h = (h ^ b[i]) * 1099511628211ull;
    return h;
}

static float f(std::uint32_t u) {
    float x;
    std::memcpy(&x, &u, 4);
    return x;
}

int main(int argc, char** argv) {
    if (argc < 3) return 2;
    const std::string mode = argv[1];
    const bool swapped = mode == "swapped";
    const std::string dir = argv[2];
    const std::uint64_t n = 100003, sub = 30000, seed = 1;
    AdamHyper h;
    h.lr = f(981668463u);
    h.beta1 = f(1063675494u);
    h.beta2 = f(1065336439u);
    h.eps = f(841731191u);
    h.weight_decay = f(1008981770u);
    try {
        float *p, *m, *v;
        uint16_t *g, *w;
        cudaMalloc(&p, n * 4);
        cudaMalloc(&m, n * 4);
        cudaMalloc(&v, n * 4);
        cudaMalloc(&g, n * 2);
        cudaMalloc(&w, n * 2);
        cudaMemset(m, 0, n * 4);
        cudaMemset(v, 0, n * 4);
        cudaStream_t st, h2d, d2h;
        cudaStreamCreate(&st);
        cudaStreamCreate(&h2d);
        cudaStreamCreate(&d2h);
        if (ma_gen_seeded_weights_async(p, w, MA_DT_BF16, n, 0, seed, st)) return 3;
        auto drv_ptr = std::make_unique<StepDriver>(h, LossScaler{}, MA_DT_BF16, MA_DT_BF16);
        std::unique_ptr<Communicator> comm;
        if (mode == "nccl" || mode == "graph")
            comm = std::make_unique<Communicator>(1, 0, Communicator::unique_id());
        std::vector<ma_subgroup> groups;
        for (std::uint64_t o = 0; o < n; o += sub) {
            const std::uint64_t k = std::min(sub, n - o);
            groups.push_back({p + o, m + o, v + o, g + o, w + o, k});
        }
        // swapped form: the state of every sub-group in the store
        const std::uint64_t slot = 32768, tb = slot * 4;
        DeviceSet devs;
        DirectIoEngine* store = nullptr;
        std::vector<ma_swap_group> sg;
        std::vector<std::string> keys;
        void* hstage = nullptr;
        float* dstage = nullptr;
        if (swapped) {
            devs = DirectIoEngine::create_virtual_devices(dir, 2, 8 << 20);
            store = new DirectIoEngine(devs, {});
            void* buf = std::aligned_alloc(4096, tb);
            cudaStreamSynchronize(st);
            for (size_t k = 0; k < groups.size(); ++k) {
                const char* names[3] = {"master", "m", "v"};
                float* src[3] = {groups[k].p, groups[k].m, groups[k].v};
                for (int t = 0; t < 3; ++t) {
                    cudaMemcpy(buf, src[t], groups[k].n * 4, cudaMemcpyDeviceToHost);
                    keys.push_back(std::string(names[t]) + ".g" + std::to_string(k));
                    store->write_tensor(keys.back(), {static_cast<std::byte*>(buf), tb},
                                        groups[k].n * 4);
                }
            }
            std::free(buf);
            for (size_t k = 0; k < groups.size(); ++k)
                sg.push_back({keys[3 * k].c_str(), keys[3 * k + 1].c_str(), keys[3 * k + 2].c_str(),
                              nullptr, nullptr, nullptr, groups[k].g, groups[k].w, groups[k].n});
            hstage = std::aligned_alloc(4096, 2 * 3 * tb);
            if (ma_host_register(hstage, 2 * 3 * tb)) return 4;
            cudaMalloc(&dstage, 2 * 3 * slot * 4);
        }
        SwapStaging staging{hstage, 2, dstage, 2, slot, h2d, d2h};
        std::unique_ptr<StepGraph> graph;
        if (mode == "graph") {
            StepDriver& d = *drv_ptr;
            d.capture_begin(st, 16);
            d.check(g, n, st);
            d.exchange(*comm, st);
            d.apply(groups, st);
            d.finish(st);
            graph = std::make_unique<StepGraph>(d.capture_end(st));
        }
        for (std::uint64_t s = 0; s < 6; ++s) {
            if (mode == "resume" && s == 3) {
                // checkpoint: the scaler and t; p/m/v/w stay where they are
                const LossScaler saved = drv_ptr->scaler();
                const std::uint64_t step_t = drv_ptr->updates();
                drv_ptr = std::make_unique<StepDriver>(h, saved, MA_DT_BF16, MA_DT_BF16, step_t);
            }
            StepDriver& drv = *drv_ptr;
            ma_gen_pseudo_grads_async(g, MA_DT_BF16, w, MA_DT_BF16, n, 0, seed, s,
                                      ma_stepper_scale(drv.handle()), 0.0f, st);
            if (s == 2) ma_plant_bits_async(g, MA_DT_BF16, 777, 32704, st);
            if (s == 4) ma_plant_bits_async(g, MA_DT_BF16, 100002, 32639, st);
            if (graph) {
                graph->launch(st);
                continue;
            }
            drv.check(g, n, st);
            if (comm) drv.exchange(*comm, st);
            if (swapped)
                drv.apply_swapped(*store, sg, staging, st);
            else
                drv.apply(groups, st);
            drv.finish(st);
        }
        StepDriver& drv = *drv_ptr;
        cudaStreamSynchronize(st);
        std::vector<float> hp(n), hm(n), hv(n);
        std::vector<uint16_t> hw(n);
        if (swapped) {
            void* buf = std::aligned_alloc(4096, tb);
            std::vector<float>* dst[3] = {&hp, &hm, &hv};
            for (size_t k = 0; k < groups.size(); ++k)
                for (int t = 0; t < 3; ++t) {
                    store->read_tensor(keys[3 * k + t], {static_cast<std::byte*>(buf), tb});
                    std::memcpy(dst[t]->data() + (groups[k].p - p), buf, groups[k].n * 4);
                }
            std::free(buf);
        } else {
            cudaMemcpy(hp.data(), p, n * 4, cudaMemcpyDeviceToHost);
            cudaMemcpy(hm.data(), m, n * 4, cudaMemcpyDeviceToHost);
            cudaMemcpy(hv.data(), v, n * 4, cudaMemcpyDeviceToHost);
        }
        cudaMemcpy(hw.data(), w, n * 2, cudaMemcpyDeviceToHost);
        const LossScaler sc = drv.scaler();
        std::printf("p %016llx\nm %016llx\nv %016llx\nw %016llx\nscale %.1f\nupdates %llu\n",
                    (unsigned long long)fnv(hp.data(), n * 4), (unsigned long long)fnv(hm.data(), n * 4),
                    (unsigned long long)fnv(hv.data(), n * 4), (unsigned long long)fnv(hw.data(), n * 2),
                    sc.scale, (unsigned long long)drv.updates());
        if (swapped) {
            ma_host_unregister(hstage);
            std::free(hstage);
            delete store;
        }
    } catch (const std::exception& e) {
        std::printf("FAIL exception: %s\n", e.what());
        return 1;
    }
    return 0;
}
