// TEST INFRASTRUCTURE ONLY (never linked into the product).
//
// On-disk compatibility of the swap store, both directions.  The SAME source
// is compiled twice by oracle/Makefile:
//   oracle/_ref/xcompat_ref   against the reference's DirectIoEngine
//                             (proj/include/memascend/direct_io.hpp, proj/src/direct_io.cpp)
//   oracle/_ref/xcompat_ours  against ours (include/memascend/direct_io.hpp -> ma_swap_*)
// `write DIR` creates three file-backed devices, stores a set of tensors
// (ragged lengths, a shrink rewrite and a grow rewrite) and saves the
// manifest; `read DIR` reopens the devices with that manifest, restores every
// tensor and checks bytes, logical lengths, extents and the restored cursor.
// tests/test_swap.py runs ref->ours and ours->ref.
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "memascend/direct_io.hpp"

using namespace memascend;

namespace {

constexpr std::uint32_t kDevices = 3;
constexpr std::uint64_t kDevBytes = 32ull << 20;

struct Item {
    const char* key;
    std::uint64_t logical;
};
// final logical lengths; "grow" is first written at 4096 then grown,
// "shrink" first at 200000 then shrunk
const Item kItems[] = {{"master.block0", 1 << 20},  {"m.block0", (1 << 20) + 123},
                       {"v.block0", 5000},          {"w.embed", 4096},
                       {"key with spaces/\"q\"", 77}, {"grow", 300001},
                       {"shrink", 9000}};

std::uint64_t mix(std::uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

std::uint8_t byte_at(const char* key, std::uint64_t i) {
    std::uint64_t h = 1469598103934665603ull;
    for (const char* p = key; *p; ++p) h = (h ^ static_cast<unsigned char>(*p)) * 1099511628211ull;
    return static_cast<std::uint8_t>(mix(h + i / 8) >> (8 * (i % 8)));
}

std::byte* aligned(std::uint64_t bytes) {
    void* p = std::aligned_alloc(4096, (bytes + 4095) / 4096 * 4096);
    std::memset(p, 0, (bytes + 4095) / 4096 * 4096);
    return static_cast<std::byte*>(p);
}

void put(DirectIoEngine& e, const char* key, std::uint64_t logical) {
    const std::uint64_t padded = (logical + 4095) / 4096 * 4096;
    std::byte* b = aligned(padded);
    for (std::uint64_t i = 0; i < logical; ++i) b[i] = static_cast<std::byte>(byte_at(key, i));
    e.write_tensor(key, {b, padded}, logical);
    std::free(b);
}

DeviceSet devices(const std::string& dir) {
    DeviceSet s;
    for (std::uint32_t d = 0; d < kDevices; ++d)
        s.devices.push_back({dir + "/vdev" + std::to_string(d) + ".img", kDevBytes,
                             DeviceKind::file_backed_virtual});
    return s;
}

int fails = 0;
void expect(bool ok, const std::string& what) {
    if (!ok) {
        std::printf("FAIL %s\n", what.c_str());
        ++fails;
    }
}

}  // namespace

int main(int argc, char** argv) {
    if (argc != 3) {
        std::fprintf(stderr, "usage: %s write|read DIR\n", argv[0]);
        return 2;
    }
    const std::string mode = argv[1], dir = argv[2];
    EngineConfig cfg;
    cfg.manifest_path = dir + "/store.manifest.json";
    try {
        if (mode == "write") {
            DirectIoEngine::create_virtual_devices(dir, kDevices, kDevBytes);
            DirectIoEngine e(devices(dir), cfg);
            put(e, "grow", 4096);
            put(e, "shrink", 200000);
            for (const Item& it : kItems) put(e, it.key, it.logical);
            expect(e.stats().abandoned_bytes == 4096, "abandoned bytes after the grow rewrite");
            e.save_manifest();
        } else if (mode == "read") {
            DirectIoEngine e(devices(dir), cfg);
            const auto all = e.all_locations();
            expect(all.size() == sizeof kItems / sizeof kItems[0], "key count");
            std::uint64_t top[kDevices] = {0, 0, 0};
            for (const auto& kv : all)
                for (const Extent& x : kv.second.extents)
                    top[x.device_index] = std::max(top[x.device_index], x.device_offset + x.length);
            for (const Item& it : kItems) {
                const TensorLocation loc = e.location(it.key);
                expect(loc.logical_length == it.logical, std::string("logical length of ") + it.key);
                std::byte* b = aligned(loc.padded_length);
                const std::uint64_t got = e.read_tensor(it.key, {b, loc.padded_length});
                expect(got == it.logical, std::string("read length of ") + it.key);
                bool same = true;
                for (std::uint64_t i = 0; i < it.logical && same; ++i)
                    same = static_cast<std::uint8_t>(b[i]) == byte_at(it.key, i);
                expect(same, std::string("payload of ") + it.key);
                std::free(b);
            }
            // the cursors were restored: fresh space lies past every stored extent
            const auto fresh = e.allocate_extents("after-restart", 3 * 4096);
            for (const Extent& x : fresh)
                expect(x.device_offset >= top[x.device_index], "cursor restored");
        } else {
            return 2;
        }
    } catch (const std::exception& ex) {
        std::printf("FAIL exception: %s\n", ex.what());
        return 1;
    }
    std::printf("%s %s: %s\n", argv[0], mode.c_str(), fails ? "FAILED" : "ok");
    return fails ? 1 : 0;
}
