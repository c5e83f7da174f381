// ORACLE — TEST INFRASTRUCTURE ONLY.
//
// Generates tests/golden/*.json from the UNMODIFIED reference (compiled from
// /root/reference/proj by oracle/Makefile).  Driven by
// tests/golden/make_golden.py; the fixtures are committed so the GPU box,
// which has no /root/reference, can check against them.
//
// The adversarial-buffer generator is taken from the reference test itself by
// compiling proj/tests/test_overflow.cpp into this translation unit (its
// TEST_CASEs register with the doctest shim and are simply not run here).
#include "test_overflow.cpp"  // NOLINT: reference test TU, provides adversarial_buffer()
#include "reference_trainer.hpp"

#include <cinttypes>
#include <array>
#include <cstdio>
#include <fstream>
#include <nlohmann/json.hpp>

#include "memascend/halfprec.hpp"
#include "memascend/optimizer.hpp"
#include "memascend/simulator.hpp"

using nlohmann::json;

namespace {

std::string hex64(std::uint64_t v) {
    char b[17];
    std::snprintf(b, sizeof b, "%016" PRIx64, v);
    return b;
}

std::uint64_t fnv(const void* data, std::size_t bytes, std::uint64_t h = 1469598103934665603ull) {
    const auto* p = static_cast<const unsigned char*>(data);
    for (std::size_t i = 0; i < bytes; ++i) {
        h ^= p[i];
        h *= 1099511628211ull;
    }
    return h;
}

template <typename T>
std::string fnv_vec(const std::vector<T>& v) {
    return hex64(fnv(v.data(), v.size() * sizeof(T)));
}

json f32_bits_list(const std::vector<float>& v) {
    json a = json::array();
    for (float f : v) a.push_back(float_bits(f));
    return a;
}

void write(const std::string& dir, const std::string& name, const json& j) {
    std::ofstream(dir + "/" + name) << j.dump(1) << "\n";
    std::printf("wrote %s/%s\n", dir.c_str(), name.c_str());
}

// test_overflow.cpp:106-145 — decisions of the reference fused check on the
// reference's adversarial generator, plus buffer digests that pin the
// generator's draw order for the restated one.
json adversarial() {
    json out;
    std::mt19937_64 rng(99);
    json rounds = json::array();
    for (int round = 0; round < 300; ++round) {
        const std::size_t n = 1 + rng() % 4096;
        const bool inject = rng() % 2 == 0;
        auto host = adversarial_buffer(rng, n, inject);
        ScanConfig cfg;
        cfg.worker_count = 1 + rng() % 4;
        cfg.chunk_bytes = 4 * (1 + rng() % 512);
        cfg.early_exit = rng() % 2 == 0;
        ScanConfig dbg;
        dbg.track_first_index = true;
        dbg.early_exit = false;
        const auto r = fused_overflow_check(std::span<const float>(host), cfg);
        const auto rf = fused_overflow_check(std::span<const float>(host), dbg);
        rounds.push_back({{"n", n},
                          {"inject", inject},
                          {"workers", cfg.worker_count},
                          {"chunk_bytes", cfg.chunk_bytes},
                          {"early_exit", cfg.early_exit},
                          {"fnv", fnv_vec(host)},
                          {"overflow", r.overflow},
                          {"first_index", rf.first_offending_index.has_value()
                                              ? json(*rf.first_offending_index)
                                              : json(nullptr)}});
    }
    out["seed"] = 99;
    out["rounds"] = rounds;

    std::mt19937_64 rng5(5);
    auto host = adversarial_buffer(rng5, 100000, true);
    out["determinism"] = {{"seed", 5},
                          {"n", 100000},
                          {"fnv", fnv_vec(host)},
                          {"overflow",
                           fused_overflow_check(std::span<const float>(host),
                                                ScanConfig{1, 1 << 20, false, false})
                               .overflow}};
    return out;
}

// test_overflow.cpp:85-104
json nan_index() {
    std::mt19937_64 rng(11);
    std::vector<float> vals(1000000);
    for (auto& x : vals) x = static_cast<float>(rng() % 1000) * 0.5f - 250.0f;
    const std::uint64_t where = rng() % vals.size();
    const std::uint32_t bits = 0x7F800001u;
    std::memcpy(&vals[where], &bits, 4);
    ScanConfig dbg;
    dbg.track_first_index = true;
    dbg.early_exit = false;
    const auto r = fused_overflow_check(std::span<const float>(vals), dbg);
    return {{"seed", 11},
            {"n", vals.size()},
            {"where", where},
            {"fnv", fnv_vec(vals)},
            {"overflow", r.overflow},
            {"first_index", *r.first_offending_index}};
}

// test_optimizer.cpp:29-98 known answers, run through the reference.
json adam_kat() {
    json out;
    {
        AdamHyper h;
        h.lr = 0.1f;
        std::vector<float> p{1.0f}, m{0.0f}, v{0.0f}, g{1.0f};
        adam_step_fp32(p, m, v, g, 1, h, 1.0f);
        out["closed_form"] = {{"p", float_bits(p[0])}, {"m", float_bits(m[0])}, {"v", float_bits(v[0])}};
    }
    {
        AdamHyper h;
        h.lr = 0.01f;
        h.weight_decay = 0.1f;
        std::vector<float> p{4.0f}, m{0.0f}, v{0.0f}, g{0.0f};
        adam_step_fp32(p, m, v, g, 1, h, 1.0f);
        out["decay"] = {{"p", float_bits(p[0])}, {"m", float_bits(m[0])}};
    }
    // 257 params, seed 31, lr 3e-3, wd 0.01, scale 1024, 100 steps (:61-98).
    std::mt19937_64 rng(31);
    constexpr std::size_t n = 257;
    std::vector<float> p(n), m(n, 0.0f), v(n, 0.0f), g(n);
    for (auto& x : p) x = static_cast<float>(rng() % 2048) / 256.0f - 4.0f;
    const std::vector<float> p0 = p;
    AdamHyper h;
    h.lr = 3e-3f;
    h.weight_decay = 0.01f;
    const float scale = 1024.0f;
    json per_step = json::array();
    json grads_fnv = json::array();
    for (std::uint64_t t = 1; t <= 100; ++t) {
        for (auto& x : g) x = (static_cast<float>(rng() % 65536) / 32768.0f - 1.0f) * scale;
        grads_fnv.push_back(fnv_vec(g));
        adam_step_fp32(p, m, v, g, t, h, scale, 2);
        std::uint64_t d = fnv(p.data(), n * 4);
        d = fnv(m.data(), n * 4, d);
        d = fnv(v.data(), n * 4, d);
        per_step.push_back(hex64(d));
    }
    out["random100"] = {{"seed", 31},     {"n", n},          {"steps", 100},
                        {"lr", float_bits(h.lr)}, {"wd", float_bits(h.weight_decay)},
                        {"scale", scale}, {"p0_fnv", fnv_vec(p0)}, {"grads_fnv", grads_fnv},
                        {"per_step_pmv_fnv", per_step},
                        {"final_p", f32_bits_list(p)}, {"final_m", f32_bits_list(m)},
                        {"final_v", f32_bits_list(v)}};
    // bc table for t = 1..4096 under the default betas (glibc powf).
    json bc = json::array();
    for (std::uint64_t t = 1; t <= 4096; ++t) {
        const float b1 = 1.0f - std::pow(0.9f, static_cast<float>(t));
        const float b2 = 1.0f - std::pow(0.999f, static_cast<float>(t));
        bc.push_back({float_bits(b1), float_bits(b2)});
    }
    out["bc_default_betas"] = bc;
    return out;
}

json halfprec() {
    constexpr int kLog2 = 20;
    const std::uint64_t nb = 1ull << (32 - kLog2);
    json out;
    out["block_log2"] = kLog2;
    for (int kind : {1, 2}) {
        std::vector<std::uint64_t> sums(nb);
        std::atomic<std::uint64_t> next{0};
        auto worker = [&] {
            for (;;) {
                const std::uint64_t b = next.fetch_add(1);
                if (b >= nb) return;
                std::uint64_t hsh = 1469598103934665603ull;
                for (std::uint64_t k = 0; k < (1ull << kLog2); ++k) {
                    const float f = bits_float(static_cast<std::uint32_t>((b << kLog2) + k));
                    const std::uint16_t r = kind == 1 ? bf16_from_float(f) : fp16_from_float(f);
                    hsh = fnv(&r, 2, hsh);
                }
                sums[b] = hsh;
            }
        };
        std::vector<std::thread> th;
        for (unsigned t = 1; t < std::max(1u, std::thread::hardware_concurrency()); ++t)
            th.emplace_back(worker);
        worker();
        for (auto& t : th) t.join();
        json a = json::array();
        for (auto s : sums) a.push_back(hex64(s));
        out[kind == 1 ? "bf16_from_float" : "fp16_from_float"] = a;
    }
    std::vector<float> f16(65536), b16(65536);
    for (std::uint32_t hh = 0; hh < 65536; ++hh) {
        f16[hh] = fp16_to_float(static_cast<std::uint16_t>(hh));
        b16[hh] = bf16_to_float(static_cast<std::uint16_t>(hh));
    }
    out["fp16_to_float_fnv"] = fnv_vec(f16);
    out["bf16_to_float_fnv"] = fnv_vec(b16);
    return out;
}

// test_simulator.cpp:35-89 — reference run_training vs reference_train.
json trainer() {
    json cases = json::array();
    struct Case {
        const char* name;
        std::uint64_t steps;
        std::uint64_t seed;
        bool bf16;
        std::int64_t fault_step;
        std::uint64_t fault_index;
        std::uint32_t fault_bits;
    };
    const Case list[] = {
        {"mixed_seed7_10", 10, 7, false, -1, 0, 0},
        {"bf16_seed7_8", 8, 7, true, -1, 0, 0},
        {"mixed_fault3_inf", 6, 7, false, 3, 0, 0x7F800000u},
        {"mixed_fault1_qnan", 3, 7, false, 1, 0, 0x7FC00000u},
        {"mixed_seed8_5", 5, 8, false, -1, 0, 0},
    };
    std::uint64_t n = 0;
    for (const auto& c : list) {
        SimConfig cfg;
        cfg.model = preset("toy-dense");
        cfg.steps = c.steps;
        cfg.seed = c.seed;
        cfg.device_bytes = 32ull << 20;
        cfg.precision = c.bf16 ? OptimPrecision::pure_bf16 : OptimPrecision::mixed_fp16_fp32master;
        if (c.fault_step >= 0)
            cfg.fault = FaultInjection{static_cast<std::uint64_t>(c.fault_step), c.fault_index, c.fault_bits};
        const auto rep = run_training(cfg);
        const auto ref = testing::reference_train(cfg);
        n = c.bf16 ? ref.weights.size() : ref.master.size();
        json steps_scale = json::array();
        for (const auto& s : rep.per_step) steps_scale.push_back(s.scale_after);
        cases.push_back({{"name", c.name},
                         {"steps", c.steps},
                         {"seed", c.seed},
                         {"pure_bf16", c.bf16},
                         {"fault", c.fault_step >= 0 ? json({{"step", c.fault_step},
                                                              {"index", c.fault_index},
                                                              {"bits", c.fault_bits}})
                                                     : json(nullptr)},
                         {"sim_digest", rep.master_digest},
                         {"ref_digest", testing::reference_digest(ref, !c.bf16)},
                         {"final_scale", rep.final_scale},
                         {"scale_after", steps_scale},
                         {"overflow_steps", rep.overflow_steps}});
    }
    return {{"preset", "toy-dense"}, {"n", n}, {"cases", cases}};
}

// The BASELINE configs' workload, composed from the reference's own functions
// exactly as simulator.cpp:427-492 composes them: pseudo-gradients scaled and
// stored (bf16 or fp32), faults planted, ONE fused check over the whole flat
// buffer, then per sub-group adam_step_fp32 and the working-weight refresh.
json workload_case(const std::string& name, std::uint64_t n, std::uint64_t steps,
                   std::uint64_t seed, bool g_bf16, bool w_bf16, std::uint64_t subgroup,
                   std::uint32_t growth, const std::vector<std::array<std::uint64_t, 3>>& faults,
                   float wd) {
    AdamHyper h;
    h.lr = 1e-3f;
    h.weight_decay = wd;
    LossScaler sc;
    sc.growth_interval = growth;
    std::vector<float> p(n), m(n, 0.0f), v(n, 0.0f), flat(n);
    std::vector<std::uint16_t> w(n), gb(n);
    for (std::uint64_t i = 0; i < n; ++i) {
        p[i] = seeded_weight(seed, i);
        w[i] = w_bf16 ? bf16_from_float(p[i]) : fp16_from_float(p[i]);
    }
    json per = json::array();
    std::uint64_t updates = 0;
    for (std::uint64_t s = 0; s < steps; ++s) {
        for (std::uint64_t i = 0; i < n; ++i) {
            const float wf = w_bf16 ? bf16_to_float(w[i]) : fp16_to_float(w[i]);
            const float gs = pseudo_gradient(seed, s, i, wf) * sc.scale;
            if (g_bf16) {
                gb[i] = bf16_from_float(gs);
            } else {
                flat[i] = gs;
            }
        }
        for (const auto& f : faults) {
            if (f[0] != s) continue;
            if (g_bf16) {
                gb[f[1] % n] = static_cast<std::uint16_t>(f[2]);
            } else {
                flat[f[1] % n] = bits_float(static_cast<std::uint32_t>(f[2]));
            }
        }
        if (g_bf16)
            for (std::uint64_t i = 0; i < n; ++i) flat[i] = bf16_to_float(gb[i]);
        ScanConfig scan;
        scan.worker_count = 4;
        const bool of = fused_overflow_check(std::span<const float>(flat), scan).overflow;
        if (of) {
            sc.on_overflow();
        } else {
            updates += 1;
            const float scale_now = sc.scale;
            for (std::uint64_t off = 0; off < n; off += subgroup) {
                const std::uint64_t len = std::min(subgroup, n - off);
                adam_step_fp32({p.data() + off, len}, {m.data() + off, len}, {v.data() + off, len},
                               {flat.data() + off, len}, updates, h, scale_now, 3);
                for (std::uint64_t k = off; k < off + len; ++k)
                    w[k] = w_bf16 ? bf16_from_float(p[k]) : fp16_from_float(p[k]);
            }
            sc.on_clean_step();
        }
        per.push_back({{"step", s},
                       {"overflow", of},
                       {"scale_after", sc.scale},
                       {"grads_fnv", g_bf16 ? fnv_vec(gb) : fnv_vec(flat)},
                       {"p_fnv", fnv_vec(p)},
                       {"m_fnv", fnv_vec(m)},
                       {"v_fnv", fnv_vec(v)},
                       {"w_fnv", fnv_vec(w)}});
    }
    json fl = json::array();
    for (const auto& f : faults) fl.push_back({{"step", f[0]}, {"index", f[1]}, {"bits", f[2]}});
    // a few raw final values for readable failures
    json sample = json::array();
    for (std::uint64_t i : {std::uint64_t{0}, std::uint64_t{1}, n / 2, n - 1}) {
        sample.push_back({{"i", i}, {"p", float_bits(p[i])}, {"m", float_bits(m[i])},
                          {"v", float_bits(v[i])}, {"w", w[i]}});
    }
    return {{"name", name},       {"n", n},         {"steps", steps},
            {"seed", seed},       {"g_kind", g_bf16 ? "bf16" : "f32"},
            {"w_kind", w_bf16 ? "bf16" : "f16"}, {"subgroup", subgroup},
            {"lr", float_bits(h.lr)}, {"beta1", float_bits(h.beta1)},
            {"beta2", float_bits(h.beta2)}, {"eps", float_bits(h.eps)},
            {"wd", float_bits(h.weight_decay)}, {"init_scale", 65536.0},
            {"growth_interval", growth}, {"faults", fl},
            {"updates", updates}, {"final_scale", sc.scale},
            {"per_step", per},    {"sample", sample}};
}

json workload() {
    json cases = json::array();
    // configs: bf16 grads, bf16 working weights, fp32 master/m/v, AdamW wd 0.01
    cases.push_back(workload_case("cfg_bf16_n100003", 100003, 6, 1, true, true, 30000, 2000,
                                  {{2, 777, 0x7FC0}, {4, 100002, 0x7F7F}}, 0.01f));
    // reference mode: fp32 grads, fp16 shadows, growth every 3 clean steps
    cases.push_back(workload_case("ref_f32_n65537", 65537, 9, 3, false, false, 20000, 3,
                                  {{1, 5, 0xFF800000u}, {5, 65536, 0x7F800001u}, {6, 9, 0x7F7FFFFFu}},
                                  0.0f));
    // cfg3-style injection patterns across many steps, tiny partition
    cases.push_back(workload_case("cfg_bf16_patterns_n4099", 4099, 12, 11, true, true, 1000, 2000,
                                  {{0, 1, 0x7F80}, {2, 2, 0xFF80}, {4, 3, 0x7F81}, {6, 4, 0x7FC0},
                                   {8, 5, 0xFFC1}, {9, 6, 0x7F7F}, {10, 7, 0xFF7F}},
                                  0.01f));
    return {{"cases", cases}};
}

// BASELINE configs[2] injection plan (paper_2505_23254_b200/shard.py
// FaultPlan, seed 2505): each step draws k in {0, 1, 3} non-finite plants
// (plus a max-finite control plant that never triggers), so the global skip
// decision of step s is k > 0 — independent of the partition size.  The
// scale sequence is the reference's own LossScaler (optimizer.hpp:19-35)
// driven by those decisions; bench.py --config cfg3 checks its ranks
// against this fixture.
json cfg3_plan() {
    const std::uint64_t seed = 2505, steps = 1024;
    LossScaler sc;  // 65536, growth 2000
    json of = json::array(), scales = json::array();
    for (std::uint64_t s = 0; s < steps; ++s) {
        std::uint64_t h = splitmix64(seed ^ splitmix64(s ^ 0xC0FFEEull));
        h = splitmix64(h);
        const std::uint64_t k = std::array<std::uint64_t, 3>{0, 1, 3}[h % 3];
        if (k) {
            sc.on_overflow();
        } else {
            sc.on_clean_step();
        }
        of.push_back(k ? 1 : 0);
        scales.push_back(float_bits(sc.scale));
    }
    return {{"seed", seed}, {"steps", steps}, {"init_scale", 65536.0},
            {"growth_interval", 2000}, {"overflow", of}, {"scale_after_bits", scales}};
}

}  // namespace

int main(int argc, char** argv) {
    const std::string dir = argc > 1 ? argv[1] : ".";
    const std::string which = argc > 2 ? argv[2] : "all";
    if (which == "all" || which == "adversarial") write(dir, "adversarial.json", adversarial());
    if (which == "all" || which == "nan_index") write(dir, "nan_index.json", nan_index());
    if (which == "all" || which == "adam_kat") write(dir, "adam_kat.json", adam_kat());
    if (which == "all" || which == "halfprec") write(dir, "halfprec.json", halfprec());
    if (which == "all" || which == "trainer") write(dir, "trainer.json", trainer());
    if (which == "all" || which == "workload") write(dir, "workload.json", workload());
    if (which == "all" || which == "cfg3") write(dir, "cfg3_plan.json", cfg3_plan());
    return 0;
}
