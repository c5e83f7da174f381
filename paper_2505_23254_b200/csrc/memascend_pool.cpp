// Model inventory (model.hpp) and the registered staging pool (pool.hpp).
//
// Inventory rules follow proj/src/model.cpp:85-202 (ceil-divided rows per
// rank, orientation-insensitive shape classes, per-layer vs global member
// counts); pool layout and ledger follow proj/src/pool.cpp:22-233.  The
// backing region comes from the registering PinnedAllocator, so checked-out
// slots are DMA-ready for the streamed optimizer.
#include <algorithm>
#include <chrono>
#include <unordered_map>
#include <mutex>
#include <condition_variable>
#include <cctype>
#include <fstream>
#include <map>
#include <sstream>

#include "memascend/error.hpp"
#include "memascend/model.hpp"
#include "memascend/device_pool.hpp"
#include "memascend/pool.hpp"
#include "memascend_b200.h"

namespace memascend {

// ------------------------------------------------------------------ model
Precision precision_from_string(const std::string& name) {
    if (name == "fp32") return Precision{PrecisionKind::fp32};
    if (name == "fp16") return Precision{PrecisionKind::fp16};
    if (name == "bf16") return Precision{PrecisionKind::bf16};
    raise(ErrorCode::invalid_argument, "unknown precision '" + name + "'");
}

const char* to_string(PrecisionKind kind) noexcept {
    switch (kind) {
        case PrecisionKind::fp32: return "fp32";
        case PrecisionKind::fp16: return "fp16";
        case PrecisionKind::bf16: return "bf16";
    }
    return "?";
}

const char* to_string(TensorRole role) noexcept {
    static const char* const names[] = {"embedding", "lm_head", "ffn_up",  "ffn_gate",
                                        "ffn_down",  "q_proj",  "k_proj",  "v_proj",
                                        "o_proj",    "expert_ffn", "other"};
    const auto i = static_cast<unsigned>(role);
    return i < 11 ? names[i] : "?";
}

bool is_per_layer_role(TensorRole role) noexcept {
    return role != TensorRole::embedding && role != TensorRole::lm_head;
}

std::uint64_t tensor_bytes(const TensorDescriptor& t) {
    if (t.rows == 0 || t.cols == 0)
        raise(ErrorCode::invalid_argument, "tensor '" + t.name + "' has a zero dimension");
    std::uint64_t elems = 0, bytes = 0;
    if (__builtin_mul_overflow(t.rows, t.cols, &elems))
        raise(ErrorCode::overflow, "element count overflow for '" + t.name + "'");
    if (__builtin_mul_overflow(elems, std::uint64_t{t.precision.bytes_per_element()}, &bytes))
        raise(ErrorCode::overflow, "byte count overflow for '" + t.name + "'");
    return bytes;
}

void ModelSpec::validate() const {
    if (vocab == 0 || hidden == 0 || layers == 0 || kv_dim == 0)
        raise(ErrorCode::invalid_argument, "model spec '" + name + "' has a zero dimension");
    if (intermediate == 0)
        raise(ErrorCode::invalid_argument,
              (num_experts ? "MoE spec '" : "dense spec '") + name +
                  (num_experts ? "' needs an expert FFN size" : "' needs an intermediate size"));
    if (ranks == 0) raise(ErrorCode::invalid_argument, "ranks must be >= 1");
}

std::vector<TensorDescriptor> enumerate_offload_tensors(const ModelSpec& spec,
                                                        std::uint64_t partition_ranks) {
    spec.validate();
    if (partition_ranks == 0) raise(ErrorCode::invalid_argument, "partition_ranks must be >= 1");
    const Precision prec = spec.compute_precision;
    const std::uint64_t q = spec.q_dim ? spec.q_dim : spec.hidden;
    std::vector<TensorDescriptor> inv;
    auto add = [&](std::string name, std::uint64_t rows, std::uint64_t cols, TensorRole role) {
        if (spec.min_offload_elements && rows * cols < spec.min_offload_elements) return;
        const std::uint64_t r = partition_ranks > 1 ? (rows + partition_ranks - 1) / partition_ranks
                                                    : rows;
        inv.push_back(TensorDescriptor{std::move(name), r, cols, prec, role});
    };
    add("embedding", spec.vocab, spec.hidden, TensorRole::embedding);
    add("lm_head", spec.vocab, spec.hidden, TensorRole::lm_head);
    for (std::uint64_t l = 0; l < spec.layers; ++l) {
        const std::string b = "layer" + std::to_string(l) + ".";
        add(b + "q_proj", q, spec.hidden, TensorRole::q_proj);
        add(b + "k_proj", spec.kv_dim, spec.hidden, TensorRole::k_proj);
        add(b + "v_proj", spec.kv_dim, spec.hidden, TensorRole::v_proj);
        add(b + "o_proj", spec.hidden, q, TensorRole::o_proj);
        if (spec.num_experts == 0) {
            add(b + "ffn_up", spec.intermediate, spec.hidden, TensorRole::ffn_up);
            add(b + "ffn_gate", spec.intermediate, spec.hidden, TensorRole::ffn_gate);
            add(b + "ffn_down", spec.hidden, spec.intermediate, TensorRole::ffn_down);
        } else {
            add(b + "router", spec.num_experts, spec.hidden, TensorRole::other);
            for (std::uint64_t e = 0; e < spec.num_experts; ++e) {
                const std::string x = b + "expert" + std::to_string(e) + ".";
                add(x + "up", spec.intermediate, spec.hidden, TensorRole::expert_ffn);
                add(x + "gate", spec.intermediate, spec.hidden, TensorRole::expert_ffn);
                add(x + "down", spec.hidden, spec.intermediate, TensorRole::expert_ffn);
            }
        }
    }
    return inv;
}

std::vector<ShapeClass> classify(const std::vector<TensorDescriptor>& tensors) {
    if (tensors.empty()) raise(ErrorCode::invalid_argument, "cannot classify an empty inventory");
    std::map<std::string, ShapeClass> by_key;  // ordered: deterministic class order
    std::uint64_t layers = 0;
    for (const auto& t : tensors) {
        const std::uint64_t big = std::max(t.rows, t.cols), small = std::min(t.rows, t.cols);
        const std::string key = std::to_string(big) + "x" + std::to_string(small) + "@" +
                                std::to_string(t.precision.bytes_per_element());
        ShapeClass& c = by_key[key];
        if (c.class_id.empty()) {
            c.class_id = key;
            c.element_count = big * small;
            c.buffer_bytes = tensor_bytes(t);
        }
        c.member_count += 1;
        (is_per_layer_role(t.role) ? c.members_per_layer : c.global_members) += 1;
        if (t.name.rfind("layer", 0) == 0) {
            const std::uint64_t idx = std::stoull(t.name.substr(5, t.name.find('.') - 5));
            layers = std::max(layers, idx + 1);
        }
    }
    std::vector<ShapeClass> out;
    for (auto& [key, c] : by_key) {
        if (c.members_per_layer > 0) {
            if (layers > 0) {
                c.members_per_layer /= layers;  // totals -> per block
            } else {
                c.global_members += c.members_per_layer;
                c.members_per_layer = 0;
            }
        }
        out.push_back(std::move(c));
    }
    std::sort(out.begin(), out.end(),
              [](const ShapeClass& a, const ShapeClass& b) { return a.buffer_bytes > b.buffer_bytes; });
    return out;
}

namespace {

ModelSpec spec(const char* name, std::uint64_t v, std::uint64_t h, std::uint64_t i, std::uint64_t kv,
               std::uint64_t q, std::uint64_t l, std::uint64_t experts, std::uint64_t params) {
    ModelSpec s;
    s.name = name;
    s.vocab = v;
    s.hidden = h;
    s.intermediate = i;
    s.kv_dim = kv;
    s.q_dim = q;
    s.layers = l;
    s.num_experts = experts;
    s.params_total = params;
    return s;
}

}  // namespace

std::vector<std::string> preset_names() {
    return {"llama3.1-8b", "qwen2.5-7b", "qwen2.5-14b", "qwen2.5-32b", "qwen3-30b-a3b", "toy-dense"};
}

ModelSpec preset(const std::string& name) {
    // dimensions and exact parameter totals of proj/src/model.cpp:228-251
    if (name == "llama3.1-8b") return spec("llama3.1-8b", 128256, 5120, 14336, 1024, 5120, 32, 0, 8030261248ull);
    if (name == "qwen2.5-7b") return spec("qwen2.5-7b", 152064, 3584, 18944, 512, 3584, 28, 0, 7615627264ull);
    if (name == "qwen2.5-14b") return spec("qwen2.5-14b", 152064, 5120, 13824, 1024, 5120, 48, 0, 14770033664ull);
    if (name == "qwen2.5-32b") return spec("qwen2.5-32b", 152064, 5120, 27648, 1024, 5120, 64, 0, 32763876352ull);
    if (name == "qwen3-30b-a3b") return spec("qwen3-30b-a3b", 151936, 2048, 768, 512, 4096, 48, 128, 30532122624ull);
    if (name == "toy-dense") return spec("toy-dense", 256, 32, 64, 16, 32, 4, 0, 0);
    raise(ErrorCode::not_found, "no preset named '" + name + "'");
}

namespace {

// Minimal reader for the flat model-config object (string / unsigned values).
std::map<std::string, std::string> read_flat_json(const std::string& text, const std::string& path) {
    std::map<std::string, std::string> kv;
    std::size_t i = 0;
    auto bad = [&](const char* why) {
        raise(ErrorCode::bad_config, "malformed model config '" + path + "': " + why);
    };
    auto ws = [&] { while (i < text.size() && std::isspace(static_cast<unsigned char>(text[i]))) ++i; };
    auto str = [&] {
        if (text[i] != '"') bad("expected a string");
        std::string s;
        for (++i; i < text.size() && text[i] != '"'; ++i) {
            if (text[i] == '\\' && i + 1 < text.size()) ++i;
            s += text[i];
        }
        if (i >= text.size()) bad("unterminated string");
        ++i;
        return s;
    };
    ws();
    if (i >= text.size() || text[i] != '{') bad("expected an object");
    ++i;
    ws();
    if (i < text.size() && text[i] == '}') return kv;
    for (;;) {
        ws();
        const std::string k = str();
        ws();
        if (i >= text.size() || text[i] != ':') bad("expected ':'");
        ++i;
        ws();
        std::string v;
        if (i < text.size() && text[i] == '"') {
            v = str();
        } else {
            while (i < text.size() && text[i] != ',' && text[i] != '}' &&
                   !std::isspace(static_cast<unsigned char>(text[i])))
                v += text[i++];
            if (v.empty()) bad("empty value");
        }
        kv[k] = v;
        ws();
        if (i < text.size() && text[i] == ',') { ++i; continue; }
        if (i < text.size() && text[i] == '}') break;
        bad("expected ',' or '}'");
    }
    return kv;
}

}  // namespace

ModelSpec load_model_spec(const std::string& path) {
    std::ifstream in(path);
    if (!in.good()) raise(ErrorCode::not_found, "cannot open model config '" + path + "'");
    std::stringstream ss;
    ss << in.rdbuf();
    const auto kv = read_flat_json(ss.str(), path);
    auto num = [&](const char* key, bool required, std::uint64_t dflt) -> std::uint64_t {
        auto it = kv.find(key);
        if (it == kv.end()) {
            if (required)
                raise(ErrorCode::bad_config, "model config '" + path + "' missing field: " + key);
            return dflt;
        }
        try {
            std::size_t used = 0;
            const unsigned long long v = std::stoull(it->second, &used);
            if (used != it->second.size()) throw std::invalid_argument(key);
            return v;
        } catch (const std::exception&) {
            raise(ErrorCode::bad_config, "model config '" + path + "' field " + key + " is not an integer");
        }
    };
    ModelSpec s;
    s.name = kv.count("name") ? kv.at("name") : path;
    s.vocab = num("vocab", true, 0);
    s.hidden = num("hidden", true, 0);
    s.intermediate = num("intermediate", true, 0);
    s.kv_dim = num("kv_dim", true, 0);
    s.q_dim = num("q_dim", false, 0);
    s.layers = num("layers", true, 0);
    s.num_experts = num("experts", false, 0);
    s.params_total = num("params_total", false, 0);
    s.ranks = num("ranks", false, 1);
    s.compute_precision = precision_from_string(kv.count("precision") ? kv.at("precision") : "fp16");
    s.min_offload_elements = num("min_offload_elements", false, 0);
    s.validate();
    return s;
}

// ------------------------------------------------------------------ pool
namespace {

constexpr std::uint64_t kGranule = 4096;  // slot starts feed O_DIRECT / DMA

struct Layout {
    std::vector<Pool::ClassInfo> classes;
    std::uint64_t payload = 0;
    std::uint64_t backing = 0;
};

Layout layout_for(const std::vector<TensorDescriptor>& inventory, PoolMode mode,
                  std::uint64_t inflight) {
    if (inventory.empty()) raise(ErrorCode::invalid_argument, "cannot build a pool over an empty inventory");
    if (inflight == 0) raise(ErrorCode::invalid_argument, "inflight_blocks must be >= 1");
    const auto shapes = classify(inventory);
    Layout L;
    if (mode == PoolMode::adaptive) {
        for (const auto& c : shapes) {
            L.classes.push_back({c.class_id, c.buffer_bytes,
                                 c.global_members + c.members_per_layer * inflight, 0, 0});
        }
    } else {
        std::uint64_t biggest = 0, per_block = 0, global = 0;
        for (const auto& c : shapes) {
            biggest = std::max(biggest, c.buffer_bytes);
            per_block += c.members_per_layer;
            global += c.global_members;
        }
        L.classes.push_back({"monolithic", biggest, per_block * inflight + global, 0, 0});
    }
    std::uint64_t off = 0;
    for (auto& c : L.classes) {
        c.base_offset = off;
        c.slot_stride = (c.slot_payload_bytes + kGranule - 1) / kGranule * kGranule;
        off += c.slot_stride * c.slot_count;
        L.payload += c.slot_payload_bytes * c.slot_count;
    }
    L.backing = off;
    return L;
}

}  // namespace

std::uint64_t pool_capacity(const std::vector<TensorDescriptor>& inventory, PoolMode mode,
                            std::uint64_t inflight_blocks) {
    return layout_for(inventory, mode, inflight_blocks).payload;
}

struct Pool::State {
    std::vector<std::vector<std::uint32_t>> free;          // per class, LIFO
    std::unordered_map<std::string, std::uint32_t> known;  // inventory key -> class
    std::unordered_map<std::string, BufferHandle> out;     // checked-out handles
    PinnedRegion backing;
    PinnedAllocator* allocator = nullptr;
    mutable std::mutex mu;
    std::condition_variable returned;
    PoolStats stats;

    std::uint32_t class_for(const std::vector<ClassInfo>& classes, const std::string& key,
                            std::uint64_t payload) const {
        if (auto it = known.find(key); it != known.end()) return it->second;
        // unknown key: the tightest class that holds the payload
        std::uint32_t best = UINT32_MAX;
        for (std::uint32_t c = 0; c < classes.size(); ++c) {
            if (classes[c].slot_payload_bytes >= payload &&
                (best == UINT32_MAX || classes[c].slot_payload_bytes < classes[best].slot_payload_bytes))
                best = c;
        }
        if (best == UINT32_MAX)
            raise(ErrorCode::size_violation,
                  "payload of " + std::to_string(payload) + " bytes fits no slot class");
        return best;
    }

    const BufferHandle& held(const BufferHandle& h, const char* what) const {
        auto it = out.find(h.key);
        if (it == out.end())
            raise(ErrorCode::lifecycle, std::string(what) + " on a handle that is not checked out");
        return it->second;
    }
};

Pool::Pool(const std::vector<TensorDescriptor>& inventory, const PoolConfig& config,
           PinnedAllocator& allocator)
    : st_(std::make_unique<State>()), config_(config) {
    Layout L = layout_for(inventory, config.mode, config.inflight_blocks);
    classes_ = std::move(L.classes);
    st_->allocator = &allocator;
    st_->free.resize(classes_.size());
    for (std::size_t c = 0; c < classes_.size(); ++c)
        for (std::uint64_t k = classes_[c].slot_count; k > 0; --k)
            st_->free[c].push_back(static_cast<std::uint32_t>(k - 1));
    for (const auto& t : inventory) {
        std::uint32_t c = 0;
        if (config.mode == PoolMode::adaptive) {
            const std::uint64_t b = tensor_bytes(t);
            while (c < classes_.size() && classes_[c].slot_payload_bytes != b) ++c;
            if (c == classes_.size()) continue;
        }
        st_->known.emplace(t.name, c);
    }
    st_->backing = allocator.allocate(std::max<std::uint64_t>(L.backing, 1), config.backing_policy,
                                      config.lock_pages);
    st_->stats.capacity_bytes = L.payload;
    st_->stats.backing_bytes = L.backing;
}

Pool::~Pool() = default;

BufferHandle Pool::checkout(const std::string& key, std::uint64_t payload_bytes) {
    if (payload_bytes == 0) raise(ErrorCode::invalid_argument, "zero-byte checkout for '" + key + "'");
    State& S = *st_;
    std::unique_lock<std::mutex> lock(S.mu);
    if (S.out.count(key)) raise(ErrorCode::already_checked_out, "'" + key + "' is already checked out");
    const std::uint32_t c = S.class_for(classes_, key, payload_bytes);
    const ClassInfo& info = classes_[c];
    if (payload_bytes > info.slot_payload_bytes)
        raise(ErrorCode::size_violation, "payload of " + std::to_string(payload_bytes) +
                                             " bytes exceeds slot size " +
                                             std::to_string(info.slot_payload_bytes) + " ('" + key + "')");
    auto& fs = S.free[c];
    if (fs.empty()) {
        if (!config_.blocking_checkout)
            raise(ErrorCode::pool_exhausted,
                  "class " + info.class_id + " has no free buffers for '" + key + "'");
        const auto t0 = std::chrono::steady_clock::now();
        S.returned.wait(lock, [&] { return !fs.empty(); });
        S.stats.blocked_time += std::chrono::steady_clock::now() - t0;
    }
    const std::uint32_t slot = fs.back();
    fs.pop_back();
    BufferHandle h{key, info.base_offset + std::uint64_t{slot} * info.slot_stride, payload_bytes, c, slot,
                   true};
    S.out[key] = h;
    S.stats.checkout_count += 1;
    S.stats.live_bytes += payload_bytes;
    S.stats.peak_live_bytes = std::max(S.stats.peak_live_bytes, S.stats.live_bytes);
    return h;
}

void Pool::checkin(const BufferHandle& handle) {
    State& S = *st_;
    std::lock_guard<std::mutex> g(S.mu);
    auto it = S.out.find(handle.key);
    if (it == S.out.end() || it->second.slot_index != handle.slot_index ||
        it->second.class_index != handle.class_index)
        raise(ErrorCode::lifecycle, "checkin of a handle the pool does not hold ('" + handle.key + "')");
    S.free[handle.class_index].push_back(handle.slot_index);
    S.stats.live_bytes -= it->second.length;
    S.stats.checkin_count += 1;
    S.out.erase(it);
    S.returned.notify_all();
}

std::span<std::byte> Pool::span(const BufferHandle& handle) {
    std::lock_guard<std::mutex> g(st_->mu);
    st_->held(handle, "span()");
    return st_->backing.bytes().subspan(handle.offset, handle.length);
}

std::span<std::byte> Pool::padded_span(const BufferHandle& handle) {
    std::lock_guard<std::mutex> g(st_->mu);
    st_->held(handle, "padded_span()");
    return st_->backing.bytes().subspan(handle.offset,
                                        (handle.length + kGranule - 1) / kGranule * kGranule);
}

void* Pool::device_span(const BufferHandle& handle) {
    std::lock_guard<std::mutex> g(st_->mu);
    st_->held(handle, "device_span()");
    if (!st_->backing.locked())
        raise(ErrorCode::capability, "pool backing is not registered with the GPU");
    // registered memory is addressed by the GPU through the same UVA pointer
    return st_->backing.data() + handle.offset;
}

PoolStats Pool::stats() const {
    std::lock_guard<std::mutex> g(st_->mu);
    return st_->stats;
}

std::vector<std::pair<std::uint64_t, std::uint64_t>> Pool::live_extents() const {
    std::lock_guard<std::mutex> g(st_->mu);
    std::vector<std::pair<std::uint64_t, std::uint64_t>> v;
    v.reserve(st_->out.size());
    for (const auto& kv : st_->out) v.emplace_back(kv.second.offset, kv.second.length);
    return v;
}

double fragmentation(std::uint64_t capacity_bytes, std::uint64_t peak_live_bytes) {
    if (capacity_bytes == 0) raise(ErrorCode::invalid_argument, "fragmentation over zero capacity");
    if (peak_live_bytes > capacity_bytes) raise(ErrorCode::invalid_argument, "peak live bytes exceed capacity");
    return static_cast<double>(capacity_bytes - peak_live_bytes) / static_cast<double>(capacity_bytes);
}

}  // namespace memascend

// ------------------------------------------------------------------ device pool
// include/memascend/device_pool.hpp: the same class plan, backed in HBM by
// ma_dpool; the prefetcher over ma_prefetcher.
namespace memascend {

namespace {

void check_status(int status) {
    if (status == MA_OK) return;
    const std::string msg = ma_last_error();
    if (status >= 1 && status <= 17) raise(static_cast<ErrorCode>(status - 1), msg);
    raise(ErrorCode::device_error, msg);
}

}  // namespace

DevicePool::DevicePool(const std::vector<TensorDescriptor>& inventory, PoolMode mode,
                       std::uint64_t inflight_blocks) {
    const Layout L = layout_for(inventory, mode, inflight_blocks);
    classes_ = L.classes;
    std::vector<std::uint64_t> bytes;
    std::vector<std::uint32_t> counts;
    for (const auto& c : classes_) {
        bytes.push_back(c.slot_payload_bytes);
        counts.push_back(static_cast<std::uint32_t>(c.slot_count));
    }
    check_status(ma_dpool_create(bytes.data(), counts.data(),
                                 static_cast<std::uint32_t>(bytes.size()), &h_));
}

DevicePool::~DevicePool() {
    if (h_) ma_dpool_destroy(h_);
}

PoolStats DevicePool::stats() const {
    ma_dpool_stats s{};
    check_status(ma_dpool_get_stats(h_, &s));
    PoolStats out;
    out.capacity_bytes = s.capacity_bytes;
    out.backing_bytes = s.backing_bytes;
    out.peak_live_bytes = s.peak_live_bytes;
    out.live_bytes = s.live_bytes;
    out.checkout_count = s.checkout_count;
    out.checkin_count = s.checkin_count;
    return out;
}

WeightPrefetcher::WeightPrefetcher(DirectIoEngine& store, DevicePool& pool,
                                   std::uint32_t host_slots, std::uint64_t host_slot_bytes) {
    const std::uint64_t slot = (host_slot_bytes + kGranule - 1) / kGranule * kGranule;
    if (host_slots == 0 || slot == 0)
        raise(ErrorCode::invalid_argument, "prefetcher needs >= 1 host slot of > 0 bytes");
    staging_ = PinnedAllocator::global().allocate(slot * host_slots,
                                                  {AllocPolicyKind::alignment_free});
    check_status(ma_prefetcher_create(store.handle(), pool.handle(), staging_.data(), slot,
                                      host_slots, &h_));
}

WeightPrefetcher::~WeightPrefetcher() {
    if (h_) ma_prefetcher_destroy(h_);
}

void WeightPrefetcher::submit(const std::string& key) {
    check_status(ma_prefetch_submit(h_, key.c_str()));
}

void* WeightPrefetcher::acquire(const std::string& key, void* stream, std::uint64_t* bytes) {
    void* d = nullptr;
    check_status(ma_prefetch_acquire(h_, key.c_str(), stream, &d, bytes));
    return d;
}

void WeightPrefetcher::release(const std::string& key, void* stream) {
    check_status(ma_prefetch_release(h_, key.c_str(), stream));
}

}  // namespace memascend
