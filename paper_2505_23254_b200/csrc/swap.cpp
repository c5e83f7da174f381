// Host-side swap engine (see swap.hpp) and its C ABI (ma_swap_*, ma_cursor_*).
//
// Reference behaviour followed, by file:line of /root/reference/proj:
//   open/O_DIRECT/capability error ........ src/direct_io.cpp:30-45
//   SharedCursor (flock'd counter file) .... src/direct_io.cpp:51-117
//   constructor validation, auto backend ... src/direct_io.cpp:128-168
//   allocate_extents (equal split, grow
//     abandons, shrink reuses) ............. src/direct_io.cpp:188-248
//   per-task chunking over workers ......... src/direct_io.cpp:334-381
//   busy-key guard, write/read checks ...... src/direct_io.cpp:383-460
//   manifest schema (version 1) ............ src/direct_io.cpp:484-578
//   create_virtual_devices ................. src/direct_io.cpp:580-604
// The io_uring backend is new; the reference has
// pread/pwrite and lio_listio only.
#include "swap.hpp"

#include <aio.h>
#include <errno.h>
#include <fcntl.h>
#include <linux/io_uring.h>
#include <sys/file.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <sys/syscall.h>
#include <unistd.h>

#include <algorithm>
#include <cctype>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <sstream>

#include "memascend_b200.h"

namespace ma {
void set_error(const std::string& msg);  // capi.cu (ma_last_error)
}

namespace ma {
namespace swp {

void fail(int code, const std::string& msg) { throw Failure{code, msg}; }

namespace {

std::uint64_t align_up(std::uint64_t v, std::uint64_t a) { return (v + a - 1) / a * a; }
bool aligned_ptr(const void* p) { return reinterpret_cast<std::uintptr_t>(p) % kGranule == 0; }

int open_device(const DeviceSpec& d, bool bypass) {
    int fd = ::open(d.path.c_str(), O_RDWR | O_CLOEXEC | (bypass ? O_DIRECT : 0));
    if (fd < 0 && bypass && (errno == EINVAL || errno == ENOTSUP))
        fail(MA_ERR_CAPABILITY, "cache bypass (O_DIRECT) unsupported for '" + d.path + "'");
    if (fd < 0)
        fail(MA_ERR_DEVICE_ERROR, "cannot open device '" + d.path + "': " + std::strerror(errno));
    return fd;
}

// ------------------------------------------------------------ io_uring
// Raw-syscall ring (no liburing in the image): one per worker thread, the
// thread is the only submitter and the only reaper.
class Ring {
public:
    ~Ring() {
        if (sqes_) ::munmap(sqes_, sqes_len_);
        if (cq_map_ && cq_map_ != sq_map_) ::munmap(cq_map_, cq_len_);
        if (sq_map_) ::munmap(sq_map_, sq_len_);
        if (fd_ >= 0) ::close(fd_);
    }
    bool init(unsigned entries) {
        io_uring_params p;
        std::memset(&p, 0, sizeof p);
        fd_ = static_cast<int>(::syscall(__NR_io_uring_setup, entries, &p));
        if (fd_ < 0) return false;
        sq_len_ = p.sq_off.array + p.sq_entries * sizeof(unsigned);
        cq_len_ = p.cq_off.cqes + p.cq_entries * sizeof(io_uring_cqe);
        const bool single = p.features & IORING_FEAT_SINGLE_MMAP;
        if (single) sq_len_ = cq_len_ = std::max(sq_len_, cq_len_);
        sq_map_ = ::mmap(nullptr, sq_len_, PROT_READ | PROT_WRITE, MAP_SHARED | MAP_POPULATE, fd_,
                         IORING_OFF_SQ_RING);
        if (sq_map_ == MAP_FAILED) return sq_map_ = nullptr, false;
        if (single) {
            cq_map_ = sq_map_;
        } else {
            cq_map_ = ::mmap(nullptr, cq_len_, PROT_READ | PROT_WRITE, MAP_SHARED | MAP_POPULATE,
                             fd_, IORING_OFF_CQ_RING);
            if (cq_map_ == MAP_FAILED) return cq_map_ = nullptr, false;
        }
        sqes_len_ = p.sq_entries * sizeof(io_uring_sqe);
        sqes_ = static_cast<io_uring_sqe*>(::mmap(nullptr, sqes_len_, PROT_READ | PROT_WRITE,
                                                  MAP_SHARED | MAP_POPULATE, fd_,
                                                  IORING_OFF_SQES));
        if (sqes_ == MAP_FAILED) return sqes_ = nullptr, false;
        auto* sq = static_cast<char*>(sq_map_);
        auto* cq = static_cast<char*>(cq_map_);
        sq_tail_ = reinterpret_cast<unsigned*>(sq + p.sq_off.tail);
        sq_mask_ = *reinterpret_cast<unsigned*>(sq + p.sq_off.ring_mask);
        sq_array_ = reinterpret_cast<unsigned*>(sq + p.sq_off.array);
        cq_head_ = reinterpret_cast<unsigned*>(cq + p.cq_off.head);
        cq_tail_ = reinterpret_cast<unsigned*>(cq + p.cq_off.tail);
        cq_mask_ = *reinterpret_cast<unsigned*>(cq + p.cq_off.ring_mask);
        cqes_ = reinterpret_cast<io_uring_cqe*>(cq + p.cq_off.cqes);
        entries_ = p.sq_entries;
        return true;
    }
    unsigned entries() const { return entries_; }
    // Ops READ/WRITE exist since 5.6; probe them so auto_probe never picks a
    // ring that would fail every request.
    bool supports_rw() {
        const size_t len = sizeof(io_uring_probe) + 256 * sizeof(io_uring_probe_op);
        std::vector<char> buf(len, 0);
        auto* pr = reinterpret_cast<io_uring_probe*>(buf.data());
        if (::syscall(__NR_io_uring_register, fd_, IORING_REGISTER_PROBE, pr, 256) < 0)
            return false;
        auto ok = [&](unsigned op) {
            return op <= pr->last_op && (pr->ops[op].flags & IO_URING_OP_SUPPORTED);
        };
        return ok(IORING_OP_READ) && ok(IORING_OP_WRITE);
    }
    void prep(bool write, int fd, void* buf, unsigned len, std::uint64_t off, void* user) {
        const unsigned tail = *sq_tail_;
        const unsigned idx = tail & sq_mask_;
        io_uring_sqe* e = &sqes_[idx];
        std::memset(e, 0, sizeof *e);
        e->opcode = write ? IORING_OP_WRITE : IORING_OP_READ;
        e->fd = fd;
        e->addr = reinterpret_cast<std::uint64_t>(buf);
        e->len = len;
        e->off = off;
        e->user_data = reinterpret_cast<std::uint64_t>(user);
        sq_array_[idx] = idx;
        __atomic_store_n(sq_tail_, tail + 1, __ATOMIC_RELEASE);
    }
    // Submits `n` prepared entries and waits for at least `min_complete`.
    // Returns 0, or -errno with *unsubmitted = the trailing prepared entries
    // the kernel did not take (already withdrawn from the ring).
    int enter(unsigned n, unsigned min_complete, unsigned* unsubmitted) {
        *unsubmitted = 0;
        for (;;) {
            const long r = ::syscall(__NR_io_uring_enter, fd_, n, min_complete,
                                     min_complete ? IORING_ENTER_GETEVENTS : 0u, nullptr, 0);
            if (r >= 0) {
                n -= std::min<unsigned>(n, static_cast<unsigned>(r));
                if (n == 0) return 0;
                continue;
            }
            if (errno == EINTR || errno == EAGAIN || errno == EBUSY) continue;
            const int e = errno;
            __atomic_store_n(sq_tail_, *sq_tail_ - n, __ATOMIC_RELEASE);
            *unsubmitted = n;
            return -e;
        }
    }
    template <typename F>
    void reap(F&& on_cqe) {
        unsigned head = *cq_head_;
        const unsigned tail = __atomic_load_n(cq_tail_, __ATOMIC_ACQUIRE);
        while (head != tail) {
            const io_uring_cqe& c = cqes_[head & cq_mask_];
            on_cqe(reinterpret_cast<void*>(c.user_data), c.res);
            ++head;
        }
        __atomic_store_n(cq_head_, head, __ATOMIC_RELEASE);
    }

private:
    int fd_ = -1;
    unsigned entries_ = 0;
    void* sq_map_ = nullptr;
    void* cq_map_ = nullptr;
    size_t sq_len_ = 0, cq_len_ = 0, sqes_len_ = 0;
    io_uring_sqe* sqes_ = nullptr;
    unsigned* sq_tail_ = nullptr;
    unsigned sq_mask_ = 0;
    unsigned* sq_array_ = nullptr;
    unsigned* cq_head_ = nullptr;
    unsigned* cq_tail_ = nullptr;
    unsigned cq_mask_ = 0;
    io_uring_cqe* cqes_ = nullptr;
};

// ------------------------------------------------------------ manifest JSON
// Minimal reader for the manifest schema (objects, arrays, strings, unsigned
// integers, booleans, null).
struct JVal {
    enum Kind { Null, Bool, Num, Str, Arr, Obj } kind = Null;
    std::uint64_t num = 0;
    std::string str;
    std::vector<JVal> arr;
    std::vector<std::pair<std::string, JVal>> obj;
    const JVal& at(const std::string& k) const {
        for (const auto& kv : obj)
            if (kv.first == k) return kv.second;
        fail(MA_ERR_BAD_CONFIG, "malformed manifest: missing key '" + k + "'");
    }
    const JVal* find(const std::string& k) const {
        for (const auto& kv : obj)
            if (kv.first == k) return &kv.second;
        return nullptr;
    }
    std::uint64_t u64() const {
        if (kind != Num) fail(MA_ERR_BAD_CONFIG, "malformed manifest: expected an integer");
        return num;
    }
    const std::string& s() const {
        if (kind != Str) fail(MA_ERR_BAD_CONFIG, "malformed manifest: expected a string");
        return str;
    }
};

class JParser {
public:
    explicit JParser(const std::string& text) : t_(text) {}
    JVal parse() {
        JVal v = value();
        ws();
        if (i_ != t_.size()) bad("trailing characters");
        return v;
    }

private:
    [[noreturn]] void bad(const char* what) {
        fail(MA_ERR_BAD_CONFIG, std::string("malformed manifest: ") + what + " at offset " +
                                    std::to_string(i_));
    }
    void ws() {
        while (i_ < t_.size() && std::isspace(static_cast<unsigned char>(t_[i_]))) ++i_;
    }
    bool eat(char c) {
        ws();
        if (i_ < t_.size() && t_[i_] == c) return ++i_, true;
        return false;
    }
    JVal value() {
        ws();
        if (i_ >= t_.size()) bad("unexpected end");
        const char c = t_[i_];
        JVal v;
        if (c == '{') {
            ++i_;
            v.kind = JVal::Obj;
            if (eat('}')) return v;
            do {
                ws();
                std::string k = string();
                if (!eat(':')) bad("expected ':'");
                v.obj.emplace_back(std::move(k), value());
            } while (eat(','));
            if (!eat('}')) bad("expected '}'");
        } else if (c == '[') {
            ++i_;
            v.kind = JVal::Arr;
            if (eat(']')) return v;
            do v.arr.push_back(value());
            while (eat(','));
            if (!eat(']')) bad("expected ']'");
        } else if (c == '"') {
            v.kind = JVal::Str;
            v.str = string();
        } else if (std::isdigit(static_cast<unsigned char>(c))) {
            v.kind = JVal::Num;
            while (i_ < t_.size() && std::isdigit(static_cast<unsigned char>(t_[i_]))) {
                v.num = v.num * 10 + static_cast<std::uint64_t>(t_[i_] - '0');
                ++i_;
            }
            if (i_ < t_.size() && (t_[i_] == '.' || t_[i_] == 'e' || t_[i_] == 'E'))
                bad("non-integer number");
        } else if (t_.compare(i_, 4, "true") == 0) {
            v.kind = JVal::Bool, v.num = 1, i_ += 4;
        } else if (t_.compare(i_, 5, "false") == 0) {
            v.kind = JVal::Bool, i_ += 5;
        } else if (t_.compare(i_, 4, "null") == 0) {
            i_ += 4;
        } else {
            bad("unexpected character");
        }
        return v;
    }
    std::string string() {
        if (i_ >= t_.size() || t_[i_] != '"') bad("expected a string");
        ++i_;
        std::string out;
        while (i_ < t_.size() && t_[i_] != '"') {
            char c = t_[i_++];
            if (c != '\\') {
                out.push_back(c);
                continue;
            }
            if (i_ >= t_.size()) bad("bad escape");
            c = t_[i_++];
            switch (c) {
                case 'n': out.push_back('\n'); break;
                case 't': out.push_back('\t'); break;
                case 'r': out.push_back('\r'); break;
                case 'b': out.push_back('\b'); break;
                case 'f': out.push_back('\f'); break;
                case 'u': {
                    if (i_ + 4 > t_.size()) bad("bad \\u escape");
                    const unsigned cp = static_cast<unsigned>(std::stoul(t_.substr(i_, 4), nullptr, 16));
                    i_ += 4;
                    if (cp < 0x80) {
                        out.push_back(static_cast<char>(cp));
                    } else if (cp < 0x800) {
                        out.push_back(static_cast<char>(0xC0 | (cp >> 6)));
                        out.push_back(static_cast<char>(0x80 | (cp & 0x3F)));
                    } else {
                        out.push_back(static_cast<char>(0xE0 | (cp >> 12)));
                        out.push_back(static_cast<char>(0x80 | ((cp >> 6) & 0x3F)));
                        out.push_back(static_cast<char>(0x80 | (cp & 0x3F)));
                    }
                    break;
                }
                default: out.push_back(c);  // \" \\ \/
            }
        }
        if (i_ >= t_.size()) bad("unterminated string");
        ++i_;
        return out;
    }
    const std::string& t_;
    size_t i_ = 0;
};

std::string jstr(const std::string& s) {
    std::string out = "\"";
    for (unsigned char c : s) {
        if (c == '"' || c == '\\') {
            out.push_back('\\');
            out.push_back(static_cast<char>(c));
        } else if (c < 0x20) {
            char b[8];
            std::snprintf(b, sizeof b, "\\u%04x", c);
            out += b;
        } else {
            out.push_back(static_cast<char>(c));
        }
    }
    return out + "\"";
}

}  // namespace

// ------------------------------------------------------------ Cursor
Cursor::Cursor(std::uint32_t devices, const std::string& path) : local_(devices) {
    for (auto& c : local_) c.store(0);
    if (path.empty()) return;
    fd_ = ::open(path.c_str(), O_CREAT | O_RDWR | O_CLOEXEC, 0644);
    if (fd_ < 0) fail(MA_ERR_DEVICE_ERROR, "cannot open cursor file '" + path + "'");
    struct stat st {};
    ::fstat(fd_, &st);
    const size_t want = devices * sizeof(std::uint64_t);
    if (static_cast<size_t>(st.st_size) < want) {
        if (::ftruncate(fd_, static_cast<off_t>(want)) != 0)
            fail(MA_ERR_DEVICE_ERROR, "cannot size cursor file '" + path + "'");
    } else {
        std::vector<std::uint64_t> v(devices);
        if (::pread(fd_, v.data(), want, 0) == static_cast<ssize_t>(want))
            for (std::uint32_t d = 0; d < devices; ++d) local_[d].store(v[d]);
    }
}

Cursor::~Cursor() {
    if (fd_ >= 0) ::close(fd_);
}

std::uint64_t Cursor::advance(std::uint32_t device, std::uint64_t bytes) {
    if (device >= local_.size()) fail(MA_ERR_INVALID_ARGUMENT, "cursor device index out of range");
    if (fd_ < 0) return local_[device].fetch_add(bytes, std::memory_order_relaxed);
    std::lock_guard<std::mutex> lock(mu_);
    if (::flock(fd_, LOCK_EX) != 0) fail(MA_ERR_DEVICE_ERROR, "flock failed on cursor file");
    const off_t at = static_cast<off_t>(device * sizeof(std::uint64_t));
    std::uint64_t cur = 0;
    if (::pread(fd_, &cur, sizeof cur, at) != sizeof cur) {
        ::flock(fd_, LOCK_UN);
        fail(MA_ERR_IO_ERROR, "cursor file read failed");
    }
    const std::uint64_t next = cur + bytes;
    if (::pwrite(fd_, &next, sizeof next, at) != sizeof next) {
        ::flock(fd_, LOCK_UN);
        fail(MA_ERR_IO_ERROR, "cursor file write failed");
    }
    ::flock(fd_, LOCK_UN);
    local_[device].store(next);
    return cur;
}

std::uint64_t Cursor::position(std::uint32_t device) const {
    if (device >= local_.size()) fail(MA_ERR_INVALID_ARGUMENT, "cursor device index out of range");
    return local_[device].load(std::memory_order_relaxed);
}

void Cursor::restore(std::uint32_t device, std::uint64_t pos) {
    if (device >= local_.size()) fail(MA_ERR_INVALID_ARGUMENT, "cursor device index out of range");
    local_[device].store(pos, std::memory_order_relaxed);
}

// ------------------------------------------------------------ Engine
bool Engine::uring_available() {
    static const bool ok = [] {
        Ring r;
        return r.init(4) && r.supports_rw();
    }();
    return ok;
}

Engine::Engine(std::vector<DeviceSpec> devices, Config cfg)
    : specs_(std::move(devices)), cfg_(std::move(cfg)) {
    if (specs_.empty()) fail(MA_ERR_INVALID_ARGUMENT, "device set is empty");
    if (cfg_.workers == 0) fail(MA_ERR_INVALID_ARGUMENT, "workers must be >= 1");
    if (cfg_.queue_depth == 0) cfg_.queue_depth = 1;
    try {
        for (const auto& d : specs_) {
            if (d.capacity == 0 || d.capacity % kGranule)
                fail(MA_ERR_INVALID_ARGUMENT,
                     "device capacity must be a positive multiple of 4096: " + d.path);
            fds_.push_back(open_device(d, cfg_.cache_bypass));
            total_capacity_ += d.capacity;
        }
        backend_ = cfg_.backend;
        if (backend_ == kAuto) {
            backend_ = uring_available() ? kUring : kAio;
            if (const char* env = std::getenv("MEMASCEND_IO_BACKEND")) {
                const std::string e(env);
                if (e == "sync") backend_ = kSync;
                if (e == "aio") backend_ = kAio;
                if (e == "uring" && uring_available()) backend_ = kUring;
            }
        } else if (backend_ == kUring && !uring_available()) {
            fail(MA_ERR_CAPABILITY, "io_uring is not available (kernel or sandbox policy)");
        } else if (backend_ != kSync && backend_ != kAio && backend_ != kUring) {
            fail(MA_ERR_INVALID_ARGUMENT, "unknown I/O backend");
        }
        cursor_ = std::make_unique<Cursor>(static_cast<std::uint32_t>(specs_.size()));
        if (!cfg_.manifest.empty() && std::filesystem::exists(cfg_.manifest)) load_manifest();
    } catch (...) {
        for (int fd : fds_) ::close(fd);
        throw;
    }
    for (std::uint32_t w = 0; w < cfg_.workers; ++w) {
        if (backend_ == kUring)
            workers_.emplace_back([this] { worker_uring(); });
        else
            workers_.emplace_back([this] { worker_blocking(); });
    }
}

Engine::~Engine() {
    {
        std::lock_guard<std::mutex> lock(q_mu_);
        stopping_ = true;
    }
    q_cv_.notify_all();
    for (auto& t : workers_) t.join();
    if (!cfg_.manifest.empty()) {
        try {
            save_manifest();
        } catch (const Failure&) {
            // destructor: save_manifest() called explicitly is the reporting path
        }
    }
    for (int fd : fds_) ::close(fd);
}

std::vector<Extent> Engine::allocate(const std::string& key, std::uint64_t logical) {
    if (logical == 0) fail(MA_ERR_INVALID_ARGUMENT, "cannot allocate zero bytes for '" + key + "'");
    const std::uint64_t padded = align_up(logical, kGranule);
    {
        std::lock_guard<std::mutex> lock(table_mu_);
        auto it = table_.find(key);
        if (it != table_.end()) {
            if (padded <= it->second.padded) {
                it->second.logical = logical;
                return it->second.extents;
            }
            stats_.abandoned_bytes += it->second.padded;
            table_.erase(it);
        }
    }
    // equal split in granules; the first (granules % devices) devices take one more
    const std::uint32_t nd = static_cast<std::uint32_t>(specs_.size());
    const std::uint64_t granules = padded / kGranule;
    Location loc;
    loc.logical = logical;
    loc.padded = padded;
    for (std::uint32_t d = 0; d < nd; ++d) {
        const std::uint64_t g = granules / nd + (d < granules % nd ? 1 : 0);
        if (g == 0) continue;
        const std::uint64_t bytes = g * kGranule;
        const std::uint64_t off = cursor_->advance(d, bytes);
        if (off + bytes > specs_[d].capacity)
            fail(MA_ERR_STORAGE_FULL,
                 "device '" + specs_[d].path + "' exhausted while allocating '" + key + "'");
        loc.extents.push_back({d, off, bytes});
    }
    std::lock_guard<std::mutex> lock(table_mu_);
    auto res = table_.emplace(key, loc);
    if (!res.second) fail(MA_ERR_INVALID_ARGUMENT, "concurrent allocation for key '" + key + "'");
    return loc.extents;
}

Op* Engine::submit(const std::string& key, char* buf, std::uint64_t buf_bytes, bool write,
                   std::uint64_t logical) {
    {
        std::lock_guard<std::mutex> lock(table_mu_);
        if (!busy_.insert(key).second)
            fail(MA_ERR_BUSY, "concurrent operation on key '" + key + "'");
    }
    auto release = [&] {
        std::lock_guard<std::mutex> lock(table_mu_);
        busy_.erase(key);
    };
    std::unique_ptr<Op> op(new Op);
    op->engine = this;
    op->key = key;
    op->write = write;
    std::vector<Task> tasks;
    TraceFn trace;
    try {
        if (write) {
            allocate(key, logical);
            std::lock_guard<std::mutex> lock(table_mu_);
            op->loc = table_.at(key);
        } else {
            {
                std::lock_guard<std::mutex> lock(table_mu_);
                auto it = table_.find(key);
                if (it == table_.end()) fail(MA_ERR_NOT_FOUND, "key '" + key + "' was never written");
                op->loc = it->second;
            }
            if (buf_bytes < op->loc.padded)
                fail(MA_ERR_SIZE_VIOLATION, "read destination for '" + key + "' must cover " +
                                                std::to_string(op->loc.padded) + " padded bytes");
        }
        // Bytes moved: the tensor's padded LOGICAL length.  A key rewritten
        // smaller keeps its larger extents (reuse, like the reference), but
        // only the granules the payload occupies are transferred — the
        // caller's buffer need not cover the old extents.  The payload maps
        // onto the extents in order.
        const std::uint64_t move = std::min(align_up(op->loc.logical, kGranule), op->loc.padded);
        op->bytes = move;
        // each extent in `workers` granule-aligned chunks, one task each
        std::uint64_t at_buf = 0;
        for (const Extent& e : op->loc.extents) {
            if (at_buf >= move) break;
            const std::uint64_t len = std::min(e.length, move - at_buf);
            const std::uint64_t chunk = align_up((len + cfg_.workers - 1) / cfg_.workers, kGranule);
            for (std::uint64_t at = 0; at < len; at += chunk) {
                Task t;
                t.fd = fds_[e.device];
                t.device = e.device;
                t.offset = e.offset + at;
                t.buf = buf + at_buf + at;
                t.length = std::min(chunk, len - at);
                t.write = write;
                t.op = op.get();
                tasks.push_back(t);
            }
            at_buf += e.length;
        }
        std::lock_guard<std::mutex> lock(table_mu_);
        trace = trace_;
    } catch (...) {
        release();
        throw;
    }
    if (trace)
        for (const Task& t : tasks) trace(t.device, t.offset, t.length, t.write);
    op->pending = op->tasks = tasks.size();
    {
        std::lock_guard<std::mutex> lock(q_mu_);
        for (const Task& t : tasks) queue_.push_back(t);
    }
    q_cv_.notify_all();
    return op.release();
}

Op* Engine::submit_write(const std::string& key, const void* src, std::uint64_t src_bytes,
                         std::uint64_t logical) {
    if (logical == 0) fail(MA_ERR_INVALID_ARGUMENT, "zero-length write for '" + key + "'");
    if (!aligned_ptr(src))
        fail(MA_ERR_ALIGNMENT, "write source for '" + key + "' is not 4096-aligned");
    const std::uint64_t padded = align_up(logical, kGranule);
    if (src_bytes < padded)
        fail(MA_ERR_SIZE_VIOLATION, "write source for '" + key + "' must cover " +
                                        std::to_string(padded) + " padded bytes");
    return submit(key, static_cast<char*>(const_cast<void*>(src)), src_bytes, true, logical);
}

Op* Engine::submit_read(const std::string& key, void* dst, std::uint64_t dst_bytes) {
    if (!aligned_ptr(dst))
        fail(MA_ERR_ALIGNMENT, "read destination for '" + key + "' is not 4096-aligned");
    return submit(key, static_cast<char*>(dst), dst_bytes, false, 0);
}

std::uint64_t Engine::wait(Op* op) {
    std::unique_ptr<Op> own(op);
    {
        std::unique_lock<std::mutex> lock(op->mu);
        op->cv.wait(lock, [&] { return op->pending == 0; });
    }
    std::lock_guard<std::mutex> lock(table_mu_);
    busy_.erase(op->key);
    if (!op->error.empty()) fail(MA_ERR_IO_ERROR, op->error);
    stats_.submitted_ios += op->tasks;
    if (op->write) {
        stats_.bytes_written += op->bytes;
        stats_.write_requests += 1;
    } else {
        stats_.bytes_read += op->bytes;
        stats_.read_requests += 1;
    }
    return op->loc.logical;
}

bool Engine::pop_task(Task* t, bool block) {
    std::unique_lock<std::mutex> lock(q_mu_);
    if (block) q_cv_.wait(lock, [&] { return stopping_ || !queue_.empty(); });
    if (queue_.empty()) return false;
    *t = queue_.front();
    queue_.pop_front();
    return true;
}

void Engine::finish_task(const Task& t, const std::string& error) {
    std::lock_guard<std::mutex> lock(t.op->mu);
    if (!error.empty() && t.op->error.empty()) t.op->error = error;
    if (--t.op->pending == 0) t.op->cv.notify_all();
}

void Engine::worker_blocking() {
    for (;;) {
        Task t;
        if (!pop_task(&t, true)) {
            std::lock_guard<std::mutex> lock(q_mu_);
            if (stopping_ && queue_.empty()) return;
            continue;
        }
        std::string err;
        try {
            if (backend_ == kAio)
                run_aio(t);
            else
                run_sync(t);
        } catch (const Failure& f) {
            err = f.msg;
        }
        finish_task(t, err);
    }
}

void Engine::run_sync(const Task& t) {
    for (std::uint64_t done = 0; done < t.length;) {
        const ssize_t n = t.write ? ::pwrite(t.fd, t.buf + done, t.length - done,
                                             static_cast<off_t>(t.offset + done))
                                  : ::pread(t.fd, t.buf + done, t.length - done,
                                            static_cast<off_t>(t.offset + done));
        if (n < 0 && errno == EINTR) continue;
        if (n <= 0)
            fail(MA_ERR_IO_ERROR, std::string(t.write ? "short write" : "short read") +
                                      " on device " + std::to_string(t.device) + " at offset " +
                                      std::to_string(t.offset + done) + ": " +
                                      (n < 0 ? std::strerror(errno) : "eof"));
        done += static_cast<std::uint64_t>(n);
    }
}

void Engine::run_aio(const Task& t) {
    // up to queue_depth concurrent granule-aligned slices via lio_listio
    const std::uint64_t qd = cfg_.queue_depth;
    const std::uint64_t slice = align_up((t.length + qd - 1) / qd, kGranule);
    std::vector<aiocb> cbs;
    for (std::uint64_t at = 0; at < t.length; at += slice) {
        aiocb cb;
        std::memset(&cb, 0, sizeof cb);
        cb.aio_fildes = t.fd;
        cb.aio_offset = static_cast<off_t>(t.offset + at);
        cb.aio_buf = t.buf + at;
        cb.aio_nbytes = std::min(slice, t.length - at);
        cb.aio_lio_opcode = t.write ? LIO_WRITE : LIO_READ;
        cbs.push_back(cb);
    }
    std::vector<aiocb*> list;
    for (auto& cb : cbs) list.push_back(&cb);
    if (::lio_listio(LIO_WAIT, list.data(), static_cast<int>(list.size()), nullptr) != 0 &&
        errno != EIO && errno != EINTR) {
        // EAGAIN: none or some queued; never leave queued requests behind
        const int e = errno;
        for (auto& cb : cbs) {
            while (::aio_error(&cb) == EINPROGRESS) {
                const aiocb* one[1] = {&cb};
                ::aio_suspend(one, 1, nullptr);
            }
            ::aio_return(&cb);
        }
        fail(MA_ERR_IO_ERROR, std::string("lio_listio failed: ") + std::strerror(e));
    }
    // a signal can end LIO_WAIT early: wait for every request to finish
    for (auto& cb : cbs) {
        while (::aio_error(&cb) == EINPROGRESS) {
            const aiocb* one[1] = {&cb};
            ::aio_suspend(one, 1, nullptr);
        }
    }
    for (auto& cb : cbs) {
        const int e = ::aio_error(&cb);
        const ssize_t n = ::aio_return(&cb);
        if (e != 0 || n != static_cast<ssize_t>(cb.aio_nbytes))
            fail(MA_ERR_IO_ERROR, std::string("aio ") + (t.write ? "write" : "read") +
                                      " failed on device " + std::to_string(t.device) + ": " +
                                      (e != 0 ? std::strerror(e) : "short transfer"));
    }
}

void Engine::worker_uring() {
    // One ring per worker, up to queue_depth requests in flight ACROSS tasks:
    // each task is cut into granule-aligned pieces (at most queue_depth per
    // task, at most 8 MiB each) and the ring is kept full from the queue.
    struct Rec {
        Task t;
        std::uint64_t remaining = 0;
        std::string err;
    };
    struct Piece {
        Rec* rec;
        char* buf;
        std::uint64_t off;
        std::uint64_t len;
    };
    const unsigned depth = std::max(1u, cfg_.queue_depth);
    Ring ring;
    const bool ring_ok = ring.init(std::max(depth, 4u));
    std::deque<Piece*> ready;
    unsigned inflight = 0;
    auto close_piece = [&](Piece* p, const std::string& err) {
        Rec* r = p->rec;
        if (!err.empty() && r->err.empty()) r->err = err;
        delete p;
        if (--r->remaining == 0) {
            finish_task(r->t, r->err);
            delete r;
        }
    };
    for (;;) {
        {
            std::unique_lock<std::mutex> lock(q_mu_);
            if (ready.empty() && inflight == 0) {
                q_cv_.wait(lock, [&] { return stopping_ || !queue_.empty(); });
                if (queue_.empty()) return;  // stopping, drained
            }
            while (ready.size() < depth && !queue_.empty()) {
                Rec* r = new Rec;
                r->t = queue_.front();
                queue_.pop_front();
                const std::uint64_t piece = std::min<std::uint64_t>(
                    8ull << 20, align_up((r->t.length + depth - 1) / depth, kGranule));
                for (std::uint64_t at = 0; at < r->t.length; at += piece) {
                    ready.push_back(new Piece{r, r->t.buf + at, r->t.offset + at,
                                              std::min(piece, r->t.length - at)});
                    r->remaining += 1;
                }
            }
        }
        if (!ring_ok) {
            while (!ready.empty()) {
                close_piece(ready.front(), "io_uring ring setup failed in worker");
                ready.pop_front();
            }
            continue;
        }
        std::vector<Piece*> batch;
        while (inflight < depth && !ready.empty()) {
            Piece* p = ready.front();
            ready.pop_front();
            ring.prep(p->rec->t.write, p->rec->t.fd, p->buf, static_cast<unsigned>(p->len),
                      p->off, p);
            batch.push_back(p);
            ++inflight;
        }
        unsigned unsubmitted = 0;
        const int rc = ring.enter(static_cast<unsigned>(batch.size()), inflight ? 1 : 0,
                                  &unsubmitted);
        if (rc < 0) {
            // the entries the kernel did not take fail; what it took completes normally
            const std::string err = std::string("io_uring_enter: ") + std::strerror(-rc);
            for (size_t k = batch.size() - unsubmitted; k < batch.size(); ++k) {
                close_piece(batch[k], err);
                --inflight;
            }
            while (!ready.empty()) {
                close_piece(ready.front(), err);
                ready.pop_front();
            }
        }
        ring.reap([&](void* u, int res) {
            Piece* p = static_cast<Piece*>(u);
            --inflight;
            const Task& t = p->rec->t;
            if (res == -EINTR || res == -EAGAIN) {
                ready.push_front(p);  // transient: resubmit as is
            } else if (res < 0) {
                close_piece(p, std::string("io_uring ") + (t.write ? "write" : "read") +
                                   " failed on device " + std::to_string(t.device) +
                                   " at offset " + std::to_string(p->off) + ": " +
                                   std::strerror(-res));
            } else if (res == 0) {
                close_piece(p, std::string(t.write ? "short write" : "short read") +
                                   " on device " + std::to_string(t.device) + " at offset " +
                                   std::to_string(p->off) + ": eof");
            } else if (static_cast<std::uint64_t>(res) < p->len) {
                p->buf += res;  // resubmit the remainder
                p->off += static_cast<std::uint64_t>(res);
                p->len -= static_cast<std::uint64_t>(res);
                ready.push_front(p);
            } else {
                close_piece(p, "");
            }
        });
    }
}

bool Engine::contains(const std::string& key) const {
    std::lock_guard<std::mutex> lock(table_mu_);
    return table_.count(key) != 0;
}

Location Engine::location(const std::string& key) const {
    std::lock_guard<std::mutex> lock(table_mu_);
    auto it = table_.find(key);
    if (it == table_.end()) fail(MA_ERR_NOT_FOUND, "key '" + key + "' has no location");
    return it->second;
}

std::vector<std::pair<std::string, Location>> Engine::locations() const {
    std::lock_guard<std::mutex> lock(table_mu_);
    return {table_.begin(), table_.end()};
}

Stats Engine::stats() const {
    std::lock_guard<std::mutex> lock(table_mu_);
    return stats_;
}

void Engine::set_trace(TraceFn fn) {
    std::lock_guard<std::mutex> lock(table_mu_);
    trace_ = std::move(fn);
}

void Engine::save_manifest() const {
    if (cfg_.manifest.empty()) fail(MA_ERR_INVALID_ARGUMENT, "engine has no manifest path configured");
    std::ostringstream o;
    o << "{\n  \"version\": 1,\n  \"devices\": [";
    for (size_t d = 0; d < specs_.size(); ++d) {
        o << (d ? ",\n" : "\n") << "    {\"path\": " << jstr(specs_[d].path)
          << ", \"capacity_bytes\": " << specs_[d].capacity << ", \"kind\": "
          << (specs_[d].kind == 0 ? "\"raw_block\"" : "\"file_backed_virtual\"") << "}";
    }
    o << "\n  ],\n  \"cursors\": [";
    for (std::uint32_t d = 0; d < specs_.size(); ++d) o << (d ? ", " : "") << cursor_->position(d);
    o << "],\n  \"tensors\": {";
    {
        std::lock_guard<std::mutex> lock(table_mu_);
        bool first = true;
        for (const auto& kv : table_) {
            o << (first ? "\n" : ",\n") << "    " << jstr(kv.first) << ": {\"logical\": "
              << kv.second.logical << ", \"padded\": " << kv.second.padded << ", \"extents\": [";
            for (size_t i = 0; i < kv.second.extents.size(); ++i) {
                const Extent& e = kv.second.extents[i];
                o << (i ? ", " : "") << "{\"device\": " << e.device << ", \"offset\": " << e.offset
                  << ", \"length\": " << e.length << "}";
            }
            o << "]}";
            first = false;
        }
    }
    o << "\n  }\n}\n";
    const std::string tmp = cfg_.manifest + ".tmp";
    {
        std::ofstream out(tmp, std::ios::trunc);
        if (!out.good()) fail(MA_ERR_IO_ERROR, "cannot write manifest '" + tmp + "'");
        out << o.str();
        if (!out.good()) fail(MA_ERR_IO_ERROR, "cannot write manifest '" + tmp + "'");
    }
    std::error_code ec;
    std::filesystem::rename(tmp, cfg_.manifest, ec);
    if (ec) fail(MA_ERR_IO_ERROR, "cannot rename manifest into '" + cfg_.manifest + "'");
}

void Engine::load_manifest() {
    std::ifstream in(cfg_.manifest);
    if (!in.good()) fail(MA_ERR_IO_ERROR, "cannot read manifest '" + cfg_.manifest + "'");
    std::stringstream ss;
    ss << in.rdbuf();
    const std::string text = ss.str();
    const JVal j = JParser(text).parse();
    if (j.kind != JVal::Obj) fail(MA_ERR_BAD_CONFIG, "malformed manifest: not an object");
    const JVal* ver = j.find("version");
    if (!ver || ver->kind != JVal::Num || ver->num != 1)
        fail(MA_ERR_BAD_CONFIG, "unsupported manifest version");
    const JVal& devs = j.at("devices");
    if (devs.arr.size() != specs_.size())
        fail(MA_ERR_BAD_CONFIG, "manifest device count does not match the engine's");
    for (size_t d = 0; d < specs_.size(); ++d)
        if (devs.arr[d].at("path").s() != specs_[d].path)
            fail(MA_ERR_BAD_CONFIG, "manifest device order mismatch at index " + std::to_string(d));
    const JVal& cur = j.at("cursors");
    if (cur.arr.size() < specs_.size()) fail(MA_ERR_BAD_CONFIG, "malformed manifest: cursors");
    for (std::uint32_t d = 0; d < specs_.size(); ++d) cursor_->restore(d, cur.arr[d].u64());
    for (const auto& kv : j.at("tensors").obj) {
        Location loc;
        loc.logical = kv.second.at("logical").u64();
        loc.padded = kv.second.at("padded").u64();
        for (const JVal& e : kv.second.at("extents").arr)
            loc.extents.push_back({static_cast<std::uint32_t>(e.at("device").u64()),
                                   e.at("offset").u64(), e.at("length").u64()});
        table_[kv.first] = std::move(loc);
    }
}

std::vector<DeviceSpec> Engine::create_virtual_devices(const std::string& dir, std::uint32_t count,
                                                       std::uint64_t bytes) {
    if (count == 0 || bytes == 0 || bytes % kGranule)
        fail(MA_ERR_INVALID_ARGUMENT,
             "virtual devices need a positive count and a 4096-multiple size");
    std::error_code ec;
    std::filesystem::create_directories(dir, ec);
    std::vector<DeviceSpec> out;
    for (std::uint32_t d = 0; d < count; ++d) {
        const std::string path = dir + "/vdev" + std::to_string(d) + ".img";
        const int fd = ::open(path.c_str(), O_CREAT | O_RDWR | O_CLOEXEC, 0644);
        if (fd < 0) fail(MA_ERR_DEVICE_ERROR, "cannot create virtual device '" + path + "'");
        if (::posix_fallocate(fd, 0, static_cast<off_t>(bytes)) != 0 &&
            ::ftruncate(fd, static_cast<off_t>(bytes)) != 0) {
            ::close(fd);
            fail(MA_ERR_DEVICE_ERROR, "cannot size virtual device '" + path + "'");
        }
        ::close(fd);
        out.push_back({path, bytes, 1});
    }
    return out;
}

}  // namespace swp
}  // namespace ma

// ================================================================ C ABI
using ma::swp::Engine;
using ma::swp::Failure;

struct ma_swap_op {
    ma::swp::Op* op;
    Engine* e;
};
struct ma_cursor {
    ma::swp::Cursor* c;
};

namespace {

template <typename F>
int guard(F&& fn) {
    try {
        fn();
        return MA_OK;
    } catch (const Failure& f) {
        ma::set_error(f.msg);
        return f.code;
    } catch (const std::bad_alloc&) {
        ma::set_error("host allocation failed");
        return MA_ERR_OUT_OF_MEMORY;
    } catch (const std::exception& e) {
        ma::set_error(e.what());
        return MA_ERR_DEVICE_ERROR;
    }
}

void need(bool ok, const char* what) {
    if (!ok) ma::swp::fail(MA_ERR_INVALID_ARGUMENT, what);
}

void put_extents(const std::vector<ma::swp::Extent>& ex, ma_swap_extent* out, uint32_t cap,
                 uint32_t* count) {
    if (count) *count = static_cast<uint32_t>(ex.size());
    if (!out) return;
    for (size_t i = 0; i < ex.size() && i < cap; ++i)
        out[i] = ma_swap_extent{ex[i].device, ex[i].offset, ex[i].length};
}

}  // namespace

extern "C" {

int ma_swap_create(const ma_swap_device* devs, uint32_t ndev, const ma_swap_config* cfg,
                   ma_swap** out) {
    return guard([&] {
        need(out != nullptr, "null output");
        need(ndev == 0 || devs != nullptr, "null device list");
        std::vector<ma::swp::DeviceSpec> specs;
        for (uint32_t d = 0; d < ndev; ++d) {
            need(devs[d].path != nullptr, "null device path");
            specs.push_back({devs[d].path, devs[d].capacity_bytes, devs[d].kind});
        }
        ma::swp::Config c;
        if (cfg) {
            c.workers = cfg->workers;
            c.queue_depth = cfg->queue_depth;
            c.backend = cfg->backend;
            c.cache_bypass = cfg->cache_bypass != 0;
            c.manifest = cfg->manifest_path ? cfg->manifest_path : "";
        }
        *out = new ma_swap{new Engine(std::move(specs), std::move(c))};
    });
}

int ma_swap_destroy(ma_swap* s) {
    return guard([&] {
        if (!s) return;
        delete s->e;
        delete s;
    });
}

int ma_swap_allocate(ma_swap* s, const char* key, uint64_t logical_bytes, ma_swap_extent* out,
                     uint32_t cap, uint32_t* count) {
    return guard([&] {
        need(s && key, "null argument");
        put_extents(s->e->allocate(key, logical_bytes), out, cap, count);
    });
}

int ma_swap_write_async(ma_swap* s, const char* key, const void* src, uint64_t src_bytes,
                        uint64_t logical_bytes, ma_swap_op** op) {
    return guard([&] {
        need(s && key && op, "null argument");
        *op = new ma_swap_op{s->e->submit_write(key, src, src_bytes, logical_bytes), s->e};
    });
}

int ma_swap_read_async(ma_swap* s, const char* key, void* dst, uint64_t dst_bytes,
                       ma_swap_op** op) {
    return guard([&] {
        need(s && key && op, "null argument");
        *op = new ma_swap_op{s->e->submit_read(key, dst, dst_bytes), s->e};
    });
}

int ma_swap_wait(ma_swap_op* op, uint64_t* logical_bytes) {
    return guard([&] {
        need(op != nullptr, "null op");
        std::unique_ptr<ma_swap_op> own(op);
        const uint64_t n = op->e->wait(op->op);
        if (logical_bytes) *logical_bytes = n;
    });
}

int ma_swap_write(ma_swap* s, const char* key, const void* src, uint64_t src_bytes,
                  uint64_t logical_bytes) {
    return guard([&] {
        need(s && key, "null argument");
        s->e->wait(s->e->submit_write(key, src, src_bytes, logical_bytes));
    });
}

int ma_swap_read(ma_swap* s, const char* key, void* dst, uint64_t dst_bytes,
                 uint64_t* logical_bytes) {
    return guard([&] {
        need(s && key, "null argument");
        const uint64_t n = s->e->wait(s->e->submit_read(key, dst, dst_bytes));
        if (logical_bytes) *logical_bytes = n;
    });
}

int ma_swap_contains(ma_swap* s, const char* key, int* out) {
    return guard([&] {
        need(s && key && out, "null argument");
        *out = s->e->contains(key) ? 1 : 0;
    });
}

int ma_swap_location(ma_swap* s, const char* key, uint64_t* logical, uint64_t* padded,
                     ma_swap_extent* out, uint32_t cap, uint32_t* count) {
    return guard([&] {
        need(s && key, "null argument");
        const ma::swp::Location loc = s->e->location(key);
        if (logical) *logical = loc.logical;
        if (padded) *padded = loc.padded;
        put_extents(loc.extents, out, cap, count);
    });
}

int ma_swap_keys(ma_swap* s, char* buf, uint64_t cap, uint64_t* needed) {
    return guard([&] {
        need(s && needed, "null argument");
        std::string all;
        for (const auto& kv : s->e->locations()) {
            all += kv.first;
            all.push_back('\0');
        }
        *needed = all.size();
        if (buf && cap >= all.size()) std::memcpy(buf, all.data(), all.size());
    });
}

int ma_swap_get_stats(ma_swap* s, ma_swap_stats* out) {
    return guard([&] {
        need(s && out, "null argument");
        const ma::swp::Stats st = s->e->stats();
        *out = ma_swap_stats{st.bytes_written, st.bytes_read,    st.write_requests,
                             st.read_requests, st.submitted_ios, st.abandoned_bytes};
    });
}

int ma_swap_info(ma_swap* s, int* backend, uint64_t* total_capacity, uint32_t* device_count) {
    return guard([&] {
        need(s != nullptr, "null engine");
        if (backend) *backend = s->e->backend();
        if (total_capacity) *total_capacity = s->e->total_capacity();
        if (device_count) *device_count = s->e->device_count();
    });
}

int ma_swap_set_trace(ma_swap* s, ma_io_trace_fn fn, void* user) {
    return guard([&] {
        need(s != nullptr, "null engine");
        if (!fn) {
            s->e->set_trace(nullptr);
            return;
        }
        s->e->set_trace([fn, user](uint32_t d, uint64_t off, uint64_t len, bool w) {
            fn(user, d, off, len, w ? 1 : 0);
        });
    });
}

int ma_swap_save_manifest(ma_swap* s) {
    return guard([&] {
        need(s != nullptr, "null engine");
        s->e->save_manifest();
    });
}

int ma_swap_create_virtual_devices(const char* dir, uint32_t count, uint64_t bytes) {
    return guard([&] {
        need(dir != nullptr, "null directory");
        Engine::create_virtual_devices(dir, count, bytes);
    });
}

int ma_swap_uring_available(void) { return Engine::uring_available() ? 1 : 0; }

int ma_cursor_open(uint32_t devices, const char* path, ma_cursor** out) {
    return guard([&] {
        need(out != nullptr, "null output");
        *out = new ma_cursor{new ma::swp::Cursor(devices, path ? path : "")};
    });
}

int ma_cursor_close(ma_cursor* c) {
    return guard([&] {
        if (!c) return;
        delete c->c;
        delete c;
    });
}

int ma_cursor_advance(ma_cursor* c, uint32_t device, uint64_t bytes, uint64_t* old) {
    return guard([&] {
        need(c && old, "null argument");
        *old = c->c->advance(device, bytes);
    });
}

int ma_cursor_position(ma_cursor* c, uint32_t device, uint64_t* pos) {
    return guard([&] {
        need(c && pos, "null argument");
        *pos = c->c->position(device);
    });
}

int ma_cursor_restore(ma_cursor* c, uint32_t device, uint64_t pos) {
    return guard([&] {
        need(c != nullptr, "null cursor");
        c->c->restore(device, pos);
    });
}

}  // extern "C"
