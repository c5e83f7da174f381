// Internal: the host-side swap engine behind ma_swap_* (include/memascend_b200.h)
// and the drop-in memascend::DirectIoEngine (include/memascend/direct_io.hpp).
//
// Behaviour follows the reference's DirectIoEngine (proj/include/memascend/
// direct_io.hpp:23-180, proj/src/direct_io.cpp): a key-addressed tensor store
// over raw or file-backed devices opened with O_DIRECT, every payload padded to
// 4096 and split in equal granule counts across the device set, space claimed
// once per key through per-device cursors (grow = fresh extents, old ones
// abandoned), a per-key busy guard, a worker pool, a JSON manifest.
//
// What is different here is the submission path and the asynchrony the B200
// pipeline needs (ma_stepper_apply_swapped streams optimizer state
// NVMe -> registered host slot -> HBM and back):
//   * an io_uring backend (raw syscalls, one ring per worker, many requests
//     in flight per worker across tasks) beside the synchronous pread/pwrite
//     and POSIX-AIO (lio_listio) backends; auto_probe picks io_uring when the
//     kernel allows it;
//   * submit_read / submit_write return an Op the caller waits on later, so
//     reads of group i+1 and write-backs of group i-1 overlap the GPU update
//     of group i.  The blocking read/write are submit + wait.
#pragma once

#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <deque>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <set>
#include <string>
#include <thread>
#include <vector>

namespace ma {
namespace swp {

constexpr std::uint64_t kGranule = 4096;

// status codes are the C ABI's (1 + memascend::ErrorCode)
struct Failure {
    int code;
    std::string msg;
};
[[noreturn]] void fail(int code, const std::string& msg);

enum Backend { kAuto = 0, kSync = 1, kAio = 2, kUring = 3 };

struct DeviceSpec {
    std::string path;
    std::uint64_t capacity = 0;
    int kind = 1;  // 0 raw_block, 1 file_backed_virtual
};

struct Extent {
    std::uint32_t device = 0;
    std::uint64_t offset = 0;
    std::uint64_t length = 0;
};

struct Location {
    std::uint64_t logical = 0;
    std::uint64_t padded = 0;
    std::vector<Extent> extents;
};

struct Stats {
    std::uint64_t bytes_written = 0;
    std::uint64_t bytes_read = 0;
    std::uint64_t write_requests = 0;
    std::uint64_t read_requests = 0;
    std::uint64_t submitted_ios = 0;
    std::uint64_t abandoned_bytes = 0;
};

struct Config {
    std::uint32_t workers = 2;
    std::uint32_t queue_depth = 8;
    int backend = kAuto;
    bool cache_bypass = true;
    std::string manifest;
};

// Per-device next-free offsets (SharedCursor, direct_io.hpp:69-92).  With a
// path, every advance is a read-modify-write of the on-disk counters under
// flock, so cooperating processes never claim overlapping spans.
class Cursor {
public:
    explicit Cursor(std::uint32_t devices, const std::string& path = "");
    ~Cursor();
    Cursor(const Cursor&) = delete;
    Cursor& operator=(const Cursor&) = delete;
    std::uint64_t advance(std::uint32_t device, std::uint64_t bytes);
    std::uint64_t position(std::uint32_t device) const;
    void restore(std::uint32_t device, std::uint64_t pos);
    std::uint32_t devices() const { return static_cast<std::uint32_t>(local_.size()); }

private:
    mutable std::mutex mu_;
    std::vector<std::atomic<std::uint64_t>> local_;
    int fd_ = -1;
};

using TraceFn = std::function<void(std::uint32_t, std::uint64_t, std::uint64_t, bool)>;

class Engine;

// One tensor-level operation in flight.  Created by submit_*, consumed by
// Engine::wait (which frees it).
struct Op {
    Engine* engine = nullptr;
    std::string key;
    bool write = false;
    Location loc;
    std::mutex mu;
    std::condition_variable cv;
    std::uint64_t pending = 0;
    std::uint64_t tasks = 0;
    std::uint64_t bytes = 0;  // transferred (padded logical length)
    std::string error;
};

class Engine {
public:
    Engine(std::vector<DeviceSpec> devices, Config cfg);
    ~Engine();
    Engine(const Engine&) = delete;
    Engine& operator=(const Engine&) = delete;

    std::vector<Extent> allocate(const std::string& key, std::uint64_t logical);
    Op* submit_write(const std::string& key, const void* src, std::uint64_t src_bytes,
                     std::uint64_t logical);
    Op* submit_read(const std::string& key, void* dst, std::uint64_t dst_bytes);
    // Blocks until the op's device I/O is complete, releases its key, frees
    // it; returns the logical length (reads) and throws Failure on error.
    std::uint64_t wait(Op* op);

    bool contains(const std::string& key) const;
    Location location(const std::string& key) const;
    std::vector<std::pair<std::string, Location>> locations() const;
    Stats stats() const;
    int backend() const { return backend_; }
    std::uint64_t total_capacity() const { return total_capacity_; }
    std::uint32_t device_count() const { return static_cast<std::uint32_t>(fds_.size()); }
    void set_trace(TraceFn fn);
    void save_manifest() const;

    static std::vector<DeviceSpec> create_virtual_devices(const std::string& dir,
                                                          std::uint32_t count,
                                                          std::uint64_t bytes);
    static bool uring_available();

private:
    struct Task {
        int fd = -1;
        std::uint32_t device = 0;
        std::uint64_t offset = 0;
        char* buf = nullptr;
        std::uint64_t length = 0;
        bool write = false;
        Op* op = nullptr;
    };

    Op* submit(const std::string& key, char* buf, std::uint64_t buf_bytes, bool write,
               std::uint64_t logical);
    void worker_blocking();
    void worker_uring();
    bool pop_task(Task* t, bool block);
    void run_sync(const Task& t);
    void run_aio(const Task& t);
    void finish_task(const Task& t, const std::string& error);
    void load_manifest();

    std::vector<DeviceSpec> specs_;
    std::vector<int> fds_;
    std::uint64_t total_capacity_ = 0;
    Config cfg_;
    int backend_ = kSync;
    std::unique_ptr<Cursor> cursor_;

    mutable std::mutex table_mu_;
    std::map<std::string, Location> table_;
    std::set<std::string> busy_;
    Stats stats_;
    TraceFn trace_;

    std::mutex q_mu_;
    std::condition_variable q_cv_;
    std::deque<Task> queue_;
    bool stopping_ = false;
    std::vector<std::thread> workers_;
};

}  // namespace swp
}  // namespace ma

struct ma_swap {
    ma::swp::Engine* e;
};
