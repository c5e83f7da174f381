// Drop-in memascend::DirectIoEngine / SharedCursor / FsBaselineStore
// (include/memascend/direct_io.hpp) over the C ABI's swap store.
//
// Reference: proj/include/memascend/direct_io.hpp:19-180, proj/src/direct_io.cpp.
// FsBaselineStore (direct_io.cpp:606-716: one O_DIRECT file per key, trimmed
// to the logical length) is plain host file I/O and lives here directly.
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <cctype>
#include <cerrno>
#include <cstring>
#include <filesystem>

#include "memascend/direct_io.hpp"
#include "memascend/error.hpp"
#include "memascend_b200.h"

namespace memascend {

namespace {

void check(int status) {
    if (status == MA_OK) return;
    const std::string msg = ma_last_error();
    if (status >= 1 && status <= 17) raise(static_cast<ErrorCode>(status - 1), msg);
    raise(ErrorCode::device_error, msg);
}

std::uint64_t align_up(std::uint64_t v, std::uint64_t a) { return (v + a - 1) / a * a; }

std::vector<Extent> to_extents(const std::vector<ma_swap_extent>& v, std::uint32_t n) {
    std::vector<Extent> out;
    for (std::uint32_t i = 0; i < n; ++i)
        out.push_back({v[i].device_index, v[i].device_offset, v[i].length});
    return out;
}

void trace_trampoline(void* user, uint32_t device, uint64_t offset, uint64_t length, int write) {
    (*static_cast<IoTraceFn*>(user))(device, offset, length, write != 0);
}

}  // namespace

// ------------------------------------------------------------ SharedCursor
SharedCursor::SharedCursor(std::uint32_t device_count) {
    check(ma_cursor_open(device_count, nullptr, &c_));
}

SharedCursor::SharedCursor(std::uint32_t device_count, const std::string& path) {
    check(ma_cursor_open(device_count, path.c_str(), &c_));
}

SharedCursor::~SharedCursor() {
    if (c_) ma_cursor_close(c_);
}

std::uint64_t SharedCursor::advance(std::uint32_t device, std::uint64_t bytes) {
    if (!c_) raise(ErrorCode::invalid_argument, "cursor device index out of range");
    std::uint64_t old = 0;
    check(ma_cursor_advance(c_, device, bytes, &old));
    return old;
}

std::uint64_t SharedCursor::position(std::uint32_t device) const {
    if (!c_) raise(ErrorCode::invalid_argument, "cursor device index out of range");
    std::uint64_t pos = 0;
    check(ma_cursor_position(c_, device, &pos));
    return pos;
}

void SharedCursor::restore(std::uint32_t device, std::uint64_t position) {
    if (!c_) raise(ErrorCode::invalid_argument, "cursor device index out of range");
    check(ma_cursor_restore(c_, device, position));
}

// ------------------------------------------------------------ DirectIoEngine
DirectIoEngine::DirectIoEngine(DeviceSet devset, EngineConfig config) {
    std::vector<ma_swap_device> devs;
    for (const auto& d : devset.devices)
        devs.push_back({d.path.c_str(), d.capacity_bytes, d.kind == DeviceKind::raw_block ? 0 : 1});
    ma_swap_config cfg{};
    cfg.workers = config.workers;
    cfg.queue_depth = config.queue_depth;
    cfg.backend = config.backend == IoBackend::sync_pio    ? MA_IO_SYNC
                  : config.backend == IoBackend::posix_aio ? MA_IO_POSIX_AIO
                  : config.backend == IoBackend::io_uring  ? MA_IO_URING
                                                           : MA_IO_AUTO;
    cfg.cache_bypass = config.cache_bypass ? 1 : 0;
    cfg.manifest_path = config.manifest_path.c_str();
    check(ma_swap_create(devs.data(), static_cast<uint32_t>(devs.size()), &cfg, &h_));
    int backend = 0;
    check(ma_swap_info(h_, &backend, &total_capacity_, &device_count_));
    backend_ = backend == MA_IO_SYNC        ? IoBackend::sync_pio
               : backend == MA_IO_POSIX_AIO ? IoBackend::posix_aio
                                            : IoBackend::io_uring;
}

DirectIoEngine::~DirectIoEngine() {
    if (h_) ma_swap_destroy(h_);
}

std::vector<Extent> DirectIoEngine::allocate_extents(const std::string& key,
                                                     std::uint64_t logical_bytes) {
    std::vector<ma_swap_extent> ext(device_count_ ? device_count_ : 1);
    std::uint32_t n = 0;
    check(ma_swap_allocate(h_, key.c_str(), logical_bytes, ext.data(),
                           static_cast<uint32_t>(ext.size()), &n));
    return to_extents(ext, std::min<std::uint32_t>(n, static_cast<std::uint32_t>(ext.size())));
}

void DirectIoEngine::write_tensor(const std::string& key, std::span<const std::byte> src,
                                  std::uint64_t logical_bytes) {
    check(ma_swap_write(h_, key.c_str(), src.data(), src.size(), logical_bytes));
}

std::uint64_t DirectIoEngine::read_tensor(const std::string& key, std::span<std::byte> dst) {
    std::uint64_t logical = 0;
    check(ma_swap_read(h_, key.c_str(), dst.data(), dst.size(), &logical));
    return logical;
}

bool DirectIoEngine::contains(const std::string& key) const {
    int yes = 0;
    check(ma_swap_contains(h_, key.c_str(), &yes));
    return yes != 0;
}

TensorLocation DirectIoEngine::location(const std::string& key) const {
    TensorLocation loc;
    std::vector<ma_swap_extent> ext(device_count_ ? device_count_ : 1);
    std::uint32_t n = 0;
    check(ma_swap_location(h_, key.c_str(), &loc.logical_length, &loc.padded_length, ext.data(),
                           static_cast<uint32_t>(ext.size()), &n));
    loc.extents = to_extents(ext, std::min<std::uint32_t>(n, static_cast<std::uint32_t>(ext.size())));
    return loc;
}

std::vector<std::pair<std::string, TensorLocation>> DirectIoEngine::all_locations() const {
    std::uint64_t need = 0;
    check(ma_swap_keys(h_, nullptr, 0, &need));
    std::string buf(need, '\0');
    for (;;) {  // the table may grow between the two calls
        std::uint64_t got = 0;
        check(ma_swap_keys(h_, buf.data(), buf.size(), &got));
        if (got <= buf.size()) {
            buf.resize(got);
            break;
        }
        buf.assign(got, '\0');
    }
    std::vector<std::pair<std::string, TensorLocation>> out;
    for (size_t at = 0; at < buf.size();) {
        const size_t end = buf.find('\0', at);
        std::string key = buf.substr(at, end - at);
        out.emplace_back(key, location(key));
        at = end + 1;
    }
    return out;
}

EngineStats DirectIoEngine::stats() const {
    ma_swap_stats st{};
    check(ma_swap_get_stats(h_, &st));
    return EngineStats{st.bytes_written, st.bytes_read,    st.write_requests,
                       st.read_requests, st.submitted_ios, st.abandoned_bytes};
}

void DirectIoEngine::set_io_trace(IoTraceFn fn) {
    check(ma_swap_set_trace(h_, nullptr, nullptr));  // detach before replacing the target
    trace_ = std::move(fn);
    if (trace_) check(ma_swap_set_trace(h_, trace_trampoline, &trace_));
}

void DirectIoEngine::save_manifest() const { check(ma_swap_save_manifest(h_)); }

DeviceSet DirectIoEngine::create_virtual_devices(const std::string& dir, std::uint32_t count,
                                                 std::uint64_t bytes) {
    check(ma_swap_create_virtual_devices(dir.c_str(), count, bytes));
    DeviceSet set;
    for (std::uint32_t d = 0; d < count; ++d)
        set.devices.push_back(
            {dir + "/vdev" + std::to_string(d) + ".img", bytes, DeviceKind::file_backed_virtual});
    return set;
}

// ------------------------------------------------------------ FsBaselineStore
namespace {

// Owns one descriptor; every transfer is a full-length positional loop.
class File {
public:
    File(const std::string& path, int flags) : path_(path), fd_(::open(path.c_str(), flags, 0644)) {}
    ~File() {
        if (fd_ >= 0) ::close(fd_);
    }
    bool ok() const { return fd_ >= 0; }
    std::uint64_t size() const {
        struct stat st {};
        return ::fstat(fd_, &st) == 0 ? static_cast<std::uint64_t>(st.st_size) : 0;
    }
    // pwrite until `bytes` are out
    void put(const std::byte* src, std::uint64_t bytes) {
        std::uint64_t at = 0;
        while (at < bytes) {
            const ssize_t k = ::pwrite(fd_, src + at, bytes - at, static_cast<off_t>(at));
            if (k <= 0) raise(ErrorCode::io_error, "write to '" + path_ + "' stopped short");
            at += static_cast<std::uint64_t>(k);
        }
    }
    // pread in `chunk`-sized requests until `bytes` are in (or end of file)
    std::uint64_t get(std::byte* dst, std::uint64_t bytes, std::uint64_t chunk) {
        std::uint64_t at = 0;
        while (at < bytes) {
            const ssize_t k = ::pread(fd_, dst + at, chunk - at, static_cast<off_t>(at));
            if (k < 0) raise(ErrorCode::io_error, "read of '" + path_ + "': " + std::strerror(errno));
            if (k == 0) break;
            at += static_cast<std::uint64_t>(k);
        }
        return at;
    }
    void truncate(std::uint64_t bytes) {
        if (::ftruncate(fd_, static_cast<off_t>(bytes)) != 0)
            raise(ErrorCode::io_error, "cannot set the length of '" + path_ + "'");
    }

private:
    std::string path_;
    int fd_;
};

void require_granule_aligned(const void* p, const std::string& what) {
    if (reinterpret_cast<std::uintptr_t>(p) % kIoGranule)
        raise(ErrorCode::alignment, what + " is not 4096-aligned");
}

}  // namespace

FsBaselineStore::FsBaselineStore(std::string dir, bool cache_bypass)
    : dir_(std::move(dir)), cache_bypass_(cache_bypass) {
    std::filesystem::create_directories(dir_);
}

std::string FsBaselineStore::path_for(const std::string& key) const {
    std::string file = dir_ + "/";
    for (unsigned char c : key) file += std::isalnum(c) ? static_cast<char>(c) : '_';
    return file + ".tensor";
}

void FsBaselineStore::write(const std::string& key, std::span<const std::byte> src,
                            std::uint64_t logical_bytes) {
    if (logical_bytes == 0)
        raise(ErrorCode::invalid_argument, "'" + key + "': a tensor file holds at least one byte");
    require_granule_aligned(src.data(), "source buffer of '" + key + "'");
    const std::uint64_t padded = align_up(logical_bytes, kIoGranule);
    if (src.size() < padded)
        raise(ErrorCode::size_violation, "source buffer of '" + key + "' is shorter than " +
                                             std::to_string(padded) + " bytes");
    File f(path_for(key), O_CREAT | O_WRONLY | O_TRUNC | O_CLOEXEC | (cache_bypass_ ? O_DIRECT : 0));
    if (!f.ok()) raise(ErrorCode::io_error, "open '" + path_for(key) + "': " + std::strerror(errno));
    f.put(src.data(), padded);  // O_DIRECT moves whole granules ...
    f.truncate(logical_bytes);  // ... and the length records the logical size
}

std::uint64_t FsBaselineStore::read(const std::string& key, std::span<std::byte> dst) {
    require_granule_aligned(dst.data(), "destination buffer of '" + key + "'");
    File f(path_for(key), O_RDONLY | O_CLOEXEC | (cache_bypass_ ? O_DIRECT : 0));
    if (!f.ok()) raise(ErrorCode::not_found, "'" + key + "' has no tensor file");
    const std::uint64_t logical = f.size();
    const std::uint64_t padded = align_up(logical, kIoGranule);
    if (dst.size() < padded)
        raise(ErrorCode::size_violation, "destination buffer of '" + key + "' is shorter than " +
                                             std::to_string(padded) + " bytes");
    if (f.get(dst.data(), logical, padded) < logical)
        raise(ErrorCode::io_error, "'" + key + "' ended before its recorded length");
    return logical;
}

}  // namespace memascend
