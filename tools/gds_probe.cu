// Probe: does cuFile (GPUDirect Storage) work on this box, and in which mode?
// Writes a 256 MiB file with O_DIRECT, reads it into HBM with cuFileRead,
// checks the bytes, reports GB/s.  nvcc -o gds_probe tools/gds_probe.cu -lcufile
#include <cuda_runtime.h>
#include <cufile.h>
#include <fcntl.h>
#include <unistd.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

int main(int argc, char** argv) {
    const char* path = argc > 1 ? argv[1] : "/tmp/gds_probe.bin";
    setvbuf(stdout, nullptr, _IONBF, 0);
    const size_t n = (argc > 2 ? std::strtoull(argv[2], nullptr, 10) : 256ull) << 20;
    void* h = nullptr;
    posix_memalign(&h, 4096, n);
    for (size_t i = 0; i < n; ++i) static_cast<unsigned char*>(h)[i] = static_cast<unsigned char>(i * 7 + 3);
    int fd = open(path, O_CREAT | O_RDWR | O_DIRECT, 0644);
    if (fd < 0 || pwrite(fd, h, n, 0) != (ssize_t)n) { std::printf("write failed\n"); return 1; }
    std::printf("file written\n");
    CUfileError_t st = cuFileDriverOpen();
    std::printf("cuFileDriverOpen: err=%d cu=%d\n", st.err, st.cu_err);
    if (st.err != CU_FILE_SUCCESS) return 2;
    CUfileDescr_t d;
    std::memset(&d, 0, sizeof d);
    d.handle.fd = fd;
    d.type = CU_FILE_HANDLE_TYPE_OPAQUE_FD;
    CUfileHandle_t fh;
    st = cuFileHandleRegister(&fh, &d);
    std::printf("cuFileHandleRegister: err=%d\n", st.err);
    if (st.err != CU_FILE_SUCCESS) return 3;
    void* dbuf = nullptr;
    cudaMalloc(&dbuf, n);
    st = cuFileBufRegister(dbuf, n, 0);
    std::printf("cuFileBufRegister: err=%d\n", st.err);
    for (int it = 0; it < 3; ++it) {
        cudaMemset(dbuf, 0, n);
        cudaDeviceSynchronize();
        auto t0 = std::chrono::steady_clock::now();
        ssize_t r = cuFileRead(fh, dbuf, n, 0, 0);
        auto t1 = std::chrono::steady_clock::now();
        double s = std::chrono::duration<double>(t1 - t0).count();
        std::vector<unsigned char> back(n);
        cudaMemcpy(back.data(), dbuf, n, cudaMemcpyDeviceToHost);
        std::printf("cuFileRead: %zd bytes, %.2f GB/s, match=%d\n", r, n / s / 1e9,
                    std::memcmp(back.data(), h, n) == 0);
    }
    cuFileBufDeregister(dbuf);
    cuFileHandleDeregister(fh);
    cuFileDriverClose();
    close(fd);
    unlink(path);
    return 0;
}
