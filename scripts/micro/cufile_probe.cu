// Probe: does cuFile (GPUDirect Storage / compat mode) work on this box?  Writes a file,
// reads it into device memory with cuFileRead from the main thread and from a second thread.
//   nvcc -o cufile_probe cufile_probe.cu -lcufile
#include <cuda_runtime.h>
#include <cufile.h>
#include <fcntl.h>
#include <unistd.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

static double now() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int main(int argc, char** argv) {
  const char* path = argc > 1 ? argv[1] : "/tmp/cufile_probe.bin";
  const size_t n = 64 << 20;
  std::vector<char> buf(n);
  for (size_t i = 0; i < n; ++i) buf[i] = static_cast<char>(i * 7 + 3);
  int fdw = open(path, O_CREAT | O_TRUNC | O_WRONLY, 0644);
  if (write(fdw, buf.data(), n) != (ssize_t)n) return 2;
  fsync(fdw);
  close(fdw);
  printf("file written\n");
  fflush(stdout);
  double t = now();
  CUfileError_t e = cuFileDriverOpen();
  printf("cuFileDriverOpen: err %d (%.3f s)\n", e.err, now() - t);
  fflush(stdout);
  if (e.err != CU_FILE_SUCCESS) return 3;
  int fd = open(path, O_RDONLY | O_DIRECT);
  printf("open O_DIRECT fd %d\n", fd);
  CUfileDescr_t d{};
  d.type = CU_FILE_HANDLE_TYPE_OPAQUE_FD;
  d.handle.fd = fd;
  CUfileHandle_t h;
  t = now();
  e = cuFileHandleRegister(&h, &d);
  printf("cuFileHandleRegister: err %d (%.3f s)\n", e.err, now() - t);
  fflush(stdout);
  if (e.err != CU_FILE_SUCCESS) return 4;
  void* dev = nullptr;
  cudaMalloc(&dev, n);
  t = now();
  ssize_t got = cuFileRead(h, dev, n, 0, 0);
  double dt = now() - t;
  printf("cuFileRead main thread: %zd bytes, %.3f s, %.2f GB/s\n", got, dt, got / dt / 1e9);
  fflush(stdout);
  std::vector<char> back(n);
  cudaMemcpy(back.data(), dev, n, cudaMemcpyDeviceToHost);
  printf("content ok: %d\n", memcmp(back.data(), buf.data(), n) == 0);
  std::thread th([&] {
    cudaSetDevice(0);
    double t0 = now();
    ssize_t g = cuFileRead(h, dev, 1 << 20, 4096, 8192);
    printf("cuFileRead worker thread: %zd bytes, %.4f s\n", g, now() - t0);
    fflush(stdout);
  });
  th.join();
  cuFileHandleDeregister(h);
  close(fd);
  cuFileDriverClose();
  printf("done\n");
  return 0;
}
