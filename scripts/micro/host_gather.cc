// Host-side random-row gather rate (the paper's host-memory batch assembly):
// T threads memcpy 1600-byte records picked at random from a 3.9 GB buffer into a batch
// buffer.  Prints GB/s of records moved per thread count.
//   g++ -O3 -pthread -o host_gather host_gather.cc
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <thread>
#include <vector>

int main() {
  const size_t rec = 1600, N = 2449029, B = 8192, batches = 64;
  std::vector<char> store(rec * N);
  for (size_t i = 0; i < store.size(); i += 4096) store[i] = static_cast<char>(i);
  std::vector<char> out(rec * B);
  std::vector<uint32_t> order(B * batches);
  std::mt19937 g(1);
  for (auto& o : order) o = g() % N;
  for (int T : {1, 4, 8, 16, 32}) {
    auto t0 = std::chrono::steady_clock::now();
    for (size_t b = 0; b < batches; ++b) {
      std::vector<std::thread> th;
      for (int t = 0; t < T; ++t)
        th.emplace_back([&, t] {
          for (size_t j = t; j < B; j += T) memcpy(&out[j * rec], &store[order[b * B + j] * rec], rec);
        });
      for (auto& x : th) x.join();
    }
    const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    printf("{\"threads\": %d, \"GBs\": %.2f, \"us_per_batch\": %.1f}\n", T, batches * B * rec / s / 1e9,
           s / batches * 1e6);
    fflush(stdout);
  }
  return 0;
}
