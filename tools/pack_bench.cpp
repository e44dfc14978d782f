// Host packer throughput from DRAM (256 MiB of acgt with 1% N runs):
// 1 thread vs the pool, slot-scatter form vs the streaming tile form.
//   g++ -O3 -std=c++17 -Ipaper_1509_01506_b200/csrc -I/usr/local/cuda/include tools/pack_bench.cpp \
//       paper_1509_01506_b200/_lib/obj/host_pack.o -lpthread -o /tmp/pack_bench
#include "host_pack.h"

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

using namespace ks;

static double secs(std::chrono::steady_clock::time_point t) {
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t).count();
}

int main() {
    const int64_t n = 256ll << 20;
    std::vector<uint8_t> in(n);
    std::mt19937 r(1);
    const char* a = "acgt";
    for (auto& c : in) c = a[r() & 3];
    for (int64_t p = 0; p + 10000 < n; p += 1000000) std::fill(in.begin() + p, in.begin() + p + 10000, 'N');
    const int lb = 4;
    const int64_t tb = 32 << lb, nb = (n + 63) / 64, nt = (nb + tb - 1) / tb, slots = nt * tb;
    uint64_t* bases = static_cast<uint64_t*>(aligned_alloc(4096, slots * 16));
    uint64_t* nm = static_cast<uint64_t*>(aligned_alloc(4096, slots * 8));
    std::vector<int32_t> ids(nt);
    HostPool pool(host_pack_threads());
    for (int it = 0; it < 5; ++it) {
        auto t = std::chrono::steady_clock::now();
        pack_ascii_blocks(in.data(), n, 0, slots, lb, bases, nm);
        const double d1 = secs(t);
        t = std::chrono::steady_clock::now();
        pool.run((nt + 3) / 4, [&](int64_t k) {
            pack_ascii_blocks(in.data(), n, k * 4 * tb, std::min(slots, (k + 1) * 4 * tb), lb, bases, nm);
        });
        const double d2 = secs(t);
        std::atomic<int32_t> nc{0};
        t = std::chrono::steady_clock::now();
        pool.run((nt + 3) / 4, [&](int64_t k) {
            pack_ascii_tiles(in.data(), n, k * 4, std::min(nt, (k + 1) * 4), lb, bases, nm, ids.data(), &nc);
        });
        const double d3 = secs(t);
        printf("1 thread %.1f GB/s  pool(%d) blocks %.1f GB/s  tiles %.1f GB/s (%d of %ld tiles with OTHER)\n",
               n / d1 / 1e9, pool.threads(), n / d2 / 1e9, n / d3 / 1e9, nc.load(), long(nt));
    }
}
