// standalone timing of the widening pool kinds (host only)
#include "../../paper_1908_05944_b200/csrc/widen_pool.h"
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
using namespace axb;
static double now() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }
int main(int argc, char **argv) {
    const int workers = argc > 1 ? atoi(argv[1]) : 15;
    const size_t n = 1000000, E = 4607698, T = 3483769, Q = 510141;
    std::vector<uint32_t> offe(n + 1), offt(n + 1);
    for (size_t a = 0; a <= n; ++a) { offe[a] = (uint32_t)(a * E / n); offt[a] = (uint32_t)(a * T / n); }
    int32_t *be = (int32_t *)aligned_alloc(64, E * 4 + 64), *bt = (int32_t *)aligned_alloc(64, T * 8 + 64), *bq = (int32_t *)aligned_alloc(64, Q * 16 + 64);
    memset(be, 1, E * 4); memset(bt, 1, T * 8); memset(bq, 1, Q * 16);
    int64_t *oe = (int64_t *)aligned_alloc(64, E * 16 + 64), *ot = (int64_t *)aligned_alloc(64, T * 24 + 64), *oq = (int64_t *)aligned_alloc(64, Q * 32 + 64), *ov = (int64_t *)aligned_alloc(64, n * 8 + 64);
    memset(oe, 0, E * 16); memset(ot, 0, T * 24); memset(oq, 0, Q * 32); memset(ov, 0, n * 8);
    WidenPool pool(workers);
    const size_t piece = 1 << 16;
    for (int rep = 0; rep < 4; ++rep) {
        double t0 = now();
        pool.begin(4096);
        pool.publish(WK_WIDEN, bq, oq, Q * 4, piece, 1, 1, nullptr, 0, 0);
        pool.finish();
        double t1 = now();
        pool.begin(4096);
        pool.publish(WK_TRI_ROWS, bt, ot, T, piece / 2, 2, 3, offt.data(), n, 0);
        pool.finish();
        double t2 = now();
        pool.begin(4096);
        pool.publish(WK_EDGE_ROWS, be, oe, E, piece, 1, 2, offe.data(), n, 0);
        pool.finish();
        double t3 = now();
        pool.begin(4096);
        pool.publish(WK_IOTA, nullptr, ov, n, piece, 0, 1, nullptr, 0, 0);
        pool.finish();
        double t4 = now();
        pool.begin(4096);
        pool.publish(WK_WIDEN, bt, ot, T * 2, piece, 1, 1, nullptr, 0, 0);
        pool.finish();
        double t5 = now();
        printf("tets widen %.3f ms (%.0f GB/s out) | tri rows %.3f ms (%.0f GB/s) | edge rows %.3f ms (%.0f GB/s) | iota %.3f ms | plain widen of %zu MB out %.3f ms (%.0f GB/s)\n",
               (t1 - t0) * 1e3, Q * 32 / (t1 - t0) / 1e9, (t2 - t1) * 1e3, T * 24 / (t2 - t1) / 1e9, (t3 - t2) * 1e3, E * 16 / (t3 - t2) / 1e9,
               (t4 - t3) * 1e3, T * 16 >> 20, (t5 - t4) * 1e3, T * 16 / (t5 - t4) / 1e9);
    }
}
