// Host unit test of csrc/widen_pool.h: the int32 -> int64 row expansion the host path runs while
// result chunks cross PCIe (plain widening, (owner, b) edge rows, (owner, b, c) triangle rows, iota),
// through the thread pool, against straightforward loops.
#include "../../paper_1908_05944_b200/csrc/widen_pool.h"

#include <cstdio>
#include <cstdlib>
#include <vector>

int main() {
    using namespace axb;
    const size_t n = 20000;
    std::vector<uint32_t> off(n + 1);
    std::vector<int32_t> b, bc;
    uint32_t tot = 0;
    srand(7);
    for (size_t a = 0; a < n; ++a) {
        off[a] = tot;
        int d = rand() % 9;
        if (a % 17 == 0 || a == 0) d = 0;              // owners without rows, including the first
        tot += d;
    }
    off[n] = tot;
    for (uint32_t r = 0; r < tot; ++r) { b.push_back(rand()); bc.push_back(rand()); bc.push_back(rand()); }
    int64_t *e = (int64_t *)aligned_alloc(64, ((size_t)tot * 2 + 8) * 8);
    int64_t *t = (int64_t *)aligned_alloc(64, ((size_t)tot * 3 + 8) * 8);
    int64_t *w = (int64_t *)aligned_alloc(64, ((size_t)tot * 2 + 8) * 8);
    int64_t *io = (int64_t *)aligned_alloc(64, (n + 8) * 8);
    int bad = 0;
    const size_t m24 = 50003;                           // odd: the high-byte plane starts at an odd multiple of 2
    std::vector<int64_t> v24(m24);
    std::vector<unsigned char> p24(3 * m24 + 64);
    for (size_t i = 0; i < m24; ++i) {
        v24[i] = (int64_t)(((unsigned)rand() << 9 ^ (unsigned)rand()) & 0xffffffu);
        const uint16_t lo16 = (uint16_t)(v24[i] & 0xffff);
        memcpy(p24.data() + 2 * i, &lo16, 2);
        p24[2 * m24 + i] = (unsigned char)(v24[i] >> 16);
    }
    int64_t *u24 = (int64_t *)aligned_alloc(64, (m24 + 8) * 8);
    WidenPool pool(3);
    for (int round = 0; round < 3; ++round) {           // the pool is reused run after run
        const size_t piece = round == 0 ? 1000 : (round == 1 ? 4099 : 70000);
        pool.begin(4 * (tot / piece + 2) + n / piece + m24 / piece + 16);
        // chunks at odd row boundaries, like the D2H chunks
        const size_t cut = tot / 3 + round;
        pool.publish(WK_EDGE_ROWS, b.data(), e, cut, piece, 1, 2, off.data(), n, 0);
        pool.publish(WK_EDGE_ROWS, b.data() + cut, e + 2 * cut, tot - cut, piece, 1, 2, off.data(), n, cut);
        pool.publish(WK_TRI_ROWS, bc.data(), t, cut, piece, 2, 3, off.data(), n, 0);
        pool.publish(WK_TRI_ROWS, bc.data() + 2 * cut, t + 3 * cut, tot - cut, piece, 2, 3, off.data(), n, cut);
        pool.publish(WK_WIDEN, bc.data(), w, (size_t)tot * 2, piece, 1, 1, nullptr, 0, 0);
        pool.publish(WK_IOTA, nullptr, io, n, piece, 0, 1, nullptr, 0, 0);
        // a 24-bit chunk: m low halves, then m high bytes; the tasks of the chunk share its base pointer
        pool.publish(WK_UNPACK24, reinterpret_cast<const int32_t *>(p24.data()), u24, m24, piece, 0, 1, nullptr, m24, 0);
        pool.finish();
        for (size_t i = 0; i < m24; ++i) if (u24[i] != v24[i]) ++bad;
        for (size_t i = 0; i < m24; ++i) u24[i] = -1;
        size_t a = 0;
        for (size_t r = 0; r < tot; ++r) {
            while (r >= off[a + 1]) ++a;
            if (e[2 * r] != (int64_t)a || e[2 * r + 1] != b[r]) ++bad;
            if (t[3 * r] != (int64_t)a || t[3 * r + 1] != bc[2 * r] || t[3 * r + 2] != bc[2 * r + 1]) ++bad;
        }
        for (size_t i = 0; i < (size_t)tot * 2; ++i) if (w[i] != bc[i]) ++bad;
        for (size_t i = 0; i < n; ++i) if (io[i] != (int64_t)i) ++bad;
        for (size_t i = 0; i < (size_t)tot * 2; ++i) { e[i] = -1; w[i] = -1; }
        for (size_t i = 0; i < (size_t)tot * 3; ++i) t[i] = -1;
        for (size_t i = 0; i < n; ++i) io[i] = -1;
    }
    printf("rows=%u bad=%d\n", tot, bad);
    return bad ? 1 : 0;
}
