// host_rng.cpp — the reference's pinned Gaussian sampler, bit-identical.
//
// gaussian_matrix (reference kernels.cpp:348-379): std::mt19937_64(seed),
// u1 = ((x >> 11) + 1) * 2^-53, u2 = (x >> 11) * 2^-53, Box-Muller with the
// cosine returned first and the sine kept as the spare, column-major fill.
// The sample depends on glibc's log/sin/cos, so it stays on the host: the
// 64-bit engine runs sequentially (cheap), the transcendental transform of
// the (u1, u2) pairs is spread over host threads.
#include <cmath>
#include <cstdint>
#include <random>
#include <thread>
#include <vector>

namespace svdk {

void gaussian_fill(int64_t rows, int64_t cols, uint64_t seed, double* out) {
    const int64_t count = rows * cols;
    const int64_t pairs = (count + 1) / 2;
    std::vector<uint64_t> raw(2 * pairs);
    std::mt19937_64 engine(seed);
    for (auto& x : raw) x = engine();
    const double pi = 3.141592653589793;
    auto work = [&](int64_t p0, int64_t p1) {
        for (int64_t p = p0; p < p1; ++p) {
            const double u1 = static_cast<double>((raw[2 * p] >> 11) + 1) * 0x1.0p-53;
            const double u2 = static_cast<double>(raw[2 * p + 1] >> 11) * 0x1.0p-53;
            const double radius = std::sqrt(-2.0 * std::log(u1));
            const double angle = 2.0 * pi * u2;
            out[2 * p] = radius * std::cos(angle);
            if (2 * p + 1 < count) out[2 * p + 1] = radius * std::sin(angle);
        }
    };
    unsigned nt = std::thread::hardware_concurrency();
    if (nt == 0) nt = 1;
    if (pairs < (1 << 15) || nt == 1) {
        work(0, pairs);
        return;
    }
    nt = std::min<unsigned>(nt, 32);
    std::vector<std::thread> th;
    const int64_t chunk = (pairs + nt - 1) / nt;
    for (unsigned t = 0; t < nt; ++t) {
        const int64_t a = t * chunk, b = std::min<int64_t>(pairs, a + chunk);
        if (a < b) th.emplace_back(work, a, b);
    }
    for (auto& x : th) x.join();
}

}  // namespace svdk
