// Host memory bandwidth of the f32 -> f64 level widening (j_inf mapping) with
// N threads into a pre-touched destination.  g++ -O3 -march=native -pthread
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>
int main() {
    const size_t n = size_t(36400000);
    std::vector<float> src(n, 3.5f);
    std::vector<double> dst(n, 0.0);
    for (int nt : {1, 4, 8, 16}) {
        double best = 1e9;
        for (int rep = 0; rep < 5; ++rep) {
            auto t0 = std::chrono::steady_clock::now();
            std::vector<std::thread> th;
            const size_t per = (n + nt - 1) / nt;
            for (int t = 0; t < nt; ++t)
                th.emplace_back([&, t] {
                    const size_t a = t * per, b = std::min(n, a + per);
                    for (size_t i = a; i < b; ++i) { const double x = src[i]; dst[i] = x < 1e6 ? x : 1e6; }
                });
            for (auto& x : th) x.join();
            const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
            if (ms < best) best = ms;
        }
        std::printf("threads %2d: %.2f ms per level (%.1f GB/s moved)\n", nt, best, n * 12.0 / best / 1e6);
    }
    return 0;
}
