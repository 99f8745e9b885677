// Host side of an fp32 solve's table download, two schemes side by side:
//   level: each 145 MB f32 level DMA'd into a 4-slot pinned ring, then widened
//          to f64 by 16 threads (the library's widen_levels today);
//   chunk: W workers, each DMA'ing its own small chunks (double-buffered
//          pinned slots on its own stream) and widening each chunk right after
//          it lands, while it is still in the last-level cache.
// Plus the int32 policies DMA'd straight into their destination.
// nvcc -O3 -std=c++17 -Xcompiler -mavx2 -o tools/widen_pipe tools/widen_pipe.cu
#include <cuda_runtime.h>
#include <immintrin.h>
#include <chrono>
#include <cstdio>
#include <thread>
#include <vector>

static void widen(const float* src, double* dst, size_t n, double cap) {
    size_t i = 0;
    const __m256d c = _mm256_set1_pd(cap);
    for (; i + 8 <= n; i += 8) {
        const __m256 v = _mm256_loadu_ps(src + i);
        _mm256_stream_pd(dst + i, _mm256_min_pd(_mm256_cvtps_pd(_mm256_castps256_ps128(v)), c));
        _mm256_stream_pd(dst + i + 4, _mm256_min_pd(_mm256_cvtps_pd(_mm256_extractf128_ps(v, 1)), c));
    }
    for (; i < n; ++i) dst[i] = src[i] < cap ? src[i] : cap;
    _mm_sfence();
}

int main(int argc, char** argv) {
    const size_t ns = 36400000, L = 21, P = 20;
    float* dJ;
    int* dP;
    cudaMalloc(&dJ, L * ns * sizeof(float));
    cudaMalloc(&dP, P * ns * sizeof(int));
    cudaMemset(dJ, 0, L * ns * sizeof(float));
    cudaMemset(dP, 0, P * ns * sizeof(int));
    double* hJ;
    int* hP;
    cudaHostAlloc(reinterpret_cast<void**>(&hJ), L * ns * sizeof(double), cudaHostAllocDefault);
    cudaHostAlloc(reinterpret_cast<void**>(&hP), P * ns * sizeof(int), cudaHostAllocDefault);
    for (size_t i = 0; i < L * ns; i += 512) hJ[i] = 0;
    for (size_t i = 0; i < P * ns; i += 1024) hP[i] = 0;
    auto now = [] { return std::chrono::steady_clock::now(); };
    auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
    cudaStream_t sp;
    cudaStreamCreateWithFlags(&sp, cudaStreamNonBlocking);

    // ---- level scheme
    {
        float* stage[4];
        cudaEvent_t ev[4];
        for (int b = 0; b < 4; ++b) {
            cudaHostAlloc(reinterpret_cast<void**>(&stage[b]), ns * sizeof(float), cudaHostAllocDefault);
            cudaEventCreateWithFlags(&ev[b], cudaEventDisableTiming);
        }
        cudaStream_t s;
        cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
        for (int rep = 0; rep < 3; ++rep) {
            auto t0 = now();
            cudaMemcpyAsync(hP, dP, P * ns * sizeof(int), cudaMemcpyDeviceToHost, sp);
            int queued = 0;
            auto enq = [&](int upto) {
                for (; queued <= upto && queued < (int)L; ++queued) {
                    const int b = queued % 4;
                    cudaMemcpyAsync(stage[b], dJ + queued * ns, ns * sizeof(float), cudaMemcpyDeviceToHost, s);
                    cudaEventRecord(ev[b], s);
                }
            };
            for (int k = 0; k < (int)L; ++k) {
                enq(k + 3);
                cudaEventSynchronize(ev[k % 4]);
                std::vector<std::thread> th;
                const size_t per = (ns + 15) / 16;
                for (int t = 0; t < 16; ++t)
                    th.emplace_back([&, t] {
                        const size_t a = t * per, b = std::min(ns, a + per);
                        widen(stage[k % 4] + a, hJ + k * ns + a, b - a, 1e30);
                    });
                for (auto& x : th) x.join();
            }
            cudaStreamSynchronize(sp);
            printf("level: %.1f ms\n", ms(t0, now()));
        }
    }
    // ---- chunk scheme
    for (size_t chunk_mb : {1, 2, 4, 8}) {
        for (int W : {8, 12, 16}) {
            const size_t cn = chunk_mb * (1 << 20) / sizeof(float);
            const size_t total = L * ns, nchunks = (total + cn - 1) / cn;
            std::vector<float*> slot(2 * W);
            std::vector<cudaStream_t> st(W);
            std::vector<cudaEvent_t> ev(2 * W);
            for (int i = 0; i < 2 * W; ++i) {
                cudaHostAlloc(reinterpret_cast<void**>(&slot[i]), cn * sizeof(float), cudaHostAllocDefault);
                cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming);
            }
            for (auto& x : st) cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking);
            double best = 1e9;
            for (int rep = 0; rep < 2; ++rep) {
                auto t0 = now();
                cudaMemcpyAsync(hP, dP, P * ns * sizeof(int), cudaMemcpyDeviceToHost, sp);
                std::vector<std::thread> th;
                for (int w = 0; w < W; ++w)
                    th.emplace_back([&, w] {
                        int j = 0;
                        auto issue = [&](size_t c, int sl) {
                            const size_t a = c * cn, n = std::min(cn, total - a);
                            cudaMemcpyAsync(slot[2 * w + sl], dJ + a, n * sizeof(float), cudaMemcpyDeviceToHost,
                                            st[w]);
                            cudaEventRecord(ev[2 * w + sl], st[w]);
                        };
                        size_t c = w;
                        if (c < nchunks) issue(c, 0);
                        for (; c < nchunks; c += W, j ^= 1) {
                            if (c + W < nchunks) issue(c + W, j ^ 1);
                            cudaEventSynchronize(ev[2 * w + j]);
                            const size_t a = c * cn, n = std::min(cn, total - a);
                            widen(slot[2 * w + j], hJ + a, n, 1e30);
                        }
                    });
                for (auto& x : th) x.join();
                cudaStreamSynchronize(sp);
                best = std::min(best, ms(t0, now()));
            }
            printf("chunk %zu MB x %d workers: %.1f ms\n", chunk_mb, W, best);
            for (int i = 0; i < 2 * W; ++i) cudaFreeHost(slot[i]);
        }
    }
    return 0;
}
