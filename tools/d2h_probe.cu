// Device -> pageable host copy strategies for mid-size outputs (the J / P
// stacks of one C2 solve are ~9 MB).  nvcc -O2 -o /tmp/d2h tools/d2h_probe.cu -lpthread
#include <cuda_runtime.h>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <sys/mman.h>
#include <thread>
#include <vector>

static double now_ms() {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

static char* fresh(size_t n) {   // like np.empty: an mmap'd block, pages not yet touched
    void* p = mmap(nullptr, n, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
    return static_cast<char*>(p);
}

int main(int argc, char** argv) {
    const size_t n = (argc > 1 ? std::atof(argv[1]) : 9.0) * (1 << 20);
    const int reps = 20;
    char* d;
    cudaMalloc(&d, n);
    cudaMemset(d, 1, n);
    char* pin;
    cudaHostAlloc(reinterpret_cast<void**>(&pin), n, cudaHostAllocDefault);
    cudaStream_t st;
    cudaStreamCreate(&st);
    cudaDeviceSynchronize();
    auto run = [&](const char* name, auto&& body) {
        double best = 1e9, sum = 0;
        char* warm = fresh(n);
        std::memset(warm, 0, n);
        for (int r = 0; r < reps + 2; ++r) {
            char* h = std::getenv("WARM") ? warm : fresh(n);
            const double t0 = now_ms();
            body(h);
            const double t = now_ms() - t0;
            if (h != warm) munmap(h, n);
            if (r >= 2) { sum += t; best = std::min(best, t); }
        }
        munmap(warm, n);
        std::printf("%-34s %8.3f ms mean  %8.3f ms best  (%.1f GB/s)\n", name, sum / reps, best,
                    n / (sum / reps) / 1e6);
    };
    run("pageable cudaMemcpyAsync", [&](char* h) {
        cudaMemcpyAsync(h, d, n, cudaMemcpyDeviceToHost, st);
        cudaStreamSynchronize(st);
    });
    run("pageable, prefaulted", [&](char* h) {
        std::memset(h, 0, n);
        cudaMemcpyAsync(h, d, n, cudaMemcpyDeviceToHost, st);
        cudaStreamSynchronize(st);
    });
    run("register + async + unregister", [&](char* h) {
        cudaHostRegister(h, n, cudaHostRegisterDefault);
        cudaMemcpyAsync(h, d, n, cudaMemcpyDeviceToHost, st);
        cudaStreamSynchronize(st);
        cudaHostUnregister(h);
    });
    run("pinned only (no host copy)", [&](char*) {
        cudaMemcpyAsync(pin, d, n, cudaMemcpyDeviceToHost, st);
        cudaStreamSynchronize(st);
    });
    for (int nth : {1, 4, 8, 16}) {
        char name[64];
        std::snprintf(name, sizeof name, "pinned + memcpy x%d threads", nth);
        run(name, [&](char* h) {
            cudaMemcpyAsync(pin, d, n, cudaMemcpyDeviceToHost, st);
            cudaStreamSynchronize(st);
            std::vector<std::thread> th;
            const size_t per = (n + nth - 1) / nth;
            for (int t = 0; t < nth; ++t)
                th.emplace_back([=] { std::memcpy(h + t * per, pin + t * per, std::min(per, n - t * per)); });
            for (auto& x : th) x.join();
        });
    }
    // 21 levels, each DMA'd into pinned staging then copied while later levels transfer
    run("pinned per-level pipelined x1", [&](char* h) {
        const int L = 21;
        const size_t per = n / L;
        std::vector<cudaEvent_t> ev(L);
        for (auto& e : ev) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
        for (int k = 0; k < L; ++k) {
            cudaMemcpyAsync(pin + k * per, d + k * per, per, cudaMemcpyDeviceToHost, st);
            cudaEventRecord(ev[k], st);
        }
        for (int k = 0; k < L; ++k) {
            cudaEventSynchronize(ev[k]);
            std::memcpy(h + k * per, pin + k * per, per);
        }
        for (auto& e : ev) cudaEventDestroy(e);
    });
    std::printf("memset-touch of a fresh block: ");
    run("  (memset only)", [&](char* h) { std::memset(h, 0, n); });
    return 0;
}
