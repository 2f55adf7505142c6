// Host-link probe for the plan's end-to-end schedule (C4 sizes): how fast
// device->host read-backs run alone and under a concurrent host->device
// stream, as copy-engine 1-D / 2-D copies and as SM stores into mapped host
// memory, and how fast the host itself fills pinned memory.
//   nvcc -O2 -gencode arch=compute_100a,code=sm_100a -o gpurun_out/pcie_probe tools/pcie_probe.cu -lpthread
#include <cuda_runtime.h>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
    std::printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); return 1; } } while (0)

// rect copy dev -> mapped host, 16 B per thread-iteration
__global__ void k_egress(const uint4* src, uint4* dst, int pitch16, int x0_16, int w16, int h) {
    const long long n = (long long)w16 * h;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const int y = (int)(i / w16), x = (int)(i % w16) + x0_16;
        dst[(size_t)y * pitch16 + x] = src[(size_t)y * pitch16 + x];
    }
}

// SM load standing in for the folds: waves of short CTAs that spin
__global__ void k_busy(long long cycles, int* sink) {
    long long t0 = clock64();
    while (clock64() - t0 < cycles) {}
    if (threadIdx.x == 0 && cycles < 0) *sink = 1;
}

int main() {
    const size_t W = 16384, H = 8192, pitch = W * 4, canvas = pitch * H;  // 537 MB
    const size_t view = 2560ull * 6144 * 4;                                // 63 MB
    const int nview = 8;
    uint8_t *dout, *hout, *dv, *hv;
    CK(cudaMalloc(&dout, canvas));
    CK(cudaMalloc(&dv, view * nview));
    CK(cudaHostAlloc(&hout, canvas, cudaHostAllocMapped));
    CK(cudaHostAlloc(&hv, view * nview, cudaHostAllocDefault));
    std::memset(hout, 1, canvas);
    std::memset(hv, 1, view * nview);
    CK(cudaMemset(dout, 2, canvas));
    uint8_t* hout_d = nullptr;
    CK(cudaHostGetDevicePointer((void**)&hout_d, hout, 0));
    cudaStream_t sa, sb;
    CK(cudaStreamCreateWithFlags(&sa, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&sb, cudaStreamNonBlocking));
    cudaEvent_t a0, a1, b0, b1;
    CK(cudaEventCreate(&a0)); CK(cudaEventCreate(&a1));
    CK(cudaEventCreate(&b0)); CK(cudaEventCreate(&b1));
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));

    auto h2d = [&](cudaStream_t st) {
        for (int k = 0; k < nview; ++k)
            cudaMemcpyAsync(dv + k * view, hv + k * view, view, cudaMemcpyHostToDevice, st);
    };
    // D2H variants, each moving the whole canvas
    auto d2h = [&](int mode, cudaStream_t st, int ctas) {
        if (mode == 0) {  // 1-D, 8 slabs of full rows
            for (int k = 0; k < 8; ++k)
                cudaMemcpyAsync(hout + k * canvas / 8, dout + k * canvas / 8, canvas / 8,
                                cudaMemcpyDeviceToHost, st);
        } else if (mode == 1 || mode == 2) {  // 2-D column strips (1536 or 512 px)
            const size_t sw = mode == 1 ? 2048 : 512;
            for (size_t x = 0; x < W; x += sw)
                cudaMemcpy2DAsync(hout + x * 4, pitch, dout + x * 4, pitch, sw * 4, H,
                                  cudaMemcpyDeviceToHost, st);
        } else {  // SM stores into mapped host memory, 2048-px strips
            for (size_t x = 0; x < W; x += 2048)
                k_egress<<<ctas, 256, 0, st>>>((const uint4*)dout, (uint4*)hout_d, (int)(pitch / 16),
                                               (int)(x * 4 / 16), 2048 * 4 / 16, (int)H);
        }
    };
    auto ms = [&](cudaEvent_t x, cudaEvent_t y) { float t; cudaEventElapsedTime(&t, x, y); return t; };
    const char* names[] = {"1d", "2d_2048px", "2d_512px", "sm_mapped"};
    // warm
    h2d(sa); d2h(0, sb, 0); CK(cudaDeviceSynchronize());
    {
        cudaEventRecord(a0, sa); h2d(sa); cudaEventRecord(a1, sa);
        CK(cudaDeviceSynchronize());
        std::printf("h2d alone: %.3f ms  %.1f GB/s\n", ms(a0, a1), view * nview / ms(a0, a1) / 1e6);
    }
    for (int mode = 0; mode < 4; ++mode)
        for (int ctas : {0, 8, 32, 148}) {
            if ((mode == 3) != (ctas != 0)) continue;
            cudaEventRecord(b0, sb); d2h(mode, sb, ctas); cudaEventRecord(b1, sb);
            CK(cudaDeviceSynchronize());
            const float tb = ms(b0, b1);
            cudaEventRecord(a0, sa); cudaEventRecord(b0, sb);
            h2d(sa); d2h(mode, sb, ctas);
            cudaEventRecord(a1, sa); cudaEventRecord(b1, sb);
            CK(cudaDeviceSynchronize());
            std::printf("d2h %-10s ctas %3d: alone %.3f ms %.1f GB/s | with h2d: d2h %.3f ms %.1f GB/s, "
                        "h2d %.3f ms %.1f GB/s\n", names[mode], ctas, tb, canvas / tb / 1e6,
                        ms(b0, b1), canvas / ms(b0, b1) / 1e6, ms(a0, a1), view * nview / ms(a0, a1) / 1e6);
        }
    // the same under SM load (short CTAs filling every SM, ~20 us each)
    {
        int* sink; CK(cudaMalloc(&sink, 4));
        cudaStream_t sc, sp;
        int lo, hi;
        CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        CK(cudaStreamCreateWithFlags(&sc, cudaStreamNonBlocking));
        CK(cudaStreamCreateWithPriority(&sp, cudaStreamNonBlocking, hi));
        for (int mode = 0; mode < 4; ++mode)
            for (int ctas : {0, 8, 32}) {
                if ((mode == 3) != (ctas != 0)) continue;
                for (int prio = 0; prio < (mode == 3 ? 2 : 1); ++prio) {
                    cudaStream_t st = prio ? sp : sb;
                    k_busy<<<sms * 8 * 60, 256, 0, sc>>>(38000, sink);  // ~20 us at 1.9 GHz
                    cudaEventRecord(b0, st); d2h(mode, st, ctas); cudaEventRecord(b1, st);
                    CK(cudaDeviceSynchronize());
                    std::printf("under SM load: d2h %-10s ctas %3d prio %d: %.3f ms %.1f GB/s\n",
                                names[mode], ctas, prio, ms(b0, b1), canvas / ms(b0, b1) / 1e6);
                }
            }
        cudaEventRecord(a0, sc);
        k_busy<<<sms * 8 * 60, 256, 0, sc>>>(38000, sink);
        cudaEventRecord(a1, sc);
        CK(cudaDeviceSynchronize());
        std::printf("busy kernel alone: %.3f ms\n", ms(a0, a1));
    }
    // host fills of pinned memory (the empty bands of C4: 2 x 1024 rows)
    const size_t band = 2 * 1024 * pitch;
    for (int nt : {1, 2, 4, 8}) {
        auto t0 = std::chrono::steady_clock::now();
        std::vector<std::thread> th;
        for (int i = 0; i < nt; ++i)
            th.emplace_back([&, i] { std::memset(hout + band / nt * i, 0, band / nt); });
        for (auto& t : th) t.join();
        double dt = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        std::printf("host memset %zu MB, %d threads: %.3f ms %.1f GB/s\n", band >> 20, nt, dt, band / dt / 1e6);
    }
    return 0;
}
