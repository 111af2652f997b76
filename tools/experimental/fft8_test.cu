// Standalone bring-up and timing of the 8-point-per-thread row-pair DST-I
// (rsolve_fft8.cuh: N/8 threads per pair, radix 8 x 8 x 8 x 2 for N = 1024)
// against the shipped 16-point-per-thread RFft (rsolve_common.cuh): one CTA per
// row pair, rows global -> DST-I -> global, 5120 rows of 1023, 8 rotating sets.
// nvcc -O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -I include -I paper_2509_23180_b200/csrc \
//      -I tools/experimental tools/experimental/fft8_test.cu -o tools/experimental/fft8_test
#include "rsolve_common.cuh"
#include "rsolve_fft8.cuh"   // next to this file

#include <cmath>
#include <vector>

namespace fd {
void *dmalloc(size_t b) {
    void *p;
    cudaMalloc(&p, b);
    return p;
}
void dfree(void *p) { cudaFree(p); }
void set_error(const std::string &) {}
}  // namespace fd
using namespace fd;

// 16-point threads: 64 threads per pair
__global__ void __launch_bounds__(64, 8) k16(const double *in, double *out, const double *al, const double2 *tw16,
                                             double h2, int n) {
    using C = RS<10>;
    using F = RFft<10>;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    double2 *buf = reinterpret_cast<double2 *>(smem_raw);
    double *scr = reinterpret_cast<double *>(smem_raw + C::REG);
    const int t = threadIdx.x, lane = t & 31;
    const double *A = in + size_t(2 * blockIdx.x) * n;
    double2 v[16];
    F::load(v, A, A + n, al, h2, t);
    F::first(buf, v, t, 0);
    F::mid(buf, tw16, t, 0);
    F::last(buf, tw16 + 16, t, 0);
    double *XA = reinterpret_cast<double *>(buf);
    F::post(buf, scr, t, 0, lane, XA, XA + C::XR);
    rsync<64>(0);
    for (int h = 0; h < 2; ++h) {
        double *oh = out + size_t(2 * blockIdx.x + h) * n;
        for (int q = t; q < n; q += 64) oh[q] = XA[h * C::XR + xi(q)];
    }
}

// 8-point threads: 128 threads per pair
template <int MINB>
__global__ void __launch_bounds__(128, MINB) k8(const double *in, double *out, const double *al, const double2 *tw8,
                                                double h2, int n) {
    using F = RFft8<10>;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    double2 *buf = reinterpret_cast<double2 *>(smem_raw);
    double *scr = reinterpret_cast<double *>(smem_raw + F::REG);
    const int t = threadIdx.x, lane = t & 31;
    const double *A = in + size_t(2 * blockIdx.x) * n;
    double *XA = reinterpret_cast<double *>(buf);
    F::run(buf, A, A + n, al, h2, tw8, scr, t, 0, lane, XA, XA + F::XR);
    rsync<128>(0);
    for (int h = 0; h < 2; ++h) {
        double *oh = out + size_t(2 * blockIdx.x + h) * n;
        for (int q = t; q < n; q += 128) oh[q] = XA[h * F::XR + xi(q)];
    }
}

// same access pattern without the transform: the memory / launch floor of the one-CTA-per-pair structure
__global__ void __launch_bounds__(128, 8) kcopy(const double *in, double *out, int n) {
    const int t = threadIdx.x;
    const double *A = in + size_t(2 * blockIdx.x) * n;
    double *O = out + size_t(2 * blockIdx.x) * n;
    for (int q = t; q < 2 * n; q += 128) O[q] = A[q] * 1.000001;
}
// compute only: the 8-point transform on synthetic data, nothing read or written
template <int MINB>
__global__ void __launch_bounds__(128, MINB) k8c(double *out, const double *al, const double2 *tw8, double h2, int n) {
    using F = RFft8<10>;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    double2 *buf = reinterpret_cast<double2 *>(smem_raw);
    double *scr = reinterpret_cast<double *>(smem_raw + F::REG);
    const int t = threadIdx.x, lane = t & 31;
    double2 v[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) v[r] = make_double2(1e-3 * (t + r), 1e-3 * (blockIdx.x + r));
    F::passes(buf, v, tw8, t, 0);
    double *XA = reinterpret_cast<double *>(buf);
    F::post(buf, scr, t, 0, lane, XA, XA + F::XR);
    rsync<128>(0);
    if (XA[t] == 1.2345) out[0] = XA[t];
}

int main() {
    const int N = 1024, n = N - 1, rows = 5120, pairs = rows / 2, NB = 8;
    std::vector<double> h(size_t(rows) * n);
    unsigned s = 1;
    for (auto &x : h) {
        s = s * 1664525u + 1013904223u;
        x = (s >> 8) * (1.0 / 16777216.0) - 0.5;
    }
    double *d_in, *d_o16, *d_o8;
    cudaMalloc(&d_in, h.size() * 8 * NB);
    cudaMalloc(&d_o16, h.size() * 8 * NB);
    cudaMalloc(&d_o8, h.size() * 8 * NB);
    for (int b = 0; b < NB; ++b) cudaMemcpy(d_in + b * h.size(), h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    const long double PI = 3.141592653589793238462643383279502884L;
    const double scale = std::sqrt(2.0 / N), h2 = 0.5 * scale;
    std::vector<double> al(N);
    for (int j = 0; j < N; ++j) al[j] = (double)(0.5L * scale * sinl(PI * j / N) + 0.25L * scale);
    auto W = [&](long double num, long double den) {
        const long double a = 2.0L * PI * num / den;
        return make_double2((double)cosl(a), (double)(-sinl(a)));
    };
    std::vector<double2> t16(16 + 256), t8(RFft8<10>::NTW);
    for (int q = 0; q < 16; ++q) t16[q] = W(q, 256);
    for (int q = 0; q < 256; ++q) t16[16 + q] = W(q, N);
    RFft8<10>::host_twiddles(t8.data());
    double *d_al;
    double2 *d_t16, *d_t8;
    cudaMalloc(&d_al, N * 8);
    cudaMalloc(&d_t16, t16.size() * 16);
    cudaMalloc(&d_t8, t8.size() * 16);
    cudaMemcpy(d_al, al.data(), N * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(d_t16, t16.data(), t16.size() * 16, cudaMemcpyHostToDevice);
    cudaMemcpy(d_t8, t8.data(), t8.size() * 16, cudaMemcpyHostToDevice);
    const int sm16 = int(RS<10>::REG) + 128, sm8 = int(RFft8<10>::REG) + 128;
    cudaFuncSetAttribute(k16, cudaFuncAttributeMaxDynamicSharedMemorySize, sm16);
    cudaFuncSetAttribute(k8<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm8);
    cudaFuncSetAttribute(k8<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm8);
    cudaFuncSetAttribute(k8<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm8);
    k16<<<pairs, 64, sm16>>>(d_in, d_o16, d_al, d_t16, h2, n);
    k8<4><<<pairs, 128, sm8>>>(d_in, d_o8, d_al, d_t8, h2, n);
    cudaDeviceSynchronize();
    printf("launch: %s\n", cudaGetErrorString(cudaGetLastError()));
    std::vector<double> a(h.size()), b(h.size());
    cudaMemcpy(a.data(), d_o16, h.size() * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(b.data(), d_o8, h.size() * 8, cudaMemcpyDeviceToHost);
    double err = 0, nrm = 0;
    for (size_t i = 0; i < a.size(); ++i) {
        err = std::max(err, std::fabs(a[i] - b[i]));
        nrm = std::max(nrm, std::fabs(a[i]));
    }
    printf("8-point vs 16-point threads: max abs diff %.3e (max |X| %.3e)\n", err, nrm);
    // involution check of the 16-point reference: DST(DST(x)) = x
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto time = [&](auto launch, const char *name) {
        for (int i = 0; i < 5; ++i) launch(i % NB);
        cudaEventRecord(e0);
        const int R = 200;
        for (int i = 0; i < R; ++i) launch(i % NB);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("%-40s %.1f us per %d rows  (%s)\n", name, ms / R * 1e3, rows, cudaGetErrorString(cudaGetLastError()));
    };
    time([&](int b) { k16<<<pairs, 64, sm16>>>(d_in + b * h.size(), d_o16 + b * h.size(), d_al, d_t16, h2, n); },
         "16 points/thread, 64 thr/pair, 8 CTA/SM");
    time([&](int b) { k8<4><<<pairs, 128, sm8>>>(d_in + b * h.size(), d_o8 + b * h.size(), d_al, d_t8, h2, n); },
         "8 points/thread, 128 thr/pair, 4 CTA/SM");
    time([&](int b) { k8<6><<<pairs, 128, sm8>>>(d_in + b * h.size(), d_o8 + b * h.size(), d_al, d_t8, h2, n); },
         "8 points/thread, 128 thr/pair, 6 CTA/SM");
    time([&](int b) { k8<8><<<pairs, 128, sm8>>>(d_in + b * h.size(), d_o8 + b * h.size(), d_al, d_t8, h2, n); },
         "8 points/thread, 128 thr/pair, 8 CTA/SM");
    time([&](int b) { kcopy<<<pairs, 128>>>(d_in + b * h.size(), d_o8 + b * h.size(), n); }, "copy only, 128 thr/pair");
    cudaFuncSetAttribute(k8c<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm8);
    cudaFuncSetAttribute(k8c<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm8);
    time([&](int b) { k8c<8><<<pairs, 128, sm8>>>(d_o8, d_al, d_t8, h2, n); }, "8 points/thread, compute only, 8 CTA/SM");
    time([&](int b) { k8c<4><<<pairs, 128, sm8>>>(d_o8, d_al, d_t8, h2, n); }, "8 points/thread, compute only, 4 CTA/SM");
    return 0;
}
