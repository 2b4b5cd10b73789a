// kmc_scan.cuh -- device exclusive scans (reduce / scan-of-sums / down-sweep), generic in
// the input functor, shared by the plan (S4) and the global order (S9).
#pragma once
#include "kmc_device.cuh"

namespace kmc {
namespace scan_detail {

constexpr int SCAN_NT = 512;
constexpr int SCAN_IPT = 8;
constexpr uint64_t SCAN_TILE = SCAN_NT * SCAN_IPT;  // 4096

template <class T> struct ArrayIn {
    const T* a;
    __device__ __forceinline__ uint64_t operator()(uint64_t i) const { return (uint64_t)a[i]; }
};

template <class F, class TO>
__global__ void __launch_bounds__(SCAN_NT) k_scan_reduce(F f, uint64_t n, TO* sums) {
    __shared__ TO ws[SCAN_NT / 32 + 1];
    const uint64_t base = blockIdx.x * SCAN_TILE + (uint64_t)threadIdx.x * SCAN_IPT;
    TO s = 0;
#pragma unroll
    for (int j = 0; j < SCAN_IPT; ++j)
        if (base + j < n) s += (TO)f(base + j);
    TO t = block_sum<SCAN_NT, TO>(s, ws);
    if (threadIdx.x == 0) sums[blockIdx.x] = t;
}

// out[i] = block_off[b] + exclusive prefix within block; out[n] written by the last element.
template <class F, class TO>
__global__ void __launch_bounds__(SCAN_NT) k_scan_down(F f, uint64_t n, const TO* block_off, TO* out) {
    __shared__ TO ws[SCAN_NT / 32 + 1];
    const uint64_t base = blockIdx.x * SCAN_TILE + (uint64_t)threadIdx.x * SCAN_IPT;
    TO v[SCAN_IPT];
    TO s = 0;
#pragma unroll
    for (int j = 0; j < SCAN_IPT; ++j) {
        v[j] = (base + j < n) ? (TO)f(base + j) : (TO)0;
        s += v[j];
    }
    TO ex = block_excl_sum<SCAN_NT, TO>(s, ws, (TO*)nullptr) + (block_off ? block_off[blockIdx.x] : (TO)0);
#pragma unroll
    for (int j = 0; j < SCAN_IPT; ++j) {
        if (base + j < n) out[base + j] = ex;
        if (base + j == n - 1) out[n] = ex + v[j];
        ex += v[j];
    }
}

template <class TO> size_t scan_temp_elems(uint64_t n) {
    size_t tot = 0;
    while (n > 1) {
        uint64_t nb = (n + SCAN_TILE - 1) / SCAN_TILE;
        tot += 2 * (nb + 1);
        n = nb;
    }
    return tot + 2;
}

// Generic recursive exclusive scan: out has n+1 entries.
template <class TO, class F>
cudaError_t scan_generic(F f, uint64_t n, TO* out, TO* temp, cudaStream_t s, int* launches) {
    if (n == 0) {
        cudaError_t e = cudaMemsetAsync(out, 0, sizeof(TO), s);
        return e;
    }
    const uint64_t nb = (n + SCAN_TILE - 1) / SCAN_TILE;
    if (nb == 1) {
        k_scan_down<F, TO><<<1, SCAN_NT, 0, s>>>(f, n, (const TO*)nullptr, out);
        if (launches) *launches += 1;
        return cudaGetLastError();
    }
    TO* sums = temp;
    TO* offs = temp + nb;  // nb + 1 entries
    TO* rest = temp + 2 * (nb + 1);
    k_scan_reduce<F, TO><<<(unsigned)nb, SCAN_NT, 0, s>>>(f, n, sums);
    if (launches) *launches += 1;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    e = scan_generic<TO>(ArrayIn<TO>{sums}, nb, offs, rest, s, launches);
    if (e != cudaSuccess) return e;
    k_scan_down<F, TO><<<(unsigned)nb, SCAN_NT, 0, s>>>(f, n, offs, out);
    if (launches) *launches += 1;
    return cudaGetLastError();
}

}  // namespace scan_detail
}  // namespace kmc
