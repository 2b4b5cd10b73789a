// k_plan.cu -- S4: device exclusive scans and the signature -> bin plan.
//
// The paper samples a fraction of the input, builds a signature histogram and merges
// the least frequent signatures until at most 512 bins remain (Sec. 2.4).
// On the B200 the histogram is exact (pass 1 counts every window and record) and bins
// are sized to on-chip capacity instead of a file count (reading R6): runs of
// consecutive small signatures are merged while their summed cost stays below half the
// single-CTA capacity; a signature above that threshold forms a bin of its own.  A bin
// never splits a signature, so every copy of a canonical k-mer lands in one bin
// (a k-mer and its reverse complement share the signature).
#include "kmc_device.cuh"
#include "kmc_internal.h"
#include "kmc_scan.cuh"

namespace kmc {

using namespace scan_detail;

namespace {

// Cost of a signature in key units: max(windows, records * recw).
struct CostIn {
    const unsigned long long* hw;
    const uint32_t* hr;
    uint32_t recw;
    uint64_t half;
    __device__ __forceinline__ uint64_t cost(uint64_t i) const {
        uint64_t w = hw[i], r = (uint64_t)hr[i] * recw;
        return w > r ? w : r;
    }
    __device__ __forceinline__ uint64_t operator()(uint64_t i) const {
        uint64_t c = cost(i);
        return c > half ? 0 : c;  // big signatures get their own bin
    }
};

// 1 where a new bin starts at signature i.
struct BoundaryIn {
    CostIn c;
    const uint64_t* P;  // exclusive scan of small costs
    __device__ __forceinline__ uint64_t operator()(uint64_t i) const {
        if (i == 0) return 1;
        const bool big = c.cost(i) > c.half, big_prev = c.cost(i - 1) > c.half;
        if (big || big_prev) return 1;
        return (P[i] / c.half) != (P[i - 1] / c.half) ? 1 : 0;
    }
};

__global__ void k_sig2bin(BoundaryIn bf, uint64_t ns, const uint64_t* B, uint32_t* sig2bin, uint64_t* bin_first,
                          const unsigned long long* hw, unsigned long long* gstats) {
    __shared__ uint32_t ws[9];
    uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t used = 0;
    if (i < ns) {
        const uint64_t bnd = bf(i);
        const uint64_t incl = B[i] + bnd;
        sig2bin[i] = (uint32_t)(incl - 1);
        if (bnd) bin_first[incl - 1] = i;
        if (i == ns - 1) bin_first[B[ns]] = ns;
        used = hw[i] != 0;
    }
    uint32_t t = block_sum<256, uint32_t>(used, ws);
    if (threadIdx.x == 0 && t) atomicAdd(&gstats[GS_SIGS_USED], (unsigned long long)t);
    unsigned long long mx = i < ns ? hw[i] : 0ull;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long y = __shfl_xor_sync(0xffffffffu, mx, o);
        mx = y > mx ? y : mx;
    }
    if ((threadIdx.x & 31) == 0 && mx) atomicMax(&gstats[GS_MAX_SIG], mx);
}

__global__ void k_bins(uint64_t ns, const uint64_t* B, const uint64_t* bin_first, const uint64_t* Wp,
                       const uint64_t* Rp, uint64_t* bin_w, uint64_t* bin_nrec, uint64_t* bin_rec_off) {
    const uint64_t n_bins = B[ns];
    for (uint64_t b = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; b < n_bins;
         b += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t fs = bin_first[b], fe = bin_first[b + 1];
        bin_w[b] = Wp[fe] - Wp[fs];
        bin_nrec[b] = Rp[fe] - Rp[fs];
        bin_rec_off[b] = Rp[fs];
    }
}

__device__ __forceinline__ uint64_t tile_src_start(const TileSrc& t, uint64_t b) {
    if (!t.base) return b == 0 ? 0 : t.total;
    const uint64_t i = b << t.sh;
    if (i >= t.nbase) return t.total;
    return (t.is64 ? reinterpret_cast<const uint64_t*>(t.base)[i] : reinterpret_cast<const uint32_t*>(t.base)[i]) - t.off;
}

__global__ void k_tile_count(TileSrc t, uint64_t nb, uint32_t TI, uint64_t* __restrict__ cnt) {
    const uint64_t b = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= nb) return;
    cnt[b] = (tile_src_start(t, b + 1) - tile_src_start(t, b) + TI - 1) / TI;
}

// thread per tile: its bucket by binary search on the tile prefix
__global__ void k_tile_fill(TileSrc t, uint64_t nb, uint32_t TI, const uint64_t* __restrict__ prefix,
                            RecTile2* __restrict__ tiles) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= prefix[nb]) return;
    uint64_t lo = 0, hi = nb;  // last b with prefix[b] <= i
    while (hi - lo > 1) {
        const uint64_t mid = (lo + hi) >> 1;
        if (prefix[mid] <= i) lo = mid;
        else hi = mid;
    }
    const uint64_t s0 = tile_src_start(t, lo), s1 = tile_src_start(t, lo + 1);
    const uint64_t beg = s0 + (i - prefix[lo]) * TI;
    tiles[i] = RecTile2{beg, (uint32_t)(s1 - beg < TI ? s1 - beg : TI), (uint32_t)lo};
}

}  // namespace

cudaError_t launch_make_tiles(const TileSrc& src, uint64_t nb, uint32_t TI, uint64_t max_tiles, uint64_t* prefix,
                              void* temp, RecTile2* tiles, cudaStream_t s) {
    cudaError_t e;
    if (nb == 0) return cudaMemsetAsync(prefix, 0, 8, s);
    k_tile_count<<<(unsigned)((nb + 255) / 256), 256, 0, s>>>(src, nb, TI, prefix);
    if ((e = cudaGetLastError())) return e;
    // in-place exclusive scan: the scan reads its input before writing each output block
    if ((e = scan_generic<uint64_t>(ArrayIn<uint64_t>{prefix}, nb, prefix, (uint64_t*)temp, s, nullptr))) return e;
    if (max_tiles == 0) return cudaSuccess;
    k_tile_fill<<<(unsigned)((max_tiles + 255) / 256), 256, 0, s>>>(src, nb, TI, prefix, tiles);
    return cudaGetLastError();
}

size_t scan_temp_bytes(uint64_t n) { return scan_temp_elems<uint64_t>(n) * sizeof(uint64_t); }

cudaError_t scan_u64(const uint64_t* in, uint64_t* out, uint64_t n, void* temp, cudaStream_t s) {
    return scan_generic<uint64_t>(ArrayIn<uint64_t>{in}, n, out, (uint64_t*)temp, s, nullptr);
}

cudaError_t scan_u32_to_u32(const uint32_t* in, uint32_t* out, uint64_t n, void* temp, cudaStream_t s) {
    return scan_generic<uint32_t>(ArrayIn<uint32_t>{in}, n, out, (uint32_t*)temp, s, nullptr);
}

size_t plan_temp_bytes(uint64_t ns) { return scan_temp_bytes(ns); }

cudaError_t launch_plan(const PlanArgs& a, cudaStream_t s, int* n_launches) {
    cudaError_t e;
    CostIn ci{a.hist_w, a.hist_r, a.recw, a.half_cap};
    uint64_t* tmp = (uint64_t*)a.temp;
    if ((e = scan_generic<uint64_t>(ci, a.ns, a.cost_scan, tmp, s, n_launches)) != cudaSuccess) return e;
    BoundaryIn bf{ci, a.cost_scan};
    if ((e = scan_generic<uint64_t>(bf, a.ns, a.bnd_scan, tmp, s, n_launches)) != cudaSuccess) return e;
    if ((e = scan_generic<uint64_t>(ArrayIn<unsigned long long>{a.hist_w}, a.ns, a.win_scan, tmp, s, n_launches)) !=
        cudaSuccess)
        return e;
    if ((e = scan_generic<uint64_t>(ArrayIn<uint32_t>{a.hist_r}, a.ns, a.rec_scan, tmp, s, n_launches)) != cudaSuccess)
        return e;
    k_sig2bin<<<(unsigned)((a.ns + 255) / 256), 256, 0, s>>>(bf, a.ns, a.bnd_scan, a.sig2bin, a.bin_first, a.hist_w,
                                                             a.gstats);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    k_bins<<<(unsigned)std::min<uint64_t>((a.ns + 255) / 256, 4096), 256, 0, s>>>(
        a.ns, a.bnd_scan, a.bin_first, a.win_scan, a.rec_scan, a.bin_w, a.bin_nrec, a.bin_rec_off);
    if (n_launches) *n_launches += 2;
    return cudaGetLastError();
}

namespace {
__global__ void k_scale_hist(unsigned long long* hw, uint32_t* hr, uint64_t ns, uint64_t num, uint64_t den,
                             uint32_t fw, uint32_t fr) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < ns; i += (uint64_t)gridDim.x * blockDim.x) {
        hw[i] = (hw[i] * num + den - 1) / den + fw;
        const uint64_t v = ((uint64_t)hr[i] * num + den - 1) / den + fr;
        hr[i] = (uint32_t)(v < 0xFFFFFFFFull ? v : 0xFFFFFFFFull);
    }
}
__global__ void k_bin_caps(const uint64_t* est, uint64_t n_bins, double F, double z, uint32_t margin, uint32_t* cap,
                           uint64_t* cap64) {
    for (uint64_t b = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; b < n_bins;
         b += (uint64_t)gridDim.x * blockDim.x) {
        const double e = (double)est[b];
        const double c = e + z * sqrt(F * e) + (double)margin;
        const uint32_t v = c >= 4.0e9 ? 0xFFFFFFFFu : (uint32_t)c;
        cap[b] = v;
        cap64[b] = v;
    }
}
__global__ void k_sig_dest(const uint32_t* sig2bin, const uint32_t* cap, const uint64_t* off, uint64_t ns,
                           uint4* out) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < ns; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t b = sig2bin[i];
        const uint64_t o = off[b];
        out[i] = make_uint4(b, cap[b], (uint32_t)o, (uint32_t)(o >> 32));
    }
}
__global__ void k_bins_exact(uint64_t ns, const uint64_t* B, const uint64_t* bin_first, const uint64_t* Wp,
                             const uint32_t* fill, uint64_t* bin_w, uint64_t* bin_nrec) {
    const uint64_t n_bins = B[ns];
    for (uint64_t b = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; b < n_bins;
         b += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t fs = bin_first[b], fe = bin_first[b + 1];
        bin_w[b] = Wp[fe] - Wp[fs];
        bin_nrec[b] = fill[b];
    }
}
__global__ void k_hist_stats(const unsigned long long* hw, uint64_t ns, unsigned long long* gstats) {
    __shared__ uint32_t ws[9];
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const unsigned long long v = i < ns ? hw[i] : 0ull;
    const uint32_t t = block_sum<256, uint32_t>(v != 0, ws);
    if (threadIdx.x == 0 && t) atomicAdd(&gstats[GS_SIGS_USED], (unsigned long long)t);
    unsigned long long mx = v;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long y = __shfl_xor_sync(0xffffffffu, mx, o);
        mx = y > mx ? y : mx;
    }
    if ((threadIdx.x & 31) == 0 && mx) atomicMax(&gstats[GS_MAX_SIG], mx);
}
}  // namespace

cudaError_t launch_scale_hist(unsigned long long* hist_w, uint32_t* hist_r, uint64_t ns, uint64_t num, uint64_t den,
                              uint32_t floor_w, uint32_t floor_r, cudaStream_t s) {
    k_scale_hist<<<(unsigned)std::min<uint64_t>((ns + 255) / 256, 4096), 256, 0, s>>>(hist_w, hist_r, ns, num, den,
                                                                                        floor_w, floor_r);
    return cudaGetLastError();
}

cudaError_t launch_sig_dest(const uint32_t* sig2bin, const uint32_t* bin_cap, const uint64_t* bin_rec_off, uint64_t ns,
                            uint4* sig_dest, cudaStream_t s) {
    k_sig_dest<<<(unsigned)std::min<uint64_t>((ns + 255) / 256, 4096), 256, 0, s>>>(sig2bin, bin_cap, bin_rec_off, ns,
                                                                                     sig_dest);
    return cudaGetLastError();
}

cudaError_t launch_bin_caps(const uint64_t* bin_nrec, uint64_t n_bins, double F, double z, uint32_t margin,
                            uint32_t* bin_cap, uint64_t* bin_cap_u64, uint64_t* out_scan, void* temp, cudaStream_t s) {
    if (n_bins == 0) return cudaMemsetAsync(out_scan, 0, 8, s);
    k_bin_caps<<<(unsigned)std::min<uint64_t>((n_bins + 255) / 256, 4096), 256, 0, s>>>(bin_nrec, n_bins, F, z, margin,
                                                                                          bin_cap, bin_cap_u64);
    cudaError_t e;
    if ((e = cudaGetLastError())) return e;
    return scan_generic<uint64_t>(ArrayIn<uint64_t>{bin_cap_u64}, n_bins, out_scan, (uint64_t*)temp, s, nullptr);
}

cudaError_t launch_exact_tables(const PlanArgs& a, uint64_t n_bins, const uint32_t* bin_fill, cudaStream_t s,
                                int* n_launches) {
    cudaError_t e;
    uint64_t* tmp = (uint64_t*)a.temp;
    if ((e = scan_generic<uint64_t>(ArrayIn<unsigned long long>{a.hist_w}, a.ns, a.win_scan, tmp, s, n_launches)) !=
        cudaSuccess)
        return e;
    k_bins_exact<<<(unsigned)std::min<uint64_t>((n_bins + 255) / 256 + 1, 4096), 256, 0, s>>>(
        a.ns, a.bnd_scan, a.bin_first, a.win_scan, bin_fill, a.bin_w, a.bin_nrec);
    if ((e = cudaGetLastError())) return e;
    k_hist_stats<<<(unsigned)((a.ns + 255) / 256), 256, 0, s>>>(a.hist_w, a.ns, a.gstats);
    if (n_launches) *n_launches += 2;
    return cudaGetLastError();
}

}  // namespace kmc
