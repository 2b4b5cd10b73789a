// kmc_api.cu -- C ABI (include/kmcgpu.h) and host orchestration of the KMC 2 hot path.
//
// Stream-ordered sequence per call:
//   [input H2D] -> tile/read index -> pass 1 (S1-S3 + histogram) -> plan (S4)
//   -> sync: bin table -> pass 2 (S1-S3 + scatter, S5) -> small bins (S6-S8)
//   -> large bins: expand (S6) + device radix sort (S7) + RLE (S8)
//   -> sync: survivor count -> [finish] global order (S9) -> output copy.
#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/kmcgpu.h"
#include "kmc_device.cuh"
#include "kmc_internal.h"

using namespace kmc;

namespace {

thread_local std::string g_err;
std::mutex g_alloc_mu;
kmc_alloc_fn g_alloc = nullptr;
kmc_free_fn g_free = nullptr;
void* g_ctx = nullptr;

void set_err(const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_err = buf;
}

struct Fail {
    kmc_status st;
};

#define CK(call)                                                                                       \
    do {                                                                                               \
        cudaError_t _e = (call);                                                                       \
        if (_e != cudaSuccess) {                                                                       \
            set_err("%s:%d: %s: %s", __FILE__, __LINE__, #call, cudaGetErrorString(_e));               \
            throw Fail{KMC_ERR_CUDA};                                                                  \
        }                                                                                              \
    } while (0)

// Default scratch allocator: a process-wide cache of cudaMalloc'd device blocks.  A call
// needs tens of GB of scratch in a few dozen blocks of nearly the same sizes every time;
// mapping that anew per call (cudaMalloc / cudaFree, or a stream-ordered pool that gives
// physical pages back and re-maps them) costs more than the count itself on the host-input
// path.  Freed blocks stay cached, tagged with the stream that freed them; an allocation
// on the same stream and device takes the smallest cached block that fits without wasting
// more than a quarter (stream order makes the reuse safe, as in a caching allocator).  On
// an out-of-memory cudaMalloc the cache is synchronised and returned to the driver, then
// the allocation is retried once.
struct CachedBlock {
    void* p;
    size_t size;
    int dev;
    cudaStream_t s;
};
std::mutex g_cache_mu;
std::multimap<size_t, CachedBlock> g_cache;

size_t cache_round(size_t bytes) {
    const size_t g = bytes >= ((size_t)1 << 20) ? ((size_t)2 << 20) : (size_t)512;
    return (bytes + g - 1) / g * g;
}
void cache_flush_locked() {
    if (g_cache.empty()) return;
    cudaDeviceSynchronize();
    for (auto& e : g_cache) cudaFree(e.second.p);
    g_cache.clear();
    cudaGetLastError();
}
// *actual receives the size of the block handed out (a cached block may be up to 1.25x the
// request); the caller gives that size back to cache_free so the block keeps its true label.
void* cache_alloc(size_t bytes, cudaStream_t s, size_t* actual) {
    int dev = 0;
    *actual = bytes;
    if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
    std::lock_guard<std::mutex> g(g_cache_mu);
    for (auto it = g_cache.lower_bound(bytes); it != g_cache.end() && it->first <= bytes + bytes / 4; ++it) {
        if (it->second.dev == dev && it->second.s == s) {
            void* p = it->second.p;
            *actual = it->second.size;
            g_cache.erase(it);
            return p;
        }
    }
    void* p = nullptr;
    if (cudaMalloc(&p, bytes) != cudaSuccess) {
        cudaGetLastError();
        cache_flush_locked();
        p = nullptr;
        if (cudaMalloc(&p, bytes) != cudaSuccess) {
            cudaGetLastError();
            return nullptr;
        }
    }
    return p;
}
// bytes of this device's blocks held by the cache (free for a call that reuses them)
size_t cache_bytes() {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 0;
    std::lock_guard<std::mutex> g(g_cache_mu);
    size_t b = 0;
    for (auto& e : g_cache)
        if (e.second.dev == dev) b += e.second.size;
    return b;
}
void cache_free(void* p, size_t bytes, cudaStream_t s) {
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> g(g_cache_mu);
    g_cache.insert({bytes, CachedBlock{p, bytes, dev, s}});
}

struct Arena {
    cudaStream_t s = 0;
    std::vector<std::pair<void*, size_t>> ptrs;
    kmc_alloc_fn af = nullptr;
    kmc_free_fn ff = nullptr;
    void* ctx = nullptr;
    void bind(cudaStream_t st) {
        s = st;
        std::lock_guard<std::mutex> g(g_alloc_mu);
        af = g_alloc;
        ff = g_free;
        ctx = g_ctx;
    }
    // nullptr instead of an error when the allocator is out of memory
    void* try_alloc(size_t bytes) {
        bytes = cache_round(bytes == 0 ? 16 : bytes);
        size_t got = bytes;
        void* p = af ? af(bytes, (void*)s, ctx) : cache_alloc(bytes, s, &got);
        if (!p) {
            cudaGetLastError();
            return nullptr;
        }
        ptrs.push_back({p, got});
        return p;
    }
    void* alloc(size_t bytes) {
        void* p = try_alloc(bytes);
        if (!p) {
            set_err("scratch allocation of %zu bytes failed", bytes);
            throw Fail{KMC_ERR_ALLOC};
        }
        return p;
    }
    template <class T> T* get(size_t n) { return reinterpret_cast<T*>(alloc(n * sizeof(T))); }
    void give_back(void* p, size_t bytes) {
        if (ff) ff(p, (void*)s, ctx);
        else cache_free(p, bytes, s);
    }
    void release(void* p) {
        if (!p) return;
        auto it = std::find_if(ptrs.begin(), ptrs.end(), [p](const std::pair<void*, size_t>& e) { return e.first == p; });
        if (it == ptrs.end()) return;
        const size_t b = it->second;
        ptrs.erase(it);
        give_back(p, b);
    }
    void release_all() {
        for (auto& e : ptrs) give_back(e.first, e.second);
        ptrs.clear();
    }
};

int n_sms() {
    int dev = 0, v = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
        return 148;
    return v;
}

bool is_device_ptr(const void* p) {
    if (!p) return false;
    cudaPointerAttributes at;
    cudaError_t e = cudaPointerGetAttributes(&at, p);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

bool is_pinned_host(const void* p) {
    if (!p) return false;
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeHost;
}

// KMC_HOST_TRACE=1: host timestamps of the call's phases on stderr (diagnostics)
void htrace(const char* what) {
    static const bool on = getenv("KMC_HOST_TRACE") != nullptr;
    if (!on) return;
    static thread_local std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
    const auto t = std::chrono::steady_clock::now();
    fprintf(stderr, "[kmc %8.3f ms] %s\n", std::chrono::duration<double, std::milli>(t - t0).count(), what);
}

// Host-resident inputs of concurrent calls cross the PCIe link one pass after another: a
// call's copy stream waits for the previous call's last input copy (an event per device).
// Sharing the link would not move the inputs faster; one after another, a call's device
// stages and output copy overlap the next call's input copy (the link is full duplex).
std::mutex g_h2d_mu;
cudaEvent_t g_h2d_ev[64] = {};
struct H2DChain {
    std::unique_lock<std::mutex> lk;
    int dev = 0;
    bool on = false;
    void begin(cudaStream_t cs) {
        lk = std::unique_lock<std::mutex>(g_h2d_mu);
        if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) {
            lk.unlock();
            return;
        }
        if (g_h2d_ev[dev]) CK(cudaStreamWaitEvent(cs, g_h2d_ev[dev], 0));
        on = true;
    }
    void end(cudaStream_t cs) {
        if (!on) return;
        on = false;
        if (!g_h2d_ev[dev]) CK(cudaEventCreateWithFlags(&g_h2d_ev[dev], cudaEventDisableTiming));
        CK(cudaEventRecord(g_h2d_ev[dev], cs));
        lk.unlock();
    }
};

std::mutex g_begin_mu;  // kmc_count_begin (S1-S8) of concurrent calls, one at a time
std::mutex g_pin_mu;
std::vector<unsigned long long*> g_pin_free;
unsigned long long* pin_acquire() {
    {
        std::lock_guard<std::mutex> g(g_pin_mu);
        if (!g_pin_free.empty()) {
            unsigned long long* p = g_pin_free.back();
            g_pin_free.pop_back();
            return p;
        }
    }
    unsigned long long* p = nullptr;
    if (cudaMallocHost(&p, 256 * sizeof(unsigned long long)) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    return p;
}
void pin_release(unsigned long long* p) {
    if (!p) return;
    std::lock_guard<std::mutex> g(g_pin_mu);
    g_pin_free.push_back(p);
}

struct StageEv {
    int stage;
    cudaEvent_t a, b;
};

}  // namespace

// State carried between the phases of a count (pass 1 -> plan -> bins/count), so that the
// sharded entry points (kmc_shard_*) can stop between them for the caller's exchanges.
// inputs of at least this many Mi bases take the sampled distribution by default
constexpr uint32_t SAMPLE_MIN_MBASES = 64;
// device slots for batches of host-resident reads: the copy stream runs up to this many
// batches ahead of pass 1 (2 GiB at the default 256 MiB batches), so the input copy keeps
// going while the device is busy with another call's counting stages
constexpr int IN_SLOTS = 8;

// Large bins of the sampled plan split into their digit regions batch by batch while pass 1
// writes their records (k_split1 on the records appended since the previous batch), so that
// with host-resident reads the split runs under the input copy (kmc_options.presplit).
struct PreSplit {
    bool active = false;
    std::vector<uint64_t> ids;  // bin ids
    std::vector<S1Bin> sb;      // their split tables (paired layout)
    std::vector<int32_t> index; // bin id -> index in ids (-1: not presplit)
    uint32_t* d_ids = nullptr;
    S1Bin* d_sbins = nullptr;
    uint32_t* done = nullptr;   // records already split, per presplit bin
    uint32_t* cur = nullptr;    // per (bin, digit) key counts
    uint32_t* fail = nullptr;   // per (bin, digit) first position beyond the pair's slots
    uint64_t* keys = nullptr;   // the digit regions
    uint64_t* ovf = nullptr;    // keys beyond their region
    uint64_t ovf_cap = 0;
    unsigned long long* ctr = nullptr;  // [3] overflow keys, [5] pieces of the last batch
    Piece* pieces = nullptr;
    uint64_t n_digits = 0;
    const uint32_t* bin_fill = nullptr;
    const uint32_t* bin_cap = nullptr;
    const uint64_t* bin_rec_off = nullptr;
    uint32_t rpp = 0;
};

// A per-bin host table (windows, records or first record of every bin) in pinned memory from
// a process-wide pool: the three tables reach the host by asynchronous copies and one
// synchronisation (pageable destinations made every copy a synchronous staged transfer).
std::mutex g_tab_mu;
std::vector<std::pair<uint64_t*, size_t>> g_tab_free;  // (block, capacity in entries)
struct HostTable {
    uint64_t* p = nullptr;
    size_t n = 0, cap = 0;
    HostTable() = default;
    HostTable(const HostTable&) = delete;
    HostTable& operator=(const HostTable&) = delete;
    ~HostTable() { release(); }
    void release() {
        if (!p) return;
        std::lock_guard<std::mutex> g(g_tab_mu);
        g_tab_free.emplace_back(p, cap);
        p = nullptr;
        n = cap = 0;
    }
    // n entries (contents undefined until written)
    void resize(size_t m) {
        if (m > cap) {
            release();
            {
                std::lock_guard<std::mutex> g(g_tab_mu);
                for (size_t i = 0; i < g_tab_free.size(); ++i)
                    if (g_tab_free[i].second >= m) {
                        p = g_tab_free[i].first;
                        cap = g_tab_free[i].second;
                        g_tab_free.erase(g_tab_free.begin() + (long)i);
                        break;
                    }
            }
            if (!p) {
                const size_t c = m + m / 4 + 1024;
                if (cudaMallocHost(&p, c * 8) != cudaSuccess) {
                    cudaGetLastError();
                    p = nullptr;
                    set_err("cudaMallocHost of a %zu-entry bin table failed", c);
                    throw Fail{KMC_ERR_ALLOC};
                }
                cap = c;
            }
        }
        n = m;
    }
    uint64_t& operator[](size_t i) { return p[i]; }
    const uint64_t& operator[](size_t i) const { return p[i]; }
    uint64_t* data() { return p; }
    const uint64_t* data() const { return p; }
    size_t size() const { return n; }
};

// An array of T in the same pinned pool (host tables copied to the device asynchronously:
// the caller keeps it unchanged until the copy has completed).
template <class T> struct PinnedArr {
    HostTable raw;
    size_t n = 0;
    void resize(size_t m) {
        raw.resize((m * sizeof(T) + 7) / 8 + 1);
        n = m;
    }
    T* data() { return reinterpret_cast<T*>(raw.data()); }
    T& operator[](size_t i) { return data()[i]; }
    size_t size() const { return n; }
};

struct PlanCtx {
    PlanArgs pa{};
    uint64_t ns = 0, n_bins = 0, n_windows = 0, n_records = 0;
    uint64_t tmp_cap = 0, tmp_n = 0;  // record stream slots (capacity, used)
    int cap = 0;                      // small-bin capacity in keys
    bool check_p1 = true;             // the plan must match the pass-1 counters (not when sharded)
    unsigned long long* hist_w = nullptr;
    uint32_t* hist_r = nullptr;
    unsigned long long* gstats = nullptr;
    uint32_t* tmp_recs = nullptr;
    uint32_t* tmp_sig = nullptr;
    HostTable bw, bn, bo;              // per bin: windows, records, first record (pinned)
    bool tables_pending = false;       // bw/bn/bo not yet copied to the host (fetch_tables)
    cudaEvent_t ev_plan = nullptr;     // recorded on the job stream right after the plan
    P1Args a{};
    std::function<int(int)> run_p1;  // pass-1 recompute (S5 fallback), unset when sharded
    // sharded: bin -> owning rank
    std::vector<uint32_t> owner;
    bool multipass = false;  // host reads beyond HBM: passes over ranges of bins (f2)
    uint32_t* bins_ready = nullptr;  // sampled distribution: pass 1 wrote the records into their bins
    PreSplit pre;
};

struct kmc_job {
    cudaStream_t s = 0;
    PlanCtx ctx;
    bool shard = false;
    int world = 1, rank = 0;
    uint64_t n_local_records = 0;
    int k = 0, p = 0, key_words = 1;
    uint32_t ci = 1, cx = 0;
    kmc_options opt{};
    Arena arena;
    void* surv_keys = nullptr;
    uint32_t* surv_counts = nullptr;
    uint64_t n_surv = 0;
    uint64_t surv_cap = 0;
    kmc_stats st{};
    int launches = 0;
    std::vector<StageEv> evs;
    int cur_stage = -1;
    cudaEvent_t cur_a = nullptr;
    unsigned long long* host_small = nullptr;  // pinned readback area
    cudaStream_t cs = nullptr;                 // copy stream for streamed input batches
    // sharded, fused exchange: this rank's receive buffers (plain cudaMalloc: IPC-mappable)
    uint32_t* sig2owner = nullptr;
    std::vector<uint64_t> send_counts;
    uint32_t* recv_recs = nullptr;
    uint32_t* recv_sigs = nullptr;
    uint64_t n_recv = 0;
    cudaEvent_t ev_copy[IN_SLOTS] = {}, ev_done[IN_SLOTS] = {};

    void make_copy_stream() {
        if (cs) return;
        CK(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
        for (int t = 0; t < IN_SLOTS; ++t) {
            CK(cudaEventCreateWithFlags(&ev_copy[t], cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&ev_done[t], cudaEventDisableTiming));
            CK(cudaEventRecord(ev_done[t], s));
        }
    }

    void stage_begin(int stage) {
        cur_stage = stage;
        if (!opt.profile) return;
        CK(cudaEventCreate(&cur_a));
        CK(cudaEventRecord(cur_a, s));
    }
    void stage_end(int launches_in_stage) {
        if (cur_stage >= 0) st.stage_launches[cur_stage] += launches_in_stage;
        if (opt.profile && cur_a) {
            cudaEvent_t b;
            CK(cudaEventCreate(&b));
            CK(cudaEventRecord(b, s));
            evs.push_back({cur_stage, cur_a, b});
        }
        cur_stage = -1;
        cur_a = nullptr;
    }
    void collect_profile() {
        for (auto& e : evs) {
            float ms = 0;
            if (cudaEventElapsedTime(&ms, e.a, e.b) == cudaSuccess) st.stage_ms[e.stage] += ms;
            cudaEventDestroy(e.a);
            cudaEventDestroy(e.b);
        }
        evs.clear();
    }
    ~kmc_job() {
        for (auto& e : evs) {
            cudaEventDestroy(e.a);
            cudaEventDestroy(e.b);
        }
        if (cur_a) cudaEventDestroy(cur_a);
        if (ctx.ev_plan) cudaEventDestroy(ctx.ev_plan);
        if (cs) {
            cudaStreamSynchronize(cs);
            for (int t = 0; t < IN_SLOTS; ++t) {
                cudaEventDestroy(ev_copy[t]);
                cudaEventDestroy(ev_done[t]);
            }
            cudaStreamDestroy(cs);
        }
        arena.release_all();
        pin_release(host_small);
        if (recv_recs) cudaFree(recv_recs);
        if (recv_sigs) cudaFree(recv_sigs);
    }
};

namespace {

kmc_status validate(int k, int p, uint32_t ci, uint32_t cx) {
    if (k < 1 || k > 64) {
        set_err("k=%d outside [1, 64]", k);
        return KMC_ERR_INVALID_ARG;
    }
    if (p < 1 || p > 15 || p > k) {  // 4^15 + 1 signature ids fit 32 bits
        set_err("p=%d outside [1, min(k, 15)] (k=%d)", p, k);
        return KMC_ERR_INVALID_ARG;
    }
    if (ci == 0) ci = 1;
    if (cx < ci) {
        set_err("cutoff_max=%u < cutoff_min=%u", cx, ci);
        return KMC_ERR_INVALID_ARG;
    }
    return KMC_OK;
}

// Reads offsets[0] and offsets[n_reads] (device or host).
void read_extent(kmc_job* j, const uint64_t* offsets, uint64_t n_reads, uint64_t* off0, uint64_t* offN) {
    if (is_device_ptr(offsets)) {
        CK(cudaMemcpyAsync(&j->host_small[0], offsets, 8, cudaMemcpyDeviceToHost, j->s));
        CK(cudaMemcpyAsync(&j->host_small[1], offsets + n_reads, 8, cudaMemcpyDeviceToHost, j->s));
        CK(cudaStreamSynchronize(j->s));
        *off0 = j->host_small[0];
        *offN = j->host_small[1];
    } else {
        *off0 = offsets[0];
        *offN = offsets[n_reads];
    }
}

void plan_phase(kmc_job* j, PlanCtx& c);
void fetch_tables(kmc_job* j, PlanCtx& c);
void count_phase(kmc_job* j, PlanCtx& c);
void count_bins(kmc_job* j, PlanCtx& c, uint32_t* bins, uint64_t b_lo, uint64_t b_hi);
void count_multipass(kmc_job* j, PlanCtx& c);
void release_plan_scratch(kmc_job* j, PlanCtx& c);
void presplit_setup(kmc_job* j, PlanCtx& c, const std::vector<uint64_t>& bw, const std::vector<uint64_t>& bn,
                    const uint32_t* bin_cap, const uint32_t* bin_fill, uint64_t total_cap);
int presplit_batch(kmc_job* j, PlanCtx& c, const uint32_t* bins);
void presplit_release(kmc_job* j, PreSplit& pre);

void run_begin(kmc_job* j, const uint8_t* reads, const uint64_t* offsets, uint64_t n_reads) {
    const int k = j->k, p = j->p, kw = j->key_words;
    const size_t ksz = kw == 1 ? 8 : 16;
    Arena& ar = j->arena;
    cudaStream_t s = j->s;
    htrace("run_begin");
    j->host_small = pin_acquire();
    if (!j->host_small) {
        set_err("pinned readback buffer allocation failed");
        throw Fail{KMC_ERR_ALLOC};
    }
    j->st.n_reads = n_reads;
    uint64_t off0 = 0, offN = 0;
    if (n_reads > 0) read_extent(j, offsets, n_reads, &off0, &offN);
    if (offN < off0) {
        set_err("read_offsets decreasing: offsets[0]=%llu > offsets[n]=%llu", (unsigned long long)off0,
                (unsigned long long)offN);
        throw Fail{KMC_ERR_INVALID_ARG};
    }
    htrace("extent read");
    const uint64_t n_bases = offN - off0;
    j->st.n_bases = n_bases;
    if (n_bases == 0 || (uint64_t)k > n_bases) {
        j->n_surv = 0;
        return;
    }
    if (n_bases >= (1ull << 36)) {
        set_err("n_bases=%llu exceeds the per-call limit 2^36", (unsigned long long)n_bases);
        throw Fail{KMC_ERR_INVALID_ARG};
    }
    // ---- inputs: device-resident reads are used in place; host-resident reads are streamed
    //      through pass 1 in read-aligned batches (f2: "pinned host memory only when the
    //      input exceeds HBM"), so the reads never need to fit in device memory.
    const bool host_reads = !is_device_ptr(reads);
    const uint8_t* d_reads = reads;
    const uint64_t* d_off = offsets;
    std::vector<uint64_t> h_off_copy;
    const uint64_t* h_off = nullptr;
    j->stage_begin(KMC_STAGE_INPUT);
    if (host_reads) {
        if (is_device_ptr(offsets)) {
            h_off_copy.resize(n_reads + 1);
            CK(cudaMemcpy(h_off_copy.data(), offsets, (n_reads + 1) * 8, cudaMemcpyDeviceToHost));
            h_off = h_off_copy.data();
        } else {
            h_off = offsets;
        }
    } else if (!is_device_ptr(offsets)) {
        uint64_t* o = ar.get<uint64_t>(n_reads + 1);
        CK(cudaMemcpyAsync(o, offsets, (n_reads + 1) * 8, cudaMemcpyHostToDevice, s));
        d_off = o;
    }
    j->stage_end(0);

    // ---- pass 1: S1-S3 + per-signature histogram
    const uint64_t ns = (1ull << (2 * p)) + 1;
    unsigned long long* hist_w = ar.get<unsigned long long>(ns);
    uint32_t* hist_r = ar.get<uint32_t>(ns);
    unsigned long long* gstats = ar.get<unsigned long long>(GS_N);
    const uint64_t n_tiles = host_reads ? 0 : p1_num_tiles(n_bases);
    uint64_t* tile_r_lo = host_reads ? nullptr : ar.get<uint64_t>(n_tiles);
    j->stage_begin(KMC_STAGE_SIGNATURE);
    CK(cudaMemsetAsync(hist_w, 0, ns * 8, s));
    CK(cudaMemsetAsync(hist_r, 0, ns * 4, s));
    CK(cudaMemsetAsync(gstats, 0, GS_N * 8, s));
    P1Args a{};
    a.reads = d_reads;
    a.offsets = d_off;
    a.n_reads = n_reads;
    a.off0 = off0;
    a.n_bases = n_bases;
    a.k = k;
    a.p = p;
    a.rules = j->opt.plain_minimizers ? 0 : 1;
    a.reads_aligned16 = ((uintptr_t)d_reads & 15) == 0;
    a.tile_r_lo = tile_r_lo;
    a.bin_lo = 0;
    a.bin_hi = 0xFFFFFFFFu;
    a.hist_w = hist_w;
    a.hist_r = hist_r;
    a.gstats = gstats;
    // temporary record stream: pass 1 appends its records so S5 is a copy, not a recompute
    // (estimate n_bases/8 records; on overflow S5 falls back to recomputing pass 1)
    const int RWt = record_words(k);
    uint32_t* tmp_recs = nullptr;
    uint32_t* tmp_sig = nullptr;
    uint64_t tmp_cap = 0;
    // Inputs beyond HBM (f2): host-resident reads whose single-pass working set (record stream
    // + bins, ~(2 RW*4 + 4) bytes per record, ~n_bases/8 records) does not fit the free device
    // memory -- or a forced pass size -- are counted in passes over ranges of bins: pass 1
    // builds only the histogram, then every pass streams the reads again and keeps the
    // records of its bins.
    j->ctx.multipass = false;
    if (host_reads && !j->shard) {
        size_t fr = 0, tot = 0;
        CK(cudaMemGetInfo(&fr, &tot));
        const double est = (double)(n_bases / 8 + 1) * (2.0 * RWt * 4 + 4) * 1.2;
        j->ctx.multipass = j->opt.pass_mb > 0 || est > 0.7 * (double)(fr + cache_bytes());
    }
    // The paper's sampled distribution: the bin plan comes from a sample of the
    // reads (every 32nd pass-1 segment; with host-resident reads segments of the first batch,
    // ~1/16 of all), bins get the sampled record count + 6 standard deviations of the estimate + a
    // margin, and pass 1 then writes every record straight into its bin while it counts the
    // exact histograms -- no record stream, no S5 re-sort.  A record beyond its bin's capacity
    // (a sample far off) makes the call plan again from the exact histograms and repeat the
    // scatter.  Small inputs keep the exact histogram + record stream + S5.
    const bool sampled = !j->shard && !j->ctx.multipass &&
                         (j->opt.distribute_path == 2 ||
                          (j->opt.distribute_path == 0 && n_bases >= ((uint64_t)SAMPLE_MIN_MBASES << 20)));
    if (j->opt.distribute_path == 0 && !sampled && !j->ctx.multipass) {
        // slots: records (~n_bases/8 at 100 bp reads) + every pass-1 warp's partly used block
        tmp_cap = std::max<uint64_t>(n_bases / 8, 4096) + (uint64_t)n_sms() * 64 * 2048;
        tmp_recs = reinterpret_cast<uint32_t*>(ar.alloc(tmp_cap * RWt * 4));
        tmp_sig = ar.get<uint32_t>(tmp_cap);
    }
    a.tmp_recs = tmp_recs;
    a.tmp_sig = tmp_sig;
    a.tmp_cap = tmp_cap;
    // batches of host-resident reads: [r0, r1) with at most batch_bytes bases (one read may
    // exceed it alone); up to IN_SLOTS device slots, H2D on a copy stream ahead of pass 1
    std::vector<std::pair<uint64_t, uint64_t>> batches;
    uint8_t* bbuf[IN_SLOTS] = {};
    uint64_t* bofs[IN_SLOTS] = {};
    uint64_t* btile[IN_SLOTS] = {};
    int NS = 1;
    if (host_reads) {
        const uint64_t batch_bytes = (uint64_t)(j->opt.input_batch_mb ? j->opt.input_batch_mb : 256) << 20;
        uint64_t max_b = 0, max_r = 0;
        for (uint64_t r0 = 0; r0 < n_reads;) {
            // the last two batches' worth of bases in halving batches (down to 1/8 of one):
            // what pass 1 still has to do after the input copy ends is the last batch's work
            const uint64_t left = h_off[n_reads] - h_off[r0];
            uint64_t bb = batch_bytes;
            if (left <= 2 * batch_bytes) bb = std::max(left / 2, batch_bytes / 8);
            const uint64_t lim = h_off[r0] + bb;
            uint64_t r1 = (uint64_t)(std::upper_bound(h_off + r0 + 1, h_off + n_reads + 1, lim) - h_off) - 1;
            if (r1 <= r0) r1 = r0 + 1;
            batches.push_back({r0, r1});
            max_b = std::max(max_b, h_off[r1] - h_off[r0]);
            max_r = std::max(max_r, r1 - r0);
            r0 = r1;
        }
        // slots: IN_SLOTS, fewer for few batches, and at least 2 when memory is short
        NS = (int)std::min<size_t>(IN_SLOTS, std::max<size_t>(batches.size(), 1));
        for (int t = 0; t < NS; ++t) {
            bbuf[t] = reinterpret_cast<uint8_t*>(t < 2 ? ar.alloc(max_b + 16) : ar.try_alloc(max_b + 16));
            if (!bbuf[t]) {
                NS = t;
                break;
            }
            bofs[t] = ar.get<uint64_t>(max_r + 1);
            btile[t] = ar.get<uint64_t>(p1_num_tiles(max_b) + 1);
        }
        j->st.n_input_batches = batches.size();
    }
    // host reads: slot_batch[t] = the batch whose reads are in device slot t (-1: none); a pass
    // with keep_slots set reuses them (the sampled distribution's scatter pass reuses the
    // first batch its sample pass copied), any other pass copies every batch
    bool tiles_ready = false, keep_slots = false;
    int64_t slot_batch[IN_SLOTS];
    for (int t = 0; t < IN_SLOTS; ++t) slot_batch[t] = -1;
    auto copy_batch = [&](size_t b) {
        const int t = (int)(b % NS);
        if (slot_batch[t] == (int64_t)b) return;
        const uint64_t r0 = batches[b].first, r1 = batches[b].second;
        CK(cudaStreamWaitEvent(j->cs, j->ev_done[t], 0));
        CK(cudaMemcpyAsync(bbuf[t], reads + (h_off[r0] - off0), h_off[r1] - h_off[r0], cudaMemcpyHostToDevice, j->cs));
        CK(cudaMemcpyAsync(bofs[t], h_off + r0, (r1 - r0 + 1) * 8, cudaMemcpyHostToDevice, j->cs));
        CK(cudaEventRecord(j->ev_copy[t], j->cs));
        slot_batch[t] = (int64_t)b;
    };
    // after every pass-1 launch of a scatter pass (the presplit of the new records)
    std::function<int()> p1_hook;
    // max_batches: stop after that many batches (the sample pass: the first one)
    auto run_p1 = [&](int mode, size_t max_batches = ~(size_t)0) -> int {
        if (!host_reads) {
            int nl = 1;
            if (!tiles_ready) {  // the segment -> first read table of device-resident reads is kept
                CK(launch_tile_reads(d_off, n_reads, off0, n_tiles, tile_r_lo, s));
                tiles_ready = true;
                ++nl;
            }
            CK(launch_p1(mode, a, n_tiles, s));
            if (mode == P1_MODE_SCATTER && p1_hook) nl += p1_hook();
            return nl;
        }
        if (!keep_slots)
            for (int t = 0; t < IN_SLOTS; ++t) slot_batch[t] = -1;
        keep_slots = false;
        const size_t nbt = batches.size(), lim = std::min(nbt, max_batches);
        for (size_t q = 0; q < (size_t)NS && q < lim; ++q) copy_batch(q);
        int nl = 0;
        for (size_t b = 0; b < lim; ++b) {
            const int t = (int)(b % NS);
            const uint64_t r0 = batches[b].first, r1 = batches[b].second;
            const uint64_t nb = h_off[r1] - h_off[r0];
            copy_batch(b);
            CK(cudaStreamWaitEvent(s, j->ev_copy[t], 0));
            P1Args ab = a;
            ab.reads = bbuf[t];
            ab.offsets = bofs[t];
            ab.n_reads = r1 - r0;
            ab.off0 = h_off[r0];
            ab.n_bases = nb;
            ab.reads_aligned16 = ((uintptr_t)bbuf[t] & 15) == 0;
            ab.tile_r_lo = btile[t];
            const uint64_t nt = p1_num_tiles(nb);
            CK(launch_tile_reads(bofs[t], r1 - r0, h_off[r0], nt, btile[t], s));
            CK(launch_p1(mode, ab, nt, s));
            CK(cudaEventRecord(j->ev_done[t], s));
            nl += 2;
            if (mode == P1_MODE_SCATTER && p1_hook) nl += p1_hook();  // (after the slot is released)
            // the batch NS ahead takes this slot once this batch's pass 1 is done
            if (b + NS < lim) copy_batch(b + NS);
        }
        return nl;
    };
    if (host_reads) j->make_copy_stream();
    H2DChain chain;
    if (host_reads && !j->ctx.multipass) chain.begin(j->cs);
    if (sampled) {
        // ---- sample pass: histogram of every step-th segment (device reads) or of the first
        //      batch's every step-th segment (host reads)
        // device reads: every 32nd segment; host reads: segments of the first batch, about one
        // in 16 of all segments (every one when the batch is <= 1/16 of the input)
#ifndef KMC_SAMPLE_STEP
#define KMC_SAMPLE_STEP 32
#endif
        uint32_t step = KMC_SAMPLE_STEP;
        if (host_reads) {
            const uint64_t seg0 = p1_num_tiles(h_off[batches[0].second] - h_off[batches[0].first]);
            step = (uint32_t)std::max<uint64_t>(1, 16 * seg0 / std::max<uint64_t>(1, p1_num_tiles(n_bases)));
        }
        a.seg_step = step;
        htrace("sample pass");
        const int nls = run_p1(P1_MODE_HIST, 1);
        htrace("sample pass enqueued");
        a.seg_step = 1;
        j->launches += nls;
        const uint64_t seg_total = p1_num_tiles(n_bases);
        const uint64_t seg_in = host_reads ? p1_num_tiles(h_off[batches[0].second] - h_off[batches[0].first]) : n_tiles;
        const uint64_t seg_sampled = std::max<uint64_t>(1, (seg_in + step - 1) / step);
        const double F = (double)seg_total / (double)seg_sampled;
        const uint32_t fl = (uint32_t)std::ceil(F);
        CK(launch_scale_hist(hist_w, hist_r, ns, seg_total, seg_sampled, fl, fl, s));
        j->stage_end(nls + 1);
        PlanCtx& c = j->ctx;
        c.ns = ns;
        c.hist_w = hist_w;
        c.hist_r = hist_r;
        c.gstats = gstats;
        c.check_p1 = false;
        plan_phase(j, c);  // the plan of the estimates
        c.check_p1 = true;
        if (c.ev_plan) {
            CK(cudaEventDestroy(c.ev_plan));
            c.ev_plan = nullptr;
        }
        c.tables_pending = false;
        PlanArgs& pa = c.pa;
        const uint64_t n_bins = c.n_bins;
        const int RWs = record_words(k);
        // ---- bin capacities: estimate + 6 standard deviations + 64 records; offsets = their scan
        uint32_t* bin_cap = ar.get<uint32_t>(n_bins + 1);
        uint64_t* cap64 = ar.get<uint64_t>(n_bins + 1);
        uint64_t* cap_scan = ar.get<uint64_t>(n_bins + 2);
        void* ctemp = ar.alloc(scan_temp_bytes(n_bins + 1));
        CK(launch_bin_caps(pa.bin_nrec, n_bins, F, 6.0, 64, bin_cap, cap64, cap_scan, ctemp, s));
        unsigned long long* hs = j->host_small;
        CK(cudaMemcpyAsync(&hs[3], cap_scan + n_bins, 8, cudaMemcpyDeviceToHost, s));
        CK(cudaMemcpyAsync(pa.bin_rec_off, cap_scan, n_bins * 8, cudaMemcpyDeviceToDevice, s));
        // presplit: the estimated per-bin windows and records pick its bins
        const bool presplit = j->opt.presplit != 2 && (j->opt.presplit == 1 || host_reads) && kw == 1 && k <= 32 &&
                              j->opt.large_path == 0 && j->opt.count_path != 1;
        std::vector<uint64_t> bw_est, bn_est;
        if (presplit) {
            bw_est.resize(n_bins);
            bn_est.resize(n_bins);
            CK(cudaMemcpyAsync(bw_est.data(), pa.bin_w, n_bins * 8, cudaMemcpyDeviceToHost, s));
            CK(cudaMemcpyAsync(bn_est.data(), pa.bin_nrec, n_bins * 8, cudaMemcpyDeviceToHost, s));
        }
        CK(cudaStreamSynchronize(s));
        const uint64_t total_cap = hs[3];
        uint32_t* bins = reinterpret_cast<uint32_t*>(ar.alloc(total_cap * RWs * 4));
        uint32_t* bin_fill = ar.get<uint32_t>(n_bins);
        // ---- pass 1: every record straight into its bin, exact histograms alongside
        j->stage_begin(KMC_STAGE_SIGNATURE);
        CK(cudaMemsetAsync(bin_fill, 0, n_bins * 4, s));
        CK(cudaMemsetAsync(hist_w, 0, ns * 8, s));
        CK(cudaMemsetAsync(hist_r, 0, ns * 4, s));
        CK(cudaMemsetAsync(gstats, 0, GS_N * 8, s));
        uint4* sig_dest = ar.get<uint4>(ns);
        CK(launch_sig_dest(pa.sig2bin, bin_cap, pa.bin_rec_off, ns, sig_dest, s));
        a.sig2bin = pa.sig2bin;
        a.bin_rec_off = pa.bin_rec_off;
        a.bin_fill = bin_fill;
        a.bins = bins;
        a.sig_dest = sig_dest;
        a.scatter_hist = 1;
        keep_slots = true;  // batch 0 is still in its slot
        if (presplit) {
            presplit_setup(j, c, bw_est, bn_est, bin_cap, bin_fill, total_cap);
            if (c.pre.active) p1_hook = [&]() { return presplit_batch(j, c, bins); };
        }
        int nl = run_p1(P1_MODE_SCATTER);
        p1_hook = nullptr;
        a.sig_dest = nullptr;
        htrace("scatter pass enqueued");
        CK(cudaMemcpyAsync(&hs[4], gstats + GS_P1_OVF, 8, cudaMemcpyDeviceToHost, s));
        j->launches += nl;
        j->stage_end(nl);
        // ---- the exact per-bin tables on the sampled plan and their copies to the host are
        //      enqueued before the capacity check (a pass whose bins overflowed discards them
        //      and replans): one synchronisation after pass 1 instead of three
        j->stage_begin(KMC_STAGE_PLAN);
        int pl = 0;
        CK(launch_exact_tables(pa, n_bins, bin_fill, s, &pl));
        j->launches += pl;
        j->stage_end(pl);
        CK(cudaMemcpyAsync(&hs[1], pa.win_scan + ns, 8, cudaMemcpyDeviceToHost, s));
        CK(cudaMemcpyAsync(&hs[16], gstats, GS_N * 8, cudaMemcpyDeviceToHost, s));
        const bool early_tables = !j->cs && n_bins > 0;
        if (early_tables) {
            c.bw.resize(n_bins);
            c.bn.resize(n_bins);
            c.bo.resize(n_bins);
            CK(cudaMemcpyAsync(c.bw.data(), pa.bin_w, n_bins * 8, cudaMemcpyDeviceToHost, s));
            CK(cudaMemcpyAsync(c.bn.data(), pa.bin_nrec, n_bins * 8, cudaMemcpyDeviceToHost, s));
            CK(cudaMemcpyAsync(c.bo.data(), pa.bin_rec_off, n_bins * 8, cudaMemcpyDeviceToHost, s));
        }
        CK(cudaStreamSynchronize(s));
        ar.release(ctemp);
        ar.release(cap64);
        ar.release(cap_scan);
        if (hs[4] == 0) {
            c.n_windows = hs[1];
            c.n_records = hs[16 + GS_RECORDS];  // (the bins' fill counters are the per-bin counts)
            j->st.n_windows = c.n_windows;
            j->st.n_superkmers = hs[16 + GS_SUPERKMERS];
            j->st.n_records = c.n_records;
            j->st.n_invalid_bases = hs[16 + GS_INVALID];
            j->st.n_signatures_used = hs[16 + GS_SIGS_USED];
            j->st.max_signature_windows = hs[16 + GS_MAX_SIG];
            if (hs[16 + GS_WINDOWS] != c.n_windows) {
                set_err("sampled distribution: histogram totals disagree with pass-1 counters");
                throw Fail{KMC_ERR_INTERNAL};
            }
            if (c.n_windows > 0 && !early_tables) {
                c.tables_pending = true;
                CK(cudaEventCreateWithFlags(&c.ev_plan, cudaEventDisableTiming));
                CK(cudaEventRecord(c.ev_plan, s));
            }
        } else {
            // ---- a bin overflowed its sampled capacity: the exact histograms (a histogram
            //      pass: the scatter pass counts windows only), the exact plan, and the
            //      scatter again with exact offsets
            j->st.n_distribute_reruns += 1;
            presplit_release(j, c.pre);
            ar.release(bins);
            j->stage_begin(KMC_STAGE_SIGNATURE);
            CK(cudaMemsetAsync(hist_w, 0, ns * 8, s));
            CK(cudaMemsetAsync(hist_r, 0, ns * 4, s));
            CK(cudaMemsetAsync(gstats, 0, GS_N * 8, s));
            a.scatter_hist = 0;
            nl = run_p1(P1_MODE_HIST);
            j->launches += nl;
            j->stage_end(nl);
            plan_phase(j, c);
            bins = reinterpret_cast<uint32_t*>(ar.alloc(std::max<uint64_t>(c.n_records, 1) * RWs * 4));
            j->stage_begin(KMC_STAGE_SCATTER);
            if (c.n_bins > n_bins) bin_fill = ar.get<uint32_t>(c.n_bins);
            CK(cudaMemsetAsync(bin_fill, 0, std::max<uint64_t>(c.n_bins, 1) * 4, s));
            a.sig2bin = c.pa.sig2bin;
            a.bin_rec_off = c.pa.bin_rec_off;
            a.bin_fill = bin_fill;
            a.bins = bins;
            a.sig_dest = nullptr;
            a.scatter_hist = 0;
            nl = run_p1(P1_MODE_SCATTER);
            j->launches += nl;
            j->stage_end(nl);
        }
        chain.end(j->cs);
        c.bins_ready = bins;
        c.a = a;
        htrace("sampled distribution done");
        count_phase(j, c);
        return;
    }
    const int nl1 = run_p1(P1_MODE_HIST);
    chain.end(j->cs);
    j->launches += nl1;
    j->stage_end(nl1);

    PlanCtx& c = j->ctx;
    c.ns = ns;
    c.hist_w = hist_w;
    c.hist_r = hist_r;
    c.gstats = gstats;
    c.tmp_recs = tmp_recs;
    c.tmp_sig = tmp_sig;
    c.tmp_cap = tmp_cap;
    c.a = a;
    if (j->shard) return;  // sharded: the caller exchanges histograms and records (kmc_shard_*)
    c.run_p1 = [&](int mode) {
        a = c.a;
        return run_p1(mode);
    };
    plan_phase(j, c);
    count_phase(j, c);
    c.run_p1 = nullptr;
}

// S4 on the histograms in c.hist_w / c.hist_r: plan arrays on the device, bin tables on the host.
void plan_phase(kmc_job* j, PlanCtx& c) {
    const int k = j->k, kw = j->key_words;
    const size_t ksz = kw == 1 ? 8 : 16;
    Arena& ar = j->arena;
    cudaStream_t s = j->s;
    const uint64_t ns = c.ns;
    unsigned long long* hist_w = c.hist_w;
    uint32_t* hist_r = c.hist_r;
    unsigned long long* gstats = c.gstats;
    (void)ksz;
    // ---- S4: plan
    const int RW = record_words(k);
    int cap = small_capacity(k);
    if (j->opt.small_bin_capacity) cap = std::min<int>(cap, (int)j->opt.small_bin_capacity);
    if (j->opt.kx) cap = std::min(cap, kx_capacity());  // the (k,x)-mer kernel's bins
    if (j->opt.force_large) cap = 0;
    c.cap = cap;
    PlanArgs& pa = c.pa;
    pa = PlanArgs{};
    pa.hist_w = hist_w;
    pa.hist_r = hist_r;
    pa.ns = ns;
    pa.half_cap = std::max<uint64_t>(1, (uint64_t)cap / 2);
    pa.recw = (uint32_t)(RW * 4 / ksz);
    pa.cost_scan = ar.get<uint64_t>(ns + 1);
    pa.bnd_scan = ar.get<uint64_t>(ns + 1);
    pa.win_scan = ar.get<uint64_t>(ns + 1);
    pa.rec_scan = ar.get<uint64_t>(ns + 1);
    pa.sig2bin = ar.get<uint32_t>(ns);
    pa.bin_first = ar.get<uint64_t>(ns + 1);
    pa.bin_w = ar.get<uint64_t>(ns);
    pa.bin_nrec = ar.get<uint64_t>(ns);
    pa.bin_rec_off = ar.get<uint64_t>(ns);
    pa.gstats = gstats;
    pa.temp = ar.alloc(plan_temp_bytes(ns));
    j->stage_begin(KMC_STAGE_PLAN);
    int pl = 0;
    CK(launch_plan(pa, s, &pl));
    j->launches += pl;
    j->stage_end(pl);
    unsigned long long* hs = j->host_small;
    CK(cudaMemcpyAsync(&hs[0], pa.bnd_scan + ns, 8, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(&hs[1], pa.win_scan + ns, 8, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(&hs[2], pa.rec_scan + ns, 8, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(&hs[16], gstats, GS_N * 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    const uint64_t n_bins = hs[0], n_windows = hs[1], n_records = hs[2];
    c.n_bins = n_bins;
    c.n_windows = n_windows;
    c.n_records = n_records;
    c.tmp_n = hs[16 + GS_TMP_RECS];
    j->st.n_windows = n_windows;
    j->st.n_superkmers = hs[16 + GS_SUPERKMERS];
    j->st.n_records = n_records;
    j->st.n_invalid_bases = hs[16 + GS_INVALID];
    j->st.n_signatures_used = hs[16 + GS_SIGS_USED];
    j->st.max_signature_windows = hs[16 + GS_MAX_SIG];
    j->st.n_bins = n_bins;
    if (c.check_p1 && (hs[16 + GS_WINDOWS] != n_windows || hs[16 + GS_RECORDS] != n_records)) {
        set_err("histogram totals disagree with pass-1 counters (%llu/%llu windows, %llu/%llu records)",
                (unsigned long long)n_windows, (unsigned long long)hs[16 + GS_WINDOWS], (unsigned long long)n_records,
                (unsigned long long)hs[16 + GS_RECORDS]);
        throw Fail{KMC_ERR_INTERNAL};
    }
    if (n_windows == 0) return;
    c.tables_pending = true;  // the per-bin tables reach the host later (fetch_tables)
    CK(cudaEventCreateWithFlags(&c.ev_plan, cudaEventDisableTiming));
    CK(cudaEventRecord(c.ev_plan, s));
}

// Per-bin host tables (windows, records, first record), copied on the copy stream once the
// plan is done, so that the caller can enqueue device work (S5) before waiting for them.
void fetch_tables(kmc_job* j, PlanCtx& c) {
    if (!c.tables_pending) return;
    htrace("fetch_tables");
    c.tables_pending = false;
    const uint64_t n_bins = c.n_bins;
    c.bw.resize(n_bins);
    c.bn.resize(n_bins);
    c.bo.resize(n_bins);
    // on the copy stream when there is one (host reads; or S5 is still running), else on the
    // job's stream (creating a stream for three small copies costs more than it saves)
    cudaStream_t fs = j->cs ? j->cs : j->s;
    if (fs != j->s) CK(cudaStreamWaitEvent(fs, c.ev_plan, 0));
    cudaEventDestroy(c.ev_plan);
    c.ev_plan = nullptr;
    CK(cudaMemcpyAsync(c.bw.data(), c.pa.bin_w, n_bins * 8, cudaMemcpyDeviceToHost, fs));
    CK(cudaMemcpyAsync(c.bn.data(), c.pa.bin_nrec, n_bins * 8, cudaMemcpyDeviceToHost, fs));
    CK(cudaMemcpyAsync(c.bo.data(), c.pa.bin_rec_off, n_bins * 8, cudaMemcpyDeviceToHost, fs));
    CK(cudaStreamSynchronize(fs));
    htrace("tables fetched");
}

// ---- presplit (kmc_options.presplit): the large bins of the sampled plan -- estimated cost
//      above twice the small-bin capacity -- get their digit regions before pass 1 writes the
//      records (paired layout, digits of about 3/4 of a hash table each: a pair is one chunk
//      when the measured distinct ratio lets it fit the table), and every batch's new records
//      of those bins are split right after the batch's pass 1.
void presplit_setup(kmc_job* j, PlanCtx& c, const std::vector<uint64_t>& bw, const std::vector<uint64_t>& bn,
                    const uint32_t* bin_cap, const uint32_t* bin_fill, uint64_t total_cap) {
    PreSplit& pre = c.pre;
    Arena& ar = j->arena;
    cudaStream_t s = j->s;
    const int k = j->k;
    const uint64_t lim = 2ull * (uint64_t)c.cap;
    const double kf = (double)chunk_hash_cap(k) * 3 / 4;
    pre.ids.clear();
    pre.sb.clear();
    uint64_t key_base = 0, dbase = 0;
    for (uint64_t b = 0; b < c.n_bins; ++b) {
        const uint64_t cost = std::max<uint64_t>(bw[b], bn[b] * c.pa.recw);
        if (cost <= lim) continue;
        uint64_t d = 2 * (uint64_t)std::ceil((double)bw[b] / (2 * kf));
        d = std::min<uint64_t>(std::max<uint64_t>(d, 2), (uint64_t)S1_DMAX);
        // (more slack than the split after pass 1: the window count is an estimate)
        uint64_t r = (uint64_t)std::ceil((double)bw[b] / (double)d * 1.4) + 512;
        r = std::min<uint64_t>((r + 1) & ~1ull, 0x7FFFFFFEull);
        pre.ids.push_back(b);
        pre.sb.push_back(S1Bin{key_base, (uint32_t)d, (uint32_t)r, (uint32_t)dbase, S1_PAIRED});
        key_base += d * r;
        dbase += d;
    }
    if (pre.ids.empty() || pre.ids.size() >= (1ull << 31)) return;
    pre.keys = reinterpret_cast<uint64_t*>(ar.try_alloc(key_base * 8 + chunk_key_slack_bytes()));
    if (!pre.keys) {  // no room next to the bins: the split after pass 1
        pre.ids.clear();
        pre.sb.clear();
        return;
    }
    const size_t n = pre.ids.size();
    pre.n_digits = dbase;
    pre.index.assign(c.n_bins, -1);
    std::vector<uint32_t> ids32(n);
    for (size_t i = 0; i < n; ++i) {
        pre.index[pre.ids[i]] = (int32_t)i;
        ids32[i] = (uint32_t)pre.ids[i];
    }
    pre.rpp = (uint32_t)split1_uniform_records(k);
    pre.d_ids = ar.get<uint32_t>(n);
    pre.d_sbins = ar.get<S1Bin>(n);
    pre.done = ar.get<uint32_t>(n);
    pre.cur = ar.get<uint32_t>(dbase);
    pre.fail = ar.get<uint32_t>(dbase);
    pre.ovf_cap = std::max<uint64_t>(1u << 20, key_base / 32);
    pre.ovf = ar.get<uint64_t>(pre.ovf_cap);
    pre.ctr = ar.get<unsigned long long>(8);
    pre.pieces = ar.get<Piece>(total_cap / pre.rpp + 2 * n + 1);  // >= the pieces of any batch
    // (pageable sources: the copies are staged before the calls return)
    CK(cudaMemcpyAsync(pre.d_ids, ids32.data(), n * 4, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(pre.d_sbins, pre.sb.data(), n * sizeof(S1Bin), cudaMemcpyHostToDevice, s));
    CK(cudaMemsetAsync(pre.done, 0, n * 4, s));
    CK(cudaMemsetAsync(pre.cur, 0, dbase * 4, s));
    CK(cudaMemsetAsync(pre.fail, 0xFF, dbase * 4, s));
    CK(cudaMemsetAsync(pre.ctr, 0, 64, s));
    pre.bin_fill = bin_fill;
    pre.bin_cap = bin_cap;
    pre.bin_rec_off = c.pa.bin_rec_off;
    pre.active = true;
}

int presplit_batch(kmc_job* j, PlanCtx& c, const uint32_t* bins) {
    PreSplit& pre = c.pre;
    cudaStream_t s = j->s;
    CK(launch_presplit_pieces(pre.d_ids, (uint32_t)pre.ids.size(), pre.bin_fill, pre.bin_cap, pre.bin_rec_off,
                              pre.done, pre.rpp, pre.pieces, pre.ctr + 5, s));
    CK(launch_split1(bins, pre.pieces, 0, pre.d_sbins, j->k, !j->opt.non_canonical, pre.cur, pre.keys, pre.ovf,
                     pre.ctr + 3, pre.ovf_cap, 2 * n_sms(), s, pre.ctr + 5, pre.fail, true));
    return 2;
}

void presplit_release(kmc_job* j, PreSplit& pre) {
    Arena& ar = j->arena;
    for (void* q : {(void*)pre.keys, (void*)pre.d_ids, (void*)pre.d_sbins, (void*)pre.done, (void*)pre.cur,
                    (void*)pre.fail, (void*)pre.ovf, (void*)pre.ctr, (void*)pre.pieces})
        ar.release(q);
    pre = PreSplit{};
}

// Large bins of the default path for k <= 32 (k_split1.cu): one sized split pass puts every
// key of a bin into the region of its hashed digit (a bin of W windows: nd ~ W / (0.8 kcap)
// digits of rc ~ 1.05 W / nd slots), then every digit that fits its region is one chunk of the
// SMEM hash count.  Digits that overflowed their region (region part + the overflow list)
// and chunks whose distinct keys overflow the hash table are counted by the device radix sort.
// Bins are processed in groups whose regions fit the device budget.
template <class DR>
void large_split1(kmc_job* j, PlanCtx& c, const uint32_t* bins, const std::vector<uint64_t>& large_ids, int kcap,
                  DR&& distinct_ratio) {
    htrace("large_split1");
    (void)distinct_ratio;
    PreSplit& pre = c.pre;
    // presplit bins that the exact plan made large are counted from their regions; the
    // others take the split below
    std::vector<uint64_t> rest_ids;
    std::vector<uint8_t> pre_used;
    if (pre.active) {
        pre_used.assign(pre.ids.size(), 0);
        for (const uint64_t b : large_ids) {
            const int32_t x = pre.index[b];
            if (x >= 0) pre_used[(size_t)x] = 1;
            else rest_ids.push_back(b);
        }
    }
    const std::vector<uint64_t>& ids = pre.active ? rest_ids : large_ids;
    const int k = j->k;
    Arena& ar = j->arena;
    cudaStream_t s = j->s;
    unsigned long long* hs = j->host_small;
    unsigned long long* gstats = c.gstats;
    const HostTable& bw = c.bw;
    const HostTable& bn = c.bn;
    const HostTable& bo = c.bo;
    // digit target = kcap keys; regions 1.25x the mean + 256 (hashed digits are near-uniform,
    // but a k-mer of multiplicity m moves m keys at once: repeat families skew them).  C4
    // (tools/stage_run.py, target / kcap 0.6 .. 1.1): 62.4, 60.8, 60.1, 60.0, 59.9 ms/step,
    // overflow 6.0 M .. 0.4 M keys; bigger digits absorb pile-ups and need fewer reservations.
    const double target = std::max(1.0, (double)kcap);
    RadixScratch rs{};
    uint64_t rs_cap = 0;
    auto sort_rle = [&](uint64_t* keys, uint64_t n, int& nlaunch) {
        if (n == 0) return;
        if (n > rs_cap) {
            ar.release(rs.keys_alt);
            ar.release(rs.tile_hist);
            ar.release(rs.tile_off);
            ar.release(rs.scan_temp);
            rs.keys_alt = ar.alloc(n * 8);
            rs.tile_hist = ar.get<uint32_t>(radix_status_words(n, 1));
            rs.tile_off = ar.get<uint32_t>(radix_aux_words());
            rs.scan_temp = ar.alloc(radix_scan_temp_bytes(n, 1));
            if (!rs.red) rs.red = ar.get<unsigned long long>(4);
            rs.red_host = hs + 40;
            rs_cap = n;
        }
        void* sorted = nullptr;
        uint32_t* dummy = nullptr;
        CK(device_radix_sort(1, keys, nullptr, n, 2 * k, rs, s, &sorted, &dummy, &nlaunch));
        CK(launch_rle(1, sorted, n, j->ci, j->cx, j->surv_keys, j->surv_counts, gstats, s));
        nlaunch += 1;
    };
    // S7-S8 of a split group: its chunks by the SMEM hash count; overflowed digits (region
    // parts + the overflow list) and chunks that overflowed the table by the device radix sort
    auto count_group = [&](uint64_t* lkeys, uint64_t* ovf, uint64_t ovf_cap, Chunk* chunks, Chunk* over, Chunk* ovd,
                           Chunk* tovf, unsigned long long* ctr, uint64_t n_chunks, uint64_t n_over, uint64_t n_ovd,
                           uint64_t n_ovk) {
        j->stage_begin(KMC_STAGE_LARGE_CHUNKS);
        CK(launch_chunk_hash(lkeys, chunks, n_chunks, k, j->ci, j->cx, j->surv_keys, j->surv_counts, gstats, tovf,
                             ctr + 4, n_sms(), s));
        j->launches += 1;
        j->stage_end(1);
        CK(cudaMemcpyAsync(&hs[52], ctr + 4, 8, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        const uint64_t n_tovf = hs[52];
        htrace("chunk_hash done");
        j->st.n_overflow_chunks += n_tovf;
        if (n_over + n_ovd + n_ovk + n_tovf == 0) return;
        int fl = 0;
        j->stage_begin(KMC_STAGE_LARGE_FALLBACK);
        if (n_ovd + n_ovk > 0) {
            // overflowed digits: their region parts join their excess keys in the overflow list
            std::vector<Chunk> od(n_ovd);
            if (n_ovd) {
                CK(cudaMemcpyAsync(od.data(), ovd, n_ovd * sizeof(Chunk), cudaMemcpyDeviceToHost, s));
                CK(cudaStreamSynchronize(s));
            }
            uint64_t need = n_ovk;
            for (const Chunk& x : od) need += x.n;
            j->st.n_split_overflow += need;
            uint64_t* all = ovf;
            if (need > ovf_cap) {
                all = ar.get<uint64_t>(need);
                if (n_ovk) CK(cudaMemcpyAsync(all, ovf, n_ovk * 8, cudaMemcpyDeviceToDevice, s));
            }
            uint64_t o = n_ovk;
            for (const Chunk& x : od) {
                CK(cudaMemcpyAsync(all + o, lkeys + x.begin, (size_t)x.n * 8, cudaMemcpyDeviceToDevice, s));
                o += x.n;
            }
            sort_rle(all, need, fl);
            if (all != ovf) ar.release(all);
        }
        if (n_over + n_tovf > 0) {
            std::vector<Chunk> ov(n_over + n_tovf);
            if (n_over) CK(cudaMemcpyAsync(ov.data(), over, n_over * sizeof(Chunk), cudaMemcpyDeviceToHost, s));
            if (n_tovf)
                CK(cudaMemcpyAsync(ov.data() + n_over, tovf, n_tovf * sizeof(Chunk), cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
            for (const Chunk& x : ov) {
                if (x.pad) {  // a pair of digits: two segments (disjoint keys)
                    const uint32_t n0 = x.pad & 0xFFFFu, gap = x.pad >> 16;
                    sort_rle(lkeys + x.begin, n0, fl);
                    sort_rle(lkeys + x.begin + n0 + gap, x.n - n0, fl);
                } else {
                    sort_rle(lkeys + x.begin, x.n, fl);
                }
            }
        }
        j->launches += fl;
        j->stage_end(fl);
        htrace("fallback enqueued");
    };
    // ---- the presplit group: its regions are filled; list the chunks (a pair of digits that
    //      fits the table together is one chunk) and count them
    if (pre.active) {
        size_t used = 0;
        for (uint8_t u : pre_used) used += u;
        if (used) {
            const size_t n = pre.ids.size();
            std::vector<S1Bin> sbl = pre.sb;
            for (size_t i = 0; i < n; ++i)
                if (!pre_used[i]) sbl[i].nd = 0;  // small after all: counted from its records
            CK(cudaMemcpyAsync(pre.d_sbins, sbl.data(), n * sizeof(S1Bin), cudaMemcpyHostToDevice, s));
            const uint64_t nd_all = std::max<uint64_t>(pre.n_digits, 1);
            Chunk* pch = ar.get<Chunk>(nd_all);
            Chunk* pov = ar.get<Chunk>(nd_all);
            Chunk* povd = ar.get<Chunk>(nd_all);
            Chunk* ptovf = ar.get<Chunk>(nd_all);
            j->stage_begin(KMC_STAGE_LARGE_SCATTER);
            CK(launch_split1_chunks(pre.d_sbins, n, pre.cur, 0xFFFFFFFFu, pch, pov, povd, pre.ctr, s, (uint32_t)kcap,
                                    pre.fail));
            j->launches += 1;
            j->stage_end(1);
            CK(cudaMemcpyAsync(&hs[48], pre.ctr, 32, cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
            if (hs[51] <= pre.ovf_cap) {
                j->st.n_presplit_bins += used;
                j->st.n_large_groups += 1;
                count_group(pre.keys, pre.ovf, pre.ovf_cap, pch, pov, povd, ptovf, pre.ctr, hs[48], hs[49], hs[50],
                            hs[51]);
            } else {
                // the overflow list overflowed during the presplit: split these bins again
                for (size_t i = 0; i < n; ++i)
                    if (pre_used[i]) rest_ids.push_back(pre.ids[i]);
                std::sort(rest_ids.begin(), rest_ids.end());
            }
            ar.release(pch);
            ar.release(pov);
            ar.release(povd);
            ar.release(ptovf);
        }
        presplit_release(j, pre);
    }
    if (ids.empty()) {
        ar.release(rs.keys_alt);
        ar.release(rs.tile_hist);
        ar.release(rs.tile_off);
        ar.release(rs.scan_temp);
        return;
    }
    htrace("split1 plan");
    const size_t nl = ids.size();
    std::vector<uint32_t> nd(nl), rc(nl), rpb(nl);
    uint64_t total = 0;
    for (size_t i = 0; i < nl; ++i) {
        const uint64_t b = ids[i];
        uint64_t d = (uint64_t)std::ceil((double)bw[b] / target);
        d = std::min<uint64_t>(std::max<uint64_t>(d, 1), (uint64_t)S1_DMAX);
        uint64_t r = j->opt.split_tight ? (bw[b] + d - 1) / d + 2
                                        : (uint64_t)std::ceil((double)bw[b] / (double)d * 1.25) + 256;
        r = std::min<uint64_t>((r + 1) & ~1ull, 0x7FFFFFFEull);
        nd[i] = (uint32_t)d;
        rc[i] = (uint32_t)r;
        rpb[i] = (uint32_t)split1_bin_records(k, bw[b], bn[b], (uint32_t)d);  // pieces sized by windows
        total += d * r;
    }
    // group budget in region keys: the option, else everything if the key buffer can be
    // allocated, else half the free device memory
    uint64_t budget = j->opt.large_group_mkeys ? ((uint64_t)j->opt.large_group_mkeys << 20) : ~0ull;
    void* lkeys = nullptr;
    if (!j->opt.large_group_mkeys) {
        lkeys = ar.try_alloc(total * 8 + chunk_key_slack_bytes());
        if (!lkeys) {
            size_t fr = 0, tot = 0;
            CK(cudaMemGetInfo(&fr, &tot));
            budget = std::max<uint64_t>((uint64_t)(fr / 2) / 9, 1u << 20);
        }
    }
    htrace("split1 keys allocated");
    std::vector<std::pair<size_t, size_t>> groups;
    uint64_t max_gk = 0, max_gd = 0, max_gp = 0, max_gn = 0;
    for (size_t i0 = 0; i0 < nl;) {
        uint64_t gk = 0, gd = 0, gp = 0;
        size_t i1 = i0;
        while (i1 < nl) {
            const uint64_t need = (uint64_t)nd[i1] * rc[i1];
            if (i1 > i0 && gk + need > budget) break;
            gk += need;
            gd += nd[i1];
            gp += (bn[ids[i1]] + rpb[i1] - 1) / rpb[i1];
            ++i1;
        }
        groups.push_back({i0, i1});
        max_gk = std::max(max_gk, gk);
        max_gd = std::max(max_gd, gd);
        max_gp = std::max(max_gp, gp);
        max_gn = std::max<uint64_t>(max_gn, i1 - i0);
        i0 = i1;
    }
    j->st.n_large_groups += groups.size();
    LargeBin* d_lbins = ar.get<LargeBin>(max_gn);
    S1Bin* d_sbins = ar.get<S1Bin>(max_gn);
    uint64_t* d_pp = ar.get<uint64_t>(max_gn + 1);
    Piece* d_pieces = ar.get<Piece>(max_gp);
    uint32_t* cur = ar.get<uint32_t>(max_gd);
    Chunk* chunks = ar.get<Chunk>(max_gd);
    Chunk* over = ar.get<Chunk>(max_gd);
    Chunk* ovd = ar.get<Chunk>(max_gd);
    Chunk* tovf = ar.get<Chunk>(max_gd);  // chunks whose distinct keys overflowed the hash table
    unsigned long long* ctr = ar.get<unsigned long long>(5);  // chunks, oversize, overflowed digits, overflow keys, table overflows
    if (!lkeys) lkeys = ar.alloc(max_gk * 8 + chunk_key_slack_bytes());
    uint64_t ovf_cap = std::max<uint64_t>(1u << 20, max_gk / 32);
    uint64_t* ovf = ar.get<uint64_t>(ovf_cap);
    htrace("split1 buffers");
    // pinned: the table copies below are asynchronous (a group's copies have completed when
    // the next group rewrites the tables -- every group ends with a stream synchronisation)
    PinnedArr<LargeBin> lbins;
    PinnedArr<S1Bin> sbins;
    PinnedArr<uint64_t> pp;
    for (const auto& g : groups) {
        const size_t gn = g.second - g.first;
        lbins.resize(gn);
        sbins.resize(gn);
        pp.resize(gn + 1);
        pp[0] = 0;
        uint64_t key_base = 0, dbase = 0;
        for (size_t i = 0; i < gn; ++i) {
            const size_t li = g.first + i;
            const uint64_t b = ids[li];
            lbins[i] = LargeBin{0, 0, bo[b], 0, (uint32_t)bw[b], 0, (uint32_t)bn[b], 0, rpb[li], 0};
            sbins[i] = S1Bin{key_base, nd[li], rc[li], (uint32_t)dbase, 0};
            key_base += (uint64_t)nd[li] * rc[li];
            dbase += nd[li];
            pp[i + 1] = pp[i] + (bn[b] + rpb[li] - 1) / rpb[li];
        }
        const uint64_t n_pieces = pp[gn];
        htrace("split1 tables");
        CK(cudaMemcpyAsync(d_lbins, lbins.data(), gn * sizeof(LargeBin), cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(d_sbins, sbins.data(), gn * sizeof(S1Bin), cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(d_pp, pp.data(), pp.size() * 8, cudaMemcpyHostToDevice, s));
        uint64_t n_chunks = 0, n_over = 0, n_ovd = 0, n_ovk = 0;
        for (;;) {
            j->stage_begin(KMC_STAGE_LARGE_SCATTER);
            CK(cudaMemsetAsync(cur, 0, dbase * 4, s));
            CK(cudaMemsetAsync(ctr, 0, 40, s));
            CK(launch_make_pieces(d_lbins, d_pp, gn, 0, d_pieces, s));  // (rpp 0: LargeBin.nseg per bin)
            htrace("split1 launch");
            CK(launch_split1(bins, d_pieces, n_pieces, d_sbins, k, !j->opt.non_canonical, cur, (uint64_t*)lkeys, ovf,
                             ctr + 3, ovf_cap, 2 * n_sms(), s));
            CK(launch_split1_chunks(d_sbins, gn, cur, 0xFFFFFFFFu, chunks, over, ovd, ctr, s));
            j->launches += 3;
            j->stage_end(3);
            CK(cudaMemcpyAsync(&hs[48], ctr, 32, cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
            n_chunks = hs[48];
            n_over = hs[49];
            n_ovd = hs[50];
            n_ovk = hs[51];
            if (n_ovk <= ovf_cap) break;
            // the overflow list was too small for the digits' excess keys (the same amount on
            // a rerun: it depends only on the keys): grow it and split the group again
            ar.release(ovf);
            ovf_cap = n_ovk + (n_ovk >> 3) + 1024;
            ovf = ar.get<uint64_t>(ovf_cap);
        }
        htrace("split1 done");
        count_group((uint64_t*)lkeys, ovf, ovf_cap, chunks, over, ovd, tovf, ctr, n_chunks, n_over, n_ovd, n_ovk);
    }
    ar.release(lkeys);
    ar.release(ovf);
    ar.release(rs.keys_alt);
    ar.release(rs.tile_hist);
    ar.release(rs.tile_off);
    ar.release(rs.scan_temp);
}

// Large bins through sub-signatures (k_subsplit.cu, large_path 4): a bin of W windows gets
// nd ~ W / kcap digits; k_subsplit cuts its records into sub-records by digit, k_subcount
// counts every digit in one CTA's SMEM hash table (in hash-range rounds when its distinct keys
// overflow the table).  A digit's sub-records fill its region (sized for 1 sub-record per 3
// windows: C4 has 5.3), then pool blocks claimed on the device; digits whose sub-records
// overflowed their block table -- and the overflow list -- are expanded and counted by the
// device radix sort.  Bins are processed in groups whose regions fit the device.
void large_subsplit(kmc_job* j, PlanCtx& c, const uint32_t* bins, const std::vector<uint64_t>& large_ids, int kcap) {
    const int k = j->k;
    Arena& ar = j->arena;
    cudaStream_t s = j->s;
    unsigned long long* hs = j->host_small;
    unsigned long long* gstats = c.gstats;
    const HostTable& bw = c.bw;
    const HostTable& bn = c.bn;
    const HostTable& bo = c.bo;
    const double target = std::max(1.0, (double)kcap);
    const uint32_t rpp = (uint32_t)subsplit_piece_records(k);
    const size_t nl = large_ids.size();
    std::vector<uint32_t> nd(nl), rc(nl);
    uint64_t total_slots = 0;
    for (size_t i = 0; i < nl; ++i) {
        const uint64_t b = large_ids[i];
        uint64_t d = (uint64_t)std::ceil((double)bw[b] / target);
        d = std::min<uint64_t>(std::max<uint64_t>(d, 1), (uint64_t)SS_DMAX);
        nd[i] = (uint32_t)d;
        const uint64_t r = (bw[b] / d) / 3 + 32;
        rc[i] = (uint32_t)std::min<uint64_t>(r, 1u << 30);
        total_slots += d * rc[i];
    }
    const size_t slot_bytes = 16;
    // group budget in region slots: the option, else everything if the pool can be allocated,
    // else half the free device memory
    uint64_t budget = j->opt.large_group_mkeys ? (((uint64_t)j->opt.large_group_mkeys << 20) / 3 + 1) : ~0ull;
    uint64_t n_blocks = std::max<uint64_t>(256, total_slots / 16 / SS_BLK);  // extra blocks (lumpy digits)
    void* pool = nullptr;
    uint64_t pool_slots = 0;
    if (!j->opt.large_group_mkeys) {
        pool = ar.try_alloc((total_slots + n_blocks * SS_BLK) * slot_bytes);
        if (pool) {
            pool_slots = total_slots;
        } else {
            size_t fr = 0, tot = 0;
            CK(cudaMemGetInfo(&fr, &tot));
            budget = std::max<uint64_t>((uint64_t)(fr / 2) / slot_bytes, 1u << 16);
        }
    }
    std::vector<std::pair<size_t, size_t>> groups;
    uint64_t max_gs = 0, max_gd = 0, max_gp = 0, max_gn = 0;
    for (size_t i0 = 0; i0 < nl;) {
        uint64_t gs = 0, gd = 0, gp = 0;
        size_t i1 = i0;
        while (i1 < nl) {
            const uint64_t need = (uint64_t)nd[i1] * rc[i1];
            if (i1 > i0 && gs + need > budget) break;
            gs += need;
            gd += nd[i1];
            gp += (bn[large_ids[i1]] + rpp - 1) / rpp;
            ++i1;
        }
        groups.push_back({i0, i1});
        max_gs = std::max(max_gs, gs);
        max_gd = std::max(max_gd, gd);
        max_gp = std::max(max_gp, gp);
        max_gn = std::max<uint64_t>(max_gn, i1 - i0);
        i0 = i1;
    }
    j->st.n_large_groups += groups.size();
    if (!pool) {
        pool_slots = max_gs;
        n_blocks = std::max<uint64_t>(256, max_gs / 16 / SS_BLK);
        pool = ar.alloc((pool_slots + n_blocks * SS_BLK) * slot_bytes);
    }
    SSBin* d_sbins = ar.get<SSBin>(max_gn);
    LargeBin* d_lbins = ar.get<LargeBin>(max_gn);
    uint64_t* d_pp = ar.get<uint64_t>(max_gn + 1);
    Piece* d_pieces = ar.get<Piece>(max_gp);
    uint32_t* cur = ar.get<uint32_t>(2 * max_gd);  // sub-records, then windows per digit
    uint32_t* btab = ar.get<uint32_t>(max_gd * SS_MAXB);
    uint32_t* fb = ar.get<uint32_t>(max_gd);
    uint2* dinfo = ar.get<uint2>(max_gd);
    uint32_t* drc = ar.get<uint32_t>(max_gd);
    unsigned long long* ctr = ar.get<unsigned long long>(4);  // blocks, overflow sub-records, fallback digits, error
    uint64_t ovf_cap = 1u << 16;
    uint4* ovf = ar.get<uint4>(ovf_cap);
    static thread_local std::vector<LargeBin> lbins;
    static thread_local std::vector<SSBin> sbins;
    static thread_local std::vector<uint64_t> pp;
    for (const auto& g : groups) {
        const size_t gn = g.second - g.first;
        lbins.resize(gn);
        sbins.resize(gn);
        pp.assign(gn + 1, 0);
        uint32_t dbase = 0;
        uint64_t rbase = 0;
        for (size_t i = 0; i < gn; ++i) {
            const size_t li = g.first + i;
            const uint64_t b = large_ids[li];
            lbins[i] = LargeBin{0, 0, bo[b], 0, (uint32_t)bw[b], 0, (uint32_t)bn[b], 0, 0, 0};
            sbins[i] = SSBin{rbase, nd[li], dbase, rc[li], 0};
            dbase += nd[li];
            rbase += (uint64_t)nd[li] * rc[li];
            pp[i + 1] = pp[i] + (bn[b] + rpp - 1) / rpp;
        }
        const uint64_t n_pieces = pp.back();
        CK(cudaMemcpyAsync(d_lbins, lbins.data(), gn * sizeof(LargeBin), cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(d_sbins, sbins.data(), gn * sizeof(SSBin), cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(d_pp, pp.data(), pp.size() * 8, cudaMemcpyHostToDevice, s));
        uint64_t n_ovs = 0;
        for (;;) {
            j->stage_begin(KMC_STAGE_LARGE_SCATTER);
            CK(cudaMemsetAsync(cur, 0, (size_t)dbase * 8, s));
            CK(cudaMemsetAsync(btab, 0, (size_t)dbase * SS_MAXB * 4, s));
            CK(cudaMemsetAsync(ctr, 0, 32, s));
            CK(launch_make_pieces(d_lbins, d_pp, gn, rpp, d_pieces, s));
            CK(launch_subsplit(bins, d_pieces, n_pieces, d_sbins, k, cur, cur + dbase, btab, pool, pool_slots, n_blocks,
                               ovf, ovf_cap, ctr, 2 * n_sms(), s));
            j->launches += 2;
            j->stage_end(2);
            CK(cudaMemcpyAsync(&hs[48], ctr, 16, cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
            const uint64_t used = hs[48];
            n_ovs = hs[49];
            if (used <= n_blocks && n_ovs <= ovf_cap) break;
            // the extra blocks (or the overflow list) were too few: the same amount on a rerun
            // (it depends only on the records), so grow them and split the group again
            if (used > n_blocks) {
                ar.release(pool);
                n_blocks = used + used / 8 + 64;
                pool = ar.alloc((pool_slots + n_blocks * SS_BLK) * slot_bytes);
            }
            if (n_ovs > ovf_cap) {
                ar.release(ovf);
                ovf_cap = n_ovs + n_ovs / 8 + 1024;
                ovf = ar.get<uint4>(ovf_cap);
            }
        }
        j->stage_begin(KMC_STAGE_LARGE_CHUNKS);
        CK(launch_subcount(pool, pool_slots, d_sbins, (uint32_t)gn, dinfo, drc, cur, cur + dbase, btab, dbase, k,
                           !j->opt.non_canonical, j->ci, j->cx, (uint64_t*)j->surv_keys, j->surv_counts, gstats, fb,
                           ctr + 2, n_sms(), s));
        j->launches += 2;
        j->stage_end(2);
        CK(cudaMemcpyAsync(&hs[52], ctr + 2, 16, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        const uint64_t n_fb = hs[52];
        if (hs[53]) {
            set_err("sub-signature count: a digit overflowed 2^20 hash-range rounds");
            throw Fail{KMC_ERR_INTERNAL};
        }
        if (n_fb == 0) continue;
        // ---- fallback: the listed digits' sub-records (region, extra blocks, the overflow
        // list) are expanded into keys and counted by the device radix sort (digits partition
        // the keys, so one sort of their union counts each of them)
        int fl = 0;
        j->stage_begin(KMC_STAGE_LARGE_FALLBACK);
        std::vector<uint32_t> fd(n_fb), fn(n_fb), fw(n_fb);
        CK(cudaMemcpyAsync(fd.data(), fb, n_fb * 4, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        std::vector<uint32_t> tabs(n_fb * (size_t)SS_MAXB);
        for (uint64_t i = 0; i < n_fb; ++i) {
            CK(cudaMemcpyAsync(&fn[i], cur + fd[i], 4, cudaMemcpyDeviceToHost, s));
            CK(cudaMemcpyAsync(&fw[i], cur + dbase + fd[i], 4, cudaMemcpyDeviceToHost, s));
            CK(cudaMemcpyAsync(tabs.data() + i * SS_MAXB, btab + (size_t)fd[i] * SS_MAXB, SS_MAXB * 4,
                               cudaMemcpyDeviceToHost, s));
        }
        CK(cudaStreamSynchronize(s));
        uint64_t nsub = n_ovs, nkeys = 0;
        for (uint64_t i = 0; i < n_fb; ++i) {
            const size_t bi = std::upper_bound(sbins.begin(), sbins.end(), fd[i],
                                               [](uint32_t d, const SSBin& x) { return d < x.dbase; }) -
                              sbins.begin() - 1;
            nsub += std::min<uint64_t>(fn[i], (uint64_t)sbins[bi].rc + (uint64_t)SS_MAXB * SS_BLK);
            nkeys += fw[i];
        }
        j->st.n_split_overflow += nkeys;
        uint4* subs = ar.get<uint4>(nsub + 1);
        uint64_t o = 0;
        for (uint64_t i = 0; i < n_fb; ++i) {
            const size_t bi = std::upper_bound(sbins.begin(), sbins.end(), fd[i],
                                               [](uint32_t d, const SSBin& x) { return d < x.dbase; }) -
                              sbins.begin() - 1;
            const SSBin& sb = sbins[bi];
            const uint64_t m = std::min<uint64_t>(fn[i], (uint64_t)sb.rc + (uint64_t)SS_MAXB * SS_BLK);
            const uint64_t mr = std::min<uint64_t>(m, sb.rc);
            CK(cudaMemcpyAsync(subs + o, (uint4*)pool + sb.rbase + (uint64_t)(fd[i] - sb.dbase) * sb.rc, mr * 16,
                               cudaMemcpyDeviceToDevice, s));
            o += mr;
            for (uint64_t q = 0; mr + q * SS_BLK < m; ++q) {
                const uint64_t e = std::min<uint64_t>(SS_BLK, m - mr - q * SS_BLK);
                CK(cudaMemcpyAsync(subs + o, (uint4*)pool + pool_slots + (uint64_t)(tabs[i * SS_MAXB + q] - 1) * SS_BLK,
                                   e * 16, cudaMemcpyDeviceToDevice, s));
                o += e;
            }
        }
        if (n_ovs) CK(cudaMemcpyAsync(subs + o, ovf, n_ovs * 16, cudaMemcpyDeviceToDevice, s));
        o += n_ovs;
        // pieces of PIECE_RECORDS sub-records over the gathered array
        std::vector<Piece> pcs;
        for (uint64_t q = 0; q < o; q += PIECE_RECORDS)
            pcs.push_back(Piece{q, (uint32_t)std::min<uint64_t>(PIECE_RECORDS, o - q), 0});
        Piece* d_fp = ar.get<Piece>(pcs.size());
        CK(cudaMemcpyAsync(d_fp, pcs.data(), pcs.size() * sizeof(Piece), cudaMemcpyHostToDevice, s));
        uint64_t* keys = ar.get<uint64_t>(nkeys + 1);
        CK(cudaMemsetAsync(gstats + GS_LARGE_KEYS, 0, 8, s));
        CK(launch_large_expand((const uint32_t*)subs, d_fp, pcs.size(), k, !j->opt.non_canonical, keys, gstats, s));
        ++fl;
        RadixScratch rs{};
        rs.keys_alt = ar.alloc(nkeys * 8 + 8);
        rs.tile_hist = ar.get<uint32_t>(radix_status_words(nkeys, 1));
        rs.tile_off = ar.get<uint32_t>(radix_aux_words());
        rs.scan_temp = ar.alloc(radix_scan_temp_bytes(nkeys, 1));
        rs.red = ar.get<unsigned long long>(4);
        rs.red_host = hs + 40;
        void* sorted = nullptr;
        uint32_t* dummy = nullptr;
        CK(device_radix_sort(1, keys, nullptr, nkeys, 2 * k, rs, s, &sorted, &dummy, &fl));
        CK(launch_rle(1, sorted, nkeys, j->ci, j->cx, j->surv_keys, j->surv_counts, gstats, s));
        ++fl;
        j->launches += fl;
        j->stage_end(fl);
        CK(cudaStreamSynchronize(s));  // the host vectors above are released on return
        ar.release(subs);
        ar.release(d_fp);
        ar.release(keys);
        ar.release(rs.keys_alt);
        ar.release(rs.tile_hist);
        ar.release(rs.tile_off);
        ar.release(rs.scan_temp);
        ar.release(rs.red);
    }
    ar.release(pool);
    ar.release(ovf);
}

// S5-S8 from the record stream in c (tmp_recs / tmp_sig, tmp_n slots) and the plan:
// bins, then small and large bins counted into the survivor buffer.
void count_phase(kmc_job* j, PlanCtx& c) {
    const int k = j->k, kw = j->key_words;
    const size_t ksz = kw == 1 ? 8 : 16;
    Arena& ar = j->arena;
    cudaStream_t s = j->s;
    const int RW = record_words(k);
    const int cap = c.cap;
    PlanArgs& pa = c.pa;
    unsigned long long* hs = j->host_small;
    unsigned long long* gstats = c.gstats;
    const uint64_t n_bins = c.n_bins, n_windows = c.n_windows, n_records = c.n_records;
    const HostTable& bw = c.bw;
    const HostTable& bn = c.bn;
    const HostTable& bo = c.bo;
    uint32_t* tmp_recs = c.tmp_recs;
    uint32_t* tmp_sig = c.tmp_sig;
    const uint64_t tmp_cap = c.tmp_cap;
    if (n_windows == 0) {
        j->n_surv = 0;
        return;
    }
    j->st.n_passes = 1;
    if (c.multipass) {
        count_multipass(j, c);
        return;
    }
    // ---- S5: records into bins -- a copy from pass 1's temporary stream, or (if the stream
    //      overflowed its estimate) pass 2 = S1-S3 recomputed + scatter; nothing when the
    //      sampled distribution has written them already
    uint32_t* bins = c.bins_ready ? c.bins_ready : reinterpret_cast<uint32_t*>(ar.alloc(n_records * RW * 4));
    const uint64_t tmp_n = c.tmp_n;
    j->stage_begin(KMC_STAGE_SCATTER);
    int s5_launches = 0;
    if (c.bins_ready) {
        // (pass 1 wrote the bins)
    } else if (tmp_recs && tmp_n <= tmp_cap) {
        // MSD passes of <= 8 bits over the bin id; the last one writes the bins
        int B = 1;
        while ((1ull << B) < n_bins) ++B;
        std::vector<int> D;
        for (int bits = 0; bits < B; bits += D.back()) D.push_back(std::min(8, B - bits));
        const int L = (int)D.size();
        const uint64_t TI = rec_tile_items(k);
        unsigned long long* cursor = ar.get<unsigned long long>((1ull << B) + 1);
        const uint64_t max_tiles = std::max(tmp_n, n_records) / TI + n_bins + 2;  // + one partial tile per bucket
        RecTile2* d_tiles = ar.get<RecTile2>(max_tiles);
        uint64_t* t_prefix = ar.get<uint64_t>(n_bins + 2);
        void* t_temp = ar.alloc(scan_temp_bytes(n_bins + 2));
        uint32_t* x_recs = L > 1 ? reinterpret_cast<uint32_t*>(ar.alloc(n_records * RW * 4)) : nullptr;
        uint32_t* x_ids = L > 1 ? ar.get<uint32_t>(n_records) : nullptr;
        const uint32_t* in_r = tmp_recs;
        const uint32_t* in_i = tmp_sig;
        int prefix = 0;
        for (int l = 0; l < L; ++l) {
            const int shift_prev = B - prefix;
            prefix += D[l];
            const int shift = B - prefix;
            // tiles (device-built): pass 0 cuts the stream, later passes every bucket of the
            // previous pass (bins [v << shift_prev, (v + 1) << shift_prev))
            uint64_t nbp = 1, mt = tmp_n / TI + 1;
            TileSrc src{nullptr, 1, 0, 0, tmp_n};
            if (l > 0) {
                nbp = (n_bins + (1ull << shift_prev) - 1) >> shift_prev;
                mt = n_records / TI + nbp;
                src = TileSrc{pa.bin_rec_off, 1, n_bins, shift_prev, n_records};
            }
            CK(launch_make_tiles(src, nbp, (uint32_t)TI, mt, t_prefix, t_temp, d_tiles, s));
            const uint64_t nbk = (n_bins + (1ull << shift) - 1) >> shift;
            CK(launch_bucket_cursors(pa.bin_rec_off, n_bins, n_records, shift, nbk, cursor, s));
            // ping-pong: the last pass writes the bins; others alternate x / tmp buffers
            uint32_t* out_r = (l == L - 1) ? bins : ((l & 1) == 0 ? x_recs : tmp_recs);
            uint32_t* out_i = (l == L - 1) ? nullptr : ((l & 1) == 0 ? x_ids : tmp_sig);
            CK(launch_rec_scatter(k, in_r, in_i, l == 0 ? pa.sig2bin : nullptr, d_tiles, mt, t_prefix + nbp, shift,
                                  D[l], cursor, out_r, out_i, s));
            // the pass reads from in_* while writing out_*: tmp is only an output from pass 2 on
            in_r = out_r;
            in_i = out_i;
            s5_launches += 5;
        }
        ar.release(x_recs);
        ar.release(x_ids);
    } else {
        if (!c.run_p1) {
            set_err("the record stream overflowed its capacity (%llu > %llu slots)", (unsigned long long)tmp_n,
                    (unsigned long long)tmp_cap);
            throw Fail{KMC_ERR_INTERNAL};
        }
        uint32_t* bin_fill = ar.get<uint32_t>(n_bins);
        CK(cudaMemsetAsync(bin_fill, 0, n_bins * 4, s));
        c.a.sig2bin = pa.sig2bin;
        c.a.bin_rec_off = pa.bin_rec_off;
        c.a.bin_fill = bin_fill;
        c.a.bins = bins;
        s5_launches = c.run_p1(P1_MODE_SCATTER);
    }
    j->launches += s5_launches;
    j->stage_end(s5_launches);
    ar.release(tmp_recs);
    ar.release(tmp_sig);
    release_plan_scratch(j, c);

    // the per-bin tables were copied to the host while S5 runs on the device
    fetch_tables(j, c);
    count_bins(j, c, bins, 0, n_bins);
    presplit_release(j, c.pre);
    ar.release(bins);
}

// Frees the histograms and the plan's scans (the per-bin tables stay).
void release_plan_scratch(kmc_job* j, PlanCtx& c) {
    Arena& ar = j->arena;
    PlanArgs& pa = c.pa;
    ar.release(c.hist_w);
    ar.release(c.hist_r);
    ar.release(pa.cost_scan);
    ar.release(pa.bnd_scan);
    ar.release(pa.win_scan);
    ar.release(pa.rec_scan);
    ar.release(pa.bin_first);
    ar.release(pa.temp);
}

// Inputs beyond HBM (f2; host-resident reads): pass 1 has built only the histogram; the bins
// are cut into consecutive ranges whose records (and their counting) fit the device budget,
// and for every range the reads are streamed through pass 1 again, which now writes the
// records of the range's bins straight into them (P1_MODE_SCATTER with a bin filter), then
// the range is counted (S6-S8) into the growing survivor buffer; S9 orders all survivors.
void count_multipass(kmc_job* j, PlanCtx& c) {
    const int RW = record_words(j->k);
    Arena& ar = j->arena;
    cudaStream_t s = j->s;
    PlanArgs& pa = c.pa;
    release_plan_scratch(j, c);
    fetch_tables(j, c);
    const HostTable& bn = c.bn;
    const HostTable& bo = c.bo;
    const uint64_t n_bins = c.n_bins;
    // records per pass: the option, else a share of the free device memory (bins 16-32 B,
    // survivors up to 12-20 B per window / ci, the large-bin key regions are grouped anyway)
    uint64_t budget;
    if (j->opt.pass_mb) {
        budget = std::max<uint64_t>(1, ((uint64_t)j->opt.pass_mb << 20) / (RW * 4));
    } else {
        // per record of a pass: the record, the survivor room of its windows (count >= ci)
        // and about 10 bytes per window of large-bin key regions (the split groups bins by
        // the memory left, so this only sizes the pass); memory = free + this process's cache
        size_t fr = 0, tot = 0;
        CK(cudaMemGetInfo(&fr, &tot));
        const double wpr = c.n_records ? (double)c.n_windows / (double)c.n_records : 10.0;
        const double per = RW * 4 + wpr * ((j->key_words == 1 ? 12.0 : 20.0) / j->ci + 10.0);
        budget = std::max<uint64_t>(1u << 20, (uint64_t)(0.6 * (double)(fr + cache_bytes()) / per));
    }
    std::vector<std::pair<uint64_t, uint64_t>> passes;
    for (uint64_t b0 = 0; b0 < n_bins;) {
        uint64_t b1 = b0, recs = 0;
        while (b1 < n_bins && (b1 == b0 || recs + bn[b1] <= budget)) recs += bn[b1++];
        passes.push_back({b0, b1});
        b0 = b1;
    }
    j->st.n_passes = passes.size();
    uint32_t* bin_fill = ar.get<uint32_t>(n_bins);
    for (const auto& ps : passes) {
        const uint64_t b0 = ps.first, b1 = ps.second;
        const uint64_t r0 = bo[b0], r1 = b1 < n_bins ? bo[b1] : c.n_records;
        if (r1 == r0) continue;
        uint32_t* buf = reinterpret_cast<uint32_t*>(ar.alloc((r1 - r0) * RW * 4 + 64));
        // the kernels address records by their global record index: a base pointer r0
        // records before the buffer makes [r0, r1) land in it
        uint32_t* bins_v = buf - r0 * RW;
        CK(cudaMemsetAsync(bin_fill, 0, n_bins * 4, s));
        c.a.sig2bin = pa.sig2bin;
        c.a.bin_rec_off = pa.bin_rec_off;
        c.a.bin_fill = bin_fill;
        c.a.bins = bins_v;
        c.a.bin_lo = (uint32_t)b0;
        c.a.bin_hi = (uint32_t)b1;
        j->stage_begin(KMC_STAGE_SCATTER);
        const int nl = c.run_p1(P1_MODE_SCATTER);
        j->launches += nl;
        j->stage_end(nl);
        count_bins(j, c, bins_v, b0, b1);
        ar.release(buf);
    }
    ar.release(bin_fill);
}

// S6-S8 of the bins [b_lo, b_hi) (records in `bins`, addressed by global record index) into
// the survivor buffer, grown to hold every survivor possible so far.
void count_bins(kmc_job* j, PlanCtx& c, uint32_t* bins, uint64_t b_lo, uint64_t b_hi) {
    htrace("count_bins");
    const int k = j->k, kw = j->key_words;
    const size_t ksz = kw == 1 ? 8 : 16;
    Arena& ar = j->arena;
    cudaStream_t s = j->s;
    const int cap = c.cap;
    PlanArgs& pa = c.pa;
    unsigned long long* hs = j->host_small;
    unsigned long long* gstats = c.gstats;
    const HostTable& bw = c.bw;
    const HostTable& bn = c.bn;
    const HostTable& bo = c.bo;
    // ---- host: classify bins (small: one CTA in SMEM; large: multi-CTA path)
    std::vector<uint32_t> small;
    std::vector<uint64_t> large_ids;
    small.reserve(b_hi - b_lo);
    large_ids.reserve(b_hi - b_lo);
    uint64_t large_windows = 0, n_large = 0, max_bin = 0, range_windows = 0;
    for (uint64_t b = b_lo; b < b_hi; ++b) {
        if (bw[b] == 0) continue;
        range_windows += bw[b];
        max_bin = std::max(max_bin, bw[b]);
        const uint64_t cost = std::max<uint64_t>(bw[b], bn[b] * pa.recw);
        if (cost <= (uint64_t)cap && !j->opt.force_large) {
            small.push_back((uint32_t)b);
        } else {
            ++n_large;
            large_windows += bw[b];
            large_ids.push_back(b);
        }
    }
    htrace("classified");
    {  // small bins by windows, largest first (ties by bin id): a counting sort, windows <= cap
        uint64_t wmax = 0;
        for (uint32_t b : small) wmax = std::max(wmax, bw[b]);
        std::vector<uint32_t> start(wmax + 2, 0), sorted(small.size());
        for (uint32_t b : small) ++start[wmax - bw[b] + 1];
        for (uint64_t v = 1; v <= wmax + 1; ++v) start[v] += start[v - 1];
        for (uint32_t b : small) sorted[start[wmax - bw[b]]++] = b;
        small.swap(sorted);
    }
    htrace("sorted");
    j->st.n_large_bins += n_large;
    j->st.large_windows += large_windows;
    j->st.max_bin_windows = std::max<uint64_t>(j->st.max_bin_windows, max_bin);

    // ---- survivors buffer: every survivor has count >= ci, the range's counts sum to its
    //      windows; grown (the survivors so far copied) when a later range needs more room
    const uint64_t need = j->n_surv + range_windows / j->ci + 1;
    if (need > j->surv_cap) {
        void* nk = ar.alloc(need * ksz);
        uint32_t* nc = ar.get<uint32_t>(need);
        if (j->n_surv) {
            CK(cudaMemcpyAsync(nk, j->surv_keys, j->n_surv * ksz, cudaMemcpyDeviceToDevice, s));
            CK(cudaMemcpyAsync(nc, j->surv_counts, j->n_surv * 4, cudaMemcpyDeviceToDevice, s));
        }
        ar.release(j->surv_keys);
        ar.release(j->surv_counts);
        j->surv_keys = nk;
        j->surv_counts = nc;
        j->surv_cap = need;
    }
    const uint64_t surv_cap = j->surv_cap;

    // ---- S6-S8 small bins
    // The hash path sizes its chunks by the distinct/window ratio of the small bins.  With
    // enough small windows, every 8th small bin runs first as the sample; its distinct-key
    // count is read back while the other small bins run, so the host's large-bin setup
    // overlaps them instead of waiting for all small bins.
    uint64_t small_w = 0, sample_w = 0;
    for (uint32_t b : small) small_w += bw[b];
    size_t n_first = small.size();
    cudaEvent_t ev_sample = nullptr;
    struct EvGuard {
        cudaEvent_t& e;
        ~EvGuard() {
            if (e) cudaEventDestroy(e);
        }
    } ev_sample_guard{ev_sample};
    const bool hash_path = large_windows > 0 && j->opt.large_path != 1 && j->opt.count_path != 1;
    if (hash_path && small_w >= (8u << 20)) {
        std::vector<uint32_t> first, rest;
        for (size_t i = 0; i < small.size(); ++i) (i % 8 == 0 ? first : rest).push_back(small[i]);
        for (uint32_t b : first) sample_w += bw[b];
        n_first = first.size();
        small = first;
        small.insert(small.end(), rest.begin(), rest.end());
    }
    if (!small.empty()) {
        uint32_t* d_small = ar.get<uint32_t>(small.size());
        CK(cudaMemcpyAsync(d_small, small.data(), small.size() * 4, cudaMemcpyHostToDevice, s));
        SmallArgs sa{};
        sa.bins = bins;
        sa.small_list = d_small;
        sa.bin_rec_off = pa.bin_rec_off;
        sa.bin_nrec = pa.bin_nrec;
        sa.bin_w = pa.bin_w;
        sa.k = k;
        sa.canonical = !j->opt.non_canonical;
        sa.ci = j->ci;
        sa.cx = j->cx;
        sa.surv_keys = j->surv_keys;
        sa.surv_counts = j->surv_counts;
        sa.gstats = gstats;
        j->stage_begin(KMC_STAGE_SMALL_BINS);
        // (k,x)-mers (kx > 0): the paper's sorter on every small bin (k_kxmer.cu)
        auto small_launch = [&](uint64_t n) {
            return j->opt.kx ? launch_small_kx(sa, n, (int)j->opt.kx, s) : launch_small_bins(sa, n, s);
        };
        CK(small_launch(n_first));
        int sl = 1;
        if (n_first < small.size()) {
            CK(cudaMemcpyAsync(&hs[64], gstats + GS_UNIQUE, 8, cudaMemcpyDeviceToHost, s));
            CK(cudaEventCreateWithFlags(&ev_sample, cudaEventDisableTiming));
            CK(cudaEventRecord(ev_sample, s));
            sa.small_list = d_small + n_first;
            CK(small_launch(small.size() - n_first));
            ++sl;
        }
        j->launches += sl;
        j->stage_end(sl);
    }
    // distinct keys per window, estimated from the sampled small bins (x margin); 1 without a
    // sample (every window distinct: the safe assumption)
    auto distinct_ratio = [&](double margin) -> double {
        double r = 1.0;
        if (ev_sample) {  // distinct keys of the sampled small bins (the rest still run)
            CK(cudaEventSynchronize(ev_sample));
            r = std::min(1.0, std::max(0.05, margin * (double)hs[64] / (double)sample_w));
        } else if (small_w >= (1u << 20)) {
            CK(cudaMemcpyAsync(&hs[16], gstats, GS_N * 8, cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
            r = std::min(1.0, std::max(0.05, margin * (double)hs[16 + GS_UNIQUE] / (double)small_w));
        }
        return r;
    };
    // chunk capacity (keys): the per-chunk radix sort holds small_capacity(k) keys; the hash
    // table holds 3/4 of its slots in DISTINCT keys, so its chunks may carry more keys by the
    // distinct/window ratio measured on the small bins (x1.5 margin; a chunk that still
    // overflows is counted by the fallback)
    auto chunk_cap = [&]() -> int {
        int kcap = small_capacity(k);
        if (j->opt.count_path != 1) {
            const uint64_t safe = (uint64_t)chunk_hash_cap(k) * 3 / 4;
            const double r = distinct_ratio(1.5);
            kcap = (int)std::min<uint64_t>(2ull * chunk_hash_cap(k), std::max<uint64_t>(safe, (uint64_t)(safe / r)));
        }
        if (j->opt.chunk_capacity) kcap = (int)std::min<uint32_t>(j->opt.chunk_capacity, 1u << 24);
        // the per-chunk radix sort holds at most small_capacity(k) keys in shared memory
        if (j->opt.count_path == 1) kcap = std::min(kcap, small_capacity(k));
        return kcap;
    };
    // ---- S6-S8 large bins
    bool large_done = false;
    if (large_windows > 0 && k <= 32 && j->opt.large_path == 3 && j->opt.count_path != 1) {
        // thread-block clusters count every large bin in their CTAs' shared-memory tables
        // (k_cluster.cu): no key spill to HBM, one expansion per window and round
        int C = (int)j->opt.cluster_size;
        if (C == 0) C = cluster_max_active(16) > 0 ? 16 : cluster_max_active(8) > 0 ? 8 : 1;
        if (C != 1 && C != 4 && C != 8 && C != 16) {
            set_err("cluster_size=%d not in {0, 1, 4, 8, 16}", C);
            throw Fail{KMC_ERR_INVALID_ARG};
        }
        if (C > 1 && cluster_max_active(C) < 1) {
            set_err("the device holds no cluster of %d CTAs", C);
            throw Fail{KMC_ERR_INVALID_ARG};
        }
        const double r = distinct_ratio(1.25);
        const double cap = j->opt.table_keys ? (double)j->opt.table_keys : (double)cl_table_slots() * 3 / 4;
        std::vector<ClItem> items;  // cluster items first, then single items
        std::vector<ClItem> singles;
        for (const uint64_t b : large_ids) {
            const double d = (double)bw[b] * r;
            if (C == 1 || d <= cap) {
                singles.push_back(ClItem{bo[b], (uint32_t)bn[b], 0, 1});
            } else {
                const uint64_t R = std::min<uint64_t>(65535, (uint64_t)std::ceil(d / ((double)C * cap)));
                for (uint64_t q = 0; q < R; ++q) items.push_back(ClItem{bo[b], (uint32_t)bn[b], (uint16_t)q, (uint16_t)R});
            }
        }
        auto by_size = [](const ClItem& x, const ClItem& y) {
            return x.nrec > y.nrec || (x.nrec == y.nrec && (x.rec_off < y.rec_off || (x.rec_off == y.rec_off && x.round < y.round)));
        };
        std::sort(items.begin(), items.end(), by_size);
        std::sort(singles.begin(), singles.end(), by_size);
        const uint64_t n_ci = items.size(), n_si = singles.size();
        items.insert(items.end(), singles.begin(), singles.end());
        ClItem* d_items = ar.get<ClItem>(items.size());
        CK(cudaMemcpyAsync(d_items, items.data(), items.size() * sizeof(ClItem), cudaMemcpyHostToDevice, s));
        unsigned long long* ctr = ar.get<unsigned long long>(4);
        CK(cudaMemsetAsync(ctr, 0, 32, s));
        const uint64_t spill_cap =
            j->opt.spill_keys ? (uint64_t)j->opt.spill_keys : std::max<uint64_t>(1u << 20, large_windows / 16);
        uint64_t* spill = ar.get<uint64_t>(spill_cap);
        unsigned long long* gsnap = ar.get<unsigned long long>(GS_N);
        CK(cudaMemcpyAsync(gsnap, gstats, GS_N * 8, cudaMemcpyDeviceToDevice, s));
        int n_ctas = 0;
        j->stage_begin(KMC_STAGE_LARGE_CHUNKS);
        CK(launch_cluster_count(bins, d_items, n_ci, d_items + n_ci, n_si, C, k, !j->opt.non_canonical, j->ci, j->cx,
                                ctr, spill, spill_cap, j->surv_keys, j->surv_counts, gstats, 0, s, &n_ctas));
        j->launches += 1;
        j->stage_end(1);
        CK(cudaMemcpyAsync(&hs[48], ctr, 24, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        const uint64_t n_spill = hs[50];
        j->st.n_cluster_items = n_ci;
        j->st.n_single_items = n_si;
        j->st.n_spilled_keys = n_spill;
        j->st.cluster_size = (uint64_t)C;
        j->st.cluster_ctas = (uint64_t)n_ctas;
        if (n_spill > spill_cap) {
            // the spill list overflowed: forget this pass's counts, take the split path
            CK(cudaMemcpyAsync(gstats, gsnap, GS_N * 8, cudaMemcpyDeviceToDevice, s));
        } else {
            if (n_spill > 0) {
                // keys that found no slot: disjoint from every table's keys (all their copies
                // fail alike), counted by the device radix sort + run pass
                RadixScratch rs{};
                rs.keys_alt = ar.alloc(n_spill * 8);
                rs.tile_hist = ar.get<uint32_t>(radix_status_words(n_spill, 1));
                rs.tile_off = ar.get<uint32_t>(radix_aux_words());
                rs.scan_temp = ar.alloc(radix_scan_temp_bytes(n_spill, 1));
                rs.red = ar.get<unsigned long long>(4);
                rs.red_host = hs + 40;
                void* sorted = nullptr;
                uint32_t* dummy = nullptr;
                int fl = 0;
                j->stage_begin(KMC_STAGE_LARGE_FALLBACK);
                CK(device_radix_sort(1, spill, nullptr, n_spill, 2 * k, rs, s, &sorted, &dummy, &fl));
                CK(launch_rle(1, sorted, n_spill, j->ci, j->cx, j->surv_keys, j->surv_counts, gstats, s));
                j->launches += fl + 1;
                j->stage_end(fl + 1);
                ar.release(rs.keys_alt);
                ar.release(rs.tile_hist);
                ar.release(rs.tile_off);
                ar.release(rs.scan_temp);
            }
            large_done = true;
        }
        ar.release(spill);
        ar.release(d_items);
    }
    if (large_done) {
    } else if (large_windows > 0 && j->opt.large_path == 1) {
        // device-wide LSD radix sort of all large-bin keys together (a bin partitions the
        // k-mer space, so sorting the union sorts every bin); kept for testing
        std::vector<LargeBin> lbins(large_ids.size());
        std::vector<uint64_t> pp(large_ids.size() + 1, 0);
        for (size_t i = 0; i < large_ids.size(); ++i) {
            const uint64_t b = large_ids[i];
            lbins[i] = LargeBin{0, 0, bo[b], 0, (uint32_t)bw[b], 0, (uint32_t)bn[b], 0, 0, 0};
            pp[i + 1] = pp[i] + (bn[b] + PIECE_RECORDS - 1) / PIECE_RECORDS;
        }
        const uint64_t n_pieces = pp.back();
        LargeBin* d_lbins = ar.get<LargeBin>(lbins.size());
        uint64_t* d_pp = ar.get<uint64_t>(pp.size());
        Piece* d_pieces = ar.get<Piece>(n_pieces);
        CK(cudaMemcpyAsync(d_lbins, lbins.data(), lbins.size() * sizeof(LargeBin), cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(d_pp, pp.data(), pp.size() * 8, cudaMemcpyHostToDevice, s));
        void* lkeys = ar.alloc(large_windows * ksz);
        j->stage_begin(KMC_STAGE_LARGE_SPLIT);
        CK(cudaMemsetAsync(gstats + GS_LARGE_KEYS, 0, 8, s));  // this range's key cursor
        CK(launch_make_pieces(d_lbins, d_pp, lbins.size(), PIECE_RECORDS, d_pieces, s));
        CK(launch_large_expand(bins, d_pieces, n_pieces, k, !j->opt.non_canonical, lkeys, gstats, s));
        j->launches += 2;
        j->stage_end(2);
        RadixScratch rs{};
        rs.keys_alt = ar.alloc(large_windows * ksz);
        rs.tile_hist = ar.get<uint32_t>(radix_status_words(large_windows, kw));
        rs.tile_off = ar.get<uint32_t>(radix_aux_words());
        rs.scan_temp = ar.alloc(radix_scan_temp_bytes(large_windows, kw));
        rs.red = ar.get<unsigned long long>(4);
        rs.red_host = hs + 40;
        void* sorted = nullptr;
        uint32_t* dummy = nullptr;
        int sl = 0;
        j->stage_begin(KMC_STAGE_LARGE_FALLBACK);
        CK(device_radix_sort(kw, lkeys, nullptr, large_windows, 2 * k, rs, s, &sorted, &dummy, &sl));
        CK(launch_rle(kw, sorted, large_windows, j->ci, j->cx, j->surv_keys, j->surv_counts, gstats, s));
        j->launches += sl + 1;
        j->stage_end(sl + 1);
        ar.release(lkeys);
        ar.release(rs.keys_alt);
        ar.release(rs.tile_hist);
        ar.release(rs.tile_off);
        ar.release(rs.scan_temp);
    } else if (large_windows > 0 && k >= SS_KMIN && k <= SS_KMAX && j->opt.large_path == 4 &&
               j->opt.count_path != 1) {
        const int kcap = chunk_cap();
        j->st.chunk_capacity = (uint64_t)kcap;
        large_subsplit(j, c, bins, large_ids, kcap);
    } else if (large_windows > 0 && k <= 32 && j->opt.large_path == 0 && j->opt.count_path != 1) {
        const int kcap = chunk_cap();
        j->st.chunk_capacity = (uint64_t)kcap;
        large_split1(j, c, bins, large_ids, kcap, distinct_ratio);
    } else if (large_windows > 0) {
        // hashed split: per large bin, a D-bit digit -> digit ranges in HBM -> chunks <= cap
        // keys.  Large bins are processed in groups whose keys fit the device budget.
        const int kcap = chunk_cap();
        j->st.chunk_capacity = (uint64_t)kcap;
        const int prec = msd_piece_records(k);
        // group budget in keys: the option, else everything at once if the key buffer can be
        // allocated, else half the free device memory
        uint64_t budget = j->opt.large_group_mkeys ? ((uint64_t)j->opt.large_group_mkeys << 20) : ~0ull;
        void* lkeys = nullptr;
        if (!j->opt.large_group_mkeys) {
            lkeys = ar.try_alloc(large_windows * ksz + chunk_key_slack_bytes());
            if (!lkeys) {
                size_t fr = 0, tot = 0;
                CK(cudaMemGetInfo(&fr, &tot));
                budget = std::max<uint64_t>((uint64_t)(fr / 2) / (ksz + 1), 1u << 20);
            }
        }
        // split positions are uint32 key indices within a group
        budget = std::min<uint64_t>(budget, 0xFFFFFFFFull - 64);
        std::vector<std::pair<size_t, size_t>> groups;
        uint64_t max_gw = 0, max_gd = 0, max_gp = 0, max_gn = 0;
        for (size_t i0 = 0; i0 < large_ids.size();) {
            uint64_t gw = 0, gd = 0, gp = 0;
            size_t i1 = i0;
            while (i1 < large_ids.size()) {
                const uint64_t b = large_ids[i1];
                if (i1 > i0 && gw + bw[b] > budget) break;
                gw += bw[b];
                gd += 1ull << msd_digit_bits(bw[b], k, kcap);
                gp += (bn[b] + prec - 1) / prec;
                ++i1;
            }
            groups.push_back({i0, i1});
            max_gw = std::max(max_gw, gw);
            max_gd = std::max(max_gd, gd);
            max_gp = std::max(max_gp, gp);
            max_gn = std::max<uint64_t>(max_gn, i1 - i0);
            i0 = i1;
        }
        j->st.n_large_groups += groups.size();
        // split ranges: one CTA each, a few per SM (the split kernels are ~40 KB of SMEM)
        const uint32_t max_ranges = (uint32_t)n_sms() * 4;
        LargeBin* d_lbins = ar.get<LargeBin>(max_gn);
        uint64_t* d_pp = ar.get<uint64_t>(max_gn + 1);
        Piece* d_pieces = ar.get<Piece>(max_gp);
        uint32_t* digit_cnt = ar.get<uint32_t>(max_gd);
        uint32_t* digit_start = ar.get<uint32_t>(max_gd);
        Chunk* chunks = ar.get<Chunk>(max_gd);
        Chunk* oversize = ar.get<Chunk>(max_gd);
        unsigned long long* counters = ar.get<unsigned long long>(3);
        if (!lkeys) lkeys = ar.alloc(max_gw * ksz + chunk_key_slack_bytes());
        uint32_t* table = nullptr;
        uint32_t* tpos = nullptr;
        void* ttemp = nullptr;
        uint64_t table_cap = 0;
        RadixScratch rs{};
        uint64_t rs_cap = 0;
        int sl = 0;
        for (const auto& g : groups) {
            const size_t gn = g.second - g.first;
            // host tables reused across calls on this thread (fresh MB-sized vectors cost
            // page faults on the critical path between the small-bin and split kernels)
            static thread_local std::vector<LargeBin> lbins;
            static thread_local std::vector<uint64_t> pp;
            lbins.resize(gn);
            pp.assign(gn + 1, 0);
            uint64_t key_base = 0, digit_base = 0;
            int dmax = 1;
            for (size_t i = 0; i < gn; ++i) {
                const uint64_t b = large_ids[g.first + i];
                const int D = msd_digit_bits(bw[b], k, kcap);
                dmax = std::max(dmax, D);
                lbins[i] = LargeBin{key_base, digit_base, bo[b], 0, (uint32_t)bw[b], (uint32_t)D, (uint32_t)bn[b], 0, 0, 0};
                key_base += bw[b];
                digit_base += 1ull << D;
                pp[i + 1] = pp[i] + (bn[b] + prec - 1) / prec;
            }
            const uint64_t n_pieces = pp.back();
            // ranges r = pieces [r*n/R, (r+1)*n/R); segments = (range, bin) pairs
            const uint32_t R = (uint32_t)std::min<uint64_t>(n_pieces, max_ranges);
            auto range_of = [&](uint64_t piece) {
                uint64_t r = piece * R / n_pieces;
                while (r + 1 < R && (r + 1) * n_pieces / R <= piece) ++r;
                while (r > 0 && r * n_pieces / R > piece) --r;
                return (uint32_t)r;
            };
            // segments: single pieces for bins in piece mode (staged coalesced scatter) while
            // the table stays small, else (range, bin) pairs
            uint64_t tb = 0;
            const int pm_dmax = split_piece_mode_dmax(k);
            for (size_t i = 0; i < gn; ++i) {
                const uint64_t np_b = pp[i + 1] - pp[i];
                const bool pm = (int)lbins[i].D <= pm_dmax && tb + (np_b << lbins[i].D) <= (1ull << 26);
                if (pm) {
                    lbins[i].first_range = (uint32_t)pp[i];
                    lbins[i].nseg = (uint32_t)np_b;
                    lbins[i].pad = 1;
                } else {
                    const uint32_t f = range_of(pp[i]), l = range_of(pp[i + 1] - 1);
                    lbins[i].first_range = f;
                    lbins[i].nseg = l - f + 1;
                }
                lbins[i].tb = tb;
                tb += (uint64_t)lbins[i].nseg << lbins[i].D;
            }
            if (tb + 1 > table_cap) {
                ar.release(table);
                ar.release(tpos);
                ar.release(ttemp);
                table_cap = tb + 1;
                table = ar.get<uint32_t>(table_cap);
                tpos = ar.get<uint32_t>(table_cap);
                ttemp = ar.alloc(scan_temp_bytes(table_cap));
            }
            CK(cudaMemcpyAsync(d_lbins, lbins.data(), gn * sizeof(LargeBin), cudaMemcpyHostToDevice, s));
            CK(cudaMemcpyAsync(d_pp, pp.data(), pp.size() * 8, cudaMemcpyHostToDevice, s));
            j->stage_begin(KMC_STAGE_LARGE_SPLIT);
            CK(cudaMemsetAsync(counters, 0, 24, s));
            CK(launch_make_pieces(d_lbins, d_pp, gn, (uint32_t)prec, d_pieces, s));
            CK(launch_split(false, bins, d_pieces, n_pieces, d_lbins, k, !j->opt.non_canonical, dmax, R, table, nullptr, s));
            CK(scan_u32_to_u32(table, tpos, tb, ttemp, s));
            CK(launch_digit_totals(d_lbins, gn, tpos, digit_cnt, digit_start, s));
            GreedyArgs ga{};
            ga.cnt = digit_cnt;
            ga.gstart = digit_start;
            ga.n_digits = digit_base;
            ga.chunks = chunks;
            ga.oversize = oversize;
            ga.counters = counters;
            ga.cap = (uint32_t)kcap;
            CK(launch_greedy_chunks(ga, key_base, s));
            j->launches += 6;
            j->stage_end(6);
            j->stage_begin(KMC_STAGE_LARGE_SCATTER);
            CK(launch_split(true, bins, d_pieces, n_pieces, d_lbins, k, !j->opt.non_canonical, dmax, R, tpos, lkeys, s));
            j->launches += 1;
            j->stage_end(1);
            CK(cudaMemcpyAsync(&hs[48], counters, 16, cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
            const uint64_t n_chunks = hs[48], n_over = hs[49];
            j->stage_begin(KMC_STAGE_LARGE_CHUNKS);
            if (j->opt.count_path == 1)
                CK(launch_chunk_sort(lkeys, chunks, n_chunks, k, j->ci, j->cx, j->surv_keys, j->surv_counts, gstats,
                                     s));
            else
                CK(launch_chunk_hash(lkeys, chunks, n_chunks, k, j->ci, j->cx, j->surv_keys, j->surv_counts, gstats,
                                     oversize + n_over, counters + 2, n_sms(), s));
            j->launches += 1;
            j->stage_end(1);
            uint64_t n_ovf = 0;
            if (j->opt.count_path != 1) {
                CK(cudaMemcpyAsync(&hs[50], counters + 2, 8, cudaMemcpyDeviceToHost, s));
                CK(cudaStreamSynchronize(s));
                n_ovf = hs[50];
                j->st.n_overflow_chunks += n_ovf;
            }
            if (n_over + n_ovf > 0) {
                // digits above the chunk capacity (identical-key pile-ups) and chunks whose
                // distinct keys overflowed the hash table: device LSD + run pass
                std::vector<Chunk> ov(n_over + n_ovf);
                CK(cudaMemcpyAsync(ov.data(), oversize, ov.size() * sizeof(Chunk), cudaMemcpyDeviceToHost, s));
                CK(cudaStreamSynchronize(s));
                uint64_t maxn = 0;
                for (auto& c : ov) maxn = std::max<uint64_t>(maxn, c.n);
                if (maxn > rs_cap) {
                    ar.release(rs.keys_alt);
                    ar.release(rs.tile_hist);
                    ar.release(rs.tile_off);
                    ar.release(rs.scan_temp);
                    rs.keys_alt = ar.alloc(maxn * ksz);
                    rs.tile_hist = ar.get<uint32_t>(radix_status_words(maxn, kw));
                    rs.tile_off = ar.get<uint32_t>(radix_aux_words());
                    rs.scan_temp = ar.alloc(radix_scan_temp_bytes(maxn, kw));
                    if (!rs.red) rs.red = ar.get<unsigned long long>(4);
                    rs.red_host = hs + 40;
                    rs_cap = maxn;
                }
                int fl = 0;
                j->stage_begin(KMC_STAGE_LARGE_FALLBACK);
                for (auto& c : ov) {
                    void* seg = (uint8_t*)lkeys + c.begin * ksz;
                    void* sorted = nullptr;
                    uint32_t* dummy = nullptr;
                    CK(device_radix_sort(kw, seg, nullptr, c.n, 2 * k, rs, s, &sorted, &dummy, &fl));
                    CK(launch_rle(kw, sorted, c.n, j->ci, j->cx, j->surv_keys, j->surv_counts, gstats, s));
                    fl += 1;
                }
                sl += fl;
                j->launches += fl;
                j->stage_end(fl);
            }
        }
        ar.release(lkeys);
        hs[16 + GS_LARGE_KEYS] = large_windows;  // the split writes exactly the planned keys
    }
    CK(cudaMemcpyAsync(&hs[16], gstats, GS_N * 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    j->n_surv = hs[16 + GS_SURV];
    j->st.n_unique = hs[16 + GS_UNIQUE];
    j->st.n_below_min = hs[16 + GS_BELOW];
    j->st.n_above_max = hs[16 + GS_ABOVE];
    j->st.n_small_sorted = hs[16 + GS_SMALL_SORTED];
    j->st.n_kxmers = hs[16 + GS_KX];
    j->st.kx_windows = hs[16 + GS_KX_WIN];
    j->st.n_overflow_chunks += hs[16 + GS_SUB_OVF];
    if (j->opt.large_path == 1 && hs[16 + GS_LARGE_KEYS] != large_windows) {
        set_err("large-bin expansion produced %llu keys, plan says %llu", (unsigned long long)hs[16 + GS_LARGE_KEYS],
                (unsigned long long)large_windows);
        throw Fail{KMC_ERR_INTERNAL};
    }
    if (j->n_surv > surv_cap) {
        set_err("survivor overflow");
        throw Fail{KMC_ERR_INTERNAL};
    }
}

void run_finish(kmc_job* j, uint64_t* out_kmers, uint32_t* out_counts) {
    htrace("finish");
    const int kw = j->key_words;
    const size_t ksz = kw == 1 ? 8 : 16;
    Arena& ar = j->arena;
    cudaStream_t s = j->s;
    const uint64_t n = j->n_surv;
    if (n == 0) return;
    // ---- S9: global ascending order, written straight into device outputs
    const bool dev_out = is_device_ptr(out_kmers) && is_device_ptr(out_counts);
    void* ok = dev_out ? (void*)out_kmers : ar.alloc(n * ksz);
    uint32_t* oc = dev_out ? out_counts : ar.get<uint32_t>(n);
    const uint64_t nd = 1ull << order_digit_bits(n, j->k);
    OrderScratch os{};
    os.hist = ar.get<uint32_t>(nd);
    os.start = ar.get<uint32_t>(nd + 1);
    os.cursor = ar.get<uint32_t>(nd);
    os.chunks = ar.get<Chunk>(nd);
    os.oversize = ar.get<Chunk>(nd);
    os.counters = ar.get<unsigned long long>(80);
    os.tiles = ar.get<OrdTile>(order_max_tiles(n, j->k));
    os.tprefix = ar.get<uint64_t>(order_prev_buckets(n, j->k) + 1);
    os.ttemp = ar.alloc(scan_temp_bytes(order_prev_buckets(n, j->k) + 1));
    os.tmp_keys = ar.alloc(n * ksz);
    os.tmp_vals = ar.get<uint32_t>(n);
    os.scan_temp = ar.alloc(order_scan_temp_bytes(nd + 1));
    os.host = j->host_small + 56;
    os.start0 = ar.get<uint32_t>(257);
    std::vector<OrderSegment> over;
    int sl = 0;
    j->stage_begin(KMC_STAGE_ORDER);
    void* seg_k = nullptr;
    uint32_t* seg_v = nullptr;
    // host outputs in pinned memory: every group of S9's final sorts is copied out on the copy
    // stream while the next group is sorted (groups holding an oversize bucket after its sort)
    const bool overlap = !dev_out && is_pinned_host(out_kmers) && is_pinned_host(out_counts) && kw == 1;
    std::vector<std::pair<uint64_t, uint64_t>> later;
    std::vector<cudaEvent_t> gev;
    OrderRangeFn range_done = [&](uint64_t lo, uint64_t hi, bool final) {
        if (hi <= lo) return;
        if (!final) {
            later.push_back({lo, hi});
            return;
        }
        cudaEvent_t ev = nullptr;
        CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        gev.push_back(ev);
        CK(cudaEventRecord(ev, s));
        CK(cudaStreamWaitEvent(j->cs, ev, 0));
        CK(cudaMemcpyAsync((uint8_t*)out_kmers + lo * ksz, (uint8_t*)ok + lo * ksz, (hi - lo) * ksz,
                           cudaMemcpyDeviceToHost, j->cs));
        CK(cudaMemcpyAsync(out_counts + lo, oc + lo, (hi - lo) * 4, cudaMemcpyDeviceToHost, j->cs));
    };
    if (overlap) j->make_copy_stream();
    htrace("order launch");
    CK(launch_order(kw, j->surv_keys, j->surv_counts, n, j->k, ok, oc, os, s, &sl, &over, &seg_k, &seg_v,
                    overlap ? &range_done : nullptr));
    htrace("order enqueued");
    if (!over.empty()) {
        // oversize buckets (more survivors than one chunk): gathered into one array, sorted
        // together by the device LSD (they are disjoint, ascending key ranges, so the sorted
        // concatenation is every bucket sorted, in bucket order), written to their places
        uint64_t tot = 0;
        for (auto& g : over) tot += g.n;
        j->st.n_order_oversize = tot;
        void* gk = ar.alloc(tot * ksz);
        uint32_t* gv = ar.get<uint32_t>(tot);
        uint64_t o = 0;
        for (auto& g : over) {
            CK(cudaMemcpyAsync((uint8_t*)gk + o * ksz, (uint8_t*)seg_k + g.begin * ksz, g.n * ksz,
                               cudaMemcpyDeviceToDevice, s));
            CK(cudaMemcpyAsync(gv + o, seg_v + g.begin, g.n * 4, cudaMemcpyDeviceToDevice, s));
            o += g.n;
        }
        RadixScratch rs{};
        rs.keys_alt = ar.alloc(tot * ksz);
        rs.vals_alt = ar.get<uint32_t>(tot);
        rs.tile_hist = ar.get<uint32_t>(radix_status_words(tot, kw));
        rs.tile_off = ar.get<uint32_t>(radix_aux_words());
        rs.scan_temp = ar.alloc(radix_scan_temp_bytes(tot, kw));
        rs.red = ar.get<unsigned long long>(4);
        rs.red_host = j->host_small + 40;
        void* rk = nullptr;
        uint32_t* rv = nullptr;
        CK(device_radix_sort(kw, gk, gv, tot, 2 * j->k, rs, s, &rk, &rv, &sl));
        o = 0;
        for (auto& g : over) {
            CK(cudaMemcpyAsync((uint8_t*)ok + g.begin * ksz, (uint8_t*)rk + o * ksz, g.n * ksz, cudaMemcpyDeviceToDevice,
                               s));
            CK(cudaMemcpyAsync(oc + g.begin, rv + o, g.n * 4, cudaMemcpyDeviceToDevice, s));
            o += g.n;
        }
    }
    j->launches += sl;
    j->stage_end(sl);
    if (overlap) {
        // (the stage covers what is left of the copies once the sorts are done)
        j->stage_begin(KMC_STAGE_OUTPUT);
        for (auto& r : later) {
            CK(cudaMemcpyAsync((uint8_t*)out_kmers + r.first * ksz, (uint8_t*)ok + r.first * ksz,
                               (r.second - r.first) * ksz, cudaMemcpyDeviceToHost, s));
            CK(cudaMemcpyAsync(out_counts + r.first, oc + r.first, (r.second - r.first) * 4, cudaMemcpyDeviceToHost, s));
        }
        cudaEvent_t done = nullptr;
        CK(cudaEventCreateWithFlags(&done, cudaEventDisableTiming));
        CK(cudaEventRecord(done, j->cs));
        CK(cudaStreamWaitEvent(s, done, 0));  // the call's stream covers every copy
        j->stage_end(0);
        cudaEventDestroy(done);
        for (cudaEvent_t e : gev) cudaEventDestroy(e);
    } else if (!dev_out) {
        j->stage_begin(KMC_STAGE_OUTPUT);
        CK(cudaMemcpyAsync(out_kmers, ok, n * ksz, cudaMemcpyDefault, s));
        CK(cudaMemcpyAsync(out_counts, oc, n * 4, cudaMemcpyDefault, s));
        j->stage_end(0);
    }
}

}  // namespace

extern "C" {

void kmc_set_allocator(kmc_alloc_fn alloc_fn, kmc_free_fn free_fn, void* ctx) {
    std::lock_guard<std::mutex> g(g_alloc_mu);
    if (alloc_fn && free_fn) {
        g_alloc = alloc_fn;
        g_free = free_fn;
        g_ctx = ctx;
    } else {
        g_alloc = nullptr;
        g_free = nullptr;
        g_ctx = nullptr;
    }
}

void kmc_empty_cache(void) {
    std::lock_guard<std::mutex> g(g_cache_mu);
    cache_flush_locked();
}

const char* kmc_last_error(void) { return g_err.c_str(); }
int kmc_version(void) { return KMCGPU_VERSION; }

kmc_status kmc_count_begin(const uint8_t* reads, const uint64_t* read_offsets, uint64_t n_reads, int k, int p,
                           uint32_t cutoff_min, uint32_t cutoff_max, void* stream, const kmc_options* opt,
                           kmc_job** job, uint64_t* n_out) {
    if (!job || !n_out) {
        set_err("job and n_out must be non-NULL");
        return KMC_ERR_INVALID_ARG;
    }
    *job = nullptr;
    *n_out = 0;
    kmc_status v = validate(k, p, cutoff_min, cutoff_max);
    if (v != KMC_OK) return v;
    if (n_reads > 0 && (!reads || !read_offsets)) {
        set_err("reads and read_offsets must be non-NULL when n_reads > 0");
        return KMC_ERR_INVALID_ARG;
    }
    kmc_job* j = new kmc_job();
    j->s = (cudaStream_t)stream;
    j->k = k;
    j->p = p;
    j->key_words = k <= 32 ? 1 : 2;
    j->ci = cutoff_min ? cutoff_min : 1;
    j->cx = cutoff_max;
    if (opt) j->opt = *opt;
    if (j->opt.non_canonical && (k == 32 || k == 64)) {
        // the all-T k-mer is the all-ones key, the empty-slot / padding marker (never a
        // canonical key, but a forward one)
        set_err("non_canonical needs k != 32 and k != 64 (k=%d)", k);
        delete j;
        return KMC_ERR_INVALID_ARG;
    }
    if (j->opt.kx && (j->opt.kx > 3 || k + (int)j->opt.kx > 31 || j->opt.non_canonical)) {
        set_err("kx=%u needs kx <= 3, k + kx <= 31 and canonical counting (k=%d)", j->opt.kx, k);
        delete j;
        return KMC_ERR_INVALID_ARG;
    }
    j->arena.bind(j->s);
    try {
        // Calls from several host threads of one process run S1-S8 one after another: two
        // overlapping calls hit an illegal address in a race not yet found (one
        // process per stream of calls is fine).  S9 and the output copy still overlap.
        std::lock_guard<std::mutex> g(g_begin_mu);
        run_begin(j, reads, read_offsets, n_reads);
    } catch (const Fail& f) {
        cudaStreamSynchronize(j->s);
        delete j;
        return f.st;
    }
    *n_out = j->n_surv;
    *job = j;
    return KMC_OK;
}

kmc_status kmc_count_finish(kmc_job* j, uint64_t* out_kmers, uint32_t* out_counts, uint64_t out_capacity,
                            kmc_stats* stats) {
    if (!j) {
        set_err("NULL job");
        return KMC_ERR_INVALID_ARG;
    }
    kmc_status st = KMC_OK;
    if (out_capacity < j->n_surv) {
        set_err("out_capacity=%llu < n_out=%llu", (unsigned long long)out_capacity, (unsigned long long)j->n_surv);
        st = KMC_ERR_OUT_CAPACITY;
    } else if (j->n_surv > 0 && (!out_kmers || !out_counts)) {
        set_err("NULL output buffers");
        st = KMC_ERR_INVALID_ARG;
    } else {
        try {
            run_finish(j, out_kmers, out_counts);
            CK(cudaStreamSynchronize(j->s));
        } catch (const Fail& f) {
            st = f.st;
        }
    }
    cudaStreamSynchronize(j->s);
    j->collect_profile();
    j->st.n_out = j->n_surv;
    j->st.n_launches = (uint64_t)j->launches;
    if (stats) *stats = j->st;
    delete j;
    return st;
}

void kmc_job_free(kmc_job* j) {
    if (!j) return;
    cudaStreamSynchronize(j->s);
    delete j;
}

kmc_status kmc_count_ex(const uint8_t* reads, const uint64_t* read_offsets, uint64_t n_reads, int k, int p,
                        uint32_t cutoff_min, uint32_t cutoff_max, uint64_t* out_kmers, uint32_t* out_counts,
                        uint64_t out_capacity, kmc_stats* stats, void* stream, const kmc_options* opt) {
    kmc_job* j = nullptr;
    uint64_t n = 0;
    kmc_status st = kmc_count_begin(reads, read_offsets, n_reads, k, p, cutoff_min, cutoff_max, stream, opt, &j, &n);
    if (st != KMC_OK) return st;
    return kmc_count_finish(j, out_kmers, out_counts, out_capacity, stats);
}

kmc_status kmc_count(const uint8_t* reads, const uint64_t* read_offsets, uint64_t n_reads, int k, int p,
                     uint32_t cutoff_min, uint32_t cutoff_max, uint64_t* out_kmers, uint32_t* out_counts,
                     uint64_t out_capacity, kmc_stats* stats, void* stream) {
    return kmc_count_ex(reads, read_offsets, n_reads, k, p, cutoff_min, cutoff_max, out_kmers, out_counts,
                        out_capacity, stats, stream, nullptr);
}

// ---------------------------------------------------------------- sharded counting
void kmc_shard_owners(const uint64_t* bin_windows, uint64_t n_bins, int world, uint32_t* owner) {
    uint64_t total = 0;
    for (uint64_t b = 0; b < n_bins; ++b) total += bin_windows[b];
    uint64_t pre = 0;
    for (uint64_t b = 0; b < n_bins; ++b) {
        // contiguous ranges of bins, balanced by windows: the rank whose share holds the bin's midpoint
        const unsigned __int128 mid2 = (unsigned __int128)(2 * pre + bin_windows[b]) * (unsigned)world;
        uint64_t r = total ? (uint64_t)(mid2 / (2 * (unsigned __int128)total)) : 0;
        owner[b] = (uint32_t)std::min<uint64_t>(r, (uint64_t)world - 1);
        pre += bin_windows[b];
    }
}

kmc_status kmc_shard_pass1(const uint8_t* reads, const uint64_t* read_offsets, uint64_t n_reads, int k, int p,
                           uint32_t cutoff_min, uint32_t cutoff_max, void* stream, const kmc_options* opt,
                           kmc_job** job, uint64_t* hist_w, uint64_t* hist_r, uint64_t* n_records) {
    if (!job || !hist_w || !hist_r || !n_records) {
        set_err("job, hist_w, hist_r and n_records must be non-NULL");
        return KMC_ERR_INVALID_ARG;
    }
    *job = nullptr;
    *n_records = 0;
    kmc_status v = validate(k, p, cutoff_min, cutoff_max);
    if (v != KMC_OK) return v;
    if (n_reads > 0 && (!reads || !read_offsets)) {
        set_err("reads and read_offsets must be non-NULL when n_reads > 0");
        return KMC_ERR_INVALID_ARG;
    }
    kmc_job* j = new kmc_job();
    j->s = (cudaStream_t)stream;
    j->k = k;
    j->p = p;
    j->key_words = k <= 32 ? 1 : 2;
    j->ci = cutoff_min ? cutoff_min : 1;
    j->cx = cutoff_max;
    if (opt) j->opt = *opt;
    if (j->opt.non_canonical && (k == 32 || k == 64)) {
        set_err("non_canonical needs k != 32 and k != 64 (k=%d)", k);
        delete j;
        return KMC_ERR_INVALID_ARG;
    }
    j->shard = true;
    j->arena.bind(j->s);
    try {
        run_begin(j, reads, read_offsets, n_reads);
        PlanCtx& c = j->ctx;
        Arena& ar = j->arena;
        cudaStream_t s = j->s;
        const uint64_t ns = (1ull << (2 * p)) + 1;
        if (!c.hist_w) {  // no window in this slice: empty histograms, empty stream
            c.ns = ns;
            c.hist_w = ar.get<unsigned long long>(ns);
            c.hist_r = ar.get<uint32_t>(ns);
            c.gstats = ar.get<unsigned long long>(GS_N);
            CK(cudaMemsetAsync(c.hist_w, 0, ns * 8, s));
            CK(cudaMemsetAsync(c.hist_r, 0, ns * 4, s));
            CK(cudaMemsetAsync(c.gstats, 0, GS_N * 8, s));
        }
        uint64_t* hr = ar.get<uint64_t>(ns);
        CK(launch_widen(c.hist_r, ns, hr, s));
        CK(cudaMemcpyAsync(hist_w, c.hist_w, ns * 8, cudaMemcpyDefault, s));
        CK(cudaMemcpyAsync(hist_r, hr, ns * 8, cudaMemcpyDefault, s));
        unsigned long long* hs = j->host_small;
        CK(cudaMemcpyAsync(&hs[16], c.gstats, GS_N * 8, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        ar.release(hr);
        c.tmp_n = hs[16 + GS_TMP_RECS];
        if (c.tmp_recs && c.tmp_n > c.tmp_cap) {
            set_err("the record stream overflowed its capacity (%llu > %llu slots)", (unsigned long long)c.tmp_n,
                    (unsigned long long)c.tmp_cap);
            throw Fail{KMC_ERR_INTERNAL};
        }
        j->n_local_records = hs[16 + GS_RECORDS];
    } catch (const Fail& f) {
        cudaStreamSynchronize(j->s);
        delete j;
        return f.st;
    }
    *n_records = j->n_local_records;
    *job = j;
    return KMC_OK;
}

namespace {

// The sharded plan (every rank derives the same one from the global histograms), the bin ->
// rank map and this rank's record count per destination (j->send_counts); j->sig2owner holds
// signature -> rank on the device.
void shard_plan(kmc_job* j, const uint64_t* global_hist_w, const uint64_t* global_hist_r, int world, int rank) {
    PlanCtx& c = j->ctx;
    Arena& ar = j->arena;
    cudaStream_t s = j->s;
    const uint64_t ns = c.ns;
    j->world = world;
    j->rank = rank;
    // the global histograms replace the local ones: every rank derives the same plan
    uint64_t* gr = ar.get<uint64_t>(ns);
    CK(cudaMemcpyAsync(c.hist_w, global_hist_w, ns * 8, cudaMemcpyDefault, s));
    CK(cudaMemcpyAsync(gr, global_hist_r, ns * 8, cudaMemcpyDefault, s));
    CK(launch_narrow(gr, ns, c.hist_r, s));
    c.check_p1 = false;
    plan_phase(j, c);
    fetch_tables(j, c);
    ar.release(gr);
    c.owner.assign(c.n_bins, 0);
    if (c.n_bins) kmc_shard_owners(c.bw.data(), c.n_bins, world, c.owner.data());
    j->send_counts.assign(world, 0);
    if (j->n_local_records == 0) return;
    uint32_t* d_owner = ar.get<uint32_t>(c.n_bins);
    j->sig2owner = ar.get<uint32_t>(ns);
    unsigned long long* counts = ar.get<unsigned long long>(world);
    CK(cudaMemcpyAsync(d_owner, c.owner.data(), c.n_bins * 4, cudaMemcpyHostToDevice, s));
    CK(launch_compose_map(c.pa.sig2bin, d_owner, ns, j->sig2owner, s));
    CK(cudaMemsetAsync(counts, 0, world * 8, s));
    CK(launch_owner_count(c.tmp_sig, c.tmp_n, j->sig2owner, world, counts, s));
    std::vector<unsigned long long> hc(world);
    CK(cudaMemcpyAsync(hc.data(), counts, world * 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    uint64_t o = 0;
    for (int r = 0; r < world; ++r) {
        j->send_counts[r] = hc[r];
        o += hc[r];
    }
    if (o != j->n_local_records) {
        set_err("partitioned %llu records, pass 1 wrote %llu", (unsigned long long)o,
                (unsigned long long)j->n_local_records);
        throw Fail{KMC_ERR_INTERNAL};
    }
    ar.release(d_owner);
    ar.release(counts);
}

// One MSD pass of k_rec_scatter over the record stream with digit = owner rank; every rank's
// run starts at cursor0[rank] of its output.  Plain mode writes into out_recs / out_sigs;
// peer mode (peer_recs != nullptr) into the device array of per-rank base pointers.
void shard_scatter(kmc_job* j, const std::vector<uint64_t>& cursor0, uint32_t* out_recs, uint32_t* out_sigs,
                   uint32_t* const* peer_recs, uint32_t* const* peer_sigs) {
    PlanCtx& c = j->ctx;
    Arena& ar = j->arena;
    cudaStream_t s = j->s;
    const int world = j->world;
    unsigned long long* cursor = ar.get<unsigned long long>(world);
    CK(cudaMemcpyAsync(cursor, cursor0.data(), world * 8, cudaMemcpyHostToDevice, s));
    int D = 1;
    while ((1 << D) < world) ++D;
    const uint64_t TI = rec_tile_items(j->k);
    const uint64_t mt = c.tmp_n / TI + 1;
    RecTile2* d_tiles = ar.get<RecTile2>(mt);
    uint64_t* t_prefix = ar.get<uint64_t>(2);
    void* t_temp = ar.alloc(scan_temp_bytes(2));
    CK(launch_make_tiles(TileSrc{nullptr, 1, 0, 0, c.tmp_n}, 1, (uint32_t)TI, mt, t_prefix, t_temp, d_tiles, s));
    CK(launch_rec_scatter(j->k, c.tmp_recs, c.tmp_sig, j->sig2owner, d_tiles, mt, t_prefix + 1, 0, D, cursor, out_recs,
                          out_sigs, s, 1, peer_recs, peer_sigs));
    j->launches += 7;
    CK(cudaStreamSynchronize(s));
    ar.release(d_tiles);
    ar.release(t_prefix);
    ar.release(t_temp);
    ar.release(cursor);
}

}  // namespace

kmc_status kmc_shard_partition(kmc_job* j, const uint64_t* global_hist_w, const uint64_t* global_hist_r, int world,
                               int rank, uint32_t* send_records, uint32_t* send_sigs, uint64_t* send_counts) {
    if (!j || !j->shard || !global_hist_w || !global_hist_r || !send_counts || world < 1 || world > 256 || rank < 0 ||
        rank >= world) {
        set_err("invalid kmc_shard_partition arguments");
        return KMC_ERR_INVALID_ARG;
    }
    if (j->n_local_records > 0 && (!send_records || !send_sigs)) {
        set_err("NULL send buffers");
        return KMC_ERR_INVALID_ARG;
    }
    try {
        shard_plan(j, global_hist_w, global_hist_r, world, rank);
        std::vector<uint64_t> cur(world, 0);
        uint64_t o = 0;
        for (int r = 0; r < world; ++r) {
            send_counts[r] = j->send_counts[r];
            cur[r] = o;
            o += j->send_counts[r];
        }
        if (j->n_local_records > 0) shard_scatter(j, cur, send_records, send_sigs, nullptr, nullptr);
    } catch (const Fail& f) {
        return f.st;
    }
    return KMC_OK;
}

kmc_status kmc_shard_plan(kmc_job* j, const uint64_t* global_hist_w, const uint64_t* global_hist_r, int world,
                          int rank, uint64_t* send_counts) {
    if (!j || !j->shard || !global_hist_w || !global_hist_r || !send_counts || world < 1 || world > 256 || rank < 0 ||
        rank >= world) {
        set_err("invalid kmc_shard_plan arguments");
        return KMC_ERR_INVALID_ARG;
    }
    try {
        shard_plan(j, global_hist_w, global_hist_r, world, rank);
        for (int r = 0; r < world; ++r) send_counts[r] = j->send_counts[r];
    } catch (const Fail& f) {
        return f.st;
    }
    return KMC_OK;
}

kmc_status kmc_shard_recv_alloc(kmc_job* j, uint64_t n_recv, uint8_t* handles) {
    if (!j || !j->shard || !handles || j->recv_recs) {
        set_err("invalid kmc_shard_recv_alloc arguments");
        return KMC_ERR_INVALID_ARG;
    }
    try {
        const int RW = record_words(j->k);
        // at least one record each, so that every rank has a mappable allocation
        const uint64_t n = n_recv > 0 ? n_recv : 1;
        CK(cudaMalloc(&j->recv_recs, n * RW * 4));
        CK(cudaMalloc(&j->recv_sigs, n * 4));
        j->n_recv = n_recv;
        cudaIpcMemHandle_t h[2];
        CK(cudaIpcGetMemHandle(&h[0], j->recv_recs));
        CK(cudaIpcGetMemHandle(&h[1], j->recv_sigs));
        static_assert(sizeof(cudaIpcMemHandle_t) == 64, "64-byte IPC handles");
        memcpy(handles, h, 128);
    } catch (const Fail& f) {
        return f.st;
    }
    return KMC_OK;
}

kmc_status kmc_shard_send_peers(kmc_job* j, const uint8_t* all_handles, const uint64_t* dst_offsets) {
    if (!j || !j->shard || !all_handles || !dst_offsets || !j->recv_recs || j->world < 1) {
        set_err("invalid kmc_shard_send_peers arguments (kmc_shard_plan and kmc_shard_recv_alloc first)");
        return KMC_ERR_INVALID_ARG;
    }
    const int world = j->world;
    std::vector<void*> opened;
    kmc_status st = KMC_OK;
    try {
        std::vector<uint32_t*> pr(world), ps(world);
        for (int r = 0; r < world; ++r) {
            if (r == j->rank) {
                pr[r] = j->recv_recs;
                ps[r] = j->recv_sigs;
                continue;
            }
            cudaIpcMemHandle_t h[2];
            memcpy(h, all_handles + 128 * (size_t)r, 128);
            void* a = nullptr;
            void* b = nullptr;
            CK(cudaIpcOpenMemHandle(&a, h[0], cudaIpcMemLazyEnablePeerAccess));
            opened.push_back(a);
            CK(cudaIpcOpenMemHandle(&b, h[1], cudaIpcMemLazyEnablePeerAccess));
            opened.push_back(b);
            pr[r] = (uint32_t*)a;
            ps[r] = (uint32_t*)b;
        }
        if (j->n_local_records > 0) {
            uint32_t** d_ptrs = j->arena.get<uint32_t*>(2 * world);
            std::vector<uint32_t*> both(pr);
            both.insert(both.end(), ps.begin(), ps.end());
            CK(cudaMemcpyAsync(d_ptrs, both.data(), 2 * world * sizeof(uint32_t*), cudaMemcpyHostToDevice, j->s));
            std::vector<uint64_t> cur(dst_offsets, dst_offsets + world);
            shard_scatter(j, cur, nullptr, nullptr, d_ptrs, d_ptrs + world);
            j->arena.release(d_ptrs);
        }
        CK(cudaStreamSynchronize(j->s));
    } catch (const Fail& f) {
        st = f.st;
    }
    for (void* p : opened) cudaIpcCloseMemHandle(p);
    return st;
}

namespace {
kmc_status shard_count_impl(kmc_job* j, const uint32_t* recv_records, const uint32_t* recv_sigs, uint64_t n_recv,
                            uint64_t* n_out, bool in_place);
}

kmc_status kmc_shard_count_recv(kmc_job* j, uint64_t* n_out) {
    if (!j || !j->shard || !n_out || !j->recv_recs) {
        set_err("invalid kmc_shard_count_recv arguments");
        return KMC_ERR_INVALID_ARG;
    }
    return shard_count_impl(j, j->recv_recs, j->recv_sigs, j->n_recv, n_out, true);
}

kmc_status kmc_shard_count(kmc_job* j, const uint32_t* recv_records, const uint32_t* recv_sigs, uint64_t n_recv,
                           uint64_t* n_out) {
    if (!j || !j->shard || !n_out || (n_recv > 0 && (!recv_records || !recv_sigs))) {
        set_err("invalid kmc_shard_count arguments");
        return KMC_ERR_INVALID_ARG;
    }
    return shard_count_impl(j, recv_records, recv_sigs, n_recv, n_out, false);
}

namespace {
// in_place: the received records already sit in job-owned buffers (the fused exchange's
// receive buffers), read where they are instead of being copied into scratch
kmc_status shard_count_impl(kmc_job* j, const uint32_t* recv_records, const uint32_t* recv_sigs, uint64_t n_recv,
                            uint64_t* n_out, bool in_place) {
    *n_out = 0;
    try {
        PlanCtx& c = j->ctx;
        Arena& ar = j->arena;
        cudaStream_t s = j->s;
        const int RW = record_words(j->k);
        // this rank's bins only: the records of every bin it owns, from all ranks
        uint64_t nrec = 0, nwin = 0;
        for (uint64_t b = 0; b < c.n_bins; ++b) {
            if (c.owner[b] != (uint32_t)j->rank) {
                c.bw[b] = 0;
                c.bn[b] = 0;
            }
            c.bo[b] = nrec;
            nrec += c.bn[b];
            nwin += c.bw[b];
        }
        if (nrec != n_recv) {
            set_err("received %llu records, the plan gives this rank %llu", (unsigned long long)n_recv,
                    (unsigned long long)nrec);
            throw Fail{KMC_ERR_INVALID_ARG};
        }
        c.n_records = nrec;
        c.n_windows = nwin;
        j->st.n_records = nrec;
        j->st.n_windows = nwin;
        if (c.n_bins) {
            CK(cudaMemcpyAsync(c.pa.bin_w, c.bw.data(), c.n_bins * 8, cudaMemcpyHostToDevice, s));
            CK(cudaMemcpyAsync(c.pa.bin_nrec, c.bn.data(), c.n_bins * 8, cudaMemcpyHostToDevice, s));
            CK(cudaMemcpyAsync(c.pa.bin_rec_off, c.bo.data(), c.n_bins * 8, cudaMemcpyHostToDevice, s));
        }
        ar.release(c.tmp_recs);
        ar.release(c.tmp_sig);
        c.tmp_recs = c.tmp_sig = nullptr;
        if (n_recv > 0 && in_place) {
            c.tmp_recs = const_cast<uint32_t*>(recv_records);  // not arena memory: release() skips it
            c.tmp_sig = const_cast<uint32_t*>(recv_sigs);
        } else if (n_recv > 0) {
            c.tmp_recs = reinterpret_cast<uint32_t*>(ar.alloc(n_recv * RW * 4));
            c.tmp_sig = ar.get<uint32_t>(n_recv);
            CK(cudaMemcpyAsync(c.tmp_recs, recv_records, n_recv * RW * 4, cudaMemcpyDefault, s));
            CK(cudaMemcpyAsync(c.tmp_sig, recv_sigs, n_recv * 4, cudaMemcpyDefault, s));
        }
        c.tmp_n = c.tmp_cap = n_recv;
        CK(cudaMemsetAsync(c.gstats, 0, GS_N * 8, s));
        count_phase(j, c);
        CK(cudaStreamSynchronize(s));
    } catch (const Fail& f) {
        return f.st;
    }
    *n_out = j->n_surv;
    return KMC_OK;
}
}  // namespace

int kmc_record_words(int k) { return record_words(k); }

kmc_status kmc_debug_signatures(const uint8_t* reads, const uint64_t* read_offsets, uint64_t n_reads, int k, int p,
                                uint32_t* out_sig, void* stream) {
    return kmc_debug_signatures_ex(reads, read_offsets, n_reads, k, p, 0, out_sig, stream);
}

kmc_status kmc_debug_signatures_ex(const uint8_t* reads, const uint64_t* read_offsets, uint64_t n_reads, int k, int p,
                                   int plain_minimizers, uint32_t* out_sig, void* stream) {
    kmc_status v = validate(k, p, 1, 1);
    if (v != KMC_OK) return v;
    kmc_job j;
    j.s = (cudaStream_t)stream;
    j.k = k;
    j.p = p;
    j.arena.bind(j.s);
    try {
        j.host_small = pin_acquire();
        if (!j.host_small) {
            set_err("pinned readback buffer allocation failed");
            throw Fail{KMC_ERR_ALLOC};
        }
        if (n_reads == 0) return KMC_OK;
        uint64_t off0, offN;
        read_extent(&j, read_offsets, n_reads, &off0, &offN);
        const uint64_t n_bases = offN - off0;
        if (n_bases == 0) return KMC_OK;
        const uint8_t* d_reads = reads;
        const uint64_t* d_off = read_offsets;
        if (!is_device_ptr(reads)) {
            uint8_t* r = j.arena.get<uint8_t>(n_bases);
            CK(cudaMemcpyAsync(r, reads, n_bases, cudaMemcpyHostToDevice, j.s));
            d_reads = r;
        }
        if (!is_device_ptr(read_offsets)) {
            uint64_t* o = j.arena.get<uint64_t>(n_reads + 1);
            CK(cudaMemcpyAsync(o, read_offsets, (n_reads + 1) * 8, cudaMemcpyHostToDevice, j.s));
            d_off = o;
        }
        uint32_t* d_out = out_sig;
        const bool host_out = !is_device_ptr(out_sig);
        if (host_out) d_out = j.arena.get<uint32_t>(n_bases);
        const uint64_t n_tiles = p1_num_tiles(n_bases);
        uint64_t* tile_r_lo = j.arena.get<uint64_t>(n_tiles);
        CK(launch_tile_reads(d_off, n_reads, off0, n_tiles, tile_r_lo, j.s));
        P1Args a{};
        a.reads = d_reads;
        a.offsets = d_off;
        a.n_reads = n_reads;
        a.off0 = off0;
        a.n_bases = n_bases;
        a.k = k;
        a.p = p;
        a.rules = plain_minimizers ? 0 : 1;
        a.reads_aligned16 = ((uintptr_t)d_reads & 15) == 0;
        a.tile_r_lo = tile_r_lo;
        a.dbg_sig = d_out;
        CK(launch_p1(P1_MODE_DEBUG, a, n_tiles, j.s));
        if (host_out) CK(cudaMemcpyAsync(out_sig, d_out, n_bases * 4, cudaMemcpyDeviceToHost, j.s));
        CK(cudaStreamSynchronize(j.s));
    } catch (const Fail& f) {
        cudaStreamSynchronize(j.s);
        return f.st;
    }
    return KMC_OK;
}

kmc_status kmc_debug_allowed(int p, uint8_t* out_allowed, void* stream) {
    if (p < 1 || p > 15) {
        set_err("p=%d outside [1, 15]", p);
        return KMC_ERR_INVALID_ARG;
    }
    cudaStream_t s = (cudaStream_t)stream;
    Arena ar;
    ar.bind(s);
    try {
        const uint64_t n = 1ull << (2 * p);
        uint8_t* d = out_allowed;
        const bool host_out = !is_device_ptr(out_allowed);
        if (host_out) d = ar.get<uint8_t>(n);
        CK(launch_debug_allowed(p, d, s));
        if (host_out) CK(cudaMemcpyAsync(out_allowed, d, n, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
    } catch (const Fail& f) {
        ar.release_all();
        return f.st;
    }
    ar.release_all();
    return KMC_OK;
}

kmc_status kmc_write_db(const void* kmers, const uint32_t* counts, uint64_t n, int k, int p, uint32_t cutoff_min,
                        uint32_t cutoff_max, uint32_t counter_max, const char* path, void* stream) {
    if (!path || k < 1 || k > 64 || p < 1 || p > 12 || p > k || counter_max == 0 ||
        (n > 0 && (!kmers || !counts)) || n >= (1ull << 32)) {
        set_err("invalid kmc_write_db arguments (path=%p k=%d p=%d counter_max=%u n=%llu)", (const void*)path, k, p,
                counter_max, (unsigned long long)n);
        return KMC_ERR_INVALID_ARG;
    }
    cudaStream_t s = (cudaStream_t)stream;
    Arena ar;
    ar.bind(s);
    try {
        const int kw = k <= 32 ? 1 : 2;
        const size_t ksz = 8 * (size_t)kw;
        const int G = db_group_shift(p), lut = db_lut_length(k, p), cb = db_counter_bytes(counter_max);
        const uint64_t na = db_n_arrays(p), entries = na << (2 * lut);
        const int nb = (k - lut) / 4, rec = nb + cb;
        std::vector<uint64_t> hpos(entries + 1, 0);
        std::vector<uint8_t> hrec((size_t)n * rec);
        if (n > 0) {
            const void* dk = kmers;
            const uint32_t* dc = counts;
            if (!is_device_ptr(kmers)) {
                void* t = ar.alloc(n * ksz);
                CK(cudaMemcpyAsync(t, kmers, n * ksz, cudaMemcpyHostToDevice, s));
                dk = t;
            }
            if (!is_device_ptr(counts)) {
                uint32_t* t = ar.get<uint32_t>(n);
                CK(cudaMemcpyAsync(t, counts, n * 4, cudaMemcpyHostToDevice, s));
                dc = t;
            }
            // ids (signature >> G), then a stable sort by id: k-mers stay ascending per id
            uint64_t* ids = ar.get<uint64_t>(n);
            uint32_t* idx = ar.get<uint32_t>(n);
            CK(launch_db_ids(kw, dk, n, k, p, ids, idx, s));
            int nbits = 1;
            while ((1ull << nbits) < na) ++nbits;
            RadixScratch rs{};
            rs.keys_alt = ar.alloc(n * 8);
            rs.vals_alt = ar.get<uint32_t>(n);
            rs.tile_hist = ar.get<uint32_t>(radix_status_words(n, 1));
            rs.tile_off = ar.get<uint32_t>(radix_aux_words());
            rs.scan_temp = ar.alloc(radix_scan_temp_bytes(n, 1));
            rs.red = ar.get<unsigned long long>(4);
            unsigned long long* red_host = nullptr;
            CK(cudaMallocHost(&red_host, 4 * sizeof(unsigned long long)));
            rs.red_host = red_host;
            void* sk = nullptr;
            uint32_t* perm = nullptr;
            int sl = 0;
            const cudaError_t se = device_radix_sort(1, ids, idx, n, nbits, rs, s, &sk, &perm, &sl);
            cudaFreeHost(red_host);
            CK(se);
            // prefixes region: exclusive scan of the records per (id, prefix), + guard
            unsigned long long* cnt = ar.get<unsigned long long>(entries + 1);
            CK(cudaMemsetAsync(cnt, 0, (entries + 1) * 8, s));
            CK(launch_db_hist(kw, dk, (const uint64_t*)sk, perm, n, k, lut, cnt, s));
            uint64_t* pos = ar.get<uint64_t>(entries + 1);
            void* temp = ar.alloc(scan_temp_bytes(entries + 1));
            CK(scan_u64((const uint64_t*)cnt, pos, entries, temp, s));
            uint8_t* recs = ar.get<uint8_t>((size_t)n * rec);
            CK(launch_db_records(kw, dk, dc, perm, n, k, lut, cb, counter_max, recs, s));
            CK(cudaMemcpyAsync(hpos.data(), pos, (entries + 1) * 8, cudaMemcpyDeviceToHost, s));
            CK(cudaMemcpyAsync(hrec.data(), recs, (size_t)n * rec, cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
        }
        // .kmc_pre
        std::vector<uint32_t> amap((1ull << (2 * p)) + 1);
        for (uint64_t sg = 0; sg < amap.size(); ++sg) amap[sg] = (uint32_t)(sg >> G);
        uint8_t hdr[68];
        auto put32 = [&](int o, uint32_t v) { memcpy(hdr + o, &v, 4); };
        memset(hdr, 0, sizeof(hdr));
        put32(0, (uint32_t)k);
        put32(4, 0u);  // mode: occurrence counters
        put32(8, (uint32_t)cb);
        put32(12, (uint32_t)lut);
        put32(16, (uint32_t)p);
        put32(20, cutoff_min);
        put32(24, cutoff_max);
        memcpy(hdr + 28, &n, 8);
        put32(64, 0x200u);  // KMC_VER (tmp[7] at 36..63 stays 0)
        const uint32_t hpos_field = sizeof(hdr);
        const std::string pre_path = std::string(path) + ".kmc_pre", suf_path = std::string(path) + ".kmc_suf";
        FILE* f = fopen(pre_path.c_str(), "wb");
        bool ok = f != nullptr;
        if (ok) {
            ok = fwrite("KMCP", 1, 4, f) == 4 && fwrite(hpos.data(), 8, hpos.size(), f) == hpos.size() &&
                 fwrite(amap.data(), 4, amap.size(), f) == amap.size() && fwrite(hdr, 1, sizeof(hdr), f) == sizeof(hdr) &&
                 fwrite(&hpos_field, 4, 1, f) == 1 && fwrite("KMCP", 1, 4, f) == 4;
            ok = (fclose(f) == 0) && ok;
        }
        if (ok) {
            f = fopen(suf_path.c_str(), "wb");
            ok = f != nullptr;
            if (ok) {
                ok = fwrite("KMCS", 1, 4, f) == 4 && fwrite(hrec.data(), 1, hrec.size(), f) == hrec.size() &&
                     fwrite("KMCS", 1, 4, f) == 4;
                ok = (fclose(f) == 0) && ok;
            }
        }
        if (!ok) {
            set_err("cannot write %s / %s", pre_path.c_str(), suf_path.c_str());
            throw Fail{KMC_ERR_IO};
        }
    } catch (const Fail& e) {
        ar.release_all();
        return e.st;
    }
    ar.release_all();
    return KMC_OK;
}

}  // extern "C"
