// Host side of the B200 acquisition path: contexts, transform plans, code
// sets, window sets, launch orchestration and the extern "C" ABI declared in
// include/tagdsp_gpu.h.  Kernels live in kernels.cuh.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <complex>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <functional>
#include <map>
#include <mutex>
#include <tuple>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "tagdsp_gpu.h"
#include "kernels.cuh"
#include "corr_v3.cuh"
#include "peak.cuh"
#include "generic.cuh"
#include <cudaTypedefs.h>

namespace {

thread_local std::string g_err;
std::atomic<uint64_t> g_launches{0};
// bumped by every device allocation and free: a captured CUDA graph is only
// replayed while no buffer it may reference has moved
std::atomic<uint64_t> g_dev_epoch{0};
// small tracking batches as CUDA graphs (track_graph): 0 = stream ops issued
// normally, 1 = being captured, 2 = replay -- host-side descriptor rebuild
// only, every stream op is skipped (the instantiated graph carries them)
thread_local int tl_graph_mode = 0;
#define STREAM_OPS (tl_graph_mode != 2)
// a replayed tracking graph: its kernels were counted as launched while the
// host pass walked the launch sites
#define LAUNCHED_GRAPH() ck(cudaGetLastError(), "graph launch")

struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] void fail(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    throw Error(code, buf);
}

void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) fail(e == cudaErrorMemoryAllocation ? TDG_ENOMEM : TDG_ECUDA, "%s: %s", what, cudaGetErrorString(e));
}

#define CK(x) ck((x), #x)
#define TDG_STR2(x) #x
#define TDG_STR(x) TDG_STR2(x)
#define LAUNCHED()                                                                  \
    do {                                                                            \
        if (tl_graph_mode != 1) g_launches.fetch_add(1, std::memory_order_relaxed); \
        ck(cudaGetLastError(), "kernel launch (" TDG_STR(__LINE__) ")");            \
    } while (0)

template <class F>
int guard(F&& f) {
    try {
        f();
        return TDG_OK;
    } catch (const Error& e) {
        g_err = e.what();
        return e.code;
    } catch (const std::bad_alloc&) {
        g_err = "host allocation failed";
        return TDG_ENOMEM;
    } catch (const std::exception& e) {
        g_err = e.what();
        return TDG_EINTERNAL;
    }
}

// ---------------------------------------------------------------------------
// Device buffer
struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() { release(); }
    void release() {
        if (p) {
            cudaFree(p);
            g_dev_epoch.fetch_add(1, std::memory_order_relaxed);
        }
        p = nullptr;
        bytes = 0;
    }
    void ensure(size_t b) {
        if (b <= bytes) return;
        release();
        CK(cudaMalloc(&p, b));
        g_dev_epoch.fetch_add(1, std::memory_order_relaxed);
        bytes = b;
        // debugging aid: TDG_POISON_ALLOC=<byte> fills new device buffers with
        // that byte (0x7f: +3.4e38 floats, 0xff: NaN), so a read before the
        // first write shows up in the results
        static const int poison = getenv("TDG_POISON_ALLOC") ? int(strtol(getenv("TDG_POISON_ALLOC"), nullptr, 0)) : -1;
        if (poison >= 0) {   // complete before any stream (non-blocking ones included) writes it
            CK(cudaMemset(p, poison, b));
            CK(cudaDeviceSynchronize());
        }
    }
    template <class T>
    T* as() const { return static_cast<T*>(p); }
};

// Descriptor staging: one pinned host buffer + one device buffer per pack,
// uploaded with a single async copy; the next reuse waits on the copy's event.
struct DescPack {
    char* host = nullptr;
    size_t cap = 0, used = 0;
    DevBuf dev;
    cudaEvent_t done = nullptr;
    bool pending = false;
    DescPack() = default;
    DescPack(const DescPack&) = delete;
    DescPack& operator=(const DescPack&) = delete;
    ~DescPack() {
        if (done) cudaEventDestroy(done);
        if (host) cudaFreeHost(host);
    }
    void begin() {
        if (pending) CK(cudaEventSynchronize(done));
        pending = false;
        used = 0;
    }
    template <class T>
    size_t add(const std::vector<T>& v) {
        const size_t off = (used + 255) & ~size_t(255);
        const size_t need = off + v.size() * sizeof(T);
        if (need > cap) {
            size_t ncap = std::max(need, cap * 2 + 4096);
            char* nh = nullptr;
            CK(cudaHostAlloc(reinterpret_cast<void**>(&nh), ncap, cudaHostAllocDefault));
            g_dev_epoch.fetch_add(1, std::memory_order_relaxed);   // staging moved
            if (host) {
                std::memcpy(nh, host, used);
                cudaFreeHost(host);
            }
            host = nh;
            cap = ncap;
        }
        if (!v.empty()) std::memcpy(host + off, v.data(), v.size() * sizeof(T));
        used = need;
        return off;
    }
    void commit(cudaStream_t st) {
        dev.ensure(std::max<size_t>(used, 256));
        if (used && STREAM_OPS) CK(cudaMemcpyAsync(dev.p, host, used, cudaMemcpyHostToDevice, st));
        if (tl_graph_mode) return;   // graph packs: the caller orders reuse (synchronous calls)
        if (!done) CK(cudaEventCreateWithFlags(&done, cudaEventDisableTiming));
        CK(cudaEventRecord(done, st));
        pending = true;
    }
    template <class T>
    T* at(size_t off) const { return reinterpret_cast<T*>(static_cast<char*>(dev.p) + off); }
};

// ---------------------------------------------------------------------------
// Supported pass lengths L = P*Q (register codelets P and Q, tools/gen_codelets.py).
#define TDG_MENU(X) \
    X(16, 4, 4)     \
    X(32, 4, 8)     \
    X(64, 8, 8)     \
    X(128, 8, 16)   \
    X(256, 16, 16)  \
    X(360, 18, 20)  \
    X(450, 18, 25)  \
    X(512, 16, 32)  \
    X(864, 27, 32)  \
    X(1008, 28, 36) \
    X(1024, 32, 32)

struct PassShape {
    int L, P, Q;
};
const PassShape kMenu[] = {
#define X(L, P, Q) {L, P, Q},
    TDG_MENU(X)
#undef X
};

const PassShape& shape_of(int L) {
    for (const auto& s : kMenu)
        if (s.L == L) return s;
    fail(TDG_ERANGE, "unsupported pass length %d", L);
}

// forward pass 1: t2 columns per CTA (16: 64-byte runs per load row; 8 was
// ~10 % slower on tracking batches, 32 where it fits ~1 % slower than 16,
// tools/ab_libs.sh)
constexpr int fwd1_tb(int) { return 16; }
constexpr int kDemodBlk = 4;

uint64_t pad_length_impl(uint64_t n) {
    if (n < 1) fail(TDG_EINVAL, "pad_length: n must be >= 1");
    for (uint64_t m = n;; ++m) {
        uint64_t r = m;
        for (uint64_t p : {2, 3, 5, 7})
            while (r % p == 0) r /= p;
        if (r == 1) return m;
    }
}

// Codelet cost (scalar ops per point of one pass, from tools/gen_codelets.py's
// counts: ops(P)/P + ops(Q)/Q) plus ~12 ops/point of per-pass overhead.
double pass_cost(int L) {
    switch (L) {
        case 16: return 8.0 + 12;
        case 32: return 10.5 + 12;
        case 64: return 13.0 + 12;
        case 128: return 15.5 + 12;
        case 256: return 18.0 + 12;
        case 360: return 25.51 + 12;
        case 450: return 28.79 + 12;
        case 512: return 20.75 + 12;
        case 864: return 27.82 + 12;
        case 1008: return 30.16 + 12;
        case 1024: return 23.5 + 12;
    }
    return 1e9;
}

// (N1, N2) splits the fused correlation kernel is instantiated for: the
// search shape (1024 x 864), the tracking shape (450 x 360) and a power-of-two
// ladder for everything else (small transforms are padded up; any
// N >= W + n - 1 gives the same lags [0, W)).
#define TDG_FUSED(X)                                                              \
    X(16, 4, 4, 16, 4, 4) X(32, 4, 8, 16, 4, 4) X(32, 4, 8, 32, 4, 8)             \
    X(64, 8, 8, 32, 4, 8) X(64, 8, 8, 64, 8, 8) X(128, 8, 16, 64, 8, 8)           \
    X(128, 8, 16, 128, 8, 16) X(256, 16, 16, 128, 8, 16)                          \
    X(256, 16, 16, 256, 16, 16) X(512, 16, 32, 256, 16, 16)                       \
    X(512, 16, 32, 512, 16, 32) X(450, 18, 25, 360, 18, 20)                       \
    X(1024, 32, 32, 512, 16, 32) X(1024, 32, 32, 864, 27, 32)                     \
    X(1024, 32, 32, 1024, 32, 32)

// Transform length N = N1*N2 >= need minimising N*(cost(N1)+cost(N2)) over
// the fused splits; any N >= W + n - 1 yields the same lags [0, W) (linear
// correlation).  N1 (pass B, 32 KB tiles) >= N2 (pass A columns).
bool choose_corr_len(uint64_t need, int* n1, int* n2) {
    double best = 0.0;
    uint64_t bestN = 0;
    int b1 = 0, b2 = 0;
    auto consider = [&](int a, int b) {
        const uint64_t n = uint64_t(a) * uint64_t(b);
        if (n < need) return;
        const double c = double(n) * (pass_cost(a) + pass_cost(b));
        if (bestN == 0 || c < best * (1.0 - 1e-9) || (c <= best * (1.0 + 1e-9) && n < bestN)) {
            best = c;
            bestN = n;
            b1 = a;
            b2 = b;
        }
    };
#define X(L1, P1, Q1, L2, P2, Q2) consider(L1, L2);
    TDG_FUSED(X)
#undef X
    if (!bestN) return false;
    *n1 = b1;
    *n2 = b2;
    return true;
}

// ---------------------------------------------------------------------------
// Kernel dispatch by pass length
template <class T>
void set_smem(T* kernel, size_t bytes) {
    // the opt-in limit only ever rises per (kernel, device): a launch with
    // fewer bytes than an earlier one must not lower it under that one.  The
    // attribute call costs a few microseconds (latency-bound tracking
    // batches), so it is made only when the limit has to rise.
    static std::mutex mu;
    static std::map<std::pair<const void*, int>, size_t> limit;
    if (bytes <= 48 * 1024) return;
    int dev = 0;
    CK(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(mu);
    size_t& cur = limit[std::make_pair(reinterpret_cast<const void*>(kernel), dev)];
    if (bytes <= cur) return;
    CK(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes)));
    cur = bytes;
}

int block_for(int tasks) {
    int t = ((tasks + 31) / 32) * 32;
    return std::min(256, std::max(32, t));
}

void launch_fwd1(int L, unsigned n_seq, cudaStream_t st, const tdg::SeqPairDesc* pairs, int N2, const float2* tw) {
    switch (L) {
#define X(LL, P, Q)                                                                        \
    case LL: {                                                                             \
        constexpr int TB = fwd1_tb(LL);                                                    \
        const size_t sm = size_t(P) * Q * TB * sizeof(float2);                             \
        const dim3 grid(unsigned((N2 + TB - 1) / TB), n_seq);                              \
        set_smem(tdg::k_fwd_pass1<P, Q, TB>, sm);                                          \
        if (STREAM_OPS) tdg::k_fwd_pass1<P, Q, TB><<<grid, block_for(std::max(P, Q) * TB), sm, st>>>(pairs, N2, tw); \
        LAUNCHED();                                                                        \
        return;                                                                            \
    }
        TDG_MENU(X)
#undef X
    }
    fail(TDG_ERANGE, "fwd1: length %d", L);
}

void launch_fwd2(int L, bool split, dim3 grid, cudaStream_t st, const tdg::SeqPairDesc* pairs, int N1,
                 const float2* tw, const float2* twI, bool pfa) {
    switch (L) {
#define X(LL, P, Q)                                                                                       \
    case LL: {                                                                                            \
        constexpr int QS = (Q % 2) ? Q : Q + 1;                                                           \
        const size_t sm = (size_t(2) * P * QS + 2 * LL + 2 * (P + Q)) * sizeof(float2);                   \
        if (split) {                                                                                      \
            set_smem(tdg::k_fwd_pass2<P, Q, true>, sm);                                                   \
            if (STREAM_OPS) tdg::k_fwd_pass2<P, Q, true><<<grid, block_for(2 * std::max(P, Q)), sm, st>>>(pairs, N1, tw, twI, pfa); \
        } else {                                                                                          \
            set_smem(tdg::k_fwd_pass2<P, Q, false>, sm);                                                  \
            if (STREAM_OPS) tdg::k_fwd_pass2<P, Q, false><<<grid, block_for(2 * std::max(P, Q)), sm, st>>>(pairs, N1, tw, twI, pfa); \
        }                                                                                                 \
        LAUNCHED();                                                                                       \
        return;                                                                                           \
    }
        TDG_MENU(X)
#undef X
    }
    fail(TDG_ERANGE, "fwd2: length %d", L);
}

// SM count of the current device (cached per device: one process may drive
// several GPUs, one context each)
int num_sms() {
    static std::mutex mu;
    static std::map<int, int> cache;
    int dev = 0;
    CK(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(dev);
    if (it != cache.end()) return it->second;
    int n = 0;
    CK(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
    cache[dev] = n;
    return n;
}

template <class K>
int persistent_grid(K* kernel, int threads, size_t smem, int n_items) {
    // attributes + occupancy once per (kernel, threads, smem) and device
    static std::mutex mu;
    static std::map<std::tuple<const void*, int, size_t, int>, int> cache;
    int dev = 0;
    CK(cudaGetDevice(&dev));
    const auto key = std::make_tuple(reinterpret_cast<const void*>(kernel), threads, smem, dev);
    int per_sm = 0;
    {
        std::lock_guard<std::mutex> lk(mu);
        auto it = cache.find(key);
        if (it != cache.end()) {
            per_sm = it->second;
        } else {
            CK(cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
            set_smem(kernel, smem);
            CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem));
            cache[key] = per_sm;
        }
    }
    if (per_sm < 1) fail(TDG_ECUDA, "kernel does not fit on an SM (smem %zu)", smem);
    return std::max(1, std::min(n_items, per_sm * num_sms()));
}

// cap: max CTAs per SM of the pass (0 = occupancy; per context, tdg_ctx::cta_cap)
template <int TYPE>
void launch_pass(int N1, int N2, cudaStream_t st, const tdg::CorrSched& S, int cap) {
    const int n_items = TYPE == 0 ? S.nA : S.nB;
#define X(L1, P1, Q1, L2, P2, Q2)                                                       \
    if (N1 == L1 && N2 == L2) {                                                         \
        using F = tdg::Fused<P2, Q2, P1, Q1>;                                           \
        auto* k = tdg::k_corr_pass<P2, Q2, P1, Q1, TYPE>;                               \
        /* + the wave's descriptors (copied to shared memory by every CTA) */          \
        const size_t sm = F::SMEM + ((TYPE == 0 ? S.ngw * sizeof(tdg::CorrGroup<tdg::kGroup>)       \
                                                : S.wave_pairs * sizeof(tdg::CorrPairOut)) + 15) / 16 * 16; \
        int grid = persistent_grid(k, F::NT, sm, n_items);                              \
        if (cap > 0) grid = std::min(grid, cap * num_sms());                            \
        if (STREAM_OPS) k<<<grid, F::NT, sm, st>>>(S);                                  \
        LAUNCHED();                                                                     \
        return;                                                                         \
    }
    TDG_FUSED(X)
#undef X
    fail(TDG_ERANGE, "correlation split %d x %d is not instantiated", N1, N2);
}

// ---------------------------------------------------------------------------
// Demodulation filter design, restated from proj/src/dsp.cpp:37-73 with the
// same float/double arithmetic (fill_bandpass, fill_matched, convolve_into).
using cfloat = std::complex<float>;

void fill_bandpass(double center, double width, size_t taps, double fs, std::vector<cfloat>& out) {
    const double pi = 3.14159265358979323846;
    double fc = width / 2.0;
    double mid = double(taps - 1) / 2.0;
    std::vector<double> lp(taps);
    double sum = 0.0;
    for (size_t k = 0; k < taps; ++k) {
        double t = double(k) - mid;
        double x = 2.0 * fc * t / fs;
        double sinc = (x == 0.0) ? 1.0 : std::sin(pi * x) / (pi * x);
        double w = (taps == 1) ? 1.0 : 0.54 - 0.46 * std::cos(2.0 * pi * double(k) / double(taps - 1));
        lp[k] = sinc * w;
        sum += lp[k];
    }
    out.resize(taps);
    for (size_t k = 0; k < taps; ++k) {
        double t = double(k) - mid;
        double a = 2.0 * pi * center * t / fs;
        double g = lp[k] / sum;
        out[k] = cfloat(float(g * std::cos(a)), float(g * std::sin(a)));
    }
}

void fill_matched(double freq, size_t spb, double fs, std::vector<cfloat>& out) {
    const double pi = 3.14159265358979323846;
    out.resize(spb);
    for (size_t k = 0; k < spb; ++k) {
        double a = 2.0 * pi * freq * double(spb - 1 - k) / fs;
        out[k] = cfloat(float(std::cos(a)), float(-std::sin(a)));
    }
}

std::vector<cfloat> convolve(const std::vector<cfloat>& a, const std::vector<cfloat>& b) {
    std::vector<cfloat> out(a.size() + b.size() - 1, cfloat{0.0f, 0.0f});
    for (size_t i = 0; i < a.size(); ++i)
        for (size_t j = 0; j < b.size(); ++j) out[i + j] += a[i] * b[j];
    return out;
}

size_t samples_per_bit(const tdg_modulation& m) {
    double spb = m.sample_rate / m.bit_rate;
    auto n = static_cast<size_t>(spb + 0.5);
    if (n < 1 || std::abs(spb - double(n)) > 1e-9)
        fail(TDG_EINVAL, "sample_rate / bit_rate must be a positive integer");
    return n;
}

void validate_cfg(const tdg_demod_config& c) {
    if (c.bandpass_taps < 1) fail(TDG_EINVAL, "design_bandpass: taps must be >= 1");
    if (c.bandpass_width <= 0.0) fail(TDG_EINVAL, "design_bandpass: width must be positive");
    if (std::abs(c.bandpass_center) + c.bandpass_width / 2.0 > c.mod.sample_rate / 2.0)
        fail(TDG_EINVAL, "design_bandpass: band outside Nyquist");
    samples_per_bit(c.mod);
}

}  // namespace

// ---------------------------------------------------------------------------
struct tdg_ctx;
struct KScope {   // records a CUDA event pair around one launch when timing is on
    tdg_ctx* ctx;
    const char* name;
    cudaEvent_t a = nullptr;
    KScope(tdg_ctx* c, const char* n);
    ~KScope();
};

struct DescPacks {
    DescPack fwd, corr, misc, stats;
};

// A small tracking batch (one correlation wave) captured as a CUDA graph:
// demod, forward transforms, both correlation passes and the statistics with
// their descriptor uploads from this entry's own pinned staging.  A replay
// rewrites the staging in place (same offsets) and launches the graph; it is
// valid while nothing it references has moved (g_dev_epoch) and the key --
// batch size, code set, window, input block and every kernel parameter that
// comes from the configuration -- matches.
struct TrackGraph {
    std::vector<double> key;
    const void* cs = nullptr;
    const void* base = nullptr;
    uint64_t epoch = 0;
    int state = 0;   // 1: seen once (every cache warm), 2: captured
    cudaGraphExec_t exec = nullptr;
    DescPacks packs;
    uint64_t last_use = 0;
    TrackGraph() = default;
    TrackGraph(const TrackGraph&) = delete;
    TrackGraph& operator=(const TrackGraph&) = delete;
    ~TrackGraph() {
        if (exec) cudaGraphExecDestroy(exec);
    }
};

struct tdg_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    std::map<int, std::unique_ptr<DevBuf>> tw;   // per pass length: w_L^{+a c}, index a*Q + c
    int clen = 0;               // composed filter length of the last filter_spectra key
    // scratch
    DevBuf T, M, keys, det_dev, stream_buf, stats_part, stats_ctr;
    DevBuf gen_a, gen_b, gen_c, gen_d;   // span-level entry points (tdg_fft, tdg_convolve, ...)
    // detect() stage split (option "detect_timings"): events around the
    // correlation stage and the statistics of the last detect
    bool detect_timings = false;
    cudaEvent_t dt_ev[3] = {nullptr, nullptr, nullptr};
    double last_corr_s = 0.0, last_stats_s = 0.0;
    // streams + events of the multi-stream correlation pipeline
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    std::vector<cudaEvent_t> ev_a, ev_b;
    std::vector<cudaStream_t> a_streams, b_streams;
    std::vector<cudaEvent_t> ev_fwd;                  // forward-transform waves done
    int64_t n_streams = 6;
    void ensure_pipeline(int ring) {   // (set_option("n_streams") drops the old streams)
        const size_t ns = size_t(std::max<int64_t>(1, std::min<int64_t>(n_streams, 8)));
        while (a_streams.size() < ns) {
            cudaStream_t x;
            CK(cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking));
            a_streams.push_back(x);
        }
        while (b_streams.size() < ns) {
            cudaStream_t x;
            CK(cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking));
            b_streams.push_back(x);
        }
        if (!ev_fork) CK(cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming));
        if (!ev_join) CK(cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming));
        while (int(ev_a.size()) < ring) {
            cudaEvent_t a, b;
            CK(cudaEventCreateWithFlags(&a, cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&b, cudaEventDisableTiming));
            ev_a.push_back(a);
            ev_b.push_back(b);
        }
    }
    tdg_windows* search_win = nullptr;   // cached window set of tdg_search (reused across calls)
    tdg_windows* track_win = nullptr;    // cached window set of tdg_track (capacity grows)
    // descriptor staging, one pack per stage (no stage waits on another's
    // staging copy); a captured tracking graph brings its own set
    DescPacks own_packs;
    DescPacks* pk = &own_packs;
    std::vector<std::unique_ptr<TrackGraph>> track_graphs;
    int64_t track_graphs_on = 1;   // small tracking batches replayed as CUDA graphs
    uint64_t graph_clock = 0;
    std::vector<char> host_stage;
    int64_t wave_pairs = 8;      // correlation pairs per wave (one pass-A + one pass-B launch)
    int64_t ring = 3;            // M wave buffers in flight
    int64_t discard = 1;         // drop consumed M tiles from L2
    int64_t one_stream = 0;      // tuning: run pass B on the context stream too (no overlap)
    int64_t fwd_wave = 32;       // sequence pairs per forward-FFT wave
    // diagnostics: option "cta_trace" = capacity; every correlation-pass CTA
    // records {smid << 8 | pass, globaltimer at start, at exit} (tdg_cta_trace)
    DevBuf trace;
    uint32_t trace_cap = 0;
    // max CTAs per SM of pass A / pass B (0 = occupancy).  Pass B at 2 of its 3
    // leaves SM room for the next waves' pass A on the other streams (A/B: +0.8 %
    // device and e2e, burst and sustained)
    int cta_cap[2] = {0, 2};
    // optional per-launch CUDA-event timing (bench.py roofline)
    bool time_kernels = false;
    struct KTime {
        const char* name;
        cudaEvent_t a, b;
    };
    std::vector<KTime> ktimes;
    std::vector<cudaEvent_t> ev_pool;
    std::map<std::string, std::pair<uint64_t, double>> kstats;   // name -> (count, total ms)
    cudaEvent_t ev() {
        if (ev_pool.empty()) {
            cudaEvent_t e;
            CK(cudaEventCreate(&e));
            return e;
        }
        cudaEvent_t e = ev_pool.back();
        ev_pool.pop_back();
        return e;
    }
    void collect() {
        if (ktimes.empty()) return;
        CK(cudaStreamSynchronize(stream));
        for (auto& k : ktimes) {
            float ms = 0.f;
            CK(cudaEventElapsedTime(&ms, k.a, k.b));
            auto& st = kstats[k.name];
            st.first += 1;
            st.second += ms;
            ev_pool.push_back(k.a);
            ev_pool.push_back(k.b);
        }
        ktimes.clear();
    }

    const float2* twiddles(int L) {
        auto it = tw.find(L);
        if (it != tw.end()) return it->second->as<float2>();
        const PassShape& s = shape_of(L);
        std::vector<float2> h(static_cast<size_t>(L));
        const double pi = 3.14159265358979323846;
        for (int a = 0; a < s.P; ++a)
            for (int c = 0; c < s.Q; ++c) {
                const long e = long(a) * c % L;
                const double ang = 2.0 * pi * double(e) / double(L);
                h[size_t(a) * s.Q + c] = make_float2(float(std::cos(ang)), float(std::sin(ang)));
            }
        auto buf = std::make_unique<DevBuf>();
        buf->ensure(h.size() * sizeof(float2));
        CK(cudaMemcpyAsync(buf->p, h.data(), h.size() * sizeof(float2), cudaMemcpyHostToDevice, stream));
        CK(cudaStreamSynchronize(stream));
        const float2* p = buf->as<float2>();
        tw[L] = std::move(buf);
        return p;
    }

    // pass-A inter-pass twiddles (csrc/corr_v3.cuh): row k1 = [w_N^{+k1 c}, c < QA]
    // [w_N^{+k1 QA e}, e < PA], computed in double with exact integer reduction
    std::map<std::pair<int, int>, std::unique_ptr<DevBuf>> twi;
    // forward pass 2: row k1 = [w_N^{+k1 a}, a < P][w_N^{+k1 P b}, b < Q]
    // (P x Q the pass-2 split of N2), computed in double
    std::map<std::pair<int, int>, std::unique_ptr<DevBuf>> twf;
    const float2* fwd_inter_twiddles(int N1, int N2) {
        auto key = std::make_pair(N1, N2);
        auto it = twf.find(key);
        if (it != twf.end()) return it->second->as<float2>();
        const PassShape& s = shape_of(N2);
        const int st = s.P + s.Q;
        const long long N = (long long)N1 * N2;
        std::vector<float2> h(size_t(N1) * st);
        const double pi = 3.14159265358979323846;
        for (int k1 = 0; k1 < N1; ++k1)
            for (int r = 0; r < st; ++r) {
                const long long e = (r < s.P ? (long long)k1 * r : (long long)k1 * s.P * (r - s.P)) % N;
                const double ang = 2.0 * pi * double(e) / double(N);
                h[size_t(k1) * st + r] = make_float2(float(std::cos(ang)), float(std::sin(ang)));
            }
        auto buf = std::make_unique<DevBuf>();
        buf->ensure(h.size() * sizeof(float2));
        CK(cudaMemcpyAsync(buf->p, h.data(), h.size() * sizeof(float2), cudaMemcpyHostToDevice, stream));
        CK(cudaStreamSynchronize(stream));
        const float2* p = buf->as<float2>();
        twf[key] = std::move(buf);
        return p;
    }

    const float2* inter_twiddles(int N1, int N2) {
        auto key = std::make_pair(N1, N2);
        auto it = twi.find(key);
        if (it != twi.end()) return it->second->as<float2>();
        const PassShape& s = shape_of(N2);
        const int tws = tdg::inter_tw_stride(s.P, s.Q);
        const long long N = (long long)N1 * N2;
        std::vector<float2> h(size_t(N1) * tws, make_float2(0.f, 0.f));
        const double pi = 3.14159265358979323846;
        // prime-factor split (corr_v3.cuh pfa_split): row k1 = [w_N^{+k1 P c}, c < QA]
        const bool pfa = tdg::pfa_split(s.P, s.Q, N1);
        for (int k1 = 0; k1 < N1; ++k1)
            for (int r = 0; r < s.P + s.Q; ++r) {
                const long long e = (pfa ? (r < s.Q ? (long long)k1 * s.P * r : 0)
                                         : r < s.Q ? (long long)k1 * r : (long long)k1 * s.Q * (r - s.Q)) % N;
                const double ang = 2.0 * pi * double(e) / double(N);
                h[size_t(k1) * tws + r] = make_float2(float(std::cos(ang)), float(std::sin(ang)));
            }
        auto buf = std::make_unique<DevBuf>();
        buf->ensure(h.size() * sizeof(float2));
        CK(cudaMemcpyAsync(buf->p, h.data(), h.size() * sizeof(float2), cudaMemcpyHostToDevice, stream));
        CK(cudaStreamSynchronize(stream));
        const float2* p = buf->as<float2>();
        twi[key] = std::move(buf);
        return p;
    }

    // single-array upload through a pack
    template <class T>
    T* upload(DescPack& pk, const std::vector<T>& v) {
        pk.begin();
        const size_t off = pk.add(v);
        pk.commit(stream);
        return pk.at<T>(off);
    }

    // FFT_1024 spectra of the LO-shifted composed filters for a bin set.  One
    // device buffer per key (configuration + bins), kept in a small LRU: a
    // buffer is never rewritten while kernels queued on the context stream
    // (or captured in a tracking graph) may still read it.  Eviction frees
    // the buffer (cudaFree waits for the device) and drops captured graphs.
    struct HSpec {
        std::vector<double> key;
        DevBuf buf;
        int clen = 0;
        uint64_t last_use = 0;
    };
    std::vector<std::unique_ptr<HSpec>> hspecs;
    uint64_t hspec_clock = 0;
    const float2* filter_spectra(const tdg_demod_config& c, const std::vector<double>& bins) {
        validate_cfg(c);
        // cache key: the parameters the composed filters depend on, then the bins
        std::vector<double> k{c.mod.sample_rate,     c.mod.bit_rate,   c.mod.freq_one,
                              c.mod.freq_zero,       double(c.mod.packet_bits),
                              c.bandpass_center,     c.bandpass_width, double(c.bandpass_taps)};
        k.insert(k.end(), bins.begin(), bins.end());
        for (auto& h : hspecs)
            if (h->key == k) {
                h->last_use = ++hspec_clock;
                clen = h->clen;
                return h->buf.as<float2>();
            }
        const size_t spb = samples_per_bit(c.mod);
        std::vector<cfloat> hbp, hm;
        fill_bandpass(c.bandpass_center, c.bandpass_width, size_t(c.bandpass_taps), c.mod.sample_rate, hbp);
        fill_matched(c.mod.freq_one, spb, c.mod.sample_rate, hm);
        const auto h1c = convolve(hbp, hm);
        fill_matched(c.mod.freq_zero, spb, c.mod.sample_rate, hm);
        const auto h0c = convolve(hbp, hm);
        const int cl = int(h1c.size());
        if (cl > 1024 - 32) fail(TDG_ERANGE, "composed filter of %d taps exceeds the 1024-point demod block", cl);
        const double pi = 3.14159265358979323846;
        std::vector<float2> H(bins.size() * 2 * 1024);
        std::vector<std::complex<double>> tw(1024);
        for (int kk = 0; kk < 1024; ++kk) tw[size_t(kk)] = std::polar(1.0, -2.0 * pi * kk / 1024.0);
        for (size_t b = 0; b < bins.size(); ++b) {
            const double om = 2.0 * pi * bins[b] / c.mod.sample_rate;
            for (int f = 0; f < 2; ++f) {
                const auto& h = f == 0 ? h1c : h0c;
                std::vector<std::complex<double>> hb(h.size());
                for (size_t j = 0; j < h.size(); ++j)
                    hb[j] = std::complex<double>(h[j].real(), h[j].imag()) * std::polar(1.0, om * double(j));
                for (int kk = 0; kk < 1024; ++kk) {
                    std::complex<double> acc = 0.0;
                    for (size_t j = 0; j < h.size(); ++j) acc += hb[j] * tw[(size_t(kk) * j) % 1024];
                    H[(b * 2 + size_t(f)) * 1024 + size_t(kk)] = make_float2(float(acc.real()), float(acc.imag()));
                }
            }
        }
        if (hspecs.size() >= 16) {   // evict the least recently used key
            auto lru = std::min_element(hspecs.begin(), hspecs.end(),
                                        [](const auto& a, const auto& b) { return a->last_use < b->last_use; });
            track_graphs.clear();
            hspecs.erase(lru);
        }
        auto e = std::make_unique<HSpec>();
        e->key = k;
        e->clen = cl;
        e->last_use = ++hspec_clock;
        e->buf.ensure(H.size() * sizeof(float2));
        // a fresh buffer: stream-ordered before every kernel that will read it
        CK(cudaMemcpyAsync(e->buf.p, H.data(), H.size() * sizeof(float2), cudaMemcpyHostToDevice, stream));
        CK(cudaStreamSynchronize(stream));   // H is pageable and local
        clen = cl;
        const float2* p = e->buf.as<float2>();
        hspecs.push_back(std::move(e));
        return p;
    }
};

KScope::KScope(tdg_ctx* c, const char* n) : ctx(c), name(n) {
    if (ctx->time_kernels && !tl_graph_mode) {
        a = ctx->ev();
        cudaEventRecord(a, ctx->stream);
    }
}
KScope::~KScope() {
    if (a) {
        cudaEvent_t b = ctx->ev();
        cudaEventRecord(b, ctx->stream);
        ctx->ktimes.push_back({name, a, b});
    }
}

struct tdg_codeset {
    tdg_ctx* ctx = nullptr;    // creating context (not owned; may be destroyed first)
    int device = 0;
    uint64_t window_len = 0;
    uint64_t n_codes = 0;
    int N1 = 0, N2 = 0;
    uint64_t H = 0;            // half-column spectrum length (N1/2+1)*N2
    uint64_t rep_cap = 0;      // replica_d stride
    uint64_t cap_codes = 0;    // codes the device buffers hold (grows by doubling on append)
    uint64_t ref_corr = 0;     // the reference's corr_len (make_transformed precondition)
    std::vector<double> cfg_key;   // prepared sets: the configuration appended codes must share
    DevBuf spec, rep, nlen_dev, energy_dev, abs_dev;
    std::vector<uint64_t> nlen;
    std::vector<float> energy, abs_sum;
    uint64_t corr_len() const { return uint64_t(N1) * uint64_t(N2); }
    // Segmented correlation (windows longer than the largest transform,
    // N = 1024 x 1024): seg_lags > 0 splits a window's lags [0, W) into
    // segments of seg_lags lags; segment g correlates d[g*B, g*B + B + nmax - 1)
    // (B = seg_lags, nmax = the longest support), which a transform of
    // N >= B + nmax - 1 holds without wrap-around, and its argmax keys merge
    // into the window's (atomicMax over the global lag).  0 = one transform
    // per window.
    uint64_t seg_lags = 0;
    uint64_t nmax = 0;
    uint64_t n_segments(uint64_t W) const { return seg_lags ? (W + seg_lags - 1) / seg_lags : 1; }
};

struct tdg_windows {
    tdg_ctx* ctx = nullptr;    // creating context (not owned; may be destroyed first)
    int device = 0;
    uint64_t W = 0, n_windows = 0, n_bins = 0;
    DevBuf d, u;
    std::vector<int64_t> start;   // window_start per slot
    DevBuf dspec;                 // [slot][segment] half-column spectra
    uint64_t dspec_N = 0;         // transform length dspec was computed for (0 = stale)
    uint64_t dspec_seg = 0;       // ... and its segment length (codeset seg_lags, nmax)
    uint64_t active = 0;          // slots in use (tracking batches reuse a larger set); 0 = all
    uint64_t slots() const { return n_windows * n_bins; }
    uint64_t used() const { return active ? active : slots(); }
};

// Device-resident CircularBuffer (include/tagdsp/scheduler.hpp:11-40,
// proj/src/scheduler.cpp:7-45): the raw int16 I/Q stream addressed by
// absolute sample index, sample t in slot t % cap.  Pushes are host->device
// copies on the ring's own stream; compute on the context stream waits for
// them through `pushed`, and each kernel that reads the ring registers its
// sample range with an event, so a later push only waits for the reads whose
// slots it overwrites (searches of second k overlap the upload of second k+1).
struct tdg_ring {
    tdg_ctx* ctx = nullptr;    // creating context (not owned)
    int device = 0;
    uint64_t cap = 0;          // complex samples
    DevBuf buf;
    int64_t head = 0, tail = 0;
    cudaStream_t copy = nullptr;
    cudaEvent_t pushed = nullptr;
    struct Read {
        int64_t s, e;
        cudaEvent_t ev;
    };
    std::vector<Read> reads;
    std::vector<cudaEvent_t> spare;
    uint64_t slot(int64_t t) const {
        const int64_t c = int64_t(cap);
        return uint64_t(((t % c) + c) % c);
    }
    cudaEvent_t event() {
        if (!spare.empty()) {
            cudaEvent_t e = spare.back();
            spare.pop_back();
            return e;
        }
        cudaEvent_t e;
        CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        return e;
    }
    // true if the sample ranges [a, a+na) and [b, b+nb) share a ring slot
    bool overlap(int64_t a, uint64_t na, int64_t b, uint64_t nb) const {
        if (!na || !nb) return false;
        const uint64_t sa = slot(a), sb = slot(b);
        return (sb + cap - sa) % cap < na || (sa + cap - sb) % cap < nb;
    }
};

namespace {

// Where a kernel's input samples live: a linear device block starting at
// stream index `origin`, or the device ring (absolute-index slots).
struct SampleSource {
    const int16_t* base;
    uint64_t len;
    int64_t origin;
    uint64_t ring_cap;
    tdg_ring* ring;
    static SampleSource linear(const int16_t* p, uint64_t n, int64_t start) { return {p, n, start, 0, nullptr}; }
    static SampleSource of(tdg_ring* r) { return {r->buf.as<int16_t>(), r->cap, 0, r->cap, r}; }
    bool holds(int64_t start, uint64_t n) const {
        if (ring) return start >= ring->head && start + int64_t(n) <= ring->tail;
        return start >= origin && uint64_t(start - origin) + n <= len;
    }
    uint64_t offset(int64_t start) const { return ring ? ring->slot(start) : uint64_t(start - origin); }
    void before_read(tdg_ctx* ctx) const;
    void after_read(tdg_ctx* ctx, int64_t s, int64_t e) const;
};

// Forward transforms of real sequences (pairs packed as r1 + i r2) into
// Hermitian half-column spectra.
struct FwdJob {
    const float* r1;
    const float* r2;
    uint64_t len1, len2;
    float2* S1;
    float2* S2;
};

// split = true: r1, r2 -> two Hermitian half-column spectra (window d's).
// split = false: the packed pair's full spectrum X (code pairs), into S1.
// chunk_done (optional): after each wave of `fwd_wave` jobs an event is
// recorded on the context stream, with the number of jobs completed by then
void run_forward(tdg_ctx* ctx, int N1, int N2, const std::vector<FwdJob>& jobs, bool split,
                 std::vector<std::pair<size_t, cudaEvent_t>>* chunk_done = nullptr) {
    const uint64_t N = uint64_t(N1) * uint64_t(N2);
    const float2* tw1 = ctx->twiddles(N1);
    const float2* tw2 = ctx->twiddles(N2);
    const float2* twI = ctx->fwd_inter_twiddles(N1, N2);
    // at least fwd_wave pairs per launch; short transforms (tracking) fill up
    // to kFwdScratch bytes of T so that one launch still covers the GPU
    constexpr size_t kFwdScratch = size_t(56) << 20;
    const size_t wave = std::min(jobs.size(), std::max(size_t(std::max<int64_t>(1, ctx->fwd_wave)),
                                                       kFwdScratch / (N * sizeof(float2))));
    ctx->T.ensure(wave * N * sizeof(float2));
    std::vector<tdg::SeqPairDesc> d(jobs.size());
    for (size_t i = 0; i < jobs.size(); ++i) {
        const auto& j = jobs[i];
        d[i] = {j.r1, j.r2, j.len1, j.len2, ctx->T.as<float2>() + (i % wave) * N, j.S1, j.S2};
    }
    tdg::SeqPairDesc* dd = ctx->upload(ctx->pk->fwd, d);
    for (size_t base = 0; base < jobs.size(); base += wave) {
        const size_t n = std::min(wave, jobs.size() - base);
        {
            KScope ks(ctx, "fwd_pass1");
            launch_fwd1(N1, unsigned(n), ctx->stream, dd + base, N2, tw1);
        }
        {
            KScope ks(ctx, "fwd_pass2");
            launch_fwd2(N2, split, dim3(unsigned(N1 / 2 + 1), unsigned(n)), ctx->stream, dd + base, N1, tw2, twI,
                        tdg::pfa_split(shape_of(N2).P, shape_of(N2).Q, N1));
        }
        if (chunk_done) {
            const size_t k = chunk_done->size();
            while (ctx->ev_fwd.size() <= k) {
                cudaEvent_t e;
                CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
                ctx->ev_fwd.push_back(e);
            }
            CK(cudaEventRecord(ctx->ev_fwd[k], ctx->stream));
            chunk_done->push_back({base + n, ctx->ev_fwd[k]});
        }
    }
}

// Window spectra of every used slot (and segment, cs->seg_lags).  slot_ready
// (optional) receives, per forward-transform wave, (spectrum slots complete,
// event on the context stream) so that correlations of early slots can start
// while later slots transform.  Spectrum slot of (slot s, segment g) =
// s * n_segments + g.
void ensure_dspec(tdg_ctx* ctx, tdg_windows* w, const tdg_codeset* cs,
                  std::vector<std::pair<size_t, cudaEvent_t>>* slot_ready = nullptr) {
    const int N1 = cs->N1, N2 = cs->N2;
    const uint64_t N = uint64_t(N1) * uint64_t(N2);
    const uint64_t seg_key = cs->seg_lags ? cs->seg_lags * (uint64_t(1) << 24) + cs->nmax : 0;
    if (w->dspec_N == N && w->dspec_seg == seg_key) return;
    const uint64_t H = uint64_t(N1 / 2 + 1) * uint64_t(N2);
    const uint64_t nseg = cs->n_segments(w->W), nss = w->used() * nseg;
    w->dspec.ensure(w->slots() * nseg * H * sizeof(float2));
    auto seq = [&](uint64_t ss, const float** r, uint64_t* len) {
        const uint64_t s = ss / nseg, g = ss % nseg;
        const uint64_t o = g * cs->seg_lags;
        *r = w->d.as<float>() + s * w->W + o;
        *len = cs->seg_lags ? std::min(w->W - o, cs->seg_lags + cs->nmax - 1) : w->W;
    };
    std::vector<FwdJob> jobs;
    for (uint64_t ss = 0; ss < nss; ss += 2) {
        const bool two = ss + 1 < nss;
        const float *r1 = nullptr, *r2 = nullptr;
        uint64_t l1 = 0, l2 = 0;
        seq(ss, &r1, &l1);
        if (two) seq(ss + 1, &r2, &l2);
        jobs.push_back({r1, r2, l1, l2, w->dspec.as<float2>() + ss * H, two ? w->dspec.as<float2>() + (ss + 1) * H : nullptr});
    }
    run_forward(ctx, N1, N2, jobs, true, slot_ready);
    if (slot_ready)
        for (auto& c : *slot_ready) c.first = std::min<size_t>(2 * c.first, nss);   // pair jobs -> spectrum slots
    w->dspec_N = N;
    w->dspec_seg = seg_key;
}

// Correlation jobs: each is one stored code pair (codes 2p, 2p+1) against
// one window slot; outputs are argmax keys and/or full xc rows.
struct CorrJob {
    uint64_t slot;               // spectrum slot (window slot * n_segments + segment)
    uint64_t pair;
    unsigned long long* key_a;
    unsigned long long* key_b;   // nullptr if the pair has one code
    float* xc_a;                 // diagnostic outputs (nullable), at the segment's first lag
    float* xc_b;
    uint32_t lag0 = 0;           // global lag of the segment's local lag 0
    uint32_t lag_lim = 0;        // local lags [0, lag_lim); 0 = the window length
};

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda)
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q{};
        void* p = nullptr;
        CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
        if (q != cudaDriverEntryPointSuccess || !p) fail(TDG_ECUDA, "cuTensorMapEncodeTiled unavailable");
        fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

// The M ring as a 4-D fp32 tensor [pair][tile t2/4][k1][t2%4 as 8 floats]:
// one pass-A TMA store writes a whole column k1 (box 8 x 1 x n_tiles x 1).
CUtensorMap m_store_map(float2* M, int N1, int n_tiles, uint64_t Mstride, int n_pairs) {
    CUtensorMap map;
    const cuuint64_t dims[4] = {8, cuuint64_t(N1), cuuint64_t(n_tiles), cuuint64_t(n_pairs)};
    const cuuint64_t strides[3] = {32, cuuint64_t(N1) * 32, Mstride * 8};
    const cuuint32_t box[4] = {8, 1, cuuint32_t(n_tiles), 1};
    const cuuint32_t estr[4] = {1, 1, 1, 1};
    if (n_tiles > 256) fail(TDG_ERANGE, "M tile count %d exceeds a TMA box", n_tiles);
    const CUresult r = tensor_map_encoder()(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, M, dims, strides, box, estr,
                                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                            CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) fail(TDG_ECUDA, "cuTensorMapEncodeTiled failed (%d)", int(r));
    return map;
}

// statistics (k_stats): one CTA per (slot, code) when there are enough of
// them to fill the GPU, else each dot product split over several CTAs
void launch_stats(tdg_ctx* ctx, const tdg::StatsDesc* sd, size_t n, uint32_t W, double fs, float threshold) {
    if (!n) return;
    const size_t want = size_t(num_sms()) * 8;
    int splits = n >= want ? 1 : int(std::min<size_t>(256, (want + n - 1) / n));
    double* partial = nullptr;
    unsigned* counters = nullptr;
    if (splits > 1) {
        ctx->stats_part.ensure(n * size_t(splits) * 5 * sizeof(double));
        if (ctx->stats_ctr.bytes < n * sizeof(unsigned)) {
            ctx->stats_ctr.ensure(n * sizeof(unsigned));
            if (STREAM_OPS) CK(cudaMemsetAsync(ctx->stats_ctr.p, 0, ctx->stats_ctr.bytes, ctx->stream));
        }
        partial = ctx->stats_part.as<double>();
        counters = ctx->stats_ctr.as<unsigned>();
    }
    KScope ks(ctx, "stats");
    if (STREAM_OPS) {
        if (splits > 1)
            tdg::k_stats<true><<<unsigned(n * size_t(splits)), 256, 0, ctx->stream>>>(sd, W, fs, threshold, splits,
                                                                                 partial, counters);
        else
            tdg::k_stats<false><<<unsigned(n), 256, 0, ctx->stream>>>(sd, W, fs, threshold, 1, nullptr, nullptr);
    }
    LAUNCHED();
}

// Waves of wave_pairs pairs; wave w's pass A on A-stream w % n_streams and its
// pass B on B-stream w % n_streams, M in a ring of `ring` wave buffers: B(w)
// waits for A(w), A(w) waits for B(w - ring).  Passes of neighbouring waves
// thus overlap and no kernel's ramp or tail leaves SMs idle.  One wave
// (small tracking batches) runs on the context stream without events.
void run_correlations(tdg_ctx* ctx, tdg_windows* w, const tdg_codeset* cs, const std::vector<CorrJob>& jobs,
                      bool write_xc) {
    if (jobs.empty()) return;
    const int N1 = cs->N1, N2 = cs->N2;
    const uint64_t N = cs->corr_len(), H = cs->H;
    // allocate the window spectra now (their addresses go into the
    // descriptors); the transforms themselves are enqueued after the fork
    w->dspec.ensure(w->slots() * cs->n_segments(w->W) * H * sizeof(float2));
    constexpr int G = tdg::kGroup;
    const int wave = int(std::max<int64_t>(G, ctx->wave_pairs / G * G));
    const int n_waves = int((jobs.size() + size_t(wave) - 1) / size_t(wave));
    const int ring = int(std::max<int64_t>(1, std::min<int64_t>(ctx->ring, n_waves)));
    const int n_tiles = (N2 + tdg::kTileB - 1) / tdg::kTileB;
    const uint64_t Mstride = uint64_t(n_tiles) * uint64_t(N1) * tdg::kTileB;   // tile-major M per pair
    ctx->M.ensure(size_t(ring) * size_t(wave) * Mstride * sizeof(float2));
    // groups: consecutive jobs of a wave that share a window spectrum, <= G each
    std::vector<std::vector<tdg::CorrGroup<G>>> wg(static_cast<size_t>(n_waves));
    int ngw = 1;
    for (int wv = 0; wv < n_waves; ++wv) {
        auto& gs = wg[size_t(wv)];
        for (int i = 0; i < wave && size_t(wv) * wave + i < jobs.size(); ++i) {
            const CorrJob& jb = jobs[size_t(wv) * wave + size_t(i)];
            const float2* D = w->dspec.as<float2>() + jb.slot * H;
            if (gs.empty() || gs.back().npairs == G || gs.back().D != D) {
                tdg::CorrGroup<G> g{};
                g.D = D;
                gs.push_back(g);
            }
            auto& g = gs.back();
            g.Ca[g.npairs] = cs->spec.as<float2>() + jb.pair * N;
            g.Cb[g.npairs] = nullptr;
            g.M[g.npairs] = ctx->M.as<float2>() + (size_t(wv % ring) * wave + size_t(i)) * Mstride;
            g.Mi[g.npairs] = (wv % ring) * wave + i;
            ++g.npairs;
        }
        ngw = std::max(ngw, int(gs.size()));
    }
    std::vector<tdg::CorrGroup<G>> groups(size_t(n_waves) * ngw);   // npairs 0 = no-op item
    std::vector<tdg::CorrPairOut> outs(size_t(n_waves) * wave);     // M null = no-op item
    for (int wv = 0; wv < n_waves; ++wv) {
        for (size_t g = 0; g < wg[size_t(wv)].size(); ++g) groups[size_t(wv) * ngw + g] = wg[size_t(wv)][g];
        for (int i = 0; i < wave && size_t(wv) * wave + i < jobs.size(); ++i) {
            const CorrJob& jb = jobs[size_t(wv) * wave + size_t(i)];
            auto& o = outs[size_t(wv) * wave + size_t(i)];
            o.M = ctx->M.as<float2>() + (size_t(wv % ring) * wave + size_t(i)) * Mstride;
            o.key_a = jb.key_a;
            o.key_b = jb.key_b;
            o.xc_a = jb.xc_a;
            o.xc_b = jb.xc_b;
            o.lag0 = jb.lag0;
            o.lag_lim = jb.lag_lim ? jb.lag_lim : uint32_t(w->W);
        }
    }
    ctx->pk->corr.begin();
    const size_t og = ctx->pk->corr.add(groups);
    const size_t oo = ctx->pk->corr.add(outs);
    ctx->pk->corr.commit(ctx->stream);
    tdg::CorrSched S{};
    S.mstore = m_store_map(ctx->M.as<float2>(), N1, n_tiles, Mstride, ring * wave);
    S.twA = ctx->twiddles(N2);
    S.twB = ctx->twiddles(N1);
    S.twI = ctx->inter_twiddles(N1, N2);
    S.ngw = ngw;
    S.wave_pairs = wave;
    S.n_tiles = n_tiles;
    S.nA = (N1 / 2 + 1) * ngw;
    S.nB = wave * n_tiles;
    S.N1 = N1;
    S.N2 = N2;
    S.write_xc = write_xc ? 1 : 0;
    S.discard = ctx->discard ? 1 : 0;
    if (ctx->trace_cap && !tl_graph_mode) {
        S.trace = reinterpret_cast<unsigned long long*>(ctx->trace.as<unsigned char>() + 16);
        S.trace_n = ctx->trace.as<unsigned int>();
        S.trace_cap = ctx->trace_cap;
    }
    S.W = uint32_t(w->W);
    S.inv_n = 1.0f / float(N);
    auto* gd = ctx->pk->corr.at<tdg::CorrGroup<G>>(og);
    auto* od = ctx->pk->corr.at<tdg::CorrPairOut>(oo);
    if (n_waves == 1) {
        // one wave (small tracking batches): nothing to overlap, so no fork,
        // events or join -- the transforms and both passes in order on the
        // context stream (API calls are most of a small batch's latency)
        ensure_dspec(ctx, w, cs);
        S.groups = gd;
        S.outs = od;
        launch_pass<0>(N1, N2, ctx->stream, S, ctx->cta_cap[0]);
        launch_pass<1>(N1, N2, ctx->stream, S, ctx->cta_cap[1]);
        return;
    }
    ctx->ensure_pipeline(ring);
    // waves alternate over n_streams pass-A and n_streams pass-B streams; more
    // launches in flight let the latency-bound passes of neighbouring waves
    // share the SMs.  The window spectra are transformed on the context stream
    // after the fork, wave by wave, and a pass-A launch only waits for the
    // transform wave that completes the slots it reads.
    const int ns = int(ctx->a_streams.size());
    CK(cudaEventRecord(ctx->ev_fork, ctx->stream));
    for (int i = 0; i < ns; ++i) {
        CK(cudaStreamWaitEvent(ctx->a_streams[size_t(i)], ctx->ev_fork, 0));
        CK(cudaStreamWaitEvent(ctx->b_streams[size_t(i)], ctx->ev_fork, 0));
    }
    std::vector<std::pair<size_t, cudaEvent_t>> ready;   // (slots transformed, event)
    ensure_dspec(ctx, w, cs, &ready);
    std::vector<size_t> waited(size_t(ns), 0);            // ready[] prefix each A stream has waited for
    for (int wv = 0; wv < n_waves; ++wv) {
        const int r = wv % ring;
        cudaStream_t sa = ctx->a_streams[size_t(wv % ns)];
        S.groups = gd + size_t(wv) * ngw;
        S.outs = od + size_t(wv) * wave;
        uint64_t top = 0;
        for (int i = 0; i < wave && size_t(wv) * wave + i < jobs.size(); ++i)
            top = std::max(top, jobs[size_t(wv) * wave + size_t(i)].slot + 1);
        size_t& wt = waited[size_t(wv % ns)];
        while (wt < ready.size() && (wt == 0 || ready[wt - 1].first < top)) {
            CK(cudaStreamWaitEvent(sa, ready[wt].second, 0));
            ++wt;
        }
        if (wv >= ring) CK(cudaStreamWaitEvent(sa, ctx->ev_b[size_t(r)], 0));
        launch_pass<0>(N1, N2, sa, S, ctx->cta_cap[0]);
        CK(cudaEventRecord(ctx->ev_a[size_t(r)], sa));
        cudaStream_t sb = ctx->one_stream ? sa : ctx->b_streams[size_t(wv % ns)];
        CK(cudaStreamWaitEvent(sb, ctx->ev_a[size_t(r)], 0));
        launch_pass<1>(N1, N2, sb, S, ctx->cta_cap[1]);
        CK(cudaEventRecord(ctx->ev_b[size_t(r)], sb));
    }
    for (int i = 0; i < ns; ++i)
        for (cudaStream_t x : {ctx->a_streams[size_t(i)], ctx->b_streams[size_t(i)]}) {
            CK(cudaEventRecord(ctx->ev_join, x));
            CK(cudaStreamWaitEvent(ctx->stream, ctx->ev_join, 0));
        }
}

}  // namespace

// ===========================================================================
extern "C" {

const char* tdg_last_error(void) { return g_err.c_str(); }
const char* tdg_version(void) { return "tagdsp_gpu 0.1 (sm_100a)"; }
uint64_t tdg_kernel_launches(void) { return g_launches.load(); }

int tdg_ctx_create(int device, tdg_ctx** out) {
    return guard([&] {
        *out = nullptr;
        CK(cudaSetDevice(device));
        auto ctx = std::make_unique<tdg_ctx>();
        ctx->device = device;
        CK(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
        *out = ctx.release();
    });
}

void tdg_ctx_destroy(tdg_ctx* ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    for (auto& k : ctx->ktimes) {
        cudaEventDestroy(k.a);
        cudaEventDestroy(k.b);
    }
    for (auto e : ctx->ev_pool) cudaEventDestroy(e);
    if (ctx->search_win) tdg_windows_destroy(ctx->search_win);
    if (ctx->track_win) tdg_windows_destroy(ctx->track_win);
    for (auto e : ctx->ev_a) cudaEventDestroy(e);
    for (auto e : ctx->ev_b) cudaEventDestroy(e);
    if (ctx->ev_fork) cudaEventDestroy(ctx->ev_fork);
    if (ctx->ev_join) cudaEventDestroy(ctx->ev_join);
    for (auto x : ctx->a_streams) cudaStreamDestroy(x);
    for (auto x : ctx->b_streams) cudaStreamDestroy(x);
    for (auto e : ctx->ev_fwd) cudaEventDestroy(e);
    for (auto e : ctx->dt_ev)
        if (e) cudaEventDestroy(e);
    cudaStreamDestroy(ctx->stream);
    delete ctx;
}

int tdg_ctx_synchronize(tdg_ctx* ctx) {
    return guard([&] { CK(cudaStreamSynchronize(ctx->stream)); });
}

void* tdg_ctx_stream(tdg_ctx* ctx) { return ctx ? static_cast<void*>(ctx->stream) : nullptr; }

uint64_t tdg_pad_length(uint64_t n) {
    uint64_t r = 0;
    if (guard([&] { r = pad_length_impl(n); })) return 0;
    return r;
}

uint64_t tdg_corr_len(uint64_t window_len, uint64_t nonzero_len) {
    int n1, n2;
    const uint64_t need = std::max<uint64_t>(1, window_len + nonzero_len - (nonzero_len ? 1 : 0));
    if (!choose_corr_len(need, &n1, &n2)) return 0;
    return uint64_t(n1) * uint64_t(n2);
}

int tdg_kernel_time(tdg_ctx* ctx, const char* name, uint64_t* count, double* total_ms) {
    return guard([&] {
        ctx->collect();
        auto it = ctx->kstats.find(name);
        *count = it == ctx->kstats.end() ? 0 : it->second.first;
        *total_ms = it == ctx->kstats.end() ? 0.0 : it->second.second;
    });
}

int tdg_cta_trace(tdg_ctx* ctx, uint64_t* out, uint64_t cap, uint64_t* n) {
    return guard([&] {
        CK(cudaSetDevice(ctx->device));
        CK(cudaStreamSynchronize(ctx->stream));
        CK(cudaDeviceSynchronize());
        uint32_t cnt = 0;
        if (ctx->trace_cap) {
            CK(cudaMemcpy(&cnt, ctx->trace.p, sizeof(cnt), cudaMemcpyDeviceToHost));
            cnt = std::min(cnt, ctx->trace_cap);
            const uint64_t m = std::min<uint64_t>(cnt, cap);
            if (out && m)
                CK(cudaMemcpy(out, ctx->trace.as<unsigned char>() + 16, m * 24, cudaMemcpyDeviceToHost));
            CK(cudaMemset(ctx->trace.p, 0, 16));
        }
        if (n) *n = cnt;
    });
}

int tdg_kernel_time_reset(tdg_ctx* ctx) {
    return guard([&] {
        ctx->collect();
        ctx->kstats.clear();
    });
}

int tdg_set_option(tdg_ctx* ctx, const char* key, int64_t value) {
    return guard([&] {
        std::string k(key);
        ctx->track_graphs.clear();   // captured launch configurations may change
        if (k == "time_kernels") {
            ctx->collect();
            ctx->time_kernels = value != 0;
        } else if (k == "wave_pairs")
            ctx->wave_pairs = value > 0 ? value : 8;
        else if (k == "n_streams") {
            CK(cudaDeviceSynchronize());
            for (auto x : ctx->a_streams) CK(cudaStreamDestroy(x));
            for (auto x : ctx->b_streams) CK(cudaStreamDestroy(x));
            ctx->a_streams.clear();
            ctx->b_streams.clear();
            ctx->n_streams = value > 0 ? value : 6;
        } else if (k == "cta_cap_a")
            ctx->cta_cap[0] = int(value);
        else if (k == "cta_cap_b")
            ctx->cta_cap[1] = int(value);
        else if (k == "one_stream")
            ctx->one_stream = value;
        else if (k == "discard")
            ctx->discard = value;
        else if (k == "ring")
            ctx->ring = value > 0 ? value : 3;
        else if (k == "track_graphs")
            ctx->track_graphs_on = value != 0;
        else if (k == "fwd_wave")
            ctx->fwd_wave = value > 0 ? value : 32;
        else if (k == "cta_trace") {
            ctx->trace_cap = uint32_t(std::max<int64_t>(0, value));
            if (ctx->trace_cap) {
                ctx->trace.ensure(size_t(ctx->trace_cap) * 24 + 16);
                CK(cudaMemsetAsync(ctx->trace.p, 0, size_t(ctx->trace_cap) * 24 + 16, ctx->stream));
            }
        }
        else if (k == "detect_timings")
            ctx->detect_timings = value != 0;
        else
            fail(TDG_EINVAL, "unknown option %s", key);
    });
}

// ---- code sets -------------------------------------------------------------
namespace {

// grow a device buffer to `bytes`, keeping its first `keep` bytes
void grow_keep(tdg_ctx* ctx, DevBuf& buf, size_t bytes, size_t keep) {
    if (bytes <= buf.bytes) return;
    DevBuf nb;
    nb.ensure(bytes);
    if (keep) CK(cudaMemcpyAsync(nb.p, buf.p, keep, cudaMemcpyDeviceToDevice, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    std::swap(nb.p, buf.p);
    std::swap(nb.bytes, buf.bytes);
}

// Append n codes to cs from their demodulated replicas (d, u at `stride`,
// lens[i] samples each): support n, energy and abs_sum (make_transformed,
// proj/src/detector.cpp:20-43), then the forward transforms of every stored
// pair the new codes touch -- or of all pairs if the longer support needs a
// longer transform.  Device buffers grow by doubling, so a roster built one
// prepare_code at a time costs O(C) transforms, not O(C^2).
void append_codes(tdg_ctx* ctx, tdg_codeset* cs, const float* d, const float* u, uint64_t stride,
                  const std::vector<uint64_t>& lens, uint64_t ref_corr_len) {
    const uint64_t n0 = cs->n_codes, n = lens.size(), nt = n0 + n;
    uint64_t rc = 0;
    for (uint64_t l : lens) rc = std::max(rc, l);
    rc = (std::max<uint64_t>(rc, 1) + 3) & ~uint64_t(3);   // 16-byte rows (stats vector loads)
    if (n0 && rc > cs->rep_cap) fail(TDG_EINVAL, "prepare_code: replica longer than the code set's stride");
    if (!n0) cs->rep_cap = rc;
    if (nt > cs->cap_codes) {
        const uint64_t cap = std::max<uint64_t>(nt, n0 ? 2 * cs->cap_codes : nt);
        grow_keep(ctx, cs->rep, cap * cs->rep_cap * sizeof(float), n0 * cs->rep_cap * sizeof(float));
        grow_keep(ctx, cs->nlen_dev, cap * sizeof(uint64_t), n0 * sizeof(uint64_t));
        grow_keep(ctx, cs->energy_dev, cap * sizeof(float), n0 * sizeof(float));
        grow_keep(ctx, cs->abs_dev, cap * sizeof(float), n0 * sizeof(float));
        cs->cap_codes = cap;
    }
    std::vector<tdg::SupportDesc> sd(n);
    for (uint64_t i = 0; i < n; ++i) {
        const uint64_t c = n0 + i;
        sd[i] = {d + i * stride, u ? u + i * stride : nullptr, lens[i], cs->rep.as<float>() + c * cs->rep_cap,
                 cs->rep_cap, cs->nlen_dev.as<uint64_t>() + c, cs->energy_dev.as<float>() + c,
                 cs->abs_dev.as<float>() + c};
    }
    auto* sdd = ctx->upload(ctx->pk->stats, sd);
    tdg::k_support<<<unsigned(n), 1024, 0, ctx->stream>>>(sdd);
    LAUNCHED();
    cs->nlen.resize(nt);
    cs->energy.resize(nt);
    cs->abs_sum.resize(nt);
    CK(cudaMemcpyAsync(cs->nlen.data() + n0, cs->nlen_dev.as<uint64_t>() + n0, n * sizeof(uint64_t),
                       cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaMemcpyAsync(cs->energy.data() + n0, cs->energy_dev.as<float>() + n0, n * sizeof(float),
                       cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaMemcpyAsync(cs->abs_sum.data() + n0, cs->abs_dev.as<float>() + n0, n * sizeof(float),
                       cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    uint64_t nmax = 1;
    for (uint64_t i = 0; i < nt; ++i) {
        // make_transformed precondition (proj/src/detector.cpp:28-29)
        if (i >= n0 && cs->window_len + cs->nlen[i] > ref_corr_len + 1) {
            cs->nlen.resize(n0);
            cs->energy.resize(n0);
            cs->abs_sum.resize(n0);
            fail(TDG_EINVAL, "make_transformed: transform too short for linear correlation");
        }
        nmax = std::max(nmax, cs->nlen[i]);
    }
    if (cs->window_len >= (uint64_t(1) << 32)) fail(TDG_ERANGE, "window_len too large");
    int N1 = 0, N2 = 0;
    uint64_t seg_lags = 0;
    if (!choose_corr_len(cs->window_len + nmax - 1, &N1, &N2)) {
        // longer than one transform: segmented correlation with the largest
        // split, each segment's lags [gB, gB + B) from B + nmax - 1 samples
        N1 = N2 = 1024;
        const uint64_t Nmax = uint64_t(N1) * uint64_t(N2);
        if (nmax > Nmax / 2) {
            cs->nlen.resize(n0);
            cs->energy.resize(n0);
            cs->abs_sum.resize(n0);
            fail(TDG_ERANGE, "code support %llu exceeds half of the largest transform", (unsigned long long)nmax);
        }
        seg_lags = Nmax - nmax + 1;
    }
    cs->n_codes = nt;
    cs->seg_lags = seg_lags;
    cs->nmax = nmax;
    const bool relen = N1 != cs->N1 || N2 != cs->N2;
    cs->N1 = N1;
    cs->N2 = N2;
    cs->H = uint64_t(N1 / 2 + 1) * uint64_t(N2);
    const uint64_t N = cs->corr_len();
    const uint64_t npairs = (nt + 1) / 2, pcap = (cs->cap_codes + 1) / 2;
    const uint64_t first_pair = relen ? 0 : n0 / 2;
    if (relen) {
        cs->spec.release();
        cs->spec.ensure(pcap * N * sizeof(float2));
    } else {
        grow_keep(ctx, cs->spec, pcap * N * sizeof(float2), first_pair * N * sizeof(float2));
    }
    std::vector<FwdJob> jobs;
    for (uint64_t p = first_pair; p < npairs; ++p) {
        const uint64_t i = 2 * p;
        const bool two = i + 1 < nt;
        jobs.push_back({cs->rep.as<float>() + i * cs->rep_cap, two ? cs->rep.as<float>() + (i + 1) * cs->rep_cap : nullptr,
                        cs->nlen[i], two ? cs->nlen[i + 1] : 0, cs->spec.as<float2>() + p * N, nullptr});
    }
    run_forward(ctx, cs->N1, cs->N2, jobs, false);
    CK(cudaStreamSynchronize(ctx->stream));
}

void demod_launch(tdg_ctx* ctx, const void* in, bool int16_input, uint64_t in_len,
                  const std::vector<tdg::DemodWindowDesc>& wins, uint64_t W, int n_bins, uint64_t slot_stride,
                  const float2* H, float eps, uint64_t ring_cap = 0) {
    if (W == 0 || wins.empty()) return;
    const int V = 1024 - (ctx->clen - 1);
    const uint64_t nblocks = (W + uint64_t(V) - 1) / uint64_t(V);
    const float2* tw = ctx->twiddles(1024);
    auto* wd = ctx->upload(ctx->pk->misc, wins);
    KScope ks(ctx, "demod");
    // launches that leave the SMs mostly idle take the two-warps-per-block
    // variant (shorter per-warp chain, one more forward transform per block)
    const bool split = nblocks * wins.size() * 2 <= uint64_t(num_sms()) * 12;
    auto go = [&](auto kern, int nblk, int warps_per_blk, const auto* src) {
        dim3 grid(unsigned((nblocks + uint64_t(nblk) - 1) / uint64_t(nblk)), unsigned(wins.size()));
        const size_t sm = size_t(nblk * warps_per_blk) * (32 * 33) * sizeof(float2) + size_t(nblk) * 1024 * sizeof(float);
        set_smem(kern, sm);
        if (STREAM_OPS)
            kern<<<grid, nblk * warps_per_blk * 32, sm, ctx->stream>>>(src, in_len, wd, uint32_t(W), ctx->clen, n_bins,
                                                                      slot_stride, H, eps, tw, ring_cap);
    };
    if (int16_input) {
        const auto* src = static_cast<const int32_t*>(in);
        if (split) go(tdg::k_demod<int32_t, 2, true>, 2, 2, src);
        else go(tdg::k_demod<int32_t, kDemodBlk>, kDemodBlk, 1, src);
    } else {
        const auto* src = static_cast<const float2*>(in);
        if (split) go(tdg::k_demod<float2, 2, true>, 2, 2, src);
        else go(tdg::k_demod<float2, kDemodBlk>, kDemodBlk, 1, src);
    }
    LAUNCHED();
}

}  // namespace

namespace {
std::vector<double> cfg_key_of(const tdg_demod_config& c) {
    return {c.mod.sample_rate, c.mod.bit_rate, c.mod.freq_one, c.mod.freq_zero, double(c.mod.packet_bits),
            c.bandpass_center, c.bandpass_width, double(c.bandpass_taps), double(c.eps)};
}

// prepare_code (proj/src/detector.cpp:50-66) for n codes, appended to cs:
// synth_replica -> demodulation with lo_freq = 0 -> support / energy ->
// forward transforms of the touched pairs, all on the GPU
void prepare_codes(tdg_ctx* ctx, tdg_codeset* cs, const tdg_demod_config& c, const uint8_t* bits, uint64_t n_codes) {
    validate_cfg(c);
    const uint64_t spb = samples_per_bit(c.mod);
    const uint64_t nbits = c.mod.packet_bits;
    const uint64_t psamp = nbits * spb;
    const uint64_t window_len = cs->window_len;
    if (window_len < psamp) fail(TDG_EINVAL, "prepare_code: window shorter than a packet");
    if (n_codes == 0) fail(TDG_EINVAL, "prepare_code: no codes");
    const std::vector<double> key = cfg_key_of(c);
    if (cs->n_codes && cs->cfg_key != key)
        fail(TDG_EINVAL, "prepare_code: the code set was prepared with another configuration");
    cs->cfg_key = key;
    const uint64_t clen_ref = c.bandpass_taps + spb - 1;
    cs->ref_corr = pad_length_impl(window_len + psamp + clen_ref);
    // filters for lo = 0 (replicas skip the local oscillator, proj/src/detector.cpp:59-61)
    const float2* H = ctx->filter_spectra(c, std::vector<double>{0.0});
    // replica demod span: the packet plus the filter tail plus one block of margin
    const uint64_t Wr = std::min<uint64_t>(window_len, psamp + uint64_t(ctx->clen) + 1024);
    DevBuf dbits, drep, dd, du;
    dbits.ensure(n_codes * nbits);
    CK(cudaMemcpyAsync(dbits.p, bits, n_codes * nbits, cudaMemcpyHostToDevice, ctx->stream));
    drep.ensure(n_codes * Wr * sizeof(float2));
    const double pi = 3.14159265358979323846;
    const double step1 = 2.0 * pi * c.mod.freq_one / c.mod.sample_rate;
    const double step0 = 2.0 * pi * c.mod.freq_zero / c.mod.sample_rate;
    tdg::k_synth_replica<<<unsigned(n_codes), 1024, nbits * sizeof(uint32_t), ctx->stream>>>(
        dbits.as<uint8_t>(), uint32_t(nbits), uint32_t(spb), step1, step0, drep.as<float2>(), Wr);
    LAUNCHED();
    dd.ensure(n_codes * Wr * sizeof(float));
    du.ensure(n_codes * Wr * sizeof(float));
    std::vector<tdg::DemodWindowDesc> wins(n_codes);
    for (uint64_t i = 0; i < n_codes; ++i) wins[i] = {i * Wr, dd.as<float>() + i * Wr, du.as<float>() + i * Wr};
    demod_launch(ctx, drep.p, false, n_codes * Wr, wins, Wr, 1, Wr, H, c.eps);
    std::vector<uint64_t> lens(n_codes, Wr);
    append_codes(ctx, cs, dd.as<float>(), du.as<float>(), Wr, lens, cs->ref_corr);
}
}  // namespace

int tdg_codeset_prepare(tdg_ctx* ctx, const tdg_demod_config* cfg, uint64_t window_len, const uint8_t* bits,
                        uint64_t n_codes, tdg_codeset** out) {
    return guard([&] {
        *out = nullptr;
        CK(cudaSetDevice(ctx->device));
        auto cs = std::make_unique<tdg_codeset>();
        cs->ctx = ctx;
        cs->device = ctx->device;
        cs->window_len = window_len;
        prepare_codes(ctx, cs.get(), *cfg, bits, n_codes);
        *out = cs.release();
    });
}

int tdg_codeset_append(tdg_ctx* ctx, tdg_codeset* cs, const tdg_demod_config* cfg, const uint8_t* bits,
                       uint64_t n_codes) {
    return guard([&] {
        CK(cudaSetDevice(ctx->device));
        if (cs->device != ctx->device) fail(TDG_EINVAL, "prepare_code: code set on another device");
        if (cs->n_codes && cs->cfg_key.empty())
            fail(TDG_EINVAL, "prepare_code: cannot append prepared codes to a make_transformed code set");
        prepare_codes(ctx, cs, *cfg, bits, n_codes);
    });
}

int tdg_codeset_from_replicas(tdg_ctx* ctx, uint64_t window_len, uint64_t corr_len, const float* const* replica_d,
                              const float* const* replica_u, const uint64_t* lengths, uint64_t n_codes,
                              tdg_codeset** out) {
    return guard([&] {
        *out = nullptr;
        CK(cudaSetDevice(ctx->device));
        if (n_codes == 0) fail(TDG_EINVAL, "make_transformed: no codes");
        uint64_t stride = 1;
        for (uint64_t i = 0; i < n_codes; ++i) stride = std::max(stride, lengths[i]);
        std::vector<float> hd(n_codes * stride, 0.f), hu;
        const bool have_u = replica_u != nullptr;
        if (have_u) hu.assign(n_codes * stride, 0.f);
        std::vector<uint64_t> lens(n_codes);
        for (uint64_t i = 0; i < n_codes; ++i) {
            lens[i] = lengths[i];
            std::memcpy(hd.data() + i * stride, replica_d[i], lengths[i] * sizeof(float));
            if (have_u && replica_u[i]) std::memcpy(hu.data() + i * stride, replica_u[i], lengths[i] * sizeof(float));
            else if (have_u) std::memcpy(hu.data() + i * stride, replica_d[i], lengths[i] * sizeof(float));
        }
        auto cs = std::make_unique<tdg_codeset>();
        cs->ctx = ctx;
        cs->device = ctx->device;
        cs->window_len = window_len;
        cs->ref_corr = corr_len;
        DevBuf dd, du;
        dd.ensure(hd.size() * sizeof(float));
        CK(cudaMemcpyAsync(dd.p, hd.data(), hd.size() * sizeof(float), cudaMemcpyHostToDevice, ctx->stream));
        if (have_u) {
            du.ensure(hu.size() * sizeof(float));
            CK(cudaMemcpyAsync(du.p, hu.data(), hu.size() * sizeof(float), cudaMemcpyHostToDevice, ctx->stream));
        }
        append_codes(ctx, cs.get(), dd.as<float>(), have_u ? du.as<float>() : nullptr, stride, lens, corr_len);
        *out = cs.release();
    });
}

void tdg_codeset_destroy(tdg_codeset* cs) {
    if (!cs) return;
    cudaSetDevice(cs->device);   // cudaFree in the buffers' destructors synchronises
    delete cs;
}

uint64_t tdg_codeset_size(const tdg_codeset* cs) { return cs ? cs->n_codes : 0; }

int tdg_codeset_info(const tdg_codeset* cs, uint64_t idx, uint64_t* nonzero_len, float* energy, float* abs_sum,
                     uint64_t* corr_len) {
    return guard([&] {
        if (idx >= cs->n_codes) fail(TDG_EINVAL, "code index out of range");
        if (nonzero_len) *nonzero_len = cs->nlen[idx];
        if (energy) *energy = cs->energy[idx];
        if (abs_sum) *abs_sum = cs->abs_sum[idx];
        if (corr_len) *corr_len = cs->corr_len();
    });
}

int tdg_codeset_replica(const tdg_codeset* cs, uint64_t idx, float* replica_d_out) {
    return guard([&] {
        if (idx >= cs->n_codes) fail(TDG_EINVAL, "code index out of range");
        CK(cudaSetDevice(cs->device));
        CK(cudaDeviceSynchronize());
        CK(cudaMemcpy(replica_d_out, cs->rep.as<float>() + idx * cs->rep_cap, cs->nlen[idx] * sizeof(float),
                      cudaMemcpyDeviceToHost));
    });
}

// ---- windows ---------------------------------------------------------------
int tdg_windows_create(tdg_ctx* ctx, uint64_t window_len, uint64_t n_windows, uint64_t n_bins, tdg_windows** out) {
    return guard([&] {
        *out = nullptr;
        CK(cudaSetDevice(ctx->device));
        if (window_len == 0 || n_windows == 0 || n_bins == 0) fail(TDG_EINVAL, "windows: empty shape");
        if (window_len >= (uint64_t(1) << 32)) fail(TDG_ERANGE, "window_len too large");
        auto w = std::make_unique<tdg_windows>();
        w->ctx = ctx;
        w->device = ctx->device;
        w->W = window_len;
        w->n_windows = n_windows;
        w->n_bins = n_bins;
        w->d.ensure(w->slots() * window_len * sizeof(float));
        w->u.ensure(w->slots() * window_len * sizeof(float));
        CK(cudaMemsetAsync(w->d.p, 0, w->d.bytes, ctx->stream));
        CK(cudaMemsetAsync(w->u.p, 0, w->u.bytes, ctx->stream));
        w->start.assign(w->slots(), 0);
        *out = w.release();
    });
}

void tdg_windows_destroy(tdg_windows* w) {
    if (!w) return;
    cudaSetDevice(w->device);
    delete w;
}

namespace {
void SampleSource::before_read(tdg_ctx* ctx) const {
    if (ring) CK(cudaStreamWaitEvent(ctx->stream, ring->pushed, 0));
}
void SampleSource::after_read(tdg_ctx* ctx, int64_t s, int64_t e) const {
    if (!ring) return;
    cudaEvent_t ev = ring->event();
    CK(cudaEventRecord(ev, ctx->stream));
    ring->reads.push_back({s, e, ev});
}

void demodulate_impl(tdg_ctx* ctx, tdg_windows* win, const tdg_demod_config* cfg, const double* lo_bins,
                     uint64_t n_bins, const SampleSource& src, int64_t first_start, uint64_t advance,
                     uint64_t n_windows) {
    if (n_bins != win->n_bins) fail(TDG_EINVAL, "demodulate: bin count %llu != window set's %llu",
                                    (unsigned long long)n_bins, (unsigned long long)win->n_bins);
    if (n_windows > win->n_windows) fail(TDG_EINVAL, "demodulate: too many windows");
    if (n_windows && !src.holds(first_start, (n_windows - 1) * advance + win->W))
        fail(TDG_EINVAL, "demodulate: windows exceed the sample block");
    std::vector<double> bins(lo_bins, lo_bins + n_bins);
    const float2* H = ctx->filter_spectra(*cfg, bins);
    std::vector<tdg::DemodWindowDesc> wins(n_windows);
    for (uint64_t w = 0; w < n_windows; ++w) {
        const uint64_t slot0 = w * n_bins;
        const int64_t st = first_start + int64_t(w * advance);
        wins[w] = {src.offset(st), win->d.as<float>() + slot0 * win->W, win->u.as<float>() + slot0 * win->W};
        for (uint64_t b = 0; b < n_bins; ++b) win->start[slot0 + b] = st;
    }
    src.before_read(ctx);
    demod_launch(ctx, src.base, true, src.len, wins, win->W, int(n_bins), win->W, H, cfg->eps, src.ring_cap);
    if (n_windows) src.after_read(ctx, first_start, first_start + int64_t((n_windows - 1) * advance + win->W));
    win->dspec_N = 0;
}
}  // namespace

int tdg_demodulate_device(tdg_ctx* ctx, tdg_windows* win, const tdg_demod_config* cfg, const double* lo_bins,
                          uint64_t n_bins, const int16_t* iq_dev, uint64_t n_complex, int64_t stream_start,
                          uint64_t advance, uint64_t n_windows) {
    return guard([&] {
        CK(cudaSetDevice(ctx->device));
        demodulate_impl(ctx, win, cfg, lo_bins, n_bins, SampleSource::linear(iq_dev, n_complex, stream_start),
                        stream_start, advance, n_windows);
    });
}

int tdg_demodulate(tdg_ctx* ctx, tdg_windows* win, const tdg_demod_config* cfg, const double* lo_bins,
                   uint64_t n_bins, const int16_t* iq, uint64_t n_complex, int64_t stream_start, uint64_t advance,
                   uint64_t n_windows) {
    return guard([&] {
        CK(cudaSetDevice(ctx->device));
        ctx->stream_buf.ensure(std::max<uint64_t>(n_complex, 1) * 2 * sizeof(int16_t));
        CK(cudaMemcpyAsync(ctx->stream_buf.p, iq, n_complex * 2 * sizeof(int16_t), cudaMemcpyHostToDevice, ctx->stream));
        demodulate_impl(ctx, win, cfg, lo_bins, n_bins,
                        SampleSource::linear(ctx->stream_buf.as<int16_t>(), n_complex, stream_start), stream_start,
                        advance, n_windows);
        CK(cudaStreamSynchronize(ctx->stream));
    });
}

int tdg_windows_set_du(tdg_ctx* ctx, tdg_windows* w, uint64_t slot, const float* d, const float* u,
                       int64_t window_start) {
    return guard([&] {
        CK(cudaSetDevice(ctx->device));
        if (slot >= w->slots()) fail(TDG_EINVAL, "slot out of range");
        CK(cudaMemcpyAsync(w->d.as<float>() + slot * w->W, d, w->W * sizeof(float), cudaMemcpyHostToDevice, ctx->stream));
        CK(cudaMemcpyAsync(w->u.as<float>() + slot * w->W, u, w->W * sizeof(float), cudaMemcpyHostToDevice, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
        w->start[slot] = window_start;
        w->dspec_N = 0;
    });
}

int tdg_windows_set_start(tdg_ctx* ctx, tdg_windows* w, uint64_t slot, int64_t window_start) {
    return guard([&] {
        (void)ctx;
        if (slot >= w->slots()) fail(TDG_EINVAL, "slot out of range");
        w->start[slot] = window_start;
    });
}

int tdg_windows_get_du(tdg_ctx* ctx, const tdg_windows* w, uint64_t slot, float* d, float* u) {
    return guard([&] {
        CK(cudaSetDevice(ctx->device));
        if (slot >= w->slots()) fail(TDG_EINVAL, "slot out of range");
        CK(cudaStreamSynchronize(ctx->stream));
        if (d) CK(cudaMemcpy(d, w->d.as<float>() + slot * w->W, w->W * sizeof(float), cudaMemcpyDeviceToHost));
        if (u) CK(cudaMemcpy(u, w->u.as<float>() + slot * w->W, w->W * sizeof(float), cudaMemcpyDeviceToHost));
    });
}

// ---- detection -------------------------------------------------------------
namespace {
// sel (optional): the code indices to detect, in output order (the
// reference's detect over a span of TransformedCode pointers,
// detector.hpp:103-106); nullptr = every code of the set.  Records are
// [slot][k] for k < |sel|.  Only the stored pairs the selection touches are
// correlated.
void detect_impl(tdg_ctx* ctx, tdg_windows* w, const tdg_codeset* cs, float threshold, double fs, tdg_detection* out,
                 bool sync = true, const std::vector<uint64_t>* sel = nullptr) {
    if (cs->window_len != w->W) fail(TDG_EINVAL, "batch_xcorr: mixed window shapes");
    const uint64_t ns = w->used(), nc = cs->n_codes;
    std::vector<uint64_t> all;
    if (!sel) {
        all.resize(nc);
        for (uint64_t i = 0; i < nc; ++i) all[i] = i;
        sel = &all;
    }
    const uint64_t nk = sel->size();
    std::vector<char> want_pair((nc + 1) / 2, 0);
    for (uint64_t c : *sel) {
        if (c >= nc) fail(TDG_EINVAL, "detect: code index out of range");
        if (!cs->seg_lags && w->W + cs->nlen[c] > cs->corr_len() + 1)
            fail(TDG_EINVAL, "batch_xcorr: window does not fit transform size");
        want_pair[c / 2] = 1;
    }
    const uint64_t nseg = cs->n_segments(w->W);
    if (!nk) return;
    // argmax keys [slot][code] of every code of a touched pair (the packed
    // IFFT yields both codes of a pair)
    ctx->keys.ensure(ns * nc * sizeof(unsigned long long));
    CK(cudaMemsetAsync(ctx->keys.p, 0, ns * nc * sizeof(unsigned long long), ctx->stream));
    std::vector<CorrJob> jobs;
    unsigned long long* keys = ctx->keys.as<unsigned long long>();
    // code-pair-major: a group of kGroup stored pairs (whose spectra stay
    // L2-resident) sweeps every window slot before the next group starts
    std::vector<uint64_t> pairs;
    for (uint64_t p = 0; p < want_pair.size(); ++p)
        if (want_pair[p]) pairs.push_back(p);
    const uint64_t G = tdg::kGroup;
    for (uint64_t i0 = 0; i0 < pairs.size(); i0 += G) {
        for (uint64_t ss = 0; ss < ns * nseg; ++ss)
            for (uint64_t i = i0; i < std::min<uint64_t>(pairs.size(), i0 + G); ++i) {
                const uint64_t p = pairs[i], s = ss / nseg, g = ss % nseg;
                CorrJob jb{ss, p, keys + s * nc + 2 * p, 2 * p + 1 < nc ? keys + s * nc + 2 * p + 1 : nullptr,
                           nullptr, nullptr};
                if (cs->seg_lags) {
                    jb.lag0 = uint32_t(g * cs->seg_lags);
                    jb.lag_lim = uint32_t(std::min(cs->seg_lags, w->W - g * cs->seg_lags));
                }
                jobs.push_back(jb);
            }
    }
    ctx->det_dev.ensure(ns * nk * sizeof(tdg_detection));
    // statistics: one CTA per (slot, code), slot-major so a window's d,u stay
    // in L2 across all codes
    std::vector<tdg::StatsDesc> sd(ns * nk);
    for (uint64_t s = 0; s < ns; ++s)
        for (uint64_t k = 0; k < nk; ++k) {
            const uint64_t c = (*sel)[k];
            auto& x = sd[s * nk + k];
            x.d = w->d.as<float>() + s * w->W;
            x.u = w->u.as<float>() + s * w->W;
            x.dc = cs->rep.as<float>() + c * cs->rep_cap;
            x.key = keys + s * nc + c;
            x.out = ctx->det_dev.as<tdg_detection>() + s * nk + k;
            x.nonzero_len = uint32_t(cs->nlen[c]);
            x.energy = cs->energy[c];
            x.window_start = w->start[s];
            x.code_index = int32_t(c);
            x.bin = int32_t(s % w->n_bins);
        }
    auto* sdd = ctx->upload(ctx->pk->stats, sd);
    const bool timed = ctx->detect_timings && !tl_graph_mode;
    if (timed) {
        for (auto& e : ctx->dt_ev)
            if (!e) CK(cudaEventCreate(&e));
        CK(cudaEventRecord(ctx->dt_ev[0], ctx->stream));
    }
    {
        // correlation stage incl. the forward transforms it overlaps (those are
        // also timed on their own as fwd_pass1/2)
        KScope ks(ctx, "corr");
        run_correlations(ctx, w, cs, jobs, false);
    }
    if (timed) CK(cudaEventRecord(ctx->dt_ev[1], ctx->stream));
    // (running each finished code group's statistics under later waves on the
    // second stream was measured slower: it delays the pass-B launches queued
    // behind it and takes SM slots from the persistent passes)
    launch_stats(ctx, sdd, sd.size(), uint32_t(w->W), fs, threshold);
    if (timed) CK(cudaEventRecord(ctx->dt_ev[2], ctx->stream));
    if (out) {
        CK(cudaMemcpyAsync(out, ctx->det_dev.p, ns * nk * sizeof(tdg_detection), cudaMemcpyDeviceToHost, ctx->stream));
        if (sync) CK(cudaStreamSynchronize(ctx->stream));
    }
    if (timed) {
        // DetectTimings (detector.hpp:95-98): correlation = forward transform +
        // spectral products + inverse transforms + argmax; peak_stats = refinement
        // and statistics
        CK(cudaEventSynchronize(ctx->dt_ev[2]));
        float a = 0.f, b = 0.f;
        CK(cudaEventElapsedTime(&a, ctx->dt_ev[0], ctx->dt_ev[1]));
        CK(cudaEventElapsedTime(&b, ctx->dt_ev[1], ctx->dt_ev[2]));
        ctx->last_corr_s = a * 1e-3;
        ctx->last_stats_s = b * 1e-3;
    }
}
}  // namespace

int tdg_detect(tdg_ctx* ctx, tdg_windows* w, const tdg_codeset* cs, float threshold, double sample_rate,
               tdg_detection* out, uint64_t out_cap) {
    return guard([&] {
        CK(cudaSetDevice(ctx->device));
        if (out && out_cap < w->used() * cs->n_codes) fail(TDG_EINVAL, "detect: output capacity too small");
        detect_impl(ctx, w, cs, threshold, sample_rate, out);
    });
}

int tdg_detect_codes(tdg_ctx* ctx, tdg_windows* w, const tdg_codeset* cs, const int64_t* idx, uint64_t n_idx,
                     float threshold, double sample_rate, tdg_detection* out, uint64_t out_cap) {
    return guard([&] {
        CK(cudaSetDevice(ctx->device));
        std::vector<uint64_t> sel(n_idx);
        for (uint64_t i = 0; i < n_idx; ++i) {
            if (idx[i] < 0 || uint64_t(idx[i]) >= cs->n_codes) fail(TDG_EINVAL, "detect: code index out of range");
            sel[i] = uint64_t(idx[i]);
        }
        if (out && out_cap < w->used() * n_idx) fail(TDG_EINVAL, "detect: output capacity too small");
        detect_impl(ctx, w, cs, threshold, sample_rate, out, true, &sel);
    });
}

int tdg_batch_xcorr(tdg_ctx* ctx, tdg_windows* w, uint64_t slot, const tdg_codeset* cs, const int64_t* idx,
                    uint64_t n_idx, float* out) {
    return guard([&] {
        CK(cudaSetDevice(ctx->device));
        if (slot >= w->slots()) fail(TDG_EINVAL, "slot out of range");
        if (cs->window_len != w->W) fail(TDG_EINVAL, "batch_xcorr: mixed window shapes");
        std::vector<int64_t> codes(idx, idx + n_idx);
        for (int64_t c : codes)
            if (c < 0 || uint64_t(c) >= cs->n_codes) fail(TDG_EINVAL, "code index out of range");
        // one row per distinct code (a code requested twice gets the same row
        // twice, like the reference's per-index loop, detector.cpp:116-118);
        // one job per stored pair touched
        std::map<uint64_t, uint64_t> row_of;   // code -> row of xc
        for (int64_t c : codes) row_of.emplace(uint64_t(c), 0);
        uint64_t nr = 0;
        for (auto& kv : row_of) kv.second = nr++;
        DevBuf xc;
        xc.ensure(std::max<uint64_t>(1, nr) * w->W * sizeof(float));
        std::map<uint64_t, std::pair<float*, float*>> per_pair;
        for (auto& [c, r] : row_of) {
            auto& pp = per_pair[c / 2];
            (c % 2 ? pp.second : pp.first) = xc.as<float>() + r * w->W;
        }
        std::vector<CorrJob> jobs;
        const uint64_t nseg = cs->n_segments(w->W);
        for (uint64_t g = 0; g < nseg; ++g)
            for (auto& [p, rows] : per_pair) {
                const uint64_t o = g * cs->seg_lags;
                CorrJob jb{slot * nseg + g, p, nullptr, nullptr, rows.first ? rows.first + o : nullptr,
                           rows.second ? rows.second + o : nullptr};
                if (cs->seg_lags) {
                    jb.lag0 = uint32_t(o);
                    jb.lag_lim = uint32_t(std::min(cs->seg_lags, w->W - o));
                }
                jobs.push_back(jb);
            }
        run_correlations(ctx, w, cs, jobs, true);
        for (uint64_t i = 0; i < n_idx; ++i)
            CK(cudaMemcpyAsync(out + i * w->W, xc.as<float>() + row_of[uint64_t(codes[i])] * w->W,
                               w->W * sizeof(float), cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
    });
}

int tdg_search(tdg_ctx* ctx, const tdg_demod_config* cfg, const double* lo_bins, uint64_t n_bins, const int16_t* iq,
               uint64_t n_complex, int64_t stream_start, uint64_t window_len, uint64_t advance, const tdg_codeset* cs,
               float threshold, tdg_detection* out, uint64_t out_cap, uint64_t* n_out) {
    return guard([&] {
        CK(cudaSetDevice(ctx->device));
        if (advance == 0) fail(TDG_EINVAL, "search: advance must be positive");
        const uint64_t n_windows = n_complex >= window_len ? (n_complex - window_len) / advance + 1 : 0;
        if (n_out) *n_out = n_windows * n_bins * cs->n_codes;
        if (n_windows == 0) return;
        if (out_cap < n_windows * n_bins * cs->n_codes) fail(TDG_EINVAL, "search: output capacity too small");
        tdg_windows* w = ctx->search_win;
        if (!w || w->W != window_len || w->n_windows != n_windows || w->n_bins != n_bins) {
            if (w) tdg_windows_destroy(w);
            ctx->search_win = nullptr;
            int rc = tdg_windows_create(ctx, window_len, n_windows, n_bins, &w);
            if (rc) fail(rc, "%s", g_err.c_str());
            ctx->search_win = w;
        }
        ctx->stream_buf.ensure(n_complex * 2 * sizeof(int16_t));
        CK(cudaMemcpyAsync(ctx->stream_buf.p, iq, n_complex * 2 * sizeof(int16_t), cudaMemcpyHostToDevice, ctx->stream));
        demodulate_impl(ctx, w, cfg, lo_bins, n_bins,
                        SampleSource::linear(ctx->stream_buf.as<int16_t>(), n_complex, stream_start), stream_start,
                        advance, n_windows);
        detect_impl(ctx, w, cs, threshold, cfg->mod.sample_rate, out);
    });
}


// ---------------------------------------------------------------------------
// Tracking (proj/src/recording.cpp:360-378, one Task of
// proj/src/scheduler.cpp:89-113 each): every task is a short window
// [start, start + W) demodulated at cfg->lo_freq and detected against ONE
// code.  A batch of tasks runs as one pipeline: one demod launch for all
// windows, the forward transforms, one correlation job per task and one
// statistics launch -- the latency-bound small batches of BASELINE configs[3].
namespace {
void track_impl(tdg_ctx* ctx, const tdg_demod_config* cfg, const SampleSource& src, const tdg_track_task* tasks,
                uint64_t n_tasks, const tdg_codeset* cs, float threshold, tdg_detection* out, bool sync = true) {
    const uint64_t W = cs->window_len;
    if (cs->seg_lags)
        fail(TDG_ERANGE, "track: windows longer than one transform (segmented code sets) are searched, not tracked");
    for (uint64_t i = 0; i < n_tasks; ++i) {
        if (tasks[i].code_index >= cs->n_codes) fail(TDG_EINVAL, "track: task %llu code index out of range",
                                                     (unsigned long long)i);
        if (!src.holds(tasks[i].start, W))
            fail(TDG_EINVAL, "track: task %llu window outside the sample block", (unsigned long long)i);
        if (W + cs->nlen[tasks[i].code_index] > cs->corr_len() + 1)
            fail(TDG_EINVAL, "batch_xcorr: window does not fit transform size");
    }
    tdg_windows* w = ctx->track_win;
    if (!w || w->W != W || w->n_windows < n_tasks) {
        if (w) tdg_windows_destroy(w);
        ctx->track_win = nullptr;
        uint64_t cap = 16;
        while (cap < n_tasks) cap *= 2;
        int rc = tdg_windows_create(ctx, W, cap, 1, &w);
        if (rc) fail(rc, "%s", g_err.c_str());
        ctx->track_win = w;
    }
    w->active = n_tasks;
    const std::vector<double> bins{cfg->lo_freq};
    const float2* H = ctx->filter_spectra(*cfg, bins);
    std::vector<tdg::DemodWindowDesc> wins(n_tasks);
    for (uint64_t i = 0; i < n_tasks; ++i) {
        wins[i] = {src.offset(tasks[i].start), w->d.as<float>() + i * W, w->u.as<float>() + i * W};
        w->start[i] = tasks[i].start;
    }
    src.before_read(ctx);
    demod_launch(ctx, src.base, true, src.len, wins, W, 1, W, H, cfg->eps, src.ring_cap);
    {
        int64_t lo = tasks[0].start, hi = tasks[0].start;
        for (uint64_t i = 0; i < n_tasks; ++i) {
            lo = std::min(lo, tasks[i].start);
            hi = std::max(hi, tasks[i].start);
        }
        src.after_read(ctx, lo, hi + int64_t(W));
    }
    w->dspec_N = 0;
    // keys[i]: argmax of task i; keys[n_tasks]: sink for the stored pair's
    // other code (its correlation comes for free in the packed IFFT)
    ctx->keys.ensure((n_tasks + 1) * sizeof(unsigned long long));
    if (STREAM_OPS) CK(cudaMemsetAsync(ctx->keys.p, 0, (n_tasks + 1) * sizeof(unsigned long long), ctx->stream));
    unsigned long long* keys = ctx->keys.as<unsigned long long>();
    std::vector<CorrJob> jobs(n_tasks);
    for (uint64_t i = 0; i < n_tasks; ++i) {
        const uint64_t c = tasks[i].code_index;
        const bool odd = c % 2 != 0;
        jobs[i] = {i, c / 2, odd ? keys + n_tasks : keys + i, odd ? keys + i : nullptr, nullptr, nullptr};
    }
    run_correlations(ctx, w, cs, jobs, false);
    ctx->det_dev.ensure(n_tasks * sizeof(tdg_detection));
    std::vector<tdg::StatsDesc> sd(n_tasks);
    for (uint64_t i = 0; i < n_tasks; ++i) {
        const uint64_t c = tasks[i].code_index;
        auto& x = sd[i];
        x.d = w->d.as<float>() + i * W;
        x.u = w->u.as<float>() + i * W;
        x.dc = cs->rep.as<float>() + c * cs->rep_cap;
        x.key = keys + i;
        x.out = ctx->det_dev.as<tdg_detection>() + i;
        x.nonzero_len = uint32_t(cs->nlen[c]);
        x.energy = cs->energy[c];
        x.window_start = tasks[i].start;
        x.code_index = int32_t(c);
        x.bin = 0;
    }
    auto* sdd = ctx->upload(ctx->pk->stats, sd);
    launch_stats(ctx, sdd, n_tasks, uint32_t(W), cfg->mod.sample_rate, threshold);
    if (out) {
        CK(cudaMemcpyAsync(out, ctx->det_dev.p, n_tasks * sizeof(tdg_detection), cudaMemcpyDeviceToHost,
                           ctx->stream));
        if (sync) CK(cudaStreamSynchronize(ctx->stream));
    }
}

// Synchronous tracking of a linear sample block: batches that fit one
// correlation wave run as CUDA graphs once seen twice with the same key
// (first call: normal, warming every cache; second: captured; later: the
// host rebuilds the descriptors in the graph's staging and launches it).
// Larger batches, or any buffer move in between, take the normal path.
void track_linear(tdg_ctx* ctx, const tdg_demod_config* cfg, const SampleSource& src, const tdg_track_task* tasks,
                  uint64_t n_tasks, const tdg_codeset* cs, float threshold, tdg_detection* out) {
    const uint64_t wave = uint64_t(std::max<int64_t>(tdg::kGroup, ctx->wave_pairs / tdg::kGroup * tdg::kGroup));
    if (!ctx->track_graphs_on || n_tasks > wave) {
        track_impl(ctx, cfg, src, tasks, n_tasks, cs, threshold, out);
        return;
    }
    const tdg_modulation& m = cfg->mod;
    // (the tasks and stream_start only enter descriptor contents, rebuilt on
    // every call; tdg_set_option drops every graph)
    const std::vector<double> key{double(n_tasks),       double(cs->window_len), double(src.len),
                                  double(threshold),     m.sample_rate,          m.bit_rate,
                                  m.freq_one,            m.freq_zero,            double(m.packet_bits),
                                  cfg->lo_freq,          cfg->bandpass_center,   cfg->bandpass_width,
                                  double(cfg->bandpass_taps), double(cfg->eps)};
    TrackGraph* g = nullptr;
    for (auto& x : ctx->track_graphs)
        if (x->cs == cs && x->base == src.base && x->key == key) g = x.get();
    const uint64_t ep = g_dev_epoch.load();
    auto finish = [&] {
        if (out) CK(cudaMemcpyAsync(out, ctx->det_dev.p, n_tasks * sizeof(tdg_detection), cudaMemcpyDeviceToHost,
                                    ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
    };
    // host pass in graph mode `mode` with the entry's staging; always restores
    auto host_pass = [&](int mode) {
        tl_graph_mode = mode;
        ctx->pk = &g->packs;
        try {
            track_impl(ctx, cfg, src, tasks, n_tasks, cs, threshold, nullptr, false);
        } catch (...) {
            tl_graph_mode = 0;
            ctx->pk = &ctx->own_packs;
            throw;
        }
        tl_graph_mode = 0;
        ctx->pk = &ctx->own_packs;
    };
    if (g && g->state == 2 && g->epoch == ep) {
        g->last_use = ++ctx->graph_clock;
        host_pass(2);
        if (g_dev_epoch.load() == ep) {
            CK(cudaGraphLaunch(g->exec, ctx->stream));
            LAUNCHED_GRAPH();
            finish();
            return;
        }
        g->state = 0;   // something moved during the host pass
    } else if (g && g->state == 1 && g->epoch == ep) {
        g->last_use = ++ctx->graph_clock;
        host_pass(2);   // validates the batch and sizes the entry's staging (its only allocations)
        const uint64_t ep2 = g_dev_epoch.load();
        cudaGraph_t graph = nullptr;
        bool ok = cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal) == cudaSuccess;
        if (ok) {
            try {
                host_pass(1);
            } catch (...) {
                ok = false;
            }
            ok = cudaStreamEndCapture(ctx->stream, &graph) == cudaSuccess && ok && graph;
        }
        if (g->exec) cudaGraphExecDestroy(g->exec);
        g->exec = nullptr;
        ok = ok && cudaGraphInstantiate(&g->exec, graph, 0) == cudaSuccess;
        if (graph) cudaGraphDestroy(graph);
        if (ok && g_dev_epoch.load() == ep2) {
            g->state = 2;
            g->epoch = ep2;
            CK(cudaGraphLaunch(g->exec, ctx->stream));
            LAUNCHED_GRAPH();
            finish();
            return;
        }
        // not capturable: this key stays on the stream path (same kernels)
        cudaGetLastError();
        g->state = -1;
        track_impl(ctx, cfg, src, tasks, n_tasks, cs, threshold, out);
        return;
    }
    track_impl(ctx, cfg, src, tasks, n_tasks, cs, threshold, out);
    if (!g) {
        if (ctx->track_graphs.size() >= 8) {   // evict the least recently used entry
            auto lru = std::min_element(ctx->track_graphs.begin(), ctx->track_graphs.end(),
                                        [](const auto& a, const auto& b) { return a->last_use < b->last_use; });
            ctx->track_graphs.erase(lru);
        }
        ctx->track_graphs.push_back(std::make_unique<TrackGraph>());
        g = ctx->track_graphs.back().get();
        g->cs = cs;
        g->base = src.base;
    }
    g->key = key;
    if (g->state != -1) g->state = 1;
    g->last_use = ++ctx->graph_clock;
    g->epoch = g_dev_epoch.load();
}
}  // namespace

int tdg_track_device(tdg_ctx* ctx, const tdg_demod_config* cfg, const int16_t* iq_dev, uint64_t n_complex,
                     int64_t stream_start, const tdg_track_task* tasks, uint64_t n_tasks, const tdg_codeset* cs,
                     float threshold, tdg_detection* out) {
    return guard([&] {
        CK(cudaSetDevice(ctx->device));
        if (n_tasks == 0) return;
        track_linear(ctx, cfg, SampleSource::linear(iq_dev, n_complex, stream_start), tasks, n_tasks, cs, threshold,
                     out);
    });
}

int tdg_track(tdg_ctx* ctx, const tdg_demod_config* cfg, const int16_t* iq, uint64_t n_complex, int64_t stream_start,
              const tdg_track_task* tasks, uint64_t n_tasks, const tdg_codeset* cs, float threshold,
              tdg_detection* out) {
    return guard([&] {
        CK(cudaSetDevice(ctx->device));
        if (n_tasks == 0) return;
        ctx->stream_buf.ensure(n_complex * 2 * sizeof(int16_t));
        CK(cudaMemcpyAsync(ctx->stream_buf.p, iq, n_complex * 2 * sizeof(int16_t), cudaMemcpyHostToDevice,
                           ctx->stream));
        track_linear(ctx, cfg, SampleSource::linear(ctx->stream_buf.as<int16_t>(), n_complex, stream_start), tasks,
                     n_tasks, cs, threshold, out);
    });
}


// ---------------------------------------------------------------------------
// Device-resident CircularBuffer and the searches/tracking tasks that read it.
namespace {
tdg_windows* search_windows(tdg_ctx* ctx, uint64_t window_len, uint64_t n_windows, uint64_t n_bins) {
    tdg_windows* w = ctx->search_win;
    if (!w || w->W != window_len || w->n_windows != n_windows || w->n_bins != n_bins) {
        if (w) tdg_windows_destroy(w);
        ctx->search_win = nullptr;
        int rc = tdg_windows_create(ctx, window_len, n_windows, n_bins, &w);
        if (rc) fail(rc, "%s", g_err.c_str());
        ctx->search_win = w;
    }
    return w;
}

void ring_prune(tdg_ring* r) {
    std::vector<tdg_ring::Read> keep;
    for (auto& rd : r->reads) {
        const cudaError_t q = cudaEventQuery(rd.ev);
        if (q == cudaSuccess) {
            r->spare.push_back(rd.ev);
        } else if (q == cudaErrorNotReady) {
            keep.push_back(rd);
        } else {
            CK(q);
        }
    }
    r->reads.swap(keep);
}
}  // namespace

int tdg_ring_create(tdg_ctx* ctx, uint64_t capacity, tdg_ring** out) {
    return guard([&] {
        *out = nullptr;
        CK(cudaSetDevice(ctx->device));
        if (capacity == 0) fail(TDG_EINVAL, "ring: capacity must be positive");
        auto r = std::make_unique<tdg_ring>();
        r->ctx = ctx;
        r->device = ctx->device;
        r->cap = capacity;
        r->buf.ensure(capacity * 2 * sizeof(int16_t));
        CK(cudaStreamCreateWithFlags(&r->copy, cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&r->pushed, cudaEventDisableTiming));
        CK(cudaMemsetAsync(r->buf.p, 0, r->buf.bytes, r->copy));
        CK(cudaEventRecord(r->pushed, r->copy));
        *out = r.release();
    });
}

void tdg_ring_destroy(tdg_ring* r) {
    if (!r) return;
    cudaSetDevice(r->device);
    cudaStreamSynchronize(r->copy);
    for (auto& rd : r->reads) {
        cudaEventSynchronize(rd.ev);
        cudaEventDestroy(rd.ev);
    }
    for (auto e : r->spare) cudaEventDestroy(e);
    if (r->pushed) cudaEventDestroy(r->pushed);
    if (r->copy) cudaStreamDestroy(r->copy);
    delete r;
}

int tdg_ring_bounds(const tdg_ring* r, int64_t* head, int64_t* tail, uint64_t* capacity) {
    return guard([&] {
        if (head) *head = r->head;
        if (tail) *tail = r->tail;
        if (capacity) *capacity = r->cap;
    });
}

// CircularBuffer::push (proj/src/scheduler.cpp:11-33): same gap / eviction
// bookkeeping; only the last `cap` samples of a block are uploaded.
int tdg_ring_push(tdg_ring* r, const int16_t* iq, uint64_t n_complex, int64_t start, tdg_ring_push_result* res) {
    return guard([&] {
        CK(cudaSetDevice(r->device));
        tdg_ring_push_result pr{};
        if (start != r->tail) {   // gap in the stream: resynchronise at the new start
            pr.gap = 1;
            pr.evicted_begin = r->head;
            pr.evicted_end = r->tail;
            r->head = r->tail = start;
        }
        const uint64_t skip = n_complex > r->cap ? n_complex - r->cap : 0;
        const int64_t t0 = start + int64_t(skip);
        const uint64_t m = n_complex - skip;
        if (m) {
            ring_prune(r);
            for (auto& rd : r->reads)
                if (r->overlap(rd.s, uint64_t(rd.e - rd.s), t0, m)) CK(cudaStreamWaitEvent(r->copy, rd.ev, 0));
            const uint64_t sl = r->slot(t0), first = std::min(m, r->cap - sl);
            int16_t* dst = r->buf.as<int16_t>();
            CK(cudaMemcpyAsync(dst + 2 * sl, iq + 2 * skip, first * 2 * sizeof(int16_t), cudaMemcpyHostToDevice,
                               r->copy));
            if (m > first)
                CK(cudaMemcpyAsync(dst, iq + 2 * (skip + first), (m - first) * 2 * sizeof(int16_t),
                                   cudaMemcpyHostToDevice, r->copy));
            CK(cudaEventRecord(r->pushed, r->copy));
        }
        r->tail += int64_t(n_complex);
        if (r->tail - r->head > int64_t(r->cap)) {
            if (!pr.gap) {
                pr.evicted_begin = r->head;
                pr.evicted_end = r->tail - int64_t(r->cap);
            }
            r->head = r->tail - int64_t(r->cap);
        }
        if (res) *res = pr;
    });
}

// CircularBuffer::read (proj/src/scheduler.cpp:35-45): *ok = 0 if any part
// of [start, end) was evicted or not yet received.
int tdg_ring_read(tdg_ring* r, int64_t start, int64_t end, int16_t* out, int* ok) {
    return guard([&] {
        CK(cudaSetDevice(r->device));
        *ok = 0;
        if (start < r->head || end > r->tail || start > end) return;
        const uint64_t m = uint64_t(end - start);
        if (m) {
            const uint64_t sl = r->slot(start), first = std::min(m, r->cap - sl);
            const int16_t* src = r->buf.as<int16_t>();
            CK(cudaMemcpyAsync(out, src + 2 * sl, first * 2 * sizeof(int16_t), cudaMemcpyDeviceToHost, r->copy));
            if (m > first)
                CK(cudaMemcpyAsync(out + 2 * first, src, (m - first) * 2 * sizeof(int16_t), cudaMemcpyDeviceToHost,
                                   r->copy));
            CK(cudaStreamSynchronize(r->copy));
        }
        *ok = 1;
    });
}

int tdg_search_ring(tdg_ctx* ctx, tdg_ring* r, const tdg_demod_config* cfg, const double* lo_bins, uint64_t n_bins,
                    int64_t first_start, uint64_t window_len, uint64_t advance, uint64_t n_windows,
                    const tdg_codeset* cs, float threshold, tdg_detection* out, uint64_t out_cap, int sync) {
    return guard([&] {
        CK(cudaSetDevice(ctx->device));
        if (advance == 0) fail(TDG_EINVAL, "search: advance must be positive");
        if (n_windows == 0) return;
        if (cs->window_len != window_len) fail(TDG_EINVAL, "batch_xcorr: mixed window shapes");
        if (out && out_cap < n_windows * n_bins * cs->n_codes) fail(TDG_EINVAL, "search: output capacity too small");
        if (r->device != ctx->device) fail(TDG_EINVAL, "search: ring and context on different devices");
        tdg_windows* w = search_windows(ctx, window_len, n_windows, n_bins);
        demodulate_impl(ctx, w, cfg, lo_bins, n_bins, SampleSource::of(r), first_start, advance, n_windows);
        detect_impl(ctx, w, cs, threshold, cfg->mod.sample_rate, out, sync != 0);
    });
}

int tdg_track_ring(tdg_ctx* ctx, tdg_ring* r, const tdg_demod_config* cfg, const tdg_track_task* tasks,
                   uint64_t n_tasks, const tdg_codeset* cs, float threshold, tdg_detection* out, int sync) {
    return guard([&] {
        CK(cudaSetDevice(ctx->device));
        if (n_tasks == 0) return;
        if (r->device != ctx->device) fail(TDG_EINVAL, "track: ring and context on different devices");
        track_impl(ctx, cfg, SampleSource::of(r), tasks, n_tasks, cs, threshold, out, sync != 0);
    });
}

// FP32 peak of the current device at its current clock (bench.py's roofline
// denominator): TFLOP/s of scalar FFMA and of packed FFMA2 (2 flops per FMA
// lane), best of 5 timed launches after a warm-up.
int tdg_fp32_peak(int device, double* ffma_tflops, double* ffma2_tflops) {
    return guard([&] {
        CK(cudaSetDevice(device));
        const int sms = num_sms();
        DevBuf out;
        out.ensure(64);
        CK(cudaMemset(out.p, 0, 64));
        cudaStream_t st;
        CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        cudaEvent_t e0, e1;
        CK(cudaEventCreate(&e0));
        CK(cudaEventCreate(&e1));
        const int iters = 2048, threads = 512, blocks = sms * 4;
        double best1 = 0, best2 = 0;
        for (int rep = 0; rep < 6; ++rep) {
            float ms = 0;
            CK(cudaEventRecord(e0, st));
            tdg::k_peak_ffma<<<blocks, threads, 0, st>>>(out.as<float>(), iters);
            CK(cudaEventRecord(e1, st));
            CK(cudaEventSynchronize(e1));
            CK(cudaEventElapsedTime(&ms, e0, e1));
            const double f1 = double(blocks) * threads * iters * 64 * 2 / (ms * 1e-3) / 1e12;
            CK(cudaEventRecord(e0, st));
            tdg::k_peak_ffma2<<<blocks, threads, 0, st>>>(out.as<float>(), iters);
            CK(cudaEventRecord(e1, st));
            CK(cudaEventSynchronize(e1));
            CK(cudaEventElapsedTime(&ms, e0, e1));
            const double f2 = double(blocks) * threads * iters * 64 * 4 / (ms * 1e-3) / 1e12;
            if (rep) {
                best1 = std::max(best1, f1);
                best2 = std::max(best2, f2);
            }
        }
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        cudaStreamDestroy(st);
        if (ffma_tflops) *ffma_tflops = best1;
        if (ffma2_tflops) *ffma2_tflops = best2;
    });
}

// ---------------------------------------------------------------------------
// Span-level entry points: the reference functions that take and return host
// arrays (the drop-in's fft.hpp / dsp.hpp / detector.hpp surface), each one a
// device round trip through the kernels of generic.cuh / kernels.cuh.
namespace {
int grid_for(uint64_t n) { return int(std::max<uint64_t>(1, std::min<uint64_t>((n + 255) / 256, uint64_t(num_sms()) * 16))); }

// {2,3,5,7}-smooth radix plan, largest radices first (8 and 4 for powers of two)
std::vector<int> radix_plan(uint64_t n) {
    std::vector<int> r;
    uint64_t m = n;
    while (m % 8 == 0) { r.push_back(8); m /= 8; }
    while (m % 4 == 0) { r.push_back(4); m /= 4; }
    while (m % 2 == 0) { r.push_back(2); m /= 2; }
    for (int p : {7, 5, 3})
        while (m % uint64_t(p) == 0) { r.push_back(p); m /= uint64_t(p); }
    if (m != 1) fail(TDG_ERANGE, "fft: length %llu is not {2,3,5,7}-smooth", (unsigned long long)n);
    return r;
}

// in-place-by-ping-pong Stockham FFT of the n complex values at a; the result
// is in a (copied back if the stage count is odd).  inverse: sign +1 and 1/n.
void fft_device(tdg_ctx* ctx, float2* a, float2* tmp, uint64_t n, bool inverse) {
    if (n >= (uint64_t(1) << 32)) fail(TDG_ERANGE, "fft: length too large");
    const auto plan = radix_plan(n);
    float2 *src = a, *dst = tmp;
    uint32_t ns = 1;
    for (size_t s = 0; s < plan.size(); ++s) {
        const float scale = (inverse && s + 1 == plan.size()) ? float(1.0 / double(n)) : 1.0f;
        const int R = plan[s];
        const int g = grid_for(n / uint64_t(R));
#define STAGE(RR)                                                                                              \
    if (R == RR) {                                                                                             \
        if (inverse) tdg::k_stockham<RR, 1><<<g, 256, 0, ctx->stream>>>(src, dst, uint32_t(n), ns, scale);     \
        else tdg::k_stockham<RR, -1><<<g, 256, 0, ctx->stream>>>(src, dst, uint32_t(n), ns, scale);            \
    }
        STAGE(2) STAGE(3) STAGE(4) STAGE(5) STAGE(7) STAGE(8)
#undef STAGE
        LAUNCHED();
        ns *= uint32_t(R);
        std::swap(src, dst);
    }
    if (src != a) CK(cudaMemcpyAsync(a, src, n * sizeof(float2), cudaMemcpyDeviceToDevice, ctx->stream));
}
}  // namespace

int tdg_fft(tdg_ctx* ctx, const float* in, float* out, uint64_t n, int inverse) {
    return guard([&] {
        CK(cudaSetDevice(ctx->device));
        if (n == 0) fail(TDG_EINVAL, "fft: empty transform");
        ctx->gen_a.ensure(n * sizeof(float2));
        ctx->gen_b.ensure(n * sizeof(float2));
        CK(cudaMemcpyAsync(ctx->gen_a.p, in, n * sizeof(float2), cudaMemcpyHostToDevice, ctx->stream));
        fft_device(ctx, ctx->gen_a.as<float2>(), ctx->gen_b.as<float2>(), n, inverse != 0);
        CK(cudaMemcpyAsync(out, ctx->gen_a.p, n * sizeof(float2), cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
    });
}

int tdg_convert(tdg_ctx* ctx, const int16_t* iq, uint64_t n_int16, float* out) {
    return guard([&] {
        CK(cudaSetDevice(ctx->device));
        if (n_int16 % 2) fail(TDG_EINVAL, "convert: odd raw sample count");
        const uint64_t n = n_int16 / 2;
        if (!n) return;
        ctx->gen_c.ensure(n * 2 * sizeof(int16_t));
        ctx->gen_a.ensure(n * sizeof(float2));
        CK(cudaMemcpyAsync(ctx->gen_c.p, iq, n * 2 * sizeof(int16_t), cudaMemcpyHostToDevice, ctx->stream));
        tdg::k_convert<<<grid_for(n), 256, 0, ctx->stream>>>(ctx->gen_c.as<short2>(), ctx->gen_a.as<float2>(), n);
        LAUNCHED();
        CK(cudaMemcpyAsync(out, ctx->gen_a.p, n * sizeof(float2), cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
    });
}

int tdg_mix(tdg_ctx* ctx, float* x, uint64_t n, double lo_freq, int64_t start_index, double sample_rate) {
    return guard([&] {
        CK(cudaSetDevice(ctx->device));
        if (lo_freq == 0.0 || n == 0) return;   // the reference's no-op (dsp.cpp:19)
        ctx->gen_a.ensure(n * sizeof(float2));
        CK(cudaMemcpyAsync(ctx->gen_a.p, x, n * sizeof(float2), cudaMemcpyHostToDevice, ctx->stream));
        tdg::k_mix<<<grid_for(n), 256, 0, ctx->stream>>>(ctx->gen_a.as<float2>(), n, lo_freq / sample_rate, start_index);
        LAUNCHED();
        CK(cudaMemcpyAsync(x, ctx->gen_a.p, n * sizeof(float2), cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
    });
}

int tdg_convolve(tdg_ctx* ctx, const float* x, uint64_t nx, const float* h, uint64_t nh, float* out) {
    return guard([&] {
        CK(cudaSetDevice(ctx->device));
        if (nh == 0) fail(TDG_EINVAL, "overlap_add_filter: empty filter");
        if (nx == 0) return;
        const uint64_t nf = nx + nh - 1, L = pad_length_impl(nf);
        ctx->gen_a.ensure(L * sizeof(float2));
        ctx->gen_b.ensure(L * sizeof(float2));
        ctx->gen_d.ensure(L * sizeof(float2));
        float2* A = ctx->gen_a.as<float2>();
        float2* B = ctx->gen_d.as<float2>();
        CK(cudaMemsetAsync(A, 0, L * sizeof(float2), ctx->stream));
        CK(cudaMemsetAsync(B, 0, L * sizeof(float2), ctx->stream));
        CK(cudaMemcpyAsync(A, x, nx * sizeof(float2), cudaMemcpyHostToDevice, ctx->stream));
        CK(cudaMemcpyAsync(B, h, nh * sizeof(float2), cudaMemcpyHostToDevice, ctx->stream));
        fft_device(ctx, A, ctx->gen_b.as<float2>(), L, false);
        fft_device(ctx, B, ctx->gen_b.as<float2>(), L, false);
        tdg::k_cmul_inplace<<<grid_for(L), 256, 0, ctx->stream>>>(A, B, L);
        LAUNCHED();
        fft_device(ctx, A, ctx->gen_b.as<float2>(), L, true);
        CK(cudaMemcpyAsync(out, A, nf * sizeof(float2), cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
    });
}

int tdg_discriminate(tdg_ctx* ctx, const float* f1, const float* f0, uint64_t n, float eps, float* d, float* u) {
    return guard([&] {
        CK(cudaSetDevice(ctx->device));
        if (!n) return;
        ctx->gen_a.ensure(n * sizeof(float2));
        ctx->gen_b.ensure(n * sizeof(float2));
        ctx->gen_c.ensure(2 * n * sizeof(float));
        CK(cudaMemcpyAsync(ctx->gen_a.p, f1, n * sizeof(float2), cudaMemcpyHostToDevice, ctx->stream));
        CK(cudaMemcpyAsync(ctx->gen_b.p, f0, n * sizeof(float2), cudaMemcpyHostToDevice, ctx->stream));
        float* dd = ctx->gen_c.as<float>();
        tdg::k_discriminate<<<grid_for(n), 256, 0, ctx->stream>>>(ctx->gen_a.as<float2>(), ctx->gen_b.as<float2>(), n, eps,
                                                                  dd, dd + n);
        LAUNCHED();
        CK(cudaMemcpyAsync(d, dd, n * sizeof(float), cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaMemcpyAsync(u, dd + n, n * sizeof(float), cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
    });
}

int tdg_find_peak(tdg_ctx* ctx, const float* xc, uint64_t n, uint64_t* j, float* value) {
    return guard([&] {
        CK(cudaSetDevice(ctx->device));
        if (n == 0) fail(TDG_EINVAL, "find_peak: empty correlation");
        if (n >= (uint64_t(1) << 32)) fail(TDG_ERANGE, "find_peak: length too large");
        ctx->gen_c.ensure(n * sizeof(float));
        ctx->gen_d.ensure(sizeof(unsigned long long));
        CK(cudaMemcpyAsync(ctx->gen_c.p, xc, n * sizeof(float), cudaMemcpyHostToDevice, ctx->stream));
        CK(cudaMemsetAsync(ctx->gen_d.p, 0, sizeof(unsigned long long), ctx->stream));
        tdg::k_argmax_abs<<<grid_for(n), 256, 0, ctx->stream>>>(ctx->gen_c.as<float>(), n,
                                                                ctx->gen_d.as<unsigned long long>());
        LAUNCHED();
        unsigned long long key = 0;
        CK(cudaMemcpyAsync(&key, ctx->gen_d.p, sizeof(key), cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
        const uint64_t jj = 0xFFFFFFFFull - (key & 0xFFFFFFFFull);
        *j = jj;
        *value = xc[jj];   // the signed value at the peak (detector.cpp:133)
    });
}

int tdg_statistics(tdg_ctx* ctx, const float* d, const float* u, uint64_t W, const float* dc, uint64_t n, uint64_t j,
                   float* w_c, float* q, float* p_c, int* partial) {
    return guard([&] {
        CK(cudaSetDevice(ctx->device));
        if (W >= (uint64_t(1) << 32) || n >= (uint64_t(1) << 32)) fail(TDG_ERANGE, "statistics: length too large");
        const uint64_t ncap = (std::max<uint64_t>(n, 1) + 3) & ~uint64_t(3);
        ctx->gen_c.ensure((2 * W + ncap + 8) * sizeof(float));
        ctx->gen_d.ensure(sizeof(unsigned long long) + sizeof(tdg_detection) + sizeof(tdg::StatsDesc) + 64);
        float* dd = ctx->gen_c.as<float>();
        float* uu = dd + W;
        // 16-byte aligned replica (the statistics kernel's vector path)
        float* cc = reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(uu + W) + 15) & ~uintptr_t(15));
        CK(cudaMemsetAsync(cc, 0, ncap * sizeof(float), ctx->stream));
        CK(cudaMemcpyAsync(dd, d, W * sizeof(float), cudaMemcpyHostToDevice, ctx->stream));
        CK(cudaMemcpyAsync(uu, u, W * sizeof(float), cudaMemcpyHostToDevice, ctx->stream));
        if (n) CK(cudaMemcpyAsync(cc, dc, n * sizeof(float), cudaMemcpyHostToDevice, ctx->stream));
        char* base = static_cast<char*>(ctx->gen_d.p);
        auto* key = reinterpret_cast<unsigned long long*>(base);
        auto* det = reinterpret_cast<tdg_detection*>(base + 64);
        auto* desc = reinterpret_cast<tdg::StatsDesc*>(base + 64 + ((sizeof(tdg_detection) + 63) & ~size_t(63)));
        const unsigned long long k = 0xFFFFFFFFull - (j & 0xFFFFFFFFull);   // peak_key(0, j)
        tdg::StatsDesc sd{dd, uu, cc, key, det, uint32_t(n), 1.0f, 0, 0, 0};
        CK(cudaMemcpyAsync(key, &k, sizeof(k), cudaMemcpyHostToDevice, ctx->stream));
        CK(cudaMemcpyAsync(desc, &sd, sizeof(sd), cudaMemcpyHostToDevice, ctx->stream));
        tdg::k_stats<false><<<1, 256, 0, ctx->stream>>>(desc, uint32_t(W), 1.0, 0.25f, 1, nullptr, nullptr);
        LAUNCHED();
        tdg_detection r;
        CK(cudaMemcpyAsync(&r, det, sizeof(r), cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
        *w_c = r.w_c;
        *q = r.q;
        *p_c = r.p_c;
        *partial = r.partial;
    });
}

int tdg_demodulate_signal(tdg_ctx* ctx, tdg_windows* win, const tdg_demod_config* cfg, double lo_freq, const float* x,
                          uint64_t n, int64_t start_index) {
    return guard([&] {
        CK(cudaSetDevice(ctx->device));
        if (win->W != n || win->slots() < 1) fail(TDG_EINVAL, "demodulate_signal: window set shape");
        std::vector<double> bins{lo_freq};
        const float2* H = ctx->filter_spectra(*cfg, bins);
        ctx->gen_a.ensure(std::max<uint64_t>(n, 1) * sizeof(float2));
        CK(cudaMemcpyAsync(ctx->gen_a.p, x, n * sizeof(float2), cudaMemcpyHostToDevice, ctx->stream));
        std::vector<tdg::DemodWindowDesc> wins{{0, win->d.as<float>(), win->u.as<float>()}};
        demod_launch(ctx, ctx->gen_a.p, false, n, wins, n, 1, n, H, cfg->eps);
        win->start[0] = start_index;
        win->dspec_N = 0;
        CK(cudaStreamSynchronize(ctx->stream));
    });
}

int tdg_detect_timings(tdg_ctx* ctx, double* correlation_s, double* peak_stats_s) {
    return guard([&] {
        if (correlation_s) *correlation_s = ctx->last_corr_s;
        if (peak_stats_s) *peak_stats_s = ctx->last_stats_s;
    });
}

}  // extern "C"
