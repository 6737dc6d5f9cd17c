// TEST INFRASTRUCTURE ONLY (oracle).  extern "C" wrapper over the UNMODIFIED
// reference library compiled in place from /root/reference/proj/src (see
// oracle/Makefile; nothing is copied into this repo).  Only tests/, the
// __graft_entry__.smoke() checker and bench.py's CPU-baseline / reference arm
// may load the resulting oracle/_ref/libtagdsp_ref.so.
//
// Every function forwards to the reference API it names; exceptions become a
// status code (1 = std::invalid_argument, 5 = anything else) plus a message.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <fstream>
#include <cstring>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "tagdsp/codegen.hpp"
#include "tagdsp/detector.hpp"
#include "tagdsp/dsp.hpp"
#include "tagdsp/harness.hpp"
#include "tagdsp/recording.hpp"
#include "tagdsp/scheduler.hpp"
#include "tagdsp_gpu_types.h"

using namespace tagdsp;

namespace {

thread_local std::string g_err;

template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 5;
    }
}

ModulationParams to_mod(const tdg_modulation& m) {
    ModulationParams p;
    p.sample_rate = m.sample_rate;
    p.bit_rate = m.bit_rate;
    p.freq_one = m.freq_one;
    p.freq_zero = m.freq_zero;
    p.packet_bits = size_t(m.packet_bits);
    return p;
}

DemodConfig to_cfg(const tdg_demod_config& c) {
    DemodConfig cfg;
    cfg.mod = to_mod(c.mod);
    cfg.lo_freq = c.lo_freq;
    cfg.bandpass_center = c.bandpass_center;
    cfg.bandpass_width = c.bandpass_width;
    cfg.bandpass_taps = size_t(c.bandpass_taps);
    cfg.eps = c.eps;
    return cfg;
}

void fill_detection(const Detection& d, int32_t code_index, int32_t bin, int64_t window_start,
                    tdg_detection* out) {
    std::memset(out, 0, sizeof(*out));
    out->code_index = code_index;
    out->bin = bin;
    out->window_start = window_start;
    out->peak_index = d.peak_index;
    out->toa_seconds = d.toa_seconds;
    out->subsample_offset = d.subsample_offset;
    out->peak_value = d.peak_value;
    out->w_c = d.w_c;
    out->q = d.q;
    out->p_c = d.p_c;
    out->score = d.score;
    out->accepted = d.accepted;
    out->partial = d.partial;
}

}  // namespace

struct tdref_session {
    PlanCache cache;
    CodeCache codes;                              // prepare_code cache
    std::vector<std::unique_ptr<TransformedCode>> owned;  // make_transformed results
    std::vector<const TransformedCode*> index;    // code_index -> code
};

extern "C" {

const char* tdref_last_error(void) { return g_err.c_str(); }

uint64_t tdref_pad_length(uint64_t n) {
    uint64_t r = 0;
    if (guard([&] { r = pad_length(size_t(n)); })) return 0;
    return r;
}

int tdref_gen_code(uint64_t seed, const tdg_modulation* mod, uint8_t* bits_out) {
    return guard([&] {
        auto code = gen_code(seed, to_mod(*mod));
        std::memcpy(bits_out, code.bits.data(), code.bits.size());
    });
}

// synth_replica (proj/src/codegen.cpp:40-60); out = interleaved re,im floats.
int tdref_synth_replica(const uint8_t* bits, uint64_t nbits, const tdg_modulation* mod,
                        uint64_t padded_len, float* out) {
    return guard([&] {
        TagCode code;
        code.mod = to_mod(*mod);
        code.bits.assign(bits, bits + nbits);
        auto r = synth_replica(code, size_t(padded_len));
        std::memcpy(out, r.data(), r.size() * sizeof(cfloat));
    });
}

// The harness/test window generator: replica of `bits` delayed through the
// channel model (apply_channel, proj/src/codegen.cpp:84-124), then quantize
// (:126-143).  Mirrors proj/src/harness.cpp:47-54 and test_detector.cpp:269-275.
int tdref_channel_window(const uint8_t* bits, uint64_t nbits, const tdg_modulation* mod,
                         double delay, double snr_db, double gain, double freq_offset,
                         uint64_t window_len, uint64_t rng_seed, float scale, int16_t* out) {
    return guard([&] {
        TagCode code;
        code.mod = to_mod(*mod);
        code.bits.assign(bits, bits + nbits);
        auto replica = synth_replica(code, code.mod.packet_samples());
        ChannelSpec chan;
        chan.delay = delay;
        chan.snr_db = snr_db;
        chan.gain = gain;
        chan.freq_offset = freq_offset;
        auto rf = apply_channel(replica, chan, size_t(window_len), rng_seed, code.mod.sample_rate);
        auto blk = quantize(rf, scale, 0, code.mod.sample_rate);
        std::memcpy(out, blk.samples.data(), blk.samples.size() * sizeof(int16_t));
    });
}

// Pure-noise window as in acceptance.cpp:217-218 (random_signal + quantize).
int tdref_noise_window(uint64_t n, uint64_t seed, float scale, int16_t* out) {
    return guard([&] {
        GaussianRng rng(seed);
        std::vector<cfloat> sig(n);
        for (auto& v : sig) v = cfloat(rng.next(), rng.next());
        auto blk = quantize(sig, scale, 0, 8.0e6);
        std::memcpy(out, blk.samples.data(), blk.samples.size() * sizeof(int16_t));
    });
}

// GaussianRng draws (proj/src/codegen.cpp:10-24).
int tdref_gaussian(uint64_t seed, uint64_t n, float* out) {
    return guard([&] {
        GaussianRng rng(seed);
        for (uint64_t i = 0; i < n; ++i) out[i] = rng.next();
    });
}

// generate_recording (proj/src/recording.cpp:177-219).  Tags are t<i> with
// seeds tag_seeds[i]; injections reference tags by index.
int64_t tdref_generate_recording(const tdg_demod_config* demod, float quantize_scale,
                                 const uint64_t* tag_seeds, uint64_t n_tags, double duration_s,
                                 double noise_snr_db, uint64_t noise_seed, const int32_t* inj_tag,
                                 const double* inj_time, const double* inj_gain,
                                 const double* inj_freq, uint64_t n_inj, int16_t* out,
                                 uint64_t cap_int16) {
    int64_t n_complex = -1;
    int rc = guard([&] {
        RunConfig cfg;
        cfg.demod = to_cfg(*demod);
        cfg.quantize_scale = quantize_scale;
        for (uint64_t i = 0; i < n_tags; ++i)
            cfg.tags.push_back({"t" + std::to_string(i), tag_seeds[i], 1.0});
        Scenario sc;
        sc.duration_s = duration_s;
        sc.noise_snr_db = noise_snr_db;
        sc.noise_seed = noise_seed;
        for (uint64_t i = 0; i < n_inj; ++i)
            sc.injections.push_back({"t" + std::to_string(inj_tag[i]), inj_time[i], inj_gain[i], inj_freq[i]});
        auto rec = generate_recording(cfg, sc, nullptr);
        if (rec.block.samples.size() > cap_int16) throw std::runtime_error("output buffer too small");
        std::memcpy(out, rec.block.samples.data(), rec.block.samples.size() * sizeof(int16_t));
        n_complex = int64_t(rec.block.num_complex());
    });
    return rc ? -rc : n_complex;
}

// demodulate_window (proj/src/dsp.cpp:193-197).
int tdref_demodulate_window(const int16_t* iq, uint64_t n_complex, int64_t start,
                            const tdg_demod_config* cfg, float* d, float* u) {
    return guard([&] {
        RawSampleBlock blk;
        blk.samples.assign(iq, iq + 2 * n_complex);
        blk.start_time = start;
        blk.sample_rate = cfg->mod.sample_rate;
        PlanCache cache;
        auto r = demodulate_window(blk, to_cfg(*cfg), cache);
        std::memcpy(d, r.d.data(), r.d.size() * sizeof(float));
        std::memcpy(u, r.u.data(), r.u.size() * sizeof(float));
    });
}

// demodulate_signal (proj/src/dsp.cpp:159-191) on interleaved complex input.
int tdref_demodulate_signal(const float* x, uint64_t n, int64_t start, double lo_freq,
                            const tdg_demod_config* cfg, float* d, float* u) {
    return guard([&] {
        std::vector<cfloat> xs(reinterpret_cast<const cfloat*>(x), reinterpret_cast<const cfloat*>(x) + n);
        PlanCache cache;
        auto r = demodulate_signal(xs, start, lo_freq, to_cfg(*cfg), cache);
        std::memcpy(d, r.d.data(), r.d.size() * sizeof(float));
        std::memcpy(u, r.u.data(), r.u.size() * sizeof(float));
    });
}

// overlap_add_filter (proj/src/dsp.cpp:137-145), Full mode.
int tdref_overlap_add(const float* x, uint64_t n, const float* h, uint64_t m, float* out) {
    return guard([&] {
        std::vector<cfloat> xs(reinterpret_cast<const cfloat*>(x), reinterpret_cast<const cfloat*>(x) + n);
        FirFilter f;
        f.coeffs.assign(reinterpret_cast<const cfloat*>(h), reinterpret_cast<const cfloat*>(h) + m);
        PlanCache cache;
        auto y = overlap_add_filter(xs, f, cache, ConvMode::Full);
        std::memcpy(out, y.data(), y.size() * sizeof(cfloat));
    });
}

// Composed demod filters exactly as demodulate_signal builds them
// (proj/src/dsp.cpp:170-178): h1c = bandpass * matched(freq_one), h0c likewise.
int tdref_composed_filters(const tdg_demod_config* c, float* h1c, float* h0c) {
    return guard([&] {
        auto cfg = to_cfg(*c);
        auto bp = design_bandpass(cfg.bandpass_center, cfg.bandpass_width, cfg.bandpass_taps,
                                  cfg.mod.sample_rate);
        auto [m1, m0] = matched_filters(cfg.mod);
        auto a = compose(bp, m1);
        auto b = compose(bp, m0);
        std::memcpy(h1c, a.coeffs.data(), a.coeffs.size() * sizeof(cfloat));
        std::memcpy(h0c, b.coeffs.data(), b.coeffs.size() * sizeof(cfloat));
    });
}

tdref_session* tdref_session_new(void) { return new tdref_session(); }
void tdref_session_free(tdref_session* s) { delete s; }

// prepare_code (proj/src/detector.cpp:50-66); returns code index or -status.
int64_t tdref_session_prepare_code(tdref_session* s, const uint8_t* bits, uint64_t nbits,
                                   const tdg_demod_config* cfg, uint64_t window_len,
                                   const char* tag_id) {
    int64_t idx = -1;
    int rc = guard([&] {
        TagCode code;
        code.tag_id = tag_id;
        code.mod = to_mod(cfg->mod);
        code.bits.assign(bits, bits + nbits);
        WindowShape shape{size_t(window_len), to_cfg(*cfg)};
        const auto& tc = prepare_code(code, shape, s->cache, s->codes);
        s->index.push_back(&tc);
        idx = int64_t(s->index.size() - 1);
    });
    return rc ? -rc : idx;
}

// make_transformed (proj/src/detector.cpp:11-48).
int64_t tdref_session_make_transformed(tdref_session* s, const float* replica_d,
                                       const float* replica_u, uint64_t len, uint64_t window_len,
                                       uint64_t corr_len) {
    int64_t idx = -1;
    int rc = guard([&] {
        auto tc = std::make_unique<TransformedCode>(make_transformed(
            "x" + std::to_string(s->index.size()), std::span<const float>(replica_d, len),
            std::span<const float>(replica_u, replica_u ? len : 0), size_t(window_len),
            size_t(corr_len), s->cache));
        s->index.push_back(tc.get());
        s->owned.push_back(std::move(tc));
        idx = int64_t(s->index.size() - 1);
    });
    return rc ? -rc : idx;
}

int tdref_session_code_info(tdref_session* s, int64_t idx, uint64_t* nonzero_len, float* energy,
                            float* abs_sum, uint64_t* corr_len) {
    return guard([&] {
        const auto* tc = s->index.at(size_t(idx));
        *nonzero_len = tc->nonzero_len;
        *energy = tc->energy;
        *abs_sum = tc->abs_sum;
        *corr_len = tc->spectrum.size();
    });
}

int tdref_session_code_replica(tdref_session* s, int64_t idx, float* out_d) {
    return guard([&] {
        const auto* tc = s->index.at(size_t(idx));
        std::memcpy(out_d, tc->replica_d.data(), tc->replica_d.size() * sizeof(float));
    });
}

int tdref_session_code_spectrum(tdref_session* s, int64_t idx, float* out) {
    return guard([&] {
        const auto* tc = s->index.at(size_t(idx));
        std::memcpy(out, tc->spectrum.data(), tc->spectrum.size() * sizeof(cfloat));
    });
}

// batch_xcorr (proj/src/detector.cpp:102-120); out is n_idx x W row-major.
int tdref_session_batch_xcorr(tdref_session* s, const float* d, uint64_t W, const int64_t* idx,
                              uint64_t n_idx, float* out) {
    return guard([&] {
        std::vector<const TransformedCode*> codes;
        for (uint64_t i = 0; i < n_idx; ++i) codes.push_back(s->index.at(size_t(idx[i])));
        auto xs = batch_xcorr(std::span<const float>(d, W), codes, s->cache);
        for (uint64_t i = 0; i < n_idx; ++i) std::memcpy(out + i * W, xs[i].data(), W * sizeof(float));
    });
}

// detect (proj/src/detector.cpp:167-206); one record per code, in order.
int tdref_session_detect(tdref_session* s, const float* d, const float* u, uint64_t W,
                         const int64_t* idx, uint64_t n_idx, float threshold, int64_t window_start,
                         double sample_rate, int32_t bin, tdg_detection* out) {
    return guard([&] {
        std::vector<const TransformedCode*> codes;
        for (uint64_t i = 0; i < n_idx; ++i) codes.push_back(s->index.at(size_t(idx[i])));
        DetectionConfig dc{threshold, window_start};
        auto dets = detect(std::span<const float>(d, W), std::span<const float>(u, W), codes, dc,
                           sample_rate, s->cache);
        for (uint64_t i = 0; i < n_idx; ++i) fill_detection(dets[i], int32_t(idx[i]), bin, window_start, out + i);
    });
}

// find_peak / interpolate_peak / statistics (proj/src/detector.cpp:122-165).
int tdref_find_peak(const float* xc, uint64_t n, uint64_t* j, float* value) {
    return guard([&] {
        auto [jj, v] = find_peak(std::span<const float>(xc, n));
        *j = jj;
        *value = v;
    });
}

float tdref_interpolate_peak(const float* xc, uint64_t n, uint64_t j) {
    return interpolate_peak(std::span<const float>(xc, n), size_t(j));
}

// CPU reference arm / baseline: the detect_recording loop
// (proj/src/recording.cpp:258-289) over `n_windows` windows of the stream
// and `n_bins` lo_freq values, with all codes, spread over `threads` host
// threads.  Each thread owns its PlanCache/CodeCache (the reference's
// single-owner contract, proj/include/tagdsp/fft.hpp:13-16) and processes
// whole (window, bin, code-chunk) tasks.  Code preparation is done before
// timing (it is the one-time prepare_code of detect_recording :271-274).
// Returns the wall time of the timed region in seconds (<0 on error) and
// writes n_windows*n_bins*n_codes detections ordered [window][bin][code].
double tdref_search_bench(const int16_t* iq, uint64_t n_complex, int64_t stream_start,
                          const tdg_demod_config* cfg, const double* lo_bins, uint64_t n_bins,
                          const uint8_t* bits, uint64_t n_codes, uint64_t window_len,
                          uint64_t advance, uint64_t n_windows, float threshold, int threads,
                          int code_chunk, tdg_detection* out) {
    double elapsed = -1.0;
    int rc = guard([&] {
        if (threads < 1) threads = 1;
        if (code_chunk < 1) code_chunk = int(n_codes);
        if (n_windows && (n_windows - 1) * advance + window_len > n_complex)
            throw std::invalid_argument("search_bench: windows exceed the stream");
        DemodConfig base = to_cfg(*cfg);
        uint64_t nbits = cfg->mod.packet_bits;
        // per-thread contexts with codes prepared up front (untimed)
        struct Ctx {
            PlanCache cache;
            CodeCache codes;
            std::vector<const TransformedCode*> tcs;
        };
        std::vector<std::unique_ptr<Ctx>> ctx(static_cast<size_t>(threads));
        std::vector<std::thread> prep;
        std::vector<std::string> errs(static_cast<size_t>(threads));
        for (int t = 0; t < threads; ++t) {
            ctx[size_t(t)] = std::make_unique<Ctx>();
            prep.emplace_back([&, t] {
                try {
                    WindowShape shape{size_t(window_len), base};
                    for (uint64_t c = 0; c < n_codes; ++c) {
                        TagCode code;
                        code.tag_id = "t" + std::to_string(c);
                        code.mod = base.mod;
                        code.bits.assign(bits + c * nbits, bits + (c + 1) * nbits);
                        ctx[size_t(t)]->tcs.push_back(&prepare_code(code, shape, ctx[size_t(t)]->cache, ctx[size_t(t)]->codes));
                    }
                } catch (const std::exception& e) {
                    errs[size_t(t)] = e.what();
                }
            });
        }
        for (auto& th : prep) th.join();
        for (auto& e : errs)
            if (!e.empty()) throw std::runtime_error(e);

        uint64_t chunks = (n_codes + uint64_t(code_chunk) - 1) / uint64_t(code_chunk);
        uint64_t n_tasks = n_windows * n_bins * chunks;
        std::atomic<uint64_t> next{0};
        auto t0 = std::chrono::steady_clock::now();
        std::vector<std::thread> pool;
        for (int t = 0; t < threads; ++t) {
            pool.emplace_back([&, t] {
                Ctx& c = *ctx[size_t(t)];
                try {
                    for (;;) {
                        uint64_t task = next.fetch_add(1);
                        if (task >= n_tasks) break;
                        uint64_t w = task / (n_bins * chunks);
                        uint64_t b = (task / chunks) % n_bins;
                        uint64_t ch = task % chunks;
                        uint64_t start = w * advance;
                        RawSampleBlock blk;
                        blk.sample_rate = base.mod.sample_rate;
                        blk.start_time = stream_start + int64_t(start);
                        blk.samples.assign(iq + 2 * start, iq + 2 * (start + window_len));
                        DemodConfig dcfg = base;
                        dcfg.lo_freq = lo_bins[b];
                        auto demod = demodulate_window(blk, dcfg, c.cache);
                        uint64_t c0 = ch * uint64_t(code_chunk);
                        uint64_t c1 = std::min(n_codes, c0 + uint64_t(code_chunk));
                        std::span<const TransformedCode* const> sub(c.tcs.data() + c0, c1 - c0);
                        DetectionConfig dc{threshold, blk.start_time};
                        auto dets = detect(demod.d, demod.u, sub, dc, base.mod.sample_rate, c.cache);
                        for (uint64_t k = 0; k < dets.size(); ++k)
                            fill_detection(dets[k], int32_t(c0 + k), int32_t(b), blk.start_time,
                                           out + (w * n_bins + b) * n_codes + c0 + k);
                    }
                } catch (const std::exception& e) {
                    errs[size_t(t)] = e.what();
                }
            });
        }
        for (auto& th : pool) th.join();
        auto t1 = std::chrono::steady_clock::now();
        for (auto& e : errs)
            if (!e.empty()) throw std::runtime_error(e);
        elapsed = std::chrono::duration<double>(t1 - t0).count();
    });
    return rc ? -double(rc) : elapsed;
}

// CPU reference arm, like for like with the reference's own loop
// (proj/src/recording.cpp:277-286): ONE demodulate_window per (window, bin),
// shared by every code, then detect() over the codes.  Spread over `threads`
// host threads in two phases: (1) the (window, bin) demodulations, (2)
// detect() over (window, bin, chunk of code_chunk codes) tasks, each thread
// with its own PlanCache (fft.hpp:13-16).  Codes are prepared before timing,
// split over the threads (each TransformedCode is read-only afterwards).
// stage_s (optional, 3 doubles) receives summed thread-seconds of
// demodulation, correlation and peak+statistics (DetectTimings,
// detector.hpp:95-98; the split of harness.hpp:7-11).  Returns the wall time
// of the two phases in seconds (<0 on error); detections [window][bin][code].
double tdref_search_bench_shared(const int16_t* iq, uint64_t n_complex, int64_t stream_start,
                                 const tdg_demod_config* cfg, const double* lo_bins, uint64_t n_bins,
                                 const uint8_t* bits, uint64_t n_codes, uint64_t window_len,
                                 uint64_t advance, uint64_t n_windows, float threshold, int threads,
                                 int code_chunk, tdg_detection* out, double* stage_s) {
    double elapsed = -1.0;
    int rc = guard([&] {
        if (threads < 1) threads = 1;
        if (code_chunk < 1) code_chunk = int(n_codes);
        if (n_windows && (n_windows - 1) * advance + window_len > n_complex)
            throw std::invalid_argument("search_bench: windows exceed the stream");
        const DemodConfig base = to_cfg(*cfg);
        const uint64_t nbits = cfg->mod.packet_bits;
        struct Ctx {
            PlanCache cache;
            CodeCache codes;
            double demod_s = 0, corr_s = 0, peak_s = 0;
        };
        std::vector<std::unique_ptr<Ctx>> ctx(static_cast<size_t>(threads));
        for (auto& c : ctx) c = std::make_unique<Ctx>();
        std::vector<const TransformedCode*> tcs(n_codes, nullptr);
        std::vector<std::string> errs(static_cast<size_t>(threads));
        auto run = [&](auto&& body) {
            std::vector<std::thread> pool;
            for (int t = 0; t < threads; ++t)
                pool.emplace_back([&, t] {
                    try {
                        body(t);
                    } catch (const std::exception& e) {
                        errs[size_t(t)] = e.what();
                    }
                });
            for (auto& th : pool) th.join();
            for (auto& e : errs)
                if (!e.empty()) throw std::runtime_error(e);
        };
        run([&](int t) {   // untimed: prepare_code (detect_recording :271-274), codes split over threads
            WindowShape shape{size_t(window_len), base};
            for (uint64_t c = uint64_t(t); c < n_codes; c += uint64_t(threads)) {
                TagCode code;
                code.tag_id = "t" + std::to_string(c);
                code.mod = base.mod;
                code.bits.assign(bits + c * nbits, bits + (c + 1) * nbits);
                tcs[c] = &prepare_code(code, shape, ctx[size_t(t)]->cache, ctx[size_t(t)]->codes);
            }
        });
        const uint64_t n_slots = n_windows * n_bins;
        std::vector<DemodResult> demod(n_slots);
        const uint64_t chunks = (n_codes + uint64_t(code_chunk) - 1) / uint64_t(code_chunk);
        std::atomic<uint64_t> next{0};
        const auto t0 = std::chrono::steady_clock::now();
        run([&](int t) {   // phase 1: one demodulation per (window, bin)
            Ctx& c = *ctx[size_t(t)];
            for (;;) {
                const uint64_t slot = next.fetch_add(1);
                if (slot >= n_slots) break;
                const uint64_t w = slot / n_bins, b = slot % n_bins, start = w * advance;
                const auto a = std::chrono::steady_clock::now();
                RawSampleBlock blk;
                blk.sample_rate = base.mod.sample_rate;
                blk.start_time = stream_start + int64_t(start);
                blk.samples.assign(iq + 2 * start, iq + 2 * (start + window_len));
                DemodConfig dcfg = base;
                dcfg.lo_freq = lo_bins[b];
                demod[slot] = demodulate_window(blk, dcfg, c.cache);
                c.demod_s += std::chrono::duration<double>(std::chrono::steady_clock::now() - a).count();
            }
        });
        next = 0;
        run([&](int t) {   // phase 2: detect over code chunks of every slot
            Ctx& c = *ctx[size_t(t)];
            for (;;) {
                const uint64_t task = next.fetch_add(1);
                if (task >= n_slots * chunks) break;
                const uint64_t slot = task / chunks, ch = task % chunks;
                const uint64_t w = slot / n_bins, b = slot % n_bins;
                const int64_t ws = stream_start + int64_t(w * advance);
                const uint64_t c0 = ch * uint64_t(code_chunk), c1 = std::min(n_codes, c0 + uint64_t(code_chunk));
                std::span<const TransformedCode* const> sub(tcs.data() + c0, c1 - c0);
                DetectTimings tm;
                auto dets = detect(demod[slot].d, demod[slot].u, sub, DetectionConfig{threshold, ws},
                                   base.mod.sample_rate, c.cache, &tm);
                c.corr_s += tm.correlation_s;
                c.peak_s += tm.peak_stats_s;
                for (uint64_t k = 0; k < dets.size(); ++k)
                    fill_detection(dets[k], int32_t(c0 + k), int32_t(b), ws, out + slot * n_codes + c0 + k);
            }
        });
        elapsed = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        if (stage_s) {
            stage_s[0] = stage_s[1] = stage_s[2] = 0.0;
            for (auto& c : ctx) {
                stage_s[0] += c->demod_s;
                stage_s[1] += c->corr_s;
                stage_s[2] += c->peak_s;
            }
        }
    });
    return rc ? -double(rc) : elapsed;
}

// Tracking tasks on the CPU (the Tracking branch of simulate_recording,
// proj/src/recording.cpp:360-378): per task demodulate_window of
// [start, start + window_len) at cfg->lo_freq, then detect() against its one
// code prepared for the tracking shape.  Single thread (the reference's
// scheduler is sequential, scheduler.hpp:90-92).  Returns seconds of the
// timed loop (<0 on error); out[i] = task i's Detection.
double tdref_track_bench(const int16_t* iq, uint64_t n_complex, int64_t stream_start, const tdg_demod_config* cfg,
                         const uint8_t* bits, uint64_t n_codes, uint64_t window_len, const int64_t* starts,
                         const uint64_t* code_idx, uint64_t n_tasks, float threshold, tdg_detection* out) {
    double elapsed = -1.0;
    int rc = guard([&] {
        const DemodConfig base = to_cfg(*cfg);
        const uint64_t nbits = cfg->mod.packet_bits;
        PlanCache cache;
        CodeCache codes;
        std::vector<const TransformedCode*> tcs(n_codes);
        WindowShape shape{size_t(window_len), base};
        for (uint64_t c = 0; c < n_codes; ++c) {
            TagCode code;
            code.tag_id = "t" + std::to_string(c);
            code.mod = base.mod;
            code.bits.assign(bits + c * nbits, bits + (c + 1) * nbits);
            tcs[c] = &prepare_code(code, shape, cache, codes);
        }
        const auto t0 = std::chrono::steady_clock::now();
        for (uint64_t i = 0; i < n_tasks; ++i) {
            const int64_t s0 = starts[i];
            if (s0 < stream_start || uint64_t(s0 - stream_start) + window_len > n_complex)
                throw std::invalid_argument("track_bench: task window outside the block");
            if (code_idx[i] >= n_codes) throw std::invalid_argument("track_bench: code index");
            RawSampleBlock blk;
            blk.sample_rate = base.mod.sample_rate;
            blk.start_time = s0;
            const uint64_t off = uint64_t(s0 - stream_start);
            blk.samples.assign(iq + 2 * off, iq + 2 * (off + window_len));
            auto demod = demodulate_window(blk, base, cache);
            const TransformedCode* one[1] = {tcs[code_idx[i]]};
            auto dets = detect(demod.d, demod.u, std::span<const TransformedCode* const>(one, 1),
                               DetectionConfig{threshold, s0}, base.mod.sample_rate, cache);
            fill_detection(dets[0], int32_t(code_idx[i]), 0, s0, out + i);
        }
        elapsed = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    });
    return rc ? -double(rc) : elapsed;
}

// detect_recording / simulate_recording (proj/src/recording.cpp:258-389) on
// a recording file + run-config file, output as the reference's JSON lines
// (detection_json_line / event_json_line) -- the oracle side of the drop-in
// tests (tests/test_gpu_dropin.py).
int tdref_run_detect_recording(const char* rec_path, const char* cfg_path, const char* out_path) {
    return guard([&] {
        auto rec = read_recording(rec_path);
        auto cfg = load_run_config(cfg_path);
        auto dets = detect_recording(rec, cfg);
        std::ofstream out(out_path);
        for (const auto& d : dets) out << detection_json_line(d) << "\n";
    });
}

int tdref_run_simulate(const char* rec_path, const char* cfg_path, const char* out_path, double compute_ratio,
                       uint64_t* detections, uint64_t* misses) {
    return guard([&] {
        auto rec = read_recording(rec_path);
        auto cfg = load_run_config(cfg_path);
        auto res = simulate_recording(rec, cfg, compute_ratio);
        std::ofstream out(out_path);
        for (const auto& e : res.events) out << event_json_line(e) << "\n";
        *detections = res.detections;
        *misses = res.misses;
    });
}

// write_recording / read_recording / detection_json_line
// (proj/src/recording.cpp:23-64,228-242) for the recording-format cross-checks
int tdref_write_recording(const char* path, const int16_t* iq, uint64_t n_complex, double sample_rate,
                          int64_t start_time, double center_freq, const char* creator) {
    return guard([&] {
        RecordingFile rec;
        rec.block.samples.assign(iq, iq + 2 * n_complex);
        rec.block.sample_rate = sample_rate;
        rec.block.start_time = start_time;
        rec.center_freq = center_freq;
        rec.creator = creator;
        write_recording(path, rec);
    });
}

int tdref_read_recording(const char* path, int16_t* iq, uint64_t cap_int16, uint64_t* n_complex, double* sample_rate,
                         int64_t* start_time, double* center_freq, char* creator, uint64_t creator_cap) {
    return guard([&] {
        auto rec = read_recording(path);
        *n_complex = rec.block.num_complex();
        if (rec.block.samples.size() > cap_int16) throw std::runtime_error("read_recording: buffer too small");
        std::memcpy(iq, rec.block.samples.data(), rec.block.samples.size() * sizeof(int16_t));
        *sample_rate = rec.block.sample_rate;
        *start_time = rec.block.start_time;
        *center_freq = rec.center_freq;
        std::snprintf(creator, creator_cap, "%s", rec.creator.c_str());
    });
}

int tdref_detection_json_line(const tdg_detection* r, const char* tag_id, char* out, uint64_t cap) {
    return guard([&] {
        Detection d;
        d.tag_id = tag_id;
        d.peak_index = size_t(r->peak_index);
        d.subsample_offset = r->subsample_offset;
        d.toa_seconds = r->toa_seconds;
        d.peak_value = r->peak_value;
        d.w_c = r->w_c;
        d.q = r->q;
        d.p_c = r->p_c;
        d.score = r->score;
        d.accepted = r->accepted != 0;
        d.partial = r->partial != 0;
        std::snprintf(out, cap, "%s", detection_json_line(d).c_str());
    });
}

// CircularBuffer (proj/src/scheduler.cpp:7-45): create / push / read / bounds,
// the oracle of the device ring tdg_ring_* (tests/test_gpu_ring.py)
void* tdref_ring_new(uint64_t capacity) { return new CircularBuffer(size_t(capacity)); }
void tdref_ring_free(void* r) { delete static_cast<CircularBuffer*>(r); }
int tdref_ring_push(void* r, const int16_t* iq, uint64_t n_complex, int64_t start, int64_t* ev_begin, int64_t* ev_end,
                    int32_t* gap) {
    return guard([&] {
        RawSampleBlock blk;
        blk.samples.assign(iq, iq + 2 * n_complex);
        blk.start_time = start;
        auto res = static_cast<CircularBuffer*>(r)->push(blk);
        *ev_begin = res.evicted_begin;
        *ev_end = res.evicted_end;
        *gap = res.gap ? 1 : 0;
    });
}
int tdref_ring_read(void* r, int64_t start, int64_t end, int16_t* out, int32_t* ok) {
    return guard([&] {
        std::vector<int16_t> v;
        *ok = static_cast<CircularBuffer*>(r)->read(start, end, v) ? 1 : 0;
        if (*ok) std::memcpy(out, v.data(), v.size() * sizeof(int16_t));
    });
}
void tdref_ring_bounds(void* r, int64_t* head, int64_t* tail) {
    *head = static_cast<CircularBuffer*>(r)->head();
    *tail = static_cast<CircularBuffer*>(r)->tail();
}

}  // extern "C"
