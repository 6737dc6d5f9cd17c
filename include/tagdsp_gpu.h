/* tagdsp_gpu.h -- C-ABI of the B200-native acquisition (searching) hot path.
 *
 * Drop-in replacement for the reference tagdsp detector path
 * (/root/reference/proj): sample block in, per-tag detections out.  The
 * reference has no FFI layer (a C++20 static library, proj/src/CMakeLists.txt:1-12);
 * each entry point below names the reference function it replaces, and the
 * header-only C++ wrapper include/tagdsp_gpu.hpp restores the reference
 * signatures on top of it.  Plain pointers and sizes only; no torch or CUDA
 * types.  Every call returns TDG_OK (0) or an error code from
 * tagdsp_gpu_types.h, with a message in tdg_last_error().
 *
 * Objects (all device-resident, "allocate once, reuse" like PlanCache,
 * proj/include/tagdsp/fft.hpp:13-16):
 *   tdg_ctx      one CUDA device + stream + FFT plans/tables (~ PlanCache)
 *   tdg_codeset  prepared codes for one window shape (~ CodeCache entries,
 *                proj/include/tagdsp/detector.hpp:26-37)
 *   tdg_windows  demodulated windows d,u for W samples x (windows x bins)
 *                (~ DemodResult, proj/include/tagdsp/dsp.hpp:62-65)
 */
#ifndef TAGDSP_GPU_H
#define TAGDSP_GPU_H
#include <stddef.h>
#include <stdint.h>

#include "tagdsp_gpu_types.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct tdg_ctx tdg_ctx;
typedef struct tdg_codeset tdg_codeset;
typedef struct tdg_windows tdg_windows;
typedef struct tdg_ring tdg_ring;

/* Message for the last failing call on this host thread. */
const char* tdg_last_error(void);
/* Library version string and number of CUDA kernels launched by this
 * process (all contexts) -- used by bench.py's gpu_launches accounting. */
const char* tdg_version(void);
uint64_t tdg_kernel_launches(void);

/* PlanCache construction (proj/src/fft.cpp:27-44 creates plans lazily; here
 * the context owns the stream and the twiddle tables of every supported
 * transform length). */
int tdg_ctx_create(int device, tdg_ctx** out);
void tdg_ctx_destroy(tdg_ctx* ctx);
int tdg_ctx_synchronize(tdg_ctx* ctx);
/* Raw cudaStream_t of the context (opaque pointer), for event timing. */
void* tdg_ctx_stream(tdg_ctx* ctx);

/* pad_length (proj/src/fft.cpp:93-101): smallest {2,3,5,7}-smooth m >= n. */
uint64_t tdg_pad_length(uint64_t n);
/* Transform length the B200 path uses for a correlation that must be linear
 * over lags [0, window_len) for supports up to nonzero_len: the smallest
 * supported N1*N2 >= window_len + nonzero_len - 1 (0 if unsupported).  Any
 * such length gives the same lags as the reference's corr_len
 * (proj/include/tagdsp/detector.hpp:19-21); only rounding differs. */
uint64_t tdg_corr_len(uint64_t window_len, uint64_t nonzero_len);

/* ---- codes ---------------------------------------------------------------
 * prepare_code (proj/src/detector.cpp:50-66) for n_codes codes at once, all
 * on the GPU: synth_replica (proj/src/codegen.cpp:40-60) -> demodulation
 * with lo_freq = 0 (proj/src/dsp.cpp:159-191) -> support / energy / abs_sum
 * (proj/src/detector.cpp:20-43) -> forward FFT of the zero-padded replica d
 * (:45-47).  bits is n_codes x cfg->mod.packet_bits bytes (0/1).
 * Errors as the reference: window_len < packet_samples -> TDG_EINVAL;
 * beyond the reference: window_len + support - 1 > 1,048,576 (the largest
 * instantiated transform, tdg_corr_len() == 0) -> TDG_ERANGE. */
int tdg_codeset_prepare(tdg_ctx* ctx, const tdg_demod_config* cfg, uint64_t window_len,
                        const uint8_t* bits, uint64_t n_codes, tdg_codeset** out);
/* make_transformed (proj/src/detector.cpp:11-48) from host replicas:
 * replica_d/replica_u are n_codes pointers to `lengths[i]` floats
 * (replica_u may be NULL -> support measured on d).  corr_len is the
 * reference's transform length and is only used for its precondition
 * (window_len + n <= corr_len + 1, else TDG_EINVAL). */
/* prepare_code for n_codes more codes of the same configuration, appended to
 * cs (indices n .. n + n_codes - 1): only the stored pairs the new codes touch
 * are transformed (all of them if a longer support needs a longer transform);
 * device buffers grow by doubling.  TDG_EINVAL for a code set made by
 * make_transformed or prepared with another configuration. */
int tdg_codeset_append(tdg_ctx* ctx, tdg_codeset* cs, const tdg_demod_config* cfg, const uint8_t* bits,
                       uint64_t n_codes);
int tdg_codeset_from_replicas(tdg_ctx* ctx, uint64_t window_len, uint64_t corr_len,
                              const float* const* replica_d, const float* const* replica_u,
                              const uint64_t* lengths, uint64_t n_codes, tdg_codeset** out);
void tdg_codeset_destroy(tdg_codeset* cs);
uint64_t tdg_codeset_size(const tdg_codeset* cs);
/* TransformedCode fields (proj/include/tagdsp/detector.hpp:26-35). */
int tdg_codeset_info(const tdg_codeset* cs, uint64_t idx, uint64_t* nonzero_len, float* energy,
                     float* abs_sum, uint64_t* corr_len);
int tdg_codeset_replica(const tdg_codeset* cs, uint64_t idx, float* replica_d_out);

/* ---- windows -------------------------------------------------------------
 * Storage for n_windows x n_bins demodulated windows of window_len samples. */
int tdg_windows_create(tdg_ctx* ctx, uint64_t window_len, uint64_t n_windows, uint64_t n_bins,
                       tdg_windows** out);
void tdg_windows_destroy(tdg_windows* w);
/* demodulate_window (proj/src/dsp.cpp:193-197) for every window w < n_windows
 * starting at stream sample w*advance of `iq` (interleaved int16 I,Q, HOST
 * memory, n_complex samples, absolute start index stream_start) and every
 * lo_freq in lo_bins (the frequency-offset sweep; the reference's single
 * DemodConfig::lo_freq is lo_bins[0] with n_bins = 1).  Slot of (w, b) is
 * w*n_bins + b.  cfg->lo_freq is ignored (the bins replace it). */
int tdg_demodulate(tdg_ctx* ctx, tdg_windows* win, const tdg_demod_config* cfg,
                   const double* lo_bins, uint64_t n_bins, const int16_t* iq, uint64_t n_complex,
                   int64_t stream_start, uint64_t advance, uint64_t n_windows);
/* Same as tdg_demodulate but `iq_dev` is a device pointer (already resident). */
int tdg_demodulate_device(tdg_ctx* ctx, tdg_windows* win, const tdg_demod_config* cfg,
                          const double* lo_bins, uint64_t n_bins, const int16_t* iq_dev,
                          uint64_t n_complex, int64_t stream_start, uint64_t advance,
                          uint64_t n_windows);
/* detect(d, u, ...) entry: upload a host d,u pair into a slot. */
int tdg_windows_set_du(tdg_ctx* ctx, tdg_windows* w, uint64_t slot, const float* d, const float* u,
                       int64_t window_start);
int tdg_windows_get_du(tdg_ctx* ctx, const tdg_windows* w, uint64_t slot, float* d, float* u);
/* DetectionConfig::window_start of a slot whose d,u are already on the device. */
int tdg_windows_set_start(tdg_ctx* ctx, tdg_windows* w, uint64_t slot, int64_t window_start);

/* ---- detection -----------------------------------------------------------
 * detect (proj/src/detector.cpp:167-206) for every slot x code: one forward
 * FFT per slot, then per (slot, code) the fused spectral product + inverse
 * FFT + |xc| first-index argmax (the xc vector never reaches HBM), then
 * parabolic refinement, (w_c, q, p_c) statistics, score, ToA and accept.
 * out receives n_slots*n_codes records ordered [slot][code] (slot = window *
 * n_bins + bin) in HOST memory (out_cap >= n_slots*n_codes, else TDG_EINVAL;
 * out may be NULL: records stay on the device).  toa uses each slot's
 * window_start. */
int tdg_detect(tdg_ctx* ctx, tdg_windows* w, const tdg_codeset* cs, float threshold,
               double sample_rate, tdg_detection* out, uint64_t out_cap);
/* detect() over a subset of the code set -- the reference's
 * span<const TransformedCode* const> (detector.hpp:103-106): records
 * [slot][k] for code idx[k] (repeats allowed); only the stored code pairs the
 * subset touches are correlated.  out may be NULL (records stay on the
 * device); else out_cap >= n_slots*n_idx. */
int tdg_detect_codes(tdg_ctx* ctx, tdg_windows* w, const tdg_codeset* cs, const int64_t* idx,
                     uint64_t n_idx, float threshold, double sample_rate, tdg_detection* out,
                     uint64_t out_cap);
/* batch_xcorr (proj/src/detector.cpp:102-120) for one slot: the full xc
 * (lags [0, W)) of each requested code, normalised like the reference
 * inverse (1/N), into HOST out (n_idx x W).  Test/diagnostic path. */
int tdg_batch_xcorr(tdg_ctx* ctx, tdg_windows* w, uint64_t slot, const tdg_codeset* cs,
                    const int64_t* idx, uint64_t n_idx, float* out);

/* ---- whole searching pass ------------------------------------------------
 * detect_recording (proj/src/recording.cpp:258-289) with a frequency-offset
 * sweep: windows of window_len every `advance` samples over a HOST int16
 * stream, every code x every bin.  H2D of the stream, demodulation, all
 * correlations, statistics and the D2H of the detections happen inside.
 * out must hold n_windows*n_bins*n_codes records, n_windows =
 * (n_complex >= window_len) ? (n_complex - window_len)/advance + 1 : 0. */
int tdg_search(tdg_ctx* ctx, const tdg_demod_config* cfg, const double* lo_bins, uint64_t n_bins,
               const int16_t* iq, uint64_t n_complex, int64_t stream_start, uint64_t window_len,
               uint64_t advance, const tdg_codeset* cs, float threshold, tdg_detection* out,
               uint64_t out_cap, uint64_t* n_out);

/* Tracking mode: a batch of short windows, one code each (what
 * proj/src/recording.cpp:360-378 does per Tracking task: demodulate_window
 * at cfg->lo_freq, prepare_code(track_shape) -> detect with that one code).
 * iq covers stream samples [stream_start, stream_start + n_complex); every
 * task window must lie inside it; the code set must be prepared for the
 * tracking window length.  out[i] is task i's Detection (accepted or not).
 * _device: iq is a device pointer (e.g. a device-resident ring buffer). */
int tdg_track(tdg_ctx* ctx, const tdg_demod_config* cfg, const int16_t* iq, uint64_t n_complex,
              int64_t stream_start, const tdg_track_task* tasks, uint64_t n_tasks, const tdg_codeset* cs,
              float threshold, tdg_detection* out);
int tdg_track_device(tdg_ctx* ctx, const tdg_demod_config* cfg, const int16_t* iq_dev, uint64_t n_complex,
                     int64_t stream_start, const tdg_track_task* tasks, uint64_t n_tasks,
                     const tdg_codeset* cs, float threshold, tdg_detection* out);

/* Device-resident CircularBuffer (tagdsp::CircularBuffer,
 * include/tagdsp/scheduler.hpp:11-40; proj/src/scheduler.cpp:7-45): the raw
 * stream addressed by absolute sample index, same push (gap resync,
 * eviction) and read semantics.  Pushes are asynchronous host->device copies
 * on the ring's own stream; searches and tracking tasks read windows straight
 * from the ring (no per-task copy, cf. the reference's read() into a vector)
 * and a later push waits only for the reads whose slots it overwrites.
 * Host buffers passed to push must stay valid until the copy completes
 * (pinned memory: until a later synchronisation). */
int tdg_ring_create(tdg_ctx* ctx, uint64_t capacity_samples, tdg_ring** out);
void tdg_ring_destroy(tdg_ring* ring);
int tdg_ring_push(tdg_ring* ring, const int16_t* iq, uint64_t n_complex, int64_t start,
                  tdg_ring_push_result* result);
int tdg_ring_read(tdg_ring* ring, int64_t start, int64_t end, int16_t* out, int* ok);
int tdg_ring_bounds(const tdg_ring* ring, int64_t* head, int64_t* tail, uint64_t* capacity);
/* Searching pass over n_windows windows [first_start + w*advance, + window_len)
 * held by the ring (all bins x codes, records [window][bin][code]); sync = 0
 * leaves the Detection copy-out in flight on the context stream
 * (tdg_ctx_synchronize before reading `out`). */
int tdg_search_ring(tdg_ctx* ctx, tdg_ring* ring, const tdg_demod_config* cfg, const double* lo_bins,
                    uint64_t n_bins, int64_t first_start, uint64_t window_len, uint64_t advance,
                    uint64_t n_windows, const tdg_codeset* cs, float threshold, tdg_detection* out,
                    uint64_t out_cap, int sync);
int tdg_track_ring(tdg_ctx* ctx, tdg_ring* ring, const tdg_demod_config* cfg, const tdg_track_task* tasks,
                   uint64_t n_tasks, const tdg_codeset* cs, float threshold, tdg_detection* out, int sync);

/* ---- span-level functions of the reference API ----------------------------
 * Host arrays in and out, each a device round trip; the drop-in
 * (include/tagdsp_b200, libtagdsp_b200.so) maps the reference's free
 * functions onto them.  Complex arrays are interleaved float pairs. */
/* PlanCache::forward / inverse (proj/src/fft.cpp:46-67): C2C DFT of any
 * {2,3,5,7}-smooth length n (else TDG_ERANGE); inverse = +sign and 1/n. */
int tdg_fft(tdg_ctx* ctx, const float* in, float* out, uint64_t n, int inverse);
/* convert (proj/src/dsp.cpp:9-16): n_int16 interleaved I,Q -> n_int16/2 complex. */
int tdg_convert(tdg_ctx* ctx, const int16_t* iq, uint64_t n_int16, float* out);
/* mix (proj/src/dsp.cpp:18-33), in place; no-op for lo_freq == 0. */
int tdg_mix(tdg_ctx* ctx, float* x, uint64_t n, double lo_freq, int64_t start_index, double sample_rate);
/* full linear convolution of x (nx complex) with h (nh complex) -> nx+nh-1
 * complex (overlap_add_filter, proj/src/dsp.cpp:137-145, ConvMode::Full). */
int tdg_convolve(tdg_ctx* ctx, const float* x, uint64_t nx, const float* h, uint64_t nh, float* out);
/* demodulate (proj/src/dsp.cpp:147-157). */
int tdg_discriminate(tdg_ctx* ctx, const float* f1, const float* f0, uint64_t n, float eps, float* d, float* u);
/* find_peak (proj/src/detector.cpp:122-134): first index of max |xc|, signed value. */
int tdg_find_peak(tdg_ctx* ctx, const float* xc, uint64_t n, uint64_t* j, float* value);
/* statistics (proj/src/detector.cpp:147-165) of replica dc (n) at lag j of d,u (W). */
int tdg_statistics(tdg_ctx* ctx, const float* d, const float* u, uint64_t W, const float* dc, uint64_t n,
                   uint64_t j, float* w_c, float* q, float* p_c, int* partial);
/* demodulate_signal (proj/src/dsp.cpp:159-191) of n complex samples at
 * lo_freq into slot 0 of win (window length n). */
int tdg_demodulate_signal(tdg_ctx* ctx, tdg_windows* win, const tdg_demod_config* cfg, double lo_freq,
                          const float* x, uint64_t n, int64_t start_index);
/* DetectTimings (proj/include/tagdsp/detector.hpp:95-98) of the last detect
 * on this context when option "detect_timings" is 1 (CUDA events). */
int tdg_detect_timings(tdg_ctx* ctx, double* correlation_s, double* peak_stats_s);

/* detection_json_line (proj/src/recording.cpp:228-242): the record as the
 * reference's JSON line (byte-identical: same nlohmann::json dump) into out
 * (cap bytes incl. the terminator; *len = its length; TDG_EINVAL if short). */
int tdg_detection_json_line(const tdg_detection* det, const char* tag_id, char* out, uint64_t cap, uint64_t* len);

/* Tuning / profiling knobs (0 = default): "wave_pairs" (8), "ring" (3),
 * "n_streams" (6), "discard" (1), "fwd_wave" (32), "one_stream",
 * "cta_cap_a" / "cta_cap_b" (CTAs per SM of the two correlation passes of
 * this context; defaults 0 = occupancy / 2, and 0 sets no cap),
 * "time_kernels" (1 = record a CUDA event pair on the context stream around
 * every launch; read back with tdg_kernel_time), "track_graphs" (default 1:
 * tdg_track / tdg_track_device batches that fit one correlation wave are
 * captured as a CUDA graph on their second call with the same shape and
 * replayed from the third; 0 = always issue the launches), "detect_timings"
 * (1 = record the correlation / statistics split of every detect, read with
 * tdg_detect_timings).  Setting any
 * option drops the context's captured graphs. */
int tdg_set_option(tdg_ctx* ctx, const char* key, int64_t value);
/* Launch count and summed device time (ms) of one kernel family since the
 * last reset: "demod", "fwd_pass1", "fwd_pass2", "corr_passA", "corr_passB",
 * "stats".  Synchronises the context stream. */
int tdg_kernel_time(tdg_ctx* ctx, const char* name, uint64_t* count, double* total_ms);
int tdg_kernel_time_reset(tdg_ctx* ctx);
/* Diagnostics (option "cta_trace" = capacity > 0): the correlation-pass CTAs
 * recorded since the last call, 3 words each {smid << 8 | pass (0 = A, 1 = B),
 * globaltimer ns at CTA start, at CTA exit}; *n = records (all of them, even
 * beyond cap); the record count is reset.  Synchronises the device. */
int tdg_cta_trace(tdg_ctx* ctx, uint64_t* out, uint64_t cap, uint64_t* n);
/* FP32 issue-rate probe (bench.py's roofline denominator): TFLOP/s of scalar
 * FFMA and of packed FFMA2 on `device` at its current clock. */
int tdg_fp32_peak(int device, double* ffma_tflops, double* ffma2_tflops);

#ifdef __cplusplus
}
#endif
#endif
