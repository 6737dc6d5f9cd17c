/* Plain-old-data records shared by the B200 C-ABI (tagdsp_gpu.h) and the
 * CPU oracle / reference wrappers used by the parity tests.  Every field
 * mirrors a reference type field-for-field (citations are to
 * /root/reference/proj).  No torch or CUDA types appear here. */
#ifndef TAGDSP_GPU_TYPES_H
#define TAGDSP_GPU_TYPES_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* tagdsp::ModulationParams, include/tagdsp/types.hpp:24-40 */
typedef struct tdg_modulation {
    double sample_rate;   /* default 8e6 */
    double bit_rate;      /* default 1e6 */
    double freq_one;      /* default +250e3 */
    double freq_zero;     /* default -250e3 */
    uint64_t packet_bits; /* default 8192 */
} tdg_modulation;

/* tagdsp::DemodConfig, include/tagdsp/dsp.hpp:25-36 */
typedef struct tdg_demod_config {
    tdg_modulation mod;
    double lo_freq;          /* default 0 */
    double bandpass_center;  /* default 0 */
    double bandpass_width;   /* default 1.5e6 */
    uint64_t bandpass_taps;  /* default 200 */
    float eps;               /* default 1e-12f */
    uint32_t reserved;
} tdg_demod_config;

/* tagdsp::Detection, include/tagdsp/detector.hpp:39-51.  tag_id is replaced
 * by code_index (position in the code set; the C++ wrapper maps it back to
 * the tag id) and two fields are added for the batched B200 path: bin (the
 * frequency-offset bin, i.e. which lo_freq of the sweep) and window_start
 * (DetectionConfig::window_start of the window the record belongs to). */
typedef struct tdg_detection {
    int32_t code_index;
    int32_t bin;
    int64_t window_start;
    uint64_t peak_index;
    double toa_seconds;
    float subsample_offset;
    float peak_value;
    float w_c;
    float q;
    float p_c;
    float score;
    uint8_t accepted;
    uint8_t partial;
    uint8_t reserved[6];
} tdg_detection;

/* One tracking task (tagdsp::Task of kind Tracking, include/tagdsp/scheduler.hpp
 * and proj/src/scheduler.cpp:89-113): the window [start, start + window_len)
 * of the stream, searched for exactly one code. */
typedef struct tdg_track_task {
    int64_t start;         /* absolute stream index of the window's first sample */
    uint64_t code_index;   /* code in the code set (prepared for the tracking window length) */
} tdg_track_task;

/* tagdsp::CircularBuffer::PushResult, include/tagdsp/scheduler.hpp:18-24 */
typedef struct tdg_ring_push_result {
    int64_t evicted_begin;
    int64_t evicted_end;   /* == evicted_begin when nothing was evicted */
    int32_t gap;           /* the block did not continue the stream: resynchronised */
    int32_t reserved;
} tdg_ring_push_result;

/* Status codes of every C-ABI entry point (0 = ok).  The C++ wrapper maps
 * TDG_EINVAL to std::invalid_argument (the reference's precondition
 * exceptions) and everything else to std::runtime_error. */
enum {
    TDG_OK = 0,
    TDG_EINVAL = 1,   /* reference would throw std::invalid_argument */
    TDG_ECUDA = 2,    /* CUDA runtime / launch failure */
    TDG_ENOMEM = 3,   /* device or pinned-host allocation failed */
    TDG_ERANGE = 4,   /* shape outside what the B200 kernels support */
    TDG_EINTERNAL = 5
};

#ifdef __cplusplus
}
#endif
#endif
