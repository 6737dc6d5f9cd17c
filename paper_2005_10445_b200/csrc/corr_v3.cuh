// Correlation engine v3: the two inverse-FFT passes of every (window slot x
// code pair) correlation as two persistent, TMA-pipelined kernels per wave
// of `wave_pairs` pairs, waves alternating over n_streams pass-A and
// n_streams pass-B CUDA streams so that the passes of neighbouring waves
// overlap (no SM idles in a launch's ramp or tail):
//
//   correlate_spectrum (proj/src/detector.cpp:78-88)  ->  pass A
//   inverse FFT + find_peak (detector.cpp:122-134)     ->  pass A + pass B
//
// Pass-A items: column pair cp x group of <= kGroup code pairs sharing one
// window spectrum.  Pass-B items: pair x tile of kTileB t2 columns of the
// inter-pass intermediate M, which lives in a ring of `ring` wave buffers
// (events order A(w) after B(w-ring)).  Jobs are ordered code-pair-major so
// a group's code spectra stay L2-resident (evict_last) while the window
// spectra stream through (evict_first), and pass B drops each M tile from L2
// after reading it (discard: no DRAM write-back of dead data).
//
// Inside a CTA, the next item's operands are bulk-copied (cp.async.bulk ->
// UBLKCP, completing on an mbarrier) into the second shared-memory slot while
// the 4 warps run the current item from the first: in pass A every warp's
// lane 0 issues its own share (its X column; warp 0 the window column, warp 1
// the twiddle rows) and the TMA store of its own staged column, in pass B
// thread 0 issues the tile.  In pass A each warp (one column role) transposes
// and stages over the X column only it reads, so an item has a single CTA
// barrier (at its end).  The search shape (N = 27 x 32768) runs as a
// prime-factor split: no step-2 twiddles in pass A (pfa_split below).
#pragma once
#include "kernels.cuh"
#include "tma.cuh"

namespace tdg {

constexpr int kTileB = 4;   // t2 columns per pass-B tile (M is stored tile-major)
constexpr int kGroup = 2;   // code pairs per pass-A item (sharing one window spectrum column)

// Build-time layout variant (A/B-timed with tools/ab_libs.sh):
//   TDG_CORR_MINB  CTAs per SM the register budget is sized for (3: 170
//                  registers; 4 spills and measured 13-17 % slower)
// Two operand slots per CTA: the next item's bulk copies overlap this item.
// Measured and removed: one slot with more CTAs per SM, pass-B
// twiddles from a full shared-memory table (-20 %: every twiddle an LDS),
// pass-B transposes in a separate region, pass A without the end-of-item
// barrier (per-warp slot release through "empty" mbarriers).
#ifndef TDG_CORR_MINB
#define TDG_CORR_MINB 3
#endif
constexpr int kSlots = 2;

__host__ __device__ constexpr int cmax(int a, int b) { return a > b ? a : b; }
__host__ __device__ constexpr int qstride_even_pad(int q) { return (q % 2) ? q : q + 1; }
// pass-B transposed row stride (float2 units): == 4 or 12 (mod 16) so that a
// half-warp of 4 a-values x 4 t2-columns hits 16 distinct 8-byte bank pairs
__host__ __device__ constexpr int passb_row(int q) {
    return ((q * kTileB) % 16 == 4 || (q * kTileB) % 16 == 12) ? q * kTileB
           : ((q * kTileB) % 16 == 0) ? q * kTileB + 4
                                      : q * kTileB + 12 - ((q * kTileB) % 16) + ((q * kTileB) % 16 > 12 ? 16 : 0);
}
__host__ __device__ constexpr int even_up(int x) { return (x + 1) & ~1; }
__host__ __device__ constexpr int up16(int x) { return (x + 15) & ~15; }   // float2 units: 128 bytes

// Inter-pass twiddle table row stride (float2): row k1 holds
// [w_N^{+k1 c}, c < QA][w_N^{+k1 QA e}, e < PA], padded to a 16-byte multiple.
__host__ __device__ constexpr int inter_tw_stride(int PA, int QA) { return even_up(PA + QA); }

__host__ __device__ constexpr int cgcd(int a, int b) { return b ? cgcd(b, a % b) : a; }

// Prime-factor (Good-Thomas) split of the correlation length: when the pass-A
// step-1 lane dimension PA is coprime to N / PA = N1 * QA (the search shape:
// N = 27 x 32768), the inverse DFT is DFT_PA (x) DFT_{N/PA} with no twiddles
// between them, and DFT_{N/PA} is the four-step N1 x QA.  Spectra are then
// stored per column k1 = k mod N1 in PFA order (element a + PA*b for
// a = k mod PA, b = (k mod N1*QA) div N1), pass A runs DFT_QA over b and
// DFT_PA over a without step-2 twiddles and with an inter-pass twiddle
// w_{N/PA}^{k1 c} that is constant per lane, and output t_a, t_b map to the
// lag t = ((N/PA) t_a + PA t_b) mod N.
__host__ __device__ constexpr bool pfa_split(int PA, int QA, int N1) { return PA > 1 && cgcd(PA, N1 * QA) == 1; }

template <int PA, int QA, int PB, int QB>
struct Fused {
    static constexpr int LA = PA * QA, LB = PB * QB;
    static constexpr bool PFA = pfa_split(PA, QA, LB);
    static constexpr int QSA = qstride_even_pad(QA);
    static constexpr int TWS = inter_tw_stride(PA, QA);
    // pass-A slot: [D column][X columns: 2 per pair][2 twiddle rows], every
    // column in a region of XS >= the padded transpose, so each warp's
    // transpose and M staging live over the X column it alone reads (no CTA
    // barrier inside an item); regions 128-byte aligned for the TMA store
    static constexpr int STG = up16(cmax(PA * QSA, LA));
    static constexpr int XS = STG;
    static constexpr int A_OPS = (1 + 2 * kGroup) * XS;
    static constexpr int A_SLOT = up16(A_OPS + 2 * TWS);
    static constexpr int ROWB = passb_row(QB);
    static constexpr int B_SLOT = up16(cmax(LB * kTileB, PB * ROWB));     // tile, transposed in place
    static constexpr int SLOT = cmax(A_SLOT, B_SLOT);
    static constexpr int NT = 128;
    // slots, then (pass B) the transpose region and the twiddle table
    static constexpr int ANC = 5 * cmax(QA, QB);   // step-2 twiddle anchors (+ pass B PFA: w_32^{-q})
    static constexpr size_t SMEM = 128 + kSlots * size_t(SLOT) * 8 + size_t(ANC) * 8;
    static_assert(cmax(PA, QA) <= 32 && cmax(PB, QB) <= 32, "one warp per column role");
    static_assert(LA % kTileB == 0, "M tiles cover the t2 columns exactly (TMA store box)");
    static_assert(kTileB * cmax(PB, QB) <= NT, "pass-B tasks fit the CTA");
};

struct CorrSched {                     // one wave
    CUtensorMap mstore;                // M ring as [pair][tile][k1][8 floats]: pass A's TMA stores
    const CorrGroup<kGroup>* groups;   // [ngw]
    const CorrPairOut* outs;           // [wave_pairs]
    const float2* twA;                 // w_{N2}^{+ac}, index a*QA + c
    const float2* twB;                 // w_{N1}^{+ac}, index a*QB + c
    const float2* twI;                 // inter-pass rows, stride inter_tw_stride
    int ngw, wave_pairs, n_tiles, nA, nB, N1, N2;
    int write_xc;                      // 1: full xc rows (batch_xcorr), 0: argmax keys
    int discard;                       // 1: drop consumed M tiles from L2 (no write-back)
    unsigned long long* trace;         // diagnostics (option "cta_trace"): per CTA {smid|type, t0, t1}
    unsigned int* trace_n;
    unsigned int trace_cap;
    uint32_t W;                        // window length (lag limits are per pair: CorrPairOut)
    float inv_n;
};


__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// threadIdx.x through a volatile read: the item bodies recompute their
// lane-dependent addresses per item instead of letting NVVM hoist them out of
// the persistent loop, where pass A's and pass B's invariants together would
// stay live across both bodies and spill.
__device__ __forceinline__ int tid_x() {
    int t;
    asm volatile("mov.u32 %0, %%tid.x;" : "=r"(t));
    return t;
}

// An item's coordinates: pass A (u, v) = (column pair cp, group), item
// u * ngw + v; pass B (u, v) = (pair, M tile), item u * n_tiles + v.  A CTA
// walks a contiguous item range, so they advance without divisions.
// warp-wide max of a float (CREDUX.MAX.F32, sm_100a)
__device__ __forceinline__ float warp_max_f32(float v) {
    float d;
    asm volatile("redux.sync.max.f32 %0, %1, 0xffffffff;" : "=f"(d) : "f"(v));
    return d;
}

// max(m, |x|, |y|) as one FMNMX3 (three-input max with |.| operand modifiers)
__device__ __forceinline__ float fmax3_abs(float m, float x, float y) {
    float d;
    asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(m), "f"(fabsf(x)), "f"(fabsf(y)));
    return d;
}

struct Ticket {
    int u, v;
};
__device__ __forceinline__ Ticket ticket_at(int item, int den) { return Ticket{item / den, item % den}; }
__device__ __forceinline__ void ticket_next(Ticket& t, int den) {
    if (++t.v == den) {
        t.v = 0;
        ++t.u;
    }
}

// the wave's descriptors, copied to shared memory once per CTA
struct Desc {
    const CorrGroup<kGroup>* groups;
    const CorrPairOut* outs;
};

template <int TYPE>
__device__ __forceinline__ bool ticket_noop(const Desc& D, const Ticket& k) {
    if (TYPE == 0) return D.groups[k.v].npairs == 0;
    return D.outs[k.u].M == nullptr;
}

// thread 0 (pass B): the bulk copy of a (non-noop) item's M tile into slot sl
template <int PA, int QA, int PB, int QB>
__device__ __forceinline__ void issue_tile(const Desc& D, const Ticket& k, float2* sl, uint64_t* bar) {
    using F = Fused<PA, QA, PB, QB>;
    constexpr int LB = F::LB;
    // earlier generic use of this slot before the async writes (no global
    // proxy fence: M is written by pass A's TMA stores and read by pass B's
    // bulk copies, both async proxy, across a kernel boundary)
    fence_proxy_async_smem();
    const CorrPairOut& po = D.outs[k.u];
    mbar_arrive_expect_tx(bar, LB * kTileB * 8);
    bulk_g2s_hint(sl, po.M + size_t(k.v) * LB * kTileB, LB * kTileB * 8, bar, policy_evict_first());
}

// lane 0 of warp `role`: this role's share of a pass-A item's
// bulk copies, with one arrive.expect_tx on the slot's barrier (initialised
// for NT/32 arrivals)
template <int PA, int QA, int PB, int QB>
__device__ __forceinline__ void issue_passA_role(const CorrSched& S, const Desc& D, const Ticket& k, float2* sl,
                                                 uint64_t* bar, int role) {
    using F = Fused<PA, QA, PB, QB>;
    constexpr int LA = F::LA, TWS = F::TWS;
    fence_proxy_async_smem();
    const int cp = k.u;
    const CorrGroup<kGroup>& gd = D.groups[k.v];
    const bool self = (cp == 0) || (2 * cp == F::LB);
    const int g = role >> 1, col = role & 1;
    const bool act = g < gd.npairs && (col == 0 || !self);
    uint32_t bytes = act ? uint32_t(LA) * 8u : 0u;
    if (role == 0) bytes += uint32_t(LA) * 8u;
    if (role == 1) bytes += 2u * TWS * 8u;
    mbar_arrive_expect_tx(bar, bytes);
    if (role == 0) bulk_g2s_hint(sl, gd.D + size_t(cp) * LA, LA * 8, bar, policy_evict_first());
    if (act) {
        const int xcol = (col == 0 && !self) ? F::LB - cp : cp;   // region 1 + role: X column of (g, col)
        bulk_g2s_hint(sl + (1 + role) * F::XS, gd.Ca[g] + size_t(xcol) * LA, LA * 8, bar, policy_evict_last());
    }
    if (role == 1) {
        const int k1b = cp == 0 ? 0 : F::LB - cp;
        bulk_g2s(sl + F::A_OPS, S.twI + size_t(cp) * TWS, TWS * 8, bar);
        bulk_g2s(sl + F::A_OPS + TWS, S.twI + size_t(k1b) * TWS, TWS * 8, bar);
    }
}

// ---------------------------------------------------------------------------
// Pass A item: column pair (cp, N1-cp) x up to kGroup code pairs of one
// window.  Code pairs are stored as the full spectrum X = FFT(dc_a + i dc_b)
// in column layout, so with the window's Hermitian half-column D:
//   Z[k]   = D[k] (conj Ca[k] + i conj Cb[k]) = D[k] X[N-k]
//   Z[N-k] = conj(D[k]) (Ca[k] + i Cb[k])     = conj(D[k]) X[k]
// i.e. one complex multiply per point; IFFT(Z) = xc_a + i xc_b.  Output: M,
// tile-major M[(t2/kTileB)*N1*kTileB + k1*kTileB + t2%kTileB], times the
// inter-pass twiddle w_N^{+k1 t2}.
template <int PA, int QA, int PB, int QB, class Mid>
__device__ __forceinline__ void item_passA(const CorrSched& S, const Desc& D, const Ticket& k, float2* sl, Mid&& mid,
                                           const float2* anc) {
    using F = Fused<PA, QA, PB, QB>;
    constexpr int P = PA, Q = QA, L = F::LA, QS = F::QSA, TWS = F::TWS;
    constexpr int N1 = F::LB;   // pass-B length == number of columns
    const int cp = k.u;
    const int tid = tid_x();
    const CorrGroup<kGroup>& gd = D.groups[k.v];
    const int npairs = gd.npairs;
    const bool self = (cp == 0) || (2 * cp == N1);
    const int role = tid >> 5;   // warp-uniform (g, col)
    const int g = role >> 1, col = role & 1;
    const int lane = tid & 31;
    const bool act = g < npairs && (col == 0 || !self);
    // ---- step 1: lane a: product + Q-point IDFT over rows r = a + P*b
    float2 v[Q];
    const bool act1 = act && lane < P;
    // row of this lane.  PFA: half-warp 0 takes rows 1..16, half-warp 1 rows
    // 0, 17..P-1, so that both a row's elements a + P*b and its mirror's
    // (P - a) % P + P*b' hit 16 distinct bank pairs per half-warp (lane a = row
    // a put rows 0 and 16 of the mirror into one bank pair: 1.5x wavefronts)
    const int arow = (F::PFA && P > 16) ? (lane < 16 ? lane + 1 : (lane == 16 ? 0 : lane)) : lane;
    if (act1 && F::PFA) {
        // PFA order: element (a, b) at a + P*b; the mirror N - k of (a, b) is
        // ((P - a) % P, Q - 1 - b) across a column pair, ((P - a) % P, (Q - b) % Q)
        // in column 0
        const int a = arow;
        const int am = a ? P - a : 0;
        const float2* D = sl;
        const float2* Xm = sl + (1 + 2 * g) * F::XS;   // X column N1-cp (or cp if self)
        if (col == 0) {
            if (cp == 0) {
#pragma unroll
                for (int b = 0; b < Q; ++b) v[b] = cmul(D[a + P * b], Xm[am + P * ((Q - b) % Q)]);
            } else {
#pragma unroll
                for (int b = 0; b < Q; ++b) v[b] = cmul(D[a + P * b], Xm[am + P * (Q - 1 - b)]);
            }
        } else {
            const float2* Xc = sl + (2 + 2 * g) * F::XS;  // X column cp
#pragma unroll
            for (int b = 0; b < Q; ++b) {
                const int m = am + P * (Q - 1 - b);   // source element of output (a, b)
                v[b] = cmulc(Xc[m], D[m]);
            }
        }
        dft<Q, +1>(v);
    } else if (act1) {
        const int a = lane;
        const float2* D = sl;
        const float2* Xm = sl + (1 + 2 * g) * F::XS;   // X column N1-cp (or cp if self)
        if (col == 0) {
            if (cp == 0) {
#pragma unroll
                for (int b = 0; b < Q; ++b) {
                    const int r = a + P * b;
                    v[b] = cmul(D[r], Xm[r == 0 ? 0 : L - r]);
                }
            } else {
#pragma unroll
                for (int b = 0; b < Q; ++b) {
                    const int r = a + P * b;
                    v[b] = cmul(D[r], Xm[L - 1 - r]);
                }
            }
        } else {
            const float2* Xc = sl + (2 + 2 * g) * F::XS;  // X column cp
#pragma unroll
            for (int b = 0; b < Q; ++b) {
                const int r = (L - 1) - (a + P * b);   // source row of output row a + P*b
                v[b] = cmulc(Xc[r], D[r]);
            }
        }
        dft<Q, +1>(v);
    }
    // the transpose goes over this warp's own X column (read only by it)
    __syncwarp();
    if (act1) {
        float2* tr = sl + (1 + role) * F::XS + arow * QS;
#pragma unroll
        for (int c = 0; c < Q; ++c) tr[c] = v[c];
    }
    __syncwarp();
    mid();   // thread 0: the next item's bulk copies (into the other slot; A/B: after the
             // transpose write beats before it by ~0.4 %, after step 2 loses ~1 %)
    // ---- step 2: lane c: twiddle, P-point IDFT over a, inter-pass twiddle, store M
    if (act && lane < Q) {
        const int c = lane;
        const float2* tr = sl + (1 + role) * F::XS + c;
        float2 w[P];
#pragma unroll
        for (int a = 0; a < P; ++a) w[a] = tr[a * QS];
        if (!F::PFA) apply_step2_twiddles_anc<P, Q>(w, anc, c);
        dft<P, +1>(w);
        const float2* twr = sl + F::A_OPS + col * TWS;
        const float2 tc = twr[c];
        if (F::PFA) {
            // inter-pass twiddle w_{N/P}^{k1 c}: one value per lane (twr row k1
            // holds w_N^{k1 P c}, c < Q)
            float2* stg = sl + (1 + role) * F::XS;
            __syncwarp(0xffffffffu >> (32 - Q));
#pragma unroll
            for (int e = 0; e < P; ++e) stg[c + Q * e] = cmul(w[e], tc);
            fence_proxy_async_smem();
            return;
        }
        // stage the column in t2 order in the warp's own region, then one TMA
        // tensor store scatters it into M's tile-major layout (N2/4 chunks of
        // 32 bytes) without occupying the LSU pipe
        float2* stg = sl + (1 + role) * F::XS;
        __syncwarp(0xffffffffu >> (32 - Q));   // the region's transposed inputs are consumed
        // w_N^{k1 (c + Q e)} = tc * w_N^{k1 Q e}: exact row values every 8th e,
        // one chained product by w_N^{k1 Q} in between
        const float2 s1 = twr[Q + 1];
        float2 tt = tc;
#pragma unroll
        for (int e = 0; e < P; ++e) {
            if (e % 8 == 0) {
                if (e) tt = cmul(tc, twr[Q + e]);
            } else {
                tt = cmul(tt, s1);
            }
            stg[c + Q * e] = cmul(w[e], tt);
        }
    }
    // staged column visible to the async proxy; thread 0 issues the stores
    // after the end-of-item barrier (store_passA)
    if (act) fence_proxy_async_smem();
}

// lane 0 of a warp, after the end-of-item barrier: the TMA tensor store of this warp's own
// staged column, if its role is active in the item
template <int PA, int QA, int PB, int QB>
__device__ __forceinline__ void store_passA_role(const CorrSched& S, const Desc& D, const Ticket& k, float2* sl,
                                                 int role) {
    using F = Fused<PA, QA, PB, QB>;
    constexpr int N1 = F::LB;
    const int cp = k.u;
    const CorrGroup<kGroup>& gd = D.groups[k.v];
    const bool self = (cp == 0) || (2 * cp == N1);
    const int g = role >> 1, col = role & 1;
    if (g < gd.npairs && (col == 0 || !self)) {
        tma_store_4d(&S.mstore, sl + (1 + role) * F::XS, 0, col ? N1 - cp : cp, 0, gd.Mi[g]);
        bulk_commit();
    }
}

// ---------------------------------------------------------------------------
// Pass B item: (pair, tile of kTileB t2 columns); tile = N1 x kTileB
// contiguous float2 of M.  y[t2 + N2*t1] = xc_a + i*xc_b (times N).
// Epilogue: first-index argmax of |Re|, |Im| over lags t < W (find_peak,
// proj/src/detector.cpp:122-134) merged with atomicMax on packed keys, or
// the full xc rows (batch_xcorr diagnostics).
template <int PA, int QA, int PB, int QB, class Pre>
__device__ __forceinline__ void item_passB(const CorrSched& S, const Desc& D, const Ticket& k, float2* sl,
                                           const float2* anc, Pre&& pre) {
    using F = Fused<PA, QA, PB, QB>;
    constexpr int P = PB, Q = QB, ROW = F::ROWB, TB = kTileB;
    const CorrPairOut& po = D.outs[k.u];
    const int tb = k.v;
    const int tid = tid_x();
    constexpr int N2 = F::LA;   // pass-A length == number of t2 columns
    // the pair's best magnitudes so far (high words of the packed keys)
    float cur_a = 0.f, cur_b = 0.f;
    if (!S.write_xc) {
        cur_a = __uint_as_float(uint32_t(ld_relaxed_u64(po.key_a) >> 32));
        if (po.key_b) cur_b = __uint_as_float(uint32_t(ld_relaxed_u64(po.key_b) >> 32));
    }
    const uint32_t W = po.lag_lim;   // valid local lags [0, W)
    // step 1: task (a, t2l), t2l fastest
    const int t2l1 = tid % TB, a1 = tid / TB;
    const bool act1 = a1 < P;
    float2 v[Q];
    float2* tr = sl;   // transposed in place
    if (act1) {
#pragma unroll
        for (int b = 0; b < Q; ++b) v[b] = sl[(a1 + P * b) * TB + t2l1];
        dft<Q, +1>(v);
    }
    __syncthreads();   // in place: every input read before any transposed write
    // every warp is past the previous item, so the other slot is free: the
    // next tile's bulk copy (no end-of-item barrier needed)
    pre();
    if (act1) {
#pragma unroll
        for (int c = 0; c < Q; ++c) tr[a1 * ROW + c * TB + t2l1] = v[c];
    }
    __syncthreads();
    // step 2: task (c, t2l)
    const int t2l = tid % TB, c = tid / TB;
    const int t2 = tb * TB + t2l;
    float best_a = -1.f, best_b = -1.f;
    int e_lim = 0;
    uint32_t pfa_base = 0, pfa_m = 0;   // PFA: lag of slot 0 and valid slots e < pfa_m
    float2 w[P];
    if (c < Q) {
#pragma unroll
        for (int a = 0; a < P; ++a) w[a] = tr[a * ROW + c * TB + t2l];
        if (F::PFA) {
            // column t2 = t_b1 + QA t_a; output e of the last DFT is the lag
            // t = ((N/PA) t_a + PA (t_b1 + QA (c + Q e))) mod N = (base + e SE) mod N,
            // base = q SE + r.  The step-2 twiddles are taken as
            // w_L^{a (c - Q q)} instead of w_L^{a c} -- the extra w_P^{-a q} rotates
            // the DFT's outputs so that slot e holds lag r + e SE: no wrap, the
            // valid lags t < W are the prefix e < m = ceil((W - r) / SE), and the
            // lags rise with e.  (anchors at a = 8j pick up a quarter turn
            // i^{-jq}; the base twiddle one multiply by w_P^{-q})
            static_assert(!F::PFA || (P == 32 && Q == 32), "rotated PFA epilogue assumes a 32 x 32 last pass");
            constexpr uint32_t NN = uint32_t(F::LA) * uint32_t(F::LB), SE = NN / P;
            constexpr uint32_t NBB = NN / PA;
            const uint32_t tb1 = uint32_t(t2) % uint32_t(QA), ta = uint32_t(t2) / uint32_t(QA);
            // (N/PA) t_a < N and PA (t_b1 + QA c) < PA QA QB <= N: one conditional subtract
            uint32_t base = NBB * ta + uint32_t(PA) * (tb1 + uint32_t(QA) * uint32_t(c));
            base = base >= NN ? base - NN : base;
            const uint32_t q = base / SE;
            pfa_base = base - q * SE;   // r: the lag of slot 0
            pfa_m = W > pfa_base ? min(uint32_t(P), (W - pfa_base + SE - 1) / SE) : 0u;
            // w_1024^{a (c - 32 q)}: base twiddle and the 8j anchors
            const float2 rq = anc[4 * Q + (q & 31u)];   // w_32^{-q}
            const float2 t1 = cmul(anc[c], rq);
            float2 t = t1;
#pragma unroll
            for (int a = 1; a < P; ++a) {
                if (a % 8 == 0) {
                    const float2 x = anc[(a / 8) * Q + c];
                    const uint32_t k = (uint32_t(4 - (a / 8)) * q) & 3u;   // i^{-(a/8) q} = i^k
                    t = k == 0 ? x : k == 1 ? make_float2(-x.y, x.x) : k == 2 ? make_float2(-x.x, -x.y)
                                                                           : make_float2(x.y, -x.x);
                } else if (a > 1) {
                    t = cmul(t, t1);
                }
                w[a] = cmul(w[a], t);
            }
            dft<P, +1>(w);
            if (S.write_xc) {
#pragma unroll
                for (int e = 0; e < P; ++e) {
                    if (uint32_t(e) < pfa_m) {
                        const uint32_t tt = pfa_base + uint32_t(e) * SE;
                        if (po.xc_a) po.xc_a[tt] = w[e].x * S.inv_n;
                        if (po.xc_b) po.xc_b[tt] = w[e].y * S.inv_n;
                    }
                }
            } else if (W >= uint32_t(P - 4) * SE) {
                // every lane's m >= P - 4 (r < SE): the first P - 4 slots unmasked,
                // three-input maxima
                // four independent FMNMX3 chains per component (short dependency
                // chains: the epilogue is latency-, not issue-bound)
                float ma[4] = {best_a, best_a, best_a, best_a}, mb[4] = {best_b, best_b, best_b, best_b};
#pragma unroll
                for (int e = 0; e < P - 4; e += 2) {
                    ma[(e / 2) & 3] = fmax3_abs(ma[(e / 2) & 3], w[e].x, w[e + 1].x);
                    mb[(e / 2) & 3] = fmax3_abs(mb[(e / 2) & 3], w[e].y, w[e + 1].y);
                }
                best_a = fmaxf(fmaxf(ma[0], ma[1]), fmaxf(ma[2], ma[3]));
                best_b = fmaxf(fmaxf(mb[0], mb[1]), fmaxf(mb[2], mb[3]));
#pragma unroll
                for (int e = P - 4; e < P; ++e) {
                    if (uint32_t(e) < pfa_m) {
                        best_a = fmaxf(best_a, fabsf(w[e].x));
                        best_b = fmaxf(best_b, fabsf(w[e].y));
                    }
                }
            } else {
#pragma unroll
                for (int e = 0; e < P; ++e) {
                    if (uint32_t(e) < pfa_m) {
                        best_a = fmaxf(best_a, fabsf(w[e].x));
                        best_b = fmaxf(best_b, fabsf(w[e].y));
                    }
                }
            }
        } else {
            apply_step2_twiddles_anc<P, Q>(w, anc, c);
            dft<P, +1>(w);
        }
        // valid lags t = t2 + N2*(c + Q*e) < W form a prefix e < e_lim
        if (!F::PFA && t2 < N2 && uint32_t(t2) < W) {
            const int t1max = int((W - 1u - uint32_t(t2)) / uint32_t(N2));
            e_lim = t1max >= c ? (t1max - c) / Q + 1 : 0;
            e_lim = e_lim < P ? e_lim : P;
        }
        if (F::PFA) {
        } else if (S.write_xc) {
#pragma unroll
            for (int e = 0; e < P; ++e) {
                if (e < e_lim) {
                    const uint32_t t = uint32_t(t2) + uint32_t(N2) * uint32_t(c + Q * e);
                    if (po.xc_a) po.xc_a[t] = w[e].x * S.inv_n;
                    if (po.xc_b) po.xc_b[t] = w[e].y * S.inv_n;
                }
            }
        } else if (e_lim == P) {
#pragma unroll
            for (int e = 0; e < P; ++e) {
                best_a = fmaxf(best_a, fabsf(w[e].x));
                best_b = fmaxf(best_b, fabsf(w[e].y));
            }
        } else {
#pragma unroll
            for (int e = 0; e < P; ++e) {
                if (e < e_lim) {
                    best_a = fmaxf(best_a, fabsf(w[e].x));
                    best_b = fmaxf(best_b, fabsf(w[e].y));
                }
            }
        }
    }
    if (!S.write_xc) {
        // first-index argmax.  Warp maxima of |Re|, |Im| first (one CREDUX
        // each); only warps whose maximum can still win against the pair's
        // best so far (read at item start -- an older value only makes more
        // warps search) locate the smallest lag holding it (per lane, then one
        // CREDUX.MIN) and merge packed keys (magnitude, then smallest lag:
        // exact first-index ties) with atomicMax.
        best_a = warp_max_f32(best_a);
        best_b = warp_max_f32(best_b);
        // each lane read the pair's best on its own, so another CTA's atomicMax
        // can land between lanes: vote, so the branch below (warp-wide
        // reductions) is taken by every lane or none
        const bool need_a = __any_sync(0xffffffffu, best_a >= 0.f && best_a >= cur_a);
        const bool need_b = __any_sync(0xffffffffu, best_b >= 0.f && po.key_b != nullptr && best_b >= cur_b);
        if (need_a || need_b) {   // warp-uniform
            uint32_t ta = 0xffffffffu, tb = 0xffffffffu;
            if (c < Q) {
                if (F::PFA) {
                    // lags rise with the slot
                    constexpr uint32_t NN = uint32_t(F::LA) * uint32_t(F::LB), SE = NN / P;
#pragma unroll
                    for (int e = P - 1; e >= 0; --e) {
                        if (uint32_t(e) < pfa_m) {
                            const uint32_t t = pfa_base + uint32_t(e) * SE;
                            if (fabsf(w[e].x) == best_a) ta = t;
                            if (fabsf(w[e].y) == best_b) tb = t;
                        }
                    }
                } else {
#pragma unroll
                    for (int e = P - 1; e >= 0; --e) {
                        if (e < e_lim) {
                            const uint32_t t = uint32_t(t2) + uint32_t(N2) * uint32_t(c + Q * e);
                            if (fabsf(w[e].x) == best_a) ta = t;
                            if (fabsf(w[e].y) == best_b) tb = t;
                        }
                    }
                }
            }
            ta = __reduce_min_sync(0xffffffffu, ta);
            tb = __reduce_min_sync(0xffffffffu, tb);
            if ((tid & 31) == 0) {
                if (need_a && ta != 0xffffffffu) atomicMax(po.key_a, peak_key(best_a, po.lag0 + ta));
                if (need_b && tb != 0xffffffffu) atomicMax(po.key_b, peak_key(best_b, po.lag0 + tb));
            }
        }
    }
}

// ---------------------------------------------------------------------------
// One pass over one wave: persistent CTAs, each walking a contiguous range of
// items with a 2-slot TMA ring (item i+1's bulk copies in flight while item i
// computes).
template <int PA, int QA, int PB, int QB, int TYPE>
__global__ void __launch_bounds__(128, TDG_CORR_MINB) k_corr_pass(const __grid_constant__ CorrSched S) {
    using F = Fused<PA, QA, PB, QB>;
    extern __shared__ __align__(128) unsigned char smraw[];
    unsigned long long trace_t0 = 0;
    if (S.trace && threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(trace_t0));
    uint64_t* bar = reinterpret_cast<uint64_t*>(smraw);   // [0..1]: slot full
    float2* slots = reinterpret_cast<float2*>(smraw + 128);
    float2* anc = slots + size_t(kSlots) * F::SLOT;      // step-2 twiddle anchors of this pass
    // the wave's descriptors live in shared memory (read by every item)
    unsigned char* dsm = smraw + F::SMEM;
    const int n_items = TYPE == 0 ? S.nA : S.nB;
    const int den = TYPE == 0 ? S.ngw : S.n_tiles;
    const int i0 = int(int64_t(blockIdx.x) * n_items / gridDim.x);
    const int i1 = int(int64_t(blockIdx.x + 1) * n_items / gridDim.x);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // pass A: every warp's lane 0 issues its share of an item's bulk copies
    // (issue_passA_role), so the slot barriers count NT/32 arrivals; pass B:
    // thread 0 issues the tile
    if (threadIdx.x == 0) {
        mbar_init(&bar[0], TYPE == 0 ? F::NT / 32 : 1);
        mbar_init(&bar[1], TYPE == 0 ? F::NT / 32 : 1);
        mbar_fence_init();
    }
    if (TYPE == 0) __syncthreads();   // barriers initialised before any warp arrives on them
    // the first item's bulk copies from the global descriptors, while the CTA
    // stages the descriptors in shared memory
    if (i0 < i1) {
        const Desc Dg{S.groups, S.outs};
        const Ticket k0 = ticket_at(i0, den);
        if (!ticket_noop<TYPE>(Dg, k0)) {
            if (TYPE == 0 && lane == 0) issue_passA_role<PA, QA, PB, QB>(S, Dg, k0, slots, &bar[0], warp);
            if (TYPE == 1 && threadIdx.x == 0) issue_tile<PA, QA, PB, QB>(Dg, k0, slots, &bar[0]);
        }
    }
    Desc D;
    {
        const int nb_g = TYPE == 0 ? int(S.ngw * sizeof(CorrGroup<kGroup>)) : 0;
        const int nb_o = TYPE == 1 ? int(S.wave_pairs * sizeof(CorrPairOut)) : 0;
        const unsigned char* src_g = reinterpret_cast<const unsigned char*>(S.groups);
        const unsigned char* src_o = reinterpret_cast<const unsigned char*>(S.outs);
        for (int i = threadIdx.x; i < (nb_g + nb_o) / 4; i += F::NT)
            reinterpret_cast<uint32_t*>(dsm)[i] =
                4 * i < nb_g ? reinterpret_cast<const uint32_t*>(src_g)[i]
                             : reinterpret_cast<const uint32_t*>(src_o)[i - nb_g / 4];
        D.groups = reinterpret_cast<const CorrGroup<kGroup>*>(dsm);
        D.outs = reinterpret_cast<const CorrPairOut*>(dsm + nb_g);
    }
    if (TYPE == 1) {
        fill_twiddle_anchors<PB, QB>(anc, S.twB, threadIdx.x, F::NT);
        if (F::PFA && threadIdx.x < 32) {
            // w_32^{-q}, q < 32: the rotation of the PFA epilogue's outputs
            double sn, cs;
            sincospi(double(threadIdx.x) / 16.0, &sn, &cs);
            anc[4 * QB + threadIdx.x] = make_float2(float(cs), float(-sn));
        }
    } else if (!F::PFA) {
        fill_twiddle_anchors<PA, QA>(anc, S.twA, threadIdx.x, F::NT);
    }
    __syncthreads();
    uint32_t phases = 0u;   // bit s: parity of slot s's mbarrier
    Ticket k = ticket_at(i0, den);
    for (int item = i0, s = 0; item < i1; ++item, s ^= 1) {
        Ticket kn = k;
        ticket_next(kn, den);
        // the next item's bulk copies into slot s^1: pass B at the top of the
        // item; pass A halfway through (after step 1), each warp once its TMA
        // store of the item that last used slot s^1 has read its staging area
        auto prefetch = [&]() {
            if (item + 1 >= i1) return;
            if (TYPE == 0 && lane == 0) {
                bulk_wait_read_all();
                if (!ticket_noop<TYPE>(D, kn))
                    issue_passA_role<PA, QA, PB, QB>(S, D, kn, slots + size_t(s ^ 1) * F::SLOT, &bar[s ^ 1], warp);
            }
            if (TYPE == 1 && threadIdx.x == 0 && !ticket_noop<TYPE>(D, kn))
                issue_tile<PA, QA, PB, QB>(D, kn, slots + size_t(s ^ 1) * F::SLOT, &bar[s ^ 1]);
        };
        if (ticket_noop<TYPE>(D, k)) {
            if (TYPE == 1) __syncthreads();   // every warp past the previous item
            prefetch();
            k = kn;
            continue;
        }
        float2* sl = slots + size_t(s) * F::SLOT;
        mbar_wait(&bar[s], (phases >> s) & 1u);
        phases ^= 1u << s;
        if (TYPE == 0) {
            item_passA<PA, QA, PB, QB>(S, D, k, sl, prefetch, anc);
        } else {
            // the M tile is in shared memory and its L2 lines are dead: drop
            // them without a DRAM write-back.  Only lines wholly inside the
            // tile: a tile that does not start on a 128-byte line (N1 * 32
            // bytes not a multiple of 128, e.g. N1 = 450) shares its edge lines
            // with the neighbouring tiles, whose items may not have read them yet.
            const CorrPairOut& po = D.outs[k.u];
            const uintptr_t t0 = reinterpret_cast<uintptr_t>(po.M + size_t(k.v) * F::LB * kTileB);
            const uintptr_t lo = (t0 + 127) & ~uintptr_t(127);
            const uintptr_t hi = (t0 + uintptr_t(F::LB) * kTileB * 8) & ~uintptr_t(127);
            if (S.discard)
                for (uintptr_t a = lo + uintptr_t(threadIdx.x) * 128; a < hi; a += uintptr_t(F::NT) * 128)
                    discard_l2(reinterpret_cast<const void*>(a));
            item_passB<PA, QA, PB, QB>(S, D, k, sl, anc, prefetch);
        }
        // pass A: slot s consumed, its staged columns complete (pass B needs no
        // end-of-item barrier: its next bulk copy waits for the in-item one)
        if (TYPE == 0) __syncthreads();
        if (TYPE == 0 && lane == 0) store_passA_role<PA, QA, PB, QB>(S, D, k, sl, warp);
        k = kn;
    }
    // the CTA's shared memory must outlive the reads of its last TMA stores;
    // the stores' global writes are complete by the end of the grid (what
    // orders pass B after them), so only the reads are waited for here
    if (TYPE == 0 && lane == 0) bulk_wait_read_all();
    if (S.trace) {
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned long long t1, smid;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
            unsigned int sm32;
            asm volatile("mov.u32 %0, %%smid;" : "=r"(sm32));
            smid = sm32;
            const unsigned int i = atomicAdd(S.trace_n, 1u);
            if (i < S.trace_cap) {
                S.trace[3 * size_t(i)] = (smid << 8) | unsigned(TYPE);
                S.trace[3 * size_t(i) + 1] = trace_t0;
                S.trace[3 * size_t(i) + 2] = t1;
            }
        }
    }
}

}  // namespace tdg
