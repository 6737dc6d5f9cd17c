// Correlation passes, persistent + TMA-pipelined (v2).  See kernels.cuh for
// the transform layout.  Each CTA walks a contiguous range of work items;
// while it runs the two FFT steps of item i from one shared-memory slot, a
// single elected thread has already issued the 1-D bulk copies
// (cp.async.bulk, SASS UBLKCP) of item i+1 into the other slot, completing on
// an mbarrier.  The transposes between the register codelets are written in
// place over the slot's consumed operands.
#pragma once
#include "kernels.cuh"
#include "tma.cuh"

namespace tdg {

constexpr int kTileB = 4;  // t2 columns per pass-B tile (M is stored tile-major)

__host__ __device__ constexpr int cmax(int a, int b) { return a > b ? a : b; }
__host__ __device__ constexpr int qstride_even_pad(int q) { return (q % 2) ? q : q + 1; }
// pass-B transposed row stride (float2 units): == 4 or 12 (mod 16) so that a
// half-warp of 4 a-values x 4 t2-columns hits 16 distinct 8-byte bank pairs
__host__ __device__ constexpr int passb_row(int q) {
    return ((q * kTileB) % 16 == 4 || (q * kTileB) % 16 == 12) ? q * kTileB
           : ((q * kTileB) % 16 == 0) ? q * kTileB + 4
                                      : q * kTileB + 12 - ((q * kTileB) % 16) + ((q * kTileB) % 16 > 12 ? 16 : 0);
}

template <int P, int Q, int GP>
struct PassA2 {
    static constexpr int L = P * Q;
    static constexpr int QS = qstride_even_pad(Q);
    static constexpr int SLOT = cmax((1 + 2 * GP) * L, GP * 2 * P * QS);  // float2
    // one warp-group of WP lanes per (pair, column) role in step 1 and step 2
    static constexpr int WP = ((cmax(P, Q) + 31) / 32) * 32;
    static constexpr int NT = GP * 2 * WP;
    static constexpr int TW_OFF = 128;                                      // bytes
    static constexpr int SLOT_OFF = TW_OFF + ((2 * (P + Q) * 8 + 127) / 128) * 128;
    static constexpr size_t SMEM = size_t(SLOT_OFF) + 2 * size_t(SLOT) * 8;
    static constexpr int MINB = cmax(P, Q) > 32 ? 2 : 3;
};

template <int P, int Q>
struct PassB2 {
    static constexpr int L = P * Q;
    static constexpr int ROW = passb_row(Q);
    static constexpr int SLOT = cmax(L * kTileB, P * ROW);
    static constexpr int NT = ((kTileB * cmax(P, Q) + 31) / 32) * 32;
    static constexpr size_t SMEM = 128 + 2 * size_t(SLOT) * 8;
    static constexpr int MINB = cmax(P, Q) > 32 ? 2 : 3;
};

// ---------------------------------------------------------------------------
// Pass A: item = (column pair cp, group of GP code pairs of one window).
// Code pairs are stored as the full spectrum X = FFT(dc_a + i dc_b) in
// column layout, so with the window's Hermitian half-column D:
//   Z[k]   = D[k] (conj Ca[k] + i conj Cb[k]) = D[k] X[N-k]
//   Z[N-k] = conj(D[k]) (Ca[k] + i Cb[k])     = conj(D[k]) X[k]
// i.e. one complex multiply per point; IFFT(Z) = xc_a + i xc_b.
template <int P, int Q, int GP>
__global__ void __launch_bounds__(PassA2<P, Q, GP>::NT, PassA2<P, Q, GP>::MINB)
    k_corr_passA2(const CorrGroup<GP>* __restrict__ groups, int n_groups, int N1, int n_items,
                  const float2* __restrict__ twL) {
    using C = PassA2<P, Q, GP>;
    constexpr int L = P * Q, QS = C::QS, WP = C::WP;
    extern __shared__ __align__(128) unsigned char smraw[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(smraw);
    float2* tw = reinterpret_cast<float2*>(smraw + C::TW_OFF);
    float2* slots = reinterpret_cast<float2*>(smraw + C::SLOT_OFF);
    const int64_t N = int64_t(N1) * L;
    const int i0 = int(int64_t(blockIdx.x) * n_items / gridDim.x);
    const int i1 = int(int64_t(blockIdx.x + 1) * n_items / gridDim.x);
    if (threadIdx.x == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        mbar_fence_init();
    }
    __syncthreads();
    // slot layout: [0,L) D column cp ; for pair g: [(1+2g)L) X column N1-cp,
    // [(2+2g)L) X column cp (self columns: only the first is used)
    auto issue = [&](int item, int s) {
        const int cp = item / n_groups;
        const CorrGroup<GP>& gd = groups[item % n_groups];
        const bool self = (cp == 0) || (2 * cp == N1);
        float2* sl = slots + size_t(s) * C::SLOT;
        const uint32_t bytes = uint32_t(L) * 8u * uint32_t(1 + gd.npairs * (self ? 1 : 2));
        mbar_arrive_expect_tx(&bar[s], bytes);
        bulk_g2s(sl, gd.D + size_t(cp) * L, L * 8, &bar[s]);
        for (int g = 0; g < gd.npairs; ++g) {
            const float2* X = gd.Ca[g];
            bulk_g2s(sl + (1 + 2 * g) * L, X + size_t(self ? cp : N1 - cp) * L, L * 8, &bar[s]);
            if (!self) bulk_g2s(sl + (2 + 2 * g) * L, X + size_t(cp) * L, L * 8, &bar[s]);
        }
    };
    if (threadIdx.x == 0 && i0 < i1) issue(i0, 0);
    uint32_t phase0 = 0, phase1 = 0;
    int last_cp = -1;
    const int role = threadIdx.x / WP;          // warp-uniform (g, col)
    const int g = role >> 1, col = role & 1;
    const int lane = threadIdx.x % WP;
    for (int item = i0, it = 0; item < i1; ++item, ++it) {
        const int s = it & 1;
        if (threadIdx.x == 0 && item + 1 < i1) {
            fence_proxy_async_smem();
            issue(item + 1, s ^ 1);
        }
        const int cp = item / n_groups;
        const CorrGroup<GP>& gd = groups[item % n_groups];
        const bool self = (cp == 0) || (2 * cp == N1);
        const bool act = g < gd.npairs && (col == 0 || !self);
        if (cp != last_cp) {
            for (int i = threadIdx.x; i < 2 * (P + Q); i += blockDim.x) {
                const int cc = i / (P + Q), r = i % (P + Q);
                const int64_t k1 = cc ? N1 - cp : cp;
                const int64_t e = r < Q ? k1 * r : k1 * Q * (r - Q);
                tw[i] = twiddle_exact(e, N, +1);
            }
            last_cp = cp;
        }
        if (s == 0) {
            mbar_wait(&bar[0], phase0);
            phase0 ^= 1;
        } else {
            mbar_wait(&bar[1], phase1);
            phase1 ^= 1;
        }
        float2* sl = slots + size_t(s) * C::SLOT;
        // ---- step 1: lane a: product + Q-point IDFT over rows r = a + P*b
        float2 v[Q];
        const bool act1 = act && lane < P;
        if (act1) {
            const int a = lane;
            const float2* D = sl;
            const float2* Xm = sl + (1 + 2 * g) * L;   // X column N1-cp (or cp if self)
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
                const float2* Xc = sl + (2 + 2 * g) * L;  // X column cp
#pragma unroll
                for (int b = 0; b < Q; ++b) {
                    const int r = (L - 1) - (a + P * b);   // source row of output row a + P*b
                    v[b] = cmulc(Xc[r], D[r]);
                }
            }
            dft<Q, +1>(v);
        }
        __syncthreads();  // operands consumed
        if (act1) {
            float2* tr = sl + role * P * QS + lane * QS;
#pragma unroll
            for (int c = 0; c < Q; ++c) tr[c] = v[c];
        }
        __syncthreads();
        // ---- step 2: lane c: twiddle, P-point IDFT over a, inter-pass twiddle, store M
        if (act && lane < Q) {
            const int c = lane;
            const float2* tr = sl + role * P * QS + c;
            float2 w[P];
#pragma unroll
            for (int a = 0; a < P; ++a) {
                const float2 x = tr[a * QS];
                w[a] = a == 0 ? x : cmul(x, __ldg(&twL[a * Q + c]));
            }
            dft<P, +1>(w);
            const int k1 = col ? N1 - cp : cp;
            const float2 tc = tw[col * (P + Q) + c];
            const float2* tb = tw + col * (P + Q) + Q;
            float2* M = gd.M[g] + size_t(k1) * kTileB + (c % kTileB) + size_t(c / kTileB) * N1 * kTileB;
#pragma unroll
            for (int e = 0; e < P; ++e) {
                // t2 = c + Q e ; tile-major: ((t2 / TB) * N1 + k1) * TB + t2 % TB
                static_assert(Q % kTileB == 0 || true, "");
                const int t2 = c + Q * e;
                const float2 tt = cmul(tc, tb[e]);
                if (Q % kTileB == 0)
                    M[size_t(Q / kTileB) * e * N1 * kTileB] = cmul(w[e], tt);
                else
                    gd.M[g][(size_t(t2 / kTileB) * N1 + k1) * kTileB + (t2 % kTileB)] = cmul(w[e], tt);
            }
        }
        __syncthreads();  // slot s free for the prefetch of item + 2
    }
}

// ---------------------------------------------------------------------------
// Pass B: item = (pair, tile of kTileB t2 columns).  Tile = N1 x kTileB
// contiguous floats2 of M.  Epilogue: running first-index argmax of |Re|, |Im|.
template <int P, int Q, bool WRITE_XC>
__global__ void __launch_bounds__(PassB2<P, Q>::NT, PassB2<P, Q>::MINB)
    k_corr_passB2(const CorrPairOut* __restrict__ pairs, int n_tiles, int N2, uint32_t W, float inv_n,
                  int n_items, const float2* __restrict__ twL) {
    using C = PassB2<P, Q>;
    constexpr int L = C::L, ROW = C::ROW, TB = kTileB;
    extern __shared__ __align__(128) unsigned char smraw[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(smraw);
    float2* slots = reinterpret_cast<float2*>(smraw + 128);
    const int i0 = int(int64_t(blockIdx.x) * n_items / gridDim.x);
    const int i1 = int(int64_t(blockIdx.x + 1) * n_items / gridDim.x);
    if (threadIdx.x == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        mbar_fence_init();
    }
    __syncthreads();
    auto issue = [&](int item, int s) {
        const CorrPairOut& po = pairs[item / n_tiles];
        const int tb = item % n_tiles;
        mbar_arrive_expect_tx(&bar[s], L * TB * 8);
        bulk_g2s(slots + size_t(s) * C::SLOT, po.M + size_t(tb) * L * TB, L * TB * 8, &bar[s]);
    };
    if (threadIdx.x == 0 && i0 < i1) issue(i0, 0);
    uint32_t phase0 = 0, phase1 = 0;
    // running best per thread (first index wins ties: strict '>' over increasing t)
    float best_a = -1.f, best_b = -1.f;
    uint32_t idx_a = 0, idx_b = 0;
    int cur_pair = i0 < i1 ? i0 / n_tiles : -1;
    const int lane = threadIdx.x & 31;
    auto flush = [&](int pair) {
        unsigned long long ka = best_a >= 0.f ? peak_key(best_a, idx_a) : 0ull;
        unsigned long long kb = best_b >= 0.f ? peak_key(best_b, idx_b) : 0ull;
        for (int o = 16; o > 0; o >>= 1) {
            const unsigned long long xa = __shfl_xor_sync(0xffffffffu, ka, o);
            const unsigned long long xb = __shfl_xor_sync(0xffffffffu, kb, o);
            ka = xa > ka ? xa : ka;
            kb = xb > kb ? xb : kb;
        }
        if (lane == 0) {
            const CorrPairOut& po = pairs[pair];
            if (ka) atomicMax(po.key_a, ka);
            if (kb && po.key_b) atomicMax(po.key_b, kb);
        }
        best_a = best_b = -1.f;
    };
    for (int item = i0, it = 0; item < i1; ++item, ++it) {
        const int s = it & 1;
        if (threadIdx.x == 0 && item + 1 < i1) {
            fence_proxy_async_smem();
            issue(item + 1, s ^ 1);
        }
        const int pair = item / n_tiles, tb = item % n_tiles;
        if (!WRITE_XC && pair != cur_pair) {
            flush(cur_pair);
            cur_pair = pair;
        }
        if (s == 0) {
            mbar_wait(&bar[0], phase0);
            phase0 ^= 1;
        } else {
            mbar_wait(&bar[1], phase1);
            phase1 ^= 1;
        }
        float2* sl = slots + size_t(s) * C::SLOT;
        // step 1: task (a, t2l), t2l fastest
        const int t2l1 = threadIdx.x % TB, a1 = threadIdx.x / TB;
        const bool act1 = a1 < P;
        float2 v[Q];
        if (act1) {
#pragma unroll
            for (int b = 0; b < Q; ++b) v[b] = sl[(a1 + P * b) * TB + t2l1];
            dft<Q, +1>(v);
        }
        __syncthreads();
        if (act1) {
#pragma unroll
            for (int c = 0; c < Q; ++c) sl[a1 * ROW + c * TB + t2l1] = v[c];
        }
        __syncthreads();
        // step 2: task (c, t2l)
        const int t2l = threadIdx.x % TB, c = threadIdx.x / TB;
        const int t2 = tb * TB + t2l;
        if (c < Q) {
            float2 w[P];
#pragma unroll
            for (int a = 0; a < P; ++a) {
                const float2 x = sl[a * ROW + c * TB + t2l];
                w[a] = a == 0 ? x : cmul(x, __ldg(&twL[a * Q + c]));
            }
            dft<P, +1>(w);
            // valid lags t = t2 + N2*(c + Q*e) < W form a prefix e < e_lim
            int e_lim = 0;
            if (t2 < N2 && uint32_t(t2) < W) {
                const int t1max = int((W - 1u - uint32_t(t2)) / uint32_t(N2));
                e_lim = t1max >= c ? (t1max - c) / Q + 1 : 0;
                e_lim = e_lim < P ? e_lim : P;
            }
            if (WRITE_XC) {
                const CorrPairOut& po = pairs[pair];
#pragma unroll
                for (int e = 0; e < P; ++e) {
                    if (e < e_lim) {
                        const uint32_t t = uint32_t(t2) + uint32_t(N2) * uint32_t(c + Q * e);
                        if (po.xc_a) po.xc_a[t] = w[e].x * inv_n;
                        if (po.xc_b) po.xc_b[t] = w[e].y * inv_n;
                    }
                }
            } else if (e_lim > 0) {
                // t increases with e: strict '>' keeps the first index
                float la = -1.f, lb = -1.f;
                int ea = 0, eb = 0;
#pragma unroll
                for (int e = 0; e < P; ++e) {
                    if (e < e_lim) {
                        const float ma = fabsf(w[e].x), mb = fabsf(w[e].y);
                        if (ma > la) {
                            la = ma;
                            ea = e;
                        }
                        if (mb > lb) {
                            lb = mb;
                            eb = e;
                        }
                    }
                }
                const uint32_t ia = uint32_t(t2) + uint32_t(N2) * uint32_t(c + Q * ea);
                const uint32_t ib = uint32_t(t2) + uint32_t(N2) * uint32_t(c + Q * eb);
                // merge across tiles, where t is not monotone: explicit tie rule
                if (la > best_a || (la == best_a && ia < idx_a)) {
                    best_a = la;
                    idx_a = ia;
                }
                if (lb > best_b || (lb == best_b && ib < idx_b)) {
                    best_b = lb;
                    idx_b = ib;
                }
            }
        }
        __syncthreads();  // slot s free
    }
    if (!WRITE_XC && cur_pair >= 0) flush(cur_pair);
}

}  // namespace tdg
