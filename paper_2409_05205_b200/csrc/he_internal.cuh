// he_internal.cuh -- context layout, 64-bit modular arithmetic and the
// shared-memory NTT passes used by every kernel of the library.
//
// Residues are < q < 2^50.  Two arithmetic families: exact FP64 modular
// products on the DFMA pipe (the default transforms, dp_* below) and
// integer Shoup products with Harvey's lazy butterflies (HE_NTT=int).  The
// folded MAC runs on the int8 tensor cores (exact byte-plane split,
// he_kernels.cu K3), not here.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/he_rotfree.h"

typedef unsigned long long u64;
typedef unsigned int u32;

// Per-limb constants (device copy in he_ctx::d_limb).
#ifndef HE_QDIV
#define HE_QDIV 1
#endif
#ifndef HE_TW_LAZY
#define HE_TW_LAZY 1      // radix-16 CT passes: the last stage's twiddles loaded at that stage
#endif

struct he_limb {
    u64 q;          // prime q_j
    u64 q2;         // 2 q_j
    u64 ninv, ninv_p;       // N^{-1} mod q and its Shoup companion
    u64 delta, delta_p;     // Delta_t mod q (R2) and Shoup companion
    u64 r25, r25_p;         // 2^25 mod q
    u64 r50, r50_p;         // 2^50 mod q
    u64 r64, r64_p;         // 2^64 mod q
    u64 r40, r40_p;         // 2^40 mod q   (byte-split MAC recombination)
    u64 r80, r80_p;         // 2^80 mod q
    u64 one_p;              // Shoup companion of 1  (floor(2^64 / q))
    double qd, qinvd;       // q and fl(1/q) for the FP64 transforms
    double tinvd;           // t^{-1} mod q, centred, as a double (enc_dp)
    double c32d, c64d, c96d;  // 2^32, 2^64, 2^96 mod q, centred (FP64 MAC recombination)
    u64 mq;                 // -q^{-1} mod 2^64 (Montgomery reduction of the int8 MAC sums)
    double mrd[3];          // 2^-64, 2^-32, 2^32 mod q, centred (FP64 form of that reduction)
    uint32_t pw8[3];        // 2^8, 2^16, 2^24 (runtime multipliers: one IMAD.WIDE per term)
    double td, t_invd, rtd; // t, fl(1/t), r_t as doubles (context-wide; K4 mask encoding)
};

struct he_ctx {
    int device;
    int mac_mode;           // 0: auto (int8 tensor-core MAC when s >= 4), 1: IMAD MAC
    uint32_t logN, N, L;
    u64 t, r_t;             // plaintext modulus, r_t = Q mod t (R2)
    u64 t_inv;              // floor(2^64 / t) (for floor(x / t))
    u64* q_host;
    u64* psi_host;
    he_limb* limb_host;
    he_limb* d_limb;        // [L]
    ulonglong2* d_tw_fwd;   // [L][N]  {psi^{brv(k)}, Shoup}
    ulonglong2* d_tw_inv;   // [L][N]  {psi^{-brv(k)}, Shoup}
    double* d_twd_fwd;      // [L][N]  psi^{brv(k)} as double (FP64 transforms)
    double* d_twd_inv;      // [L][N]  psi^{-brv(k)} as double
    int ntt_mode;           // 0: FP64 butterflies (default), 1: integer (HE_NTT=int)
    int ntt_cluster;        // HE_NTT_COLS: 0 auto, 1 cluster kernels only, 2 columns forced
    int ntt_r8;             // HE_NTT_R8 set: radix-8 full forward transforms (A/B only)
    int mac_tc;             // HE_MAC_TC: 0 never, 1 always, 2 (default) when B >= 128
    u64* d_enc;             // [L][t] enc_j(m) table (t <= 2^20), else nullptr
};

// enc_j(m) via the context table when present (one L2-resident load).
__device__ __forceinline__ u64 enc_lookup(const u64* __restrict__ tab, int l, u64 t, u64 m,
                                          const struct he_limb& L, u64 r_t, u64 t_inv);

// ------------------------------------------------------------ arithmetic
// x * w mod q in [0, 2q) for any x < 2^64 (Shoup): wp = floor(w 2^64 / q).
__device__ __forceinline__ u64 shoup_mul(u64 x, u64 w, u64 wp, u64 q) {
    u64 qh = __umul64hi(x, wp);
    return x * w - qh * q;
}

__device__ __forceinline__ u64 csub(u64 x, u64 m) { return x >= m ? x - m : x; }

// Cooley-Tukey butterfly, inputs/outputs in [0, 4q).
__device__ __forceinline__ void ct_bfly(u64& X, u64& Y, ulonglong2 w, u64 q,
                                        u64 q2) {
    u64 x = csub(X, q2);
    u64 t = shoup_mul(Y, w.x, w.y, q);
    X = x + t;
    Y = x - t + q2;
}

// Shoup product with an approximate quotient: Q' = x1 w1 + hi(x1 w0) +
// hi(x0 w1) (32-bit halves; the x0 w0 term and the carries are dropped), so
// Q - 2 <= Q' <= Q and the result x w - Q' q lies in [0, 4q) for any x < 2^64.
__device__ __forceinline__ u64 shoup_mul4(u64 x, u64 w, u64 wp, u64 q) {
    const u32 x0 = (u32)x, x1 = (u32)(x >> 32);
    const u32 p0 = (u32)wp, p1 = (u32)(wp >> 32);
    u64 qh = (u64)__umulhi(x0, p1) + __umulhi(x1, p0);
    asm("mad.wide.u32 %0, %1, %2, %0;" : "+l"(qh) : "r"(x1), "r"(p1));
    return x * w - qh * q;
}

// Lazy Cooley-Tukey butterfly without the conditional subtraction: with
// inputs < a q the outputs are < (a + 4) q (T = Shoup4(Y) < 4q for any
// 64-bit Y).  15 stages keep every value below 61 q < 2^56.
__device__ __forceinline__ void ct_bfly_lazy(u64& X, u64& Y, ulonglong2 w, u64 q, u64 q2) {
    const u64 x = X;
    const u64 t = shoup_mul4(Y, w.x, w.y, q);
    X = x + t;
    Y = x - t + 2 * q2;
}

// Lazy Gentleman-Sande butterfly for stage `lt` (t = 2^lt) of a transform
// whose inputs are < 2q: inputs of stage lt are < 2^(lt+1) q (X' = X + Y
// doubles the bound, Y' = Shoup4(.) < 4q <= 2^(lt+2) q), so
// X - Y + 2^(lt+1) q >= 0.  Valid while 2^(stages+1) q < 2^64 (<= 12
// stages for q < 2^50).
__device__ __forceinline__ void gs_bfly_lazy(u64& X, u64& Y, ulonglong2 w, u64 q, u64 off) {
    const u64 x = X, y = Y;
    X = x + y;
    Y = shoup_mul4(x - y + off, w.x, w.y, q);      // < 4q <= offset of the next stage
}

// Full reduction of a lazy value v < 2^64 to [0, q).
__device__ __forceinline__ u64 reduce_full(u64 v, u64 q, u64 one_p) {
    const u64 r = v - __umul64hi(v, one_p) * q;     // [0, 2q)
    return csub(r, q);
}

// Gentleman-Sande butterfly, inputs/outputs in [0, 2q).
__device__ __forceinline__ void gs_bfly(u64& X, u64& Y, ulonglong2 w, u64 q,
                                        u64 q2) {
    u64 x = X, y = Y;
    X = csub(x + y, q2);
    Y = shoup_mul(x - y + q2, w.x, w.y, q);
}

// floor(x / t) for x < 2^63 with t_inv = floor(2^64 / t).
__device__ __forceinline__ u64 div_by_t(u64 x, u64 t, u64 t_inv) {
    u64 d = __umul64hi(x, t_inv);
    return (x - d * t >= t) ? d + 1 : d;
}

// enc_j(m) = (Delta_t mod q) m + floor((r_t m + floor(t/2)) / t)  mod q,
// m in [0, t)  (R2; equals round(Q m / t) mod q_j).
__device__ __forceinline__ u64 enc_plain(u64 m, const he_limb& L, u64 t,
                                         u64 r_t, u64 t_inv) {
    u64 a = shoup_mul(m, L.delta, L.delta_p, L.q);                  // [0, 2q)
    u64 f = div_by_t(r_t * m + (t >> 1), t, t_inv);                 // < t
    f = shoup_mul(f, 1, L.one_p, L.q);              // [0, 2q) even if t > q
    return csub(csub(a + f, 2 * L.q), L.q);
}

// acc += a * b (32 x 32 -> 64, 64-bit accumulate): one IMAD.WIDE.U32.
// (Plain C `acc += (u64)a * b` makes nvcc add the zero high words too.)
// x / d for 0 <= x < 2^20, 1 <= d < 2^20 without an integer division (the
// kernels' block-index decompositions): floor((x + 1/2) r) with r the
// hardware reciprocal of d (relative error < 2^-22) is exact there --
// (x + 1/2)/d is at least 1/(2d) away from an integer and the float error is
// below (x + 1/2)/d 1.25 2^-22 < 1/(2d); larger x take the integer division.
__device__ __forceinline__ int qdiv(int x, int d) {
#if HE_QDIV
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"((float)d));
    return x < (1 << 20) ? (int)(((float)x + 0.5f) * r) : x / d;
#else
    return x / d;
#endif
}

__device__ __forceinline__ void madw(u64& acc, u32 a, u32 b) {
    asm("mad.wide.u32 %0, %1, %2, %0;" : "+l"(acc) : "r"(a), "r"(b));
}

__device__ __forceinline__ u64 enc_lookup(const u64* __restrict__ tab, int l, u64 t, u64 m,
                                          const he_limb& L, u64 r_t, u64 t_inv) {
    return tab ? __ldg(&tab[(size_t)l * t + m]) : enc_plain(m, L, t, r_t, t_inv);
}

__device__ __forceinline__ u64 addmod(u64 a, u64 b, u64 q) {
    return csub(a + b, q);
}

// Canonical value -> "split25" word (hi25 << 32 | lo25) used by the MAC.
__device__ __forceinline__ u64 to_split25(u64 v) {
    return ((v >> 25) << 32) | (v & ((1ull << 25) - 1));
}

// 4 x 4 byte transpose: p_i = byte_i(a) | byte_i(b) << 8 | byte_i(c) << 16 |
// byte_i(d) << 24  (8 PRMT).
__device__ __forceinline__ void byte_transpose4(u32 a, u32 b, u32 c, u32 d, u32& p0,
                                                u32& p1, u32& p2, u32& p3) {
    const u32 t0 = __byte_perm(a, b, 0x5140), t1 = __byte_perm(a, b, 0x7362);
    const u32 t2 = __byte_perm(c, d, 0x5140), t3 = __byte_perm(c, d, 0x7362);
    p0 = __byte_perm(t0, t2, 0x5410);
    p1 = __byte_perm(t0, t2, 0x7632);
    p2 = __byte_perm(t1, t3, 0x5410);
    p3 = __byte_perm(t1, t3, 0x7632);
}

// Padding: one 8-byte word per 16 (kills bank conflicts for every stride).
__device__ __forceinline__ int PAD(int i) { return i + (i >> 4); }
__host__ __device__ constexpr int padded_words(int n) { return n + (n >> 4); }

// ------------------------------------------------------- FP64 residues
// Residues as integer-valued doubles (|x| < 2^52), so the modular products
// run on the FP64 pipe.  The twiddle tables are centred, |w| <= (q-1)/2, so
// |y| w / q < 2^51 holds for every |y| <= 4q + 8 (q <= 2^50 - 3):
//   p = fl(y w), e = fma(y, w, -p) = y w - p        (exact two-product)
//   k = rint(p qinv) via the 1.5 2^52 magic constant: |p/q - k| <= 0.5 +
//       |p/q| 2^-53 <= 0.75
//   r = fma(-k, q, p) = p - k q                     (exact, |.| <= 0.75 q)
//   T = r + e = y w - k q,  |T| <= 0.75 q + ulp(p)/2 <= q   (|p| <= 2 q^2)
static constexpr double DP_MAGIC = 6755399441055744.0;     // 1.5 * 2^52

__device__ __forceinline__ double dp_mulmod(double y, double w, double q, double qinv) {
    const double p = y * w;
    const double e = fma(y, w, -p);
    const double k = fma(p, qinv, DP_MAGIC) - DP_MAGIC;
    return fma(-k, q, p) + e;
}

// |result| <= q/2 + 2 for integer-valued |y| < 2^53 (k = rint(y qinv) is
// within 0.5 + 2^-49 of y / q).
__device__ __forceinline__ double dp_reduce(double y, double q, double qinv) {
    const double k = fma(y, qinv, DP_MAGIC) - DP_MAGIC;
    return fma(-k, q, y);
}

// n consecutive twiddles tw[b .. b+n) (n a power of two; b a multiple of
// min(n, 2)): 16-byte loads, so a warp whose lanes read different runs
// touches half as many L1 sectors per twiddle.
__device__ __forceinline__ void load_tw_run(double* dst, const double* __restrict__ tw, int b,
                                            int nt) {
    if (nt == 1) {
        dst[0] = __ldg(&tw[b]);
    } else {
#pragma unroll
        for (int z = 0; z < nt; z += 2) {
            const double2 v = __ldg(reinterpret_cast<const double2*>(tw + b + z));
            dst[z] = v.x;
            dst[z + 1] = v.y;
        }
    }
}

// enc_j(m) = round(Q m / t) mod q_j without a table (R2): Q m = t X + c
// with X = round(Q m / t) and c the centred remainder of Q m mod t, and
// Q = 0 mod q_j, so X = -c t^{-1} mod q_j; c = r_t m mods t (r_t = Q mod t).
// For t <= 2^20 (odd) and m < t: x = r_t m < 2^40 is exact, rint(x / t)
// is exact (|x/t| 2^-52 << 1/(2t), and t odd has no ties), |c| <= t/2.
// Result: an integer-valued double with |.| <= q.
__device__ __forceinline__ double enc_dp(double md, double rtd, double td, double t_inv,
                                         double tinvq, double q, double qinv) {
    const double x = rtd * md;                              // exact
    const double k = fma(x, t_inv, DP_MAGIC) - DP_MAGIC;    // rint(x / t)
    const double c = fma(-k, td, x);                        // centred remainder
    return dp_mulmod(-c, tinvq, q, qinv);
}

// exact u64 (< 2^52) <-> double
__device__ __forceinline__ double u2d(u64 x) {
    return __longlong_as_double((long long)(x | 0x4330000000000000ull)) - 4503599627370496.0;
}
// integer-valued |y| < 2^52 -> a residue congruent to y in [q/2 - 1, 3q/2 + 1]
// (not canonical: for the int8 MAC operand, whose byte split takes any
// value below 2^56)
__device__ __forceinline__ u64 d2lazy(double y, double q, double qinv) {
    // r + (q + 2^52) in one rounding: exact, the sum is an integer in [2^52, 2^53)
    const double r = dp_reduce(y, q, qinv);
    return (u64)(__double_as_longlong(r + (q + 4503599627370496.0)) & 0xFFFFFFFFFFFFFull);
}
// integer-valued |y| < 2^53 -> canonical residue in [0, q)
__device__ __forceinline__ u64 d2canon(double y, double q, double qinv) {
    const double r = dp_reduce(y, q, qinv); // |r| <= q/2 + 2 < q
    // one conditional add suffices; it rides on the 2^52 shift (one DADD)
    const double off = r < 0.0 ? q + 4503599627370496.0 : 4503599627370496.0;
    return (u64)(__double_as_longlong(r + off) & 0xFFFFFFFFFFFFFull);
}

// FP64 Cooley-Tukey butterfly: X' = X + T, Y' = X - T, T = Y w mod q.
// Caller guarantees |Y| < 4 q and |w| <= (q-1)/2 (so |Y| w / q < 2^51).
__device__ __forceinline__ void ct_bfly_dp(double& X, double& Y, double w, double q,
                                           double qinv) {
    const double t = dp_mulmod(Y, w, q, qinv);
    const double x = X;
    X = x + t;
    Y = x - t;
}

// One radix-2^K pass of FP64 CT stages (as ct_pass).  Inputs are reduced
// to |x| <= q/2 + 1 at the start of the pass; stage r inputs are then below
// (0.5 + r) q + 1 (|T| <= q), so for K <= 4 every stage multiplies directly
// (multiplicand < 3.5 q + 1 < 4 q).  Outputs < 4.5 q + 1.
template <int K, bool NORED = false, bool LZ = false, bool LIN = false>
__device__ __forceinline__ void ct_pass_dp(double* sm, int logN, int NS, int st0, int seg,
                                           int split, const double* __restrict__ tw,
                                           double q, double qinv) {
    const int lt0 = logN - st0 - 1;
    const int ltk = lt0 - (K - 1);
    const int tk = 1 << ltk;
    const int ngroups = NS >> K;
    for (int g = threadIdx.x; g < ngroups; g += blockDim.x) {
        const int blk = g >> ltk, off = g & (tk - 1);
        const int base = (blk << (lt0 + 1)) + off;
        double tws[(1 << K) - 1];
        // LZ (the 64-register conv-path kernels): the last HE_TW_LAZY stages'
        // twiddles are loaded when each stage starts -- fewer live registers
        // in radix-16 passes, spills 72 -> 40 bytes, s = 8 forward NTT 62.4 ->
        // 60.2 us; the 80-register full transforms keep loading them up front
        constexpr int RUP = (LZ && HE_TW_LAZY && K == 4) ? K - HE_TW_LAZY : K;
#pragma unroll
        for (int r = 0, o = 0; r < RUP; o += (1 << r), ++r) {
            const int twb = (1 << (st0 + r)) + (seg << (st0 + r - split)) + (blk << r);
            load_tw_run(tws + o, tw, twb, 1 << r);
        }
        // LIN: PAD(base + (c << ltk)) = PAD(base) + PAD(c << ltk) -- base's
        // residue mod 16 plus that of c << ltk never reaches 16 (off < 2^ltk,
        // and base is a multiple of 2^(ltk+K) plus off) -- so with a
        // compile-time ltk (the unrolled plain-20 instances) every element is
        // an immediate offset from one base: no per-element address
        // arithmetic and no addresses kept live (spilled) for the stores.
        // (With a run-time ltk the 16 offsets would stay live in registers
        // across the group loop: the full transforms keep the direct form.)
        const int pb = PAD(base);
        auto ai = [&](int c) { return LIN ? pb + PAD(c << ltk) : PAD(base + (c << ltk)); };
        double x[1 << K];
#pragma unroll
        for (int c = 0; c < (1 << K); ++c)
            x[c] = NORED ? sm[ai(c)] : dp_reduce(sm[ai(c)], q, qinv);
#pragma unroll
        for (int r = 0, o = 0; r < K; o += (1 << r), ++r) {
            if (r >= RUP) {
                const int twb = (1 << (st0 + r)) + (seg << (st0 + r - split)) + (blk << r);
                load_tw_run(tws + o, tw, twb, 1 << r);
            }
            const int half = 1 << (K - 1 - r);
#pragma unroll
            for (int c = 0; c < (1 << K); ++c) {
                if (c & half) continue;
                if (r >= 4) x[c + half] = dp_reduce(x[c + half], q, qinv);
                ct_bfly_dp(x[c], x[c + half], tws[o + (c >> (K - r))], q, qinv);
            }
        }
#pragma unroll
        for (int c = 0; c < (1 << K); ++c) sm[ai(c)] = x[c];
    }
}

template <int RMAX, bool LZ = false, bool UNR = false, bool LIN = UNR>
__device__ __forceinline__ void ct_all_dp(double* sm, int logN, int NS, int seg, int split,
                                          const double* tw, double q, double qinv,
                                          int end) {
    // stages [split, end): end < logN stops early (incomplete transform)
    int st = split;
    if (st >= end) return;
    const int rem = (end - split) % RMAX;
    // the first pass reads the register stages' outputs: canonical inputs
    // plus at most `split` added |T| <= q, so its stage-r multiplicands stay
    // below (1 + split + r) q <= 4q when split + K <= 4 -- no reduction
    if (rem) {
        const bool nr = split + rem <= 4;
        if (rem == 1) ct_pass_dp<1, true, false, LIN>(sm, logN, NS, st, seg, split, tw, q, qinv);
        else if (rem == 2 && nr)
            ct_pass_dp<2, true, false, LIN>(sm, logN, NS, st, seg, split, tw, q, qinv);
        else if (rem == 2) ct_pass_dp<2, false, false, LIN>(sm, logN, NS, st, seg, split, tw, q, qinv);
        else if (nr) ct_pass_dp<3, true, false, LIN>(sm, logN, NS, st, seg, split, tw, q, qinv);
        else ct_pass_dp<3, false, false, LIN>(sm, logN, NS, st, seg, split, tw, q, qinv);
        st += rem;
        __syncthreads();
    } else if (split + RMAX <= 4) {
        ct_pass_dp<RMAX, true, LZ, LIN>(sm, logN, NS, st, seg, split, tw, q, qinv);
        st += RMAX;
        __syncthreads();
    }
    if (UNR) {
        // compile-time geometry (the plain-20 instances): unrolled, so every
        // pass's stage offset and strides are immediates
#pragma unroll
        for (int p = 0; p < 8; ++p) {
            if (st + p * RMAX >= end) break;
            ct_pass_dp<RMAX, false, LZ, LIN>(sm, logN, NS, st + p * RMAX, seg, split, tw, q,
                                             qinv);
            __syncthreads();
        }
        return;
    }
    for (; st < end; st += RMAX) {
        ct_pass_dp<RMAX, false, LZ, LIN>(sm, logN, NS, st, seg, split, tw, q, qinv);
        __syncthreads();
    }
}

// Column form of the incomplete forward transform: the first T = log2(M)
// stages of the N-point CT transform never mix residues mod s = N/M, so
// they are s independent M-point transforms of the columns {c + s k}, with
// the N-point twiddles of stage st and block k >> (T - st).  One radix-2^K
// pass over narr column arrays (arr_stride words apart) in shared memory;
// value bounds as ct_pass_dp.
template <int K, bool RAW = false, bool LIN = false>
__device__ __forceinline__ void ct_pass_cols_dp(double* sm, int arr_stride, int narr, int T,
                                                int st0, const double* __restrict__ tw,
                                                double q, double qinv) {
    const int lt0 = T - st0 - 1;
    const int ltk = lt0 - (K - 1);
    const int tk = 1 << ltk;
    const int gper = 1 << (T - K);
    const int total = narr * gper;
    for (int G = threadIdx.x; G < total; G += blockDim.x) {
        const int a = G >> (T - K), g = G & (gper - 1);
        double* s = sm + a * arr_stride;
        const int blk = g >> ltk, off = g & (tk - 1);
        const int base = (blk << (lt0 + 1)) + off;
        double tws[(1 << K) - 1];
#pragma unroll
        for (int r = 0, o = 0; r < K; o += (1 << r), ++r) {
            const int twb = (1 << (st0 + r)) + (blk << r);
            load_tw_run(tws + o, tw, twb, 1 << r);
        }
        // (LIN: the immediate-offset form of ct_pass_dp's addresses)
        const int pb = PAD(base);
        auto ai = [&](int c) { return LIN ? pb + PAD(c << ltk) : PAD(base + (c << ltk)); };
        double x[1 << K];
#pragma unroll
        for (int c = 0; c < (1 << K); ++c)
            // RAW: canonical u64 residues as copied by cp.async (< q: stage r
            // multiplicands stay below (1 + r) q <= 4q without a reduction)
            x[c] = RAW ? u2d(reinterpret_cast<const u64*>(s)[ai(c)]) : dp_reduce(s[ai(c)], q, qinv);
#pragma unroll
        for (int r = 0, o = 0; r < K; o += (1 << r), ++r) {
            const int half = 1 << (K - 1 - r);
#pragma unroll
            for (int c = 0; c < (1 << K); ++c) {
                if (c & half) continue;
                if (r >= 4) x[c + half] = dp_reduce(x[c + half], q, qinv);
                ct_bfly_dp(x[c], x[c + half], tws[o + (c >> (K - r))], q, qinv);
            }
        }
#pragma unroll
        for (int c = 0; c < (1 << K); ++c) s[ai(c)] = x[c];
    }
}

template <int RMAX, bool RAW = false, bool LIN = false>
__device__ __forceinline__ void ct_all_cols_dp(double* sm, int arr_stride, int narr, int T,
                                               const double* tw, double q, double qinv) {
    int st = 0;
    const int rem = T % RMAX;
    if (rem) {
        if (rem == 1) ct_pass_cols_dp<1, RAW, LIN>(sm, arr_stride, narr, T, st, tw, q, qinv);
        else if (rem == 2) ct_pass_cols_dp<2, RAW, LIN>(sm, arr_stride, narr, T, st, tw, q, qinv);
        else ct_pass_cols_dp<3, RAW, LIN>(sm, arr_stride, narr, T, st, tw, q, qinv);
        st += rem;
        __syncthreads();
    } else if (RAW && T > 0) {
        ct_pass_cols_dp<RMAX, true, LIN>(sm, arr_stride, narr, T, st, tw, q, qinv);
        st += RMAX;
        __syncthreads();
    }
    if (LIN) {                  // compile-time T: unrolled, strides are immediates
#pragma unroll
        for (int p = 0; p < 8; ++p) {
            if (st >= T) break;
            ct_pass_cols_dp<RMAX, false, LIN>(sm, arr_stride, narr, T, st, tw, q, qinv);
            __syncthreads();
            st += RMAX;
        }
        return;
    }
    for (; st < T; st += RMAX) {
        ct_pass_cols_dp<RMAX>(sm, arr_stride, narr, T, st, tw, q, qinv);
        __syncthreads();
    }
}


// One radix-2^K pass of FP64 Gentleman-Sande stages over narr M-point arrays
// (as gs_pass).  Inputs are reduced to |x| <= q/2 + 1 at the start of the
// pass; X' = X + Y, Y' = (X - Y) w mod q (|Y'| <= q).  Stage v: |X - Y| <=
// 2^v (q + 2): stages 0-2 multiply directly (4q + 8 is within dp_mulmod's
// 4q + 8 bound with centred twiddles); stage 3 reduces X - Y first.
// Outputs < 2^K (q/2 + 1).
template <int K, bool RAW = false>
__device__ __forceinline__ void gs_pass_dp(double* sm, int arr_stride, int narr, int logM,
                                           int lt0, int seg, int logMfull,
                                           const double* __restrict__ tw, double q,
                                           double qinv) {
    // RAW: the arrays still hold u64 residues (< 4q < 2^52) as loaded by cp.async
    const int tk = 1 << lt0;
    const int gper = 1 << (logM - K);
    const int total = narr * gper;
    for (int G = threadIdx.x; G < total; G += blockDim.x) {
        const int a = G >> (logM - K), g = G & (gper - 1);
        double* s = sm + a * arr_stride;
        const int blk = g >> lt0, off = g & (tk - 1);
        const int base = (blk << (lt0 + K)) + off;
        double tws[(1 << K) - 1];
#pragma unroll
        for (int v = 0, o = 0; v < K; o += (1 << (K - 1 - v)), ++v) {
            const int lt = lt0 + v;
            const int tb = (1 << (logMfull - lt - 1)) + (seg << (logM - lt - 1)) +
                           (blk << (K - 1 - v));
            load_tw_run(tws + o, tw, tb, 1 << (K - 1 - v));
        }
        // element c sits at PAD(base + c 2^lt0); for lt0 >= 4 that is
        // PAD(base) + c (2^lt0 + 2^(lt0-4)) (base's low lt0 bits are off < 2^lt0):
        // linear addresses, no per-element padding arithmetic (the forward
        // passes keep PAD(): their 64-register cap spills otherwise)
        // (and for any lt0: PAD(base + (c << lt0)) = PAD(base) + PAD(c << lt0),
        //  as in ct_pass_dp)
        const int pbo = PAD(base);
        auto ai = [&](int c) { return pbo + PAD(c << lt0); };
        double x[1 << K];
#pragma unroll
        for (int c = 0; c < (1 << K); ++c) {
            const double v = RAW ? u2d(reinterpret_cast<const u64*>(s)[ai(c)]) : s[ai(c)];
            // raw inputs are lazy residues in [0, 4q) (the MAC's output):
            // stage 0 multiplies X - Y (|.| < 4q) directly and reduces only
            // its sums, after which the bounds below hold as for reduced
            // inputs; other passes reduce every input to |x| <= q/2 + 2
            x[c] = RAW ? v : dp_reduce(v, q, qinv);
        }
#pragma unroll
        for (int v = 0, o = 0; v < K; o += (1 << (K - 1 - v)), ++v) {
            const int half = 1 << v;
#pragma unroll
            for (int c = 0; c < (1 << K); ++c) {
                if (c & half) continue;
                const double X = x[c], Y = x[c + half];
                double u = X - Y;
                if (v >= 3) u = dp_reduce(u, q, qinv);
                x[c] = (RAW && v == 0) ? dp_reduce(X + Y, q, qinv) : X + Y;
                x[c + half] = dp_mulmod(u, tws[o + (c >> (v + 1))], q, qinv);
            }
        }
#pragma unroll
        for (int c = 0; c < (1 << K); ++c) s[ai(c)] = x[c];
    }
}

template <int RMAX, bool RAW = false>
__device__ __forceinline__ void gs_all_dp(double* sm, int arr_stride, int narr, int logM,
                                          int seg, int logMfull, const double* tw, double q,
                                          double qinv) {
    int lt = 0;
    const int rem = logM % RMAX;
    if (RAW) {                                  // first pass converts the raw residues
        if (logM >= RMAX) {
            gs_pass_dp<RMAX, true>(sm, arr_stride, narr, logM, lt, seg, logMfull, tw, q, qinv);
            lt += RMAX;
        } else if (rem == 1) {
            gs_pass_dp<1, true>(sm, arr_stride, narr, logM, lt, seg, logMfull, tw, q, qinv);
            lt += 1;
        } else if (rem == 2) {
            gs_pass_dp<2, true>(sm, arr_stride, narr, logM, lt, seg, logMfull, tw, q, qinv);
            lt += 2;
        } else if (rem == 3) {
            gs_pass_dp<3, true>(sm, arr_stride, narr, logM, lt, seg, logMfull, tw, q, qinv);
            lt += 3;
        }
        __syncthreads();
        if (lt >= logM) return;
    }
    for (; lt + RMAX <= logM; lt += RMAX) {
        gs_pass_dp<RMAX>(sm, arr_stride, narr, logM, lt, seg, logMfull, tw, q, qinv);
        __syncthreads();
    }
    if (lt < logM) {
        if (rem == 1) gs_pass_dp<1>(sm, arr_stride, narr, logM, lt, seg, logMfull, tw, q, qinv);
        else if (rem == 2) gs_pass_dp<2>(sm, arr_stride, narr, logM, lt, seg, logMfull, tw, q, qinv);
        else gs_pass_dp<3>(sm, arr_stride, narr, logM, lt, seg, logMfull, tw, q, qinv);
        __syncthreads();
    }
}

// ---------------------------------------------------- shared-memory NTT

// One pass of K radix-2 Cooley-Tukey stages (forward NTT, bit-reversed
// output), on a segment of NS words of an N-point transform held in shared
// memory.  Stages st0 .. st0+K-1 (stage st has m = 2^st blocks, stride
// t = N >> (st+1)).  `seg` / `split`: this CTA holds words
// [seg*NS, (seg+1)*NS) of the transform (N = NS << split).
template <int K, bool LAZY = false>
__device__ __forceinline__ void ct_pass(u64* sm, int logN, int NS, int st0,
                                        int seg, int split,
                                        const ulonglong2* __restrict__ tw,
                                        u64 q, u64 q2) {
    const int lt0 = logN - st0 - 1;        // log2 t0
    const int ltk = lt0 - (K - 1);         // log2 tk
    const int tk = 1 << ltk;
    const int ngroups = NS >> K;
    for (int g = threadIdx.x; g < ngroups; g += blockDim.x) {
        const int blk = g >> ltk, off = g & (tk - 1);
        const int base = (blk << (lt0 + 1)) + off;
        // all 2^K - 1 twiddles of the group first (independent loads in flight)
        ulonglong2 tws[(1 << K) - 1];
#pragma unroll
        for (int r = 0, o = 0; r < K; o += (1 << r), ++r) {
            const int twb = (1 << (st0 + r)) + (seg << (st0 + r - split)) + (blk << r);
#pragma unroll
            for (int z = 0; z < (1 << r); ++z) tws[o + z] = __ldg(&tw[twb + z]);
        }
        u64 x[1 << K];
#pragma unroll
        for (int c = 0; c < (1 << K); ++c) x[c] = sm[PAD(base + (c << ltk))];
#pragma unroll
        for (int r = 0, o = 0; r < K; o += (1 << r), ++r) {
            const int half = 1 << (K - 1 - r);
#pragma unroll
            for (int c = 0; c < (1 << K); ++c) {
                if (c & half) continue;
                if (LAZY) ct_bfly_lazy(x[c], x[c + half], tws[o + (c >> (K - r))], q, q2);
                else ct_bfly(x[c], x[c + half], tws[o + (c >> (K - r))], q, q2);
            }
        }
#pragma unroll
        for (int c = 0; c < (1 << K); ++c) sm[PAD(base + (c << ltk))] = x[c];
    }
}

// One pass of K radix-2 Gentleman-Sande stages (inverse NTT, bit-reversed
// input, natural output) over `narr` independent M-point transforms stored
// at sm + a * arr_stride.  Strides t = 2^lt0 .. 2^(lt0+K-1); the twiddle of
// block i at stride t is tw_inv[M/(2t) + i] (the prefix of the N-point
// table serves every M = N/s: brv_N(k) = s brv_M(k) for k < M).  `seg`:
// offset of this segment's blocks when the M-point transform is one of
// 2^split segments of a larger transform (logMS = log2 of the full size).
template <int K, bool LAZY = false>
__device__ __forceinline__ void gs_pass(u64* sm, int arr_stride, int narr,
                                        int logM, int lt0, int seg,
                                        int logMfull,
                                        const ulonglong2* __restrict__ tw,
                                        u64 q, u64 q2) {
    const int tk = 1 << lt0;
    const int gper = 1 << (logM - K);
    const int total = narr * gper;
    for (int G = threadIdx.x; G < total; G += blockDim.x) {
        const int a = G >> (logM - K), g = G & (gper - 1);
        u64* s = sm + a * arr_stride;
        const int blk = g >> lt0, off = g & (tk - 1);
        const int base = (blk << (lt0 + K)) + off;
        // all 2^K - 1 twiddles of the group first (independent loads in flight)
        ulonglong2 tws[(1 << K) - 1];
#pragma unroll
        for (int v = 0, o = 0; v < K; o += (1 << (K - 1 - v)), ++v) {
            const int lt = lt0 + v;                       // log2 t
            const int tb = (1 << (logMfull - lt - 1)) + (seg << (logM - lt - 1)) +
                           (blk << (K - 1 - v));
#pragma unroll
            for (int z = 0; z < (1 << (K - 1 - v)); ++z) tws[o + z] = __ldg(&tw[tb + z]);
        }
        u64 x[1 << K];
#pragma unroll
        for (int c = 0; c < (1 << K); ++c) x[c] = s[PAD(base + (c << lt0))];
#pragma unroll
        for (int v = 0, o = 0; v < K; o += (1 << (K - 1 - v)), ++v) {
            const int half = 1 << v;
#pragma unroll
            for (int c = 0; c < (1 << K); ++c) {
                if (c & half) continue;
                if (LAZY) gs_bfly_lazy(x[c], x[c + half], tws[o + (c >> (v + 1))], q,
                                       q << (lt0 + v + 1));
                else gs_bfly(x[c], x[c + half], tws[o + (c >> (v + 1))], q, q2);
            }
        }
#pragma unroll
        for (int c = 0; c < (1 << K); ++c) s[PAD(base + (c << lt0))] = x[c];
    }
}

// Full forward pass schedule on a segment: stages split .. logN-1 in passes
// of up to RMAX stages (the remainder first).
template <int RMAX, bool LAZY = false>
__device__ __forceinline__ void ct_all(u64* sm, int logN, int NS, int seg,
                                       int split, const ulonglong2* tw, u64 q,
                                       u64 q2, int end) {
    int st = split;
    if (st >= end) return;
    const int rem = (end - split) % RMAX;
    if (rem) {
        if (rem == 1) ct_pass<1, LAZY>(sm, logN, NS, st, seg, split, tw, q, q2);
        else if (rem == 2) ct_pass<2, LAZY>(sm, logN, NS, st, seg, split, tw, q, q2);
        else ct_pass<3, LAZY>(sm, logN, NS, st, seg, split, tw, q, q2);
        st += rem;
        __syncthreads();
    }
    for (; st < end; st += RMAX) {
        ct_pass<RMAX, LAZY>(sm, logN, NS, st, seg, split, tw, q, q2);
        __syncthreads();
    }
}

// Full inverse schedule on narr M-point arrays: strides 1 .. M/2.
template <int RMAX, bool LAZY = false>
__device__ __forceinline__ void gs_all(u64* sm, int arr_stride, int narr,
                                       int logM, int seg, int logMfull,
                                       const ulonglong2* tw, u64 q, u64 q2) {
    int lt = 0;
    const int rem = logM % RMAX;
    for (; lt + RMAX <= logM; lt += RMAX) {
        gs_pass<RMAX, LAZY>(sm, arr_stride, narr, logM, lt, seg, logMfull, tw, q, q2);
        __syncthreads();
    }
    if (rem) {
        if (rem == 1) gs_pass<1, LAZY>(sm, arr_stride, narr, logM, lt, seg, logMfull, tw, q, q2);
        else if (rem == 2) gs_pass<2, LAZY>(sm, arr_stride, narr, logM, lt, seg, logMfull, tw, q, q2);
        else gs_pass<3, LAZY>(sm, arr_stride, narr, logM, lt, seg, logMfull, tw, q, q2);
        __syncthreads();
    }
}
