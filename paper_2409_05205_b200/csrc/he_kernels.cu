// he_kernels.cu -- sm_100a kernels and the C-ABI entry points of the
// rotation-free HE Conv/FC server path (arXiv 2409.05205).
//
// Pipeline of he_conv:
//   K1 k_ntt_fwd      c0 -> NTT spectra (bit-reversed), "split25" words
//   K3 k_mac_fold     per (limb l, fold group g): modular GEMM over the
//                     K = n_ib*s spectrum words of the group,
//                     out_fold[l][g][b][n] = sum_k C[b][k] F[k][n]
//   K4 k_intt_scatter per (b, ob, l): (N/s)-point inverse NTTs of the
//                     folded products (root psi^s), scatter to s*j + t_n,
//                     + enc(phi1), full coalesced output row.
// The fold: the server needs only coefficients s*j + t_n of each product
// (PAPER.md:197).  Coefficient s*j of r = c*f equals
// s^{-1} INTT_{N/s, psi^s}( sum of the s spectrum values over the s-th
// roots of each psi^{s(2k+1)} )_j, and in bit-reversed order those s
// values are contiguous.  N^{-1} = s^{-1} (N/s)^{-1} is folded into the
// filter spectra at he_pack_filters time.
#include <cooperative_groups.h>

#include <string.h>

#include <algorithm>

#include "he_internal.cuh"

namespace cg = cooperative_groups;

#define HE_CHECK_LAUNCH()                                   \
    do {                                                    \
        if (cudaGetLastError() != cudaSuccess) return HE_ECUDA; \
    } while (0)

static inline cudaStream_t STREAM(void* s) { return (cudaStream_t)s; }

template <typename F>
static bool set_smem(F* f, size_t bytes) {
    if (bytes <= 48 * 1024) return true;
    return cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)bytes) == cudaSuccess;
}

static inline int ntt_threads(int NS) { return std::min(512, std::max(16, NS / 16)); }

// ===================================================================== K1
// Forward negacyclic NTT, one CTA per limb (N <= 16384; the N = 32768
// variant is k_ntt_fwd_split below).  Smem-staged radix-2^4 passes,
// Shoup twiddles from L1/L2, 16-byte coalesced global loads and stores.
// OUT_FMT 0: canonical, 1: split25 words for the MAC.
template <int OUT_FMT>
__global__ void __launch_bounds__(512)
k_ntt_fwd_body(const u64* in, u64* out, int logN, int L,
               const he_limb* __restrict__ limbs,
               const ulonglong2* __restrict__ tw_all) {
    extern __shared__ u64 sm[];
    const int N = 1 << logN;
    const int li = blockIdx.x, l = li % L;
    const u64 q = limbs[l].q, q2 = 2 * q;
    const ulonglong2* tw = tw_all + (size_t)l * N;
    const u64* src = in + (size_t)li * N;
    for (int i = 2 * threadIdx.x; i < N; i += 2 * blockDim.x) {
        const ulonglong2 v = *reinterpret_cast<const ulonglong2*>(src + i);
        sm[PAD(i)] = v.x;
        sm[PAD(i + 1)] = v.y;
    }
    __syncthreads();
    ct_all(sm, logN, N, 0, 0, tw, q, q2);
    u64* dst = out + (size_t)li * N;
    for (int i = 2 * threadIdx.x; i < N; i += 2 * blockDim.x) {
        u64 x = csub(csub(sm[PAD(i)], q2), q), y = csub(csub(sm[PAD(i + 1)], q2), q);
        if (OUT_FMT == 1) { x = to_split25(x); y = to_split25(y); }
        *reinterpret_cast<ulonglong2*>(dst + i) = make_ulonglong2(x, y);
    }
}

// N = 32768: a 2-CTA cluster per limb; both CTAs read the whole limb, apply
// stage 0 and keep their half (the cluster barrier makes in-place use safe).
template <int OUT_FMT>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(512)
k_ntt_fwd_split(const u64* in, u64* out, int logN,
                int L, const he_limb* __restrict__ limbs,
                const ulonglong2* __restrict__ tw_all) {
    extern __shared__ u64 sm[];
    const int N = 1 << logN, NS = N >> 1;
    const int li = blockIdx.x >> 1, seg = blockIdx.x & 1;
    const int l = li % L;
    const u64 q = limbs[l].q, q2 = 2 * q;
    const ulonglong2* tw = tw_all + (size_t)l * N;
    const u64* src = in + (size_t)li * N;
    const ulonglong2 w = tw[1];
    for (int i = 2 * threadIdx.x; i < NS; i += 2 * blockDim.x) {
        const ulonglong2 a = *reinterpret_cast<const ulonglong2*>(src + i);
        const ulonglong2 b = *reinterpret_cast<const ulonglong2*>(src + i + NS);
        const u64 t0 = shoup_mul(b.x, w.x, w.y, q), t1 = shoup_mul(b.y, w.x, w.y, q);
        sm[PAD(i)] = seg ? a.x - t0 + q2 : a.x + t0;
        sm[PAD(i + 1)] = seg ? a.y - t1 + q2 : a.y + t1;
    }
    cg::this_cluster().sync();          // both halves read before any write
    ct_all(sm, logN, NS, seg, 1, tw, q, q2);
    u64* dst = out + (size_t)li * N + (size_t)seg * NS;
    for (int i = 2 * threadIdx.x; i < NS; i += 2 * blockDim.x) {
        u64 x = csub(csub(sm[PAD(i)], q2), q), y = csub(csub(sm[PAD(i + 1)], q2), q);
        if (OUT_FMT == 1) { x = to_split25(x); y = to_split25(y); }
        *reinterpret_cast<ulonglong2*>(dst + i) = make_ulonglong2(x, y);
    }
}

// Launch the forward NTT over nlimbs = batch * L limbs.
static he_status launch_ntt_fwd(const he_ctx* c, const u64* in, u64* out,
                                long nlimbs, int out_fmt, cudaStream_t st) {
    if (nlimbs <= 0) return HE_OK;
    const int logN = c->logN, N = c->N;
    if (logN <= 14) {
        const int threads = ntt_threads(N);
        const size_t smem = sizeof(u64) * padded_words(N);
        auto k = out_fmt ? k_ntt_fwd_body<1> : k_ntt_fwd_body<0>;
        if (!set_smem(k, smem)) return HE_ECUDA;
        k<<<(unsigned)nlimbs, threads, smem, st>>>(in, out, logN, c->L, c->d_limb,
                                                   c->d_tw_fwd);
    } else {
        const int NS = N / 2;
        const int threads = ntt_threads(NS);
        const size_t smem = sizeof(u64) * padded_words(NS);
        auto k = out_fmt ? k_ntt_fwd_split<1> : k_ntt_fwd_split<0>;
        if (!set_smem(k, smem)) return HE_ECUDA;
        k<<<(unsigned)(2 * nlimbs), threads, smem, st>>>(in, out, logN, c->L,
                                                         c->d_limb, c->d_tw_fwd);
    }
    HE_CHECK_LAUNCH();
    return HE_OK;
}

// ============================================================ inverse NTT
// Full N-point inverse (bit-reversed in, natural out, x N^{-1}).
__global__ void __launch_bounds__(512)
k_ntt_inv(const u64* in, u64* out, int logN, int L,
          const he_limb* __restrict__ limbs, const ulonglong2* __restrict__ twi_all) {
    extern __shared__ u64 sm[];
    const int N = 1 << logN;
    const int li = blockIdx.x, l = li % L;
    const he_limb& Lm = limbs[l];
    const u64 q = Lm.q, q2 = 2 * q;
    const u64* src = in + (size_t)li * N;
    for (int i = 2 * threadIdx.x; i < N; i += 2 * blockDim.x) {
        const ulonglong2 v = *reinterpret_cast<const ulonglong2*>(src + i);
        sm[PAD(i)] = v.x;
        sm[PAD(i + 1)] = v.y;
    }
    __syncthreads();
    gs_all(sm, 0, 1, logN, 0, logN, twi_all + (size_t)l * N, q, q2);
    u64* dst = out + (size_t)li * N;
    const u64 ni = Lm.ninv, nip = Lm.ninv_p;
    for (int i = 2 * threadIdx.x; i < N; i += 2 * blockDim.x) {
        const u64 x = csub(shoup_mul(sm[PAD(i)], ni, nip, q), q);
        const u64 y = csub(shoup_mul(sm[PAD(i + 1)], ni, nip, q), q);
        *reinterpret_cast<ulonglong2*>(dst + i) = make_ulonglong2(x, y);
    }
}

// N = 32768: each CTA of a 2-CTA cluster runs the 14 stages inside its half,
// then the last stage (t = N/2) reads the partner half through DSMEM.
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(512)
k_ntt_inv_split(const u64* in, u64* out, int logN,
                int L, const he_limb* __restrict__ limbs,
                const ulonglong2* __restrict__ twi_all) {
    extern __shared__ u64 sm[];
    const int N = 1 << logN, NS = N >> 1;
    const int li = blockIdx.x >> 1, seg = blockIdx.x & 1, l = li % L;
    const he_limb& Lm = limbs[l];
    const u64 q = Lm.q, q2 = 2 * q;
    const ulonglong2* twi = twi_all + (size_t)l * N;
    const u64* src = in + (size_t)li * N + (size_t)seg * NS;
    for (int i = 2 * threadIdx.x; i < NS; i += 2 * blockDim.x) {
        const ulonglong2 v = *reinterpret_cast<const ulonglong2*>(src + i);
        sm[PAD(i)] = v.x;
        sm[PAD(i + 1)] = v.y;
    }
    __syncthreads();
    gs_all(sm, 0, 1, logN - 1, seg, logN, twi, q, q2);
    cg::cluster_group cl = cg::this_cluster();
    cl.sync();
    const u64* lo = seg ? cl.map_shared_rank(sm, 0) : sm;
    const u64* hi = seg ? sm : cl.map_shared_rank(sm, 1);
    const ulonglong2 w = twi[1];
    u64* dst = out + (size_t)li * N + (size_t)seg * NS;
    for (int i = threadIdx.x; i < NS; i += blockDim.x) {
        u64 x = lo[PAD(i)], y = hi[PAD(i)];
        u64 v = seg ? shoup_mul(x - y + q2, w.x, w.y, q) : csub(x + y, q2);
        dst[i] = csub(shoup_mul(v, Lm.ninv, Lm.ninv_p, q), q);
    }
    cl.sync();                          // keep smem alive for the partner
}

static he_status launch_ntt_inv(const he_ctx* c, const u64* in, u64* out,
                                long nlimbs, cudaStream_t st) {
    if (nlimbs <= 0) return HE_OK;
    const int N = c->N;
    if (c->logN <= 14) {
        const size_t smem = sizeof(u64) * padded_words(N);
        if (!set_smem(k_ntt_inv, smem)) return HE_ECUDA;
        k_ntt_inv<<<(unsigned)nlimbs, ntt_threads(N), smem, st>>>(
            in, out, c->logN, c->L, c->d_limb, c->d_tw_inv);
    } else {
        const size_t smem = sizeof(u64) * padded_words(N / 2);
        if (!set_smem(k_ntt_inv_split, smem)) return HE_ECUDA;
        k_ntt_inv_split<<<(unsigned)(2 * nlimbs), ntt_threads(N / 2), smem, st>>>(
            in, out, c->logN, c->L, c->d_limb, c->d_tw_inv);
    }
    HE_CHECK_LAUNCH();
    return HE_OK;
}

extern "C" he_status he_ntt_forward(const he_ctx* c, uint64_t* d, int batch,
                                    void* stream) {
    if (!c || !d || batch < 0) return HE_EINVAL;
    return launch_ntt_fwd(c, (const u64*)d, (u64*)d, (long)batch * c->L, 0,
                          STREAM(stream));
}

extern "C" he_status he_ntt_inverse(const he_ctx* c, uint64_t* d, int batch,
                                    void* stream) {
    if (!c || !d || batch < 0) return HE_EINVAL;
    return launch_ntt_inv(c, (const u64*)d, (u64*)d, (long)batch * c->L,
                          STREAM(stream));
}

// ===================================================================== K5
// a1: input packing (Eq. (5)) + encoding (+ optional v*b + e0).
struct PlanDev {
    int c_i, c_o, w_i, h_i, f_w, f_h, stride, padw, padh;
    int s, logs, c_ib, n_ib, c_ob, n_ob, w_p, h_p, w_o, h_o, n_valid, step;
};

static PlanDev plan_dev(const he_conv_plan* p) {
    PlanDev d;
    d.c_i = p->d.c_i; d.c_o = p->d.c_o; d.w_i = p->d.w_i; d.h_i = p->d.h_i;
    d.f_w = p->d.f_w; d.f_h = p->d.f_h; d.stride = p->d.stride;
    d.padw = (p->w_p - p->d.w_i) / 2; d.padh = (p->h_p - p->d.h_i) / 2;
    d.s = p->s; d.logs = 0;
    while ((1 << d.logs) < p->s) ++d.logs;
    d.c_ib = p->c_ib; d.n_ib = p->n_ib; d.c_ob = p->c_ob; d.n_ob = p->n_ob;
    d.w_p = p->w_p; d.h_p = p->h_p; d.w_o = p->w_o; d.h_o = p->h_o;
    d.n_valid = p->n_valid; d.step = p->s / p->c_ob;
    return d;
}

static bool plan_ok(const he_ctx* c, const he_conv_plan* p) {
    he_conv_plan chk;
    if (he_conv_plan_make(c, &p->d, p->s, &chk) != HE_OK) return false;
    return memcmp(&chk, p, sizeof(chk)) == 0;
}

__device__ __forceinline__ int floordiv(int a, int b) {
    int q = a / b;
    return (a % b != 0 && ((a < 0) != (b < 0))) ? q - 1 : q;
}

__global__ void k_pack_input(const int32_t* __restrict__ img, const u64* __restrict__ ve,
                             u64* __restrict__ out, PlanDev P, int B, int L, int logN,
                             const he_limb* __restrict__ limbs, u64 t, u64 r_t, u64 t_inv) {
    const long N = 1L << logN;
    const long total = (long)B * P.n_ib * L * N;
    for (long idx = blockIdx.x * (long)blockDim.x + threadIdx.x; idx < total;
         idx += (long)gridDim.x * blockDim.x) {
        const int i = (int)(idx & (N - 1));
        const long r = idx >> logN;
        const int l = (int)(r % L);
        const long bb = r / L;
        const int beta = (int)(bb % P.n_ib), b = (int)(bb / P.n_ib);
        long coef = 0;
#pragma unroll
        for (int cand = 0; cand < 2; ++cand) {
            const int e = cand ? i - (int)N : i;
            const int m = e & (P.s - 1);                  // e mod s (floor)
            const int Pq = (e - m) >> P.logs;             // exact
            const int kk = floordiv(Pq, P.h_p);
            const int ll = Pq - kk * P.h_p;
            const int k = kk + P.f_w;
            const int ch = beta * P.c_ib + m;
            if (k >= 0 && k < P.w_p && m < P.c_ib && ch < P.c_i) {
                const int ki = k - P.padw, li = ll - P.padh;
                long pix = 0;
                if (ki >= 0 && ki < P.w_i && li >= 0 && li < P.h_i)
                    pix = img[(((long)b * P.c_i + ch) * P.w_i + ki) * P.h_i + li];
                coef = cand ? -pix : pix;
                break;
            }
        }
        long mt = coef % (long)t;
        if (mt < 0) mt += t;
        const he_limb& Lm = limbs[l];
        u64 v = enc_plain((u64)mt, Lm, t, r_t, t_inv);
        if (ve) v = addmod(v, ve[idx], Lm.q);
        out[idx] = v;
    }
}

static unsigned grid_for(long total, int threads) {
    long g = (total + threads - 1) / threads;
    return (unsigned)std::max(1L, std::min(g, 148L * 32));
}

extern "C" he_status he_pack_input(const he_ctx* c, const he_conv_plan* p,
                                   const int32_t* d_img, int B, const uint64_t* d_ve,
                                   uint64_t* d_pt, void* stream) {
    if (!c || !p || !d_img || !d_pt || B < 0) return HE_EINVAL;
    if (!plan_ok(c, p)) return HE_ESHAPE;
    if (B == 0) return HE_OK;
    const long total = (long)B * p->n_ib * c->L * c->N;
    k_pack_input<<<grid_for(total, 256), 256, 0, STREAM(stream)>>>(
        d_img, (const u64*)d_ve, (u64*)d_pt, plan_dev(p), B, c->L, c->logN,
        c->d_limb, c->t, c->r_t, c->t_inv);
    HE_CHECK_LAUNCH();
    return HE_OK;
}

// ===================================================================== K6
// a2: dense filter polynomials f_beta^{(n)} (Eq. (6), UNshifted: the
// Eq. (7) shift X^{t_n} is realised by K4's scatter offset), per limb.
__global__ void k_pack_filter_coeffs(const int32_t* __restrict__ W, u64* __restrict__ out,
                                     PlanDev P, int L, int logN,
                                     const he_limb* __restrict__ limbs) {
    const long N = 1L << logN;
    const long total = (long)P.c_o * P.n_ib * L * N;
    for (long idx = blockIdx.x * (long)blockDim.x + threadIdx.x; idx < total;
         idx += (long)gridDim.x * blockDim.x) {
        const int i = (int)(idx & (N - 1));
        const long r = idx >> logN;
        const int l = (int)(r % L);
        const long nb = r / L;
        const int beta = (int)(nb % P.n_ib), n = (int)(nb / P.n_ib);
        long w = 0;
        for (int cand = 0; cand < 2; ++cand) {
            const int e = cand ? i + (int)N : i;            // e in (0, N]
            if (e == 0) continue;
            const int m = (P.s - (e & (P.s - 1))) & (P.s - 1);
            const int Pp = (e + m) >> P.logs;
            const int Z = P.h_p * P.f_w - Pp;               // = k h_p + l
            if (Z < 0) continue;
            const int k = Z / P.h_p, ll = Z % P.h_p;
            const int ch = beta * P.c_ib + m;
            if (k < P.f_w && ll < P.f_h && m < P.c_ib && ch < P.c_i) {
                const long wv = W[(((long)n * P.c_i + ch) * P.f_w + k) * P.f_h + ll];
                w = cand ? -wv : wv;
                break;
            }
        }
        const u64 q = limbs[l].q;
        out[idx] = w >= 0 ? (u64)w % q : q - ((u64)(-w) % q);
    }
}

// spectra [c_o][n_ib][L][N] (canonical, bit-reversed) -> MAC layout
// F[l][g][k][n] = split25(spec[n][beta][l][g s + u] * N^{-1}), k = beta s + u.
__global__ void k_filter_to_mac(const u64* __restrict__ spec, u64* __restrict__ F,
                                PlanDev P, int L, int logN,
                                const he_limb* __restrict__ limbs) {
    const long N = 1L << logN;
    const int K = P.n_ib * P.s;
    const long total = (long)L * N * P.n_ib * P.c_o;  // = L * M * K * c_o
    for (long idx = blockIdx.x * (long)blockDim.x + threadIdx.x; idx < total;
         idx += (long)gridDim.x * blockDim.x) {
        const int n = (int)(idx % P.c_o);
        long r = idx / P.c_o;
        const int k = (int)(r % K);
        r /= K;
        const int M = (int)(N >> P.logs);
        const int g = (int)(r % M);
        const int l = (int)(r / M);
        const int beta = k >> P.logs, u = k & (P.s - 1);
        const he_limb& Lm = limbs[l];
        const u64 v = spec[(((long)n * P.n_ib + beta) * L + l) * N + ((long)g << P.logs) + u];
        F[idx] = to_split25(csub(shoup_mul(v, Lm.ninv, Lm.ninv_p, Lm.q), Lm.q));
    }
}

extern "C" size_t he_filter_bytes(const he_ctx* c, const he_conv_plan* p) {
    if (!c || !p) return 0;
    return sizeof(u64) * (size_t)p->d.c_o * p->n_ib * c->L * c->N;
}

extern "C" size_t he_pack_filters_workspace_bytes(const he_ctx* c,
                                                  const he_conv_plan* p) {
    return he_filter_bytes(c, p);
}

extern "C" he_status he_pack_filters(const he_ctx* c, const he_conv_plan* p,
                                     const int32_t* d_w, uint64_t* d_fspec,
                                     void* d_ws, size_t ws_bytes, void* stream) {
    if (!c || !p || !d_w || !d_fspec || !d_ws) return HE_EINVAL;
    if (!plan_ok(c, p)) return HE_ESHAPE;
    if (ws_bytes < he_pack_filters_workspace_bytes(c, p)) return HE_ENOMEM;
    cudaStream_t st = STREAM(stream);
    const PlanDev P = plan_dev(p);
    u64* ws = (u64*)d_ws;
    const long total = (long)P.c_o * P.n_ib * c->L * c->N;
    k_pack_filter_coeffs<<<grid_for(total, 256), 256, 0, st>>>(d_w, ws, P, c->L,
                                                                c->logN, c->d_limb);
    HE_CHECK_LAUNCH();
    he_status s = launch_ntt_fwd(c, ws, ws, (long)P.c_o * P.n_ib * c->L, 0, st);
    if (s != HE_OK) return s;
    k_filter_to_mac<<<grid_for(total, 256), 256, 0, st>>>(ws, (u64*)d_fspec, P, c->L,
                                                           c->logN, c->d_limb);
    HE_CHECK_LAUNCH();
    return HE_OK;
}

// ===================================================================== K3
// Folded NTT-domain MAC: for each (l, g), the modular GEMM
//   out[l][g][b][n] = sum_{k < K} C[b][beta][l][g s + u] * F[l][g][k][n] mod q
// (k = beta s + u).  Operands are split25 words: v = hi * 2^25 + lo, so each
// term is 4 IMAD.WIDE.U32 into three 64-bit accumulators (acc0: lo*lo,
// acc1: cross, acc2: hi*hi), reduced once per output.  K <= 4096 keeps the
// accumulators below 2^64.
__device__ __forceinline__ u64 mac_reduce(u64 a0, u64 a1, u64 a2, const he_limb& Lm) {
    const u64 q = Lm.q;
    u64 r = shoup_mul(a0, 1, Lm.one_p, q) + shoup_mul(a1, Lm.r25, Lm.r25_p, q) +
            shoup_mul(a2, Lm.r50, Lm.r50_p, q);          // < 6q
    r = csub(r, 4 * q);
    r = csub(r, 2 * q);
    return csub(r, q);
}

template <int TM, int TN>
__global__ void __launch_bounds__(256)
k_mac_fold(const u64* __restrict__ C, const u64* __restrict__ F, u64* __restrict__ out,
           int B, int n_ib, int L, int logN, int logs, int c_o, int GC,
           const he_limb* __restrict__ limbs) {
    constexpr int TBc = 16 * TM, TNc = 16 * TN, KC = 32;
    __shared__ u64 sC[KC][TBc + 1];
    __shared__ u64 sF[KC][TNc];
    const int N = 1 << logN, s = 1 << logs, M = N >> logs, K = n_ib * s;
    const int nG = (M + GC - 1) / GC;
    const int l = blockIdx.x / nG, g0 = (blockIdx.x % nG) * GC;
    const int b0 = blockIdx.y * TBc, n0 = blockIdx.z * TNc;
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    const he_limb Lm = limbs[l];
    for (int g = g0; g < min(g0 + GC, M); ++g) {
        u64 a0[TM][TN], a1[TM][TN], a2[TM][TN];
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
            for (int j = 0; j < TN; ++j) a0[i][j] = a1[i][j] = a2[i][j] = 0;
        const u64* Fg = F + ((size_t)l * M + g) * K * c_o;
        for (int k0 = 0; k0 < K; k0 += KC) {
            const int kc = min(KC, K - k0);
            for (int idx = threadIdx.x; idx < TBc * kc; idx += 256) {
                const int bl = idx / kc, kk = idx - bl * kc;
                const int b = b0 + bl, k = k0 + kk;
                u64 v = 0;
                if (b < B)
                    v = C[(((size_t)b * n_ib + (k >> logs)) * L + l) * N +
                          ((size_t)g << logs) + (k & (s - 1))];
                sC[kk][bl] = v;
            }
            for (int idx = threadIdx.x; idx < kc * TNc; idx += 256) {
                const int kk = idx / TNc, nl = idx - kk * TNc;
                const int n = n0 + nl;
                sF[kk][nl] = n < c_o ? Fg[(size_t)(k0 + kk) * c_o + n] : 0;
            }
            __syncthreads();
            for (int kk = 0; kk < kc; ++kk) {
                u32 c0[TM], c1[TM], f0[TN], f1[TN];
#pragma unroll
                for (int i = 0; i < TM; ++i) {
                    const u64 v = sC[kk][ty + 16 * i];
                    c0[i] = (u32)v;
                    c1[i] = (u32)(v >> 32);
                }
#pragma unroll
                for (int j = 0; j < TN; ++j) {
                    const u64 v = sF[kk][tx + 16 * j];
                    f0[j] = (u32)v;
                    f1[j] = (u32)(v >> 32);
                }
#pragma unroll
                for (int i = 0; i < TM; ++i)
#pragma unroll
                    for (int j = 0; j < TN; ++j) {
                        a0[i][j] += (u64)c0[i] * f0[j];
                        a1[i][j] += (u64)c0[i] * f1[j];
                        a1[i][j] += (u64)c1[i] * f0[j];
                        a2[i][j] += (u64)c1[i] * f1[j];
                    }
            }
            __syncthreads();
        }
        u64* og = out + ((size_t)l * M + g) * B * c_o;
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
            for (int j = 0; j < TN; ++j) {
                const int b = b0 + ty + 16 * i, n = n0 + tx + 16 * j;
                if (b < B && n < c_o)
                    og[(size_t)b * c_o + n] = mac_reduce(a0[i][j], a1[i][j], a2[i][j], Lm);
            }
    }
}

template <int TM, int TN>
static void launch_mac_t(const u64* C, const u64* F, u64* out, int B, int n_ib, int L,
                         int logN, int logs, int c_o, const he_limb* limbs,
                         cudaStream_t st) {
    const int M = (1 << logN) >> logs, K = n_ib << logs;
    int GC = std::max(1, 256 / K);
    GC = std::min(GC, M);
    const int nG = (M + GC - 1) / GC;
    dim3 grid(L * nG, (B + 16 * TM - 1) / (16 * TM), (c_o + 16 * TN - 1) / (16 * TN));
    k_mac_fold<TM, TN><<<grid, 256, 0, st>>>(C, F, out, B, n_ib, L, logN, logs, c_o, GC,
                                             limbs);
}

static void launch_mac(const u64* C, const u64* F, u64* out, int B, int n_ib, int L,
                       int logN, int logs, int c_o, const he_limb* limbs, cudaStream_t st) {
    const int tm = B > 32 ? 4 : (B > 16 ? 2 : 1);
    const int tn = c_o > 32 ? 4 : (c_o > 16 ? 2 : 1);
#define MAC_CASE(A, Bt) \
    if (tm == A && tn == Bt) { launch_mac_t<A, Bt>(C, F, out, B, n_ib, L, logN, logs, c_o, limbs, st); return; }
    MAC_CASE(1, 1) MAC_CASE(1, 2) MAC_CASE(1, 4)
    MAC_CASE(2, 1) MAC_CASE(2, 2) MAC_CASE(2, 4)
    MAC_CASE(4, 1) MAC_CASE(4, 2) MAC_CASE(4, 4)
#undef MAC_CASE
}

// ===================================================================== K4
// Per (b, ob, l): (N/s)-point inverse NTTs (root psi^s, no scaling: N^{-1}
// is in the filter spectra) of the folded products of the block's channels,
// then the full output row: slot s*j + t_n <- result_n[j] (Alg. 1 Lines
// 15-17; Eq. (7) shift as offset t_n), other slots 0, + enc(phi1) at every
// coefficient.  Channels are processed in chunks of `cc`
// that fit shared memory; a slot owned by no channel is written with the
// first chunk.
__global__ void __launch_bounds__(512)
k_intt_scatter(const u64* __restrict__ fold, const u32* __restrict__ phi1,
               u64* __restrict__ out, PlanDev P, int B, int L, int logN, int cc,
               const he_limb* __restrict__ limbs, const ulonglong2* __restrict__ twi_all,
               u64 t, u64 r_t, u64 t_inv) {
    extern __shared__ u64 sm[];
    const int N = 1 << logN, M = N >> P.logs, logM = logN - P.logs;
    const int stride = padded_words(M);
    const int l = blockIdx.x % L;
    const int bo = blockIdx.x / L, ob = bo % P.n_ob, b = bo / P.n_ob;
    const he_limb Lm = limbs[l];
    const u64 q = Lm.q, q2 = 2 * q;
    const ulonglong2* twi = twi_all + (size_t)l * N;
    const u32* ph = phi1 ? phi1 + ((size_t)b * P.n_ob + ob) * N : nullptr;
    u64* orow = out + (((size_t)b * P.n_ob + ob) * L + l) * N;
    for (int ch0 = 0; ch0 < P.c_ob; ch0 += cc) {
        const int ncc = min(cc, P.c_ob - ch0);
        for (int idx = threadIdx.x; idx < ncc * M; idx += blockDim.x) {
            const int g = idx / ncc, a = idx - g * ncc;
            const int n = ob * P.c_ob + ch0 + a;
            sm[a * stride + PAD(g)] =
                n < P.c_o ? fold[(((size_t)l * M + g) * B + b) * P.c_o + n] : 0;
        }
        __syncthreads();
        gs_all(sm, stride, ncc, logM, 0, logM, twi, q, q2);
        for (int i = threadIdx.x; i < N; i += blockDim.x) {
            const int u = i & (P.s - 1), j = i >> P.logs;
            const int nl = u / P.step;
            const bool owned = (u - nl * P.step == 0) && nl < P.c_ob;
            u64 v;
            if (owned && nl >= ch0 && nl < ch0 + ncc) v = csub(sm[(nl - ch0) * stride + PAD(j)], q);
            else if (!owned && ch0 == 0) v = 0;
            else continue;
            if (ph) v = addmod(v, enc_plain(ph[i], Lm, t, r_t, t_inv), q);
            orow[i] = v;
        }
        __syncthreads();
    }
}

extern "C" size_t he_conv_workspace_bytes(const he_ctx* c, const he_conv_plan* p, int B) {
    if (!c || !p || B < 0) return 0;
    const size_t M = (size_t)c->N / p->s;
    const size_t spec = (size_t)B * p->n_ib * c->L * c->N;
    const size_t fold = (size_t)c->L * M * B * p->d.c_o;
    return sizeof(u64) * (spec + fold) + 256;
}

static inline void rec(void* const* ev, int i, cudaStream_t st) {
    if (ev && ev[i]) cudaEventRecord((cudaEvent_t)ev[i], st);
}

extern "C" he_status he_conv(const he_ctx* c, const he_conv_plan* p, const uint64_t* d_c0,
                             int B, const uint64_t* d_fspec, const uint32_t* d_phi1,
                             uint64_t* d_out, void* d_ws, size_t ws_bytes, void* stream) {
    return he_conv_ex(c, p, d_c0, B, d_fspec, d_phi1, d_out, d_ws, ws_bytes, stream, nullptr);
}

extern "C" he_status he_conv_ex(const he_ctx* c, const he_conv_plan* p, const uint64_t* d_c0,
                                int B, const uint64_t* d_fspec, const uint32_t* d_phi1,
                                uint64_t* d_out, void* d_ws, size_t ws_bytes, void* stream,
                                void* const* ev) {
    if (!c || !p || B < 0) return HE_EINVAL;
    if (!plan_ok(c, p)) return HE_ESHAPE;
    if (B == 0) return HE_OK;
    if (!d_c0 || !d_fspec || !d_out || !d_ws) return HE_EINVAL;
    if (ws_bytes < he_conv_workspace_bytes(c, p, B)) return HE_ENOMEM;
    cudaStream_t st = STREAM(stream);
    const PlanDev P = plan_dev(p);
    u64* spec = (u64*)d_ws;
    u64* fold = spec + (size_t)B * P.n_ib * c->L * c->N;
    rec(ev, 0, st);
    he_status s = launch_ntt_fwd(c, (const u64*)d_c0, spec, (long)B * P.n_ib * c->L, 1, st);
    if (s != HE_OK) return s;
    rec(ev, 1, st);
    launch_mac(spec, (const u64*)d_fspec, fold, B, P.n_ib, c->L, c->logN, P.logs, P.c_o,
               c->d_limb, st);
    HE_CHECK_LAUNCH();
    const int M = c->N >> P.logs;
    const int max_words = 16384;                  // 128 KB of shared memory
    int cc = std::max(1, std::min(P.c_ob, max_words / padded_words(M)));
    const size_t smem = sizeof(u64) * (size_t)cc * padded_words(M);
    if (!set_smem(k_intt_scatter, smem)) return HE_ECUDA;
    rec(ev, 2, st);
    k_intt_scatter<<<(unsigned)(B * P.n_ob * c->L), 512, smem, st>>>(
        fold, d_phi1, (u64*)d_out, P, B, c->L, c->logN, cc, c->d_limb, c->d_tw_inv, c->t,
        c->r_t, c->t_inv);
    HE_CHECK_LAUNCH();
    rec(ev, 3, st);
    return HE_OK;
}

// ===================================================================== K7
__global__ void k_mask_extract(const u64* __restrict__ full, const u32* __restrict__ phi1,
                               u64* __restrict__ comp, PlanDev P, int B, int L, int logN,
                               const he_limb* __restrict__ limbs, u64 t, u64 r_t, u64 t_inv) {
    const long N = 1L << logN;
    const long total = (long)B * P.n_ob * L * P.n_valid;
    for (long idx = blockIdx.x * (long)blockDim.x + threadIdx.x; idx < total;
         idx += (long)gridDim.x * blockDim.x) {
        const int v = (int)(idx % P.n_valid);
        const long r = idx / P.n_valid;
        const int l = (int)(r % L);
        const long bo = r / L;
        const int nl = v % P.c_ob, Pq = v / P.c_ob;
        const int Lc = Pq % P.h_o, Kr = Pq / P.h_o;
        const long i = (long)P.s * (P.stride * Kr * (long)P.h_p + P.stride * Lc) +
                       (long)nl * P.step;
        u64 x = full[r * N + i];
        if (phi1) {
            const he_limb& Lm = limbs[l];
            x = addmod(x, enc_plain(phi1[bo * N + i], Lm, t, r_t, t_inv), Lm.q);
        }
        comp[idx] = x;
    }
}

extern "C" he_status he_mask_extract(const he_ctx* c, const he_conv_plan* p,
                                     const uint64_t* d_out, int B, const uint32_t* d_phi1,
                                     uint64_t* d_compact, void* stream) {
    if (!c || !p || !d_out || !d_compact || B < 0) return HE_EINVAL;
    if (!plan_ok(c, p)) return HE_ESHAPE;
    if (B == 0) return HE_OK;
    const long total = (long)B * p->n_ob * c->L * p->n_valid;
    k_mask_extract<<<grid_for(total, 256), 256, 0, STREAM(stream)>>>(
        (const u64*)d_out, d_phi1, (u64*)d_compact, plan_dev(p), B, c->L, c->logN, c->d_limb,
        c->t, c->r_t, c->t_inv);
    HE_CHECK_LAUNCH();
    return HE_OK;
}

// ===================================================================== FC
static bool fc_ok(const he_ctx* c, const he_fc_desc* f) {
    return f && f->n_i >= 1 && f->n_o >= 1 && (long)f->n_i * f->n_o <= (long)c->N &&
           c->logN <= 14;
}

__global__ void k_pack_fc_input(const int32_t* __restrict__ in, const u64* __restrict__ ve,
                                u64* __restrict__ out, int n_i, int n_o, int B, int L,
                                int logN, const he_limb* __restrict__ limbs, u64 t, u64 r_t,
                                u64 t_inv) {
    const long N = 1L << logN;
    const long total = (long)B * L * N;
    for (long idx = blockIdx.x * (long)blockDim.x + threadIdx.x; idx < total;
         idx += (long)gridDim.x * blockDim.x) {
        const int i = (int)(idx & (N - 1));
        const long r = idx >> logN;
        const int l = (int)(r % L), b = (int)(r / L);
        long m = 0;
        if (i % n_o == 0 && i / n_o < n_i) m = in[(long)b * n_i + i / n_o];   // Eq. (9)
        long mt = m % (long)t;
        if (mt < 0) mt += t;
        const he_limb& Lm = limbs[l];
        u64 v = enc_plain((u64)mt, Lm, t, r_t, t_inv);
        if (ve) v = addmod(v, ve[idx], Lm.q);
        out[idx] = v;
    }
}

extern "C" he_status he_pack_fc_input(const he_ctx* c, const he_fc_desc* f,
                                      const int32_t* d_in, int B, const uint64_t* d_ve,
                                      uint64_t* d_pt, void* stream) {
    if (!c || !f || !d_in || !d_pt || B < 0) return HE_EINVAL;
    if (!fc_ok(c, f)) return HE_ESHAPE;
    if (B == 0) return HE_OK;
    const long total = (long)B * c->L * c->N;
    k_pack_fc_input<<<grid_for(total, 256), 256, 0, STREAM(stream)>>>(
        d_in, (const u64*)d_ve, (u64*)d_pt, f->n_i, f->n_o, B, c->L, c->logN, c->d_limb, c->t,
        c->r_t, c->t_inv);
    HE_CHECK_LAUNCH();
    return HE_OK;
}

// dense w(X) (R17) per limb
__global__ void k_fc_weight_coeffs(const int32_t* __restrict__ W, u64* __restrict__ out,
                                   int n_i, int n_o, int L, int logN,
                                   const he_limb* __restrict__ limbs) {
    const long N = 1L << logN;
    for (long idx = blockIdx.x * (long)blockDim.x + threadIdx.x; idx < L * N;
         idx += (long)gridDim.x * blockDim.x) {
        const int i = (int)(idx & (N - 1)), l = (int)(idx >> logN);
        long w = 0;
        if (i < n_o) {
            w = W[(long)i * n_i];                                  // W_{i,0} X^i
        } else {
            const long d = N - i;                                  // = l' n_o - k
            const long lp = (d + n_o - 1) / n_o;
            const long k = lp * n_o - d;
            if (lp >= 1 && lp < n_i) w = -(long)W[k * n_i + lp];   // -W_{k,l'}
        }
        const u64 q = limbs[l].q;
        out[idx] = w >= 0 ? (u64)w % q : q - ((u64)(-w) % q);
    }
}

// spectrum -> {w N^{-1}, Shoup}; bias -> enc
__global__ void k_fc_finish_weights(const u64* __restrict__ spec, ulonglong2* __restrict__ wspec,
                                    const int32_t* __restrict__ bias, u64* __restrict__ bias_enc,
                                    int n_o, int L, int logN, const he_limb* __restrict__ limbs,
                                    u64 t, u64 r_t, u64 t_inv) {
    const long N = 1L << logN;
    for (long idx = blockIdx.x * (long)blockDim.x + threadIdx.x; idx < L * N;
         idx += (long)gridDim.x * blockDim.x) {
        const int l = (int)(idx >> logN), i = (int)(idx & (N - 1));
        const he_limb& Lm = limbs[l];
        const u64 w = csub(shoup_mul(spec[idx], Lm.ninv, Lm.ninv_p, Lm.q), Lm.q);
        wspec[idx] = make_ulonglong2(w, (u64)(((unsigned __int128)w << 64) / Lm.q));
        if (i < n_o) {
            long m = bias ? bias[i] : 0;
            long mt = m % (long)t;
            if (mt < 0) mt += t;
            bias_enc[(long)l * n_o + i] = enc_plain((u64)mt, Lm, t, r_t, t_inv);
        }
    }
}

extern "C" size_t he_fc_wspec_bytes(const he_ctx* c, const he_fc_desc* f) {
    if (!c || !f) return 0;
    return sizeof(ulonglong2) * (size_t)c->L * c->N;
}

extern "C" size_t he_fc_workspace_bytes(const he_ctx* c, const he_fc_desc* f, int B) {
    if (!c || !f || B < 0) return 0;
    return sizeof(u64) * (size_t)std::max(B, 1) * c->L * c->N;
}

extern "C" he_status he_pack_fc_weights(const he_ctx* c, const he_fc_desc* f,
                                        const int32_t* d_W, const int32_t* d_bias,
                                        uint64_t* d_wspec, uint64_t* d_bias_enc, void* d_ws,
                                        size_t ws_bytes, void* stream) {
    if (!c || !f || !d_W || !d_wspec || !d_bias_enc || !d_ws) return HE_EINVAL;
    if (!fc_ok(c, f)) return HE_ESHAPE;
    if (ws_bytes < sizeof(u64) * (size_t)c->L * c->N) return HE_ENOMEM;
    cudaStream_t st = STREAM(stream);
    u64* ws = (u64*)d_ws;
    const long total = (long)c->L * c->N;
    k_fc_weight_coeffs<<<grid_for(total, 256), 256, 0, st>>>(d_W, ws, f->n_i, f->n_o, c->L,
                                                             c->logN, c->d_limb);
    HE_CHECK_LAUNCH();
    he_status s = launch_ntt_fwd(c, ws, ws, c->L, 0, st);
    if (s != HE_OK) return s;
    k_fc_finish_weights<<<grid_for(total, 256), 256, 0, st>>>(
        ws, (ulonglong2*)d_wspec, d_bias, (u64*)d_bias_enc, f->n_o, c->L, c->logN, c->d_limb,
        c->t, c->r_t, c->t_inv);
    HE_CHECK_LAUNCH();
    return HE_OK;
}

// Per (b, l): pointwise product with the weight spectrum, N-point inverse
// NTT (N^{-1} pre-folded), first n_o coefficients + enc(bias) + enc(phi1).
__global__ void __launch_bounds__(512)
k_fc_inv(const u64* __restrict__ spec, const ulonglong2* __restrict__ wspec,
         const u64* __restrict__ bias_enc, const u32* __restrict__ phi1, u64* __restrict__ out,
         int n_o, int L, int logN, const he_limb* __restrict__ limbs,
         const ulonglong2* __restrict__ twi_all, u64 t, u64 r_t, u64 t_inv) {
    extern __shared__ u64 sm[];
    const int N = 1 << logN;
    const int li = blockIdx.x, l = li % L, b = li / L;
    const he_limb Lm = limbs[l];
    const u64 q = Lm.q, q2 = 2 * q;
    const u64* src = spec + (size_t)li * N;
    const ulonglong2* ws = wspec + (size_t)l * N;
    for (int i = threadIdx.x; i < N; i += blockDim.x) {
        const ulonglong2 w = __ldg(&ws[i]);
        sm[PAD(i)] = shoup_mul(src[i], w.x, w.y, q);      // [0, 2q)
    }
    __syncthreads();
    gs_all(sm, 0, 1, logN, 0, logN, twi_all + (size_t)l * N, q, q2);
    for (int k = threadIdx.x; k < n_o; k += blockDim.x) {
        u64 v = csub(sm[PAD(k)], q);
        v = addmod(v, bias_enc[(size_t)l * n_o + k], q);
        if (phi1) v = addmod(v, enc_plain(phi1[(size_t)b * n_o + k], Lm, t, r_t, t_inv), q);
        out[(size_t)li * n_o + k] = v;
    }
}

extern "C" he_status he_fc(const he_ctx* c, const he_fc_desc* f, const uint64_t* d_c0, int B,
                           const uint64_t* d_wspec, const uint64_t* d_bias_enc,
                           const uint32_t* d_phi1, uint64_t* d_out, void* d_ws,
                           size_t ws_bytes, void* stream) {
    return he_fc_ex(c, f, d_c0, B, d_wspec, d_bias_enc, d_phi1, d_out, d_ws, ws_bytes, stream,
                    nullptr);
}

extern "C" he_status he_fc_ex(const he_ctx* c, const he_fc_desc* f, const uint64_t* d_c0,
                              int B, const uint64_t* d_wspec, const uint64_t* d_bias_enc,
                              const uint32_t* d_phi1, uint64_t* d_out, void* d_ws,
                              size_t ws_bytes, void* stream, void* const* ev) {
    if (!c || !f || B < 0) return HE_EINVAL;
    if (!fc_ok(c, f)) return HE_ESHAPE;
    if (B == 0) return HE_OK;
    if (!d_c0 || !d_wspec || !d_bias_enc || !d_out || !d_ws) return HE_EINVAL;
    if (ws_bytes < he_fc_workspace_bytes(c, f, B)) return HE_ENOMEM;
    cudaStream_t st = STREAM(stream);
    u64* spec = (u64*)d_ws;
    rec(ev, 0, st);
    he_status s = launch_ntt_fwd(c, (const u64*)d_c0, spec, (long)B * c->L, 0, st);
    if (s != HE_OK) return s;
    const size_t smem = sizeof(u64) * padded_words(c->N);
    if (!set_smem(k_fc_inv, smem)) return HE_ECUDA;
    rec(ev, 1, st);
    k_fc_inv<<<(unsigned)(B * c->L), ntt_threads(c->N), smem, st>>>(
        spec, (const ulonglong2*)d_wspec, (const u64*)d_bias_enc, d_phi1, (u64*)d_out, f->n_o,
        c->L, c->logN, c->d_limb, c->d_tw_inv, c->t, c->r_t, c->t_inv);
    HE_CHECK_LAUNCH();
    rec(ev, 2, st);
    return HE_OK;
}
