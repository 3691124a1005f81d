// he_host.cu -- context creation (ring validation, psi, twiddle tables),
// the packing plan and status strings.  Host code only.
#include <stdlib.h>
#include <string.h>

#include <vector>

#include <algorithm>

#include "he_internal.cuh"

typedef unsigned __int128 u128;

static u64 h_mulmod(u64 a, u64 b, u64 q) { return (u64)(((u128)a * b) % q); }
static u64 h_powmod(u64 a, u64 e, u64 q) {
    u64 r = 1 % q;
    a %= q;
    while (e) {
        if (e & 1) r = h_mulmod(r, a, q);
        a = h_mulmod(a, a, q);
        e >>= 1;
    }
    return r;
}
static u64 h_shoup(u64 w, u64 q) { return (u64)(((u128)w << 64) / q); }
static u64 h_inv(u64 a, u64 q) { return h_powmod(a, q - 2, q); }  // q prime

// Deterministic Miller-Rabin for 64-bit n (bases 2..37).
static bool h_is_prime(u64 n) {
    static const u64 B[] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
    if (n < 2) return false;
    for (u64 p : B)
        if (n % p == 0) return n == p;
    u64 d = n - 1;
    int r = 0;
    while (!(d & 1)) { d >>= 1; ++r; }
    for (u64 a : B) {
        u64 x = h_powmod(a, d, n);
        if (x == 1 || x == n - 1) continue;
        bool comp = true;
        for (int i = 1; i < r; ++i) {
            x = h_mulmod(x, x, n);
            if (x == n - 1) { comp = false; break; }
        }
        if (comp) return false;
    }
    return true;
}

static uint32_t brv(uint32_t x, int bits) {
    uint32_t r = 0;
    for (int i = 0; i < bits; ++i) { r = (r << 1) | (x & 1); x >>= 1; }
    return r;
}

// Smallest primitive 2N-th root of unity (reading R9): find one root x with
// x^N = -1, then the minimum over its N odd powers.
static u64 h_min_psi(u64 q, uint32_t N) {
    u64 x = 0;
    for (u64 g = 2;; ++g) {
        x = h_powmod(g, (q - 1) / (2 * (u64)N), q);
        if (h_powmod(x, N, q) == q - 1) break;
    }
    u64 best = x, x2 = h_mulmod(x, x, q), cur = x;
    for (uint32_t i = 1; i < N; ++i) {
        cur = h_mulmod(cur, x2, q);
        if (cur < best) best = cur;
    }
    return best;
}

extern "C" const char* he_status_str(he_status s) {
    switch (s) {
        case HE_OK: return "HE_OK";
        case HE_EINVAL: return "HE_EINVAL: invalid argument";
        case HE_ESHAPE: return "HE_ESHAPE: layer does not fit the ring / unsupported geometry";
        case HE_EPARAM: return "HE_EPARAM: invalid ring parameters";
        case HE_ECUDA: return "HE_ECUDA: CUDA error";
        case HE_ENOMEM: return "HE_ENOMEM: workspace too small";
    }
    return "HE_?: unknown status";
}

extern "C" void he_ctx_destroy(he_ctx* c) {
    if (!c) return;
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(c->device);
    cudaFree(c->d_limb);
    cudaFree(c->d_tw_fwd);
    cudaFree(c->d_tw_inv);
    cudaFree(c->d_enc);
    cudaFree(c->d_twd_fwd);
    cudaFree(c->d_twd_inv);
    cudaSetDevice(prev);
    free(c->q_host);
    free(c->psi_host);
    free(c->limb_host);
    free(c);
}

extern "C" he_status he_ctx_create(const he_ring_desc* r, int device,
                                   he_ctx** out) {
    if (!r || !out || !r->q) return HE_EINVAL;
    *out = nullptr;
    if (r->log2N < 8 || r->log2N > 15 || r->L < 1 || r->L > 64) return HE_EPARAM;
    if (r->t < 3 || !(r->t & 1) || r->t >= (1ull << 32)) return HE_EPARAM;
    const uint32_t N = 1u << r->log2N, L = r->L;
    for (uint32_t j = 0; j < L; ++j) {
        u64 q = r->q[j];
        if (q >= (1ull << 50) || q < 3 || (q - 1) % (2 * (u64)N) != 0 || !h_is_prime(q))
            return HE_EPARAM;
        if (q % r->t == 0) return HE_EPARAM;
        for (uint32_t i = 0; i < j; ++i)
            if (r->q[i] == q) return HE_EPARAM;
    }
    he_ctx* c = (he_ctx*)calloc(1, sizeof(he_ctx));
    c->device = device;
    {
        const char* m = getenv("HE_MAC");
        c->mac_mode = (m && m[0] == 'i') ? 1 : 0;     // HE_MAC=imad forces the IMAD MAC
        const char* t = getenv("HE_NTT");
        c->ntt_mode = (t && t[0] == 'i') ? 1 : 0;     // HE_NTT=int: integer butterflies
        const char* k = getenv("HE_NTT_COLS");
        // HE_NTT_COLS=0: cluster kernels only; =1: column kernel whenever possible
        c->ntt_cluster = (k && k[0] == '0') ? 1 : ((k && k[0] == '1') ? 2 : 0);
        // read once here: the hot path never calls getenv
        c->ntt_r8 = getenv("HE_NTT_R8") != nullptr;
        const char* tc = getenv("HE_MAC_TC");
        c->mac_tc = tc ? atoi(tc) : 2;
    }
    c->logN = r->log2N;
    c->N = N;
    c->L = L;
    c->t = r->t;
    // r_t = Q mod t = prod (q_j mod t) mod t  (no big integers needed)
    u64 rt = 1 % r->t;
    for (uint32_t j = 0; j < L; ++j) rt = h_mulmod(rt, r->q[j] % r->t, r->t);
    c->r_t = rt;
    c->t_inv = (u64)(((u128)1 << 64) / r->t);
    c->q_host = (u64*)malloc(sizeof(u64) * L);
    c->psi_host = (u64*)malloc(sizeof(u64) * L);
    c->limb_host = (he_limb*)malloc(sizeof(he_limb) * L);
    std::vector<ulonglong2> fwd((size_t)L * N), inv((size_t)L * N);
    std::vector<double> fwdd((size_t)L * N), invd((size_t)L * N);
    for (uint32_t j = 0; j < L; ++j) {
        const u64 q = r->q[j];
        c->q_host[j] = q;
        const u64 psi = h_min_psi(q, N);
        c->psi_host[j] = psi;
        const u64 psi_inv = h_inv(psi, q);
        // powers psi^e, psi^{-e} for e < N
        std::vector<u64> pw(N), pwi(N);
        pw[0] = pwi[0] = 1;
        for (uint32_t e = 1; e < N; ++e) {
            pw[e] = h_mulmod(pw[e - 1], psi, q);
            pwi[e] = h_mulmod(pwi[e - 1], psi_inv, q);
        }
        for (uint32_t k = 0; k < N; ++k) {
            const u64 w = pw[brv(k, r->log2N)], wi = pwi[brv(k, r->log2N)];
            fwd[(size_t)j * N + k] = make_ulonglong2(w, h_shoup(w, q));
            inv[(size_t)j * N + k] = make_ulonglong2(wi, h_shoup(wi, q));
            // FP64 twiddles centred into (-q/2, q/2): |w| <= (q-1)/2 lets the
            // FP64 butterflies multiply operands up to 4q without a prior
            // reduction (he_internal.cuh, dp_mulmod)
            fwdd[(size_t)j * N + k] = w > q / 2 ? -(double)(q - w) : (double)w;
            invd[(size_t)j * N + k] = wi > q / 2 ? -(double)(q - wi) : (double)wi;
        }
        he_limb& Lm = c->limb_host[j];
        Lm.q = q;
        Lm.q2 = 2 * q;
        Lm.ninv = h_inv(N % q, q);
        Lm.ninv_p = h_shoup(Lm.ninv, q);
        // Delta_t = floor(Q/t) = (Q - r_t)/t, and Q = 0 mod q_j:
        // Delta_t mod q_j = -r_t * t^{-1} mod q_j.
        Lm.delta = h_mulmod((q - rt % q) % q, h_inv(r->t % q, q), q);
        Lm.delta_p = h_shoup(Lm.delta, q);
        Lm.r25 = (1ull << 25) % q;
        Lm.r25_p = h_shoup(Lm.r25, q);
        Lm.r50 = (1ull << 50) % q;
        Lm.r50_p = h_shoup(Lm.r50, q);
        Lm.r40 = (u64)(((u128)1 << 40) % q);
        Lm.r40_p = h_shoup(Lm.r40, q);
        Lm.r80 = h_mulmod(Lm.r40, Lm.r40, q);
        Lm.r80_p = h_shoup(Lm.r80, q);
        Lm.r64 = (u64)(((u128)1 << 64) % q);
        Lm.r64_p = h_shoup(Lm.r64, q);
        Lm.one_p = h_shoup(1, q);
        {   // -q^{-1} mod 2^64 by Newton iteration (q odd): x <- x (2 - q x)
            u64 x = q;                      // q q = 1 mod 8: 3 correct bits
            for (int it = 0; it < 5; ++it) x *= 2 - q * x;
            Lm.mq = (u64)0 - x;
            auto centred = [q](u64 v) { return v > q / 2 ? -(double)(q - v) : (double)v; };
            const u64 i32 = h_inv((1ull << 32) % q, q);            // 2^-32
            Lm.mrd[0] = centred(h_mulmod(i32, i32, q));          // 2^-64
            Lm.mrd[1] = centred(i32);
            Lm.mrd[2] = centred((1ull << 32) % q);               // 2^32
            Lm.pw8[0] = 1u << 8;
            Lm.pw8[1] = 1u << 16;
            Lm.pw8[2] = 1u << 24;
        }
        Lm.td = (double)r->t;
        Lm.t_invd = 1.0 / (double)r->t;
        Lm.rtd = (double)rt;
        Lm.qd = (double)q;
        Lm.qinvd = 1.0 / (double)q;
        {
            const u64 ti = h_inv(r->t % q, q);
            Lm.tinvd = ti > q / 2 ? -(double)(q - ti) : (double)ti;
            auto centred = [q](u64 v) { return v > q / 2 ? -(double)(q - v) : (double)v; };
            const u64 c32 = (1ull << 32) % q;
            const u64 c64 = (u64)(((u128)1 << 64) % q);
            Lm.c32d = centred(c32);
            Lm.c64d = centred(c64);
            Lm.c96d = centred(h_mulmod(c64, c32, q));
        }
    }
    int prev = 0;
    cudaGetDevice(&prev);
    if (cudaSetDevice(device) != cudaSuccess) { he_ctx_destroy(c); return HE_ECUDA; }
    bool ok = cudaMalloc(&c->d_limb, sizeof(he_limb) * L) == cudaSuccess &&
              cudaMalloc(&c->d_tw_fwd, sizeof(ulonglong2) * L * N) == cudaSuccess &&
              cudaMalloc(&c->d_tw_inv, sizeof(ulonglong2) * L * N) == cudaSuccess &&
              cudaMemcpy(c->d_limb, c->limb_host, sizeof(he_limb) * L,
                         cudaMemcpyHostToDevice) == cudaSuccess &&
              cudaMemcpy(c->d_tw_fwd, fwd.data(), sizeof(ulonglong2) * L * N,
                         cudaMemcpyHostToDevice) == cudaSuccess &&
              cudaMemcpy(c->d_tw_inv, inv.data(), sizeof(ulonglong2) * L * N,
                         cudaMemcpyHostToDevice) == cudaSuccess &&
              cudaMalloc(&c->d_twd_fwd, sizeof(double) * L * N) == cudaSuccess &&
              cudaMalloc(&c->d_twd_inv, sizeof(double) * L * N) == cudaSuccess &&
              cudaMemcpy(c->d_twd_fwd, fwdd.data(), sizeof(double) * L * N,
                         cudaMemcpyHostToDevice) == cudaSuccess &&
              cudaMemcpy(c->d_twd_inv, invd.data(), sizeof(double) * L * N,
                         cudaMemcpyHostToDevice) == cudaSuccess;
    if (ok && r->t <= (1u << 20)) {
        // enc_j(m) = (Delta_t mod q_j) m + floor((r_t m + floor(t/2)) / t) mod q_j
        const u64 t = r->t;
        std::vector<u64> tab((size_t)L * t);
        for (uint32_t j = 0; j < L; ++j) {
            const u64 q = c->q_host[j], d = c->limb_host[j].delta;
            for (u64 m = 0; m < t; ++m)
                tab[(size_t)j * t + m] =
                    (u64)(((u128)d * m + ((u128)rt * m + t / 2) / t) % q);
        }
        ok = cudaMalloc(&c->d_enc, sizeof(u64) * tab.size()) == cudaSuccess &&
             cudaMemcpy(c->d_enc, tab.data(), sizeof(u64) * tab.size(),
                        cudaMemcpyHostToDevice) == cudaSuccess;
    }
    cudaSetDevice(prev);
    if (!ok) { cudaGetLastError(); he_ctx_destroy(c); return HE_ECUDA; }
    *out = c;
    return HE_OK;
}

extern "C" uint64_t he_ctx_psi(const he_ctx* c, uint32_t j) {
    return (c && j < c->L) ? c->psi_host[j] : 0;
}

extern "C" he_status he_conv_plan_make(const he_ctx* c, const he_conv_desc* d,
                                       int s_override, he_conv_plan* out) {
    if (!c || !d || !out) return HE_EINVAL;
    if (d->c_i < 1 || d->c_o < 1 || d->w_i < 1 || d->h_i < 1 || d->f_w < 1 ||
        d->f_h < 1 || d->stride < 1 || (d->stride & (d->stride - 1)) ||
        (d->pad != 0 && d->pad != 1))
        return HE_ESHAPE;
    const long N = c->N;
    const int padw = d->pad ? (d->f_w - 1) / 2 : 0;
    const int padh = d->pad ? (d->f_h - 1) / 2 : 0;
    const long w_p = d->w_i + 2 * padw, h_p = d->h_i + 2 * padh;
    if (w_p < d->f_w || h_p < d->f_h || w_p * h_p > N) return HE_ESHAPE;
    long s;
    if (s_override) {
        s = s_override;
        if (s < 1 || (s & (s - 1)) || s * w_p * h_p > N) return HE_ESHAPE;
    } else {
        s = 1;
        while (2 * s * w_p * h_p <= N) s *= 2;
    }
    he_conv_plan p;
    p.d = *d;
    p.s = (int32_t)s;
    p.c_ib = d->c_i < s ? d->c_i : (int32_t)s;
    p.n_ib = (d->c_i + p.c_ib - 1) / p.c_ib;
    p.c_ob = d->c_o < s ? d->c_o : (int32_t)s;
    p.n_ob = (d->c_o + p.c_ob - 1) / p.c_ob;
    p.w_p = (int32_t)w_p;
    p.h_p = (int32_t)h_p;
    p.w_o = (int32_t)((w_p - d->f_w + 1) / d->stride);
    p.h_o = (int32_t)((h_p - d->f_h + 1) / d->stride);
    p.n_valid = p.c_ob * p.w_o * p.h_o;
    // columns of each fold group that meet nonzero filter operands
    p.k_u = std::min<int32_t>((int32_t)s, (p.c_ib + 3) & ~3);
    if ((long)p.n_ib * s > 4096) return HE_ESHAPE;       // MAC headroom
    *out = p;
    return HE_OK;
}

extern "C" he_status he_conv_plan_dense(const he_conv_plan* p, he_conv_plan* out) {
    if (!p || !out) return HE_EINVAL;
    *out = *p;
    out->k_u = p->s;
    return HE_OK;
}
