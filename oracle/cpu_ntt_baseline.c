/*
 * cpu_ntt_baseline.c -- the "CPU textbook-NTT path" of SURVEY §8(d)(ii): the
 * server's Conv work unit computed on the host with the standard
 * NTT-domain polynomial products, as a fairer CPU baseline than the
 * sparse-direct oracle.  TEST / BENCHMARK INFRASTRUCTURE ONLY (bench.py's
 * cpu_baseline leg and tests/); it is not a parity reference -- a not-gpu
 * test pins it against the oracle's definition (he_oracle.c
 * orc_conv_server) -- and it shares no code with the CUDA path.
 *
 * Textbook choices: negacyclic NTT by twisting (a_i psi^i, then the cyclic
 * radix-2 Cooley-Tukey NTT with omega = psi^2, bit-reversal permutation,
 * natural order in and out); Shoup multiplication by precomputed constants;
 * no incomplete transform, no fold (PAPER.md:28 cites NTT as the standard
 * product speed-up; Alg. 1 Line 14 computes c0 * fhat^{(n)} in full).
 *   out[b][ob][l][i] = (sum_beta c0_beta * fhat_beta^{(n)})_i   for i = s j + t_n,
 *                      n in block ob; 0 at other i; + enc_l(phi1) everywhere.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef unsigned __int128 u128;

static uint64_t mulm(uint64_t a, uint64_t b, uint64_t q) { return (uint64_t)(((u128)a * b) % q); }
static uint64_t powm(uint64_t a, uint64_t e, uint64_t q) {
    uint64_t r = 1 % q;
    a %= q;
    for (; e; e >>= 1, a = mulm(a, a, q))
        if (e & 1) r = mulm(r, a, q);
    return r;
}
/* x w mod q with wp = floor(w 2^64 / q): result in [0, q) */
static inline uint64_t shoup(uint64_t x, uint64_t w, uint64_t wp, uint64_t q) {
    uint64_t qh = (uint64_t)(((u128)x * wp) >> 64);
    uint64_t r = x * w - qh * q;
    return r >= q ? r - q : r;
}

typedef struct {
    int N, logN;
    uint64_t q;
    uint64_t *tw, *twp;     /* omega^{brv-free} per stage: tw[m + j] for stage length m */
    uint64_t *itw, *itwp;
    uint64_t *psi, *psip, *ipsi, *ipsip;   /* psi^i, N^{-1} psi^{-i} */
} tables;

static void make_tables(tables* T, int N, uint64_t q, uint64_t psi) {
    T->N = N;
    T->logN = 0;
    while ((1 << T->logN) < N) ++T->logN;
    T->q = q;
    size_t n = (size_t)N;
    T->tw = malloc(8 * n); T->twp = malloc(8 * n); T->itw = malloc(8 * n); T->itwp = malloc(8 * n);
    T->psi = malloc(8 * n); T->psip = malloc(8 * n); T->ipsi = malloc(8 * n); T->ipsip = malloc(8 * n);
    uint64_t om = mulm(psi, psi, q), iom = powm(om, q - 2, q), ipsi = powm(psi, q - 2, q);
    uint64_t ninv = powm((uint64_t)N % q, q - 2, q);
    for (int m = 1; m < N; m <<= 1) {           /* stage with butterflies of span m */
        uint64_t w = powm(om, (uint64_t)(N / (2 * m)), q), iw = powm(iom, (uint64_t)(N / (2 * m)), q);
        uint64_t c = 1, ic = 1;
        for (int j = 0; j < m; ++j) {
            T->tw[m + j] = c; T->twp[m + j] = (uint64_t)(((u128)c << 64) / q);
            T->itw[m + j] = ic; T->itwp[m + j] = (uint64_t)(((u128)ic << 64) / q);
            c = mulm(c, w, q);
            ic = mulm(ic, iw, q);
        }
    }
    uint64_t p = 1, ip = ninv;
    for (int i = 0; i < N; ++i) {
        T->psi[i] = p; T->psip[i] = (uint64_t)(((u128)p << 64) / q);
        T->ipsi[i] = ip; T->ipsip[i] = (uint64_t)(((u128)ip << 64) / q);
        p = mulm(p, psi, q);
        ip = mulm(ip, ipsi, q);
    }
}
static void free_tables(tables* T) {
    free(T->tw); free(T->twp); free(T->itw); free(T->itwp);
    free(T->psi); free(T->psip); free(T->ipsi); free(T->ipsip);
}

static void bitrev(uint64_t* a, int N, int logN) {
    for (int i = 0; i < N; ++i) {
        int r = 0;
        for (int b = 0; b < logN; ++b) r |= ((i >> b) & 1) << (logN - 1 - b);
        if (r > i) { uint64_t t = a[i]; a[i] = a[r]; a[r] = t; }
    }
}
/* cyclic NTT (inv = 0) or INTT (inv = 1) in place, natural order in and out */
static void cyc(uint64_t* a, const tables* T, int inv) {
    const int N = T->N;
    const uint64_t q = T->q;
    const uint64_t* w = inv ? T->itw : T->tw;
    const uint64_t* wp = inv ? T->itwp : T->twp;
    bitrev(a, N, T->logN);
    for (int m = 1; m < N; m <<= 1)
        for (int k = 0; k < N; k += 2 * m)
            for (int j = 0; j < m; ++j) {
                uint64_t u = a[k + j], v = shoup(a[k + j + m], w[m + j], wp[m + j], q);
                uint64_t x = u + v, y = u + q - v;
                a[k + j] = x >= q ? x - q : x;
                a[k + j + m] = y >= q ? y - q : y;
            }
}
static void ntt_neg(uint64_t* a, const tables* T) {
    for (int i = 0; i < T->N; ++i) a[i] = shoup(a[i], T->psi[i], T->psip[i], T->q);
    cyc(a, T, 0);
}
static void intt_neg(uint64_t* a, const tables* T) {
    cyc(a, T, 1);
    for (int i = 0; i < T->N; ++i) a[i] = shoup(a[i], T->ipsi[i], T->ipsip[i], T->q);
}

/* In place: spectra of the filter polynomials fhat [nf][L][N] (canonical,
 * Eq. (6)-(7) with the shift; server initialisation, not timed). */
void cpu_ntt_forward(uint64_t* a, int64_t nf, int L, int N, const uint64_t* q,
                     const uint64_t* psi) {
    for (int l = 0; l < L; ++l) {
        tables T;
        make_tables(&T, N, q[l], psi[l]);
#pragma omp parallel for schedule(dynamic)
        for (int64_t f = 0; f < nf; ++f) ntt_neg(a + ((size_t)f * L + l) * N, &T);
        free_tables(&T);
    }
}

/* Shoup companions floor(f 2^64 / q) of the filter spectra (server init). */
void cpu_ntt_companions(const uint64_t* f, uint64_t* fp, int64_t nf, int L, int N,
                        const uint64_t* q) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < nf * L; ++i) {
        const uint64_t ql = q[i % L];
        for (int k = 0; k < N; ++k)
            fp[(size_t)i * N + k] = (uint64_t)(((u128)f[(size_t)i * N + k] << 64) / ql);
    }
}

/* The timed server unit.  c0 [B][n_ib][L][N]; fspec [c_o][n_ib][L][N]
 * (cpu_ntt_forward of the shifted filter polynomials); phi1 [B][n_ob][N] or
 * NULL; enc per limb: delta[l] = Delta_t mod q_l, r_t, t; out [B][n_ob][L][N]. */
void cpu_ntt_conv_server(const uint64_t* c0, int B, int n_ib, int L, int N, const uint64_t* q,
                         const uint64_t* psi, int s, int c_o, int c_ob, int n_ob,
                         const uint64_t* fspec, const uint64_t* fspec_p, const uint32_t* phi1,
                         const uint64_t* delta, uint64_t r_t, uint64_t t, uint64_t* out) {
    const int step = s / c_ob;
    for (int l = 0; l < L; ++l) {
        tables T;
        make_tables(&T, N, q[l], psi[l]);
        const uint64_t ql = q[l];
#pragma omp parallel for schedule(dynamic)
        for (int b = 0; b < B; ++b) {
            uint64_t* C = malloc(sizeof(uint64_t) * (size_t)n_ib * N);
            uint64_t* acc = malloc(sizeof(uint64_t) * (size_t)N);
            for (int beta = 0; beta < n_ib; ++beta) {
                memcpy(C + (size_t)beta * N, c0 + (((size_t)b * n_ib + beta) * L + l) * N,
                       sizeof(uint64_t) * N);
                ntt_neg(C + (size_t)beta * N, &T);
            }
            for (int ob = 0; ob < n_ob; ++ob) {
                uint64_t* o = out + (((size_t)b * n_ob + ob) * L + l) * N;
                memset(o, 0, sizeof(uint64_t) * N);
                for (int nl = 0; nl < c_ob; ++nl) {
                    const int n = ob * c_ob + nl;
                    if (n >= c_o) break;
                    for (int k = 0; k < N; ++k) {
                        uint64_t a = 0;
                        for (int beta = 0; beta < n_ib; ++beta) {
                            const size_t fi = (((size_t)n * n_ib + beta) * L + l) * N + k;
                            a += shoup(C[(size_t)beta * N + k], fspec[fi], fspec_p[fi], ql);
                            a = a >= ql ? a - ql : a;
                        }
                        acc[k] = a;
                    }
                    intt_neg(acc, &T);
                    for (int i = nl * step; i < N; i += s) o[i] = acc[i];   /* slots s j + t_n */
                }
                if (phi1) {
                    const uint32_t* ph = phi1 + ((size_t)b * n_ob + ob) * N;
                    for (int i = 0; i < N; ++i) {
                        uint64_t m = ph[i] % t;
                        uint64_t e = (uint64_t)((((u128)delta[l] * m) + ((u128)r_t * m + t / 2) / t) % ql);
                        uint64_t v = o[i] + e;
                        o[i] = v >= ql ? v - ql : v;
                    }
                }
            }
            free(C);
            free(acc);
        }
        free_tables(&T);
    }
}
