/*
 * he_oracle.c -- plain, slow, obviously-correct CPU oracle for the
 * rotation-free HE Conv/FC server path of arXiv 2409.05205.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or constant generator with the CUDA
 * path (paper_2409_05205_b200/), and the CUDA path never links it.
 *
 * Every routine is the textbook definition written out with unsigned
 * __int128 arithmetic; no NTT, no blocking, no lazy reduction.  Citations
 * are PAPER.md line (section, equation / algorithm).  The readings R1..R26
 * are listed in DESIGN.md ("Readings of the paper").
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef unsigned __int128 u128;
typedef __int128 i128;

static uint64_t mulmod(uint64_t a, uint64_t b, uint64_t q) {
    return (uint64_t)(((u128)a * b) % q);
}

static uint64_t powmod(uint64_t a, uint64_t e, uint64_t q) {
    uint64_t r = 1 % q;
    a %= q;
    while (e) {
        if (e & 1) r = mulmod(r, a, q);
        a = mulmod(a, a, q);
        e >>= 1;
    }
    return r;
}

/* signed 128-bit value -> canonical residue in [0, q) */
static uint64_t smod(i128 x, uint64_t q) {
    i128 r = x % (i128)q;
    if (r < 0) r += q;
    return (uint64_t)r;
}

uint64_t orc_powmod(uint64_t a, uint64_t e, uint64_t q) { return powmod(a, e, q); }
uint64_t orc_mulmod(uint64_t a, uint64_t b, uint64_t q) { return mulmod(a, b, q); }

/*
 * Negacyclic product coefficients (§II-A: "modular reduction
 * by X^N+1 is carried out after polynomial multiplications"):
 *   c_k = sum_{i+j=k} a_i b_j - sum_{i+j=k+N} a_i b_j  (mod q)
 * evaluated only at the requested positions (pos == NULL: all k < N).
 * a, b canonical residues.  O(N) per position.
 */
void orc_negacyclic_at(const uint64_t* a, const uint64_t* b, int N, uint64_t q,
                       const int32_t* pos, int npos, uint64_t* out) {
    int n = pos ? npos : N;
#pragma omp parallel for schedule(static)
    for (int p = 0; p < n; ++p) {
        int k = pos ? pos[p] : p;
        u128 plus = 0, minus = 0;
        for (int i = 0; i < N; ++i) {
            int j = k - i;
            if (j >= 0) plus += (u128)a[i] * b[j];
            else minus += (u128)a[i] * b[j + N];
            /* keep the sums well inside 128 bits */
            if ((i & 1023) == 1023) { plus %= q; minus %= q; }
        }
        uint64_t P = (uint64_t)(plus % q), M = (uint64_t)(minus % q);
        out[p] = P >= M ? P - M : P + q - M;
    }
}

/*
 * Product of a dense residue polynomial a with a sparse integer polynomial
 * sum_t w_t X^{e_t} (0 <= e_t < N), full negacyclic result mod q.
 * Definition: X^{e} * X^{i} = X^{i+e} if i+e < N, else -X^{i+e-N}.
 */
void orc_sparse_mul(const uint64_t* a, int N, uint64_t q, const int32_t* e,
                    const int64_t* w, int nterms, uint64_t* out) {
#pragma omp parallel for schedule(static)
    for (int k = 0; k < N; ++k) {
        i128 acc = 0;
        for (int t = 0; t < nterms; ++t) {
            int i = k - e[t];
            if (i >= 0) acc += (i128)w[t] * (i128)a[i];
            else acc -= (i128)w[t] * (i128)a[i + N];
        }
        out[k] = smod(acc, q);
    }
}

/*
 * BFV-style encoding (R2):  enc_j(m) = round(Q * m / t) mod q_j
 *   = (Delta_t mod q_j) * m + floor((r_t * m + floor(t/2)) / t)   (mod q_j)
 * with Delta_t = floor(Q/t), r_t = Q mod t, m in [0, t).  The constants
 * Delta_t mod q_j and r_t come from the oracle's own big-integer code
 * (oracle/ref.py); a not-gpu test checks this routine against the literal
 * big-integer round(Q*m/t).
 */
static uint64_t enc1(uint64_t m, uint64_t q, uint64_t delta_mod_q, uint64_t r_t,
                     uint64_t t) {
    uint64_t frac = (uint64_t)(((u128)r_t * m + t / 2) / t);
    return (uint64_t)(((u128)delta_mod_q * m + frac) % q);
}

void orc_encode(const uint32_t* m, int64_t n, uint64_t q, uint64_t delta_mod_q,
                uint64_t r_t, uint64_t t, uint64_t* out) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) out[i] = enc1(m[i] % t, q, delta_mod_q, r_t, t);
}

/*
 * Server side of Algorithm 1 + the additive mask
 * (PAPER.md:280), written as the plain definition:
 *
 *   c0^{(n)} = sum_beta c0_beta * fhat_beta^{(n)}     (Alg.1 Line 14, R13)
 *   c0^r_{ob}[s*j + t_n] = c0^{(n)}[s*j + t_n]         (Lines 15-17, R11/R14)
 *   c0^r_{ob}[i] = 0 at every other i
 *   c0^r_{ob}[i] += enc_l(phi1[b][ob][i])  for all i   (mask, R15)
 *
 * Each needed coefficient is computed directly from the definition of the
 * negacyclic product with the sparse filter polynomial fhat (which already
 * contains the Eq. (7) shift X^{t_n}; exponents are reduced to [0, N) with
 * the sign folded into the weight by the caller).
 *
 * c0     : uint64 [B][n_ib][L][N]
 * t_off  : int32 [c_o + 1]  (terms for channel n, all blocks beta, are in
 *          [t_off[n], t_off[n+1]); term t has block tb[t], exponent te[t],
 *          signed weight tw[t])
 * phi1   : uint32 [B][n_ob][N] or NULL
 * out    : uint64 [B][n_ob][L][N]
 */
void orc_conv_server(const uint64_t* c0, int B, int n_ib, int L, int N,
                     const uint64_t* q, int s, int c_o, int c_ob, int n_ob,
                     const int32_t* t_off, const int32_t* tb, const int32_t* te,
                     const int64_t* tw, const uint32_t* phi1,
                     const uint64_t* delta_mod_q, uint64_t r_t, uint64_t t,
                     uint64_t* out) {
    const int step = s / c_ob;      /* t_n = (n mod c_ob) * s / c_ob */
#pragma omp parallel for collapse(3) schedule(dynamic)
    for (int b = 0; b < B; ++b)
        for (int ob = 0; ob < n_ob; ++ob)
            for (int l = 0; l < L; ++l) {
                uint64_t* o = out + (((size_t)b * n_ob + ob) * L + l) * N;
                memset(o, 0, sizeof(uint64_t) * (size_t)N);
                for (int nl = 0; nl < c_ob; ++nl) {
                    int n = ob * c_ob + nl;
                    if (n >= c_o) break;
                    int tn = nl * step;
                    for (int j = 0; j < N / s; ++j) {
                        int i = s * j + tn;
                        i128 acc = 0;
                        for (int k = t_off[n]; k < t_off[n + 1]; ++k) {
                            const uint64_t* cb =
                                c0 + (((size_t)b * n_ib + tb[k]) * L + l) * N;
                            int idx = i - te[k];
                            if (idx >= 0) acc += (i128)tw[k] * (i128)cb[idx];
                            else acc -= (i128)tw[k] * (i128)cb[idx + N];
                        }
                        o[i] = smod(acc, q[l]);
                    }
                }
                if (phi1) {
                    const uint32_t* ph = phi1 + ((size_t)b * n_ob + ob) * N;
                    for (int i = 0; i < N; ++i) {
                        uint64_t e = enc1(ph[i] % t, q[l], delta_mod_q[l], r_t, t);
                        uint64_t v = o[i] + e;
                        o[i] = v >= q[l] ? v - q[l] : v;
                    }
                }
            }
}

/*
 * Server side of Algorithm 2 (Line 13) restricted to the
 * first n_o coefficients, plus the mask:
 *   out[b][l][k] = (c0 * w)_k + enc_l(B_k) + enc_l(phi1[b][k]),  k < n_o
 * w given as sparse terms (exponent, signed weight) in [0, N).
 * c0: uint64 [B][L][N]; bias_m, phi1 values in [0,t) (phi1 may be NULL);
 * out: uint64 [B][L][n_o].
 */
void orc_fc_server(const uint64_t* c0, int B, int L, int N, const uint64_t* q,
                   int n_o, const int32_t* te, const int64_t* tw, int nterms,
                   const uint32_t* bias_m, const uint32_t* phi1,
                   const uint64_t* delta_mod_q, uint64_t r_t, uint64_t t,
                   uint64_t* out) {
#pragma omp parallel for collapse(2) schedule(static)
    for (int b = 0; b < B; ++b)
        for (int l = 0; l < L; ++l) {
            const uint64_t* c = c0 + ((size_t)b * L + l) * N;
            for (int k = 0; k < n_o; ++k) {
                i128 acc = 0;
                for (int tt = 0; tt < nterms; ++tt) {
                    int idx = k - te[tt];
                    if (idx >= 0) acc += (i128)tw[tt] * (i128)c[idx];
                    else acc -= (i128)tw[tt] * (i128)c[idx + N];
                }
                uint64_t v = smod(acc, q[l]);
                if (bias_m) v = (uint64_t)(((u128)v + enc1(bias_m[k] % t, q[l], delta_mod_q[l], r_t, t)) % q[l]);
                if (phi1) v = (uint64_t)(((u128)v + enc1(phi1[(size_t)b * n_o + k] % t, q[l], delta_mod_q[l], r_t, t)) % q[l]);
                out[((size_t)b * L + l) * n_o + k] = v;
            }
        }
}

/*
 * Definition of the negacyclic NTT (R9): A[k] = a(psi^{2k+1}) mod q for the
 * requested k (natural order).  O(N) per k, Horner-free direct sum.
 */
void orc_ntt_def(const uint64_t* a, int N, uint64_t q, uint64_t psi,
                 const int32_t* ks, int nk, uint64_t* out) {
#pragma omp parallel for schedule(static)
    for (int p = 0; p < nk; ++p) {
        uint64_t x = powmod(psi, 2 * (uint64_t)ks[p] + 1, q);
        uint64_t xp = 1, acc = 0;
        for (int i = 0; i < N; ++i) {
            acc = (uint64_t)(((u128)acc + (u128)a[i] * xp) % q);
            xp = mulmod(xp, x, q);
        }
        out[p] = acc;
    }
}

/*
 * Definition of the inverse: a_i = N^{-1} sum_k A[k] psi^{-(2k+1) i}.
 * A in natural order, full N outputs.  O(N^2).
 */
void orc_intt_def(const uint64_t* A, int N, uint64_t q, uint64_t psi,
                  uint64_t* out) {
    uint64_t psi_inv = powmod(psi, q - 2, q);
    uint64_t n_inv = powmod((uint64_t)N, q - 2, q);
    uint64_t* pw = (uint64_t*)malloc(sizeof(uint64_t) * 2 * (size_t)N);
    pw[0] = 1;
    for (int e = 1; e < 2 * N; ++e) pw[e] = mulmod(pw[e - 1], psi_inv, q);
#pragma omp parallel for schedule(static)
    for (int i = 0; i < N; ++i) {
        uint64_t acc = 0;
        for (int k = 0; k < N; ++k) {
            uint64_t e = ((2 * (uint64_t)k + 1) * (uint64_t)i) % (2 * (uint64_t)N);
            acc = (uint64_t)(((u128)acc + (u128)A[k] * pw[e]) % q);
        }
        out[i] = mulmod(acc, n_inv, q);
    }
    free(pw);
}
