/*
 * he_rotfree.h -- C ABI of the B200 (sm_100a) server hot path of
 * arXiv 2409.05205, "Efficient Homomorphically Encrypted Convolutional
 * Neural Network Without Rotation" (Akherati & Zhang).
 *
 * The library evaluates, on the GPU, the server side of the paper's
 * rotation-free Conv procedure (Algorithm 1: Line 14
 * product c0 * fhat^(n), Lines 15-17 valid-slot extraction) and FC
 * procedure (Algorithm 2, Line 13: c0 * w + b), plus the
 * additive mask phi1 of the garbled-circuit bridge, in an
 * RNS ring Z_Q[X]/(X^N+1), Q = q_0 ... q_{L-1}, each q_j prime, q_j < 2^50,
 * q_j = 1 (mod 2N) (§II-A; BASELINE.json north_star).
 *
 * Conventions (all entry points):
 *  - Every device buffer is allocated and owned by the caller.  The
 *    library owns only the context tables (allocated in he_ctx_create) and
 *    never allocates or synchronises in the hot path; all work is enqueued
 *    on the caller's stream (`stream` is a cudaStream_t, NULL = legacy
 *    default stream) and the call returns without waiting.
 *  - Residue buffers are uint64_t, canonical (each value in [0, q_j)); the
 *    library's outputs are always canonical.  Inputs that are not
 *    canonical give unspecified (but memory-safe) results.
 *  - Polynomials are stored coefficient-major: the innermost axis is the
 *    N coefficients of one limb, the next axis the L limbs.
 *  - Errors: argument / shape checks are synchronous and return a status
 *    before anything is enqueued.  HE_ECUDA reports a launch error from
 *    cudaGetLastError(); asynchronous faults surface at the caller's next
 *    synchronisation.  he_status_str() names each status.
 *  - Plaintext-scale values (image pixels, mask phi1, FC bias) are encoded
 *    as enc_j(m) = round(Q * (m mod t) / t) mod q_j (BFV-style, DESIGN.md
 *    reading R2; the paper's CKKS ⌈Δm⌋ of Eq. (1)).
 */
#ifndef HE_ROTFREE_H
#define HE_ROTFREE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    HE_OK = 0,
    HE_EINVAL = 1,   /* null pointer, non-positive batch, bad argument      */
    HE_ESHAPE = 2,   /* layer does not fit the ring / unsupported geometry  */
    HE_EPARAM = 3,   /* ring parameters: q not prime, q >= 2^50, q != 1 mod
                        2N, duplicate q, t even or t >= 2^32, N unsupported  */
    HE_ECUDA = 4,    /* CUDA launch / allocation error                      */
    HE_ENOMEM = 5    /* caller workspace too small                          */
} he_status;

const char* he_status_str(he_status s);
/* Text of the CUDA error behind the last HE_ECUDA returned on the calling
 * host thread ("no error" if none).  The pointer is static. */
const char* he_last_cuda_error(void);

/* ------------------------------------------------------------------ ring */
/* Ring description.  log2N in [8, 15]; 1 <= L <= 64; q[L]
 * host array (copied); t odd, 3 <= t < 2^32. */
typedef struct {
    uint32_t log2N;
    uint32_t L;
    const uint64_t* q;
    uint64_t t;
} he_ring_desc;

typedef struct he_ctx he_ctx;

/* Creates an immutable context on CUDA device `device`: validates the ring
 * (HE_EPARAM), picks psi_j = the smallest primitive 2N-th root of unity mod
 * q_j (reading R9), and uploads the twiddle tables (psi^{brv(k)} and its
 * inverse with Shoup companions) and per-limb constants.  The context may
 * be used concurrently from several streams. */
he_status he_ctx_create(const he_ring_desc* r, int device, he_ctx** out);
void he_ctx_destroy(he_ctx* ctx);
/* psi_j used for limb j (host value). */
uint64_t he_ctx_psi(const he_ctx* ctx, uint32_t j);

/* ------------------------------------------------------------------ conv */
/* Conv layer geometry in the paper's notation (§II-B):
 * w_i = image rows, h_i = row length, f_w = filter rows, f_h = filter
 * columns, stride s_w = s_h = stride, pad 1 = "same" (client zero-pads
 * (f-1)/2 on each side), 0 = valid. */
typedef struct {
    int32_t c_i, c_o, w_i, h_i, f_w, f_h, stride, pad;
} he_conv_desc;

/* Packing plan (reading R11).  s = largest power of two with
 * s * w_p * h_p <= N (the paper's spacing s = c_i of Eq. (5)-(7) when its
 * preconditions hold); c_ib = min(c_i, s) input
 * channels per input ciphertext (n_ib blocks), c_ob = min(c_o, s) output
 * channels per output ciphertext (n_ob blocks); output channel n of a block
 * sits at offset t_n = (n mod c_ob) * (s / c_ob) (Eq. (7) shift n c_i/c_o);
 * n_valid = c_ob * w_o * h_o valid slots per output block. */
typedef struct {
    he_conv_desc d;
    int32_t s, c_ib, n_ib, c_ob, n_ob, w_p, h_p, w_o, h_o, n_valid;
    /* columns u < k_u of each fold group enter the MAC (K = n_ib k_u).  The
     * filter polynomials of Eq. (6) have exponents -m mod s (m < c_ib), so
     * after the incomplete transform their operand is zero for u >= c_ib:
     * he_conv_plan_make sets k_u = c_ib rounded up to a multiple of 4 (<= s).
     * A dense second operand (the client's p of Alg. 1 Line 5) needs
     * k_u = s: he_conv_plan_dense. */
    int32_t k_u;
} he_conv_plan;

/* Host-only, deterministic.  s_override = 0 applies R11; otherwise it must
 * be a power of two with s_override * w_p * h_p <= N (paper-literal layouts
 * use s = c_i).  HE_ESHAPE if the padded image does not fit, if
 * n_ib * s > 4096 (MAC accumulator headroom), for c_i, c_o, sizes < 1 or
 * for a stride that is not a power of two. */
he_status he_conv_plan_make(const he_ctx* ctx, const he_conv_desc* d,
                            int s_override, he_conv_plan* out);

/* The same plan with k_u = s, for he_pack_client_p / he_conv on the
 * client's dense operand.  HE_EINVAL on NULL. */
he_status he_conv_plan_dense(const he_conv_plan* p, he_conv_plan* out);

/* a1, client side (Eq. (5); Alg. 1 Line 2).  Packs
 * d_img int32 [B][c_i][w_i][h_i] into the input polynomials
 *   i_beta(X) = sum_m sum_{k,l} Ip^{(beta c_ib + m)}_{k,l} X^{s((k-f_w)h_p+l)+m}
 * (negacyclic sign on negative exponents) and encodes every coefficient
 * with enc_j, giving d_pt uint64 [B][n_ib][L][N].  If d_ve is non-NULL
 * (uint64 [B][n_ib][L][N], the caller's v*b + e0 residues of Eq. (1)) it
 * is added mod q_j, so d_pt becomes the c0-only encryption of Alg. 1
 * Line 9.  d_ve may alias d_pt. */
he_status he_pack_input(const he_ctx* ctx, const he_conv_plan* p,
                        const int32_t* d_img, int B, const uint64_t* d_ve,
                        uint64_t* d_pt, void* stream);

/* a2, server initialisation (Eq. (6)-(7); Alg. 1
 * Line 4).  Packs d_w int32 [c_o][c_i][f_w][f_h] (weights, any sign, used
 * unscaled: R3) into the filter polynomials, runs the incomplete forward
 * transform (the first log2(N/s) stages) and stores the fold
 * operand F'_{g,u} = (N/s)^{-1} (u ? zeta_g F_{g,s-u} : F_{g,0}), u < k_u,
 * in the opaque layout d_fspec (he_filter_bytes() bytes) consumed by
 * he_conv: byte planes for the int8 tensor-core MAC, 25-bit split words for
 * the IMAD MAC.  d_ws: workspace of he_pack_filters_workspace_bytes()
 * bytes (the coefficient polynomials). */
size_t he_filter_bytes(const he_ctx* ctx, const he_conv_plan* p);
size_t he_pack_filters_workspace_bytes(const he_ctx* ctx,
                                       const he_conv_plan* p);
he_status he_pack_filters(const he_ctx* ctx, const he_conv_plan* p,
                          const int32_t* d_w, uint64_t* d_fspec, void* d_ws,
                          size_t ws_bytes, void* stream);

/* a3-a7, the server hot path (Alg. 1 Lines 13-17; mask
 * PAPER.md:280).  d_c0 uint64 [B][n_ib][L][N] (c0 of each input block);
 * d_fspec from he_pack_filters; d_phi1 uint32 [B][n_ob][N] mask values in
 * [0, t) or NULL (no mask).  Writes the full output polynomials
 *   d_out[b][ob][j][s*k + t_n] = (sum_beta c0_beta * fhat_beta^{(n)})_{s*k+t_n}
 * for every k < N/s and channel n of block ob, 0 at every other
 * coefficient, then + enc_j(phi1[b][ob][i]) at every coefficient i.
 * d_out uint64 [B][n_ob][L][N].  d_ws: he_conv_workspace_bytes(B) bytes
 * (HE_ENOMEM if smaller); the workspace must not overlap d_c0, d_fspec,
 * d_phi1 or the outputs (the forward transform reads d_c0 while it writes
 * the workspace). */
size_t he_conv_workspace_bytes(const he_ctx* ctx, const he_conv_plan* p,
                               int B);
he_status he_conv(const he_ctx* ctx, const he_conv_plan* p,
                  const uint64_t* d_c0, int B, const uint64_t* d_fspec,
                  const uint32_t* d_phi1, uint64_t* d_out, void* d_ws,
                  size_t ws_bytes, void* stream);

/* he_conv with the payload fused in and stage events.  d_out (full
 * output, as he_conv) and d_compact (uint64 [B][n_ob][L][n_valid], the
 * masked valid slots exactly as he_mask_extract would gather them from
 * d_out) are each nullable, not both.  If `events` is non-NULL it holds 4
 * cudaEvent_t handles, recorded on `stream` before K1 (forward NTT of c0),
 * before K3 (folded MAC), before K4 (inverse NTT + scatter + mask) and
 * after K4 (measurement). */
he_status he_conv_ex(const he_ctx* ctx, const he_conv_plan* p,
                     const uint64_t* d_c0, int B, const uint64_t* d_fspec,
                     const uint32_t* d_phi1, uint64_t* d_out,
                     uint64_t* d_compact, void* d_ws, size_t ws_bytes,
                     void* stream, void* const* events);

/* a7-a8 ("invalid slots ... do not need to be sent").
 * Gathers the n_valid valid slots of each output block, in increasing
 * coefficient order (row K < w_o, column L < h_o, channel n of the block:
 * i = s*(stride*K*h_p + stride*L) + t_n), from d_out uint64
 * [B][n_ob][L][N] into d_compact uint64 [B][n_ob][L][n_valid].  If d_phi1
 * is non-NULL the mask enc_j(phi1[b][ob][i]) is added to each gathered
 * slot (for outputs produced by he_conv without a mask). */
he_status he_mask_extract(const he_ctx* ctx, const he_conv_plan* p,
                          const uint64_t* d_out, int B,
                          const uint32_t* d_phi1, uint64_t* d_compact,
                          void* stream);

/* ------------------------------------------------ multi-image packing */
/* SURVEY §8(f) row 4b, reading R31, a protocol extension
 * beyond the paper (which keeps one image per ciphertext):
 * P images share one input ciphertext at offsets p*D,
 *   c(X) = sum_{p<P} X^{p D} i_p(X)  (mod X^N + 1),  i_p = Eq. (5) packing,
 * and he_conv on it (unchanged plan, filters and kernels) leaves image p's
 * conv outputs at p*D + the single-image valid slots.  D is the least
 * multiple of s with D > hi and D + lo > v_hi, where [lo, hi] holds the
 * exponents of i_p f (nonzero pixels, Eq. (6)-(7) filter) and [0, v_hi] the
 * valid slots; P = floor(N / D).  he_multi_image_spacing returns them
 * (HE_ESHAPE if P < 1). */
he_status he_multi_image_spacing(const he_ctx* ctx, const he_conv_plan* p,
                                 int32_t* D, int32_t* P);

/* a1 for multi-image ciphertexts: d_img int32 [B][c_i][w_i][h_i] (image
 * b = c*P + p goes to slot p of ciphertext c; a short last ciphertext has
 * zero images) -> d_pt uint64 [Bc][n_ib][L][N], Bc = ceil(B / P), enc_j of
 * c(X) (R2), plus the optional d_ve [Bc][n_ib][L][N] (v b + e0) as in
 * he_pack_input.  P and D must be he_multi_image_spacing's (or P smaller). */
he_status he_pack_input_multi(const he_ctx* ctx, const he_conv_plan* p,
                              const int32_t* d_img, int B, int P, int D,
                              const uint64_t* d_ve, uint64_t* d_pt, void* stream);

/* a7-a8 for multi-image ciphertexts: from d_out uint64 [Bc][n_ob][L][N]
 * (he_conv on he_pack_input_multi ciphertexts) gather, for p < P, image p's
 * valid slots p*D + i (i as he_mask_extract) into d_compact uint64
 * [Bc][n_ob][L][P n_valid] (image-major); + enc_j(phi1[c][ob][p*D + i]) if
 * d_phi1 uint32 [Bc][n_ob][N] is non-NULL. */
he_status he_mask_extract_multi(const he_ctx* ctx, const he_conv_plan* p,
                                const uint64_t* d_out, int Bc, int P, int D,
                                const uint32_t* d_phi1, uint64_t* d_compact,
                                void* stream);

/* -------------------------------------------------------------------- FC */
/* FC layer with n_i inputs, n_o outputs, any sizes.
 * When n_i n_o > N the weight matrix is decomposed into sub-matrices
 * (reading R27): input blocks of n_it = min(n_i, N) columns
 * (n_ib = ceil(n_i / n_it) input ciphertexts) and output tiles of
 * n_ot = min(n_o, floor(N / n_it)) rows (n_t = ceil(n_o / n_ot) products per
 * input block: Table III's ceil(n_o / floor(N / n_i)) when n_i <= N).
 * N up to 32768. */
typedef struct {
    int32_t n_i, n_o;
} he_fc_desc;

/* Eq. (9) per input block: block beta holds
 * I[beta n_it + l] at X^{l n_ot}, encoded with enc_j; d_in int32 [B][n_i] ->
 * d_pt uint64 [B][n_ib][L][N]; optional d_ve (same layout) as in
 * he_pack_input. */
he_status he_pack_fc_input(const he_ctx* ctx, const he_fc_desc* f,
                           const int32_t* d_in, int B, const uint64_t* d_ve,
                           uint64_t* d_pt, void* stream);

/* Server initialisation of Algorithm 2 (Lines 3-4):
 * per sub-matrix (beta, t) of n_ot x n_it (zero-padded), w(X) per Eq. (10)
 * generalised to N >= n_it n_ot (reading R17):
 *   w(X) = sum_k W_{k,0} X^k - sum_{l>=1} sum_k W_{k,l} X^{N - l n_ot + k},
 * d_W int32 [n_o][n_i]; stored NTT-domain (times N^{-1}, Shoup pairs) in
 * d_wspec [n_ib][n_t][L][N] (he_fc_wspec_bytes()).  d_bias int32 [n_o] (or
 * NULL = 0) is encoded into d_bias_enc uint64 [L][n_o].  d_ws:
 * he_fc_workspace_bytes(ctx, f, 1) bytes. */
size_t he_fc_wspec_bytes(const he_ctx* ctx, const he_fc_desc* f);
he_status he_pack_fc_weights(const he_ctx* ctx, const he_fc_desc* f,
                             const int32_t* d_W, const int32_t* d_bias,
                             uint64_t* d_wspec, uint64_t* d_bias_enc,
                             void* d_ws, size_t ws_bytes, void* stream);

/* a9, Algorithm 2 Line 13, first coefficients only
 * (PAPER.md:267), per output tile t:
 *   d_out[b][j][t n_ot + k] = (sum_beta c0_{b,beta} w_{beta,t})_k
 *                             + bias_enc[j][t n_ot + k] + enc_j(phi1[b][.]),
 * k < min(n_ot, n_o - t n_ot).  d_c0 uint64 [B][n_ib][L][N]; d_phi1 uint32
 * [B][n_o] or NULL; d_out uint64 [B][L][n_o]; d_ws:
 * he_fc_workspace_bytes(B) bytes. */
size_t he_fc_workspace_bytes(const he_ctx* ctx, const he_fc_desc* f, int B);
he_status he_fc(const he_ctx* ctx, const he_fc_desc* f, const uint64_t* d_c0,
                int B, const uint64_t* d_wspec, const uint64_t* d_bias_enc,
                const uint32_t* d_phi1, uint64_t* d_out, void* d_ws,
                size_t ws_bytes, void* stream);

/* he_fc with stage events: 3 cudaEvent_t (before the forward NTT, before
 * the pointwise-product + inverse-NTT kernel, after it) or NULL. */
he_status he_fc_ex(const he_ctx* ctx, const he_fc_desc* f,
                   const uint64_t* d_c0, int B, const uint64_t* d_wspec,
                   const uint64_t* d_bias_enc, const uint32_t* d_phi1,
                   uint64_t* d_out, void* d_ws, size_t ws_bytes, void* stream,
                   void* const* events);

/* ------------------------------------------------------------ wire format */
/* Residue wire format.  The paper counts ceil(log2 Q) bits per transmitted
 * coefficient (Table II); here every residue (< 2^50) is
 * bit-packed at 50 bits, little-endian: element i occupies bits
 * [50 i, 50 i + 50) of the byte stream.  n must be a multiple of 32 (the
 * stream is 50 n / 8 bytes, a multiple of 8); d_packed 8-byte aligned.
 * Used for c0 arriving at the server (Alg. 1 Line 10) and the payload
 * leaving it (Line 18).  Elements >= 2^50 give unspecified results. */
he_status he_residues_pack50(const uint64_t* d_in, size_t n, uint8_t* d_packed,
                             void* stream);
he_status he_residues_unpack50(const uint8_t* d_packed, size_t n,
                               uint64_t* d_out, void* stream);

/* Server-side mask phi1 ("two random polynomials ... are
 * generated"; reading R15): d_phi1[i] = SplitMix64(seed, i) mod t for
 * i < n, a counter-based stream (z = seed + (i + 1) 0x9E3779B97F4A7C15,
 * then the SplitMix64 finaliser), reproducible on any device and in the
 * oracle.  FOR REPRODUCIBLE TESTS AND BENCHMARKS ONLY: SplitMix64 is not a
 * cryptographic generator and a small or guessable seed makes phi1
 * predictable, and phi1 is what hides the server's conv output from the
 * client.  A deployment supplies phi1 from a keyed
 * cryptographic PRF (e.g. ChaCha20 or AES-CTR under a server secret) as the
 * caller-owned d_phi1 buffer of he_conv / he_fc. */
he_status he_phi1_generate(const he_ctx* ctx, uint64_t seed, size_t n,
                           uint32_t* d_phi1, void* stream);

/* ------------------------------------------------------------ transforms */
/* Batched negacyclic NTT over `batch` x L limbs stored [batch][L][N]
 * (the primitive behind a2, a3, a9; PAPER.md:28 cites NTT as the standard
 * polynomial-product speed-up).  In place.  Forward: canonical natural-
 * order coefficients in, canonical evaluations out in bit-reversed order:
 * out[p] = a(psi_j^{2 brv(p) + 1}).  Inverse: exactly undoes the forward
 * (bit-reversed in, natural out, includes N^{-1}). */
he_status he_ntt_forward(const he_ctx* ctx, uint64_t* d_data, int batch,
                         void* stream);
he_status he_ntt_inverse(const he_ctx* ctx, uint64_t* d_data, int batch,
                         void* stream);
/* The first log2(N) - skip stages of he_ntt_forward (the incomplete
 * transform the conv fold runs): block g of 2^skip
 * consecutive outputs holds the coefficients of a mod (X^{2^skip} - zeta_g),
 * zeta_g = psi^{brv(2^{logN-skip-1} + g/2)} for even g and its negative for
 * odd g (zeta = -1 when skip = log2 N).  In place, canonical. */
he_status he_ntt_forward_partial(const he_ctx* ctx, uint64_t* d_data, int batch,
                                 int skip, void* stream);

/* ----------------------------------------------- client mirror path (§8 f) */
/* Server initialisation, Alg. 1 Line 5:
 *   p_beta^{(n)} = fhat_beta^{(n)} a + e_f,
 * fhat the Eq. (7)-shifted filter polynomial of the same
 * weights he_pack_filters takes.  d_w int32 [c_o][c_i][f_w][f_h];
 * d_a uint64 [L][N] canonical residues of the public a; d_ef int32
 * [c_o][n_ib][N] signed noise e_f (NULL = 0); d_p uint64 [c_o][n_ib][L][N]
 * (output, canonical).  Full negacyclic products via NTT.  Workspace
 * he_server_p_workspace_bytes, caller-owned.  Errors: HE_EINVAL null
 * pointer, HE_ESHAPE foreign plan, HE_ENOMEM workspace too small. */
size_t he_server_p_workspace_bytes(const he_ctx* ctx, const he_conv_plan* plan);
he_status he_server_init_p(const he_ctx* ctx, const he_conv_plan* plan,
                           const int32_t* d_w, const uint64_t* d_a,
                           const int32_t* d_ef, uint64_t* d_p, void* d_ws,
                           size_t ws_bytes, void* stream);

/* Client side of Alg. 1 Lines 21-24: from the server's
 * p (layout of he_server_init_p) build, in he_pack_filters' layout, the
 * spectra of X^{-t_n} p_beta^{(n)}, so that
 *   he_conv(ctx, plan, d_vs, B, d_pspec, NULL, d_c1r, ...)
 * with d_vs[b][beta] = residues of v_beta s returns c1^r: the coefficients
 * s j + t_n of sum_beta v_beta s p_beta^{(n)} at exactly the slots of c0^r
 * (zeros elsewhere; d_compact gives the packed payload order).  d_pspec
 * needs he_filter_bytes; workspace he_pack_filters_workspace_bytes. */
he_status he_pack_client_p(const he_ctx* ctx, const he_conv_plan* plan,
                           const uint64_t* d_p, uint64_t* d_pspec, void* d_ws,
                           size_t ws_bytes, void* stream);

/* Signed small integers -> residues: d_out[i][j][k] = d_x[i][k] mod q_j.
 * d_x int32 [n_polys][N]; d_out uint64 [n_polys][L][N]. (encryption
 * randomness v, s, e of Alg. 1 as RNS polynomials) */
he_status he_residues_from_int(const he_ctx* ctx, const int32_t* d_x,
                               long n_polys, uint64_t* d_out, void* stream);

/* Negacyclic products in R_Q:
 *   d_out[b] = d_x[b] * d_y[y_batch == 1 ? 0 : b],  b < B,
 * all [.][L][N] canonical residues (d_out may alias d_x, not d_y).
 * Workspace: y_batch x L x N x 8 bytes (the spectra of y).  y_batch must be
 * 1 or B. */
he_status he_poly_mul(const he_ctx* ctx, const uint64_t* d_x,
                      const uint64_t* d_y, int B, int y_batch, uint64_t* d_out,
                      void* d_ws, size_t ws_bytes, void* stream);

/* Decryption rounding, Eq. (2) in the BFV reading (R1):
 *   m = round(t r / Q) mod t,  r = CRT(c0r + c1r)   (c1r NULL = 0),
 * per coefficient of n_polys polynomials of `len` coefficients, stored
 * [n_polys][L][len] (len = N for full rows, n_valid for the compact
 * payload).  Computed in RNS: sum_j floor/frac of y_j t / q_j with
 * y_j = r_j (Q/q_j)^{-1} mod q_j; the integer parts are exact and the
 * fractional parts are summed in FP64 (error < L 2^-52: a coefficient
 * decodes differently from the exact definition only if t r / Q lies within
 * that distance of a half-integer, which a valid ciphertext's noise bound
 * excludes).  d_m uint32 [n_polys][len]. */
he_status he_decrypt_round(const he_ctx* ctx, const uint64_t* d_c0r,
                           const uint64_t* d_c1r, long n_polys, long len,
                           uint32_t* d_m, void* stream);

/* Modulus switching before the wire (§8(f); the BFV counterpart of the
 * paper's rescale to Q', Table II's log Q' factor; reading
 * R28): each residue polynomial is mapped to Q' = q_0 ... q_{L_keep-1},
 *   x' = round(Q' x / Q) mod q_j,  j < L_keep,
 * x the canonical CRT value in [0, Q).  Applied to the server's payload
 * (c0^r) and, by the client, to its share c1^r; r' = c0' + c1' then
 * decrypts under Q' (he_decrypt_round on a context over the first L_keep
 * primes) while the wire carries L_keep / L of the bytes.  The division
 * by P = Q / Q' is exact in RNS except for the final rounding of
 * sum_i y_i / p_i, done in FP64 (differs from the exact definition only
 * within ~L 2^-52 of a half-integer).  d_in [n_polys][L][len], d_out
 * [n_polys][L_keep][len].  HE_EPARAM if more than 16 limbs are dropped or
 * L_keep (L - L_keep) + L > 400. */
he_status he_mod_switch(const he_ctx* ctx, const uint64_t* d_in, long n_polys,
                        long len, int L_keep, uint64_t* d_out, void* stream);

/* --------------------------------------- chained pipeline (§8(f), R29) */
/* Public-key mask of the c0-only encryption, Eq. (1):
 *   d_ve[i] = v_i b + e_i  in R_Q,  i < n_polys,
 * d_v, d_e int32 [n_polys][N] small signed (d_e NULL = 0), d_b uint64
 * [L][N] the public key; d_ve uint64 [n_polys][L][N], passed to
 * he_pack_input / he_pack_fc_input as d_ve.  Workspace L N 8 bytes. */
he_status he_pk_mask(const he_ctx* ctx, const int32_t* d_v, const int32_t* d_e,
                     long n_polys, const uint64_t* d_b, uint64_t* d_ve,
                     void* d_ws, size_t ws_bytes, void* stream);

/* Trusted stub of the garbled-circuit stage between layers (Fig. 5,
 * PAPER.md:270-281; reading R29, phi2 = 0): from the decrypted valid slots
 * d_m uint32 [B][n_ob][n_valid] (he_decrypt_round of the compact shares)
 *   x = centered((m - phi1) mod t),  y = min(qmax, max(x, 0) >> shift),
 * written as the next layer's image d_img int32 [B][c_o][w_o][h_o].
 * d_phi1 uint32 [B][n_ob][N] (the server's mask) or NULL. */
he_status he_relu_requant(const he_ctx* ctx, const he_conv_plan* plan,
                          const uint32_t* d_m, int B, const uint32_t* d_phi1,
                          int shift, int qmax, int32_t* d_img, void* stream);

/* Global average pooling before the FC (plain-20): d_out[r] =
 * floor(sum_{i < hw} d_x[r][i] / hw), d_x int32 [rows][hw]. */
he_status he_avgpool(const int32_t* d_x, long rows, int hw, int32_t* d_out,
                     void* stream);

/* FC client mirror path (Alg. 2 Lines 5-6, 16-17):
 * p_{beta,t} = w_{beta,t} a + e (sub-matrices as he_pack_fc_weights),
 * d_p uint64 [n_ib][n_t][L][N], d_e int32 [n_ib][n_t][N] or NULL; then
 * he_pack_fc_client_p stores the spectra of p in the d_wspec format, so
 * he_fc(ctx, f, d_vs, B, d_pspec, zero bias_enc, NULL, d_c1r, ...) with
 * d_vs[b][beta] = v_beta s returns the client share c1^r [B][L][n_o]. */
size_t he_fc_server_p_workspace_bytes(const he_ctx* ctx, const he_fc_desc* f);
he_status he_fc_server_init_p(const he_ctx* ctx, const he_fc_desc* f,
                              const int32_t* d_W, const uint64_t* d_a,
                              const int32_t* d_e, uint64_t* d_p, void* d_ws,
                              size_t ws_bytes, void* stream);
he_status he_pack_fc_client_p(const he_ctx* ctx, const he_fc_desc* f,
                              const uint64_t* d_p, uint64_t* d_pspec, void* d_ws,
                              size_t ws_bytes, void* stream);

/* FC output stub (R29): d_out[i] = centered((d_m[i] - d_phi1[i]) mod t),
 * int32; d_phi1 NULL = 0. */
he_status he_unmask(const he_ctx* ctx, const uint32_t* d_m, const uint32_t* d_phi1,
                    long n, int32_t* d_out, void* stream);

/* Sparse c0 upload (protocol extension): he_conv reads c0
 * only on the columns u < k_u of each fold group -- the coefficients
 * g s + u that some filter tap reaches -- so the client may send only those.
 * he_c0_compact gathers d_c0 [B][n_ib][L][N] into d_c0c [B][n_ib][L][M k_u]
 * (M = N / s, element g k_u + u); he_c0_expand scatters it back with zeros
 * elsewhere, and he_conv on the expanded c0 returns exactly the output of
 * the full c0.  plan: the he_conv_plan_make plan (its k_u). */
he_status he_c0_compact(const he_ctx* ctx, const he_conv_plan* plan,
                        const uint64_t* d_c0, int B, uint64_t* d_c0c, void* stream);
he_status he_c0_expand(const he_ctx* ctx, const he_conv_plan* plan,
                       const uint64_t* d_c0c, int B, uint64_t* d_c0, void* stream);

/* a2 debug export for parity: the coefficient-domain filter polynomials of
 * Eq. (6), f_beta^{(n)} (shifted = 0) or the Eq. (7)-shifted
 * fhat_beta^{(n)} = X^{t_n} f_beta^{(n)} (shifted = 1),
 * residues per limb, d_f uint64 [c_o][n_ib][L][N].  d_ws (c_o n_ib L N 8
 * bytes) is needed only when shifted.  Not on the hot path: he_pack_filters
 * stores the transformed operand instead. */
he_status he_filter_coeffs(const he_ctx* ctx, const he_conv_plan* plan,
                           const int32_t* d_w, int shifted, uint64_t* d_f, void* d_ws,
                           size_t ws_bytes, void* stream);

/* Unfolded reference path (ablation; SURVEY §8(a) "plain variant"): Alg. 1
 * Lines 14-17 computed literally -- full N-point NTT-domain products
 * sum_beta c0_beta f_beta^{(n)}, an N-point inverse per (b, n, l), then the
 * slots s j + t_n extracted and masked.  Output identical to he_conv's full
 * c0^r; costs the full transforms the fold avoids.  d_fplain uint64
 * [c_o][n_ib][L][N] from he_pack_filters_plain (plain NTT spectra). */
size_t he_conv_plain_workspace_bytes(const he_ctx* ctx, const he_conv_plan* plan, int B);
he_status he_pack_filters_plain(const he_ctx* ctx, const he_conv_plan* plan,
                                const int32_t* d_w, uint64_t* d_fplain, void* stream);
he_status he_conv_plain(const he_ctx* ctx, const he_conv_plan* plan, const uint64_t* d_c0,
                        int B, const uint64_t* d_fplain, const uint32_t* d_phi1,
                        uint64_t* d_out, void* d_ws, size_t ws_bytes, void* stream);

/* The client's per-layer randomness in one pass, sharing NTT(v):
 * d_ve[i] = v_i b + e_i (Eq. (1)) and d_vs[i] = v_i s (Alg. 1 Line 21),
 * d_s uint64 [L][N] the residues of the secret key.  Workspace 2 L N 8
 * bytes. */
he_status he_pk_mask_vs(const he_ctx* ctx, const int32_t* d_v, const int32_t* d_e,
                        long n_polys, const uint64_t* d_b, const uint64_t* d_s,
                        uint64_t* d_ve, uint64_t* d_vs, void* d_ws, size_t ws_bytes,
                        void* stream);

#ifdef __cplusplus
}
#endif
#endif /* HE_ROTFREE_H */
