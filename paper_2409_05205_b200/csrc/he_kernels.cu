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
#include <cuda.h>             // CUtensorMap (the TMA descriptors; encoded through the runtime entry point)

#include <string.h>

#include <algorithm>
#include <map>
#include <mutex>

#include "he_internal.cuh"

namespace cg = cooperative_groups;

#ifndef HE_MAC_OB
#define HE_MAC_OB 2          // fold groups per MAC output run (k_mac_imma)
#endif
#ifndef HE_K4_ROWS
#define HE_K4_ROWS 1         // K4: row-writer kernel k_intt_rows
#endif
#ifndef HE_NTT_T
#define HE_NTT_T 512         // forward NTT (cluster kernels): threads per CTA
#endif
#ifndef HE_NTT_MINB
#define HE_NTT_MINB 2        // forward NTT (cluster kernels): CTAs per SM (register cap)
#endif
#ifndef HE_NTT_UNR5
#define HE_NTT_UNR5 1        // s = 32 forward-NTT instance: pass loop unrolled too
#endif
#ifndef HE_NTT_NOCL
#define HE_NTT_NOCL 1        // conv-path forward NTT (N = 16384): no cluster barrier (out != in)
#endif
#ifndef HE_INV_RADIX
#define HE_INV_RADIX 3       // inverse cluster kernel: log2 of the pass radix
#endif
#ifndef HE_INV_FUSE
#define HE_INV_FUSE 1        // inverse cluster kernel: last stages in registers, fused with the store
#endif
#ifndef HE_INV_CL
#define HE_INV_CL 1          // full inverse NTT at N >= 16384: FP64 cluster kernel
#endif
#ifndef HE_FC_PRUNE
#define HE_FC_PRUNE 1        // FC inverse: pruned to the tile's output coefficients
#endif
#ifndef HE_MAC_TC_TMA
#define HE_MAC_TC_TMA 1      // tcgen05 MAC: operands staged by two TMA tensor copies
#endif
#ifndef HE_MAC_TMA16
#define HE_MAC_TMA16 1       // K = 16 mma.sync MAC instance: operands staged by TMA tensor copies
#endif
#ifndef HE_NTT_SPEC
#define HE_NTT_SPEC 1        // forward NTT: compile-time instances for plain-20 layers
#endif
#ifndef HE_TC_PWR
#define HE_TC_PWR 0       // tcgen05 MAC recombination with run-time power-of-two multipliers
#endif
#ifndef HE_K4_PF
#define HE_K4_PF 1        // K4 scatter writer: phi1 loads one batch ahead
#endif
#ifndef HE_NTT_UNR
#define HE_NTT_UNR 1      // s = 8 forward-NTT instances: pass loop unrolled (59.3 vs 60.1 us;
                          // the s = 32 instance measured slower, 34.1 vs 31.1 us)
#endif
#ifndef HE_FOLD_GN
#define HE_FOLD_GN 1      // s = 32 / s = 128 plain-20 layers: fold in [l][b][g][n] layout
#endif
#ifndef HE_FOLD_GN8
#define HE_FOLD_GN8 3     // s = 8 layers (scatter K4, cc = 2): fold [l][b][n/2][g][2] (3), [l][b][g][n] (1), off (0)
#endif
#ifndef HE_FOLD_GN5
#define HE_FOLD_GN5 1     // config 5 (tcgen05 MAC + row writer): fold in [l][b][g][n]
#endif
#ifndef HE_K4_SPEC
#define HE_K4_SPEC 1         // K4: compile-time instance for the plain-20 s = 8 layers
#endif
#ifndef HE_MAC_TB2_MAXNNT
#define HE_MAC_TB2_MAXNNT 4  // MAC: 32-image tiles when c_o <= 8 * this (else 16-image tiles)
#endif
#ifndef HE_MAC_CT16
#define HE_MAC_CT16 1        // MAC: 16-channel tiles for K = 16, c_o = 32 layers
#endif
#ifndef HE_MAC_KCMAX
#define HE_MAC_KCMAX 64      // MAC: largest k-chunk per staged unit when K does not fit
#endif
#ifndef HE_MAC_SPEC
#define HE_MAC_SPEC 1        // MAC: compile-time specialised instances for plain-20 shapes
#endif
#ifndef HE_MAC_DPE
#define HE_MAC_DPE 0         // K <= 16 MAC: outputs (of 4 per thread) reduced on the FP64 pipe
#endif
#ifndef HE_K4_MINW
#define HE_K4_MINW 2         // K4: minimum slot columns per channel chunk
#endif
#ifndef HE_K4_ROWS_MAXM
#define HE_K4_ROWS_MAXM 512  // K4: row-writer kernel for (N/s)-point transforms up to this
#endif
#ifndef HE_K4_ROWS_MINB
#define HE_K4_ROWS_MINB 4    // K4 row writer: CTAs per SM (register cap)
#endif
#ifndef HE_K4_W8
#define HE_K4_W8 1           // K4 s = 8 instances: unrolled writer with immediate offsets
#endif
#ifndef HE_K4_W8_EB
#define HE_K4_W8_EB 4        // K4 s = 8 writer: phi1 loads per batch (one batch ahead)
#endif
#ifndef HE_K4_RW
#define HE_K4_RW 1           // K4 row-writer instances: per-thread constant slot columns
#endif
#ifndef HE_K4_PRE
#define HE_K4_PRE 1          // K4 s = 8 writer: first phi1 batch loaded before the transform
#endif
#ifndef HE_K4_FUSE
#define HE_K4_FUSE 1         // K4 s = 8 instances: last radix-8 GS pass in the writer's registers
#endif
#ifndef HE_K4_FUSE_PU
#define HE_K4_FUSE_PU 1      // (its two radix-8 groups per thread: loop unroll factor)
#endif
#ifndef HE_K4_CC32
#define HE_K4_CC32 8         // K4 row writer, plain-20 s = 32 layers: channels per CTA
#endif
#ifndef HE_K4_CC128
#define HE_K4_CC128 32       // K4 row writer, plain-20 s = 128 layers: channels per CTA
#endif
// the array strides the host derives for those chunks (16/cc mod 16, or odd)
constexpr int k4_stride(int M, int cc) {
    int st = M + (M >> 4);
    while ((st & 15) != (cc < 16 ? (16 / cc) & 15 : 1) && !(cc >= 16 && (st & 1))) ++st;
    return st;
}
constexpr int K4_ST32 = k4_stride(512, HE_K4_CC32), K4_ST128 = k4_stride(128, HE_K4_CC128);
#ifndef HE_K4_WORDS
#define HE_K4_WORDS 6144     // K4: fold-array budget per CTA (words)
#endif

// The CUDA error behind the last HE_ECUDA returned on this host thread
// (he_last_cuda_error), so a caller can report what failed.
static thread_local cudaError_t g_last_cuda_error = cudaSuccess;
extern "C" const char* he_last_cuda_error(void) { return cudaGetErrorString(g_last_cuda_error); }

#define HE_CHECK_LAUNCH()                                   \
    do {                                                    \
        const cudaError_t e_ = cudaGetLastError();          \
        if (e_ != cudaSuccess) {                            \
            g_last_cuda_error = e_;                         \
            return HE_ECUDA;                                \
        }                                                   \
    } while (0)

static inline cudaStream_t STREAM(void* s) { return (cudaStream_t)s; }

// Raise a kernel's dynamic shared-memory limit.  The limit only ever grows
// (per device and kernel, under a mutex), so a launch from one host thread
// can never be undercut by another thread lowering it, and the
// attribute call is made once per size class instead of before every launch.
template <typename F>
static bool set_smem(F* f, size_t bytes) {
    if (bytes <= 48 * 1024) return true;
    static std::mutex mu;
    static std::map<std::pair<int, const void*>, size_t> cur;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> g(mu);
    size_t& have = cur[{dev, (const void*)f}];
    if (bytes <= have) return true;
    const cudaError_t e =
        cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e != cudaSuccess) {
        cudaGetLastError();
        g_last_cuda_error = e;
        return false;
    }
    have = bytes;
    return true;
}

static inline int ntt_threads(int NS) { return std::min(512, std::max(16, NS / 16)); }

// ===================================================================== K1
// Forward negacyclic NTT (natural in, bit-reversed out) of one limb by a
// cluster of 2^S CTAs (S = 0 for N <= 8192, 1 for 16384, 2 for 32768), so
// every CTA holds NS = N >> S <= 8192 words (69.6 KB of shared memory) and
// two 512-thread CTAs fit on an SM.  Each CTA reads the 2^S words
// x[i + r NS] of its output index i, applies the first S stages to them and
// keeps the value of its own segment; the remaining stages run in shared
// memory as radix-8 passes (ct_pass) with Shoup twiddles from L1/L2.  The
// cluster barrier after the loads makes in-place use safe.  16-byte
// coalesced global loads and stores.  OUT_FMT 0: canonical, 1: split25,
// 2: byte planes (int8 tensor-core MAC operand).
// MAC-tile layout of the forward spectra (OUT_FMT 2): byte j (j < 7) of the
// coefficient at position g s + u of limb (b, beta, l), g = gb Gt + gi, is
//   A[((((l (M/Gt) + gb) 7 + j) B + b) Gt + gi) Kp + beta s + u]   (bytes),
// with zeros in [K, Kp) of every row: a (plane, image) row holds Gt
// consecutive groups, so a limb writes runs of Gt*s bytes (n_ib = 1) and the
// int8 MAC stages each operand tile as contiguous blocks.
// cp.async helpers (Ampere-style async copies, used by several kernels)
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n"); }
template <int NW>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(NW)); }
template <int CHUNK>
__device__ __forceinline__ void cp_async_n(void* smem_dst, const void* gsrc, bool valid) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
    if (CHUNK == 16)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(gsrc),
                     "r"(valid ? 16 : 0));
    else
        asm volatile("cp.async.ca.shared.global [%0], [%1], %2, %3;\n" ::"r"(d), "l"(gsrc),
                     "n"(CHUNK), "r"(valid ? CHUNK : 0));
}

__device__ __forceinline__ bool mbar_try_wait(uint32_t bar, uint32_t phase) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}\n"
        : "=r"(ok) : "r"(bar), "r"(phase) : "memory");
    return ok != 0;
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_arrive_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes)
                 : "memory");
}

struct TileLay {
    int B, n_ib, logs, Kp, Gt;
    int skip;       // trailing stages not run: log2(s) for the fold (0 = full)
    int Ku;         // MAC-tile: columns u < Ku of each block are stored (k = beta Ku + u)
};
static inline int tile_gt(int M) { return M < 16 ? M : 16; }

// Store phase of the forward NTT: canonical values from `val(i)` (local
// index i of this CTA's segment) in format OUT_FMT.
template <int OUT_FMT, class F>
__device__ __forceinline__ void ntt_store(u64* out, int li, int seg, int NS, int N, int L,
                                          int l, const TileLay& T, F val) {
    if (OUT_FMT == 2) {
        unsigned char* A = reinterpret_cast<unsigned char*>(out);
        const int bb = qdiv(li, L), b = bb / T.n_ib, beta = bb - b * T.n_ib;
        const int s = 1 << T.logs, M = N >> T.logs, K = T.n_ib * T.Ku;
        const int lgt = __ffs(T.Gt) - 1;
        for (int i = 4 * threadIdx.x; i < NS; i += 4 * blockDim.x) {
            if (((seg * NS + i) & (s - 1)) >= T.Ku) continue;     // column unused by the MAC
            u64 x[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) x[e] = val(i + e);
            u32 pl[8];
            byte_transpose4((u32)x[0], (u32)x[1], (u32)x[2], (u32)x[3], pl[0], pl[1], pl[2],
                            pl[3]);
            byte_transpose4((u32)(x[0] >> 32), (u32)(x[1] >> 32), (u32)(x[2] >> 32),
                            (u32)(x[3] >> 32), pl[4], pl[5], pl[6], pl[7]);
            const int pos = seg * NS + i;
            const int g = pos >> T.logs, u = pos & (s - 1);
            const int gb = g >> lgt, gi = g & (T.Gt - 1);     // Gt is a power of two
            unsigned char* row =
                A + (((((size_t)l * (M / T.Gt) + gb) * 7) * T.B + b) * T.Gt + gi) * T.Kp +
                beta * T.Ku + u;
            const size_t pstride = (size_t)T.B * T.Gt * T.Kp;
            const bool tail = (beta == T.n_ib - 1) && (u + 4 == T.Ku) && (T.Kp > K);
#pragma unroll
            for (int j = 0; j < 7; ++j) {
                *reinterpret_cast<u32*>(row + j * pstride) = pl[j];
                if (tail)
                    for (int z = 4; z < T.Kp - K + 4; z += 4)
                        *reinterpret_cast<u32*>(row + j * pstride + z) = 0u;
            }
        }
        return;
    }
    u64* dst = out + (size_t)li * N + (size_t)seg * NS;
    for (int i = 2 * threadIdx.x; i < NS; i += 2 * blockDim.x) {
        u64 x = val(i), y = val(i + 1);
        if (OUT_FMT == 1) { x = to_split25(x); y = to_split25(y); }
        *reinterpret_cast<ulonglong2*>(dst + i) = make_ulonglong2(x, y);
    }
}

#ifndef HE_NTT_PF
#define HE_NTT_PF 1   // full forward transforms' register stage: input vectors in flight
#endif
#ifndef HE_NTT_PF_CONV
#define HE_NTT_PF_CONV 2   // conv path (2: 1.606 -> 1.585 ms once it dropped its cluster; 1 was faster with it)
#endif
// FP64 variant of ntt_fwd_segment (default; HE_NTT=int selects the integer
// one): residues as integer-valued doubles, exact FP64 butterflies
// (he_internal.cuh), twiddles psi^{brv(k)} as doubles.
template <int S, int OUT_FMT, int RM = 3, bool UNR = false>
__device__ __forceinline__ void ntt_fwd_segment_dp(const u64* in, u64* out, int logN, int L,
                                                   const he_limb* __restrict__ limbs,
                                                   const double* __restrict__ twd_all,
                                                   TileLay T) {
    extern __shared__ u64 sm_raw[];
    double* sm = reinterpret_cast<double*>(sm_raw);
    const int N = 1 << logN, NS = N >> S;
    const int li = blockIdx.x >> S, seg = blockIdx.x & ((1 << S) - 1);
    const int l = li - qdiv(li, L) * L;
    const double q = limbs[l].qd, qinv = limbs[l].qinvd;
    const double* tw = twd_all + (size_t)l * N;
    const u64* src = in + (size_t)li * N;
    const int end = logN - T.skip;
    // software-pipelined loads: the vectors of the next PF iterations are
    // in flight while this one's register stages run
    constexpr int PF = OUT_FMT == 2 ? HE_NTT_PF_CONV : HE_NTT_PF;
    const int step = 2 * blockDim.x;
    ulonglong2 buf[PF][1 << S];
#pragma unroll
    for (int p = 0; p < PF; ++p) {
        const int ip = 2 * threadIdx.x + p * step;
#pragma unroll
        for (int r = 0; r < (1 << S); ++r)
            if (ip < NS) buf[p][r] = *reinterpret_cast<const ulonglong2*>(src + ip + r * NS);
    }
    for (int i0 = 2 * threadIdx.x; i0 < NS; i0 += PF * step) {
#pragma unroll
        for (int p = 0; p < PF; ++p) {
            const int i = i0 + p * step;
            if (i >= NS) break;
            double vx[1 << S], vy[1 << S];
#pragma unroll
            for (int r = 0; r < (1 << S); ++r) {
                vx[r] = u2d(buf[p][r].x);
                vy[r] = u2d(buf[p][r].y);
            }
            const int in_ = i + PF * step;
#pragma unroll
            for (int r = 0; r < (1 << S); ++r)
                if (in_ < NS) buf[p][r] = *reinterpret_cast<const ulonglong2*>(src + in_ + r * NS);
#pragma unroll
            for (int st = 0; st < S; ++st) {
                if (st >= end) break;
                const int half = 1 << (S - 1 - st);
#pragma unroll
                for (int r = 0; r < (1 << S); ++r) {
                    if (r & half) continue;
                    const double w = __ldg(&tw[(1 << st) + (r >> (S - st))]);
                    // canonical inputs: stage st multiplicands < (1 + st) q < 4 q
                    ct_bfly_dp(vx[r], vx[r + half], w, q, qinv);
                    ct_bfly_dp(vy[r], vy[r + half], w, q, qinv);
                }
            }
            double ox = vx[0], oy = vy[0];
#pragma unroll
            for (int r = 1; r < (1 << S); ++r)
                if (r == seg) { ox = vx[r]; oy = vy[r]; }
            sm[PAD(i)] = ox;
            sm[PAD(i + 1)] = oy;
        }
    }
    // the cluster barrier keeps an in-place transform safe (a CTA must not
    // overwrite its segment before the partner has read it); the MAC-tile
    // output (OUT_FMT 2, he_conv_ex only) never aliases the input, so there
    // the CTAs need no cluster and synchronise only themselves
    if (S && !(OUT_FMT == 2 && HE_NTT_NOCL)) cg::this_cluster().sync();
    else __syncthreads();
    // (conv path: immediate-offset pass addressing, LIN; the full transforms
    //  keep the direct form, measured faster there)
    ct_all_dp<RM, OUT_FMT == 2, UNR, OUT_FMT == 2>(sm, logN, NS, seg, S, tw, q, qinv, end);
    ntt_store<OUT_FMT>(out, li, seg, NS, N, L, l, T,
                       [&](int i) {
                           return OUT_FMT == 2 ? d2lazy(sm[PAD(i)], q, qinv)
                                               : d2canon(sm[PAD(i)], q, qinv);
                       });
}

template <int S, int OUT_FMT>
__device__ __forceinline__ void ntt_fwd_segment(const u64* in, u64* out, int logN, int L,
                                                const he_limb* __restrict__ limbs,
                                                const ulonglong2* __restrict__ tw_all,
                                                TileLay T) {
    extern __shared__ u64 sm[];
    const int N = 1 << logN, NS = N >> S;
    const int li = blockIdx.x >> S, seg = blockIdx.x & ((1 << S) - 1);
    const int l = li % L;
    const u64 q = limbs[l].q, q2 = 2 * q;
    const ulonglong2* tw = tw_all + (size_t)l * N;
    const u64* src = in + (size_t)li * N;
    const int end = logN - T.skip;
    for (int i = 2 * threadIdx.x; i < NS; i += 2 * blockDim.x) {
        u64 vx[1 << S], vy[1 << S];
#pragma unroll
        for (int r = 0; r < (1 << S); ++r) {
            const ulonglong2 v = *reinterpret_cast<const ulonglong2*>(src + i + r * NS);
            vx[r] = v.x;
            vy[r] = v.y;
        }
#pragma unroll
        for (int st = 0; st < S; ++st) {
            if (st >= end) break;
            const int half = 1 << (S - 1 - st);
#pragma unroll
            for (int r = 0; r < (1 << S); ++r) {
                if (r & half) continue;
                const ulonglong2 w = __ldg(&tw[(1 << st) + (r >> (S - st))]);
                ct_bfly(vx[r], vx[r + half], w, q, q2);
                ct_bfly(vy[r], vy[r + half], w, q, q2);
            }
        }
        u64 ox = vx[0], oy = vy[0];
#pragma unroll
        for (int r = 1; r < (1 << S); ++r)
            if (r == seg) { ox = vx[r]; oy = vy[r]; }
        sm[PAD(i)] = ox;
        sm[PAD(i + 1)] = oy;
    }
    if (S) cg::this_cluster().sync();
    else __syncthreads();
    ct_all<3, true>(sm, logN, NS, seg, S, tw, q, q2, end); // lazy: values < 61 q
    const u64 one_p = limbs[l].one_p;
    ntt_store<OUT_FMT>(out, li, seg, NS, N, L, l, T,
                       [&](int i) { return reduce_full(sm[PAD(i)], q, one_p); });
}

template <int OUT_FMT>
__global__ void __launch_bounds__(512, 2)
k_ntt_fwd_s0(const u64* in, u64* out, int logN, int L, const he_limb* __restrict__ limbs,
             const ulonglong2* __restrict__ tw_all, TileLay T) {
    ntt_fwd_segment<0, OUT_FMT>(in, out, logN, L, limbs, tw_all, T);
}

template <int OUT_FMT>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(512, 2)
k_ntt_fwd_s1(const u64* in, u64* out, int logN, int L, const he_limb* __restrict__ limbs,
             const ulonglong2* __restrict__ tw_all, TileLay T) {
    ntt_fwd_segment<1, OUT_FMT>(in, out, logN, L, limbs, tw_all, T);
}

template <int OUT_FMT>
__global__ void __cluster_dims__(4, 1, 1) __launch_bounds__(512, 2)
k_ntt_fwd_s2(const u64* in, u64* out, int logN, int L, const he_limb* __restrict__ limbs,
             const ulonglong2* __restrict__ tw_all, TileLay T) {
    ntt_fwd_segment<2, OUT_FMT>(in, out, logN, L, limbs, tw_all, T);
}

template <int OUT_FMT>
__global__ void __launch_bounds__(HE_NTT_T, HE_NTT_MINB)
k_ntt_fwd_dp_s0(const u64* in, u64* out, int logN, int L, const he_limb* __restrict__ limbs,
                const double* __restrict__ tw_all, TileLay T) {
    ntt_fwd_segment_dp<0, OUT_FMT>(in, out, logN, L, limbs, tw_all, T);
}
// LN, SK, NIB, KU, KP, GT nonzero: log2 N, the skipped stages and the MAC-tile
// geometry fixed at compile time (the plain-20 conv layers' instances: the
// index arithmetic of the passes and of the byte-plane store folds away)
template <int OUT_FMT, int LN = 0, int SK = 0, int NIB = 0, int KU = 0, int KP = 0, int GT = 0>
__global__ void __cluster_dims__((OUT_FMT == 2 && HE_NTT_NOCL) ? 1 : 2, 1, 1)
    __launch_bounds__(HE_NTT_T, HE_NTT_MINB)
k_ntt_fwd_dp_s1(const u64* in, u64* out, int logN, int L, const he_limb* __restrict__ limbs,
                const double* __restrict__ tw_all, TileLay T) {
    if (LN) {
        T.logs = SK;
        T.skip = SK;
        T.n_ib = NIB;
        T.Ku = KU;
        T.Kp = KP;
        T.Gt = GT;
    }
    // conv path (MAC-tile output): radix-16 passes (measured 0.839 -> 0.826 ms per step)
    ntt_fwd_segment_dp<1, OUT_FMT, (OUT_FMT == 2 ? 4 : 3), (HE_NTT_UNR && LN != 0 && (SK == 3 || (HE_NTT_UNR5 && SK == 5)))>(
        in, out, LN ? LN : logN, L, limbs, tw_all, T);
}
template <int OUT_FMT>
__global__ void __cluster_dims__(4, 1, 1) __launch_bounds__(HE_NTT_T, HE_NTT_MINB)
k_ntt_fwd_dp_s2(const u64* in, u64* out, int logN, int L, const he_limb* __restrict__ limbs,
                const double* __restrict__ tw_all, TileLay T) {
    ntt_fwd_segment_dp<2, OUT_FMT>(in, out, logN, L, limbs, tw_all, T);
}
// Full transforms (canonical output: filter preparation, FC, client, the
// NTT limbs/s figure): radix-16 passes, 256 threads, 3 CTAs per SM.
__global__ void __launch_bounds__(256, 3)
k_ntt_fwd_dp16_s0(const u64* in, u64* out, int logN, int L, const he_limb* __restrict__ limbs,
                  const double* __restrict__ tw_all, TileLay T) {
    ntt_fwd_segment_dp<0, 0, 4>(in, out, logN, L, limbs, tw_all, T);
}
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(256, 3)
k_ntt_fwd_dp16_s1(const u64* in, u64* out, int logN, int L, const he_limb* __restrict__ limbs,
                  const double* __restrict__ tw_all, TileLay T) {
    ntt_fwd_segment_dp<1, 0, 4>(in, out, logN, L, limbs, tw_all, T);
}
__global__ void __cluster_dims__(4, 1, 1) __launch_bounds__(256, 3)
k_ntt_fwd_dp16_s2(const u64* in, u64* out, int logN, int L, const he_limb* __restrict__ limbs,
                  const double* __restrict__ tw_all, TileLay T) {
    ntt_fwd_segment_dp<2, 0, 4>(in, out, logN, L, limbs, tw_all, T);
}

// Column-tiled incomplete forward transform (FP64): CTA =
// (limb, C consecutive columns c0..c0+C-1 of the s = 2^skip columns), each
// column an M-point transform (M = N / s) held in shared memory at an odd
// word stride; coalesced row loads (C consecutive words per row k), and the
// store writes the same positions p = k s + c in format OUT_FMT.  No
// cluster, no read amplification: used when skip >= 2 (C >= 4).
// TNC, LCC, STC nonzero: log2 M, log2 C and the array stride at compile time
// (the M = 128, 32-column shape of config 4's s = 128 layers and config 5):
// the passes' strides become immediates (LIN addressing)
template <int OUT_FMT, int TNC = 0, int LCC = 0, int STC = 0>
__global__ void __launch_bounds__(256, 4)
k_ntt_fwd_cols(const u64* __restrict__ in, u64* __restrict__ out, int logN, int L,
               const he_limb* __restrict__ limbs, const double* __restrict__ twd_all, TileLay T,
               int logC_, int stride_, int nct) {
    extern __shared__ u64 sm_raw[];
    double* sm = reinterpret_cast<double*>(sm_raw);
    const int logC = LCC ? LCC : logC_, stride = STC ? STC : stride_;
    const int N = 1 << logN, logs = T.skip, s = 1 << logs, Tn = TNC ? TNC : logN - logs,
              M = 1 << Tn;
    const int C = 1 << logC;                 // nct column tiles of C columns per limb
    const int li = blockIdx.x / nct, c0 = (blockIdx.x - li * nct) << logC;
    const int l = li % L;
    const double q = limbs[l].qd, qinv = limbs[l].qinvd;
    const double* tw = twd_all + (size_t)l * N;
    const u64* src = in + (size_t)li * N + c0;
    const int tot = M << logC;
    // the whole tile in flight at once: 8-byte cp.async of the raw residues
    // into the padded column arrays; the first pass converts them
    for (int idx = threadIdx.x; idx < tot; idx += blockDim.x)
        cp_async_n<8>(sm_raw + (idx & (C - 1)) * stride + PAD(idx >> logC),
                      src + (size_t)(idx >> logC) * s + (idx & (C - 1)), true);
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
    if (Tn == 0) {                           // no stage: convert in place
        for (int idx = threadIdx.x; idx < tot; idx += blockDim.x) {
            const int a = (idx & (C - 1)) * stride + PAD(idx >> logC);
            sm[a] = u2d(sm_raw[a]);
        }
        __syncthreads();
    }
    ct_all_cols_dp<4, true, TNC != 0>(sm, stride, C, Tn, tw, q, qinv);
    if (OUT_FMT == 2) {
        unsigned char* A = reinterpret_cast<unsigned char*>(out);
        const int bb = li / L, beta = bb % T.n_ib, b = bb / T.n_ib;
        const int K = T.n_ib * T.Ku;
        const size_t pstride = (size_t)T.B * T.Gt * T.Kp;
        const int lgt = __ffs(T.Gt) - 1;
        const int nq = C >> 2;                                  // 4-column quads per row
        for (int e = threadIdx.x; e < (M * nq); e += blockDim.x) {
            const int k = e / nq, c = (e - k * nq) * 4;
            u64 x[4];
#pragma unroll
            for (int z = 0; z < 4; ++z) x[z] = d2lazy(sm[(c + z) * stride + PAD(k)], q, qinv);
            u32 pl[8];
            byte_transpose4((u32)x[0], (u32)x[1], (u32)x[2], (u32)x[3], pl[0], pl[1], pl[2], pl[3]);
            byte_transpose4((u32)(x[0] >> 32), (u32)(x[1] >> 32), (u32)(x[2] >> 32),
                            (u32)(x[3] >> 32), pl[4], pl[5], pl[6], pl[7]);
            const int g = k, u = c0 + c;
            if (u >= T.Ku) continue;                            // column unused by the MAC
            const int gb = g >> lgt, gi = g & (T.Gt - 1);     // Gt is a power of two
            unsigned char* row =
                A + (((((size_t)l * (M / T.Gt) + gb) * 7) * T.B + b) * T.Gt + gi) * T.Kp +
                beta * T.Ku + u;
            const bool tail = (beta == T.n_ib - 1) && (u + 4 == T.Ku) && (T.Kp > K);
#pragma unroll
            for (int j = 0; j < 7; ++j) {
                *reinterpret_cast<u32*>(row + j * pstride) = pl[j];
                if (tail)
                    for (int z = 4; z < T.Kp - K + 4; z += 4)
                        *reinterpret_cast<u32*>(row + j * pstride + z) = 0u;
            }
        }
    } else {
        u64* dst = out + (size_t)li * N + c0;
        for (int idx = threadIdx.x; idx < tot; idx += blockDim.x) {
            u64 v = d2canon(sm[(idx & (C - 1)) * stride + PAD(idx >> logC)], q, qinv);
            if (OUT_FMT == 1) v = to_split25(v);
            dst[(size_t)(idx >> logC) * s + (idx & (C - 1))] = v;
        }
    }
}

// columns per CTA and the odd-ish array stride for the column kernel
static void cols_geometry(int logN, int skip, int& logC, int& stride) {
    const int Tn = logN - skip, M = 1 << Tn;
    logC = std::max(2, std::min(skip, 12 - Tn));               // C M <= 4096 when possible
    const int C = 1 << logC;
    stride = padded_words(M);
    const int want = C < 16 ? (16 / C) & 15 : 1;                // 16/C (mod 16), or odd
    while ((stride & 15) != want && !(C >= 16 && (stride & 1))) ++stride;
}

// Launch the forward NTT over nlimbs = batch * L limbs.
static he_status launch_ntt_fwd(const he_ctx* c, const u64* in, u64* out,
                                long nlimbs, int out_fmt, cudaStream_t st,
                                TileLay T = TileLay{1, 1, 0, 16, 1, 0, 0}) {
    if (nlimbs <= 0) return HE_OK;
    const int logN = c->logN;
    const int S = logN <= 13 ? 0 : logN - 13;
    const int NS = c->N >> S;
    const int threads = std::min(512, std::max(32, NS / 16));
    const size_t smem = sizeof(u64) * padded_words(NS);
    typedef void (*kfn)(const u64*, u64*, int, int, const he_limb*, const ulonglong2*, TileLay);
    kfn k;
    static kfn const tab[3][3] = {
        {k_ntt_fwd_s0<0>, k_ntt_fwd_s0<1>, k_ntt_fwd_s0<2>},
        {k_ntt_fwd_s1<0>, k_ntt_fwd_s1<1>, k_ntt_fwd_s1<2>},
        {k_ntt_fwd_s2<0>, k_ntt_fwd_s2<1>, k_ntt_fwd_s2<2>}};
    // incomplete transform as independent column transforms, no cluster:
    // for s >= 256 (config 5: forward NTT 0.92 -> 0.73 ms) and whenever the
    // MAC uses at most half of the columns; otherwise the cluster kernels
    // measured as fast or faster (config 4).  HE_NTT_COLS=0/1 forces.
    // With the MAC-tile output only the Ku < s used columns are transformed.
    const bool cols_ok = c->ntt_mode == 0 && T.skip >= 2 && c->ntt_cluster != 1;
    const bool cols_pick = c->ntt_cluster == 2 || T.skip >= 8 ||
                           (out_fmt == 2 && T.skip >= 5 && 2 * T.Ku <= (1 << T.skip));
    if (cols_ok && cols_pick) {
        int logC, stride;
        cols_geometry(logN, T.skip, logC, stride);
        const size_t smem_c = sizeof(u64) * (size_t)(1 << logC) * stride;
        const int ncols = out_fmt == 2 ? T.Ku : (1 << T.skip);
        const int nct = (ncols + (1 << logC) - 1) >> logC;
        typedef void (*kfc)(const u64*, u64*, int, int, const he_limb*, const double*, TileLay,
                            int, int, int);
        static kfc const tabc[3] = {k_ntt_fwd_cols<0>, k_ntt_fwd_cols<1>, k_ntt_fwd_cols<2>};
        kfc kc = tabc[out_fmt];
        if (HE_NTT_SPEC && out_fmt == 2 && logN - T.skip == 7 && logC == 5 && stride == 137)
            kc = k_ntt_fwd_cols<2, 7, 5, 137>;
        if (!set_smem(kc, smem_c)) return HE_ECUDA;
        kc<<<(unsigned)(nlimbs * nct), 256, smem_c, st>>>(
            in, out, logN, c->L, c->d_limb, c->d_twd_fwd, T, logC, stride, nct);
        HE_CHECK_LAUNCH();
        return HE_OK;
    }
    if (c->ntt_mode == 0 && out_fmt == 0 && T.skip == 0 && !c->ntt_r8) {
        typedef void (*kfd)(const u64*, u64*, int, int, const he_limb*, const double*, TileLay);
        static kfd const tab16[3] = {k_ntt_fwd_dp16_s0, k_ntt_fwd_dp16_s1, k_ntt_fwd_dp16_s2};
        kfd kd = tab16[S];
        if (!set_smem(kd, smem)) return HE_ECUDA;
        kd<<<(unsigned)(nlimbs << S), std::min(threads, 256), smem, st>>>(
            in, out, logN, c->L, c->d_limb, c->d_twd_fwd, T);
        HE_CHECK_LAUNCH();
        return HE_OK;
    }
    if (c->ntt_mode == 0) {
        typedef void (*kfd)(const u64*, u64*, int, int, const he_limb*, const double*, TileLay);
        static kfd const tabd[3][3] = {
            {k_ntt_fwd_dp_s0<0>, k_ntt_fwd_dp_s0<1>, k_ntt_fwd_dp_s0<2>},
            {k_ntt_fwd_dp_s1<0>, k_ntt_fwd_dp_s1<1>, k_ntt_fwd_dp_s1<2>},
            {k_ntt_fwd_dp_s2<0>, k_ntt_fwd_dp_s2<1>, k_ntt_fwd_dp_s2<2>}};
        kfd kd = tabd[S][out_fmt];
        // compile-time instances for the plain-20 conv layers (N = 16384)
        if (HE_NTT_SPEC && S == 1 && out_fmt == 2 && logN == 14 && T.Gt == 16 &&
            T.logs == T.skip) {
            if (T.skip == 3 && T.n_ib == 2 && T.Ku == 8 && T.Kp == 16)
                kd = k_ntt_fwd_dp_s1<2, 14, 3, 2, 8, 16, 16>;
            else if (T.skip == 3 && T.n_ib == 1 && T.Ku == 4 && T.Kp == 16)
                kd = k_ntt_fwd_dp_s1<2, 14, 3, 1, 4, 16, 16>;
            else if (T.skip == 5 && T.n_ib == 1 && T.Ku == 32 && T.Kp == 32)
                kd = k_ntt_fwd_dp_s1<2, 14, 5, 1, 32, 32, 16>;
        }
        if (!set_smem(kd, smem)) return HE_ECUDA;
        kd<<<(unsigned)(nlimbs << S), std::min(threads, HE_NTT_T), smem, st>>>(in, out, logN, c->L, c->d_limb,
                                                           c->d_twd_fwd, T);
        HE_CHECK_LAUNCH();
        return HE_OK;
    }
    k = tab[S][out_fmt];
    if (!set_smem(k, smem)) return HE_ECUDA;
    k<<<(unsigned)(nlimbs << S), threads, smem, st>>>(in, out, logN, c->L, c->d_limb,
                                                      c->d_tw_fwd, T);
    HE_CHECK_LAUNCH();
    return HE_OK;
}

// ============================================================ inverse NTT
// Full N-point inverse (bit-reversed in, natural out, x N^{-1}).
template <bool DP>
__global__ void __launch_bounds__(1024)
k_ntt_inv(const u64* in, u64* out, int logN, int L, const he_limb* __restrict__ limbs,
          const ulonglong2* __restrict__ twi_all, const double* __restrict__ twid_all) {
    extern __shared__ u64 sm[];
    double* smd = reinterpret_cast<double*>(sm);
    const int N = 1 << logN;
    const int li = blockIdx.x, l = li % L;
    const he_limb& Lm = limbs[l];
    const u64 q = Lm.q, q2 = 2 * q;
    const u64* src = in + (size_t)li * N;
    for (int i = 2 * threadIdx.x; i < N; i += 2 * blockDim.x) {
        const ulonglong2 v = *reinterpret_cast<const ulonglong2*>(src + i);
        if (DP) {
            smd[PAD(i)] = u2d(v.x);
            smd[PAD(i + 1)] = u2d(v.y);
        } else {
            sm[PAD(i)] = v.x;
            sm[PAD(i + 1)] = v.y;
        }
    }
    __syncthreads();
    if (DP) gs_all_dp<3>(smd, 0, 1, logN, 0, logN, twid_all + (size_t)l * N, Lm.qd, Lm.qinvd);
    else gs_all<4>(sm, 0, 1, logN, 0, logN, twi_all + (size_t)l * N, q, q2);
    u64* dst = out + (size_t)li * N;
    const u64 ni = Lm.ninv, nip = Lm.ninv_p;
    const double nid = (double)Lm.ninv;
    for (int i = 2 * threadIdx.x; i < N; i += 2 * blockDim.x) {
        u64 x, y;
        if (DP) {
            x = d2canon(dp_mulmod(dp_reduce(smd[PAD(i)], Lm.qd, Lm.qinvd), nid, Lm.qd, Lm.qinvd),
                        Lm.qd, Lm.qinvd);
            y = d2canon(dp_mulmod(dp_reduce(smd[PAD(i + 1)], Lm.qd, Lm.qinvd), nid, Lm.qd,
                                  Lm.qinvd), Lm.qd, Lm.qinvd);
        } else {
            x = csub(shoup_mul(sm[PAD(i)], ni, nip, q), q);
            y = csub(shoup_mul(sm[PAD(i + 1)], ni, nip, q), q);
        }
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
    gs_all<4>(sm, 0, 1, logN - 1, seg, logN, twi, q, q2);
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

// FP64 inverse for N >= 2048 (N = 16384 / 32768: a cluster of 2^S CTAs per limb, the
// mirror of the forward cluster kernels): each CTA runs the first log2 N - S
// Gentleman-Sande stages on its own 8192-word segment in shared memory, then
// the S stages whose span crosses segments read the partner's segment over
// DSMEM (values in registers across the cluster barrier), then N^{-1} and the
// canonical store.  Replaces one 1024-thread CTA with 139 KB of shared memory
// (one per SM) at N = 16384 and the integer split kernel at N = 32768.
template <int S>
__global__ void __cluster_dims__(1 << S, 1, 1) __launch_bounds__(256, 3)
k_ntt_inv_dp_cl(const u64* __restrict__ in, u64* __restrict__ out, int logN, int L,
                const he_limb* __restrict__ limbs, const double* __restrict__ twid_all) {
    extern __shared__ u64 sm_raw[];
    double* sm = reinterpret_cast<double*>(sm_raw);
    const int N = 1 << logN, NS = N >> S;
    const int li = blockIdx.x >> S, seg = blockIdx.x & ((1 << S) - 1), l = li % L;
    const he_limb& Lm = limbs[l];
    const double q = Lm.qd, qi = Lm.qinvd;
    const double* tw = twid_all + (size_t)l * N;
    const u64* src = in + (size_t)li * N + (size_t)seg * NS;
    // the whole segment in flight by cp.async (raw canonical residues); the
    // first pass converts them (RAW)
    for (int i = threadIdx.x; i < NS; i += blockDim.x)
        cp_async_n<8>(sm_raw + PAD(i), src + i, true);
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
    cg::cluster_group cl = cg::this_cluster();
    const double nid = (double)Lm.ninv;
    if (HE_INV_FUSE) {
        // In-segment stages 0 .. logM - 2 as radix-8 passes in shared memory
        // (the same passes gs_all_dp runs), then one register step per index
        // i < NS/2 for the last in-segment stage (span NS/2) and the S
        // cross-segment stages: its 2^(S+1) elements i + h NS/2 of every
        // segment a are read (the partners' over DSMEM), transformed, scaled
        // by N^{-1} and stored to global memory directly -- no radix-2 pass,
        // no DSMEM writes, no separate store pass, one cluster barrier fewer.
        // The CTAs split the indices (no redundant work).  Same operations
        // in the same order as the unfused path.
        static_assert(HE_INV_RADIX == 3, "fused inverse: radix-8 passes");
        const int logM = logN - S, end = logM - 1;
        gs_pass_dp<3, true>(sm, 0, 1, logM, 0, seg, logN, tw, q, qi);
        __syncthreads();
        int lt = 3;
        for (; lt + 3 <= end; lt += 3) {
            gs_pass_dp<3>(sm, 0, 1, logM, lt, seg, logN, tw, q, qi);
            __syncthreads();
        }
        if (end - lt == 1) gs_pass_dp<1>(sm, 0, 1, logM, lt, seg, logN, tw, q, qi);
        else if (end - lt == 2) gs_pass_dp<2>(sm, 0, 1, logM, lt, seg, logN, tw, q, qi);
        if (S) cl.sync();
        else __syncthreads();
        constexpr int NSG = 1 << S;
        const int H = NS >> 1, per = H >> S;
        const double* sg[NSG];
        double wl[NSG];                      // stage logM - 1: block a of the N-point table
#pragma unroll
        for (int a = 0; a < NSG; ++a) {
            sg[a] = (a == seg) ? sm : cl.map_shared_rank(sm, a);
            wl[a] = __ldg(tw + NSG + a);
        }
        u64* dst = out + (size_t)li * N;
        for (int i = seg * per + threadIdx.x; i < (seg + 1) * per; i += blockDim.x) {
            double x[2 * NSG];
#pragma unroll
            for (int a = 0; a < NSG; ++a) {
#pragma unroll
                for (int h = 0; h < 2; ++h) x[2 * a + h] = dp_reduce(sg[a][PAD(i + h * H)], q, qi);
                const double X = x[2 * a], Y = x[2 * a + 1];
                x[2 * a] = X + Y;
                x[2 * a + 1] = dp_mulmod(X - Y, wl[a], q, qi);
            }
#pragma unroll
            for (int t = 0; t < S; ++t) {
#pragma unroll
                for (int a = 0; a < NSG; ++a) {
                    if (a & (1 << t)) continue;
                    const double w = __ldg(tw + (1 << (S - 1 - t)) + (a >> (t + 1)));
                    const double wn = t == S - 1 ? dp_mulmod(w, nid, q, qi) : w;
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        double& lo = x[2 * a + h];
                        double& hi = x[2 * (a + (1 << t)) + h];
                        const double X = dp_reduce(lo, q, qi), Y = dp_reduce(hi, q, qi);
                        lo = t == S - 1 ? dp_mulmod(X + Y, nid, q, qi) : X + Y;
                        hi = dp_mulmod(X - Y, wn, q, qi);
                    }
                }
            }
#pragma unroll
            for (int k = 0; k < 2 * NSG; ++k) {
                const double v = S ? x[k] : dp_mulmod(dp_reduce(x[k], q, qi), nid, q, qi);
                dst[(size_t)(k >> 1) * NS + (k & 1) * H + i] = d2canon(v, q, qi);
            }
        }
        if (S) cl.sync();                    // partners may still read this segment
        return;
    }
    gs_all_dp<HE_INV_RADIX, true>(sm, 0, 1, logN - S, seg, logN, tw, q, qi);   // in-segment stages
    for (int t = 0; t < S; ++t) {                                 // span NS << t
        // pair (lower segment a, upper segment a + 2^t): the lower CTA
        // takes indices i < NS/2, the upper one i >= NS/2, and each reads
        // both inputs and writes both outputs of its indices (one of them
        // over DSMEM), so no value is overwritten before its last read
        cl.sync();
        const int partner = seg ^ (1 << t);
        const bool upper = (seg >> t) & 1;
        const double w = tw[(1 << (S - 1 - t)) + (seg >> (t + 1))];
        double* lo = upper ? cl.map_shared_rank(sm, partner) : sm;
        double* hi = upper ? sm : cl.map_shared_rank(sm, partner);
        const int i0 = upper ? NS / 2 : 0;
        if (t == S - 1) {
            // last stage: N^{-1} rides on it -- X' = (X + Y) n^{-1},
            // Y' = (X - Y)(w n^{-1}) (|X +- Y| <= q + 4, |w n^{-1}| <= q keep
            // dp_mulmod's operand bound), so the store only canonicalises
            const double wn = dp_mulmod(w, nid, q, qi);
            for (int i = i0 + threadIdx.x; i < i0 + NS / 2; i += blockDim.x) {
                const double X = dp_reduce(lo[PAD(i)], q, qi), Y = dp_reduce(hi[PAD(i)], q, qi);
                lo[PAD(i)] = dp_mulmod(X + Y, nid, q, qi);
                hi[PAD(i)] = dp_mulmod(X - Y, wn, q, qi);
            }
        } else {
            for (int i = i0 + threadIdx.x; i < i0 + NS / 2; i += blockDim.x) {
                const double X = dp_reduce(lo[PAD(i)], q, qi), Y = dp_reduce(hi[PAD(i)], q, qi);
                lo[PAD(i)] = X + Y;
                hi[PAD(i)] = dp_mulmod(X - Y, w, q, qi);
            }
        }
    }
    if (S) cl.sync();
    u64* dst = out + (size_t)li * N + (size_t)seg * NS;
    for (int i = 2 * threadIdx.x; i < NS; i += 2 * blockDim.x) {
        // (S >= 1: already scaled and |.| <= q)
        const double a = S ? sm[PAD(i)] : dp_mulmod(dp_reduce(sm[PAD(i)], q, qi), nid, q, qi);
        const double b = S ? sm[PAD(i + 1)]
                           : dp_mulmod(dp_reduce(sm[PAD(i + 1)], q, qi), nid, q, qi);
        *reinterpret_cast<ulonglong2*>(dst + i) = make_ulonglong2(d2canon(a, q, qi),
                                                                  d2canon(b, q, qi));
    }
}

static he_status launch_ntt_inv(const he_ctx* c, const u64* in, u64* out,
                                long nlimbs, cudaStream_t st) {
    if (nlimbs <= 0) return HE_OK;
    const int N = c->N;
    if (c->ntt_mode == 0 && c->logN >= 11 && HE_INV_CL) {
        const int S = c->logN > 13 ? c->logN - 13 : 0;
        const size_t smem = sizeof(u64) * padded_words(N >> S);
        auto k = S == 0 ? k_ntt_inv_dp_cl<0> : (S == 1 ? k_ntt_inv_dp_cl<1> : k_ntt_inv_dp_cl<2>);
        if (!set_smem(k, smem)) return HE_ECUDA;
        k<<<(unsigned)(nlimbs << S), 256, smem, st>>>(in, out, c->logN, c->L, c->d_limb,
                                                     c->d_twd_inv);
        HE_CHECK_LAUNCH();
        return HE_OK;
    }
    if (c->logN <= 14) {
        const size_t smem = sizeof(u64) * padded_words(N);
        auto k = c->ntt_mode == 0 ? k_ntt_inv<true> : k_ntt_inv<false>;
        if (!set_smem(k, smem)) return HE_ECUDA;
        k<<<(unsigned)nlimbs, std::min(1024, std::max(32, N / 16)), smem, st>>>(
            in, out, c->logN, c->L, c->d_limb, c->d_tw_inv, c->d_twd_inv);
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

extern "C" he_status he_ntt_forward_partial(const he_ctx* c, uint64_t* d, int batch,
                                            int skip, void* stream) {
    if (!c || !d || batch < 0 || skip < 0 || skip > c->logN) return HE_EINVAL;
    return launch_ntt_fwd(c, (const u64*)d, (u64*)d, (long)batch * c->L, 0, STREAM(stream),
                          TileLay{1, 1, 0, 16, 1, skip, 0});
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
    int Ku;     // columns u < Ku of each fold group carry the MAC (K = n_ib Ku)
};

// Only the c_ib columns u < c_ib of each fold group meet nonzero filter
// operands (F'_{g,u} = 0 for u >= c_ib: the filter's exponents are
// -m mod s, m < c_ib), so the MAC runs over K = n_ib Ku with Ku = c_ib
// rounded up to a multiple of 4 (<= s), and the forward transform of c0 is
// needed on those columns only.


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
    d.Ku = p->k_u;
    return d;
}

static bool plan_ok(const he_ctx* c, const he_conv_plan* p) {
    he_conv_plan chk;
    if (he_conv_plan_make(c, &p->d, p->s, &chk) != HE_OK) return false;
    if (p->k_u != chk.k_u && p->k_u != p->s) return false;   // default or dense
    chk.k_u = p->k_u;
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

// Filter operand of the fold on the incomplete transform:
// after the first nst = log2(N/s) forward stages, group g (s contiguous
// words) of the filter holds f mod (X^s - zeta_g), and coefficient 0 of
// c f mod (X^s - zeta_g) is  sum_u c_{g,u} F'_{g,u}  with
//   F'_{g,u} = (N/s)^{-1} (u == 0 ? f_{g,0} : zeta_g f_{g,s-u}),
// zeta_g = +-psi^{brv(2^{nst-1} + g/2)} (the last stage's twiddle, - for
// odd g; -1 when nst = 0).  spec_l: this (n, beta, limb) row.
__device__ __forceinline__ u64 fold_filter_operand(const u64* __restrict__ spec_l, int g,
                                                   int u, int logs, int nst,
                                                   const he_limb& Lm,
                                                   const ulonglong2* __restrict__ tw_l) {
    const int s = 1 << logs;
    const u64 v = spec_l[((long)g << logs) + ((s - u) & (s - 1))];
    const double q = Lm.qd, qi = Lm.qinvd;
    u64 fac = d2canon(dp_mulmod(u2d(Lm.ninv), (double)s, q, qi), q, qi);   // (N/s)^{-1}
    if (u) {
        u64 z = Lm.q - 1;
        if (nst) {
            z = tw_l[(1 << (nst - 1)) + (g >> 1)].x;
            if (g & 1) z = Lm.q - z;
        }
        fac = d2canon(dp_mulmod(u2d(z), u2d(fac), q, qi), q, qi);
    }
    return d2canon(dp_mulmod(u2d(v), u2d(fac), q, qi), q, qi);
}

// incomplete spectra [c_o][n_ib][L][N] (canonical) -> MAC layout
// F[l][g][k][n] = split25(F'_{g,u} of (n, beta, l)), k = beta s + u.
__global__ void k_filter_to_mac(const u64* __restrict__ spec, u64* __restrict__ F,
                                PlanDev P, int L, int logN,
                                const he_limb* __restrict__ limbs,
                                const ulonglong2* __restrict__ tw_fwd) {
    const long N = 1L << logN;
    const int K = P.n_ib * P.Ku, M = (int)(N >> P.logs);
    const long total = (long)L * M * K * P.c_o;
    for (long idx = blockIdx.x * (long)blockDim.x + threadIdx.x; idx < total;
         idx += (long)gridDim.x * blockDim.x) {
        const int n = (int)(idx % P.c_o);
        long r = idx / P.c_o;
        const int k = (int)(r % K);
        r /= K;
        const int g = (int)(r % M);
        const int l = (int)(r / M);
        const int beta = k / P.Ku, u = k - beta * P.Ku;
        const he_limb& Lm = limbs[l];
        F[idx] = to_split25(fold_filter_operand(spec + (((long)n * P.n_ib + beta) * L + l) * N,
                                                g, u, P.logs, logN - P.logs, Lm,
                                                tw_fwd + (long)l * N));
    }
}

// Which MAC kernel a plan uses (deterministic; he_pack_filters and he_conv
// agree): the int8 tensor-core MAC for s >= 4 (its operand staging moves
// whole s-byte runs), else the IMAD MAC.  HE_MAC=imad forces the IMAD MAC.
static bool use_imma(const he_ctx* c, const PlanDev& P) {
    // (the tensor-core kernel holds all output channels of a group in one
    // CTA, one warp per 8: c_o <= 256; wider layers take the IMAD MAC)
    return c->mac_mode == 0 && P.s >= 4 && P.c_o <= 256;
}
static inline int imma_kp(int K) { return (K + 15) & ~15; }
static inline int imma_sw(int Kp) { return Kp / 4 + ((4 - Kp / 4) & 7); }   // = 4 mod 8
__device__ __forceinline__ int imma_sw_dev(int Kp) { return Kp / 4 + ((4 - Kp / 4) & 7); }

// spectra [c_o][n_ib][L][N] -> byte planes Fpl[l][g][7][c_o][Kp] of
// spec * N^{-1} (k = beta s + u < K; zero for K <= k < Kp).
__global__ void k_filter_to_imma(const u64* __restrict__ spec, unsigned char* __restrict__ F,
                                 PlanDev P, int L, int logN, int Kp,
                                 const he_limb* __restrict__ limbs,
                                 const ulonglong2* __restrict__ tw_fwd) {
    const long N = 1L << logN;
    const int K = P.n_ib * P.Ku, M = (int)(N >> P.logs);
    const long total = (long)L * M * P.c_o * Kp;
    for (long idx = blockIdx.x * (long)blockDim.x + threadIdx.x; idx < total;
         idx += (long)gridDim.x * blockDim.x) {
        const int k = (int)(idx % Kp);
        long r = idx / Kp;
        const int n = (int)(r % P.c_o);
        r /= P.c_o;
        const int g = (int)(r % M), l = (int)(r / M);
        u64 v = 0;
        if (k < K) {
            const he_limb& Lm = limbs[l];
            const int beta = k / P.Ku, u = k - beta * P.Ku;
            v = fold_filter_operand(spec + (((long)n * P.n_ib + beta) * L + l) * N, g, u,
                                    P.logs, logN - P.logs, Lm, tw_fwd + (long)l * N);
            // Montgomery form (x R mod q, R = 2^64) for the MAC's REDC (redc128)
            v = d2canon(dp_mulmod(u2d(v), u2d(Lm.r64), Lm.qd, Lm.qinvd), Lm.qd, Lm.qinvd);
        }
        unsigned char* dst = F + (((long)l * M + g) * 7 * P.c_o + n) * Kp + k;
#pragma unroll
        for (int j = 0; j < 7; ++j) dst[(long)j * P.c_o * Kp] = (unsigned char)(v >> (8 * j));
    }
}

extern "C" size_t he_filter_bytes(const he_ctx* c, const he_conv_plan* p) {
    if (!c || !p) return 0;
    const size_t M = c->N / p->s;
    const size_t K = (size_t)p->n_ib * p->k_u;
    const size_t split = sizeof(u64) * (size_t)p->d.c_o * c->L * M * K;
    const size_t planes = (size_t)c->L * M * 7 * p->d.c_o * imma_kp((int)K);
    return std::max(split, (planes + 15) & ~(size_t)15);
}

extern "C" size_t he_pack_filters_workspace_bytes(const he_ctx* c,
                                                  const he_conv_plan* p) {
    if (!c || !p) return 0;
    return sizeof(u64) * (size_t)p->d.c_o * p->n_ib * c->L * c->N;   // coefficient polys
}

static he_status finish_filter_spectra(const he_ctx* c, const PlanDev& P, u64* ws,
                                       uint64_t* d_fspec, cudaStream_t st);

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
    return finish_filter_spectra(c, P, ws, d_fspec, st);
}

// coefficient polynomials ws [c_o][n_ib][L][N] -> NTT (in place) -> the MAC
// layout of he_pack_filters (times N^{-1}).
static he_status finish_filter_spectra(const he_ctx* c, const PlanDev& P, u64* ws,
                                       uint64_t* d_fspec, cudaStream_t st) {
    // incomplete forward transform: the first log2(N/s) stages only
    he_status s = launch_ntt_fwd(c, ws, ws, (long)P.c_o * P.n_ib * c->L, 0, st,
                                 TileLay{1, 1, 0, 16, 1, P.logs, 0});
    if (s != HE_OK) return s;
    if (use_imma(c, P)) {
        const int Kp = imma_kp(P.n_ib * P.Ku);
        const long tot = (long)c->L * (c->N >> P.logs) * P.c_o * Kp;
        k_filter_to_imma<<<grid_for(tot, 256), 256, 0, st>>>(ws, (unsigned char*)d_fspec, P,
                                                              c->L, c->logN, Kp, c->d_limb,
                                                              c->d_tw_fwd);
    } else {
        const long totm = (long)c->L * (c->N >> P.logs) * P.n_ib * P.Ku * P.c_o;
        k_filter_to_mac<<<grid_for(totm, 256), 256, 0, st>>>(ws, (u64*)d_fspec, P, c->L,
                                                              c->logN, c->d_limb, c->d_tw_fwd);
    }
    HE_CHECK_LAUNCH();
    return HE_OK;
}

// ===================================================================== K3
// Folded NTT-domain MAC: for each (l, g), the modular GEMM
//   out[l][g][b][n] = sum_{k < K} C[b][beta][l][g s + u] * F[l][g][k][n] mod q
// (k = beta s + u, K = n_ib s).  Operands are split25 words v = hi 2^25 + lo,
// so each term is 4 IMAD.WIDE.U32 into three 64-bit accumulators (acc0:
// lo*lo, acc1: cross terms, acc2: hi*hi), reduced once per output.
// K <= 4096 keeps every accumulator below 2^63.
//
// CTA = 8 warps over GC consecutive groups g of one limb, a 32-image tile
// and a TNT-channel tile; warp (gl, nt) owns a 32 x 8 output tile of group
// gl, lane (ty, tx) = (lane / 4, lane % 4) the 4 x 2 outputs
// b = ty + 8 i, n = 8 nt + tx + 4 j.  C and F chunks of KC = 16 k-values
// are staged in shared memory ([k][row] layout: broadcast-free, conflict-free
// reads).
__device__ __forceinline__ u64 mac_reduce(u64 a0, u64 a1, u64 a2, const he_limb& Lm) {
    // V = a0 + a1 2^25 + a2 2^50 as a 128-bit (hi, lo), then
    // V mod q = (hi * (2^64 mod q) + lo) mod q via two Shoup products.
    const u64 q = Lm.q;
    u64 lo = a0 + (a1 << 25);
    u64 hi = (a1 >> 39) + (lo < a0);
    const u64 t = lo + (a2 << 50);
    hi += (a2 >> 14) + (t < lo);
    lo = t;
    u64 r = shoup_mul(hi, Lm.r64, Lm.r64_p, q) + shoup_mul(lo, 1, Lm.one_p, q);  // < 4q
    r = csub(r, 2 * q);
    return csub(r, q);
}

__device__ __forceinline__ void cp_async8(void* smem_dst, const void* gsrc, bool valid) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(d), "l"(gsrc),
                 "r"(valid ? 8 : 0));
}

template <int TNT>
struct MacTile {
    static constexpr int WPG = TNT / 8;   // warps per group
    static constexpr int GC = 8 / WPG;    // groups per CTA iteration
    static constexpr int KC = 16;         // k per chunk
    static constexpr int CW = KC + 1;     // padded sC row (conflict-free reads)
    static constexpr int C_WORDS = GC * 32 * CW;
    static constexpr int F_WORDS = GC * KC * TNT;
    static constexpr size_t SMEM = 2 * sizeof(u64) * (C_WORDS + F_WORDS);
};

template <int TNT>
__global__ void __launch_bounds__(256, 2)
k_mac_fold(const u64* __restrict__ C, const u64* __restrict__ F, u64* __restrict__ out,
           int B, int n_ib, int L, int logN, int logs, int c_o, int GI,
           const he_limb* __restrict__ limbs, int Ku) {
    typedef MacTile<TNT> T;
    constexpr int GC = T::GC, KC = T::KC, CW = T::CW, WPG = T::WPG;
    extern __shared__ u64 smem[];
    u64* sCb = smem;                       // [2][GC][32][CW]
    u64* sFb = smem + 2 * T::C_WORDS;      // [2][GC][KC][TNT]
    const int N = 1 << logN, M = N >> logs, K = n_ib * Ku;
    const int nG = (M + GC * GI - 1) / (GC * GI);
    const int l = blockIdx.x / nG, g0 = (blockIdx.x - l * nG) * GC * GI;
    const int b0 = blockIdx.y * 32, n0 = blockIdx.z * TNT;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int gl = warp / WPG, nt = warp - gl * WPG;
    const int ty = lane >> 2, tx = lane & 3;
    const int nK = (K + KC - 1) / KC, nchunks = GI * nK;

    auto issue = [&](int c, int buf) {
        const int it = c / nK, k0 = (c - it * nK) * KC;
        const int gb = g0 + it * GC;
        u64* sC = sCb + buf * T::C_WORDS;
        u64* sF = sFb + buf * T::F_WORDS;
        for (int e = threadIdx.x; e < GC * 32 * KC; e += 256) {
            const int kk = e & (KC - 1), r = e >> 4;
            const int gg = r & (GC - 1), bl = r / GC;
            const int k = k0 + kk, b = b0 + bl, gq = gb + gg;
            const bool ok = k < K && b < B && gq < M;
            const int beta = k / Ku;
            const u64* src = ok ? C + (((size_t)b * n_ib + beta) * L + l) * N +
                                      ((size_t)gq << logs) + (k - beta * Ku)
                                : C;
            cp_async8(sC + (gg * 32 + bl) * CW + kk, src, ok);
        }
        for (int e = threadIdx.x; e < GC * KC * TNT; e += 256) {
            const int nl = e & (TNT - 1), r = e / TNT;
            const int kk = r & (KC - 1), gg = r >> 4;
            const int k = k0 + kk, n = n0 + nl, gq = gb + gg;
            const bool ok = k < K && n < c_o && gq < M;
            const u64* src = ok ? F + (((size_t)l * M + gq) * K + k) * c_o + n : F;
            cp_async8(sF + (gg * KC + kk) * TNT + nl, src, ok);
        }
        cp_async_commit();
    };

    u64 a0[4][2], a1[4][2], a2[4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) a0[i][j] = a1[i][j] = a2[i][j] = 0;
    const he_limb Lm = limbs[l];
    issue(0, 0);
    for (int c = 0; c < nchunks; ++c) {
        if (c + 1 < nchunks) {
            issue(c + 1, (c + 1) & 1);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();
        const int it = c / nK, k0 = (c - it * nK) * KC;
        const int kc = min(KC, K - k0);
        const u64* sC = sCb + (c & 1) * T::C_WORDS + gl * 32 * CW;
        const u64* sF = sFb + (c & 1) * T::F_WORDS + gl * KC * TNT;
#pragma unroll 4
        for (int kk = 0; kk < kc; ++kk) {
            u32 c0[4], c1[4], f0[2], f1[2];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const u64 v = sC[(ty + 8 * i) * CW + kk];
                c0[i] = (u32)v;
                c1[i] = (u32)(v >> 32);
            }
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                const u64 v = sF[kk * TNT + nt * 8 + tx + 4 * j];
                f0[j] = (u32)v;
                f1[j] = (u32)(v >> 32);
            }
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 2; ++j) {
                    madw(a0[i][j], c0[i], f0[j]);
                    madw(a1[i][j], c0[i], f1[j]);
                    madw(a1[i][j], c1[i], f0[j]);
                    madw(a2[i][j], c1[i], f1[j]);
                }
        }
        if (k0 + KC >= K) {                      // last chunk of this iteration
            const int g = g0 + it * GC + gl;
            if (g < M) {
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < 2; ++j) {
                        const int b = b0 + ty + 8 * i, n = n0 + nt * 8 + tx + 4 * j;
                        if (b < B && n < c_o)
                            out[(((size_t)l * B + b) * c_o + n) * M + g] =
                                mac_reduce(a0[i][j], a1[i][j], a2[i][j], Lm);
                    }
            }
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 2; ++j) a0[i][j] = a1[i][j] = a2[i][j] = 0;
        }
        __syncthreads();
    }
}

template <int TNT>
static he_status launch_mac_t(const u64* C, const u64* F, u64* out, int B, int n_ib, int L,
                              int logN, int logs, int c_o, const he_limb* limbs,
                              cudaStream_t st, int Ku) {
    typedef MacTile<TNT> T;
    const int M = (1 << logN) >> logs;
    const int btiles = (B + 31) / 32, ntiles = (c_o + TNT - 1) / TNT;
    const long work = (long)L * ((M + T::GC - 1) / T::GC) * btiles * ntiles;
    int GI = (int)std::max(1L, std::min(16L, work / (148 * 8)));
    GI = std::min(GI, (M + T::GC - 1) / T::GC);
    const int nG = (M + T::GC * GI - 1) / (T::GC * GI);
    if (!set_smem(k_mac_fold<TNT>, T::SMEM)) return HE_ECUDA;
    dim3 grid(L * nG, btiles, ntiles);
    k_mac_fold<TNT><<<grid, 256, T::SMEM, st>>>(C, F, out, B, n_ib, L, logN, logs, c_o, GI,
                                                 limbs, Ku);
    return HE_OK;
}

static he_status launch_mac(const u64* C, const u64* F, u64* out, int B, int n_ib, int L,
                            int logN, int logs, int c_o, const he_limb* limbs,
                            cudaStream_t st, int Ku) {
    if (c_o <= 16) return launch_mac_t<16>(C, F, out, B, n_ib, L, logN, logs, c_o, limbs, st, Ku);
    if (c_o <= 32) return launch_mac_t<32>(C, F, out, B, n_ib, L, logN, logs, c_o, limbs, st, Ku);
    return launch_mac_t<64>(C, F, out, B, n_ib, L, logN, logs, c_o, limbs, st, Ku);
}

// ============================================================ K3 (int8)
// Folded MAC on the tensor cores, exact: with C = sum_i c_i 2^{8i} and
// F = sum_j f_j 2^{8j} (bytes, i, j < 7; C, F < q < 2^50),
//   sum_k C F = sum_{d=0}^{12} 2^{8d} S_d,   S_d = sum_{i+j=d} sum_k c_i f_j,
// so each (l, g) GEMM [B x K] x [K x c_o] becomes 49 u8 x u8 -> s32 MMAs
// (mma.sync m16n8k32 / m16n8k16) accumulated into 13 diagonal fragments
// (S_d < 7 K 255^2 < 2^31 for K <= 4096), then one modular recombination per
// output.  A operand: byte planes written by the forward NTT (OUT_FMT 2);
// B operand: byte planes packed by he_pack_filters.  One CTA per (l, g,
// 32-image tile); each warp owns 16 x 8 output tiles.
__device__ __forceinline__ void mma_k32(int (&d)[4], u32 a0, u32 a1, u32 a2, u32 a3, u32 b0,
                                        u32 b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
        "{%8,%9}, {%0,%1,%2,%3};"
        : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void mma_k16(int (&d)[4], u32 a0, u32 a1, u32 b0) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5}, {%6}, "
        "{%0,%1,%2,%3};"
        : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
        : "r"(a0), "r"(a1), "r"(b0));
}
// D = A B (zero accumulator input: the first product into a diagonal, so the
// 52 accumulator registers need no zeroing instructions)
__device__ __forceinline__ void mma_k32_z(int (&d)[4], u32 a0, u32 a1, u32 a2, u32 a3, u32 b0,
                                          u32 b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
        "{%8,%9}, {%10,%10,%10,%10};"
        : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1), "r"(0));
}
__device__ __forceinline__ void mma_k16_z(int (&d)[4], u32 a0, u32 a1, u32 b0) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5}, {%6}, "
        "{%7,%7,%7,%7};"
        : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3])
        : "r"(a0), "r"(a1), "r"(b0), "r"(0));
}

// Montgomery form of the recombination (R = 2^64): the filter operand of the
// int8 MAC paths is stored pre-multiplied by R mod q (k_filter_to_imma), so
// the exact 128-bit sum V = lo + hi 2^64 = R (C . F) needs one REDC instead
// of two Shoup products:  m = lo (-q^{-1}) mod 2^64,
//   t = (V + m q) / 2^64 = hi + hi64(m q) + (lo != 0)  =  C . F  (mod q),
// t < V / 2^64 + q < 2q because V < 1.5 K q^2 < q 2^64 (K <= 4096, q < 2^50).
struct Redc {
    u64 q, mq;      // q and -q^{-1} mod 2^64, held in registers by the MAC kernels
    const he_limb* L;   // FP64 constants (reduce13_mdp)
    u32 p8, p16, p24;   // 2^8, 2^16, 2^24 loaded at run time (HE_MAC_PWR)
};
__device__ __forceinline__ u64 redc128(u64 lo, u64 hi, Redc R, bool lazy) {
    const u64 m = lo * R.mq;
    const u64 t = hi + __umul64hi(m, R.q) + (lo != 0 ? 1ull : 0ull);
    return lazy ? t : csub(t, R.q);
}
// The same REDC done as two 32-bit word steps straight on the partial sums
// (no 128-bit (lo, hi) assembly, no 64 x 64-bit products): with q' = -q^{-1}
// mod 2^32 (the low word of R.mq) and V = P0 + P1 2^32 + P2 2^64 + P3 2^96,
//   m0 = lo32(P0) q' mod 2^32,  A = (V + m0 q) / 2^32
//      = hi32(P0) + P1 + m0 qhi + hi32(m0 qlo) + [lo32(P0) != 0]
// (lo32(P0) + lo32(m0 qlo) is 0 mod 2^32, so its carry is that test, taken
// from the carry flag of one mad.lo.cc), then the same step on A + P2 2^32 +
// P3 2^64.  Result (V + m q) / 2^64 with m < 2^64: congruent to V R^{-1} and
// below V / 2^64 + q < 2q (bound as redc128).  The running sums stay below
// 2^57 (P_k < 2^55, m qhi < 2^50).
#ifndef HE_MAC_GUNR
#define HE_MAC_GUNR 1       // MAC instances: the unit's group loop unrolled (compile-time GS)
#endif
#ifndef HE_MAC_PWR32
#define HE_MAC_PWR32 0      // K = 32 MAC: run-time power-of-two multipliers too
#endif
#ifndef HE_REDC_W
#define HE_REDC_W 1
#endif
__device__ __forceinline__ u64 redc_words(u64 P0, u64 P1, u64 P2, u32 P3, Redc R, bool lazy) {
    const u32 qlo = (u32)R.q, qhi = (u32)(R.q >> 32), qp = (u32)R.mq;
    u32 lo, hi;
    asm("{\n\t"
        ".reg .u32 m, x0, x1, d, p0l, p0h, p1l, p1h, p2l, p2h;\n\t"
        "mov.b64 {p0l, p0h}, %2;\n\t"
        "mov.b64 {p1l, p1h}, %3;\n\t"
        "mov.b64 {p2l, p2h}, %4;\n\t"
        "mul.lo.u32 m, p0l, %6;\n\t"
        "add.cc.u32 x0, p1l, p0h;\n\t"
        "addc.u32 x1, p1h, 0;\n\t"
        "mad.lo.cc.u32 x0, m, %8, x0;\n\t"
        "madc.hi.u32 x1, m, %8, x1;\n\t"
        "mad.lo.cc.u32 d, m, %7, p0l;\n\t"
        "madc.hi.cc.u32 x0, m, %7, x0;\n\t"
        "addc.u32 x1, x1, 0;\n\t"
        "mul.lo.u32 m, x0, %6;\n\t"
        "add.cc.u32 %0, p2l, x1;\n\t"
        "addc.u32 %1, p2h, %5;\n\t"
        "mad.lo.cc.u32 %0, m, %8, %0;\n\t"
        "madc.hi.u32 %1, m, %8, %1;\n\t"
        "mad.lo.cc.u32 d, m, %7, x0;\n\t"
        "madc.hi.cc.u32 %0, m, %7, %0;\n\t"
        "addc.u32 %1, %1, 0;\n\t"
        "}"
        : "=r"(lo), "=r"(hi)
        : "l"(P0), "l"(P1), "l"(P2), "r"(P3), "r"(qp), "r"(qlo), "r"(qhi));
    const u64 t = ((u64)hi << 32) | lo;
    return lazy ? t : csub(t, R.q);
}
// V = sum_{d<13} S_d 2^{8d} as (lo, hi): P_k = sum_{d=4k..4k+3} S_d 2^{8(d-4k)}
// (three mad.wide each, or the 32-bit pairs when S_d < 2^23, i.e. K <= 16),
// V = P0 + P1 2^32 + P2 2^64 + P3 2^96.
template <bool K16, bool PWR, class S>
__device__ __forceinline__ u64 reduce13_mont(S sd, Redc Lm, bool lazy) {
    u64 P[3];
    // PWR: the powers of two come from registers loaded at run time, so each
    // term is one IMAD.WIDE.U32 (an immediate power of two is rewritten by
    // ptxas into SHL + HI + two adds).  Measured per layer: K = 16 43.2 ->
    // 41.0 us, K = 64 33.3 -> 32.9 us, but K = 32 39.0 -> 41.0 us (kept off).
    const u32 c8 = PWR ? Lm.p8 : 1u << 8, c16 = PWR ? Lm.p16 : 1u << 16,
              c24 = PWR ? Lm.p24 : 1u << 24;
    // (no unroll pragma: the compiler's choice measured faster than forcing
    // it -- K = 16 MAC 41.0 vs 43.0 us -- and `unroll 1` puts P in local memory)
    for (int k = 0; k < 3; ++k) {
        if (K16) {
            const u32 a = (u32)sd(4 * k) + ((u32)sd(4 * k + 1) << 8);
            const u32 b = (u32)sd(4 * k + 2) + ((u32)sd(4 * k + 3) << 8);
            P[k] = a;
            madw(P[k], b, c16);
        } else {
            P[k] = (u64)(u32)sd(4 * k);
            madw(P[k], (u32)sd(4 * k + 1), c8);
            madw(P[k], (u32)sd(4 * k + 2), c16);
            madw(P[k], (u32)sd(4 * k + 3), c24);
        }
    }
#if HE_REDC_W
    return redc_words(P[0], P[1], P[2], (u32)sd(12), Lm, lazy);
#else
    const u64 P3 = (u64)(u32)sd(12);
    const u64 lo = P[0] + (P[1] << 32);
    const u64 hi = P[2] + (P[1] >> 32) + (P3 << 32) + (lo < P[0] ? 1 : 0);
    return redc128(lo, hi, Lm, lazy);
#endif
}

// The same Montgomery-domain result on the FP64 pipe (otherwise idle in the
// MAC): V 2^-64 = P0 2^-64 + P1 2^-32 + P2 + P3 2^32 (mod q).  For K <= 16
// the P_k are below 2^48 (exact doubles); three exact dp_mulmod by the
// centred constants, P2 added as is: |sum| < 2^48 + 3q, one dp_reduce and
// the lazy conversion give a residue in [q/2 - 2, 3q/2 + 2].
template <class S>
__device__ __forceinline__ u64 reduce13_mdp(S sd, Redc R, bool lazy) {
    u64 P[4];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const u32 a = (u32)sd(4 * k) + ((u32)sd(4 * k + 1) << 8);
        const u32 b = (u32)sd(4 * k + 2) + ((u32)sd(4 * k + 3) << 8);
        P[k] = a;
        madw(P[k], b, 1u << 16);
    }
    P[3] = (u64)(u32)sd(12);
    const double q = R.L->qd, qi = R.L->qinvd;
    double v = u2d(P[2]);
    v += dp_mulmod(u2d(P[0]), R.L->mrd[0], q, qi);
    v += dp_mulmod(u2d(P[1]), R.L->mrd[1], q, qi);
    v += dp_mulmod(u2d(P[3]), R.L->mrd[2], q, qi);
    return lazy ? d2lazy(v, q, qi) : d2canon(v, q, qi);
}

// x / d for 0 <= x < 2^31 with d fixed per kernel: a shift when d is a power
// of two, otherwise a plain division.
struct FastDiv {
    int d, sh;
    bool p2;
    __device__ __forceinline__ explicit FastDiv(int dd) : d(dd), sh(0),
                                                         p2((dd & (dd - 1)) == 0) {
#ifdef __CUDA_ARCH__
        sh = 31 - __clz(dd);
#else
        while ((1 << sh) < dd) ++sh;
#endif
    }
    __device__ __forceinline__ int div(int x) const { return p2 ? (x >> sh) : (x / d); }
};


// CTA = (limb l, G consecutive groups, 16*TB16-image tile); one warp per
// 16 x 8 output tile (bt, nt).  Work proceeds in "units" (GS groups x a
// KC-byte k-chunk): for small K a unit is all G groups with the whole K, for
// large K one group and a 64-byte k-chunk.  Each unit's A tile (7 planes x
// rows x KC bytes per group, MAC-tile layout) and F tile (7 x c_o x KC) are
// contiguous in global memory and are copied with 16-byte cp.async into
// padded shared rows (stride = 4 mod 8 words: conflict-free fragments).
// Reduced outputs go straight to the transposed fold out[l][b][n][g].
// Compile-time specialisations (KPC, KCC, COC, GSC nonzero: Kp, KC, c_o, GS
// fixed; LZ 1/0: lazy fixed, -1 runtime) turn the shared-memory strides into
// immediates (the generic form spends about a fifth of its instructions on
// address arithmetic); 0 / -1 keep the runtime arguments.
template <int TB16, int MINB = 1, int KPC = 0, int KCC = 0, int COC = 0, int GSC = 0, int LZ = -1,
          int FL = 0>
__global__ void __launch_bounds__(MINB > 1 ? 128 : 512, MINB)
k_mac_imma(const unsigned char* __restrict__ A, const unsigned char* __restrict__ Fpl,
           u64* __restrict__ out, int B, int L, int M, int c_o_, int Kp_, int G, int GS_,
           int KC_, int Gt, int nbuf, const he_limb* __restrict__ limbs, int lazy_,
           int c_full, int use_tma, const __grid_constant__ CUtensorMap tmA,
           const __grid_constant__ CUtensorMap tmF) {
    extern __shared__ __align__(1024) u32 sm32[];
    // K = 16 instance (config 4's s = 8 layers): with use_tma the unit's A tile
    // arrives by one 3-D TMA copy (64-byte rows, SWIZZLE_64B: the 16-byte
    // chunk of row r sits at chunk ^ ((r >> 1) & 3), conflict-free fragment
    // loads without padding) and its F tile by one 2-D copy, instead of
    // 10.5 cp.async (and their address arithmetic) per thread
    constexpr bool TK16 = HE_MAC_TMA16 && KPC == 16 && KCC == 16 && COC == 16 && GSC == 4 &&
                          TB16 == 2 && MINB == 5;
    const bool tma = TK16 && use_tma;
    constexpr int rows = 16 * TB16;
    // channel tile: channels [n0, n0 + c_o) of the c_full output channels
    // (blockIdx.z; c_o = c_full when the layer is not tiled)
    const int c_o = COC ? COC : c_o_, Kp = KPC ? KPC : Kp_;
    const int n0 = blockIdx.z * c_o;
    const int GS = GSC ? GSC : GS_, KC = KCC ? KCC : KC_;
    const bool lazy = LZ >= 0 ? (LZ == 1) : (lazy_ != 0);
    const int nrow = (c_o + 7) & ~7, nnt = nrow >> 3;
    const int swc = imma_sw_dev(KC);
    const int rw = tma ? (GS * KC) >> 2 : imma_sw_dev(GS * KC);   // A row: GS groups x KC bytes
    const int gb = 7 * nrow * swc;                        // B words per group
    const int buf_words = 7 * rows * rw + GS * gb;        // one staging buffer
    // M = N / s, G and Gt are powers of two: the block index splits by shifts
    // (a run-time division here cost ~25 instructions per thread)
    const int lgG = __ffs(G) - 1, lgN = max(__ffs(M) - 1 - lgG, 0);
    const int l = blockIdx.x >> lgN, g0 = (blockIdx.x & ((1 << lgN) - 1)) << lgG;
    const int b0 = blockIdx.y * rows;
    const int gcnt = min(G, M - g0);
    const int nkc = Kp / KC;
    const int nunits = ((gcnt + GS - 1) / GS) * nkc;      // (group block, k-chunk)
    // padded B rows (n >= c_o) stay zero for the whole kernel (every buffer)
    for (int bf = 0; bf < nbuf && nrow > c_o; ++bf) {
        u32* sB = sm32 + bf * buf_words + 7 * rows * rw;
        const int pad_rows = nrow > c_o ? nrow - c_o : 1;
        for (int e = threadIdx.x; e < GS * 7 * (nrow - c_o) * swc; e += blockDim.x) {
            const int w = e % swc, r = e / swc;
            const int n = c_o + r % pad_rows, gj = r / pad_rows;
            sB[(gj * nrow + n) * swc + w] = 0;
        }
    }
    // cp.async one unit into staging buffer `bf`
    auto issue = [&](int u, int bf) {
        const int uq = nkc == 1 ? u : u / nkc;
        const int gu = uq * GS, kc = u - uq * nkc;
        const int gsn = min(GS, gcnt - gu), k0 = kc * KC;
        u32* sA = sm32 + bf * buf_words;
        u32* sB = sA + 7 * rows * rw;
        {   // A: per (plane, image) the unit's gsn groups x KC bytes are contiguous
            const int lgt = __ffs(Gt) - 1;
            const int gbk = (g0 + gu) >> lgt, gi0 = (g0 + gu) & (Gt - 1);
            const int rcpr = (gsn * KC) >> 4;     // a power of two when KC is (gsn is)
            const int lrc = __ffs(rcpr) - 1;
            const FastDiv drc(rcpr);
            constexpr bool KCP2 = KCC > 0 && (KCC & (KCC - 1)) == 0;
            const int per = rows * rcpr;
            const size_t plane_stride = (size_t)B * Gt * Kp;
            const unsigned char* a0 = A + ((((size_t)l * (M / Gt) + gbk) * 7) * B + b0) * Gt * Kp +
                                      (size_t)gi0 * Kp + k0;
            for (int e = threadIdx.x; e < per; e += blockDim.x) {
                const int bl = KCP2 ? e >> lrc : drc.div(e), c = e - bl * rcpr;
                const bool ok = b0 + bl < B;
                // rows past the batch: zero-fill from a valid address (row 0)
                const unsigned char* src = a0 + (size_t)(ok ? bl : 0) * Gt * Kp + c * 16;
                unsigned char* dst = reinterpret_cast<unsigned char*>(sA + (size_t)bl * rw) + c * 16;
#pragma unroll
                for (int j = 0; j < 7; ++j)
                    cp_async_n<16>(dst + (size_t)j * rows * rw * 4, src + j * plane_stride, ok);
            }
        }
        {   // B: per (group, plane) a contiguous c_o x KC block
            const int cpr2 = KC >> 4;
            const FastDiv dc(cpr2), dn(c_o * cpr2);
            const int per = c_o * cpr2, total = gsn * per;
            const unsigned char* f0 =
                Fpl + ((((size_t)l * M + g0 + gu) * 7) * c_full + n0) * Kp + k0;
            for (int e = threadIdx.x; e < total; e += blockDim.x) {
                const int gi = dn.div(e), rem = e - gi * per;
                const int n = dc.div(rem), c = rem - n * cpr2;
                const unsigned char* src = f0 + ((size_t)gi * 7 * c_full + n) * Kp + c * 16;
                unsigned char* dst =
                    reinterpret_cast<unsigned char*>(sB + ((size_t)gi * 7 * nrow + n) * swc) + c * 16;
#pragma unroll
                for (int j = 0; j < 7; ++j)
                    cp_async_n<16>(dst + (size_t)j * nrow * swc * 4, src + (size_t)j * c_full * Kp,
                                   true);
            }
        }
        cp_async_commit();
    };

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int gq = lane >> 2, tq = lane & 3;
    const int bt = warp / nnt, nt = warp - bt * nnt;
    const Redc Lm = {limbs[l].q, limbs[l].mq, limbs + l, limbs[l].pw8[0], limbs[l].pw8[1],
                     limbs[l].pw8[2]};
    int acc[13][4];
    u64 ob[HE_MAC_OB][4];
    int nob = 0;
    if (tma) {
        __shared__ __align__(8) uint64_t s_tbar;
        const uint32_t tb = (uint32_t)__cvta_generic_to_shared(&s_tbar);
        if (threadIdx.x == 0) {
            mbar_init(tb, 1);
            asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            const int lgt = __ffs(Gt) - 1;
            const int gbk = g0 >> lgt, gi0 = g0 & (Gt - 1);
            mbar_arrive_tx(tb, (uint32_t)(7 * rows * GS * KC + GS * 7 * c_o * Kp));
            const uint32_t da = (uint32_t)__cvta_generic_to_shared(sm32);
            const uint32_t df = da + (uint32_t)(7 * rows * rw * 4);
            asm volatile(
                "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
                " [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(da),
                "l"(reinterpret_cast<uint64_t>(&tmA)), "r"(gi0 * Kp), "r"(b0),
                "r"((l * (M >> lgt) + gbk) * 7), "r"(tb)
                : "memory");
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
                " [%0], [%1, {%2, %3}], [%4];\n" ::"r"(df),
                "l"(reinterpret_cast<uint64_t>(&tmF)), "r"(n0 * Kp), "r"((l * M + g0) * 7),
                "r"(tb)
                : "memory");
        }
        while (!mbar_try_wait(tb, 0)) {
        }
    } else {
        issue(0, 0);
    }
    for (int u = 0; u < nunits; ++u) {
        if (nbuf == 2 && u + 1 < nunits) {                 // prefetch the next unit
            issue(u + 1, (u + 1) & 1);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();
        const int uq = nkc == 1 ? u : u / nkc;
        const int gu = uq * GS, kc = u - uq * nkc;
        const int gsn = min(GS, gcnt - gu);
        const u32* sA = sm32 + (nbuf == 2 ? (u & 1) : 0) * buf_words;
        const u32* sB = sA + 7 * rows * rw;
        // one fold group of the unit (a lambda so the full-unit case below can
        // run with a compile-time trip count: the HE_MAC_OB output shift
        // register then needs no register moves)
        auto group = [&](int gi) {
            // (TMA tile: 16-byte chunk gi of row bt 16 + gq at gi ^ (gq >> 1))
            const u32* ab = tma ? sA + (bt * 16 + gq) * rw + ((gi ^ (gq >> 1)) << 2) + tq
                                : sA + (bt * 16 + gq) * rw + gi * (KC >> 2) + tq;
            const u32* bb = sB + (size_t)gi * gb + (nt * 8 + gq) * swc + tq;
            const int Kw = KC >> 2;
            int kw = 0;
            // the first k-step of a group writes each diagonal's first product
            // with a zero accumulator input (diagonal d = i + j is first met at
            // i = 0, or at j = 6 for i >= 1 in this loop order)
            bool first = kc == 0;
            for (; kw + 8 <= Kw; kw += 8) {
                u32 bf0[7], bf1[7];
#pragma unroll
                for (int j = 0; j < 7; ++j) {
                    bf0[j] = bb[j * nrow * swc + kw];
                    bf1[j] = bb[j * nrow * swc + kw + 4];
                }
                if (first) {
#pragma unroll
                    for (int i = 0; i < 7; ++i) {
                        const u32* ap = ab + i * rows * rw + kw;
                        const u32 a0 = ap[0], a1 = ap[8 * rw], a2 = ap[4], a3 = ap[8 * rw + 4];
#pragma unroll
                        for (int j = 0; j < 7; ++j) {
                            if (i == 0 || j == 6) mma_k32_z(acc[i + j], a0, a1, a2, a3, bf0[j], bf1[j]);
                            else mma_k32(acc[i + j], a0, a1, a2, a3, bf0[j], bf1[j]);
                        }
                    }
                    first = false;
                } else {
#pragma unroll
                    for (int i = 0; i < 7; ++i) {
                        const u32* ap = ab + i * rows * rw + kw;
                        const u32 a0 = ap[0], a1 = ap[8 * rw], a2 = ap[4], a3 = ap[8 * rw + 4];
#pragma unroll
                        for (int j = 0; j < 7; ++j)
                            mma_k32(acc[i + j], a0, a1, a2, a3, bf0[j], bf1[j]);
                    }
                }
            }
            if (kw < Kw) {                                   // one k16 step
                // Two plane products of the same diagonal share one m16n8k32:
                // its K halves carry (c_i1, f_d-i1) and (c_i2, f_d-i2), so the
                // 49 k16 products take 28 k32 instructions (the k16 form
                // costs a k32 issue slot for half the work) and each
                // diagonal's dependency chain is at most 4 long.  Round r
                // issues the r-th pair of every diagonal (independent
                // accumulators back to back).
                u32 bf0[7], xa[7], xb[7];
#pragma unroll
                for (int j = 0; j < 7; ++j) bf0[j] = bb[j * nrow * swc + kw];
#pragma unroll
                for (int i = 0; i < 7; ++i) {
                    const u32* ap = ab + i * rows * rw + kw;
                    xa[i] = ap[0];
                    xb[i] = ap[8 * rw];
                }
#pragma unroll
                for (int r = 0; r < 4; ++r) {
#pragma unroll
                    for (int d = 0; d < 13; ++d) {
                        const int lo = d > 6 ? d - 6 : 0, hi = d < 6 ? d : 6;
                        const int i1 = lo + 2 * r, i2 = i1 + 1;
                        if (i1 > hi) continue;
                        if (i2 <= hi) {
                            if (first && r == 0)
                                mma_k32_z(acc[d], xa[i1], xb[i1], xa[i2], xb[i2], bf0[d - i1],
                                          bf0[d - i2]);
                            else
                                mma_k32(acc[d], xa[i1], xb[i1], xa[i2], xb[i2], bf0[d - i1],
                                        bf0[d - i2]);
                        } else {
                            if (first && r == 0) mma_k16_z(acc[d], xa[i1], xb[i1], bf0[d - i1]);
                            else mma_k16(acc[d], xa[i1], xb[i1], bf0[d - i1]);
                        }
                    }
                }
            }
            if (FL == 1 && kc == nkc - 1) {
                // fold layout [l][b][g][n] (FL = 1): the 4 outputs of a lane are
                // two channel pairs, each one 16-byte store; the 4 lanes of a
                // quad cover 8 consecutive channels (64 contiguous bytes)
                const int g = g0 + gu + gi;
                u64 v[4];
#pragma unroll
                for (int e = 0; e < 4; ++e)
                    v[e] = MINB > 1
                               ? reduce13_mont<true, true>([&](int d) { return acc[d][e]; }, Lm, lazy)
                               : reduce13_mont<false, (KPC != 32 || HE_MAC_PWR32)>([&](int d) { return acc[d][e]; },
                                                                 Lm, lazy);
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int b = b0 + bt * 16 + gq + 8 * h;
                    const int n = nt * 8 + 2 * tq;
                    if (b < B && n < c_o)
                        *reinterpret_cast<ulonglong2*>(
                            out + (((size_t)l * B + b) * M + g) * c_full + n0 + n) =
                            make_ulonglong2(v[2 * h], v[2 * h + 1]);
                }
            } else if (kc == nkc - 1) {
                // outputs of HE_MAC_OB consecutive groups are kept (shift
                // register ob, newest last) and leave as one run of HE_MAC_OB
                // words per (b, n) row of the fold, instead of 8-byte writes
                // scattered over 32 rows per warp instruction
                constexpr int OB = HE_MAC_OB;
                const int g = g0 + gu + gi;
#pragma unroll
                for (int e = 0; e < 4; ++e) {
#pragma unroll
                    for (int z = 0; z < OB - 1; ++z) ob[z][e] = ob[z + 1][e];
                    if (MINB > 1 && lazy && e >= 4 - HE_MAC_DPE)   // K <= 16: FP64 pipe share
                        ob[OB - 1][e] = reduce13_mdp([&](int d) { return acc[d][e]; }, Lm, lazy);
                    else
                        ob[OB - 1][e] =
                            MINB > 1 ? reduce13_mont<true, true>([&](int d) { return acc[d][e]; }, Lm, lazy)
                                     : reduce13_mont<false, (KPC != 32 || HE_MAC_PWR32)>([&](int d) { return acc[d][e]; },
                                                                       Lm, lazy);
                }
                ++nob;
                if (FL == 3 && (nob == OB || gu + gi == gcnt - 1)) {
                    // fold layout [l][b][n/2][g][2] (FL = 3): a lane's channel
                    // pair (2tq, 2tq + 1) over its OB = 2 groups is 32
                    // contiguous bytes
                    static_assert(FL != 3 || HE_MAC_OB == 2, "FL = 3 pairs groups");
                    const int gs0 = g - (OB - 1);
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int b = b0 + bt * 16 + gq + 8 * h;
                        const int n = nt * 8 + 2 * tq;
                        if (b >= B || n >= c_o) continue;
                        u64* pr = out + (((size_t)l * B + b) * (c_full >> 1) + ((n0 + n) >> 1)) *
                                            (2 * (size_t)M);
                        if (nob == OB && (gs0 & 1) == 0) {
                            ulonglong2* q2 = reinterpret_cast<ulonglong2*>(pr + 2 * gs0);
                            q2[0] = make_ulonglong2(ob[0][2 * h], ob[0][2 * h + 1]);
                            q2[1] = make_ulonglong2(ob[1][2 * h], ob[1][2 * h + 1]);
                        } else {
#pragma unroll
                            for (int z = 0; z < OB; ++z)
                                if (z >= OB - nob) {
                                    pr[2 * (gs0 + z)] = ob[z][2 * h];
                                    pr[2 * (gs0 + z) + 1] = ob[z][2 * h + 1];
                                }
                        }
                    }
                    nob = 0;
                }
                if (FL != 3 && (nob == OB || gu + gi == gcnt - 1)) {
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const int b = b0 + bt * 16 + gq + 8 * (e >> 1);
                        const int n = nt * 8 + 2 * tq + (e & 1);
                        if (b >= B || n >= c_o) continue;
                        u64* row = out + (((size_t)l * B + b) * c_full + n0 + n) * M + (g - (OB - 1));
                        if (nob == OB && ((g - (OB - 1)) & (OB - 1)) == 0) {
#pragma unroll
                            for (int z = 0; z < OB; z += 2)
                                reinterpret_cast<ulonglong2*>(row)[z / 2] =
                                    make_ulonglong2(ob[z][e], ob[z + 1][e]);
                        } else {
#pragma unroll
                            for (int z = 0; z < OB; ++z)
                                if (z >= OB - nob) row[z] = ob[z][e];
                        }
                    }
                    nob = 0;
                }
            }
        };
        if (GSC > 0 && HE_MAC_GUNR && gsn == GS) {
#pragma unroll
            for (int gi = 0; gi < (GSC > 0 ? GSC : 1); ++gi) group(gi);
        } else {
            for (int gi = 0; gi < gsn; ++gi) group(gi);
        }
        __syncthreads();                                   // buffer free for refill
    }
}

#ifndef HE_MAC_K16_MINB
#define HE_MAC_K16_MINB 5
#endif
#ifndef HE_MAC_UG
#define HE_MAC_UG 4
#endif
#ifndef HE_MAC_GMAX
#define HE_MAC_GMAX 16
#endif

// ------------------------------------------------------------------ K3 (tcgen05)
// Folded MAC on the 5th-generation tensor cores for batches of >= 128
// images (config 5): one CTA per (limb l, group g, 128-image tile).  The
// A operand is the 128 x K byte plane i of the image spectra, the B
// operand the c_o x K byte plane j of the filter operand, both staged in
// shared memory in the canonical K-major no-swizzle layout (8-row x
// 16-byte core matrices); D_{i+j} += A_i B_j^T accumulates each of the 13
// byte diagonals in its own TMEM region (M = 128 lanes = images, 16
// columns per 16-channel chunk: 13 x 16 = 208 of a 256-column allocation,
// two CTAs per SM).  One thread issues the 49 (x K/32) tcgen05.mma.kind::i8
// per chunk and commits them to an mbarrier; then every thread owns one
// image row (its TMEM lane) and recombines its outputs with reduce13_mont after
// tcgen05.ld -- the 13 partial sums of an output sit in one lane, so no
// cross-thread exchange is needed.
#ifndef HE_MAC_TC_BT
#define HE_MAC_TC_BT 128
#endif
__device__ __forceinline__ uint64_t tc_smem_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    // K-major, SWIZZLE_NONE: start >> 4 [0,14), LBO >> 4 [16,30), SBO >> 4
    // [32,46), version 1 [46,48), base offset 0, layout type 0 [61,64)
    return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}
__device__ __forceinline__ void tc_mma_i8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                          uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void tc_ld8(uint32_t taddr, int (&v)[8]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]),
                   "=r"(v[6]), "=r"(v[7])
                 : "r"(taddr));
}

// TMEM budget: 256 columns per CTA, and 128 registers x 256 threads cap the
// kernel at two CTAs per SM (512 columns, the whole TMEM), so an allocation
// never waits on another CTA of this kernel; no other kernel uses TMEM.
template <int FL = 0, bool TMA = false>
__global__ void __launch_bounds__(256, 2)
k_mac_tc(const unsigned char* __restrict__ A, const unsigned char* __restrict__ Fpl,
         u64* __restrict__ out, int B, int L, int M, int c_o, int Kp, int Gt,
         const he_limb* __restrict__ limbs, int lazy, const __grid_constant__ CUtensorMap tmA,
         const __grid_constant__ CUtensorMap tmB) {
    constexpr int BT = HE_MAC_TC_BT;           // images per CTA (= UMMA M)
    extern __shared__ __align__(1024) unsigned char smc[];
    const int Kt = (Kp + 31) & ~31;            // K rounded to the UMMA K step (32 bytes)
    const int kch = Kt >> 4;                   // 16-byte K chunks per row
    const int nrow = (c_o + 15) & ~15;         // B rows (channels), 16-column chunks
    const uint32_t sbo = (uint32_t)kch * 128;  // bytes between 8-row core-matrix groups
    const size_t a_plane = (size_t)BT * Kt, b_plane = (size_t)nrow * Kt;
    unsigned char* sA = smc;                   // [7][BT rows][Kt] canonical
    unsigned char* sB = smc + 7 * a_plane;     // [7][nrow][Kt] canonical
    __shared__ uint32_t s_tmem;
    __shared__ __align__(8) uint64_t s_bar;
    const int nGc = M;
    const int l = blockIdx.x / nGc, g = blockIdx.x - l * nGc;
    const int b0 = blockIdx.y * BT;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;\n" ::"r"(
            (uint32_t)__cvta_generic_to_shared(&s_tmem)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(
            (uint32_t)__cvta_generic_to_shared(&s_bar)));
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    // ---- stage the operands
    if (TMA) {
        // two TMA tensor copies (one elected thread): each 5-D box lands
        // directly in the canonical K-major core-matrix layout -- dims
        // (16 bytes of k, row mod 8, 16-byte k chunk, row / 8, plane) with the
        // row / 8 and plane strides of the global MAC-tile layouts, so the
        // box's dense order is (r & 7) 16 + c 128 + (r >> 3) SBO + j plane.
        // Out-of-range rows (ragged image tiles, channels past c_o) arrive as
        // zeros; completion is counted in bytes on an mbarrier.
        __shared__ __align__(8) uint64_t s_tbar;
        const uint32_t tb = (uint32_t)__cvta_generic_to_shared(&s_tbar);
        if (threadIdx.x == 0) {
            mbar_init(tb, 1);
            asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            const int gb = g / Gt, gi = g - gb * Gt;
            mbar_arrive_tx(tb, (uint32_t)(7 * (BT + nrow) * Kt));
            const uint32_t da = (uint32_t)__cvta_generic_to_shared(sA);
            const uint32_t db = (uint32_t)__cvta_generic_to_shared(sB);
            asm volatile(
                "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
                " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];\n" ::"r"(da),
                "l"(reinterpret_cast<uint64_t>(&tmA)), "r"(0), "r"(0), "r"(gi * (Kp >> 4)),
                "r"(b0 >> 3), "r"((l * (M / Gt) + gb) * 7), "r"(tb)
                : "memory");
            asm volatile(
                "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
                " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];\n" ::"r"(db),
                "l"(reinterpret_cast<uint64_t>(&tmB)), "r"(0), "r"(0), "r"(0), "r"(0),
                "r"((l * M + g) * 7), "r"(tb)
                : "memory");
        }
        while (!mbar_try_wait(tb, 0)) {
        }
    } else {   // 16-byte cp.async into the core-matrix layout
        const int gb = g / Gt, gi = g - gb * Gt;
        const size_t plane_stride = (size_t)B * Gt * Kp;
        const unsigned char* a0 = A + (((size_t)l * (M / Gt) + gb) * 7 * B) * Gt * Kp +
                                  (size_t)gi * Kp;
        const int cpr = Kt >> 4;                          // chunks per row
        // (index split without run-time division -- it was a quarter of the
        //  kernel's instructions -- and padding chunks zero-filled from a
        //  valid address instead of a pointer select)
        const FastDiv dcpr(cpr), dnrow(nrow);
        constexpr int LBT = __builtin_ctz(BT);
        for (int e = threadIdx.x; e < 7 * BT * cpr; e += blockDim.x) {
            const int q1 = dcpr.div(e), c = e - q1 * cpr;
            const int r = q1 & (BT - 1), j = q1 >> LBT;
            const int b = b0 + r;
            const bool ok = b < B && c * 16 < Kp;
            const unsigned char* src =
                a0 + j * plane_stride + (size_t)(ok ? b : b0) * Gt * Kp + (ok ? c * 16 : 0);
            unsigned char* dst = sA + j * a_plane + (r >> 3) * sbo + c * 128 + (r & 7) * 16;
            cp_async_n<16>(dst, src, ok);
        }
        const unsigned char* f0 = Fpl + (((size_t)l * M + g) * 7) * c_o * Kp;
        for (int e = threadIdx.x; e < 7 * nrow * cpr; e += blockDim.x) {
            const int q1 = dcpr.div(e), c = e - q1 * cpr;
            const int j = dnrow.div(q1), n = q1 - j * nrow;
            const bool ok = n < c_o && c * 16 < Kp;
            const unsigned char* src =
                f0 + ((size_t)j * c_o + (ok ? n : 0)) * Kp + (ok ? c * 16 : 0);
            unsigned char* dst = sB + j * b_plane + (n >> 3) * sbo + c * 128 + (n & 7) * 16;
            cp_async_n<16>(dst, src, ok);
        }
        cp_async_commit();
        cp_async_wait<0>();
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    const uint32_t tmem = s_tmem;
    const uint32_t bar = (uint32_t)__cvta_generic_to_shared(&s_bar);
    const uint32_t sA_addr = (uint32_t)__cvta_generic_to_shared(sA);
    const uint32_t sB_addr = (uint32_t)__cvta_generic_to_shared(sB);
    // instruction descriptor: S32 accumulate, u8 x u8, K-major A and B,
    // N = 16, M = BT
    const uint32_t idesc = (2u << 4) | ((16u >> 3) << 17) | ((uint32_t)(BT >> 4) << 24);
    const Redc Lm = {limbs[l].q, limbs[l].mq, limbs + l, limbs[l].pw8[0], limbs[l].pw8[1],
                     limbs[l].pw8[2]};
    const int quarter = warp & 3, half = warp >> 2;      // TMEM lane quarter, column half
    const int r = quarter * 32 + lane;                   // this thread's image row
    const int b = b0 + r;
    const int nchunks = nrow >> 4;
    // chunk ch's MMAs run while the threads recombine chunk ch - 1: once a
    // chunk's partial sums are in registers the TMEM region is reissued
    auto issue = [&](int ch) {
        for (int ks = 0; ks < (Kt >> 5); ++ks) {
#pragma unroll
            for (int i = 0; i < 7; ++i) {
                const uint64_t ad =
                    tc_smem_desc(sA_addr + i * (uint32_t)a_plane + ks * 256, 128, sbo);
#pragma unroll
                for (int j = 0; j < 7; ++j) {
                    const int d = i + j;
                    const uint64_t bd = tc_smem_desc(
                        sB_addr + j * (uint32_t)b_plane + (ch * 2) * sbo + ks * 256, 128, sbo);
                    // the first product into diagonal d overwrites it
                    const uint32_t acc = (ks > 0 || i > (d > 6 ? d - 6 : 0)) ? 1u : 0u;
                    tc_mma_i8(tmem + d * 16, ad, bd, idesc, acc);
                }
            }
        }
        asm volatile(
            "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                bar)
            : "memory");
    };
    if (threadIdx.x == 0) issue(0);
    for (int ch = 0; ch < nchunks; ++ch) {
        while (!mbar_try_wait(bar, (uint32_t)(ch & 1))) {
        }
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        // each thread: image row r, columns half*8 .. half*8+7 of the chunk
        int Sv[13][8];
#pragma unroll
        for (int d = 0; d < 13; ++d)
            tc_ld8(tmem + ((uint32_t)(quarter * 32) << 16) + d * 16 + half * 8, Sv[d]);
        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
        asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
        __syncthreads();                       // every lane read: TMEM free for chunk ch + 1
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        if (threadIdx.x == 0 && ch + 1 < nchunks) issue(ch + 1);
        if (FL == 1 && b < B && ch * 16 + half * 8 + 8 <= c_o) {
            // fold layout [l][b][g][n]: the thread's 8 channels are 64
            // contiguous bytes (four 16-byte stores, not eight rows)
            u64 v[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                int S[13];
#pragma unroll
                for (int d = 0; d < 13; ++d) S[d] = Sv[d][e];
                v[e] = reduce13_mont<false, HE_TC_PWR>([&](int d) { return S[d]; }, Lm, lazy);
            }
            ulonglong2* o2 = reinterpret_cast<ulonglong2*>(
                out + (((size_t)l * B + b) * M + g) * c_o + ch * 16 + half * 8);
#pragma unroll
            for (int e = 0; e < 8; e += 2) o2[e / 2] = make_ulonglong2(v[e], v[e + 1]);
        } else if (b < B) {
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                const int n = ch * 16 + half * 8 + e;
                if (n >= c_o) break;
                int S[13];
#pragma unroll
                for (int d = 0; d < 13; ++d) S[d] = Sv[d][e];
                const u64 v = reduce13_mont<false, HE_TC_PWR>([&](int d) { return S[d]; }, Lm, lazy);
                if (FL == 1) out[(((size_t)l * B + b) * M + g) * c_o + n] = v;
                else out[(((size_t)l * B + b) * c_o + n) * M + g] = v;
            }
        }
    }
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;\n" ::"r"(tmem));
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda)
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncodeTiledFn encode_tiled() {
    static EncodeTiledFn fn = [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) !=
                cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            f = nullptr;
        return reinterpret_cast<EncodeTiledFn>(f);
    }();
    return fn;
}
static he_status launch_mac_tc(const unsigned char* A, const unsigned char* Fpl, u64* out, int B,
                               int L, int M, int c_o, int Kp, const he_limb* limbs,
                               cudaStream_t st, int lazy, int fl = 0) {
    const int Kt = (Kp + 31) & ~31, nrow = (c_o + 15) & ~15;
    const size_t smem = 7 * ((size_t)HE_MAC_TC_BT * Kt + (size_t)nrow * Kt);
    if (smem > 110 * 1024) return HE_ESHAPE;
    auto k = fl == 1 ? k_mac_tc<1> : k_mac_tc<0>;
    const int Gt = tile_gt(M);
    CUtensorMap tmA, tmB;
    memset(&tmA, 0, sizeof tmA);
    memset(&tmB, 0, sizeof tmB);
    // TMA staging when the boxes tile the operands exactly: whole 32-byte K
    // steps (Kt = Kp), image and channel counts in rows of 8
    if (HE_MAC_TC_TMA && Kt == Kp && B % 8 == 0 && c_o % 8 == 0 && encode_tiled() != nullptr) {
        const cuuint32_t kch = (cuuint32_t)(Kt >> 4), one[5] = {1, 1, 1, 1, 1};
        const cuuint64_t gA[5] = {16, 8, (cuuint64_t)Gt * Kp / 16, (cuuint64_t)B / 8,
                                  (cuuint64_t)L * (M / Gt) * 7};
        const cuuint64_t sAst[4] = {(cuuint64_t)Gt * Kp, 16, (cuuint64_t)8 * Gt * Kp,
                                    (cuuint64_t)B * Gt * Kp};
        const cuuint32_t bA[5] = {16, 8, kch, HE_MAC_TC_BT / 8, 7};
        const cuuint64_t gB[5] = {16, 8, (cuuint64_t)Kp / 16, (cuuint64_t)c_o / 8,
                                  (cuuint64_t)L * M * 7};
        const cuuint64_t sBst[4] = {(cuuint64_t)Kp, 16, (cuuint64_t)8 * Kp, (cuuint64_t)c_o * Kp};
        const cuuint32_t bB[5] = {16, 8, kch, (cuuint32_t)nrow / 8, 7};
        auto enc = encode_tiled();
        const bool ok =
            enc(&tmA, CU_TENSOR_MAP_DATA_TYPE_UINT8, 5, (void*)A, gA, sAst, bA, one,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
                CUDA_SUCCESS &&
            enc(&tmB, CU_TENSOR_MAP_DATA_TYPE_UINT8, 5, (void*)Fpl, gB, sBst, bB, one,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
                CUDA_SUCCESS;
        if (ok) k = fl == 1 ? k_mac_tc<1, true> : k_mac_tc<0, true>;
    }
    if (!set_smem(k, smem)) return HE_ECUDA;
    dim3 grid(L * M, (B + HE_MAC_TC_BT - 1) / HE_MAC_TC_BT);
    k<<<grid, 256, smem, st>>>(A, Fpl, out, B, L, M, c_o, Kp, Gt, limbs, lazy, tmA, tmB);
    return HE_OK;
}

// lazy: outputs in [0, 4q) instead of canonical (the FP64 inverse in K4
// reduces its raw inputs anyway)
static he_status launch_mac_imma(const unsigned char* A, const unsigned char* Fpl, u64* out,
                                 int B, int n_ib, int L, int logN, int logs, int c_o,
                                 const he_limb* limbs, cudaStream_t st, int Ku, int lazy,
                                 int mac_tc, int fl_req = 0, int* fl_used = nullptr) {
    if (fl_used) *fl_used = 0;
    const int M = (1 << logN) >> logs, K = n_ib * Ku;
    const int Kp = imma_kp(K);
    if (c_o > 256) return HE_ESHAPE;
    {
        // batches of >= 128 images: tcgen05 MAC (HE_MAC_TC=0 disables, =1 forces)
        const int mode = mac_tc;
        const int Kt = (Kp + 31) & ~31, nr16 = (c_o + 15) & ~15;
        const bool fits = 7 * ((size_t)HE_MAC_TC_BT * Kt + (size_t)nr16 * Kt) <= 110 * 1024;
        if (fits && (mode == 1 || (mode == 2 && B >= HE_MAC_TC_BT))) {
            // ([l][b][g][n] fold when the caller's K4 instance reads it)
            const int fl = fl_req == 4 ? 1 : 0;
            if (fl_used) *fl_used = fl ? 4 : 0;
            return launch_mac_tc(A, Fpl, out, B, L, M, c_o, Kp, limbs, st, lazy, fl);
        }
    }
    const int c_full = c_o;
    // K = 16 layers with 32 channels: two 16-channel tiles (grid.z) of the
    // small-CTA form (5 CTAs per SM) instead of one 8-warp CTA
    const int ctile = (HE_MAC_CT16 && Kp == 16 && c_o == 32 && B >= 32) ? 16 : c_o;
    const int nct = c_full / ctile;
    c_o = ctile;
    const int nrow = (c_o + 7) & ~7, nnt = nrow / 8;
    const int Gt = tile_gt(M);
    // per staging buffer; the K = 16 small-CTA case targets 5 CTAs per SM
    const bool k16c = Kp == 16 && HE_MAC_K16_MINB > 1;
    const size_t budget = k16c ? 227 * 1024 / HE_MAC_K16_MINB - 1024 : 48 * 1024;
    auto unit_bytes = [&](int rows, int gs, int kc) {
        return sizeof(u32) * 7 * ((size_t)rows * imma_sw(gs * kc) + (size_t)gs * nrow * imma_sw(kc));
    };
    // 32-image tiles for small c_o; 16-image tiles (<= 256 threads, two
    // CTAs per SM) when the whole K does not fit one buffer
    int TB16 = (nnt <= HE_MAC_TB2_MAXNNT && B > 16) ? 2 : 1;
    if (TB16 == 2 && unit_bytes(32, 1, Kp) > budget) TB16 = 1;
    const int rows = 16 * TB16, warps = TB16 * nnt;
    int KC = Kp, GS = 1, G = 1;
    if (unit_bytes(rows, 1, Kp) <= budget) {
        GS = 1;
        while (GS < Gt && GS < HE_MAC_GMAX && unit_bytes(rows, GS * 2, Kp) <= budget) GS *= 2;
        G = GS;
        // CTAs of > 4 warps (not the 5-per-SM small-K variant): walk several
        // units through the double buffer so loads overlap the MMAs and the
        // per-CTA setup is amortised, keeping >= ~3 CTAs of work per SM
        if (!k16c && Kp >= 32) {
            const long ctas1 = (long)L * ((M + GS - 1) / GS) * ((B + rows - 1) / rows);
            int ug = 1;
            while (ug < HE_MAC_UG && G * 2 <= Gt * 4 && ctas1 / (ug * 2) >= 3 * 148 &&
                   2 * unit_bytes(rows, GS, Kp) <= 227 * 1024)
                ug *= 2;
            G = GS * ug;
        }
    } else {
        KC = (Kp % 64 == 0 && HE_MAC_KCMAX >= 64) ? 64 : ((Kp % 32 == 0) ? 32 : 16);
        GS = 1;
        // several groups per CTA so the k-chunk pipeline has depth, while
        // keeping >= ~4 CTAs of work per SM
        const long ctas1 = (long)L * M * ((B + rows - 1) / rows);
        G = 1;
        while (G < Gt && ctas1 / (G * 2) >= 4 * 148) G *= 2;
    }
    const int nunits = ((G + GS - 1) / GS) * (Kp / KC);
    const int nbuf = nunits > 1 ? 2 : 1;
    const size_t smem = nbuf * unit_bytes(rows, GS, KC);
    if (smem > 227 * 1024) return HE_ESHAPE;
    // K = 16 with one unit per CTA and <= 4 warps: cap registers so five
    // CTAs share an SM (occupancy-bound small-K case)
    const bool k16 = k16c && nunits == 1 && 32 * warps <= 128;
    auto k = TB16 == 2 ? (k16 ? k_mac_imma<2, HE_MAC_K16_MINB> : k_mac_imma<2>)
                       : (k16 ? k_mac_imma<1, HE_MAC_K16_MINB> : k_mac_imma<1>);
    // specialised instances for the plain-20 layer shapes (32-image tiles)
    if (HE_MAC_SPEC && TB16 == 1 && lazy && k16 && Kp == 16 && KC == 16 && c_o == 32 &&
        GS == 4)
        k = k_mac_imma<1, HE_MAC_K16_MINB, 16, 16, 32, 4, 1>;
    if (HE_MAC_SPEC && TB16 == 1 && lazy && !k16) {       // 16-image tiles, c_o >= 32
        if (Kp == 32 && KC == 32 && c_o == 32 && GS == 2)
            k = k_mac_imma<1, 1, 32, 32, 32, 2, 1>;
        else if (Kp == 32 && KC == 32 && c_o == 64 && GS == 1)
            k = k_mac_imma<1, 1, 32, 32, 64, 1, 1>;
        else if (Kp == 64 && KC == 64 && c_o == 64 && GS == 1)
            k = k_mac_imma<1, 1, 64, 64, 64, 1, 1>;
    }
    if (HE_MAC_SPEC && TB16 == 2 && lazy) {
        if (k16 && Kp == 16 && KC == 16 && c_o == 16 && GS == 4)
            k = k_mac_imma<2, HE_MAC_K16_MINB, 16, 16, 16, 4, 1>;
        else if (!k16 && Kp == 16 && KC == 16 && c_o == 32 && GS == 4)
            k = k_mac_imma<2, 1, 16, 16, 32, 4, 1>;
        else if (!k16 && Kp == 32 && KC == 32 && c_o == 32 && GS == 2)
            k = k_mac_imma<2, 1, 32, 32, 32, 2, 1>;
        else if (!k16 && Kp == 32 && KC == 32 && c_o == 64 && GS == 1)
            k = k_mac_imma<2, 1, 32, 32, 64, 1, 1>;
        else if (!k16 && Kp == 64 && KC == 64 && c_o == 64 && GS == 1)
            k = k_mac_imma<2, 1, 64, 64, 64, 1, 1>;
        else if (!k16 && Kp == 64 && KC == 32 && c_o == 64 && GS == 1)
            k = k_mac_imma<2, 1, 64, 32, 64, 1, 1>;
    }
    // fold layout [l][b][g][n] for the instances K4's row writer reads it from
    // (plain-20 s = 32 / s = 128 layers; the caller asks only then)
    if (HE_MAC_SPEC && (fl_req == 1 || fl_req == 3) && lazy) {
        auto kf = k;
        if (k16 && TB16 == 2 && Kp == 16 && KC == 16 && c_o == 16 && GS == 4)
            kf = fl_req == 3 ? k_mac_imma<2, HE_MAC_K16_MINB, 16, 16, 16, 4, 1, 3>
                             : k_mac_imma<2, HE_MAC_K16_MINB, 16, 16, 16, 4, 1, 1>;
        else if (k16 || nct != 1)
            ;
        else if (TB16 == 2 && Kp == 32 && KC == 32 && c_o == 32 && GS == 2)
            kf = k_mac_imma<2, 1, 32, 32, 32, 2, 1, 1>;
        else if (TB16 == 1 && Kp == 32 && KC == 32 && c_o == 64 && GS == 1)
            kf = k_mac_imma<1, 1, 32, 32, 64, 1, 1, 1>;
        else if (TB16 == 1 && Kp == 64 && KC == 64 && c_o == 64 && GS == 1)
            kf = k_mac_imma<1, 1, 64, 64, 64, 1, 1, 1>;
        if (kf != k) {
            k = kf;
            if (fl_used) *fl_used = (k16 && fl_req == 3) ? 3 : 1;
        }
    }
    if (!set_smem(k, smem)) return HE_ECUDA;
    // TMA staging for the K = 16 instance (one unit per CTA, whole groups)
    CUtensorMap tmA, tmF;
    memset(&tmA, 0, sizeof tmA);
    memset(&tmF, 0, sizeof tmF);
    int use_tma = 0;
    if (HE_MAC_TMA16 && k16 && TB16 == 2 && Kp == 16 && KC == 16 && c_o == 16 && GS == 4 &&
        G == GS && M % G == 0 && Gt % GS == 0 && encode_tiled() != nullptr) {
        const cuuint32_t one[3] = {1, 1, 1};
        const cuuint64_t gA[3] = {(cuuint64_t)Gt * Kp, (cuuint64_t)B, (cuuint64_t)L * (M / Gt) * 7};
        const cuuint64_t sA_[2] = {(cuuint64_t)Gt * Kp, (cuuint64_t)B * Gt * Kp};
        const cuuint32_t bA[3] = {(cuuint32_t)(GS * KC), (cuuint32_t)rows, 7};
        const cuuint64_t gF[2] = {(cuuint64_t)c_full * Kp, (cuuint64_t)L * M * 7};
        const cuuint64_t sF_[1] = {(cuuint64_t)c_full * Kp};
        const cuuint32_t bF[2] = {(cuuint32_t)(c_o * Kp), (cuuint32_t)(GS * 7)};
        auto enc = encode_tiled();
        if (enc(&tmA, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, (void*)A, gA, sA_, bA, one,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
                CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
                CUDA_SUCCESS &&
            enc(&tmF, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, (void*)Fpl, gF, sF_, bF, one,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
                CUDA_SUCCESS)
            use_tma = 1;
    }
    dim3 grid(L * ((M + G - 1) / G), (B + rows - 1) / rows, nct);
    k<<<grid, 32 * warps, smem, st>>>(A, Fpl, out, B, L, M, c_o, Kp, G, GS, KC, Gt, nbuf, limbs,
                                      lazy, c_full, use_tma, tmA, tmF);
    return HE_OK;
}

// ===================================================================== K4
// One CTA per (b, ob, l, channel chunk): (N/s)-point inverse NTTs (root
// psi^s, no scaling: N^{-1} is in the filter spectra) of the folded products
// of `cc` channels of block ob, then the output slots of those channels
// (Alg. 1 Lines 15-17; Eq. (7) shift realised as the offset t_n):
//   out[b][ob][l][s j + u] for j < N/s and u in [u0, u1),
//   u0 = ch0 * step, u1 = (last chunk ? s : (ch0 + cc) * step),
// value result_{u/step}[j] when step | u, else 0, then + enc(phi1) at every
// coefficient.  The chunks tile [0, s), so every coefficient
// of the row is written exactly once, in contiguous runs of u1 - u0 words.
// Channel arrays sit in shared memory at an odd word stride (conflict-free).
// Template arguments LN, LS, CCC, STC, NCH, COB (nonzero): log2 N, log2 s,
// cc, the array stride, nchunk and c_ob fixed at compile time -- the plain-20
// s = 8 instance turns the transform's and the writer's index arithmetic
// into immediates; 0 keeps the runtime values.
template <bool DP, int LN = 0, int LS = 0, int CCC = 0, int STC = 0, int NCH = 0, int COB = 0,
          int HP = 0, int WO = 0, int CST = 0, int FL = 0>
__global__ void __launch_bounds__(256, 4)
k_intt_scatter(const u64* __restrict__ fold, const u32* __restrict__ phi1,
               u64* __restrict__ out, u64* __restrict__ comp, PlanDev P, int B, int L,
               int logN_, int cc_, int nchunk_, int stride_, const he_limb* __restrict__ limbs,
               const ulonglong2* __restrict__ twi_all, const double* __restrict__ twid_all,
               const u64* __restrict__ enc_tab, u64 t, u64 r_t, u64 t_inv) {
    extern __shared__ u64 sm[];
    const int logN = LN ? LN : logN_, logs = LS ? LS : P.logs;
    const int cc = CCC ? CCC : cc_, nchunk = NCH ? NCH : nchunk_, stride = STC ? STC : stride_;
    const int c_ob = COB ? COB : P.c_ob, s_ = 1 << logs, step = COB ? s_ / COB : P.step;
    const int N = 1 << logN, M = N >> logs, logM = logN - logs;
    // (HP, WO, CST: padded row length h_p, output side w_o = h_o, conv stride)
    const int h_p = HP ? HP : P.h_p, w_o = WO ? WO : P.w_o, h_o = WO ? WO : P.h_o;
    const int cstr = CST ? CST : P.stride;
    int r = NCH ? (int)blockIdx.x / NCH : qdiv(blockIdx.x, nchunk);
    const int ch = blockIdx.x - r * nchunk;
    const int rl = qdiv(r, L);
    const int l = r - rl * L;
    const int b = qdiv(rl, P.n_ob), ob = rl - b * P.n_ob;
    const he_limb Lm = limbs[l];
    const u64 q = Lm.q, q2 = 2 * q;
    const ulonglong2* twi = twi_all + (size_t)l * N;
    const int ch0 = ch * cc, ncc = min(cc, c_ob - ch0);
    // fold layout [l][b][n][g]: the chunk's channel rows are contiguous in g
    const u64* fb = fold + (((size_t)l * B + b) * P.c_o + ob * c_ob + ch0) * M;
    const int tot = ncc * M, nvalid_a = min(ncc, P.c_o - (ob * c_ob + ch0));
    const bool raw = DP && logM >= 1;       // cp.async the residues, first pass converts
    if (raw && FL == 3) {
        // fold layout [l][b][n/2][g][2] (FL = 3, cc = 2: the chunk is one
        // channel pair, 2 M contiguous words)
        static_assert(FL != 3 || CCC == 2, "FL = 3 reads channel pairs");
        const u64* fg = fold + (((size_t)l * B + b) * (P.c_o >> 1) + ((ob * c_ob + ch0) >> 1)) *
                                   (2 * (size_t)M);
        for (int idx = threadIdx.x; idx < tot; idx += blockDim.x) {
            const int chn = idx & 1, g = idx >> 1;
            const bool ok = chn < nvalid_a;
            cp_async_n<8>(sm + chn * stride + PAD(g), ok ? fg + idx : fold, ok);
        }
        cp_async_commit();
        cp_async_wait<0>();
    } else if (raw && FL) {
        // fold layout [l][b][g][n] (FL = 1, k_mac_imma FL = 1): consecutive
        // threads take consecutive channels of one group
        constexpr int LCC = FL ? __builtin_ctz(CCC > 0 ? CCC : 1) : 0;
        const u64* fg = fold + ((size_t)l * B + b) * M * P.c_o + ob * c_ob + ch0;
        for (int idx = threadIdx.x; idx < tot; idx += blockDim.x) {
            const int chn = idx & (CCC - 1), g = idx >> LCC;
            const bool ok = chn < nvalid_a;
            cp_async_n<8>(sm + chn * stride + PAD(g), ok ? fg + (size_t)g * P.c_o + chn : fold, ok);
        }
        cp_async_commit();
        cp_async_wait<0>();
    } else if (raw) {
        for (int idx = threadIdx.x; idx < tot; idx += blockDim.x) {
            const bool ok = (idx >> logM) < nvalid_a;
            cp_async_n<8>(sm + (idx >> logM) * stride + PAD(idx & (M - 1)), ok ? fb + idx : fb,
                          ok);
        }
        cp_async_commit();
        cp_async_wait<0>();
    }
    for (int base = 0; !raw && base < tot; base += 8 * blockDim.x) {   // 8 loads in flight
        u64 v[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            const int idx = base + e * blockDim.x + threadIdx.x;
            v[e] = (idx < tot && (idx >> logM) < nvalid_a) ? fb[idx] : 0;
        }
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            const int idx = base + e * blockDim.x + threadIdx.x;
            if (idx < tot) {
                const int a = (idx >> logM) * stride + PAD(idx & (M - 1));
                if (DP) reinterpret_cast<double*>(sm)[a] = u2d(v[e]);
                else sm[a] = v[e];
            }
        }
    }
    __syncthreads();
    // Plain-20 s = 8 instances (two 2048-point channels per CTA, step 1, 256
    // threads, mask on): the writer below with immediate offsets
    constexpr bool W8 = FL == 3 && LN == 14 && LS == 3 && CCC == 2 && COB == 8 && HP == 34 &&
                        WO > 0 && CST > 0;
    constexpr int HPD = HP ? HP : 1;         // (divisor of the W8-only index steps; W8 implies HP = 34)
    const bool w8 = W8 && HE_K4_W8 && phi1 != nullptr && enc_tab != nullptr &&
                    blockDim.x == 256;
    // (its first phi1 batch is requested before the transform, so it has
    //  landed when the writer starts)
    u32 pre[4] = {0u, 0u, 0u, 0u};
    // (HE_K4_FUSE: the writer visits e = 0, 2, ..., 14 first, see below)
    constexpr int PSTEP = HE_K4_FUSE ? 2 : 1;
    if (w8 && HE_K4_PRE) {
        const u32* pp0 = phi1 + ((size_t)b * P.n_ob + ob) * N + ((threadIdx.x >> 1) << 3) +
                         ch * CCC + (threadIdx.x & 1);
#pragma unroll
        for (int z = 0; z < 4; ++z) pre[z] = pp0[z * PSTEP * (128 << 3)];
    }
    if (W8 && HE_K4_FUSE && w8) {
        // stages 0-7 as two radix-16 passes; stages 8-10 (the last radix-8
        // pass) run in the writer's registers below
        gs_pass_dp<4, true>(reinterpret_cast<double*>(sm), stride, ncc, logM, 0, 0, logM,
                            twid_all + (size_t)l * N, Lm.qd, Lm.qinvd);
        __syncthreads();
        gs_pass_dp<4>(reinterpret_cast<double*>(sm), stride, ncc, logM, 4, 0, logM,
                      twid_all + (size_t)l * N, Lm.qd, Lm.qinvd);
        __syncthreads();
    } else if (DP && raw)
        gs_all_dp<4, true>(reinterpret_cast<double*>(sm), stride, ncc, logM, 0, logM,
                           twid_all + (size_t)l * N, Lm.qd, Lm.qinvd);
    else if (DP)
        gs_all_dp<4>(reinterpret_cast<double*>(sm), stride, ncc, logM, 0, logM,
                     twid_all + (size_t)l * N, Lm.qd, Lm.qinvd);
    else if (logM <= 12)
        gs_all<3, true>(sm, stride, ncc, logM, 0, logM, twi, q, q2);
    else
        gs_all<3>(sm, stride, ncc, logM, 0, logM, twi, q, q2);
    const int u0 = ch0 * step;
    const int u1 = (ch == nchunk - 1) ? s_ : (ch0 + ncc) * step;
    const int w = u1 - u0;
    const u32* ph = phi1 ? phi1 + ((size_t)b * P.n_ob + ob) * N : nullptr;
    u64* orow = out ? out + (((size_t)b * P.n_ob + ob) * L + l) * N : nullptr;
    u64* crow = comp ? comp + (((size_t)b * P.n_ob + ob) * L + l) * P.n_valid : nullptr;
    int lstr = 0;                         // stride is a power of two (checked on host)
    while ((1 << lstr) < cstr) ++lstr;
    // Row writer.  Thread (uo, jt) owns slot column u = u0 + uo of every
    // group j = jt, jt + jstep, ...: its channel, ownership and smem base are
    // per-thread constants, and the (row, column) of j for the payload test
    // are advanced incrementally.  Four phi1 loads in flight; the mask encoding is
    // FP64 arithmetic (enc_dp) when the context has a table-sized t.
    // Plain-20 s = 8 instances (two 2048-point channels per CTA, step 1, 256
    // threads, mask on): the writer with every address an immediate offset.
    // Thread (uo, jt) writes slot u0 + uo of groups j = jt + 128 e, e < 16,
    // unrolled: phi1, the output row and the channel array advance by
    // compile-time strides, and the payload index follows (kr, lc) of j
    // (128 = 3 h_p + 26).  Same values and stores as the generic writer.
    if (w8) {
        constexpr int JS = 128, NE = 2048 / JS, EBW = HE_K4_W8_EB;
        constexpr int LST = CST == 1 ? 0 : (CST == 2 ? 1 : 2);
        const int uo = threadIdx.x & 1, jt = threadIdx.x >> 1;
        const int u = u0 + uo;                  // = the channel n of the block (step 1)
        const double* xs = reinterpret_cast<const double*>(sm) + (u - ch0) * stride + PAD(jt);
        const u32* pp = ph + (jt << 3) + u;
        u64* op = orow ? orow + (jt << 3) + u : nullptr;
        const double td = Lm.td, t_inv_d = Lm.t_invd, rtd = Lm.rtd, tinvq = Lm.tinvd;
        const double qd = Lm.qd, qi = Lm.qinvd;
        if (HE_K4_FUSE) {
            // The last GS pass (stages 8-10, radix 8) fused into the writer:
            // its group at offset off = jt + 128 p holds the elements
            // j = off + 256 c (c < 8), i.e. e = 2 c + p -- exactly this
            // thread's column u -- so the pass's outputs go from registers
            // to the mask add and the store (no shared-memory round trip,
            // one barrier fewer).  Block 0 of stages 8, 9, 10 for every
            // group: twiddles tw[4..7], tw[2..3], tw[1] (gs_pass_dp's
            // indexing with lt0 = 8, K = 3, seg = 0).  Same values as the
            // unfused pass + writer.
            static_assert(!W8 || EBW == 4, "fused s = 8 writer: phi1 batches of 4");
            const double* tw = twid_all + (size_t)l * N;
            u32 mn[4];
#pragma unroll
            for (int z = 0; z < 4; ++z) mn[z] = HE_K4_PRE ? pre[z] : pp[(2 * z) * (JS << 3)];
            constexpr int PU = HE_K4_FUSE_PU;
#pragma unroll PU
            for (int p = 0; p < 2; ++p) {
                double x[8];
#pragma unroll
                for (int c = 0; c < 8; ++c)
                    x[c] = dp_reduce(xs[(2 * c + p) * (JS + JS / 16)], qd, qi);
#pragma unroll
                for (int v = 0; v < 3; ++v) {
                    // (twiddles loaded per stage: L1 hits, fewer live registers)
                    double tws[4];
                    load_tw_run(tws, tw, 4 >> v, 4 >> v);
                    const int half = 1 << v;
#pragma unroll
                    for (int c = 0; c < 8; ++c) {
                        if (c & half) continue;
                        const double X = x[c], Y = x[c + half];
                        x[c] = X + Y;
                        x[c + half] = dp_mulmod(X - Y, tws[c >> (v + 1)], qd, qi);
                    }
                }
                const int j0 = jt + 128 * p;    // < 256: (j0 1928) >> 16 = j0 / 34
                int kr = (j0 * 1928) >> 16;
                int lc = j0 - kr * HP;
#pragma unroll
                for (int c0 = 0; c0 < 8; c0 += 4) {
                    u32 m[4];
#pragma unroll
                    for (int z = 0; z < 4; ++z) m[z] = mn[z];
                    if (p == 0 || c0 == 0) {    // next batch: (p, 4) or (1, 0)
                        const int np = c0 == 4 ? 1 : p, nc = c0 == 4 ? 0 : 4;
#pragma unroll
                        for (int z = 0; z < 4; ++z) mn[z] = pp[(2 * (nc + z) + np) * (JS << 3)];
                    }
#pragma unroll
                    for (int z = 0; z < 4; ++z) {
                        const int c = c0 + z, e = 2 * c + p;
                        const int K_ = kr >> LST, L_ = lc >> LST;
                        const bool valid = crow && ((kr | lc) & (CST - 1)) == 0 && K_ < WO && L_ < WO;
                        kr += 256 / HPD;
                        lc += 256 % HPD;
                        if (lc >= HP) { lc -= HP; ++kr; }
                        if (!op && !valid) continue;
                        const double y = enc_dp(u2d(m[z]), rtd, td, t_inv_d, tinvq, qd, qi) + x[c];
                        const u64 v = d2canon(y, qd, qi);
                        if (op) op[e * (JS << 3)] = v;
                        if (valid) crow[(K_ * WO + L_) * COB + u] = v;
                    }
                }
            }
            return;
        }
        int kr = (jt * 1928) >> 16;             // jt / 34 for jt < 128
        int lc = jt - kr * HP;
        u32 mnext[EBW];
#pragma unroll
        for (int z = 0; z < EBW; ++z)
            mnext[z] = (HE_K4_PRE && EBW == 4) ? pre[z < 4 ? z : 0] : pp[z * (JS << 3)];
#pragma unroll
        for (int e0 = 0; e0 < NE; e0 += EBW) {
            u32 m[EBW];
#pragma unroll
            for (int z = 0; z < EBW; ++z) m[z] = mnext[z];
            if (e0 + EBW < NE) {
#pragma unroll
                for (int z = 0; z < EBW; ++z) mnext[z] = pp[(e0 + EBW + z) * (JS << 3)];
            }
#pragma unroll
            for (int z = 0; z < EBW; ++z) {
                const int e = e0 + z;
                const int K_ = kr >> LST, L_ = lc >> LST;
                const bool valid = crow && ((kr | lc) & (CST - 1)) == 0 && K_ < WO && L_ < WO;
                kr += JS / HPD;
                lc += JS % HPD;
                if (lc >= HP) { lc -= HP; ++kr; }
                if (!op && !valid) continue;
                double y = enc_dp(u2d(m[z]), rtd, td, t_inv_d, tinvq, qd, qi);
                y += xs[e * (JS + JS / 16)];    // PAD(jt + 128 e) = PAD(jt) + 136 e
                const u64 v = d2canon(y, qd, qi);
                if (op) op[e * (JS << 3)] = v;
                if (valid) crow[(K_ * WO + L_) * COB + u] = v;
            }
        }
        return;
    }
    const int jstep = blockDim.x / w;
    const int uo = threadIdx.x % w, jt = threadIdx.x / w;
    if (jstep > 0 && jt < jstep) {
        const int u = u0 + uo;
        const int nl = u / step;
        const bool owned = u == nl * step && nl < ch0 + ncc;
        const int abase = owned ? (nl - ch0) * stride : 0;
        const bool want_c = crow && owned;
        // j = kr * h_p + lc, tracked incrementally
        int kr = jt / h_p, lc = jt - kr * h_p;
        const int dk = jstep / h_p, dl = jstep - dk * h_p;
        constexpr int EB = 4;
        // FP64 mask encoding (enc_dp) when the context has a table (t <= 2^20):
        // no random table gathers in the writer
        const bool encd = DP && enc_tab != nullptr;
        const double td = Lm.td, t_inv_d = Lm.t_invd, rtd = Lm.rtd;   // host-computed
        // transform outputs < 8q + 16 when the last pass is radix-16: reduce
        // before adding the encoding (|sum| must stay below 2^52)
        const bool xred = (logM & 3) == 0;
        if (HE_K4_PF && encd) {
            // software-pipelined phi1 loads: batch k + 1 is in flight while
            // batch k is encoded, added and stored
            u32 mn[EB];
            int vn[EB];
            auto fetch = [&](int j0) {
#pragma unroll
                for (int e = 0; e < EB; ++e) {
                    const int j = j0 + e * jstep;
                    vn[e] = -1;
                    if (want_c && j < M) {
                        const int K_ = kr >> lstr, L_ = lc >> lstr;
                        if (((kr | lc) & (cstr - 1)) == 0 && K_ < w_o && L_ < h_o)
                            vn[e] = (K_ * h_o + L_) * c_ob + nl;
                    }
                    mn[e] = (ph && j < M && (orow || vn[e] >= 0)) ? ph[(j << logs) + u] : 0u;
                    kr += dk;
                    lc += dl;
                    if (lc >= h_p) { lc -= h_p; ++kr; }
                }
            };
            fetch(jt);
            for (int j0 = jt; j0 < M; j0 += EB * jstep) {
                u32 m[EB];
                int vi[EB];
#pragma unroll
                for (int e = 0; e < EB; ++e) { m[e] = mn[e]; vi[e] = vn[e]; }
                if (j0 + EB * jstep < M) fetch(j0 + EB * jstep);
#pragma unroll
                for (int e = 0; e < EB; ++e) {
                    const int j = j0 + e * jstep;
                    if (j >= M || (!orow && vi[e] < 0)) continue;
                    double y = ph ? enc_dp(u2d(m[e]), rtd, td, t_inv_d, Lm.tinvd, Lm.qd, Lm.qinvd)
                                  : 0.0;
                    if (owned) {
                        double x = reinterpret_cast<const double*>(sm)[abase + PAD(j)];
                        if (xred) x = dp_reduce(x, Lm.qd, Lm.qinvd);
                        y += x;
                    }
                    const u64 v = d2canon(y, Lm.qd, Lm.qinvd);
                    if (orow) orow[(j << logs) + u] = v;
                    if (vi[e] >= 0) crow[vi[e]] = v;
                }
            }
        }
        for (int j0 = jt; j0 < M && !(HE_K4_PF && encd); j0 += EB * jstep) {
            u32 m[EB];
            int vi[EB];
#pragma unroll
            for (int e = 0; e < EB; ++e) {
                const int j = j0 + e * jstep;
                vi[e] = -1;
                if (want_c && j < M) {
                    const int K_ = kr >> lstr, L_ = lc >> lstr;
                    if (((kr | lc) & (cstr - 1)) == 0 && K_ < w_o && L_ < h_o)
                        vi[e] = (K_ * h_o + L_) * c_ob + nl;
                }
                m[e] = (ph && j < M && (orow || vi[e] >= 0)) ? ph[(j << logs) + u] : 0u;
                kr += dk;
                lc += dl;
                if (lc >= h_p) { lc -= h_p; ++kr; }
            }
            if (encd) {
#pragma unroll
                for (int e = 0; e < EB; ++e) {
                    const int j = j0 + e * jstep;
                    if (j >= M || (!orow && vi[e] < 0)) continue;
                    double y = ph ? enc_dp(u2d(m[e]), rtd, td, t_inv_d, Lm.tinvd, Lm.qd, Lm.qinvd)
                                  : 0.0;
                    if (owned) {
                        double x = reinterpret_cast<const double*>(sm)[abase + PAD(j)];
                        if (xred) x = dp_reduce(x, Lm.qd, Lm.qinvd);
                        y += x;
                    }
                    const u64 v = d2canon(y, Lm.qd, Lm.qinvd);
                    if (orow) orow[(j << logs) + u] = v;
                    if (vi[e] >= 0) crow[vi[e]] = v;
                }
                continue;
            }
            u64 en[EB];
#pragma unroll
            for (int e = 0; e < EB; ++e) {
                const int j = j0 + e * jstep;
                en[e] = (ph && j < M && (orow || vi[e] >= 0))
                            ? enc_lookup(enc_tab, l, t, m[e], Lm, r_t, t_inv) : 0;
            }
#pragma unroll
            for (int e = 0; e < EB; ++e) {
                const int j = j0 + e * jstep;
                if (j >= M || (!orow && vi[e] < 0)) continue;
                u64 v = 0;
                if (owned)
                    v = DP ? d2canon(reinterpret_cast<const double*>(sm)[abase + PAD(j)], Lm.qd,
                                     Lm.qinvd)
                           : reduce_full(sm[abase + PAD(j)], q, Lm.one_p);
                v = addmod(v, en[e], q);
                if (orow) orow[(j << logs) + u] = v;
                if (vi[e] >= 0) crow[vi[e]] = v;
            }
        }
    }
    // (w > blockDim, i.e. more than 256 slot columns per chunk: jstep = 0,
    //  the writer above is skipped and this sweep covers every column)
    for (int ub = jstep > 0 ? w : 0; ub < w; ub += blockDim.x) {
        const int u = u0 + ub + threadIdx.x;
        if (u >= u1) continue;
        const int nl = u / step;
        const bool owned = u == nl * step && nl < ch0 + ncc;
        for (int j = 0; j < M; ++j) {
            const int kr = j / h_p, lc = j - kr * h_p;
            int vidx = -1;
            if (crow && owned) {
                const int K_ = kr >> lstr, L_ = lc >> lstr;
                if (((kr | lc) & (cstr - 1)) == 0 && K_ < w_o && L_ < h_o)
                    vidx = (K_ * h_o + L_) * c_ob + nl;
            }
            if (!orow && vidx < 0) continue;
            u64 v = 0;
            if (owned)
                v = DP ? d2canon(reinterpret_cast<const double*>(sm)[(nl - ch0) * stride + PAD(j)],
                                 Lm.qd, Lm.qinvd)
                       : reduce_full(sm[(nl - ch0) * stride + PAD(j)], q, Lm.one_p);
            if (ph) v = addmod(v, enc_lookup(enc_tab, l, t, ph[(j << logs) + u], Lm, r_t, t_inv), q);
            if (orow) orow[(j << logs) + u] = v;
            if (vidx >= 0) crow[vidx] = v;
        }
    }
}

// K4, row-writer form (FP64 transforms, t <= 2^20): the same CTA work as
// k_intt_scatter -- (N/s)-point inverse transforms of the cc channels of one
// (b, ob, l) chunk, then the chunk's slot columns [u0, u1) of every group j
// -- but the writer maps threads to (j, V consecutive columns): V = 2 words
// leave as one 16-byte store and their phi1 as one 8-byte load, a warp
// covers whole runs of the row, and the valid-slot payload index comes from
// a per-CTA table jv[j] = K w_o' + L (or -1), built while the fold rows load,
// instead of per-element row/column tracking.  FL = 1: the fold arrives in
// the [l][b][g][n] layout (k_mac_imma FL = 1; CCC, COB fixed).
template <int V, int LN = 0, int LS = 0, int CCC = 0, int STC = 0, int NCH = 0, int COB = 0,
          int FL = 0>
__global__ void __launch_bounds__(256, HE_K4_ROWS_MINB)
k_intt_rows(const u64* __restrict__ fold, const u32* __restrict__ phi1,
            u64* __restrict__ out, u64* __restrict__ comp, PlanDev P, int B, int L, int logN_,
            int cc_, int nchunk_, int stride_, const he_limb* __restrict__ limbs,
            const double* __restrict__ twid_all, double rtd, double td, double t_inv_d) {
    extern __shared__ u64 sm[];
    // (compile-time geometry as k_intt_scatter's template arguments; 0 = runtime)
    const int logN = LN ? LN : logN_, logs = LS ? LS : P.logs;
    const int cc = CCC ? CCC : cc_, nchunk = NCH ? NCH : nchunk_, stride = STC ? STC : stride_;
    const int c_ob = COB ? COB : P.c_ob, s_ = 1 << logs, step = COB ? s_ / COB : P.step;
    const int N = 1 << logN, M = N >> logs, logM = logN - logs;
    int r = NCH ? (int)blockIdx.x / NCH : qdiv(blockIdx.x, nchunk);
    const int ch = blockIdx.x - r * nchunk;
    const int rl = qdiv(r, L);
    const int l = r - rl * L;
    const int b = qdiv(rl, P.n_ob), ob = rl - b * P.n_ob;
    const double qd = limbs[l].qd, qi = limbs[l].qinvd, tinvq = limbs[l].tinvd;
    const int ch0 = ch * cc, ncc = min(cc, c_ob - ch0);
    const u64* fb = fold + (((size_t)l * B + b) * P.c_o + ob * c_ob + ch0) * M;
    const int tot = ncc * M, nvalid_a = min(ncc, P.c_o - (ob * c_ob + ch0));
    if (FL) {
        // [l][b][g][n]: consecutive threads take consecutive channels of one group
        static_assert(!FL || (CCC > 0 && COB > 0), "FL needs the compile-time chunk");
        constexpr int LCC = FL ? __builtin_ctz(CCC > 0 ? CCC : 1) : 0;
        const u64* fg = fold + ((size_t)l * B + b) * M * P.c_o + ob * c_ob + ch0;
        for (int idx = threadIdx.x; idx < tot; idx += blockDim.x) {
            const int chn = idx & (CCC - 1), g = idx >> LCC;
            const bool ok = chn < nvalid_a;
            cp_async_n<8>(sm + chn * stride + PAD(g), ok ? fg + (size_t)g * P.c_o + chn : fold, ok);
        }
    } else {
        for (int idx = threadIdx.x; idx < tot; idx += blockDim.x) {
            const bool ok = (idx >> logM) < nvalid_a;
            cp_async_n<8>(sm + (idx >> logM) * stride + PAD(idx & (M - 1)), ok ? fb + idx : fb,
                          ok);
        }
    }
    cp_async_commit();
    int* jv = reinterpret_cast<int*>(sm + (size_t)cc * stride);
    u64* crow = comp ? comp + (((size_t)b * P.n_ob + ob) * L + l) * P.n_valid : nullptr;
    if (crow) {
        // j = kr h_p + lc without integer division: kr = floor((j + 1/2) / h_p)
        // in float is exact for j < 2^22 ((j + 1/2) / h_p is >= 1/(2 h_p) away
        // from an integer, the float error below that); the conv stride is a
        // power of two (checked by he_conv_plan_make)
        const float ihp = __frcp_rn((float)P.h_p);
        const int lstr = __ffs(P.stride) - 1;
        for (int j = threadIdx.x; j < M; j += blockDim.x) {
            const int kr = (int)(((float)j + 0.5f) * ihp), lc = j - kr * P.h_p;
            const int K_ = kr >> lstr, L_ = lc >> lstr;
            jv[j] = (((kr | lc) & (P.stride - 1)) == 0 && K_ < P.w_o && L_ < P.h_o)
                        ? (K_ * P.h_o + L_) * c_ob : -1;
        }
    }
    const int u0 = ch0 * step;
    const int u1 = (ch == nchunk - 1) ? s_ : (ch0 + ncc) * step;
    const int w = u1 - u0;                         // a multiple of V (host)
    // Compile-time instances (LN, LS, CCC, COB fixed; 256 threads): 256 is a
    // multiple of the threads per group, so every thread keeps the same two
    // slot columns (ua, ua + 1) for all the groups j = jt + e JSTEP it
    // visits -- their channels, ownership and array rows are per-thread
    // constants and phi1 / the output row advance by compile-time strides.
    // Same values and stores as the generic loop below.
    constexpr bool RW = HE_K4_RW && V == 2 && LN > 0 && LS > 0 && CCC > 0 && COB > 0;
    constexpr int STEP = (1 << LS) / (COB > 0 ? COB : 1), W = CCC * STEP;
    constexpr int TPJ = W / 2 > 0 ? W / 2 : 1;
    constexpr int LSTEP = __builtin_ctz(STEP), LTPJ = __builtin_ctz(TPJ);
    constexpr int JSTEP = 256 / TPJ, MM = (1 << LN) >> LS, NE = MM / JSTEP > 0 ? MM / JSTEP : 1;
    constexpr int EB = 4;
    const bool rw = RW && blockDim.x == 256 && phi1 != nullptr && w == W;
    // (its first phi1 batch is requested before the transform)
    uint2 pre[EB];
    if (rw && HE_K4_PRE) {
        const u32* pp0 = phi1 + ((size_t)b * P.n_ob + ob) * N +
                         ((size_t)(threadIdx.x >> LTPJ) << LS) + u0 + (threadIdx.x & (TPJ - 1)) * 2;
#pragma unroll
        for (int z = 0; z < EB; ++z)
            pre[z] = *reinterpret_cast<const uint2*>(pp0 + ((size_t)(z * JSTEP) << LS));
    }
    cp_async_wait<0>();
    __syncthreads();
    gs_all_dp<4, true>(reinterpret_cast<double*>(sm), stride, ncc, logM, 0, logM,
                       twid_all + (size_t)l * N, qd, qi);
    const int tpj = w / V;                         // threads per group j (a power of two)
    const int ltpj = __ffs(tpj) - 1;
    const u32* ph = phi1 ? phi1 + ((size_t)b * P.n_ob + ob) * N : nullptr;
    u64* orow = out ? out + (((size_t)b * P.n_ob + ob) * L + l) * N : nullptr;
    const bool xred = (logM & 3) == 0;             // radix-16 last pass: outputs < 8q + 16
    const double* smd = reinterpret_cast<const double*>(sm);
    const int lstep = __ffs(step) - 1;           // step = s / c_ob, a power of two
    if (rw) {
        static_assert(!RW || (TPJ >= 1 && 256 % TPJ == 0 && MM % (JSTEP * EB) == 0),
                      "row-writer instance geometry");
        const int uo = (threadIdx.x & (TPJ - 1)) * 2, jt = threadIdx.x >> LTPJ;
        const int ua = u0 + uo;
        const int nla = ua >> LSTEP, nlb = (ua + 1) >> LSTEP;
        const bool owna = (ua & (STEP - 1)) == 0 && nla < ch0 + ncc;
        const bool ownb = ((ua + 1) & (STEP - 1)) == 0 && nlb < ch0 + ncc;
        const double* xa = smd + (owna ? nla - ch0 : 0) * STC;
        const double* xb = smd + (ownb ? nlb - ch0 : 0) * STC;
        const u32* pp = ph + ((size_t)jt << LS) + ua;
        u64* op = orow ? orow + ((size_t)jt << LS) + ua : nullptr;
        uint2 mn[EB];
#pragma unroll
        for (int z = 0; z < EB; ++z)
            mn[z] = HE_K4_PRE ? pre[z] : *reinterpret_cast<const uint2*>(pp + ((size_t)(z * JSTEP) << LS));
#pragma unroll 1
        for (int e0 = 0; e0 < NE; e0 += EB) {
            uint2 m[EB];
#pragma unroll
            for (int z = 0; z < EB; ++z) m[z] = mn[z];
            if (e0 + EB < NE) {
#pragma unroll
                for (int z = 0; z < EB; ++z)
                    mn[z] = *reinterpret_cast<const uint2*>(
                        pp + ((size_t)((e0 + EB + z) * JSTEP) << LS));
            }
#pragma unroll
            for (int z = 0; z < EB; ++z) {
                const int j = jt + (e0 + z) * JSTEP;
                const int jvj = crow ? jv[j] : -1;
                if (!op && jvj < 0) continue;
                double ya = enc_dp(u2d(m[z].x), rtd, td, t_inv_d, tinvq, qd, qi);
                double yb = enc_dp(u2d(m[z].y), rtd, td, t_inv_d, tinvq, qd, qi);
                if (owna) {
                    double x = xa[PAD(j)];
                    if (xred) x = dp_reduce(x, qd, qi);
                    ya += x;
                }
                if (ownb) {
                    double x = xb[PAD(j)];
                    if (xred) x = dp_reduce(x, qd, qi);
                    yb += x;
                }
                const u64 va = d2canon(ya, qd, qi), vb = d2canon(yb, qd, qi);
                if (op)
                    *reinterpret_cast<ulonglong2*>(op + ((size_t)((e0 + z) * JSTEP) << LS)) =
                        make_ulonglong2(va, vb);
                if (jvj >= 0) {
                    if (owna) crow[jvj + nla] = va;
                    if (ownb) crow[jvj + nlb] = vb;
                }
            }
        }
        return;
    }
    constexpr int UB = 4;                          // elements per thread in flight
    const int nel = M * tpj;
    for (int e0 = threadIdx.x; e0 < nel; e0 += UB * blockDim.x) {
        uint2 m2[UB];
        u32 m1[UB];
#pragma unroll
        for (int z = 0; z < UB; ++z) {
            const int e = e0 + z * blockDim.x;
            const int j = e >> ltpj, uo = (e & (tpj - 1)) * V;
            m2[z] = make_uint2(0u, 0u);
            m1[z] = 0u;
            if (e < nel && ph && (orow || (crow && jv[j] >= 0))) {
                const u32* pp = ph + ((size_t)j << logs) + u0 + uo;
                if (V == 2) m2[z] = *reinterpret_cast<const uint2*>(pp);
                else m1[z] = *pp;
            }
        }
#pragma unroll
        for (int z = 0; z < UB; ++z) {
            const int e = e0 + z * blockDim.x;
            if (e >= nel) break;
            const int j = e >> ltpj, uo = (e & (tpj - 1)) * V;
            const int jvj = crow ? jv[j] : -1;
            if (!orow && jvj < 0) continue;
            u64 v[V];
#pragma unroll
            for (int k = 0; k < V; ++k) {
                const int u = u0 + uo + k;
                const u32 mm = V == 2 ? (k ? m2[z].y : m2[z].x) : m1[z];
                double y = ph ? enc_dp(u2d(mm), rtd, td, t_inv_d, tinvq, qd, qi) : 0.0;
                const int nl = u >> lstep;
                const bool owned = (u & (step - 1)) == 0 && nl < ch0 + ncc;
                if (owned) {
                    double x = smd[(nl - ch0) * stride + PAD(j)];
                    if (xred) x = dp_reduce(x, qd, qi);
                    y += x;
                }
                v[k] = d2canon(y, qd, qi);
                if (jvj >= 0 && owned) crow[jvj + nl] = v[k];
            }
            if (orow) {
                u64* op = orow + ((size_t)j << logs) + u0 + uo;
                if (V == 2) *reinterpret_cast<ulonglong2*>(op) = make_ulonglong2(v[0], v[V - 1]);
                else op[0] = v[0];
            }
        }
    }
}

// Workspace of he_conv: forward spectra (split25 words, or the MAC-tile
// byte layout, whichever is larger) followed by the folded products.
static size_t spec_words(const he_ctx* c, const he_conv_plan* p, int B) {
    const size_t M = (size_t)c->N / p->s;
    const size_t split = (size_t)B * p->n_ib * c->L * c->N;
    const size_t tile =
        ((size_t)c->L * M * 7 * B * imma_kp(p->n_ib * p->k_u) + 7) / 8;
    return std::max(split, tile);
}

extern "C" size_t he_conv_workspace_bytes(const he_ctx* c, const he_conv_plan* p, int B) {
    if (!c || !p || B < 0) return 0;
    const size_t M = (size_t)c->N / p->s;
    const size_t fold = (size_t)c->L * M * B * p->d.c_o;
    return sizeof(u64) * (spec_words(c, p, B) + fold) + 256;
}

static inline void rec(void* const* ev, int i, cudaStream_t st) {
    if (ev && ev[i]) cudaEventRecord((cudaEvent_t)ev[i], st);
}

extern "C" he_status he_conv(const he_ctx* c, const he_conv_plan* p, const uint64_t* d_c0,
                             int B, const uint64_t* d_fspec, const uint32_t* d_phi1,
                             uint64_t* d_out, void* d_ws, size_t ws_bytes, void* stream) {
    if (!d_out && B > 0) return HE_EINVAL;
    return he_conv_ex(c, p, d_c0, B, d_fspec, d_phi1, d_out, nullptr, d_ws, ws_bytes, stream,
                      nullptr);
}

extern "C" he_status he_conv_ex(const he_ctx* c, const he_conv_plan* p, const uint64_t* d_c0,
                                int B, const uint64_t* d_fspec, const uint32_t* d_phi1,
                                uint64_t* d_out, uint64_t* d_compact, void* d_ws,
                                size_t ws_bytes, void* stream, void* const* ev) {
    if (!c || !p || B < 0) return HE_EINVAL;
    if (!plan_ok(c, p)) return HE_ESHAPE;
    if (B == 0) return HE_OK;
    if (!d_c0 || !d_fspec || (!d_out && !d_compact) || !d_ws) return HE_EINVAL;
    if (ws_bytes < he_conv_workspace_bytes(c, p, B)) return HE_ENOMEM;
    cudaStream_t st = STREAM(stream);
    const PlanDev P = plan_dev(p);
    u64* spec = (u64*)d_ws;
    u64* fold = spec + spec_words(c, p, B);
    const bool imma = use_imma(c, P);
    rec(ev, 0, st);
    he_status s = launch_ntt_fwd(c, (const u64*)d_c0, spec, (long)B * P.n_ib * c->L,
                                 imma ? 2 : 1, st,
                                 TileLay{B, P.n_ib, P.logs, imma_kp(P.n_ib * P.Ku),
                                         tile_gt(c->N >> P.logs), P.logs, P.Ku});
    if (s != HE_OK) return s;
    rec(ev, 1, st);
    // K4 row-writer instances that read the [l][b][g][n] fold (see below)
    const int Mq = c->N >> P.logs;
    const bool rows_path = c->ntt_mode == 0 && c->d_enc != nullptr && Mq >= 2 &&
                           Mq <= HE_K4_ROWS_MAXM && HE_K4_ROWS;
    const bool fl_rows = HE_FOLD_GN && HE_K4_SPEC && rows_path && c->logN == 14 &&
                         ((P.logs == 5 && P.c_ob == 32) || (P.logs == 7 && P.c_ob == 64));
    // the s = 8 scatter instances (K4 below: cc = 2, stride 2184, 4 chunks)
    const bool fl_s8 = HE_FOLD_GN8 && HE_K4_SPEC && c->ntt_mode == 0 && c->logN == 14 &&
                       P.logs == 3 && P.c_ob == 8 && P.h_p == 34 &&
                       ((P.w_o == 32 && P.h_o == 32 && P.stride == 1) ||
                        (P.w_o == 16 && P.h_o == 16 && P.stride == 2));
    // config 5 (N = 32768, s = 256, 64 channels): the tcgen05 MAC writes
    // [l][b][g][n] for the k_intt_rows<2, 15, 8, 32, 137, 2, 64, 1> instance
    const bool fl_c5 = HE_FOLD_GN5 && HE_K4_SPEC && rows_path && c->logN == 15 &&
                       P.logs == 8 && P.c_ob == 64;
    const int fl_req = fl_rows ? 1 : (fl_s8 ? HE_FOLD_GN8 : (fl_c5 ? 4 : 0));
    int fl_used = 0;
    if (imma)
        s = launch_mac_imma((const unsigned char*)spec, (const unsigned char*)d_fspec, fold, B,
                            P.n_ib, c->L, c->logN, P.logs, P.c_o, c->d_limb, st, P.Ku,
                            c->ntt_mode == 0, c->mac_tc, fl_req, &fl_used);
    else
        s = launch_mac(spec, (const u64*)d_fspec, fold, B, P.n_ib, c->L, c->logN, P.logs,
                       P.c_o, c->d_limb, st, P.Ku);
    if (s != HE_OK) return s;
    HE_CHECK_LAUNCH();
    const int M = c->N >> P.logs;
    // row-writer K4 (k_intt_rows): FP64 transforms and the FP64 mask encoding
    // (t <= 2^20); chunks of at least HE_K4_MINW slot columns when the block
    // has them, so a chunk's run of each group is at least 32 bytes
    if (c->ntt_mode == 0 && c->d_enc != nullptr && M >= 2 && M <= HE_K4_ROWS_MAXM &&
        HE_K4_ROWS) {
        int cc = std::max(1, std::min(P.c_ob, HE_K4_WORDS / (padded_words(M) + 16)));
        while (cc & (cc - 1)) cc &= cc - 1;
        while (cc < P.c_ob && cc * P.step < HE_K4_MINW) cc *= 2;
        if (HE_K4_SPEC && c->logN == 14 && P.logs == 5 && P.c_ob == 32) cc = HE_K4_CC32;
        if (HE_K4_SPEC && c->logN == 14 && P.logs == 7 && P.c_ob == 64) cc = HE_K4_CC128;
        int stride = padded_words(M);
        const int want = cc < 16 ? (16 / cc) & 15 : 1;
        while ((stride & 15) != want && !(cc >= 16 && (stride & 1))) ++stride;
        const int nchunk = (P.c_ob + cc - 1) / cc;
        const int wl = P.s - (nchunk - 1) * cc * P.step;          // last chunk's width
        const bool v2 = ((cc * P.step) & 1) == 0 && (wl & 1) == 0;
        auto pow2 = [](int x) { return x > 0 && (x & (x - 1)) == 0; };
        // (thread -> (j, column) by shifts: step and both chunk widths powers of two)
        if (pow2(P.step) && pow2(cc * P.step) && pow2(wl) && wl == cc * P.step) {
        const size_t smem = sizeof(u64) * (size_t)cc * stride + sizeof(int) * (size_t)M;
        auto k4 = v2 ? k_intt_rows<2> : k_intt_rows<1>;
        if (HE_K4_SPEC && v2 && c->logN == 14) {       // plain-20 s = 32 and s = 128 layers
            if (P.logs == 5 && cc == HE_K4_CC32 && stride == K4_ST32 && P.c_ob == 32)
                k4 = fl_used ? k_intt_rows<2, 14, 5, HE_K4_CC32, K4_ST32, 32 / HE_K4_CC32, 32, 1>
                             : k_intt_rows<2, 14, 5, HE_K4_CC32, K4_ST32, 32 / HE_K4_CC32, 32>;
            else if (P.logs == 7 && cc == HE_K4_CC128 && stride == K4_ST128 && P.c_ob == 64)
                k4 = fl_used ? k_intt_rows<2, 14, 7, HE_K4_CC128, K4_ST128, 64 / HE_K4_CC128, 64, 1>
                             : k_intt_rows<2, 14, 7, HE_K4_CC128, K4_ST128, 64 / HE_K4_CC128, 64>;
        }
        // (fl_req is set exactly for these two instances' shapes, so a fold in
        //  the [l][b][g][n] layout always meets its reader; guard regardless)
        if (fl_used == 4 && HE_K4_SPEC && v2 && c->logN == 15 && P.logs == 8 && cc == 32 &&
            stride == 137 && nchunk == 2 && P.c_ob == 64)
            k4 = k_intt_rows<2, 15, 8, 32, 137, 2, 64, 1>;
        if (fl_used && k4 != k_intt_rows<2, 14, 5, HE_K4_CC32, K4_ST32, 32 / HE_K4_CC32, 32, 1> &&
            k4 != k_intt_rows<2, 15, 8, 32, 137, 2, 64, 1> &&
            k4 != k_intt_rows<2, 14, 7, HE_K4_CC128, K4_ST128, 64 / HE_K4_CC128, 64, 1>)
            return HE_ESHAPE;
        if (!set_smem(k4, smem)) return HE_ECUDA;
        rec(ev, 2, st);
        const double td = (double)c->t;
        k4<<<(unsigned)(B * P.n_ob * c->L * nchunk), 256, smem, st>>>(
            fold, d_phi1, (u64*)d_out, (u64*)d_compact, P, B, c->L, c->logN, cc, nchunk, stride,
            c->d_limb, c->d_twd_inv, (double)c->r_t, td, 1.0 / td);
        HE_CHECK_LAUNCH();
        rec(ev, 3, st);
        return HE_OK;
        }
    }
    int cc = std::max(1, std::min(P.c_ob, 6144 / (padded_words(M) + 16)));  // <= 48 KB
    while (cc & (cc - 1)) cc &= cc - 1;                       // power of two
    // array stride (words) = 16/cc (mod 16) for cc < 16, odd otherwise: the
    // row writer reads (channel-fastest) 16 consecutive threads conflict-free
    int stride = padded_words(M);
    const int want = cc < 16 ? (16 / cc) & 15 : 1;
    while ((stride & 15) != want && !(cc >= 16 && (stride & 1))) ++stride;
    const int nchunk = (P.c_ob + cc - 1) / cc;
    const size_t smem = sizeof(u64) * (size_t)cc * stride;
    auto k4 = c->ntt_mode == 0 ? k_intt_scatter<true> : k_intt_scatter<false>;
    if (HE_K4_SPEC && c->ntt_mode == 0 && c->logN == 14 && P.logs == 3 && cc == 2 &&
        stride == 2184 && nchunk == 4 && P.c_ob == 8) {
        k4 = k_intt_scatter<true, 14, 3, 2, 2184, 4, 8>;
        if (P.h_p == 34 && P.w_o == 32 && P.h_o == 32 && P.stride == 1)
            k4 = fl_used == 3 ? k_intt_scatter<true, 14, 3, 2, 2184, 4, 8, 34, 32, 1, 3>
               : fl_used ? k_intt_scatter<true, 14, 3, 2, 2184, 4, 8, 34, 32, 1, 1>
                         : k_intt_scatter<true, 14, 3, 2, 2184, 4, 8, 34, 32, 1>;
        else if (P.h_p == 34 && P.w_o == 16 && P.h_o == 16 && P.stride == 2)
            k4 = fl_used == 3 ? k_intt_scatter<true, 14, 3, 2, 2184, 4, 8, 34, 16, 2, 3>
               : fl_used ? k_intt_scatter<true, 14, 3, 2, 2184, 4, 8, 34, 16, 2, 1>
                         : k_intt_scatter<true, 14, 3, 2, 2184, 4, 8, 34, 16, 2>;
    }
    if (fl_used && k4 != k_intt_scatter<true, 14, 3, 2, 2184, 4, 8, 34, 32, 1, 1> &&
        k4 != k_intt_scatter<true, 14, 3, 2, 2184, 4, 8, 34, 16, 2, 1> &&
        k4 != k_intt_scatter<true, 14, 3, 2, 2184, 4, 8, 34, 32, 1, 3> &&
        k4 != k_intt_scatter<true, 14, 3, 2, 2184, 4, 8, 34, 16, 2, 3>)
        return HE_ESHAPE;                     // (unreachable: fl_req matches these shapes)
    if (!set_smem(k4, smem)) return HE_ECUDA;
    rec(ev, 2, st);
    k4<<<(unsigned)(B * P.n_ob * c->L * nchunk), 256, smem, st>>>(
        fold, d_phi1, (u64*)d_out, (u64*)d_compact, P, B, c->L, c->logN, cc, nchunk, stride,
        c->d_limb, c->d_tw_inv, c->d_twd_inv, c->d_enc, c->t, c->r_t, c->t_inv);
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

// ===================================================== multi-image packing
// P images at offsets p D of one ciphertext.
static void multi_spacing(const PlanDev& P, long N, int* D, int* Pn) {
    const long s = P.s, hp = P.h_p;
    const long pw = P.padw, ph = P.padh;
    const long in_lo = s * ((pw - P.f_w) * hp + ph);
    const long in_hi = s * ((pw + P.w_i - 1 - P.f_w) * hp + ph + P.h_i - 1) + P.c_ib - 1;
    const long f_lo = s * (hp - P.f_h + 1) - (P.c_ib - 1);
    const long f_hi = s * hp * P.f_w + (s - 1);
    const long lo = in_lo + f_lo, hi = in_hi + f_hi;
    const long S = P.stride;
    const long v_hi = s * (S * (P.w_o - 1) * hp + S * (P.h_o - 1)) + s - 1;
    long d = std::max(hi + 1, v_hi - lo + 1);
    d = (d + s - 1) / s * s;
    *D = (int)d;
    *Pn = (int)(N / d);
}

extern "C" he_status he_multi_image_spacing(const he_ctx* c, const he_conv_plan* p, int32_t* D,
                                            int32_t* Pn) {
    if (!c || !p || !D || !Pn) return HE_EINVAL;
    if (!plan_ok(c, p)) return HE_ESHAPE;
    int d, n;
    multi_spacing(plan_dev(p), c->N, &d, &n);
    if (n < 1) return HE_ESHAPE;
    *D = d;
    *Pn = n;
    return HE_OK;
}

// coefficient i of ciphertext (cb, beta, l): for each slot p the raw Eq. (5)
// exponent E with E + p D = i (mod N) is one of i - p D, i - p D -+ N (sign -1
// for the wrapped ones); at most one (p, E) lands on an image pixel.
__global__ void k_pack_input_multi(const int32_t* __restrict__ img, const u64* __restrict__ ve,
                                   u64* __restrict__ out, PlanDev P, int B, int Pn, int D,
                                   int Bc, int L, int logN, const he_limb* __restrict__ limbs,
                                   u64 t, u64 r_t, u64 t_inv) {
    const long N = 1L << logN;
    const long total = (long)Bc * P.n_ib * L * N;
    for (long idx = blockIdx.x * (long)blockDim.x + threadIdx.x; idx < total;
         idx += (long)gridDim.x * blockDim.x) {
        const int i = (int)(idx & (N - 1));
        const long r = idx >> logN;
        const int l = (int)(r % L);
        const long bb = r / L;
        const int beta = (int)(bb % P.n_ib), cb = (int)(bb / P.n_ib);
        long coef = 0;
        for (int p = 0; p < Pn; ++p) {
            const int b = cb * Pn + p;
            if (b >= B) break;
#pragma unroll
            for (int cand = 0; cand < 3; ++cand) {
                const long E = (long)i - (long)p * D + (cand == 0 ? 0 : (cand == 1 ? -N : N));
                const int m = (int)(E & (P.s - 1));          // E mod s (floor)
                const long Pq = (E - m) >> P.logs;
                const int kk = floordiv((int)Pq, P.h_p);
                const int ll = (int)Pq - kk * P.h_p;
                const int k = kk + P.f_w;
                const int ch = beta * P.c_ib + m;
                if (k >= 0 && k < P.w_p && m < P.c_ib && ch < P.c_i) {
                    const int ki = k - P.padw, li = ll - P.padh;
                    if (ki >= 0 && ki < P.w_i && li >= 0 && li < P.h_i) {
                        const long pix = img[(((long)b * P.c_i + ch) * P.w_i + ki) * P.h_i + li];
                        coef += cand == 0 ? pix : -pix;
                    }
                }
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

extern "C" he_status he_pack_input_multi(const he_ctx* c, const he_conv_plan* p,
                                         const int32_t* d_img, int B, int Pn, int D,
                                         const uint64_t* d_ve, uint64_t* d_pt, void* stream) {
    if (!c || !p || B < 0 || Pn < 1 || D < 1) return HE_EINVAL;
    if (!plan_ok(c, p)) return HE_ESHAPE;
    int Dm, Pm;
    multi_spacing(plan_dev(p), c->N, &Dm, &Pm);
    if (D % p->s || D < Dm || (long)Pn * D > (long)c->N) return HE_ESHAPE;
    if (B == 0) return HE_OK;
    if (!d_img || !d_pt) return HE_EINVAL;
    const int Bc = (B + Pn - 1) / Pn;
    const long total = (long)Bc * p->n_ib * c->L * c->N;
    k_pack_input_multi<<<grid_for(total, 256), 256, 0, STREAM(stream)>>>(
        d_img, (const u64*)d_ve, (u64*)d_pt, plan_dev(p), B, Pn, D, Bc, c->L, c->logN,
        c->d_limb, c->t, c->r_t, c->t_inv);
    HE_CHECK_LAUNCH();
    return HE_OK;
}

__global__ void k_mask_extract_multi(const u64* __restrict__ full, const u32* __restrict__ phi1,
                                     u64* __restrict__ comp, PlanDev P, int Bc, int Pn, int D,
                                     int L, int logN, const he_limb* __restrict__ limbs, u64 t,
                                     u64 r_t, u64 t_inv) {
    const long N = 1L << logN;
    const long per = (long)Pn * P.n_valid;
    const long total = (long)Bc * P.n_ob * L * per;
    for (long idx = blockIdx.x * (long)blockDim.x + threadIdx.x; idx < total;
         idx += (long)gridDim.x * blockDim.x) {
        const long w = idx % per;
        const long r = idx / per;                      // (cb, ob, l)
        const int l = (int)(r % L);
        const long bo = r / L;
        const int p = (int)(w / P.n_valid), v = (int)(w - (long)p * P.n_valid);
        const int nl = v % P.c_ob, Pq = v / P.c_ob;
        const int Lc = Pq % P.h_o, Kr = Pq / P.h_o;
        const long i = (long)p * D + (long)P.s * (P.stride * Kr * (long)P.h_p + P.stride * Lc) +
                       (long)nl * P.step;
        u64 x = full[r * N + i];
        if (phi1) {
            const he_limb& Lm = limbs[l];
            x = addmod(x, enc_plain(phi1[bo * N + i], Lm, t, r_t, t_inv), Lm.q);
        }
        comp[idx] = x;
    }
}

extern "C" he_status he_mask_extract_multi(const he_ctx* c, const he_conv_plan* p,
                                           const uint64_t* d_out, int Bc, int Pn, int D,
                                           const uint32_t* d_phi1, uint64_t* d_compact,
                                           void* stream) {
    if (!c || !p || Bc < 0 || Pn < 1 || D < 1) return HE_EINVAL;
    if (!plan_ok(c, p)) return HE_ESHAPE;
    int Dm, Pm;
    multi_spacing(plan_dev(p), c->N, &Dm, &Pm);
    if (D % p->s || D < Dm || (long)Pn * D > (long)c->N) return HE_ESHAPE;
    if (Bc == 0) return HE_OK;
    if (!d_out || !d_compact) return HE_EINVAL;
    const long total = (long)Bc * p->n_ob * c->L * Pn * p->n_valid;
    k_mask_extract_multi<<<grid_for(total, 256), 256, 0, STREAM(stream)>>>(
        (const u64*)d_out, d_phi1, (u64*)d_compact, plan_dev(p), Bc, Pn, D, c->L, c->logN,
        c->d_limb, c->t, c->r_t, c->t_inv);
    HE_CHECK_LAUNCH();
    return HE_OK;
}

// ===================================================================== FC
// Sub-matrix plan (reading R27, "decomposed into sub-matrices
// whose sizes are smaller or equal to N"): input blocks of n_it = min(n_i, N)
// columns, output tiles of n_ot = min(n_o, N / n_it) rows.  Input block beta
// is packed with stride n_ot (Eq. (9)); tile t = sum_beta c0_beta w_{beta,t}.
struct FcP {
    int n_i, n_o, n_it, n_ib, n_ot, n_t;
};
static FcP fc_plan(const he_ctx* c, const he_fc_desc* f) {
    FcP p;
    p.n_i = f->n_i;
    p.n_o = f->n_o;
    p.n_it = std::min<int>(f->n_i, c->N);
    p.n_ib = (f->n_i + p.n_it - 1) / p.n_it;
    p.n_ot = std::min<int>(f->n_o, c->N / p.n_it);
    p.n_t = (f->n_o + p.n_ot - 1) / p.n_ot;
    return p;
}

static bool fc_ok(const he_ctx* c, const he_fc_desc* f) {
    return c && f && f->n_i >= 1 && f->n_o >= 1;
}

// out [B][n_ib][L][N]: block beta holds I[beta n_it + l'] at X^{l' n_ot}
__global__ void k_pack_fc_input(const int32_t* __restrict__ in, const u64* __restrict__ ve,
                                u64* __restrict__ out, FcP P, int B, int L, int logN,
                                const he_limb* __restrict__ limbs, u64 t, u64 r_t,
                                u64 t_inv) {
    const long N = 1L << logN;
    const long total = (long)B * P.n_ib * L * N;
    for (long idx = blockIdx.x * (long)blockDim.x + threadIdx.x; idx < total;
         idx += (long)gridDim.x * blockDim.x) {
        const int i = (int)(idx & (N - 1));
        const long r = idx >> logN;
        const int l = (int)(r % L);
        const long bb = r / L;
        const int beta = (int)(bb % P.n_ib), b = (int)(bb / P.n_ib);
        const int col = i / P.n_ot, gcol = beta * P.n_it + col;
        long m = 0;
        if (i - col * P.n_ot == 0 && col < P.n_it && gcol < P.n_i)
            m = in[(long)b * P.n_i + gcol];                                 // Eq. (9)
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
    const FcP P = fc_plan(c, f);
    const long total = (long)B * P.n_ib * c->L * c->N;
    k_pack_fc_input<<<grid_for(total, 256), 256, 0, STREAM(stream)>>>(
        d_in, (const u64*)d_ve, (u64*)d_pt, P, B, c->L, c->logN, c->d_limb, c->t, c->r_t,
        c->t_inv);
    HE_CHECK_LAUNCH();
    return HE_OK;
}

// dense w_{beta,t}(X) (R17 on the n_ot x n_it sub-matrix), [n_ib][n_t][L][N]
__global__ void k_fc_weight_coeffs(const int32_t* __restrict__ W, u64* __restrict__ out, FcP P,
                                   int L, int logN, const he_limb* __restrict__ limbs) {
    const long N = 1L << logN;
    const long total = (long)P.n_ib * P.n_t * L * N;
    for (long idx = blockIdx.x * (long)blockDim.x + threadIdx.x; idx < total;
         idx += (long)gridDim.x * blockDim.x) {
        const int i = (int)(idx & (N - 1));
        const long r = idx >> logN;
        const int l = (int)(r % L);
        const long bt = r / L;
        const int tt = (int)(bt % P.n_t), beta = (int)(bt / P.n_t);
        long k, lp;
        if (i < P.n_ot) {
            k = i;                                                   // W_{k,0} X^k
            lp = 0;
        } else {
            const long d = N - i;                                    // = l' n_ot - k
            lp = (d + P.n_ot - 1) / P.n_ot;
            k = lp * P.n_ot - d;
        }
        const long row = (long)tt * P.n_ot + k, col = (long)beta * P.n_it + lp;
        long w = 0;
        if (lp < P.n_it && row < P.n_o && col < P.n_i) {
            w = W[row * P.n_i + col];
            if (lp) w = -w;                                          // -W_{k,l'}
        }
        const u64 q = limbs[l].q;
        out[idx] = w >= 0 ? (u64)w % q : q - ((u64)(-w) % q);
    }
}

// spectrum -> {w N^{-1}, Shoup}
__global__ void k_fc_finish_weights(const u64* __restrict__ spec, ulonglong2* __restrict__ wspec,
                                    long nlimbs, int L, int logN,
                                    const he_limb* __restrict__ limbs) {
    const long N = 1L << logN;
    for (long idx = blockIdx.x * (long)blockDim.x + threadIdx.x; idx < nlimbs * N;
         idx += (long)gridDim.x * blockDim.x) {
        const int l = (int)((idx >> logN) % L);
        const he_limb& Lm = limbs[l];
        const u64 w = csub(shoup_mul(spec[idx], Lm.ninv, Lm.ninv_p, Lm.q), Lm.q);
        wspec[idx] = make_ulonglong2(w, (u64)(((unsigned __int128)w << 64) / Lm.q));
    }
}

__global__ void k_fc_bias(const int32_t* __restrict__ bias, u64* __restrict__ bias_enc, int n_o,
                          int L, const he_limb* __restrict__ limbs, u64 t, u64 r_t,
                          u64 t_inv) {
    for (long idx = blockIdx.x * (long)blockDim.x + threadIdx.x; idx < (long)L * n_o;
         idx += (long)gridDim.x * blockDim.x) {
        const int l = (int)(idx / n_o), k = (int)(idx % n_o);
        long m = bias ? bias[k] : 0;
        long mt = m % (long)t;
        if (mt < 0) mt += t;
        bias_enc[idx] = enc_plain((u64)mt, limbs[l], t, r_t, t_inv);
    }
}

extern "C" size_t he_fc_wspec_bytes(const he_ctx* c, const he_fc_desc* f) {
    if (!fc_ok(c, f)) return 0;
    const FcP P = fc_plan(c, f);
    return sizeof(ulonglong2) * (size_t)P.n_ib * P.n_t * c->L * c->N;
}

extern "C" size_t he_fc_workspace_bytes(const he_ctx* c, const he_fc_desc* f, int B) {
    if (!fc_ok(c, f) || B < 0) return 0;
    const FcP P = fc_plan(c, f);
    return sizeof(u64) * (size_t)P.n_ib * std::max(std::max(B, 1), P.n_t) * c->L * c->N;
}

extern "C" he_status he_pack_fc_weights(const he_ctx* c, const he_fc_desc* f,
                                        const int32_t* d_W, const int32_t* d_bias,
                                        uint64_t* d_wspec, uint64_t* d_bias_enc, void* d_ws,
                                        size_t ws_bytes, void* stream) {
    if (!c || !f || !d_W || !d_wspec || !d_bias_enc || !d_ws) return HE_EINVAL;
    if (!fc_ok(c, f)) return HE_ESHAPE;
    const FcP P = fc_plan(c, f);
    const long nl = (long)P.n_ib * P.n_t * c->L;
    if (ws_bytes < sizeof(u64) * (size_t)nl * c->N) return HE_ENOMEM;
    cudaStream_t st = STREAM(stream);
    u64* ws = (u64*)d_ws;
    const long total = nl * c->N;
    k_fc_weight_coeffs<<<grid_for(total, 256), 256, 0, st>>>(d_W, ws, P, c->L, c->logN,
                                                             c->d_limb);
    HE_CHECK_LAUNCH();
    he_status s = launch_ntt_fwd(c, ws, ws, nl, 0, st);
    if (s != HE_OK) return s;
    k_fc_finish_weights<<<grid_for(total, 256), 256, 0, st>>>(ws, (ulonglong2*)d_wspec, nl, c->L,
                                                              c->logN, c->d_limb);
    HE_CHECK_LAUNCH();
    k_fc_bias<<<grid_for((long)c->L * f->n_o, 256), 256, 0, st>>>(
        d_bias, (u64*)d_bias_enc, f->n_o, c->L, c->d_limb, c->t, c->r_t, c->t_inv);
    HE_CHECK_LAUNCH();
    return HE_OK;
}

// Per (b, tile t, l): sum over input blocks of the pointwise products with
// the weight spectra, N-point inverse NTT (N^{-1} pre-folded), the tile's
// first coefficients + enc(bias) + enc(phi1) at outputs t n_ot + k.
template <bool DP>
__global__ void __launch_bounds__(1024)
k_fc_inv(const u64* __restrict__ spec, const ulonglong2* __restrict__ wspec,
         const u64* __restrict__ bias_enc, const u32* __restrict__ phi1, u64* __restrict__ out,
         FcP P, int L, int logN, const he_limb* __restrict__ limbs,
         const ulonglong2* __restrict__ twi_all, const double* __restrict__ twid_all, u64 t,
         u64 r_t, u64 t_inv) {
    extern __shared__ u64 sm[];
    double* smd = reinterpret_cast<double*>(sm);
    const int N = 1 << logN;
    const int l = blockIdx.x % L, bt = blockIdx.x / L;
    const int tt = bt % P.n_t, b = bt / P.n_t;
    const he_limb Lm = limbs[l];
    const u64 q = Lm.q, q2 = 2 * q;
    for (int i = threadIdx.x; i < N; i += blockDim.x) {
        double accd = 0.0;
        u64 acc = 0;
        for (int beta = 0; beta < P.n_ib; ++beta) {
            const u64 x = spec[(((size_t)b * P.n_ib + beta) * L + l) * N + i];
            const ulonglong2 w = __ldg(&wspec[(((size_t)beta * P.n_t + tt) * L + l) * N + i]);
            if (DP) accd = dp_reduce(accd + dp_mulmod(u2d(x), (double)w.x, Lm.qd, Lm.qinvd),
                                     Lm.qd, Lm.qinvd);
            else acc = csub(acc + shoup_mul(x, w.x, w.y, q), q2);          // [0, 2q)
        }
        if (DP) smd[PAD(i)] = accd;
        else sm[PAD(i)] = acc;
    }
    __syncthreads();
    const int k0 = tt * P.n_ot, nk = min(P.n_ot, P.n_o - k0);
    if (DP && HE_FC_PRUNE) {
        // Pruned inverse: only coefficients k < nk <= 2^kb leave.  A GS stage
        // v (pair distance 2^v) with v >= kb feeds those outputs only through
        // its sum outputs X + Y (no twiddle), so the transform runs stages
        // v < kb in full and each output is the plain sum
        //   out[k] = sum_m y[k + m 2^kb]   (y: after stage kb - 1),
        // a column sum instead of logN - kb stages of butterflies (config 4:
        // 7 of 14 stages' multiplications).
        int kb = 0;
        while ((1 << kb) < P.n_ot) ++kb;
        const double* twd = twid_all + (size_t)l * N;
        int lt = 0;
        for (; lt + 4 <= kb; lt += 4) {
            gs_pass_dp<4>(smd, 0, 1, logN, lt, 0, logN, twd, Lm.qd, Lm.qinvd);
            __syncthreads();
        }
        if (kb - lt == 1) gs_pass_dp<1>(smd, 0, 1, logN, lt, 0, logN, twd, Lm.qd, Lm.qinvd);
        else if (kb - lt == 2) gs_pass_dp<2>(smd, 0, 1, logN, lt, 0, logN, twd, Lm.qd, Lm.qinvd);
        else if (kb - lt == 3) gs_pass_dp<3>(smd, 0, 1, logN, lt, 0, logN, twd, Lm.qd, Lm.qinvd);
        if (kb > lt) __syncthreads();
        // column sums: thread (k, part) adds terms m = part, part + parts, ...
        // (each reduced to |.| <= q/2 + 2 first; 8 of them stay below 2^53)
        const int KN = 1 << kb, T = N >> kb;
        // (parts * KN <= blockDim <= 1024 words of partial sums; parts = 1
        //  reduces in place: element k is read only by its own thread)
        const int parts = min(T, max(1, (int)blockDim.x / KN));
        double* part_s = parts > 1 ? smd + padded_words(N) : smd;   // [parts][KN]
        for (int e = threadIdx.x; e < parts * KN; e += blockDim.x) {
            const int k = e & (KN - 1), pt = e >> kb;
            double acc = 0.0;
            int cnt = 0;
            for (int m = pt; m < T; m += parts) {
                acc += dp_reduce(smd[PAD(k + (m << kb))], Lm.qd, Lm.qinvd);
                if (++cnt == 8) { acc = dp_reduce(acc, Lm.qd, Lm.qinvd); cnt = 0; }
            }
            part_s[parts > 1 ? e : PAD(e)] = dp_reduce(acc, Lm.qd, Lm.qinvd);
        }
        __syncthreads();
        for (int k = threadIdx.x; k < nk; k += blockDim.x) {
            double acc = 0.0;
            for (int pt = 0; pt < parts; ++pt) {
                acc += part_s[parts > 1 ? pt * KN + k : PAD(k)];   // |.| <= q/2 + 2 each
                if ((pt & 7) == 7) acc = dp_reduce(acc, Lm.qd, Lm.qinvd);
            }
            u64 v = d2canon(acc, Lm.qd, Lm.qinvd);
            v = addmod(v, bias_enc[(size_t)l * P.n_o + k0 + k], q);
            if (phi1)
                v = addmod(v, enc_plain(phi1[(size_t)b * P.n_o + k0 + k], Lm, t, r_t, t_inv), q);
            out[((size_t)b * L + l) * P.n_o + k0 + k] = v;
        }
        return;
    }
    if (DP) gs_all_dp<3>(smd, 0, 1, logN, 0, logN, twid_all + (size_t)l * N, Lm.qd, Lm.qinvd);
    else gs_all<4>(sm, 0, 1, logN, 0, logN, twi_all + (size_t)l * N, q, q2);
    for (int k = threadIdx.x; k < nk; k += blockDim.x) {
        u64 v = DP ? d2canon(smd[PAD(k)], Lm.qd, Lm.qinvd) : csub(sm[PAD(k)], q);
        v = addmod(v, bias_enc[(size_t)l * P.n_o + k0 + k], q);
        if (phi1)
            v = addmod(v, enc_plain(phi1[(size_t)b * P.n_o + k0 + k], Lm, t, r_t, t_inv), q);
        out[((size_t)b * L + l) * P.n_o + k0 + k] = v;
    }
}

// N = 32768: a 2-CTA cluster per (b, t, l) as k_ntt_inv_split; only the
// tile's first coefficients leave the last (cross-half) stage.
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(512)
k_fc_inv_split(const u64* __restrict__ spec, const ulonglong2* __restrict__ wspec,
               const u64* __restrict__ bias_enc, const u32* __restrict__ phi1,
               u64* __restrict__ out, FcP P, int L, int logN,
               const he_limb* __restrict__ limbs, const ulonglong2* __restrict__ twi_all,
               u64 t, u64 r_t, u64 t_inv) {
    extern __shared__ u64 sm[];
    const int N = 1 << logN, NS = N >> 1;
    const int li = blockIdx.x >> 1, seg = blockIdx.x & 1;
    const int l = li % L, bt = li / L;
    const int tt = bt % P.n_t, b = bt / P.n_t;
    const he_limb Lm = limbs[l];
    const u64 q = Lm.q, q2 = 2 * q;
    const ulonglong2* twi = twi_all + (size_t)l * N;
    for (int i = threadIdx.x; i < NS; i += blockDim.x) {
        const int gi = seg * NS + i;
        u64 acc = 0;
        for (int beta = 0; beta < P.n_ib; ++beta) {
            const u64 x = spec[(((size_t)b * P.n_ib + beta) * L + l) * N + gi];
            const ulonglong2 w = __ldg(&wspec[(((size_t)beta * P.n_t + tt) * L + l) * N + gi]);
            acc = csub(acc + shoup_mul(x, w.x, w.y, q), q2);
        }
        sm[PAD(i)] = acc;
    }
    __syncthreads();
    gs_all<4>(sm, 0, 1, logN - 1, seg, logN, twi, q, q2);
    cg::cluster_group cl = cg::this_cluster();
    cl.sync();
    const u64* lo = seg ? cl.map_shared_rank(sm, 0) : sm;
    const u64* hi = seg ? sm : cl.map_shared_rank(sm, 1);
    const ulonglong2 w = twi[1];
    const int k0 = tt * P.n_ot, nk = min(P.n_ot, P.n_o - k0);
    for (int i = threadIdx.x; i < NS; i += blockDim.x) {
        const int k = seg * NS + i;
        if (k >= nk) break;
        const u64 x = lo[PAD(i)], y = hi[PAD(i)];
        u64 v = seg ? shoup_mul(x - y + q2, w.x, w.y, q) : csub(x + y, q2);
        v = csub(v, q);
        v = addmod(v, bias_enc[(size_t)l * P.n_o + k0 + k], q);
        if (phi1)
            v = addmod(v, enc_plain(phi1[(size_t)b * P.n_o + k0 + k], Lm, t, r_t, t_inv), q);
        out[((size_t)b * L + l) * P.n_o + k0 + k] = v;
    }
    cl.sync();                          // keep smem alive for the partner
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
    const FcP P = fc_plan(c, f);
    u64* spec = (u64*)d_ws;
    rec(ev, 0, st);
    he_status s = launch_ntt_fwd(c, (const u64*)d_c0, spec, (long)B * P.n_ib * c->L, 0, st);
    if (s != HE_OK) return s;
    rec(ev, 1, st);
    const unsigned nblk = (unsigned)((long)B * P.n_t * c->L);
    if (c->logN <= 14) {
        // (+ the pruned inverse's partial column sums, <= 1024 words)
        const size_t smem = sizeof(u64) * (padded_words(c->N) + (HE_FC_PRUNE ? 1024 : 0));
        auto kf = c->ntt_mode == 0 ? k_fc_inv<true> : k_fc_inv<false>;
        if (!set_smem(kf, smem)) return HE_ECUDA;
        kf<<<nblk, std::min(1024, std::max(32, (int)(c->N / 16))), smem, st>>>(
            spec, (const ulonglong2*)d_wspec, (const u64*)d_bias_enc, d_phi1, (u64*)d_out, P,
            c->L, c->logN, c->d_limb, c->d_tw_inv, c->d_twd_inv, c->t, c->r_t, c->t_inv);
    } else {
        const size_t smem = sizeof(u64) * padded_words(c->N / 2);
        if (!set_smem(k_fc_inv_split, smem)) return HE_ECUDA;
        k_fc_inv_split<<<2 * nblk, ntt_threads(c->N / 2), smem, st>>>(
            spec, (const ulonglong2*)d_wspec, (const u64*)d_bias_enc, d_phi1, (u64*)d_out, P,
            c->L, c->logN, c->d_limb, c->d_tw_inv, c->t, c->r_t, c->t_inv);
    }
    HE_CHECK_LAUNCH();
    rec(ev, 2, st);
    return HE_OK;
}

// ============================================================ wire format
// 50-bit packing, 4096 residues (3200 words) per CTA through shared memory:
// coalesced word loads/stores, per-element shifts.
static constexpr int PK_ELEMS = 4096, PK_WORDS = PK_ELEMS * 50 / 64;   // 3200
static constexpr u64 MASK50 = (1ull << 50) - 1;

__global__ void __launch_bounds__(256)
k_unpack50(const u64* __restrict__ in, u64* __restrict__ out, size_t n) {
    __shared__ u64 w[PK_WORDS + 1];
    const size_t e0 = (size_t)blockIdx.x * PK_ELEMS;
    const int ne = (int)min((size_t)PK_ELEMS, n - e0);
    const int nw = ne * 50 / 64;                 // ne multiple of 32 -> exact
    const u64* src = in + e0 / 64 * 50;
    for (int i = threadIdx.x; i < nw; i += blockDim.x) w[i] = src[i];
    if (threadIdx.x == 0) w[nw] = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < ne; i += blockDim.x) {
        const int bit = 50 * i, wi = bit >> 6, sh = bit & 63;
        u64 v = w[wi] >> sh;
        if (sh > 14) v |= w[wi + 1] << (64 - sh);
        out[e0 + i] = v & MASK50;
    }
}

__global__ void __launch_bounds__(256)
k_pack50(const u64* __restrict__ in, u64* __restrict__ out, size_t n) {
    __shared__ u64 x[PK_ELEMS + 2];
    const size_t e0 = (size_t)blockIdx.x * PK_ELEMS;
    const int ne = (int)min((size_t)PK_ELEMS, n - e0);
    const int nw = ne * 50 / 64;
    for (int i = threadIdx.x; i < ne; i += blockDim.x) x[i] = in[e0 + i] & MASK50;
    if (threadIdx.x < 2) x[ne + threadIdx.x] = 0;
    __syncthreads();
    u64* dst = out + e0 / 64 * 50;
    for (int wi = threadIdx.x; wi < nw; wi += blockDim.x) {
        const int lo = 64 * wi, i0 = lo / 50;
        u64 v = 0;
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            const int i = i0 + d, off = 50 * i - lo;      // bit of x_i's LSB in word
            if (off >= 64) break;
            v |= off >= 0 ? x[i] << off : x[i] >> (-off);
        }
        dst[wi] = v;
    }
}

extern "C" he_status he_residues_pack50(const uint64_t* d_in, size_t n, uint8_t* d_packed,
                                        void* stream) {
    if (n % 32) return HE_EINVAL;
    if (n == 0) return HE_OK;
    if (!d_in || !d_packed || ((uintptr_t)d_packed & 7)) return HE_EINVAL;
    k_pack50<<<(unsigned)((n + PK_ELEMS - 1) / PK_ELEMS), 256, 0, STREAM(stream)>>>(
        (const u64*)d_in, (u64*)d_packed, n);
    HE_CHECK_LAUNCH();
    return HE_OK;
}

extern "C" he_status he_residues_unpack50(const uint8_t* d_packed, size_t n, uint64_t* d_out,
                                          void* stream) {
    if (n % 32) return HE_EINVAL;
    if (n == 0) return HE_OK;
    if (!d_out || !d_packed || ((uintptr_t)d_packed & 7)) return HE_EINVAL;
    k_unpack50<<<(unsigned)((n + PK_ELEMS - 1) / PK_ELEMS), 256, 0, STREAM(stream)>>>(
        (const u64*)d_packed, (u64*)d_out, n);
    HE_CHECK_LAUNCH();
    return HE_OK;
}

// ================================================================ phi1
__global__ void k_phi1(u64 seed, size_t n, u32* __restrict__ out, u64 t) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
         i += (size_t)gridDim.x * blockDim.x) {
        u64 z = seed + (i + 1) * 0x9E3779B97F4A7C15ull;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        z ^= z >> 31;
        out[i] = (u32)(z % t);
    }
}

extern "C" he_status he_phi1_generate(const he_ctx* c, uint64_t seed, size_t n, uint32_t* d_phi1,
                                      void* stream) {
    if (!c) return HE_EINVAL;
    if (n == 0) return HE_OK;
    if (!d_phi1) return HE_EINVAL;
    k_phi1<<<grid_for((long)n, 256), 256, 0, STREAM(stream)>>>(seed, n, d_phi1, c->t);
    HE_CHECK_LAUNCH();
    return HE_OK;
}

// ================================================= client mirror path (§8 f)
__device__ __forceinline__ u64 int_to_res(long w, u64 q) {
    return w >= 0 ? (u64)w % q : q - 1 - ((u64)(-w) - 1) % q;
}

__global__ void k_residues_from_int(const int32_t* __restrict__ x, long n_polys, int L,
                                    int logN, const he_limb* __restrict__ limbs,
                                    u64* __restrict__ out) {
    const long N = 1L << logN;
    const long total = n_polys * L * N;
    for (long idx = blockIdx.x * (long)blockDim.x + threadIdx.x; idx < total;
         idx += (long)gridDim.x * blockDim.x) {
        const long k = idx & (N - 1), r = idx >> logN;
        const int l = (int)(r % L);
        const long i = r / L;
        out[idx] = int_to_res(x[i * N + k], limbs[l].q);
    }
}

// x[i][l][k] <- x[i][l][k] * y[(ybc ? 0 : i)][l][k] mod q_l (canonical in/out)
__global__ void k_pointwise_mul(u64* __restrict__ x, const u64* __restrict__ y, long nx,
                                int ybc, int L, int logN, const he_limb* __restrict__ limbs) {
    const long N = 1L << logN;
    const long total = nx * L * N;
    for (long idx = blockIdx.x * (long)blockDim.x + threadIdx.x; idx < total;
         idx += (long)gridDim.x * blockDim.x) {
        const long k = idx & (N - 1), r = idx >> logN;
        const int l = (int)(r % L);
        const long yi = ybc ? (long)l * N + k : idx;
        const he_limb& Lm = limbs[l];
        x[idx] = d2canon(dp_mulmod(u2d(x[idx]), u2d(y[yi]), Lm.qd, Lm.qinvd), Lm.qd, Lm.qinvd);
    }
}

// Negacyclic shift by +-t_n per output channel n (t_n of Eq. (7)):
//   dir = +1: out[n][beta][l][i] = (X^{t_n} in)[i] + e[n][beta][i]
//   dir = -1: out[n][beta][l][i] = (X^{-t_n} in)[i]
__global__ void k_negashift(const u64* __restrict__ in, const int32_t* __restrict__ e,
                            u64* __restrict__ out, PlanDev P, int dir, int L, int logN,
                            const he_limb* __restrict__ limbs) {
    const long N = 1L << logN;
    const long total = (long)P.c_o * P.n_ib * L * N;
    for (long idx = blockIdx.x * (long)blockDim.x + threadIdx.x; idx < total;
         idx += (long)gridDim.x * blockDim.x) {
        const long i = idx & (N - 1), r = idx >> logN;
        const long nb = r / L;
        const int l = (int)(r % L), n = (int)(nb / P.n_ib);
        const long tn = (long)(n % P.c_ob) * P.step;
        const u64 q = limbs[l].q;
        long src = dir > 0 ? i - tn : i + tn;
        bool neg = false;
        if (src < 0) { src += N; neg = true; }
        if (src >= N) { src -= N; neg = true; }
        u64 v = in[(r << logN) + src];
        if (neg && v) v = q - v;
        if (e) v = addmod(v, int_to_res(e[nb * N + i], q), q);
        out[idx] = v;
    }
}

extern "C" size_t he_server_p_workspace_bytes(const he_ctx* c, const he_conv_plan* p) {
    if (!c || !p) return 0;
    return sizeof(u64) * ((size_t)p->d.c_o * p->n_ib + 1) * c->L * c->N;
}

extern "C" he_status he_server_init_p(const he_ctx* c, const he_conv_plan* p,
                                      const int32_t* d_w, const uint64_t* d_a,
                                      const int32_t* d_ef, uint64_t* d_p, void* d_ws,
                                      size_t ws_bytes, void* stream) {
    if (!c || !p || !d_w || !d_a || !d_p || !d_ws) return HE_EINVAL;
    if (!plan_ok(c, p)) return HE_ESHAPE;
    if (ws_bytes < he_server_p_workspace_bytes(c, p)) return HE_ENOMEM;
    cudaStream_t st = STREAM(stream);
    const PlanDev P = plan_dev(p);
    const long nf = (long)P.c_o * P.n_ib;
    u64* fa = (u64*)d_ws;                          // [c_o][n_ib][L][N]
    u64* aspec = fa + nf * c->L * c->N;            // [L][N]
    const long total = nf * c->L * c->N;
    k_pack_filter_coeffs<<<grid_for(total, 256), 256, 0, st>>>(d_w, fa, P, c->L, c->logN,
                                                                c->d_limb);
    HE_CHECK_LAUNCH();
    he_status s = launch_ntt_fwd(c, fa, fa, nf * c->L, 0, st);
    if (s != HE_OK) return s;
    s = launch_ntt_fwd(c, (const u64*)d_a, aspec, c->L, 0, st);
    if (s != HE_OK) return s;
    k_pointwise_mul<<<grid_for(total, 256), 256, 0, st>>>(fa, aspec, nf, 1, c->L, c->logN,
                                                           c->d_limb);
    HE_CHECK_LAUNCH();
    s = launch_ntt_inv(c, fa, fa, nf * c->L, st);                 // f a (unshifted)
    if (s != HE_OK) return s;
    k_negashift<<<grid_for(total, 256), 256, 0, st>>>(fa, d_ef, (u64*)d_p, P, +1, c->L,
                                                       c->logN, c->d_limb);
    HE_CHECK_LAUNCH();
    return HE_OK;
}

extern "C" he_status he_pack_client_p(const he_ctx* c, const he_conv_plan* p,
                                      const uint64_t* d_p, uint64_t* d_pspec, void* d_ws,
                                      size_t ws_bytes, void* stream) {
    if (!c || !p || !d_p || !d_pspec || !d_ws) return HE_EINVAL;
    if (!plan_ok(c, p) || p->k_u != p->s) return HE_ESHAPE;     // dense plan required
    if (ws_bytes < he_pack_filters_workspace_bytes(c, p)) return HE_ENOMEM;
    cudaStream_t st = STREAM(stream);
    const PlanDev P = plan_dev(p);
    u64* ws = (u64*)d_ws;
    const long total = (long)P.c_o * P.n_ib * c->L * c->N;
    k_negashift<<<grid_for(total, 256), 256, 0, st>>>((const u64*)d_p, nullptr, ws, P, -1,
                                                       c->L, c->logN, c->d_limb);
    HE_CHECK_LAUNCH();
    return finish_filter_spectra(c, P, ws, d_pspec, st);
}

extern "C" he_status he_residues_from_int(const he_ctx* c, const int32_t* d_x, long n_polys,
                                          uint64_t* d_out, void* stream) {
    if (!c || n_polys < 0) return HE_EINVAL;
    if (n_polys == 0) return HE_OK;
    if (!d_x || !d_out) return HE_EINVAL;
    const long total = n_polys * c->L * c->N;
    k_residues_from_int<<<grid_for(total, 256), 256, 0, STREAM(stream)>>>(
        d_x, n_polys, c->L, c->logN, c->d_limb, (u64*)d_out);
    HE_CHECK_LAUNCH();
    return HE_OK;
}

extern "C" he_status he_poly_mul(const he_ctx* c, const uint64_t* d_x, const uint64_t* d_y,
                                 int B, int y_batch, uint64_t* d_out, void* d_ws,
                                 size_t ws_bytes, void* stream) {
    if (!c || B < 0 || (y_batch != 1 && y_batch != B)) return HE_EINVAL;
    if (B == 0) return HE_OK;
    if (!d_x || !d_y || !d_out || !d_ws) return HE_EINVAL;
    if (ws_bytes < sizeof(u64) * (size_t)y_batch * c->L * c->N) return HE_ENOMEM;
    cudaStream_t st = STREAM(stream);
    u64* yspec = (u64*)d_ws;
    he_status s = launch_ntt_fwd(c, (const u64*)d_y, yspec, (long)y_batch * c->L, 0, st);
    if (s != HE_OK) return s;
    s = launch_ntt_fwd(c, (const u64*)d_x, (u64*)d_out, (long)B * c->L, 0, st);
    if (s != HE_OK) return s;
    const long total = (long)B * c->L * c->N;
    k_pointwise_mul<<<grid_for(total, 256), 256, 0, st>>>((u64*)d_out, yspec, B,
                                                           y_batch == 1 && B > 1, c->L,
                                                           c->logN, c->d_limb);
    HE_CHECK_LAUNCH();
    return launch_ntt_inv(c, (u64*)d_out, (u64*)d_out, (long)B * c->L, st);
}

// Decryption constants: y_j = r_j * ((Q/q_j)^{-1} mod q_j) (Shoup pair).
struct DecConst {
    u64 inv[64], invp[64];
};

__global__ void k_decrypt_round(const u64* __restrict__ c0r, const u64* __restrict__ c1r,
                                long n_polys, long len, int L,
                                const he_limb* __restrict__ limbs, DecConst dc, u64 t,
                                u32* __restrict__ m) {
    const long total = n_polys * len;
    const double td = (double)t;
    for (long idx = blockIdx.x * (long)blockDim.x + threadIdx.x; idx < total;
         idx += (long)gridDim.x * blockDim.x) {
        const long i = idx / len, k = idx - i * len;
        const u64* r0 = c0r + i * L * len + k;
        const u64* r1 = c1r ? c1r + i * L * len + k : nullptr;
        u64 ai = 0;
        double fr = 0.0;
        for (int j = 0; j < L; ++j) {
            const u64 q = limbs[j].q;
            u64 r = r0[(long)j * len];
            if (r1) r = addmod(r, r1[(long)j * len], q);
            const u64 y = csub(shoup_mul(r, dc.inv[j], dc.invp[j], q), q);
            // y t = a q + b, 0 <= b < q  (y t < 2^82; a < t)
            long long a = (long long)((double)y * td / (double)q);
            long long b = (long long)(y * t - (u64)a * q);          // exact mod 2^64
            while (b < 0) { b += (long long)q; --a; }
            while (b >= (long long)q) { b -= (long long)q; ++a; }
            ai += (u64)a;
            fr += (double)b / (double)q;
        }
        m[idx] = (u32)((ai + (u64)rint(fr)) % t);
    }
}

static u64 mulmod_h(u64 a, u64 b, u64 q) { return (u64)((unsigned __int128)a * b % q); }
static u64 powmod_h(u64 a, u64 e, u64 q) {
    u64 r = 1;
    for (; e; e >>= 1, a = mulmod_h(a, a, q))
        if (e & 1) r = mulmod_h(r, a, q);
    return r;
}

extern "C" he_status he_decrypt_round(const he_ctx* c, const uint64_t* d_c0r,
                                      const uint64_t* d_c1r, long n_polys, long len,
                                      uint32_t* d_m, void* stream) {
    if (!c || n_polys < 0 || len < 0) return HE_EINVAL;
    if (n_polys == 0 || len == 0) return HE_OK;
    if (!d_c0r || !d_m) return HE_EINVAL;
    DecConst dc;
    memset(&dc, 0, sizeof(dc));
    for (int j = 0; j < c->L; ++j) {
        const u64 q = c->q_host[j];
        u64 qh = 1;                                    // (Q / q_j) mod q_j
        for (int i = 0; i < c->L; ++i)
            if (i != j) qh = mulmod_h(qh, c->q_host[i] % q, q);
        dc.inv[j] = powmod_h(qh, q - 2, q);
        dc.invp[j] = (u64)(((unsigned __int128)dc.inv[j] << 64) / q);
    }
    const long total = n_polys * len;
    k_decrypt_round<<<grid_for(total, 256), 256, 0, STREAM(stream)>>>(
        (const u64*)d_c0r, (const u64*)d_c1r, n_polys, len, c->L, c->d_limb, dc, c->t, d_m);
    HE_CHECK_LAUNCH();
    return HE_OK;
}

// ====================================================== modulus switching
// x' = round(x / P) mod q_j (j < Lk), P = q_Lk ... q_{L-1} (reading R28).
// With y_i = x_i ((P/p_i)^{-1} mod p_i) for the dropped limbs i,
//   round(x / P) = (x - sum_i y_i P/p_i) / P + round(sum_i y_i / p_i),
// so x'_j = (x_j - sum_i y_i [P/p_i]_{q_j}) [P^{-1}]_{q_j} + u  (mod q_j),
// u = rint(sum_i y_i / p_i) in FP64 (the exact rounding differs only when
// the fraction is within ~L 2^-52 of one half).  Constants: dinv[i],
// pinv[j], m[i * Lk + j] = [P/p_i]_{q_j}.
struct MsConst {
    int Lk, Ld;
    u64 v[400];           // dinv[Ld], pinv[Lk], m[Ld * Lk]
};

__global__ void __launch_bounds__(256)
k_mod_switch(const u64* __restrict__ in, u64* __restrict__ out, long n_polys, long len, int L,
             const he_limb* __restrict__ limbs, MsConst C) {
    const long total = n_polys * len;
    const u64* dinv = C.v;
    const u64* pinv = C.v + C.Ld;
    const u64* mm = C.v + C.Ld + C.Lk;
    for (long idx = blockIdx.x * (long)blockDim.x + threadIdx.x; idx < total;
         idx += (long)gridDim.x * blockDim.x) {
        const long i = idx / len, k = idx - i * len;
        const u64* x = in + i * L * len + k;
        u64* o = out + i * C.Lk * len + k;
        double u = 0.0;
#pragma unroll 1
        for (int j = 0; j < C.Lk; ++j) {            // y_d recomputed per kept limb
            const he_limb& Qm = limbs[j];
            double acc = 0.0, fr = 0.0;
#pragma unroll 4
            for (int d = 0; d < C.Ld; ++d) {
                const he_limb& Pm = limbs[C.Lk + d];
                const u64 y = d2canon(dp_mulmod(u2d(x[(long)(C.Lk + d) * len]), u2d(dinv[d]),
                                                Pm.qd, Pm.qinvd), Pm.qd, Pm.qinvd);
                if (j == 0) fr += (double)y * Pm.qinvd;
                acc = dp_reduce(acc + dp_mulmod(u2d(y), u2d(mm[d * C.Lk + j]), Qm.qd, Qm.qinvd),
                                Qm.qd, Qm.qinvd);
            }
            if (j == 0) u = rint(fr);
            const double dif = u2d(x[(long)j * len]) - acc;                 // |.| < 1.5 q
            const double v = dp_mulmod(dif, u2d(pinv[j]), Qm.qd, Qm.qinvd) + u;
            o[(long)j * len] = d2canon(v, Qm.qd, Qm.qinvd);
        }
    }
}

extern "C" he_status he_mod_switch(const he_ctx* c, const uint64_t* d_in, long n_polys,
                                   long len, int L_keep, uint64_t* d_out, void* stream) {
    if (!c || n_polys < 0 || len < 0 || L_keep < 1 || L_keep > c->L) return HE_EINVAL;
    if (n_polys == 0 || len == 0) return HE_OK;
    if (!d_in || !d_out) return HE_EINVAL;
    MsConst C;
    memset(&C, 0, sizeof(C));
    C.Lk = L_keep;
    C.Ld = c->L - L_keep;
    if (C.Ld > 16 || C.Ld + C.Lk + C.Ld * C.Lk > 400) return HE_EPARAM;
    const u64* q = c->q_host;
    for (int d = 0; d < C.Ld; ++d) {            // (P/p_d)^{-1} mod p_d
        const u64 p = q[C.Lk + d];
        u64 r = 1;
        for (int e = 0; e < C.Ld; ++e)
            if (e != d) r = mulmod_h(r, q[C.Lk + e] % p, p);
        C.v[d] = powmod_h(r, p - 2, p);
    }
    for (int j = 0; j < C.Lk; ++j) {            // P^{-1} mod q_j
        u64 r = 1;
        for (int e = 0; e < C.Ld; ++e) r = mulmod_h(r, q[C.Lk + e] % q[j], q[j]);
        C.v[C.Ld + j] = powmod_h(r, q[j] - 2, q[j]);
    }
    for (int d = 0; d < C.Ld; ++d)              // [P/p_d]_{q_j}
        for (int j = 0; j < C.Lk; ++j) {
            u64 r = 1;
            for (int e = 0; e < C.Ld; ++e)
                if (e != d) r = mulmod_h(r, q[C.Lk + e] % q[j], q[j]);
            C.v[C.Ld + C.Lk + d * C.Lk + j] = r;
        }
    const long total = n_polys * len;
    k_mod_switch<<<grid_for(total, 256), 256, 0, STREAM(stream)>>>(
        (const u64*)d_in, (u64*)d_out, n_polys, len, c->L, c->d_limb, C);
    HE_CHECK_LAUNCH();
    return HE_OK;
}

// ============================================ chained pipeline (§8(f), R29)
// Public-key mask of the c0-only encryption, Eq. (1):
// ve = v b + e0 per polynomial, v and e0 small signed integers.
__global__ void k_add_small(u64* __restrict__ x, const int32_t* __restrict__ e, long n_polys,
                            int L, int logN, const he_limb* __restrict__ limbs) {
    const long N = 1L << logN;
    const long total = n_polys * L * N;
    for (long idx = blockIdx.x * (long)blockDim.x + threadIdx.x; idx < total;
         idx += (long)gridDim.x * blockDim.x) {
        const long k = idx & (N - 1), r = idx >> logN;
        const int l = (int)(r % L);
        const u64 q = limbs[l].q;
        x[idx] = addmod(x[idx], int_to_res(e[(r / L) * N + k], q), q);
    }
}

extern "C" he_status he_pk_mask(const he_ctx* c, const int32_t* d_v, const int32_t* d_e,
                                long n_polys, const uint64_t* d_b, uint64_t* d_ve, void* d_ws,
                                size_t ws_bytes, void* stream) {
    if (!c || n_polys < 0) return HE_EINVAL;
    if (n_polys == 0) return HE_OK;
    if (!d_v || !d_b || !d_ve || !d_ws) return HE_EINVAL;
    if (ws_bytes < sizeof(u64) * (size_t)c->L * c->N) return HE_ENOMEM;
    cudaStream_t st = STREAM(stream);
    const long total = n_polys * c->L * c->N;
    k_residues_from_int<<<grid_for(total, 256), 256, 0, st>>>(d_v, n_polys, c->L, c->logN,
                                                              c->d_limb, (u64*)d_ve);
    HE_CHECK_LAUNCH();
    u64* bspec = (u64*)d_ws;
    he_status s = launch_ntt_fwd(c, (const u64*)d_b, bspec, c->L, 0, st);
    if (s != HE_OK) return s;
    s = launch_ntt_fwd(c, (const u64*)d_ve, (u64*)d_ve, n_polys * c->L, 0, st);
    if (s != HE_OK) return s;
    k_pointwise_mul<<<grid_for(total, 256), 256, 0, st>>>((u64*)d_ve, bspec, n_polys, 1, c->L,
                                                           c->logN, c->d_limb);
    HE_CHECK_LAUNCH();
    s = launch_ntt_inv(c, (u64*)d_ve, (u64*)d_ve, n_polys * c->L, st);
    if (s != HE_OK) return s;
    if (d_e) {
        k_add_small<<<grid_for(total, 256), 256, 0, st>>>((u64*)d_ve, d_e, n_polys, c->L,
                                                           c->logN, c->d_limb);
        HE_CHECK_LAUNCH();
    }
    return HE_OK;
}

// Stub between layers (R29): decrypted compact slots -> next layer image.
__global__ void k_relu_requant(const u32* __restrict__ m, const u32* __restrict__ phi1,
                               PlanDev P, int B, int logN, u64 t, int shift, int qmax,
                               int32_t* __restrict__ img) {
    const long N = 1L << logN;
    const long total = (long)B * P.n_ob * P.n_valid;
    for (long idx = blockIdx.x * (long)blockDim.x + threadIdx.x; idx < total;
         idx += (long)gridDim.x * blockDim.x) {
        const int v = (int)(idx % P.n_valid);
        const long bo = idx / P.n_valid;
        const int ob = (int)(bo % P.n_ob), b = (int)(bo / P.n_ob);
        const int nl = v % P.c_ob, Pq = v / P.c_ob;
        const int Lc = Pq % P.h_o, Kr = Pq / P.h_o;
        const int n = ob * P.c_ob + nl;
        if (n >= P.c_o) continue;
        long x = (long)m[idx];
        if (phi1) {
            const long i = (long)P.s * (P.stride * Kr * (long)P.h_p + P.stride * Lc) +
                           (long)nl * P.step;
            x -= (long)phi1[bo * N + i];
            if (x < 0) x += (long)t;
        }
        if (x > (long)(t / 2)) x -= (long)t;                  // centered mod t
        const long y = x > 0 ? min((long)qmax, x >> shift) : 0;
        img[(((long)b * P.c_o + n) * P.w_o + Kr) * P.h_o + Lc] = (int32_t)y;
    }
}

extern "C" he_status he_relu_requant(const he_ctx* c, const he_conv_plan* p, const uint32_t* d_m,
                                     int B, const uint32_t* d_phi1, int shift, int qmax,
                                     int32_t* d_img, void* stream) {
    if (!c || !p || B < 0 || shift < 0 || shift > 62 || qmax < 0) return HE_EINVAL;
    if (!plan_ok(c, p)) return HE_ESHAPE;
    if (B == 0) return HE_OK;
    if (!d_m || !d_img) return HE_EINVAL;
    const PlanDev P = plan_dev(p);
    const long total = (long)B * P.n_ob * P.n_valid;
    k_relu_requant<<<grid_for(total, 256), 256, 0, STREAM(stream)>>>(
        d_m, d_phi1, P, B, c->logN, c->t, shift, qmax, d_img);
    HE_CHECK_LAUNCH();
    return HE_OK;
}

__global__ void k_avgpool(const int32_t* __restrict__ x, long rows, int hw,
                          int32_t* __restrict__ out) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    for (long r = warp; r < rows; r += nw) {
        long sacc = 0;
        for (int i = lane; i < hw; i += 32) sacc += x[r * hw + i];
        for (int o = 16; o; o >>= 1) sacc += __shfl_xor_sync(0xffffffffu, sacc, o);
        if (lane == 0) {
            long q = sacc / hw;
            if (sacc % hw != 0 && sacc < 0) --q;              // floor
            out[r] = (int32_t)q;
        }
    }
}

extern "C" he_status he_avgpool(const int32_t* d_x, long rows, int hw, int32_t* d_out,
                                void* stream) {
    if (rows < 0 || hw < 1) return HE_EINVAL;
    if (rows == 0) return HE_OK;
    if (!d_x || !d_out) return HE_EINVAL;
    k_avgpool<<<grid_for(rows * 32, 256), 256, 0, STREAM(stream)>>>(d_x, rows, hw, d_out);
    HE_CHECK_LAUNCH();
    return HE_OK;
}

// FC client mirror path (Alg. 2 Lines 5-6 and 16-17):
// p_{beta,t} = w_{beta,t} a + e, and its spectra in the he_pack_fc_weights
// format so that he_fc(vs, pspec, zero bias, NULL) gives c1^r.
extern "C" size_t he_fc_server_p_workspace_bytes(const he_ctx* c, const he_fc_desc* f) {
    if (!fc_ok(c, f)) return 0;
    const FcP P = fc_plan(c, f);
    return sizeof(u64) * ((size_t)P.n_ib * P.n_t + 1) * c->L * c->N;
}

extern "C" he_status he_fc_server_init_p(const he_ctx* c, const he_fc_desc* f, const int32_t* d_W,
                                         const uint64_t* d_a, const int32_t* d_e, uint64_t* d_p,
                                         void* d_ws, size_t ws_bytes, void* stream) {
    if (!c || !f || !d_W || !d_a || !d_p || !d_ws) return HE_EINVAL;
    if (!fc_ok(c, f)) return HE_ESHAPE;
    if (ws_bytes < he_fc_server_p_workspace_bytes(c, f)) return HE_ENOMEM;
    cudaStream_t st = STREAM(stream);
    const FcP P = fc_plan(c, f);
    const long nl = (long)P.n_ib * P.n_t * c->L, total = nl * c->N;
    u64* aspec = (u64*)d_ws;
    u64* wp = (u64*)d_p;
    k_fc_weight_coeffs<<<grid_for(total, 256), 256, 0, st>>>(d_W, wp, P, c->L, c->logN,
                                                             c->d_limb);
    HE_CHECK_LAUNCH();
    he_status s = launch_ntt_fwd(c, wp, wp, nl, 0, st);
    if (s != HE_OK) return s;
    s = launch_ntt_fwd(c, (const u64*)d_a, aspec, c->L, 0, st);
    if (s != HE_OK) return s;
    k_pointwise_mul<<<grid_for(total, 256), 256, 0, st>>>(wp, aspec, (long)P.n_ib * P.n_t, 1,
                                                           c->L, c->logN, c->d_limb);
    HE_CHECK_LAUNCH();
    s = launch_ntt_inv(c, wp, wp, nl, st);
    if (s != HE_OK) return s;
    if (d_e) {
        k_add_small<<<grid_for(total, 256), 256, 0, st>>>(wp, d_e, (long)P.n_ib * P.n_t, c->L,
                                                           c->logN, c->d_limb);
        HE_CHECK_LAUNCH();
    }
    return HE_OK;
}

extern "C" he_status he_pack_fc_client_p(const he_ctx* c, const he_fc_desc* f,
                                         const uint64_t* d_p, uint64_t* d_pspec, void* d_ws,
                                         size_t ws_bytes, void* stream) {
    if (!c || !f || !d_p || !d_pspec || !d_ws) return HE_EINVAL;
    if (!fc_ok(c, f)) return HE_ESHAPE;
    const FcP P = fc_plan(c, f);
    const long nl = (long)P.n_ib * P.n_t * c->L;
    if (ws_bytes < sizeof(u64) * (size_t)nl * c->N) return HE_ENOMEM;
    cudaStream_t st = STREAM(stream);
    u64* ws = (u64*)d_ws;
    he_status s = launch_ntt_fwd(c, (const u64*)d_p, ws, nl, 0, st);
    if (s != HE_OK) return s;
    k_fc_finish_weights<<<grid_for(nl * c->N, 256), 256, 0, st>>>(ws, (ulonglong2*)d_pspec, nl,
                                                                  c->L, c->logN, c->d_limb);
    HE_CHECK_LAUNCH();
    return HE_OK;
}

// FC stub (R29): logits = centered((m - phi1) mod t).
__global__ void k_unmask(const u32* __restrict__ m, const u32* __restrict__ phi1, long n, u64 t,
                         int32_t* __restrict__ out) {
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n;
         i += (long)gridDim.x * blockDim.x) {
        long x = (long)m[i] - (phi1 ? (long)phi1[i] : 0);
        if (x < 0) x += (long)t;
        if (x > (long)(t / 2)) x -= (long)t;
        out[i] = (int32_t)x;
    }
}

extern "C" he_status he_unmask(const he_ctx* c, const uint32_t* d_m, const uint32_t* d_phi1,
                               long n, int32_t* d_out, void* stream) {
    if (!c || n < 0) return HE_EINVAL;
    if (n == 0) return HE_OK;
    if (!d_m || !d_out) return HE_EINVAL;
    k_unmask<<<grid_for(n, 256), 256, 0, STREAM(stream)>>>(d_m, d_phi1, n, c->t, d_out);
    HE_CHECK_LAUNCH();
    return HE_OK;
}

// ====================================== sparse c0 upload (protocol extension)
// The conv reads c0 only on the columns u < k_u of each fold group (DESIGN.md
// §4), so the client can send just those: [B][n_ib][L][M][k_u].
__global__ void k_c0_cols(const u64* __restrict__ in, u64* __restrict__ out, long npoly, int logN,
                          int logs, int Ku, int dir) {
    const long N = 1L << logN;
    const int s = 1 << logs, M = (int)(N >> logs);
    const long per = (long)M * Ku;
    const long total = npoly * (dir ? N : per);
    for (long idx = blockIdx.x * (long)blockDim.x + threadIdx.x; idx < total;
         idx += (long)gridDim.x * blockDim.x) {
        if (dir == 0) {                                         // compact: gather
            const long pl = idx / per, r = idx - pl * per;
            const long g = r / Ku, u = r - g * Ku;
            out[idx] = in[pl * N + g * s + u];
        } else {                                                // expand: scatter + zeros
            const long pl = idx >> logN, i = idx & (N - 1);
            const int u = (int)(i & (s - 1));
            out[idx] = u < Ku ? in[pl * per + (i >> logs) * Ku + u] : 0;
        }
    }
}

extern "C" he_status he_c0_compact(const he_ctx* c, const he_conv_plan* p, const uint64_t* d_c0,
                                   int B, uint64_t* d_c0c, void* stream) {
    if (!c || !p || B < 0) return HE_EINVAL;
    if (!plan_ok(c, p)) return HE_ESHAPE;
    if (B == 0) return HE_OK;
    if (!d_c0 || !d_c0c) return HE_EINVAL;
    const PlanDev P = plan_dev(p);
    const long npoly = (long)B * P.n_ib * c->L;
    k_c0_cols<<<grid_for(npoly * (c->N >> P.logs) * P.Ku, 256), 256, 0, STREAM(stream)>>>(
        (const u64*)d_c0, (u64*)d_c0c, npoly, c->logN, P.logs, P.Ku, 0);
    HE_CHECK_LAUNCH();
    return HE_OK;
}

extern "C" he_status he_c0_expand(const he_ctx* c, const he_conv_plan* p, const uint64_t* d_c0c,
                                  int B, uint64_t* d_c0, void* stream) {
    if (!c || !p || B < 0) return HE_EINVAL;
    if (!plan_ok(c, p)) return HE_ESHAPE;
    if (B == 0) return HE_OK;
    if (!d_c0 || !d_c0c) return HE_EINVAL;
    const PlanDev P = plan_dev(p);
    const long npoly = (long)B * P.n_ib * c->L;
    k_c0_cols<<<grid_for(npoly * c->N, 256), 256, 0, STREAM(stream)>>>(
        (const u64*)d_c0c, (u64*)d_c0, npoly, c->logN, P.logs, P.Ku, 1);
    HE_CHECK_LAUNCH();
    return HE_OK;
}

// ============================================== a2 debug export (parity)
extern "C" he_status he_filter_coeffs(const he_ctx* c, const he_conv_plan* p, const int32_t* d_w,
                                      int shifted, uint64_t* d_f, void* d_ws, size_t ws_bytes,
                                      void* stream) {
    if (!c || !p || !d_w || !d_f) return HE_EINVAL;
    if (!plan_ok(c, p)) return HE_ESHAPE;
    cudaStream_t st = STREAM(stream);
    const PlanDev P = plan_dev(p);
    const long total = (long)P.c_o * P.n_ib * c->L * c->N;
    if (!shifted) {
        k_pack_filter_coeffs<<<grid_for(total, 256), 256, 0, st>>>(d_w, (u64*)d_f, P, c->L,
                                                                    c->logN, c->d_limb);
        HE_CHECK_LAUNCH();
        return HE_OK;
    }
    if (!d_ws) return HE_EINVAL;
    if (ws_bytes < sizeof(u64) * (size_t)total) return HE_ENOMEM;
    k_pack_filter_coeffs<<<grid_for(total, 256), 256, 0, st>>>(d_w, (u64*)d_ws, P, c->L,
                                                                c->logN, c->d_limb);
    HE_CHECK_LAUNCH();
    k_negashift<<<grid_for(total, 256), 256, 0, st>>>((const u64*)d_ws, nullptr, (u64*)d_f, P,
                                                       +1, c->L, c->logN, c->d_limb);
    HE_CHECK_LAUNCH();
    return HE_OK;
}

// ============================== unfolded reference path (ablation of the fold)
// Alg. 1 Lines 14-17 computed literally: every c0_beta x f_beta^{(n)} as a
// full N-point NTT-domain product, an N-point inverse per (b, n, l), then the
// slots s j + t_n extracted (SURVEY §8(a) "plain variant").  Same output as
// he_conv; kept to measure what the fold and the incomplete transform save.
__global__ void k_mac_plain(const u64* __restrict__ C, const u64* __restrict__ F,
                            u64* __restrict__ P, PlanDev Pd, int B, int L, int logN,
                            const he_limb* __restrict__ limbs) {
    const long N = 1L << logN;
    const long total = (long)B * Pd.c_o * L * N;
    for (long idx = blockIdx.x * (long)blockDim.x + threadIdx.x; idx < total;
         idx += (long)gridDim.x * blockDim.x) {
        const long k = idx & (N - 1), r = idx >> logN;
        const int l = (int)(r % L);
        const long bn = r / L;
        const int n = (int)(bn % Pd.c_o), b = (int)(bn / Pd.c_o);
        const he_limb& Lm = limbs[l];
        double acc = 0.0;
        for (int beta = 0; beta < Pd.n_ib; ++beta) {
            const u64 x = C[(((long)b * Pd.n_ib + beta) * L + l) * N + k];
            const u64 y = F[(((long)n * Pd.n_ib + beta) * L + l) * N + k];
            acc = dp_reduce(acc + dp_mulmod(u2d(x), u2d(y), Lm.qd, Lm.qinvd), Lm.qd, Lm.qinvd);
        }
        P[idx] = d2canon(acc, Lm.qd, Lm.qinvd);
    }
}

__global__ void k_extract_plain(const u64* __restrict__ P, const u32* __restrict__ phi1,
                                u64* __restrict__ out, PlanDev Pd, int B, int L, int logN,
                                const he_limb* __restrict__ limbs, const u64* __restrict__ enc_tab,
                                u64 t, u64 r_t, u64 t_inv) {
    const long N = 1L << logN;
    const long total = (long)B * Pd.n_ob * L * N;
    for (long idx = blockIdx.x * (long)blockDim.x + threadIdx.x; idx < total;
         idx += (long)gridDim.x * blockDim.x) {
        const long i = idx & (N - 1), r = idx >> logN;
        const int l = (int)(r % L);
        const long bo = r / L;
        const int ob = (int)(bo % Pd.n_ob), b = (int)(bo / Pd.n_ob);
        const int u = (int)(i & (Pd.s - 1));
        const int nl = u / Pd.step, n = ob * Pd.c_ob + nl;
        u64 v = 0;
        if (u == nl * Pd.step && nl < Pd.c_ob && n < Pd.c_o)
            v = P[(((long)b * Pd.c_o + n) * L + l) * N + (i - u)];
        const he_limb& Lm = limbs[l];
        if (phi1) v = addmod(v, enc_lookup(enc_tab, l, t, phi1[bo * N + i], Lm, r_t, t_inv), Lm.q);
        out[idx] = v;
    }
}

extern "C" size_t he_conv_plain_workspace_bytes(const he_ctx* c, const he_conv_plan* p, int B) {
    if (!c || !p || B < 0) return 0;
    return sizeof(u64) * (size_t)std::max(B, 1) * (p->n_ib + p->d.c_o) * c->L * c->N;
}

extern "C" he_status he_pack_filters_plain(const he_ctx* c, const he_conv_plan* p,
                                           const int32_t* d_w, uint64_t* d_fplain, void* stream) {
    if (!c || !p || !d_w || !d_fplain) return HE_EINVAL;
    if (!plan_ok(c, p)) return HE_ESHAPE;
    cudaStream_t st = STREAM(stream);
    const PlanDev P = plan_dev(p);
    const long total = (long)P.c_o * P.n_ib * c->L * c->N;
    k_pack_filter_coeffs<<<grid_for(total, 256), 256, 0, st>>>(d_w, (u64*)d_fplain, P, c->L,
                                                                c->logN, c->d_limb);
    HE_CHECK_LAUNCH();
    return launch_ntt_fwd(c, (u64*)d_fplain, (u64*)d_fplain, (long)P.c_o * P.n_ib * c->L, 0, st);
}

extern "C" he_status he_conv_plain(const he_ctx* c, const he_conv_plan* p, const uint64_t* d_c0,
                                   int B, const uint64_t* d_fplain, const uint32_t* d_phi1,
                                   uint64_t* d_out, void* d_ws, size_t ws_bytes, void* stream) {
    if (!c || !p || B < 0) return HE_EINVAL;
    if (!plan_ok(c, p)) return HE_ESHAPE;
    if (B == 0) return HE_OK;
    if (!d_c0 || !d_fplain || !d_out || !d_ws) return HE_EINVAL;
    if (ws_bytes < he_conv_plain_workspace_bytes(c, p, B)) return HE_ENOMEM;
    cudaStream_t st = STREAM(stream);
    const PlanDev P = plan_dev(p);
    u64* Cs = (u64*)d_ws;
    u64* Ps = Cs + (size_t)B * P.n_ib * c->L * c->N;
    he_status s = launch_ntt_fwd(c, (const u64*)d_c0, Cs, (long)B * P.n_ib * c->L, 0, st);
    if (s != HE_OK) return s;
    const long tp = (long)B * P.c_o * c->L * c->N;
    k_mac_plain<<<grid_for(tp, 256), 256, 0, st>>>(Cs, (const u64*)d_fplain, Ps, P, B, c->L,
                                                   c->logN, c->d_limb);
    HE_CHECK_LAUNCH();
    s = launch_ntt_inv(c, Ps, Ps, (long)B * P.c_o * c->L, st);
    if (s != HE_OK) return s;
    const long to = (long)B * P.n_ob * c->L * c->N;
    k_extract_plain<<<grid_for(to, 256), 256, 0, st>>>(Ps, d_phi1, (u64*)d_out, P, B, c->L,
                                                       c->logN, c->d_limb, c->d_enc, c->t,
                                                       c->r_t, c->t_inv);
    HE_CHECK_LAUNCH();
    return HE_OK;
}

// out[i][l][k] = x[i][l][k] * y[l][k] mod q_l (y broadcast; out may alias x)
__global__ void k_pointwise_mul_to(const u64* __restrict__ x, const u64* __restrict__ y,
                                   u64* __restrict__ out, long nx, int L, int logN,
                                   const he_limb* __restrict__ limbs) {
    const long N = 1L << logN;
    const long total = nx * L * N;
    for (long idx = blockIdx.x * (long)blockDim.x + threadIdx.x; idx < total;
         idx += (long)gridDim.x * blockDim.x) {
        const long k = idx & (N - 1), r = idx >> logN;
        const int l = (int)(r % L);
        const he_limb& Lm = limbs[l];
        out[idx] = d2canon(dp_mulmod(u2d(x[idx]), u2d(y[(long)l * N + k]), Lm.qd, Lm.qinvd),
                           Lm.qd, Lm.qinvd);
    }
}

// Client randomness of one layer in one pass: ve = v b + e (Eq. (1)) and
// vs = v s (the client's share factor, Alg. 1 Line 21), sharing NTT(v).
extern "C" he_status he_pk_mask_vs(const he_ctx* c, const int32_t* d_v, const int32_t* d_e,
                                   long n_polys, const uint64_t* d_b, const uint64_t* d_s,
                                   uint64_t* d_ve, uint64_t* d_vs, void* d_ws, size_t ws_bytes,
                                   void* stream) {
    if (!c || n_polys < 0) return HE_EINVAL;
    if (n_polys == 0) return HE_OK;
    if (!d_v || !d_b || !d_s || !d_ve || !d_vs || !d_ws) return HE_EINVAL;
    if (ws_bytes < 2 * sizeof(u64) * (size_t)c->L * c->N) return HE_ENOMEM;
    cudaStream_t st = STREAM(stream);
    const long total = n_polys * c->L * c->N;
    u64* bspec = (u64*)d_ws;
    u64* sspec = bspec + (size_t)c->L * c->N;
    he_status s = launch_ntt_fwd(c, (const u64*)d_b, bspec, c->L, 0, st);
    if (s != HE_OK) return s;
    s = launch_ntt_fwd(c, (const u64*)d_s, sspec, c->L, 0, st);
    if (s != HE_OK) return s;
    k_residues_from_int<<<grid_for(total, 256), 256, 0, st>>>(d_v, n_polys, c->L, c->logN,
                                                              c->d_limb, (u64*)d_vs);
    HE_CHECK_LAUNCH();
    s = launch_ntt_fwd(c, (const u64*)d_vs, (u64*)d_vs, n_polys * c->L, 0, st);   // V
    if (s != HE_OK) return s;
    k_pointwise_mul_to<<<grid_for(total, 256), 256, 0, st>>>((const u64*)d_vs, bspec,
                                                              (u64*)d_ve, n_polys, c->L,
                                                              c->logN, c->d_limb);
    k_pointwise_mul_to<<<grid_for(total, 256), 256, 0, st>>>((const u64*)d_vs, sspec,
                                                              (u64*)d_vs, n_polys, c->L,
                                                              c->logN, c->d_limb);
    HE_CHECK_LAUNCH();
    s = launch_ntt_inv(c, (u64*)d_ve, (u64*)d_ve, n_polys * c->L, st);
    if (s != HE_OK) return s;
    s = launch_ntt_inv(c, (u64*)d_vs, (u64*)d_vs, n_polys * c->L, st);
    if (s != HE_OK) return s;
    if (d_e) {
        k_add_small<<<grid_for(total, 256), 256, 0, st>>>((u64*)d_ve, d_e, n_polys, c->L,
                                                           c->logN, c->d_limb);
        HE_CHECK_LAUNCH();
    }
    return HE_OK;
}
