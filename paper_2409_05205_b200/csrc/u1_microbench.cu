// u1_microbench.cu -- U1: register-resident throughput of the
// integer operations the hot path is built from, measured on the B200 that
// runs the bench.  These are the "alu" roofline denominators bench.py uses
// (DESIGN.md "Roofline").  Not part of the product C-ABI (separate .so).
//
//   which 0: IMAD      (mad.lo.u32)                      -> IMAD / s
//   which 1: IMAD.WIDE (mad.wide.u32, 64-bit addend)     -> IMAD.WIDE / s
//   which 2: lazy modular MAC, 25-bit split (4 mad.wide + 2 LOP3 for the
//            loop-carried operands)                   -> MAC / s
//   which 3: Shoup Cooley-Tukey butterfly (ct_bfly)      -> butterflies / s
//   which 4: Shoup Gentleman-Sande butterfly (gs_bfly)   -> butterflies / s
//   which 5: int8 mma.sync; 6: DFMA; 7/8: FP64 CT / GS butterflies (the
//            default transforms, he_internal.cuh)
//   which 9..14: tcgen05.mma.cta_group::1.kind::i8 (u8 x u8 -> s32, K = 32,
//            operands in shared memory, accumulator in TMEM) issued back to
//            back by one thread per CTA, one CTA per SM:
//            9: M=128 N=16, 10: M=128 N=32, 11: M=128 N=64, 12: M=128 N=256,
//            13: M=64 N=32, 14: M=64 N=256           -> int8 MACs / s
#include <cuda_runtime.h>
#include <stdint.h>

#include "he_internal.cuh"

__global__ void u1_imad(const u32* in, u32* out, int iters, long long* cyc) {
    u32 a = in[0], b = in[1];
    u32 x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x + i;
    long long c0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i)
            asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(x[i]) : "r"(a), "r"(b));
    }
    long long c1 = clock64();
    u32 s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s ^= x[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (blockIdx.x == 0 && threadIdx.x == 0) *cyc = c1 - c0;
}

__global__ void u1_imad_wide(const u32* in, u32* out, int iters, long long* cyc) {
    u32 b = in[1];
    u64 acc[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] = i;
    long long c0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i)   // multiplier is loop-carried: not hoistable
            asm volatile("mad.wide.u32 %0, %1, %2, %0;" : "+l"(acc[i]) : "r"((u32)acc[i]), "r"(b));
    }
    long long c1 = clock64();
    u64 s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s ^= acc[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = (u32)(s ^ (s >> 32));
    if (blockIdx.x == 0 && threadIdx.x == 0) *cyc = c1 - c0;
}

// 2 independent lazy MACs per iteration (acc0 += c0 f0; acc1 += c0 f1 + c1 f0;
// acc2 += c1 f1), i.e. 8 mad.wide per iteration.
__global__ void u1_mac(const u32* in, u32* out, int iters, long long* cyc) {
    u32 c0 = in[0] + threadIdx.x, c1 = in[1], f0 = in[2], f1 = in[3];
    u64 a[2][3] = {{0, 0, 0}, {1, 1, 1}};
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int m = 0; m < 2; ++m) {
            // operands change every iteration (as the C spectrum words do in
            // k_mac_fold), so ptxas cannot hoist the products out of the loop
            const u32 x0 = c0 ^ (u32)a[m][2], x1 = c1 ^ (u32)a[m][0];
            asm volatile("mad.wide.u32 %0, %1, %2, %0;" : "+l"(a[m][0]) : "r"(x0), "r"(f0));
            asm volatile("mad.wide.u32 %0, %1, %2, %0;" : "+l"(a[m][1]) : "r"(x0), "r"(f1));
            asm volatile("mad.wide.u32 %0, %1, %2, %0;" : "+l"(a[m][1]) : "r"(x1), "r"(f0));
            asm volatile("mad.wide.u32 %0, %1, %2, %0;" : "+l"(a[m][2]) : "r"(x1), "r"(f1));
        }
    }
    long long t1 = clock64();
    u64 s = a[0][0] ^ a[0][1] ^ a[0][2] ^ a[1][0] ^ a[1][1] ^ a[1][2];
    out[blockIdx.x * blockDim.x + threadIdx.x] = (u32)(s ^ (s >> 32));
    if (blockIdx.x == 0 && threadIdx.x == 0) *cyc = t1 - t0;
}

template <bool GS>
__global__ void u1_bfly(const u64* in, u32* out, int iters, long long* cyc) {
    const u64 q = in[0], q2 = 2 * q;
    const ulonglong2 w = make_ulonglong2(in[1], in[2]);
    u64 X[8], Y[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) { X[i] = (threadIdx.x + i) % q; Y[i] = (threadIdx.x * 7 + i) % q; }
    long long c0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            // the lazy forms the kernels use (ct: no conditional subtraction;
            // gs: offset q << (stage + 1), here a fixed 2^12 q)
            if (GS) gs_bfly_lazy(X[i], Y[i], w, q, q << 12);
            else ct_bfly_lazy(X[i], Y[i], w, q, q2);
        }
    }
    long long c1 = clock64();
    u64 s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s ^= X[i] ^ Y[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = (u32)(s ^ (s >> 32));
    if (blockIdx.x == 0 && threadIdx.x == 0) *cyc = c1 - c0;
}

// which 5: legacy int8 tensor-core MMA (mma.sync m16n8k32 u8 x u8 -> s32),
// 4 independent accumulators per warp -> int8 MACs / s (per lane-thread
// count converted by the host: 4096 MACs per warp-instruction).
__global__ void u1_imma(const u32* in, u32* out, int iters, long long* cyc) {
    u32 a0 = in[0] + threadIdx.x, a1 = in[1], a2 = in[2], a3 = in[3];
    u32 b0 = in[1] ^ threadIdx.x, b1 = in[2];
    int acc[4][4] = {};
    long long c0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int m = 0; m < 4; ++m)
            asm volatile(
                "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
                "{%8,%9}, {%0,%1,%2,%3};"
                : "+r"(acc[m][0]), "+r"(acc[m][1]), "+r"(acc[m][2]), "+r"(acc[m][3])
                : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
    long long c1 = clock64();
    int s = 0;
#pragma unroll
    for (int m = 0; m < 4; ++m) s ^= acc[m][0] ^ acc[m][1] ^ acc[m][2] ^ acc[m][3];
    out[blockIdx.x * blockDim.x + threadIdx.x] = (u32)s;
    if (blockIdx.x == 0 && threadIdx.x == 0) *cyc = c1 - c0;
}

// which 6: FP64 DFMA chains.
__global__ void u1_dfma(const u32* in, u32* out, int iters, long long* cyc) {
    double a = 1.0 + in[0] * 1e-9, b = 1e-7 * in[1];
    double x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x + i;
    long long c0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
    }
    long long c1 = clock64();
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += x[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = (u32)(long long)s;
    if (blockIdx.x == 0 && threadIdx.x == 0) *cyc = c1 - c0;
}

// which 7: exact FP64 Cooley-Tukey butterfly on signed residues (|x| < 2^51):
// reduce the multiplicand, T = Y w mod q via an exact two-product and a
// magic-number rounded quotient (|T| < 0.9 q), X' = X + T, Y' = X - T.
__global__ void u1_dbfly(const u64* in, u32* out, int iters, long long* cyc) {
    const double q = (double)in[0], w = (double)in[1], qinv = 1.0 / q;
    double X[8], Y[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) { X[i] = (double)((threadIdx.x + i) % in[0]); Y[i] = (double)((threadIdx.x * 7 + i) % in[0]); }
    long long c0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            // the kernels' mix: about one reduction per butterfly (pass-start
            // reductions + the stage-2 multiplicand reduction)
            Y[i] = dp_reduce(Y[i], q, qinv);
            ct_bfly_dp(X[i], Y[i], w, q, qinv);
        }
    }
    long long c1 = clock64();
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += X[i] + Y[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = (u32)(long long)s;
    if (blockIdx.x == 0 && threadIdx.x == 0) *cyc = c1 - c0;
}

// which 8: FP64 Gentleman-Sande butterfly as in gs_pass_dp (X' = X + Y,
// Y' = (X - Y) w mod q, about one reduction per butterfly).
__global__ void u1_dgsbfly(const u64* in, u32* out, int iters, long long* cyc) {
    const double q = (double)in[0], w = (double)in[1], qinv = 1.0 / q;
    double X[8], Y[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) { X[i] = (double)((threadIdx.x + i) % in[0]); Y[i] = (double)((threadIdx.x * 7 + i) % in[0]); }
    long long c0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const double x = dp_reduce(X[i], q, qinv), y = Y[i];
            X[i] = x + y;
            Y[i] = dp_mulmod(x - y, w, q, qinv);
        }
    }
    long long c1 = clock64();
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += X[i] + Y[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = (u32)(long long)s;
    if (blockIdx.x == 0 && threadIdx.x == 0) *cyc = c1 - c0;
}

// which 9..14: tcgen05 int8 MMA issue throughput.  Operands are zero
// (the tensor datapath's cost does not depend on values); 8 MMAs per
// iteration rotate over 4 accumulator regions so no two consecutive MMAs
// write the same TMEM columns.
__device__ __forceinline__ uint64_t u1_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}
template <int M, int N>
__global__ void __launch_bounds__(128, 1) u1_tc(u32* out, int iters, long long* cyc) {
    __shared__ __align__(1024) unsigned char sA[M * 32];
    __shared__ __align__(1024) unsigned char sB[N * 32];
    __shared__ uint32_t s_tmem;
    __shared__ __align__(8) uint64_t s_bar;
    for (int i = threadIdx.x; i < M * 8; i += blockDim.x) reinterpret_cast<u32*>(sA)[i] = 0;
    for (int i = threadIdx.x; i < N * 8; i += blockDim.x) reinterpret_cast<u32*>(sB)[i] = 0;
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(
            (uint32_t)__cvta_generic_to_shared(&s_tmem)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(
            (uint32_t)__cvta_generic_to_shared(&s_bar)));
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    const uint32_t tmem = s_tmem;
    long long c0 = clock64();
    if (threadIdx.x == 0) {
        const uint64_t ad = u1_desc((uint32_t)__cvta_generic_to_shared(sA), 128, 256);
        const uint64_t bd = u1_desc((uint32_t)__cvta_generic_to_shared(sB), 128, 256);
        const uint32_t idesc = (2u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
        const int stride = N < 128 ? N : 128;
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const uint32_t d = tmem + (uint32_t)((k & 3) * stride) % 512u;
                asm volatile(
                    "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                    "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d),
                    "l"(ad), "l"(bd), "r"(idesc), "r"(1u));
            }
        }
        asm volatile(
            "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                (uint32_t)__cvta_generic_to_shared(&s_bar))
            : "memory");
    }
    __syncwarp();
    {
        uint32_t ok = 0;
        const uint32_t bar = (uint32_t)__cvta_generic_to_shared(&s_bar);
        while (!ok)
            asm volatile(
                "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\t"
                "selp.u32 %0, 1, 0, p;\n\t}\n"
                : "=r"(ok) : "r"(bar) : "memory");
    }
    long long c1 = clock64();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    __syncthreads();
    if (threadIdx.x < 32)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
    if (threadIdx.x == 0) out[blockIdx.x] = tmem;
    if (blockIdx.x == 0 && threadIdx.x == 0) *cyc = c1 - c0;
}

// Runs kernel `which` once (after one warm-up launch); returns the elapsed
// milliseconds, the in-kernel cycle count of block 0 (SM clock estimate)
// and the number of operations executed.  0 on success.
extern "C" int u1_run(int which, int blocks, int threads, int iters, float* ms,
                      long long* cycles, double* ops) {
    u32* d_in = nullptr;
    u32* d_out = nullptr;
    long long* d_cyc = nullptr;
    u64 h_in64[4] = {1125899906826241ull, 11286399139ull, 0, 0};
    h_in64[2] = (u64)(((unsigned __int128)h_in64[1] << 64) / h_in64[0]);
    if (cudaMalloc(&d_in, 64) || cudaMalloc(&d_out, sizeof(u32) * blocks * threads) ||
        cudaMalloc(&d_cyc, sizeof(long long)))
        return 1;
    if (which == 3 || which == 4 || which == 7 || which == 8) cudaMemcpy(d_in, h_in64, sizeof(h_in64), cudaMemcpyHostToDevice);
    else {
        u32 h[4] = {3u, 5u, 0x1ffffffu, 0x1234567u};
        cudaMemcpy(d_in, h, sizeof(h), cudaMemcpyHostToDevice);
    }
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    double per_iter = 0;
    for (int rep = 0; rep < 2; ++rep) {
        if (rep == 1) cudaEventRecord(e0);
        switch (which) {
            case 0: u1_imad<<<blocks, threads>>>(d_in, d_out, iters, d_cyc); per_iter = 8; break;
            case 1: u1_imad_wide<<<blocks, threads>>>(d_in, d_out, iters, d_cyc); per_iter = 8; break;
            case 2: u1_mac<<<blocks, threads>>>(d_in, d_out, iters, d_cyc); per_iter = 2; break;
            case 3: u1_bfly<false><<<blocks, threads>>>((const u64*)d_in, d_out, iters, d_cyc); per_iter = 8; break;
            case 4: u1_bfly<true><<<blocks, threads>>>((const u64*)d_in, d_out, iters, d_cyc); per_iter = 8; break;
            case 5: u1_imma<<<blocks, threads>>>(d_in, d_out, iters, d_cyc); per_iter = 4 * 4096.0 / 32; break;
            case 6: u1_dfma<<<blocks, threads>>>(d_in, d_out, iters, d_cyc); per_iter = 8; break;
            case 7: u1_dbfly<<<blocks, threads>>>((const u64*)d_in, d_out, iters, d_cyc); per_iter = 8; break;
            case 8: u1_dgsbfly<<<blocks, threads>>>((const u64*)d_in, d_out, iters, d_cyc); per_iter = 8; break;
            // tcgen05: one 128-thread CTA per SM (blocks = the SM count);
            // ops counted per thread below, so per_iter = 8 MMAs x M N K / 128
            case 9: u1_tc<128, 16><<<blocks, 128>>>(d_out, iters, d_cyc); per_iter = 8.0 * 128 * 16 * 32 / threads; break;
            case 10: u1_tc<128, 32><<<blocks, 128>>>(d_out, iters, d_cyc); per_iter = 8.0 * 128 * 32 * 32 / threads; break;
            case 11: u1_tc<128, 64><<<blocks, 128>>>(d_out, iters, d_cyc); per_iter = 8.0 * 128 * 64 * 32 / threads; break;
            case 12: u1_tc<128, 256><<<blocks, 128>>>(d_out, iters, d_cyc); per_iter = 8.0 * 128 * 256 * 32 / threads; break;
            case 13: u1_tc<64, 32><<<blocks, 128>>>(d_out, iters, d_cyc); per_iter = 8.0 * 64 * 32 * 32 / threads; break;
            case 14: u1_tc<64, 256><<<blocks, 128>>>(d_out, iters, d_cyc); per_iter = 8.0 * 64 * 256 * 32 / threads; break;
            default: return 2;
        }
        if (rep == 1) cudaEventRecord(e1);
    }
    cudaEventSynchronize(e1);
    int rc = cudaGetLastError() != cudaSuccess ? 3 : 0;
    cudaEventElapsedTime(ms, e0, e1);
    cudaMemcpy(cycles, d_cyc, sizeof(long long), cudaMemcpyDeviceToHost);
    *ops = (double)blocks * threads * iters * per_iter;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(d_in);
    cudaFree(d_out);
    cudaFree(d_cyc);
    return rc;
}
