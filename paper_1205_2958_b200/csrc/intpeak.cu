// intpeak.cu -- integer-pipe throughput microbenchmarks (roofline denominators).
//
// MEASURED_PEAKS.json only carries HBM and bf16 tensor peaks; the sketch
// kernels are integer-issue bound, so their roofline needs the B200's
// per-SM integer throughputs. Each kernel runs a persistent grid (every SM
// full) with 8 independent dependency chains per thread and reports, via
// clock64 on each CTA, instructions per SM clock. Built into a separate
// libbbmh_intpeak.so (not part of the product ABI).
#include <cuda_runtime.h>

#include <cstdint>

namespace {

constexpr int kIlp = 8;
constexpr int kIters = 32768;

enum Op : int {
    OP_IMAD = 0,       // IMAD R, R, R, R          (fma pipe)
    OP_IMAD_WIDE = 1,  // IMAD.WIDE.U32 + LEA.HI   (the 4U Mersenne fold, 2 instructions)
    OP_VIMNMX3 = 2,    // 3-input unsigned min     (alu pipe)
    OP_IADD3 = 3,      // IADD3                    (alu pipe)
    OP_LOP3 = 4,       // LOP3.LUT                 (alu pipe)
    OP_MIX_2U = 5,     // 2 IMAD : 1 VIMNMX3 -- the 2U inner loop mix
    OP_LEAHI = 6,      // LEA.HI (hi + lo>>1)      (alu pipe)
    OP_VIADDMNMX = 7,  // min(x + c, x)            (alu pipe)
    OP_WIDE_XOR = 8,   // IMAD.WIDE.U32 + LOP3     (64-bit product rate)
    OP_IMAD_HI = 9,    // IMAD.HI.U32              (high-word product rate)
    OP_WIDE_RZ = 10,   // IMAD.WIDE.U32 a, b, RZ + LOP3 (no 64-bit addend: 2 register reads)
    OP_MIX_4U = 11,    // the 4U-bit fold step: IMAD.WIDE(+pair) + LEA.HI + VIADDMNMX
    OP_MIX_2U_REUSE = 12,  // 2 IMAD : 1 VIMNMX3 with the coefficients in fixed operand slots
    OP_MIX_2U_CONST = 13,  // 2 IMAD : 1 VIMNMX3 with the multiplier from the constant bank
    OP_IMAD_IMM = 14,      // IMAD R, R, imm32, R (immediate multiplier)
    OP_MIX_2U_IMM = 15,    // 2 IMAD(imm) : 1 VIMNMX3
    OP_MIX_2U_MIN2 = 16,   // 2 IMAD : 2 two-input VIMNMX (fewer ALU operands)
    OP_MIX_1TO1 = 17,      // 1 IMAD : 1 VIMNMX3
    OP_MIX_IADD_IMM = 18,  // 2 IMAD(imm) : 1 IADD3 with an immediate (1 register read)
    OP_MIX_2U_G4 = 19,     // 4 IMAD sharing both coefficients : 2 VIMNMX3 (coefficient-major)
    OP_MIX_2U_MOV = 20,    // 2 IMAD(imm) : 1 VIMNMX3, IMAD addend = fresh register
    OP_MIX_2U_UR = 21,     // 2 IMAD(uniform-register multiplier) : 1 VIMNMX3
    OP_DFMA = 22,          // DFMA (fp64 pipe)
    OP_MIX_DFMA_IMAD = 23, // 1 DFMA : 1 IMAD (separate pipes?)
    OP_EVAL_4U_HORNER = 24,  // one full 4U-bit evaluation as shipped (Horner, %D by IMAD.HI)
    OP_EVAL_4U_POWERS = 25,  // 4U-bit from precomputed powers, one 64-bit reduction, %D in fp32
};

constexpr uint32_t kP = 0x7fffffffu;
constexpr uint32_t kD = 16609143u;

template <int OP>
__global__ void __launch_bounds__(256) intpeak_kernel(uint32_t seed, uint32_t* sink,
                                                     unsigned long long* cycles,
                                                     unsigned long long* clk) {
    uint32_t a[kIlp], c1 = seed * 3 + 1, c2 = seed ^ 0x9e3779b9u;
    const uint32_t c1v = c1 + threadIdx.x * 0x10001u;  // per-lane (not uniform) addend
    uint64_t w[kIlp];
    double dv[kIlp];
    const double dc1 = 1.0000001 + seed * 1e-9, dc2 = 0.5;
#pragma unroll
    for (int i = 0; i < kIlp; ++i) {
        a[i] = threadIdx.x * 7 + i + seed;
        w[i] = a[i];
        dv[i] = a[i] * 1e-3;
    }
    __syncthreads();
    unsigned long long g0 = 0, g1 = 0;
    if (blockIdx.x == 0 && threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
    const unsigned long long t0 = clock64();
    for (int it = 0; it < kIters; ++it) {
#pragma unroll
        for (int i = 0; i < kIlp; ++i) {
            if constexpr (OP == OP_IMAD) {
                asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a[i]) : "r"(c1), "r"(c2));
            } else if constexpr (OP == OP_IMAD_WIDE) {
                // the 4U Mersenne fold: IMAD.WIDE.U32 (h*t2 + c) then LEA.HI (hi + lo>>1)
                const uint64_t v = (uint64_t)a[i] * c1 + c2;
                a[i] = (uint32_t)(v >> 32) + ((uint32_t)v >> 1);
                asm volatile("" : "+r"(a[i]));
            } else if constexpr (OP == OP_VIMNMX3) {
                a[i] = min(min(a[i], c1 + i), c2);
                asm volatile("" : "+r"(a[i]));
            } else if constexpr (OP == OP_IADD3) {
                asm volatile("add.u32 %0, %0, %1;\n\tadd.u32 %0, %0, %2;" : "+r"(a[i]) : "r"(c1), "r"(c2));
            } else if constexpr (OP == OP_LOP3) {
                asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(a[i]) : "r"(c1), "r"(c2));
            } else if constexpr (OP == OP_MIX_2U) {
                uint32_t h0, h1;
                asm volatile("mad.lo.u32 %0, %1, %2, %3;" : "=r"(h0) : "r"(a[i]), "r"(c1), "r"(c2));
                asm volatile("mad.lo.u32 %0, %1, %2, %3;" : "=r"(h1) : "r"(a[i]), "r"(c2), "r"(c1));
                a[i] = min(min(a[i], h0), h1);
                asm volatile("" : "+r"(a[i]));
            } else if constexpr (OP == OP_LEAHI) {
                a[i] = c1 + (a[i] >> 1);
                asm volatile("" : "+r"(a[i]));
            } else if constexpr (OP == OP_VIADDMNMX) {
                a[i] = min(a[i] + 0x80000001u, a[i]);
                asm volatile("" : "+r"(a[i]));
            } else if constexpr (OP == OP_WIDE_XOR) {
                const uint64_t v = (uint64_t)a[i] * c1 + c2;
                a[i] = (uint32_t)(v >> 32) ^ (uint32_t)v;
                asm volatile("" : "+r"(a[i]));
            } else if constexpr (OP == OP_IMAD_HI) {
                asm volatile("mad.hi.u32 %0, %0, %1, %2;" : "+r"(a[i]) : "r"(c1), "r"(c2));
            } else if constexpr (OP == OP_WIDE_RZ) {
                const uint64_t v = (uint64_t)a[i] * c1;
                a[i] = (uint32_t)(v >> 32) ^ (uint32_t)v;
                asm volatile("" : "+r"(a[i]));
            } else if constexpr (OP == OP_MIX_4U) {
                const uint64_t v = (uint64_t)a[i] * c1 + c2;
                const uint32_t s = (uint32_t)(v >> 32) + ((uint32_t)v >> 1);
                a[i] = min(s, s + 0x80000001u);
                asm volatile("" : "+r"(a[i]));
            } else if constexpr (OP == OP_IMAD_IMM) {
                asm volatile("mad.lo.u32 %0, %0, 0x9e3779b1, %1;" : "+r"(a[i]) : "r"(c2));
            } else if constexpr (OP == OP_MIX_2U_IMM) {
                uint32_t h0, h1;
                asm volatile("mad.lo.u32 %0, %1, 0x9e3779b1, %2;" : "=r"(h0) : "r"(a[i]), "r"(c2));
                asm volatile("mad.lo.u32 %0, %1, 0x85ebca6b, %2;" : "=r"(h1) : "r"((uint32_t)w[i]), "r"(c1));
                w[i] = h0;
                a[i] = min(min(a[i], h0), h1);
                asm volatile("" : "+r"(a[i]));
            } else if constexpr (OP == OP_MIX_2U_MIN2) {
                uint32_t h0, h1;
                asm volatile("mad.lo.u32 %0, %1, %2, %3;" : "=r"(h0) : "r"(a[i]), "r"(c1), "r"(c2));
                asm volatile("mad.lo.u32 %0, %1, %2, %3;" : "=r"(h1) : "r"((uint32_t)w[i]), "r"(c1), "r"(c2));
                w[i] = h0;
                asm volatile("min.u32 %0, %0, %1;" : "+r"(a[i]) : "r"(h0));
                asm volatile("min.u32 %0, %0, %1;" : "+r"(a[i]) : "r"(h1));
            } else if constexpr (OP == OP_MIX_1TO1) {
                uint32_t h0;
                asm volatile("mad.lo.u32 %0, %1, %2, %3;" : "=r"(h0) : "r"(a[i]), "r"(c1), "r"(c2));
                a[i] = min(min(a[i], h0), (uint32_t)w[i]);
                asm volatile("" : "+r"(a[i]));
            } else if constexpr (OP == OP_MIX_IADD_IMM) {
                uint32_t h0, h1;
                asm volatile("mad.lo.u32 %0, %1, 0x9e3779b1, %2;" : "=r"(h0) : "r"(a[i]), "r"(c2));
                asm volatile("mad.lo.u32 %0, %1, 0x85ebca6b, %2;" : "=r"(h1) : "r"((uint32_t)w[i]), "r"(c1));
                w[i] = h0;
                asm volatile("add.u32 %0, %1, 0x1234567;" : "=r"(a[i]) : "r"(h1));
            } else if constexpr (OP == OP_MIX_2U_G4) {
                // 4 ids t0..t3 (a[i], w lo/hi, a[i^1]) through one coefficient pair
                uint32_t h0, h1, h2, h3;
                const uint32_t t2 = (uint32_t)(w[i] >> 32), t3 = a[i ^ 1];
                asm volatile("mad.lo.u32 %0, %1, %2, %3;" : "=r"(h0) : "r"(a[i]), "r"(c1), "r"(c2));
                asm volatile("mad.lo.u32 %0, %1, %2, %3;" : "=r"(h1) : "r"((uint32_t)w[i]), "r"(c1), "r"(c2));
                asm volatile("mad.lo.u32 %0, %1, %2, %3;" : "=r"(h2) : "r"(t2), "r"(c1), "r"(c2));
                asm volatile("mad.lo.u32 %0, %1, %2, %3;" : "=r"(h3) : "r"(t3), "r"(c1), "r"(c2));
                w[i] = ((uint64_t)h2 << 32) | h0;
                a[i] = min(min(a[i], h0), h1);
                a[i] = min(min(a[i], h2), h3);
                asm volatile("" : "+r"(a[i]));
            } else if constexpr (OP == OP_MIX_2U_MOV) {
                uint32_t h0, h1;
                asm volatile("mad.lo.u32 %0, %1, 0x9e3779b1, %2;" : "=r"(h0) : "r"(a[i]), "r"((uint32_t)(w[i] >> 32)));
                asm volatile("mad.lo.u32 %0, %1, 0x85ebca6b, %2;" : "=r"(h1) : "r"((uint32_t)w[i]), "r"(a[i ^ 1]));
                w[i] = ((uint64_t)h1 << 32) | h0;
                a[i] = min(min(a[i], h0), h1);
                asm volatile("" : "+r"(a[i]));
            } else if constexpr (OP == OP_MIX_2U_UR) {
                // multiplier warp-uniform (kernel parameter -> uniform register), addend per lane
                uint32_t h0, h1;
                asm volatile("mad.lo.u32 %0, %1, %2, %3;" : "=r"(h0) : "r"(a[i]), "r"(c2), "r"(c1v));
                asm volatile("mad.lo.u32 %0, %1, %2, %3;" : "=r"(h1) : "r"((uint32_t)w[i]), "r"(c2), "r"(c1v));
                w[i] = h0;
                a[i] = min(min(a[i], h0), h1);
                asm volatile("" : "+r"(a[i]));
            } else if constexpr (OP == OP_DFMA) {
                asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(dv[i]) : "d"(dc1), "d"(dc2));
            } else if constexpr (OP == OP_MIX_DFMA_IMAD) {
                asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(dv[i]) : "d"(dc1), "d"(dc2));
                asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a[i]) : "r"(c1), "r"(c2));
            } else if constexpr (OP == OP_EVAL_4U_HORNER) {
                // t2 = 2t (< 2^32), coefficients a3, 2a2, 2a1, 2a0 (c1, c2, c1^5, c2^7 stand-ins)
                const uint32_t t2 = (a[i] & kP) << 1;
                auto fold = [](uint32_t h, uint32_t t, uint32_t c) {
                    const uint64_t v = (uint64_t)h * t + c;
                    return (uint32_t)(v >> 32) + ((uint32_t)v >> 1);
                };
                uint32_t x = fold(c1 & kP, t2, c2 & ~1u);
                x = min(x, x - kP);
                x = fold(x, t2, (c1 ^ 5) & ~1u);
                x = min(x, x - kP);
                x = fold(x, t2, (c2 ^ 7) & ~1u);
                x = min(min(x, x - kP), x - 2 * kP);
                const uint32_t q = __umulhi(x, 0x8150ee2bu) >> 23;
                x = x + q * (0u - kD);
                w[i] = min((uint32_t)w[i], x);
                a[i] += x;
                asm volatile("" : "+r"(a[i]));
            } else if constexpr (OP == OP_EVAL_4U_POWERS) {
                // T1..T3 < p precomputed per id (here derived cheaply from the chain value)
                const uint32_t T1 = a[i] & kP, T2 = (a[i] * 3) & kP, T3 = (a[i] ^ 0x5555) & kP;
                uint64_t x = (uint64_t)(c1 & kP) * T3 + (c2 & kP);
                x += (uint64_t)((c1 ^ 5) & kP) * T2;
                x += (uint64_t)((c2 ^ 7) & kP) * T1;  // < 3 p^2 + p
                const uint32_t hi = (uint32_t)(x >> 32), lo = (uint32_t)x;
                uint32_t h2 = min(hi, hi - kP);                 // hi mod p (hi < 3*2^30)
                uint32_t l2 = (lo >> 31) + (lo & kP);           // lo mod p, lazily (<= p)
                uint32_t s = h2 + l2;                           // < 2^32
                s = (s >> 31) + (s & kP);
                s = s + h2;                                     // x = 2 hi + lo (mod p)
                s = (s >> 31) + (s & kP);
                s = min(s, s - kP);
                // s % D in fp32: q in {floor(s/D) - 1, floor(s/D)}, then one correction
                const float sf = __int_as_float(0x4B000000u + (s >> 8)) - 8388608.0f;
                const float y = __fmaf_rn(sf, 256.0f / kD * (1.0f - 1.0f / 1048576.0f), 12582911.5f);
                const int qq = __float_as_int(y) - 0x4B400000;
                uint32_t r = s - (uint32_t)qq * kD;
                r = min(r, r - kD);
                w[i] = min((uint32_t)w[i], r);
                a[i] += r;
                asm volatile("" : "+r"(a[i]));
            } else if constexpr (OP == OP_MIX_2U_CONST) {
                // multiplier straight from the kernel-parameter constant bank
                uint32_t h0, h1;
                asm volatile("mad.lo.u32 %0, %1, %2, %3;" : "=r"(h0) : "r"(a[i]), "r"(seed), "r"(c2));
                asm volatile("mad.lo.u32 %0, %1, %2, %3;" : "=r"(h1) : "r"((uint32_t)w[i]), "r"(seed), "r"(c2));
                w[i] = h0;
                a[i] = min(min(a[i], h0), h1);
                asm volatile("" : "+r"(a[i]));
            } else {
                // two products with (c1, c2) in the same slots -> operand-reuse friendly
                uint32_t h0, h1;
                asm volatile("mad.lo.u32 %0, %1, %2, %3;" : "=r"(h0) : "r"(a[i]), "r"(c1), "r"(c2));
                asm volatile("mad.lo.u32 %0, %1, %2, %3;" : "=r"(h1) : "r"((uint32_t)w[i]), "r"(c1), "r"(c2));
                w[i] = h0;
                a[i] = min(min(a[i], h0), h1);
                asm volatile("" : "+r"(a[i]));
            }
        }
    }
    const unsigned long long t1 = clock64();
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
        clk[0] = t0;
        clk[1] = t1;
        clk[2] = g0;
        clk[3] = g1;
    }
    uint32_t acc = 0;
#pragma unroll
    for (int i = 0; i < kIlp; ++i) acc ^= a[i] ^ (uint32_t)w[i] ^ (uint32_t)(w[i] >> 32) ^ (uint32_t)__double2uint_rz(dv[i]);
    if (acc == 0x12345678u) sink[0] = acc;
    if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

template <int OP>
float run(int blocks, int threads, uint32_t* sink, unsigned long long* cyc, unsigned long long* clk,
          cudaStream_t st) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    intpeak_kernel<OP><<<blocks, threads, 0, st>>>(1, sink, cyc, clk);  // warm-up
    cudaEventRecord(e0, st);
    intpeak_kernel<OP><<<blocks, threads, 0, st>>>(2, sink, cyc, clk);
    cudaEventRecord(e1, st);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return ms;
}

}  // namespace

extern "C" {

// Instructions issued per thread per kernel for `op` (source-level count;
// OP_IADD3 issues 2 adds per step that ptxas may merge into one IADD3).
__attribute__((visibility("default"))) double bbmh_intpeak_ops_per_thread(int op) {
    const double base = double(kIters) * kIlp;
    switch (op) {
        case OP_MIX_2U: return base * 3;  // 2 IMAD + 1 VIMNMX3
        case OP_IMAD_WIDE: return base * 2;  // IMAD.WIDE + LEA.HI
        case OP_WIDE_XOR: return base * 2;   // IMAD.WIDE + LOP3
        case OP_WIDE_RZ: return base * 2;    // IMAD.WIDE (RZ addend) + LOP3
        case OP_MIX_4U: return base * 3;     // IMAD.WIDE + LEA.HI + VIADDMNMX
        case OP_MIX_2U_REUSE: return base * 3;
        case OP_MIX_2U_CONST: return base * 3;
        case OP_MIX_2U_IMM: return base * 3;
        case OP_MIX_2U_MIN2: return base * 4;
        case OP_MIX_1TO1: return base * 2;
        case OP_MIX_IADD_IMM: return base * 3;
        case OP_MIX_2U_G4: return base * 6;
        case OP_MIX_2U_MOV: return base * 3;
        case OP_MIX_2U_UR: return base * 3;
        case OP_MIX_DFMA_IMAD: return base * 2;
        case OP_EVAL_4U_HORNER: return base;  // evaluations, not instructions
        case OP_EVAL_4U_POWERS: return base;
        default: return base;
    }
}

// Runs one microbenchmark; returns elapsed ms and the mean per-CTA cycles.
__attribute__((visibility("default"))) int bbmh_intpeak_run(int op, int blocks, int threads,
                                                           float* ms_out, double* cycles_out,
                                                           double* sm_mhz_out) {
    uint32_t* sink = nullptr;
    unsigned long long* cyc = nullptr;
    unsigned long long* clk = nullptr;
    if (cudaMalloc(&sink, 4) != cudaSuccess) return -1;
    if (cudaMalloc(&clk, 4 * sizeof(unsigned long long)) != cudaSuccess) return -1;
    if (cudaMalloc(&cyc, sizeof(unsigned long long) * blocks) != cudaSuccess) return -1;
    cudaStream_t st;
    cudaStreamCreate(&st);
    float ms = -1;
    switch (op) {
        case OP_IMAD: ms = run<OP_IMAD>(blocks, threads, sink, cyc, clk, st); break;
        case OP_IMAD_WIDE: ms = run<OP_IMAD_WIDE>(blocks, threads, sink, cyc, clk, st); break;
        case OP_VIMNMX3: ms = run<OP_VIMNMX3>(blocks, threads, sink, cyc, clk, st); break;
        case OP_IADD3: ms = run<OP_IADD3>(blocks, threads, sink, cyc, clk, st); break;
        case OP_LOP3: ms = run<OP_LOP3>(blocks, threads, sink, cyc, clk, st); break;
        case OP_MIX_2U: ms = run<OP_MIX_2U>(blocks, threads, sink, cyc, clk, st); break;
        case OP_LEAHI: ms = run<OP_LEAHI>(blocks, threads, sink, cyc, clk, st); break;
        case OP_VIADDMNMX: ms = run<OP_VIADDMNMX>(blocks, threads, sink, cyc, clk, st); break;
        case OP_WIDE_XOR: ms = run<OP_WIDE_XOR>(blocks, threads, sink, cyc, clk, st); break;
        case OP_IMAD_HI: ms = run<OP_IMAD_HI>(blocks, threads, sink, cyc, clk, st); break;
        case OP_WIDE_RZ: ms = run<OP_WIDE_RZ>(blocks, threads, sink, cyc, clk, st); break;
        case OP_MIX_4U: ms = run<OP_MIX_4U>(blocks, threads, sink, cyc, clk, st); break;
        case OP_MIX_2U_REUSE: ms = run<OP_MIX_2U_REUSE>(blocks, threads, sink, cyc, clk, st); break;
        case OP_MIX_2U_CONST: ms = run<OP_MIX_2U_CONST>(blocks, threads, sink, cyc, clk, st); break;
        case OP_IMAD_IMM: ms = run<OP_IMAD_IMM>(blocks, threads, sink, cyc, clk, st); break;
        case OP_MIX_2U_IMM: ms = run<OP_MIX_2U_IMM>(blocks, threads, sink, cyc, clk, st); break;
        case OP_MIX_2U_MIN2: ms = run<OP_MIX_2U_MIN2>(blocks, threads, sink, cyc, clk, st); break;
        case OP_MIX_1TO1: ms = run<OP_MIX_1TO1>(blocks, threads, sink, cyc, clk, st); break;
        case OP_MIX_IADD_IMM: ms = run<OP_MIX_IADD_IMM>(blocks, threads, sink, cyc, clk, st); break;
        case OP_MIX_2U_G4: ms = run<OP_MIX_2U_G4>(blocks, threads, sink, cyc, clk, st); break;
        case OP_MIX_2U_MOV: ms = run<OP_MIX_2U_MOV>(blocks, threads, sink, cyc, clk, st); break;
        case OP_MIX_2U_UR: ms = run<OP_MIX_2U_UR>(blocks, threads, sink, cyc, clk, st); break;
        case OP_DFMA: ms = run<OP_DFMA>(blocks, threads, sink, cyc, clk, st); break;
        case OP_MIX_DFMA_IMAD: ms = run<OP_MIX_DFMA_IMAD>(blocks, threads, sink, cyc, clk, st); break;
        case OP_EVAL_4U_HORNER: ms = run<OP_EVAL_4U_HORNER>(blocks, threads, sink, cyc, clk, st); break;
        case OP_EVAL_4U_POWERS: ms = run<OP_EVAL_4U_POWERS>(blocks, threads, sink, cyc, clk, st); break;
        default: return -2;
    }
    unsigned long long* h = new unsigned long long[blocks];
    cudaMemcpy(h, cyc, sizeof(unsigned long long) * blocks, cudaMemcpyDeviceToHost);
    double s = 0;
    for (int i = 0; i < blocks; ++i) s += double(h[i]);
    delete[] h;
    *ms_out = ms;
    *cycles_out = s / blocks;
    unsigned long long hc[4];
    cudaMemcpy(hc, clk, sizeof hc, cudaMemcpyDeviceToHost);
    *sm_mhz_out = hc[3] > hc[2] ? double(hc[1] - hc[0]) / double(hc[3] - hc[2]) * 1e3 : 0;
    cudaFree(clk);
    cudaFree(sink);
    cudaFree(cyc);
    cudaStreamDestroy(st);
    return cudaGetLastError() == cudaSuccess ? 0 : -3;
}
}

// ---- L2 random-gather throughput (roofline denominator of permutation mode) ----
namespace {
__global__ void __launch_bounds__(256) l2gather_kernel(const uint32_t* __restrict__ tab, uint32_t mask,
                                                       uint32_t iters, uint32_t seed, uint32_t* sink) {
    uint32_t x = (blockIdx.x * blockDim.x + threadIdx.x) * 0x9e3779b9u ^ seed;
    uint32_t m = 0xffffffffu;
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    for (uint32_t it = 0; it < iters; ++it) {
        uint32_t v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            x = x * 1664525u + 1013904223u;  // LCG: independent addresses, 8 loads in flight
            asm volatile("ld.global.nc.L2::cache_hint.u32 %0, [%1], %2;"
                         : "=r"(v[u]) : "l"(tab + ((x >> 5) & mask)), "l"(pol));
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) m = min(m, v[u]);
    }
    if (m == 0x12345678u) sink[0] = m;
}
}  // namespace

extern "C" __attribute__((visibility("default"))) int bbmh_l2gather_run(uint64_t table_bytes, int blocks,
                                                                       int threads, uint32_t iters,
                                                                       double* gathers_per_s) {
    uint32_t* tab = nullptr;
    uint32_t* sink = nullptr;
    const uint64_t n = table_bytes / 4;
    if ((n & (n - 1)) != 0) return -1;  // power of two entries
    if (cudaMalloc(&tab, table_bytes) != cudaSuccess) return -2;
    if (cudaMalloc(&sink, 4) != cudaSuccess) return -2;
    cudaMemset(tab, 0x11, table_bytes);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    l2gather_kernel<<<blocks, threads>>>(tab, (uint32_t)(n - 1), iters, 1, sink);  // warm L2
    cudaEventRecord(e0);
    l2gather_kernel<<<blocks, threads>>>(tab, (uint32_t)(n - 1), iters, 2, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    *gathers_per_s = (double)blocks * threads * iters * 8 / (ms * 1e-3);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(tab);
    cudaFree(sink);
    return cudaGetLastError() == cudaSuccess ? 0 : -3;
}
