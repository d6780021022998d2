// mlp_tc.cu -- A1 and A6/A7 on the 5th-generation tensor cores (tcgen05 + TMEM), sm_100a.
//
// The network PINN(x,y) = 16x(1-x)y(1-y) net_theta(x,y) (readings R5/R6) is
// evaluated over all P = N^2 MLP points in tiles of 128 points. Every hidden-to-hidden layer
// is a 128 x WP x WP GEMM on tcgen05.mma kind::f16 with fp32 accumulators in TMEM:
//  * forward (k_tc_forward, all layers fused per tile): activations t are split t = hi + lo
//    with hi = fp16(t), lo = fp16(t - hi), and Z = T_hi W^T + T_lo W^T (2 MMAs) -- the
//    activation rounding of a single 10-bit-mantissa pass is what breaks loss parity at 512^2
//    (SURVEY.md key finding 4); weights are rounded once to fp16 (10-bit mantissa, as TF32).
//    Epilogue warps read TMEM, add bias, apply tanh, split, write the next A operand into
//    shared memory (SWIZZLE_128B K-major) and stream t_hi to HBM with bulk copies.
//  * backward: Delta_{a} = (Delta_{a+1} W) (.) (1 - t_a^2) and dW = sum_p Delta^T t, both on
//    tcgen05 in one launch per hidden GEMM (k_tc_bwd2: CTA pairs, Delta multicast, W^T resident),
//    or all hidden GEMMs in one spatial-pipeline launch (k_tc_bwdc, small problems), or
//    k_tc_out_bwd + k_tc_bwd_layer for WP = 64. Delta is stored in fp16 after a power-of-two
//    scaling of dLOSS/dnet (DevState::gscale) so that it stays in fp16's normal range; partial
//    sums are unscaled in the reduction.
// Weights are streamed into shared memory by cp.async.bulk (the TMA engine) from fp16 copies
// that k_tc_refresh re-lays out after every Adam step (zero-padded to WP = 64*ceil(w/64)).
#include "mlp_tc.cuh"
#include "tc_ptx.cuh"
#include "../../include/crvpinn.h"
#include <math.h>
#include <cstdlib>
#include <type_traits>

namespace crv {

using namespace ptx;

constexpr uint32_t CHUNK_BYTES = 128 * 128;   // one tile-chunk block: 128 rows x 128 B
constexpr int CHUNK_HALVES = 128 * 64;
constexpr int NST_W = 2;                      // weight ring stages
constexpr int EPI_THREADS = 256;              // 8 epilogue warps
constexpr int TC_THREADS = 64 + EPI_THREADS;  // producer warp + MMA warp + epilogue

__device__ __forceinline__ uint8_t *align1024(uint8_t *p) {
    return (uint8_t *)(((uintptr_t)p + 1023) & ~(uintptr_t)1023);
}

// byte offset of element (r, f%64) inside a tile-chunk block
__device__ __forceinline__ uint32_t blk_off(int r, int f) {
    return (uint32_t)(r * 128 + ((((f & 63) >> 3) ^ (r & 7)) << 4) + ((f & 7) << 1));
}

// Butterfly reduce-scatter: on entry v[k] is this lane's value for column k (0..31); on exit
// v[0] holds the sum over the warp's 32 lanes of column `lane`.
__device__ __forceinline__ void warp_reduce_scatter32(float (&v)[32], int lane) {
#pragma unroll
    for (int s = 16; s >= 1; s >>= 1) {
        const bool upper = (lane & s) != 0;
#pragma unroll
        for (int i = 0; i < s; ++i) {
            float send = upper ? v[i] : v[i + s];
            float keep = upper ? v[i + s] : v[i];
            v[i] = keep + __shfl_xor_sync(0xffffffffu, send, s);
        }
    }
}

// ================================================================ forward
struct FwdArgs {
    int N, ntiles, L, G;
    const __half *Wf;      // [G][KC] blocks
    const float *W1p, *bp, *Wop;
    __half *act;           // [L][ntiles][KC] blocks
    float *u;              // lattice (N+1)^2 (EVAL: [npts], one value per point)
    long long *trace;      // debug timeline (CTA 0), nullptr normally
    const float *xy;       // EVAL only: point coordinates [npts][2]
    int npts;              // EVAL only: number of points (ntiles = ceil(npts / 128), ragged tail)
    int p0;                // first MLP point of this shard (tile0 * 128); 0 unsharded
    const DevState *st;    // per-GEMM weight exponents (wexp, written by k_wscale)
};
// clock64 timelines (FTRACE / BTRACE / CTRACE, the CRVPINN_*_TRACE debug paths) are compiled in only with
// -DCRV_TRACE=1 (scripts/ab_build_tc.sh trace -DCRV_TRACE=1): their run-time checks sit in the hot loops
#ifndef CRV_TRACE
#define CRV_TRACE 0
#endif
// the trace file name from the environment; a library built without CRV_TRACE says so instead of writing zeros
static inline const char *trace_env(const char *name) {
    const char *e = getenv(name);
#if !CRV_TRACE
    if (e) {
        static bool warned = false;
        if (!warned) fprintf(stderr, "crvpinn: %s ignored: this library was built without -DCRV_TRACE=1\n", name);
        warned = true;
        return nullptr;
    }
#endif
    return e;
}
#if CRV_TRACE
#define FTRACE(slot) do { if (a.trace && blockIdx.x == 0 && (slot) < 4096) a.trace[(slot)] = clock64(); } while (0)
#else
#define FTRACE(slot) do { } while (0)
#endif



constexpr int NQ = 2;   // N-parts of the last K chunk of each GEMM, each committed on its own barrier
// the MMA issuer's waits suspend (try_wait with a time hint) so they do not take the epilogue warps'
// issue slots on the shared SMSP; the epilogue's accumulator waits poll
#define FWD_MMA_WAIT mbar_wait_sleep
#define FWD_EPI_WAIT mbar_wait

constexpr float TANH_C = 2.8853900817779268f;   // 2 log2(e): tanh(z) = 1 - 2 / (1 + 2^(TANH_C z))
// activation scale of every fp16 activation operand and stored activation: t' = 2^14 t
constexpr float ACT_INV = 1.0f / 16384.0f;
// the backward's factor on (Delta_out W~)(.)(1 - t^2) for GEMM g: 2^(wexp - fexp), and with t' = 2^14 t,
// k (1 - t^2) = k - (k 2^-28) t'^2
__device__ __forceinline__ float bwd_k(const DevState *st, int g) { return ldexpf(1.0f, st->wexp[g] - st->fexp[g]); }
constexpr int FWD_EPI_WARPS = 16;                       // 4 per TMEM lane quarter
constexpr int FWD_THREADS = 64 + 32 * FWD_EPI_WARPS;     // producer warp + MMA warp + epilogue

// the forward keeps its activations (A operands) in TMEM; shared memory holds the weight ring
template <int WP>
__host__ __device__ constexpr int fwd_nstw() { return WP == 256 ? 4 : (WP == 128 ? 4 : 2); }
template <int WP>
__host__ __device__ constexpr uint32_t fwd_smem_bytes(int L) {
    return 1024 + (WP / 64) * CHUNK_BYTES + fwd_nstw<WP>() * WP * 128 + (2 * WP + L * WP + WP + 1 + 2 * 4 * 128 + 2 * L) * 4 +
           40 * 8 + 16;
}

// Pipelining: two TMEM accumulators (GEMMs alternate) and per-64-feature-chunk
// barriers a_full[c]: the epilogue producing activation t_a chunk c releases it to the MMA of the
// next GEMM immediately, so that GEMM runs under the rest of the epilogue. 16 epilogue warps work
// on the same chunk at a time (the 4 warps sharing a TMEM lane quarter take 16 columns each);
// there is no block-wide barrier inside a tile. t_hi goes to HBM straight from registers
// (one 32-byte sector per thread and chunk). (Pre-scaling the fp16 weights by 2 log2 e to save
// the multiply in tanh was measured 3-4x less accurate in u on B200 and is not used.)
// EVAL = true: the same network at arbitrary points a.xy (continuous evaluation, f1 / SPEC.md:493-501):
// no activations are stored and u[p] = cutoff(x_p, y_p) net(x_p, y_p) for p < npts.
// EW epilogue warps: 16 (one CTA per SM; 18 warps -> <= 96 regs) or 8 (two CTAs per SM at WP <= 128, so
// that two tiles are in flight per SM: one CTA's epilogue runs while the other's MMAs do)
template <int EW>
__host__ __device__ constexpr int fwd_threads() { return 64 + 32 * EW; }
template <int WP, bool EVAL = false, int EW = FWD_EPI_WARPS>
__global__ void __launch_bounds__(fwd_threads<EW>(), EW == 8 ? 2 : 1) k_tc_forward(FwdArgs a) {
    constexpr int KC = WP / 64;
    constexpr int WQ = EW / 4;      // epilogue warps per TMEM lane quarter
    constexpr int SPW = 4 / WQ;     // 16-column slices per warp and 64-column chunk
    constexpr uint32_t WBLK = WP * 128;
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = align1024(smem_raw);
    constexpr int NSW = fwd_nstw<WP>();
    uint8_t *Th = smem;                  // [KC] chunks: t'_hi staging for the bulk copies to HBM
    uint8_t *Wr = Th + KC * CHUNK_BYTES;
    float *sW1 = (float *)(Wr + NSW * WBLK);
    float *sB = sW1 + 2 * WP;
    float *sWo = sB + a.L * WP;          // WP + 1 (bias last)
    float *sRed = sWo + WP + 1;          // [2 parity][4][128]
    float *sC = sRed + 2 * 4 * 128;      // [G] epilogue factor of GEMM g: 2 log2(e) 2^(wexp[g] - 14)
    int *sAcc = (int *)(sC + a.L);       // [L] layer l's tanh must be accurate for small |t| (next GEMM's gain >= 16)
    uint64_t *bars = (uint64_t *)(((uintptr_t)(sAcc + a.L) + 7) & ~(uintptr_t)7);
    uint64_t *w_full = bars, *w_empty = bars + NSW;
    uint64_t *a_full = bars + 2 * NSW;            // [KC]
    uint64_t *acc_full = a_full + KC;             // [2 accumulators][NQ N-parts]
    uint32_t *tmem_slot = (uint32_t *)(acc_full + 2 * NQ);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < NSW; ++s) {
            mbar_init(&w_full[s], 1);
            mbar_init(&w_empty[s], 1);
        }
        for (int c = 0; c < KC; ++c) mbar_init(&a_full[c], EW);
        for (int i = 0; i < 2 * NQ; ++i) mbar_init(&acc_full[i], 1);
        fence_mbar_init();
    }
    if (warp == 1) tmem_alloc(tmem_slot, 2 * WP);
    // everything above is local; the weights (written by the previous iteration's Adam) are read
    // only after the programmatic dependency resolves
    pdl_wait();
    pdl_trigger();
    for (int i = threadIdx.x; i < 2 * WP; i += blockDim.x) sW1[i] = a.W1p[i];
    for (int i = threadIdx.x; i < a.L * WP; i += blockDim.x) sB[i] = a.bp[i];
    for (int i = threadIdx.x; i < WP + 1; i += blockDim.x) sWo[i] = a.Wop[i];
    // GEMM g accumulates t' W~ = 2^(14 - wexp[g]) t W (activations t' = 2^14 t, weights W 2^-wexp[g])
    for (int i = threadIdx.x; i < a.G; i += blockDim.x) sC[i] = ldexpf(TANH_C, a.st->wexp[i] - 14);
    for (int i = threadIdx.x; i < a.L; i += blockDim.x) sAcc[i] = i < a.G && a.st->fexp[i] >= 4;
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        // ---------------- producer: weight K-chunks through the ring (bulk copies)
        if (lane == 0 && a.G > 0) {
            int stage = 0;
            uint32_t ph = 0;
            for (int tile = blockIdx.x; tile < a.ntiles; tile += gridDim.x)
                for (int g = 0; g < a.G; ++g)
                    for (int c = 0; c < KC; ++c) {
                        mbar_wait_sleep(&w_empty[stage], ph ^ 1);
                        mbar_arrive_expect_tx(&w_full[stage], WBLK);
                        bulk_g2s(Wr + stage * WBLK, (const uint8_t *)a.Wf + (size_t)(g * KC + c) * WBLK, WBLK,
                                 &w_full[stage]);
                        if (++stage == NSW) { stage = 0; ph ^= 1; }
                    }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer (one thread). GEMM gi accumulates into TMEM region (gi & 1) and
        // takes its A operand (hi/lo activations) from region ((gi + 1) & 1), where the epilogue wrote it
        // in place of the accumulator it read (16-feature slice k of chunk c: hi in the slice's first 8
        // columns, lo in the next 8)
        if (lane == 0 && a.G > 0) {
            constexpr uint32_t idesc = idesc_f16(128, WP, 0, 0);
            constexpr uint32_t idesc_h = idesc_f16(128, WP / NQ, 0, 0);
            int stage = 0;
            uint32_t ph = 0, aph = 0;
            uint32_t dph = 0u;   // bit i: parity of acc_full[i] as seen by this thread
            int gi = 0;          // running GEMM counter
            const uint32_t wr = smem_u32(Wr);
            for (int tile = blockIdx.x; tile < a.ntiles; tile += gridDim.x)
                for (int g = 0; g < a.G; ++g, ++gi) {
                    const uint32_t acc = tmem + (uint32_t)((gi & 1) * WP);
                    const uint32_t asrc = tmem + (uint32_t)(((gi + 1) & 1) * WP);
                    // region (gi & 1) held GEMM gi-1's A operand: its MMAs must be complete before the
                    // first MMA of GEMM gi overwrites it
                    if (gi > 0) {
                        const int pb = ((gi - 1) & 1) * NQ + NQ - 1;
                        FWD_MMA_WAIT(&acc_full[pb], (dph >> pb) & 1u);
                    }
                    if (gi > 0) {
                        const int pb0 = ((gi - 1) & 1) * NQ;
                        for (int hh = 0; hh < NQ; ++hh) dph ^= 1u << (pb0 + hh);
                    }
                    for (int c = 0; c < KC; ++c) {
                        FWD_MMA_WAIT(&a_full[c], aph);
                        FTRACE(2048 + (gi * KC + c) * 4 + 0);
                        if constexpr (!EVAL) {   // t'_hi chunk c of layer g+1 -> HBM
                            bulk_s2g(a.act + ((size_t)g * a.ntiles + tile) * (KC * CHUNK_HALVES) + c * CHUNK_HALVES,
                                     Th + c * CHUNK_BYTES, CHUNK_BYTES);
                            bulk_commit();
                        }
                        FWD_MMA_WAIT(&w_full[stage], ph);
                        FTRACE(2048 + (gi * KC + c) * 4 + 1);
                        tc_fence_after();
                        if (c + 1 < KC) {
#pragma unroll
                            for (int kk = 0; kk < 4; ++kk) {
                                const uint64_t bd = sdesc_sw128(wr + stage * WBLK + kk * 32, 16, 1024);
                                const uint32_t ah = asrc + (uint32_t)(c * 64 + kk * 16);
                                mma_f16_ts(acc, ah, bd, idesc, (c | kk) != 0);
                                mma_f16_ts(acc, ah + 8, bd, idesc, 1u);
                            }
                            if (c + 1 == KC) {
                                if constexpr (!EVAL) bulk_wait_read0();
                                for (int hh = 0; hh < NQ; ++hh) mma_commit(&acc_full[(gi & 1) * NQ + hh]);
                            }
                        } else {
                            // last K chunk in N parts, each committed on its own barrier: the next
                            // epilogue starts on the first part while the MMAs for the rest still run
                            // -- and rewrites the staging chunks, so their HBM copies must have read them
                            if constexpr (!EVAL) bulk_wait_read0();
#pragma unroll
                            for (int hh = 0; hh < NQ; ++hh) {
#pragma unroll
                                for (int kk = 0; kk < 4; ++kk) {
                                    const uint64_t bd =
                                        sdesc_sw128(wr + stage * WBLK + hh * (WP / NQ) * 128 + kk * 32, 16, 1024);
                                    const uint32_t ah = asrc + (uint32_t)(c * 64 + kk * 16);
                                    mma_f16_ts(acc + hh * (WP / NQ), ah, bd, idesc_h, (c | kk) != 0);
                                    mma_f16_ts(acc + hh * (WP / NQ), ah + 8, bd, idesc_h, 1u);
                                }
                                mma_commit(&acc_full[(gi & 1) * NQ + hh]);
                            }
                        }
                        FTRACE(2048 + (gi * KC + c) * 4 + 2);
                        mma_commit(&w_empty[stage]);
                        if (++stage == NSW) { stage = 0; ph ^= 1; }
                    }
                    aph ^= 1;
                }
            bulk_wait0();
        }
    } else {
        // ---------------- epilogue: EW warps; warp % 4 = TMEM lane quarter (rows), wq = which
        // 16-column slices of each 64-column chunk
        const int q = warp & 3;
        const int row = q * 32 + lane;
        const int wq = (warp - 2) >> 2;                           // slices wq, wq + WQ, ... of each chunk
        const uint32_t t_lane = tmem + ((uint32_t)(q * 32) << 16);
        const bool swap = (row & 1) != 0;
        // slice sl = 16 columns = logical granules 2 sl, 2 sl + 1: shared-memory offsets and 32-byte sector
        auto off0 = [&](int sl) { return (uint32_t)(row * 128 + (((2 * sl) ^ (row & 7)) << 4)); };
        auto off1 = [&](int sl) { return (uint32_t)(row * 128 + (((2 * sl + 1) ^ (row & 7)) << 4)); };
        auto pos = [&](int sl) { return ((2 * sl) ^ (row & 7)) & ~1; };
        uint32_t acc_ph = 0u;   // bit i: parity of acc_full[i]
        int gi = 0, par = 0;
        const int N = a.N;
        for (int tile = blockIdx.x; tile < a.ntiles; tile += gridDim.x, par ^= 1) {
            const int p = tile * 128 + row;
            int pi = 0, pj = 0;
            float x, y;
            if constexpr (EVAL) {
                const bool ok = p < a.npts;
                x = ok ? __ldg(a.xy + 2 * (long)p) : 0.0f;
                y = ok ? __ldg(a.xy + 2 * (long)p + 1) : 0.0f;
            } else {
                point_ij(a.p0 + p, N, pi, pj);
                x = (float)pi / (float)N;
                y = (float)pj / (float)N;
            }
            float dot = 0.0f;
            for (int layer = 1; layer <= a.L; ++layer) {
                const bool last = layer == a.L;
                uint32_t acc = 0;
                // where this layer's activations go (the A operand of GEMM gi', the next one): region
                // ((gi' + 1) & 1) -- for layer 1 (gi' = gi) the previous GEMM's region, for layer > 1
                // (gi' = gi + 1 after the wait) the accumulator region read here, in place
                uint32_t aout = (uint32_t)(((gi + 1) & 1) * WP);
                int ab = 0;          // first acc_full barrier of this layer's accumulator
                uint32_t got = ~0u;  // bit p: output part [p WP/NQ, (p+1) WP/NQ) available
                if (layer > 1) {
                    const int ai = gi & 1;
                    ab = ai * NQ;
                    if (warp == 2 && lane == 0) FTRACE(gi * 16 + 0);
                    FWD_EPI_WAIT(&acc_full[ab], (acc_ph >> ab) & 1u);
                    if (warp == 2 && lane == 0) FTRACE(gi * 16 + 1);
                    if (lane == 0 && gi < 12) FTRACE(1024 + (gi * (KC + 1)) * 16 + (warp - 2));
                    acc_ph ^= 1u << ab;
                    acc = (uint32_t)(ai * WP);
                    aout = acc;
                    got = 1u;
                    ++gi;
                    tc_fence_after();
                }
                const float *bias = sB + (layer - 1) * WP;
                // 2 log2(e) 2^(wexp - 14): undoes the operand scales (one shared-memory load per layer)
                const float cg = layer > 1 ? lds_f32(sC + layer - 2) : 0.0f;
                uint8_t *grow = (uint8_t *)(a.act + ((size_t)(layer - 1) * a.ntiles + tile) * (KC * CHUNK_HALVES)) +
                                row * 128;
                // TMEM loads run one slice ahead of the math; every layer stores t'_hi to HBM from
                // registers (there is no shared-memory A operand any more, hence no proxy fence).
                uint32_t rbuf[16];
                auto need_half1 = [&](int col) {   // wait for the N-part holding column col
                    const int pp = col / (WP / NQ);
                    if (!((got >> pp) & 1u)) {
                        for (int q2 = 1; q2 <= pp; ++q2)
                            if (!((got >> q2) & 1u)) {
                                FWD_EPI_WAIT(&acc_full[ab + q2], (acc_ph >> (ab + q2)) & 1u);
                                acc_ph ^= 1u << (ab + q2);
                                got |= 1u << q2;
                            }
                        tc_fence_after();
                    }
                };
                if (layer > 1) {
                    need_half1(wq * 16);
                    tmem_ld16_async(t_lane + acc + wq * 16, rbuf);
                }
                // release chunk c to the next GEMM (and its HBM copy); one arrival per warp
                auto release = [&](int c) {
                    if constexpr (!EVAL) fence_proxy_async_smem();
                    tmem_wait_st();
                    tc_fence_before();
                    __syncwarp();
                    if (warp == 2 && lane == 0) FTRACE(gi * 16 + 2 + c);
                    if (lane == 0 && gi < 12) FTRACE(1024 + (gi * (KC + 1) + 1 + c) * 16 + (warp - 2));
                    if (lane == 0) mbar_arrive(&a_full[c]);
                };
                // work items (chunk c, slice sl = wq + s WQ) in order; TMEM loads run one item ahead
                // the chunk loop, instantiated for the accurate-tanh layers and for the rest (a uniform
                // branch per layer, so the common path carries no code of the other)
                auto chunks = [&](auto EXACT) {
#pragma unroll
                for (int it = 0; it < KC * SPW; ++it) {
                    const int c = it / SPW, sp = it % SPW, sl = wq + sp * WQ;
                    const int cc = c * 64 + sl * 16;
                    float v[16];
                    if (layer == 1) {
#pragma unroll
                        for (int k = 0; k < 16; k += 4) {
                            const float4 w4a = lds_f4(sW1 + 2 * (cc + k)), w4b = lds_f4(sW1 + 2 * (cc + k) + 4);
                            const float4 b4 = lds_f4(bias + cc + k);
                            v[k] = fmaf(w4a.x, x, fmaf(w4a.y, y, b4.x));
                            v[k + 1] = fmaf(w4a.z, x, fmaf(w4a.w, y, b4.y));
                            v[k + 2] = fmaf(w4b.x, x, fmaf(w4b.y, y, b4.z));
                            v[k + 3] = fmaf(w4b.z, x, fmaf(w4b.w, y, b4.w));
                        }
                    } else {
                        tmem_wait_ld16(rbuf);
                        const f32x2_t C2 = pk2(cg, cg);
#pragma unroll
                        for (int k = 0; k < 16; k += 4) {
                            const float4 b4 = lds_f4(bias + cc + k);   // 2 log2(e) b
                            upk2(ffma2(pk2(__uint_as_float(rbuf[k]), __uint_as_float(rbuf[k + 1])), C2, pk2(b4.x, b4.y)),
                                 v[k], v[k + 1]);
                            upk2(ffma2(pk2(__uint_as_float(rbuf[k + 2]), __uint_as_float(rbuf[k + 3])), C2, pk2(b4.z, b4.w)),
                                 v[k + 2], v[k + 3]);
                        }
                        if (it + 1 < KC * SPW) {
                            const int nc = (it + 1) / SPW * 64 + (wq + (it + 1) % SPW * WQ) * 16;
                            need_half1(nc);
                            tmem_ld16_async(t_lane + acc + nc, rbuf);
                        }
                    }
                    // v = 2 log2(e) z; tanh(z) = 1 - 2 / (1 + 2^v) for 16 elements as a skewed pipeline:
                    // ex2 of element i, the reciprocal of element i-2 and the finish (t' = 2^14 t, hi/lo
                    // split, fp16 pack) of pair (i-5, i-4) are issued together, so MUFU and ALU work
                    // interleave. Even elements take the MUFU reciprocal, odd ones a Newton reciprocal on
                    // the FMA pipe, two of them (k-2, k) per packed step (FFMA2) when k = 3 mod 4 (MUFU : ALU
                    // balance); only the Newton elements need a finite 1 + 2^v (rcp.approx(inf) = 0).
                    uint32_t hw[8], lw[8];
                    float e[16], r[16];
                    if constexpr (decltype(EXACT)::value) {
                        // accurate-tanh layer (its activations feed a GEMM with a large gain):
                        // the formula below is accurate to ~2^-22 ABSOLUTE, which that gain would amplify
                        // for small |t|; here |z| < 1/8 takes the odd Taylor polynomial (relative error
                        // < 2e-9), the rest the same exp formula
#pragma unroll
                        for (int k = 0; k < 16; ++k) {
                            const float tb = fmaf(-2.0f, rcp_v(1.0f + ex2_v(fminf(v[k], 60.0f))), 1.0f);
                            const float z = v[k] * (1.0f / TANH_C), z2 = z * z;
                            const float ts = z * fmaf(z2, fmaf(z2, fmaf(z2, -17.0f / 315.0f, 2.0f / 15.0f), -1.0f / 3.0f), 1.0f);
                            r[k] = fabsf(z) < 0.125f ? ts : tb;   // r holds t on this path
                        }
#pragma unroll
                        for (int m = 0; m < 8; ++m) finish_pair_t(r[2 * m], r[2 * m + 1], hw[m], lw[m]);
                        if (last) {
#pragma unroll
                            for (int k = 0; k < 16; ++k) v[k] = r[k];
                        }
                    } else {
#pragma unroll
                    for (int i = 0; i < 16 + 5; ++i) {
                        if (i < 16) e[i] = ex2_v((i & 1) ? fminf(v[i], 60.0f) : v[i]);
                        if (i >= 2 && i < 18) {
                            const int k = i - 2;
                            if ((k & 1) == 0) {
                                r[k] = rcp_v(1.0f + e[k]);
                            } else if ((k & 3) == 3) {
                                const float da = 1.0f + e[k - 2], db = 1.0f + e[k];
                                f32x2_t R = pk2(__int_as_float(0x7EF311C3 - __float_as_int(da)),
                                                __int_as_float(0x7EF311C3 - __float_as_int(db)));
                                const f32x2_t ND = pk2(-da, -db), ONE = pk2(1.0f, 1.0f);
#pragma unroll
                                for (int it = 0; it < 3; ++it) R = ffma2(R, ffma2(ND, R, ONE), R);
                                upk2(R, r[k - 2], r[k]);
                            }
                        }
                        if (i >= 5 && ((i - 5) & 1) == 0) {
                            const int m = (i - 5) >> 1;
                            if (m < 8) finish_pair(r[2 * m], r[2 * m + 1], hw[m], lw[m]);
                        }
                    }
                    if (last) {   // the output layer takes t itself (fp32)
#pragma unroll
                        for (int k = 0; k < 16; ++k) v[k] = fmaf(-2.0f, r[k], 1.0f);
                    }
                    }
                    if (!last) {
                        // the next GEMM's A operand, in place of the accumulator slice just read; t'_hi
                        // also into the staging chunk that the MMA thread bulk-copies to HBM (the
                        // backward's operand: stores from the epilogue's registers cost ~20 % of the
                        // forward, the TMA engine does them for free)
                        tmem_st16(t_lane + aout + (uint32_t)cc, hw, lw);
                        if constexpr (!EVAL) {
                            const uint32_t bh = smem_u32(Th) + c * CHUNK_BYTES;
                            st_shared_v4(bh + off0(sl), hw[0], hw[1], hw[2], hw[3]);
                            st_shared_v4(bh + off1(sl), hw[4], hw[5], hw[6], hw[7]);
                        }
                        if (sp == SPW - 1) release(c);
                    } else {
#pragma unroll
                        for (int k = 0; k < 16; k += 4) {
                            const float4 w4 = lds_f4(sWo + cc + k);
                            dot = fmaf(w4.x, v[k], fmaf(w4.y, v[k + 1], fmaf(w4.z, v[k + 2], fmaf(w4.w, v[k + 3], dot))));
                        }
                        if constexpr (!EVAL) {
                            uint8_t *gp = grow + c * CHUNK_BYTES + pos(sl) * 16;
                            if (swap)
                                st_global_v8(gp, hw[4], hw[5], hw[6], hw[7], hw[0], hw[1], hw[2], hw[3]);
                            else
                                st_global_v8(gp, hw[0], hw[1], hw[2], hw[3], hw[4], hw[5], hw[6], hw[7]);
                        }
                    }
                }
                };
                if (sAcc[layer - 1]) chunks(std::true_type{});
                else chunks(std::false_type{});
            }
            // output layer: net = W_out t_L + b_out; u = cutoff * net (WQ partial dots per row)
            sRed[(par * 4 + wq) * 128 + row] = dot;
            named_bar(1, 32 * EW);
            if (wq == 0) {
                const float *r = sRed + par * 4 * 128 + row;
                const float net = (WQ == 4 ? ((r[0] + r[128]) + (r[256] + r[384])) : (r[0] + r[128])) + sWo[WP];
                if constexpr (EVAL) {
                    if (p < a.npts) a.u[p] = cutoff(x, y) * net;
                } else {
                    a.u[(long)pj * (N + 1) + pi] = cutoff(x, y) * net;
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) tmem_dealloc(tmem, 2 * WP);
}

// ================================================================ backward: output layer
// Delta_L = s * gbar * W_out (.) (1 - t_L^2) (fp16, tile-chunk format), with
// s = 2^(7 - ceil(log2 max|gbar|)) so max|s gbar| is in (64, 128].
// Partials per block: [WP] sum s*gbar*t_L (dW_out) | [WP] sum Delta_L (db) | [1] sum s*gbar (db_out).
// ew = ceil(log2 max|W_out|) (0 for a zero output layer): Delta_L = s gbar W_out (1 - t_L^2) then has
// max |Delta_L| <= 128 whatever the magnitudes of gbar and W_out (fp16 holds 65504)
__device__ __forceinline__ int wout_exp(float womax) {
    return (womax > 0.0f && isfinite(womax)) ? (int)ceilf(log2f(womax)) : 0;
}
__device__ __forceinline__ float grad_scale(const DevState *st, int ew) {
    float gm = __uint_as_float(st->gmax_bits);
    if (!(gm > 0.0f) || !isfinite(gm)) return 1.0f;
    int e = 7 - (int)ceilf(log2f(gm)) - ew;
    e = e < -126 ? -126 : (e > 126 ? 126 : e);
    return exp2f((float)e);
}

constexpr int OB_THREADS = 256;

// Vectorised: thread T owns logical granule lg = T%8 (8 features) of chunk c = (T/8)%KC for the
// rows r = rg, rg+NRG, ... (rg = T/(8 KC)); a warp covers whole 128-byte rows (coalesced).
// STORE = false: only the output-layer gradient sums (dW_out, db_L, db_out), no Delta_L -- run on the
// side stream next to the first k_tc_bwd2 launch, which then forms Delta_L without the sums
template <int WP, bool STORE = true>
__global__ void __launch_bounds__(OB_THREADS) k_tc_out_bwd(int ntiles, const __half *__restrict__ actL,
                                                           const float *__restrict__ gbar,
                                                           const float *__restrict__ Wop,
                                                           __half *__restrict__ deltaL,
                                                           float *__restrict__ partial, DevState *st) {
    constexpr int KC = WP / 64;
    constexpr int NRG = OB_THREADS / (8 * KC);   // row groups
    constexpr int RPT = 128 / NRG;               // rows per thread per tile
    __shared__ float sred[2][NRG][WP];
    __shared__ float sgsum[NRG];
    __shared__ float swo;
    const int T = threadIdx.x;
    const int lg = T & 7, c = (T >> 3) % KC, rg = T / (8 * KC);
    const int f0 = c * 64 + lg * 8;
    // a thread's RPT rows of one tile: t_L granules and gbar, loaded together (every input is complete
    // at launch); the next tile's are in flight while this one is transformed
    uint4 raw[RPT];
    float gr[RPT];
    auto fetch = [&](int tl) {
        const uint8_t *src = (const uint8_t *)actL + ((size_t)tl * KC + c) * CHUNK_BYTES;
#pragma unroll
        for (int k = 0; k < RPT; ++k) {
            const int r = rg + k * NRG;
            raw[k] = __ldg((const uint4 *)(src + (uint32_t)(r * 128 + ((lg ^ (r & 7)) << 4))));
            gr[k] = __ldg(gbar + tl * 128 + r);
        }
    };
    if ((int)blockIdx.x < ntiles) fetch(blockIdx.x);
    if (T < 32) {   // max |W_out| (order-independent: every block gets the same value)
        float m = 0.0f;
        for (int f = T; f < WP; f += 32) m = fmaxf(m, fabsf(Wop[f]));
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
        if (T == 0) swo = m;
    }
    __syncthreads();
    const float s = grad_scale(st, wout_exp(swo));
    if (blockIdx.x == 0 && T == 0) {
        st->gscale = s;
        st->inv_gscale = 1.0f / s;
    }
    float wo[8], aw[8], ab[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) { wo[e] = Wop[f0 + e]; aw[e] = 0.0f; ab[e] = 0.0f; }
    float ag = 0.0f;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        uint4 cur[RPT];
        float gc[RPT];
#pragma unroll
        for (int k = 0; k < RPT; ++k) { cur[k] = raw[k]; gc[k] = gr[k]; }
        if (tile + (int)gridDim.x < ntiles) fetch(tile + gridDim.x);
        uint8_t *dst = (uint8_t *)deltaL + ((size_t)tile * KC + c) * CHUNK_BYTES;
#pragma unroll
        for (int k = 0; k < RPT; ++k) {
            const int r = rg + k * NRG;
            const uint32_t off = (uint32_t)(r * 128 + ((lg ^ (r & 7)) << 4));
            const float g = gc[k] * s;
            ag += g;
            uint32_t w[4] = {cur[k].x, cur[k].y, cur[k].z, cur[k].w};
#pragma unroll
            for (int m = 0; m < 4; ++m) {
                float2 t = __half22float2(*reinterpret_cast<__half2 *>(&w[m]));
                t.x *= ACT_INV;   // stored activations are t' = 2^14 t
                t.y *= ACT_INV;
                const float d0 = g * wo[2 * m] * (1.0f - t.x * t.x);
                const float d1 = g * wo[2 * m + 1] * (1.0f - t.y * t.y);
                aw[2 * m] = fmaf(g, t.x, aw[2 * m]);
                aw[2 * m + 1] = fmaf(g, t.y, aw[2 * m + 1]);
                ab[2 * m] += d0;
                ab[2 * m + 1] += d1;
                if constexpr (STORE) w[m] = pack_half2(d0, d1);
            }
            if constexpr (STORE) *(uint4 *)(dst + off) = make_uint4(w[0], w[1], w[2], w[3]);
        }
    }
    // fixed-order combination over row groups
#pragma unroll
    for (int e = 0; e < 8; ++e) {
        sred[0][rg][f0 + e] = aw[e];
        sred[1][rg][f0 + e] = ab[e];
    }
    if (c == 0 && lg == 0) sgsum[rg] = ag;
    __syncthreads();
    float *pb = partial + (size_t)blockIdx.x * (2 * WP + 1);
    for (int f = T; f < WP; f += OB_THREADS) {
        float sw = 0.0f, sb = 0.0f;
        for (int q = 0; q < NRG; ++q) { sw += sred[0][q][f]; sb += sred[1][q][f]; }
        pb[f] = sw;
        pb[WP + f] = sb;
    }
    if (T == 0) {
        float sgt = 0.0f;
        for (int q = 0; q < NRG; ++q) sgt += sgsum[q];
        pb[2 * WP] = sgt;
    }
}

// ================================================================ backward: fused layer (dX + dW)
// One launch per hidden GEMM g: reads Delta_out (= Delta_{g+2}) and t_in (= t_{g+1}) ONCE and
// produces both Delta_in = (Delta_out W) (.) (1 - t_in^2) and this CTA's share of
// dW = sum_p Delta_out^T t_in. TMEM: dX accumulator (WP columns) + dW accumulator (WP columns,
// M = 128 out features). For WP = 256 the 256 out features do not fit one CTA's TMEM next to
// the dX accumulator, so CTAs work in PAIRS on the same tile sequence: CTA k of a pair owns dW
// rows [128k, 128k+128) for every tile of the pair and computes dX for every other tile; the
// second read of each tile is an L2 hit. For WP <= 128 (PF = 1) each CTA does everything.
struct BwdArgs {
    int N, ntiles, first, npairs;
    const __half *dout;   // Delta_{g+2}  [ntiles][KC] blocks
    const __half *tin;    // t_{g+1}      [ntiles][KC]
    __half *din;          // Delta_{g+1}  [ntiles][KC]
    const __half *WTf;    // [KC] blocks of W^T
    float *part_dx;       // [grid][3*WP]   column sums (xy-weighted | plain)
    float *part_dw;       // [npairs][WP*WP] rows = out features
    int p0;               // first MLP point of this shard
    const DevState *st;   // weight / Delta exponents of GEMM g
    int g;
};

template <int WP>
__host__ __device__ constexpr int bwd_pf() { return WP > 128 ? 2 : 1; }

template <int WP>
__host__ __device__ constexpr uint32_t bwd_smem_bytes() {
    return 1024 + 2 * (WP / 64) * CHUNK_BYTES + (WP == 64 ? CHUNK_BYTES : 0) + NST_W * WP * 128 +
           4 * 3 * WP * 4 + 16 * 8 + 16;
}

template <int WP>
__global__ void __launch_bounds__(TC_THREADS, 1) k_tc_bwd_layer(BwdArgs a) {
    constexpr int KC = WP / 64;
    constexpr int PF = bwd_pf<WP>();
    constexpr uint32_t WBLK = WP * 128;
    constexpr uint32_t TILE_BYTES = KC * CHUNK_BYTES;
    // Delta_out buffer is followed by a zero block when WP = 64 (dW M = 128 reads 2 chunks)
    constexpr uint32_t ABUF = TILE_BYTES + (WP == 64 ? CHUNK_BYTES : 0);
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = align1024(smem_raw);
    uint8_t *Ab = smem;
    uint8_t *Tb = Ab + ABUF;
    uint8_t *Wr = Tb + TILE_BYTES;
    float *sRed = (float *)(Wr + NST_W * WBLK);
    uint64_t *bars = (uint64_t *)(sRed + 4 * 3 * WP);
    uint64_t *w_full = bars, *w_empty = bars + NST_W;
    uint64_t *ld_full = bars + 2 * NST_W, *ld_empty = ld_full + 1, *acc_full = ld_full + 2,
             *acc_empty = ld_full + 3, *dw_full = ld_full + 4;
    uint32_t *tmem_slot = (uint32_t *)(dw_full + 1);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int pair = blockIdx.x / PF, kk_pf = blockIdx.x % PF;
    if (WP == 64) {
        for (int i = threadIdx.x; i < (int)(CHUNK_BYTES / 16); i += blockDim.x)
            ((uint4 *)(Ab + TILE_BYTES))[i] = make_uint4(0, 0, 0, 0);
        fence_proxy_async_smem();
    }
    if (threadIdx.x == 0) {
        for (int s = 0; s < NST_W; ++s) {
            mbar_init(&w_full[s], 1);
            mbar_init(&w_empty[s], 1);
        }
        mbar_init(ld_full, 1);
        mbar_init(ld_empty, 1);
        mbar_init(acc_full, 1);
        mbar_init(acc_empty, EPI_THREADS / 32);
        mbar_init(dw_full, 1);
        fence_mbar_init();
    }
    if (warp == 1) tmem_alloc(tmem_slot, 2 * WP);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const uint32_t tm_dx = tmem, tm_dw = tmem + WP;

    if (warp == 0) {
        if (lane == 0) {
            int stage = 0;
            uint32_t ph = 0;
            int i = 0;
            for (int tile = pair; tile < a.ntiles; tile += a.npairs, ++i) {
                mbar_wait_sleep(ld_empty, (i & 1) ^ 1);
                mbar_arrive_expect_tx(ld_full, 2 * TILE_BYTES);
                bulk_g2s(Ab, (const uint8_t *)a.dout + (size_t)tile * TILE_BYTES, TILE_BYTES, ld_full);
                bulk_g2s(Tb, (const uint8_t *)a.tin + (size_t)tile * TILE_BYTES, TILE_BYTES, ld_full);
                if (i % PF == kk_pf) {
                    for (int c = 0; c < KC; ++c) {
                        mbar_wait(&w_empty[stage], ph ^ 1);
                        mbar_arrive_expect_tx(&w_full[stage], WBLK);
                        bulk_g2s(Wr + stage * WBLK, (const uint8_t *)a.WTf + (size_t)c * WBLK, WBLK, &w_full[stage]);
                        if (++stage == NST_W) { stage = 0; ph ^= 1; }
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            constexpr uint32_t idesc_dx = idesc_f16(128, WP, 0, 0);
            constexpr uint32_t idesc_dw = idesc_f16(128, WP, 1, 1);
            int stage = 0;
            uint32_t ph = 0;
            int i = 0, ndx = 0;
            const uint32_t ab = smem_u32(Ab), tb = smem_u32(Tb), wr = smem_u32(Wr);
            const uint32_t a_dw = ab + (uint32_t)(2 * kk_pf) * CHUNK_BYTES;   // out-feature chunks 2k, 2k+1
            for (int tile = pair; tile < a.ntiles; tile += a.npairs, ++i) {
                mbar_wait(ld_full, i & 1);
                tc_fence_after();
                // dW share: D[o][i] += sum_p Delta_out[p][o] t_in[p][i], K = 128 points (8 x 16)
#pragma unroll
                for (int ks = 0; ks < 8; ++ks) {
                    const uint64_t ad = sdesc_sw128(a_dw + ks * 2048, CHUNK_BYTES, 1024);
                    const uint64_t bd = sdesc_sw128(tb + ks * 2048, CHUNK_BYTES, 1024);
                    mma_f16(tm_dw, ad, bd, idesc_dw, (i | ks) != 0);
                }
                if (i % PF == kk_pf) {
                    mbar_wait(acc_empty, (ndx & 1) ^ 1);
                    tc_fence_after();
                    for (int c = 0; c < KC; ++c) {
                        mbar_wait(&w_full[stage], ph);
                        tc_fence_after();
#pragma unroll
                        for (int kq = 0; kq < 4; ++kq) {
                            const uint64_t ad = sdesc_sw128(ab + c * CHUNK_BYTES + kq * 32, 16, 1024);
                            const uint64_t bd = sdesc_sw128(wr + stage * WBLK + kq * 32, 16, 1024);
                            mma_f16(tm_dx, ad, bd, idesc_dx, (c | kq) != 0);
                        }
                        mma_commit(&w_empty[stage]);
                        if (++stage == NST_W) { stage = 0; ph ^= 1; }
                    }
                    mma_commit(acc_full);
                    ++ndx;
                }
                mma_commit(ld_empty);
            }
            mma_commit(dw_full);
        }
    } else {
        const int q = warp & 3;
        const int row = q * 32 + lane;
        const int hf = (warp - 2) >> 2;
        constexpr int HALF = WP / 2;
        constexpr int NCH = HALF / 32;
        const int col0 = hf * HALF;
        const int ep_tid = threadIdx.x - 64;
        const uint32_t t_lane = (uint32_t)(q * 32) << 16;
        float cs[NCH], csx[NCH], csy[NCH];
#pragma unroll
        for (int k = 0; k < NCH; ++k) cs[k] = csx[k] = csy[k] = 0.0f;
        const int N = a.N;
        const float kx = bwd_k(a.st, a.g), mx = kx * (ACT_INV * ACT_INV);
        int i = 0, ndx = 0;
        for (int tile = pair; tile < a.ntiles; tile += a.npairs, ++i) {
            if (i % PF != kk_pf) continue;
            int pi, pj;
            point_ij(a.p0 + tile * 128 + row, N, pi, pj);
            const float x = (float)pi / (float)N, y = (float)pj / (float)N;
            const uint8_t *trow = (const uint8_t *)a.tin + (size_t)tile * TILE_BYTES + row * 128;
            uint8_t *drow = (uint8_t *)a.din + (size_t)tile * TILE_BYTES + row * 128;
            mbar_wait(acc_full, ndx & 1);
            ++ndx;
            tc_fence_after();
#pragma unroll
            for (int k = 0; k < NCH; ++k) {
                const int cc = col0 + 32 * k;
                const uint32_t cbase = (cc >> 6) * CHUNK_BYTES;
                uint4 tg[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const int lg = ((cc & 63) >> 3) + j;
                    tg[j] = __ldg((const uint4 *)(trow + cbase + ((lg ^ (row & 7)) << 4)));
                }
                float v[32];
                tmem_ld32(tm_dx + t_lane + cc, v);
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    uint32_t w[4] = {tg[j].x, tg[j].y, tg[j].z, tg[j].w};
#pragma unroll
                    for (int m = 0; m < 4; ++m) {
                        float2 tf = __half22float2(*reinterpret_cast<__half2 *>(&w[m]));
                        v[8 * j + 2 * m] *= fmaf(-mx * tf.x, tf.x, kx);
                        v[8 * j + 2 * m + 1] *= fmaf(-mx * tf.y, tf.y, kx);
                        w[m] = pack_half2(v[8 * j + 2 * m], v[8 * j + 2 * m + 1]);
                    }
                    const int lg = ((cc & 63) >> 3) + j;
                    *(uint4 *)(drow + cbase + ((lg ^ (row & 7)) << 4)) = make_uint4(w[0], w[1], w[2], w[3]);
                }
                if (a.first) {
                    float vx[32], vy[32];
#pragma unroll
                    for (int e = 0; e < 32; ++e) { vx[e] = v[e] * x; vy[e] = v[e] * y; }
                    warp_reduce_scatter32(vx, lane);
                    warp_reduce_scatter32(vy, lane);
                    csx[k] += vx[0];
                    csy[k] += vy[0];
                }
                warp_reduce_scatter32(v, lane);
                cs[k] += v[0];
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(acc_empty);
        }
        // column-sum partials (fixed order over the 4 row quarters)
#pragma unroll
        for (int k = 0; k < NCH; ++k) {
            const int col = col0 + 32 * k + lane;
            sRed[(q * 3 + 0) * WP + col] = csx[k];
            sRed[(q * 3 + 1) * WP + col] = csy[k];
            sRed[(q * 3 + 2) * WP + col] = cs[k];
        }
        named_bar(1, EPI_THREADS);
        float *pb = a.part_dx + (size_t)blockIdx.x * 3 * WP;
        for (int col = ep_tid; col < WP; col += EPI_THREADS) {
            float sx = 0.f, sy = 0.f, sb = 0.f;
            for (int qq = 0; qq < 4; ++qq) {
                sx += sRed[(qq * 3 + 0) * WP + col];
                sy += sRed[(qq * 3 + 1) * WP + col];
                sb += sRed[(qq * 3 + 2) * WP + col];
            }
            pb[2 * col] = sx;
            pb[2 * col + 1] = sy;
            pb[2 * WP + col] = sb;
        }
        // dW share -> part_dw[pair][o][i] (rows o = 128k + lane quarter)
        const bool any = pair < a.ntiles;
        if (any) {
            mbar_wait(dw_full, 0);
            tc_fence_after();
        }
        const int o = kk_pf * 128 + row;
        float *pw = a.part_dw + (size_t)pair * WP * WP;
#pragma unroll 1
        for (int cc = hf * HALF; cc < hf * HALF + HALF; cc += 32) {
            float v[32];
            if (any) {
                tmem_ld32(tm_dw + t_lane + cc, v);
            } else {
#pragma unroll
                for (int k = 0; k < 32; ++k) v[k] = 0.0f;
            }
            if (o < WP) {
                float4 *dst = (float4 *)(pw + (size_t)o * WP + cc);
#pragma unroll
                for (int k = 0; k < 8; ++k) dst[k] = make_float4(v[4 * k], v[4 * k + 1], v[4 * k + 2], v[4 * k + 3]);
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) tmem_dealloc(tmem, 2 * WP);
}

// ================================================================ backward v2 (WP >= 128): cluster pairs
// One launch per hidden GEMM g. A cluster of NS = WP/128 CTAs walks a tile sequence; CTA c of
// the cluster owns the input features i in [128c, 128c+128):
//   dX : Delta_in[p, i] = sum_o Delta_out[p, o] W[o, i]      M = 128 points, N = 128 (own i), K = WP
//   dW : dW^T[i, o]    += sum_p t_in[p, i] Delta_out[p, o]   M = 128 (own i), N = WP, K = 128 points
// so every CTA needs the FULL Delta_out tile (bulk-loaded once per cluster with multicast: CTA r
// issues chunks j = r mod NS for both CTAs), only its own half of t_in (unicast), and only its
// own half of W^T, which stays resident in shared memory for the whole launch. Shared memory:
// W^T half (KC x 16 KiB) + Delta ring (KC+2 chunk slots) + t ring (2 tiles x 2 chunks) = 224 KiB
// at WP = 256. L2 traffic per tile is the algorithmic 3 x 64 KiB (Delta_out, t_in, Delta_in).
// TMEM: dX accumulators (2 x 128 columns, double buffered) + dW accumulator (WP columns).
// For the first backward GEMM (outl = 1) the Delta ring receives t_L instead, and the epilogue
// warps turn it into Delta_L = s*gbar*W_out (.) (1 - t_L^2) in place (the output-layer backward,
// fused), reducing the output-layer gradients on the way. The last GEMM (g = 0) does not store
// Delta_1 (only its column sums are needed: bias and first-layer weights).
// SWIZZLE_NONE shared-memory descriptor (LBO/SBO in bytes); with LBO = SBO = 0 every core matrix
// of the operand aliases one 128-byte block -- used for an all-ones A operand (column sums by MMA)
__device__ __forceinline__ uint64_t sdesc_none(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
    d |= (uint64_t)1 << 46;
    return d;
}

struct Bwd2Args {
    int N, ntiles, npairs, first, outl;
    int rev;              // walk the tile sequence backwards (alternating launches: L2 reuse)
    const __half *dsrc;   // Delta_{g+2} (or t_L when outl)   [ntiles][KC] blocks
    const __half *tin;    // t_{g+1}                           [ntiles][KC]
    __half *din;          // Delta_{g+1}                       [ntiles][KC] (unused when first)
    const __half *WTf;    // [KC] blocks of W^T (WP rows each)
    const float *gbar;    // dLOSS/dnet per MLP point (outl)
    const float *Wop;     // output weights (outl)
    float *part_ob;       // [npairs][2*WP+1]  (outl)
    float *part_dx;       // [npairs][3*WP]
    float *part_dw;       // [npairs][WP*WP]   rows = out features
    DevState *st;
    long long *trace;     // debug timeline (CTA 0), nullptr normally
    float *part_cb;       // unused by k_tc_bwd2 (the chain's 1^T Delta_out partials)
    int outl_sums;        // outl: also reduce dW_out / db_L / db_out (else a side-stream k_tc_out_bwd does)
    int p0;               // first MLP point of this shard (gbar is passed offset by it)
    int g;                // hidden GEMM index (weight / Delta exponents)
};
#if CRV_TRACE
#define BTRACE(slot) do { if (a.trace && blockIdx.x == 0 && (slot) < 4096) a.trace[(slot)] = clock64(); } while (0)
#else
#define BTRACE(slot) do { } while (0)
#endif
#define B2_MMA_WAIT mbar_wait

constexpr int B2_EPI_WARPS = 8;    // 2 per TMEM lane quarter
constexpr int B2_EPI_THREADS = 32 * B2_EPI_WARPS;
constexpr int B2_THREADS = 64 + B2_EPI_THREADS;

template <int WP, int MODE = 1>
struct B2 {   // ring geometry; MODE as in k_tc_bwd2 (the output-layer launch keeps 1.5 Delta tiles + 2 t tiles:
              // with one t slot its transform would wait on Delta chunks queued behind t)
    static constexpr int NS = WP / 128;
    static constexpr int KC = WP / 64;
    // Delta ring slots: a tile in flight plus the next pair of chunks (measured: one slot fewer -- 5 at
    // WP = 256 -- hangs the launches, like a single t slot with the output layer fused)
    static constexpr int DS = KC + 2;
    static constexpr int NT = 2;                 // t ring depth (tiles of 2 chunks)
    static constexpr uint32_t SMEM = 1024 + (uint32_t)(KC + DS + 2 * NT) * CHUNK_BYTES + 256 + 64 * 8;   // + ones
};

// MODE bit 0: the first launch (output layer fused, OUTL); bit 1: the last one (g = 0, FIRST).
// Each mode is its own instantiation, so the registers the output-layer transform or the
// first-layer sums need are not reserved in the others.
template <int WP, int MODE>
__global__ void __launch_bounds__(B2_THREADS, 1) k_tc_bwd2(Bwd2Args a) {
    constexpr bool OUTL = (MODE & 1) != 0, FIRST = (MODE & 2) != 0;
    // middle GEMMs release the t slot right after xfull (t values in registers); bias column sums:
    // one butterfly level per tile, the rest once at the end (the g = 0 launch also defers its x-
    // and y-sums); a tile's t_in load goes out before its Delta chunks (with a single t slot it
    // must not sit in front of them)
    constexpr bool EARLY_T = MODE == 0;
    constexpr bool DEFER_CS = true;
    constexpr bool T_FIRST = B2<WP, MODE>::NT > 1;
    constexpr bool DEFER_FIRST = FIRST;
    constexpr int NS = B2<WP, MODE>::NS, KC = B2<WP, MODE>::KC, DS = B2<WP, MODE>::DS, NT = B2<WP, MODE>::NT;
    constexpr uint16_t MASK = (uint16_t)((1u << NS) - 1u);
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = align1024(smem_raw);
    uint8_t *Wt = smem;                          // [KC] x 16 KiB: W^T rows i in [128c, 128c+128)
    uint8_t *Dr = Wt + KC * CHUNK_BYTES;         // [DS] x 16 KiB
    uint8_t *Tr = Dr + DS * CHUNK_BYTES;         // [NT tiles][2 chunks] x 16 KiB
    uint8_t *ones = Tr + 2 * NT * CHUNK_BYTES;   // 256 B of fp16 ones (A operand of the bias MMA)
    uint64_t *bars = (uint64_t *)(ones + 256);
    uint64_t *wfull = bars;
    uint64_t *dfull = bars + 1, *dempty = dfull + DS, *dready = dempty + DS;
    uint64_t *tfull = dready + DS, *tempty = tfull + NT, *xfull = tempty + NT, *xempty = xfull + 2;
    uint64_t *wdone = xempty + 2;
    uint32_t *tmem_slot = (uint32_t *)(wdone + 1);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = NS > 1 ? cluster_rank() : 0u;
    const int pair = blockIdx.x / NS;
    const int nk = pair < a.ntiles ? (a.ntiles - pair + a.npairs - 1) / a.npairs : 0;
    if (threadIdx.x == 0) {
        mbar_init(wfull, 1);
        for (int s = 0; s < DS; ++s) {
            mbar_init(&dfull[s], 1);
            mbar_init(&dempty[s], NS);
            mbar_init(&dready[s], B2_EPI_THREADS);
        }
        for (int s = 0; s < NT; ++s) {
            mbar_init(&tfull[s], 1);
            mbar_init(&tempty[s], 1 + B2_EPI_WARPS);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(&xfull[s], 1);
            mbar_init(&xempty[s], B2_EPI_WARPS);
        }
        mbar_init(wdone, 1);
        fence_mbar_init();
    }
    if (threadIdx.x < 64) reinterpret_cast<uint32_t *>(ones)[threadIdx.x] = 0x3C003C00u;   // fp16 1.0 pairs
    fence_proxy_async_smem();
    if (warp == 1) tmem_alloc(tmem_slot, 512);
    pdl_wait();   // inputs of this GEMM come from the previous launch
    pdl_trigger();
    tc_fence_before();
    if (NS > 1) cluster_sync_all();   // every CTA's barriers exist before any multicast lands
    else __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const uint32_t tm_w = tmem + 256;   // dW^T accumulator; dX accumulators at columns 0 / 128
    constexpr int XB = 2;   // dX accumulator buffers

    if (warp == 0) {
        // ---------------- producer
        if (lane == 0) {
            mbar_arrive_expect_tx(wfull, KC * CHUNK_BYTES);
            for (int kc = 0; kc < KC; ++kc)
                bulk_g2s(Wt + kc * CHUNK_BYTES, (const uint8_t *)a.WTf + ((size_t)kc * WP + 128 * rank) * 128,
                         CHUNK_BYTES, wfull);
            // L2 prefetch PD tiles ahead: the shared-memory rings hold < 2 tiles, so the loads
            // that refill them must hit L2, not wait a full HBM round trip
            constexpr int PD = 3;
            auto prefetch = [&](int kp) {
                if (kp >= nk) return;
                const int tp = pair + (a.rev ? nk - 1 - kp : kp) * a.npairs;
                for (int j = (int)rank; j < KC; j += NS)
                    bulk_prefetch_l2((const uint8_t *)a.dsrc + ((size_t)tp * KC + j) * CHUNK_BYTES, CHUNK_BYTES);
                bulk_prefetch_l2((const uint8_t *)a.tin + ((size_t)tp * KC + 2 * rank) * CHUNK_BYTES,
                                 2 * CHUNK_BYTES);
            };
            for (int kp = 1; kp < PD; ++kp) prefetch(kp);
            int dn = 0;   // running Delta chunk counter
            auto load_t = [&](int k, int tile) {
                const int tb = k % NT;
                BTRACE(k * 16 + 0);
                mbar_wait_sleep(&tempty[tb], ((k / NT) & 1) ^ 1);
                BTRACE(k * 16 + 1);
                mbar_arrive_expect_tx(&tfull[tb], 2 * CHUNK_BYTES);
                bulk_g2s(Tr + tb * 2 * CHUNK_BYTES,
                         (const uint8_t *)a.tin + ((size_t)tile * KC + 2 * rank) * CHUNK_BYTES, 2 * CHUNK_BYTES,
                         &tfull[tb]);
            };
            for (int k = 0; k < nk; ++k) {
                const int tile = pair + (a.rev ? nk - 1 - k : k) * a.npairs;
                prefetch(k + PD);
                // t first: its ring is independent of the Delta ring, whose slots free up late
                if (T_FIRST) load_t(k, tile);
                for (int j = 0; j < KC; ++j, ++dn) {
                    const int slot = dn % DS;
                    mbar_wait_sleep(&dempty[slot], ((dn / DS) & 1) ^ 1);
                    mbar_arrive_expect_tx(&dfull[slot], CHUNK_BYTES);
                    const uint8_t *src = (const uint8_t *)a.dsrc + ((size_t)tile * KC + j) * CHUNK_BYTES;
                    if (NS == 1) bulk_g2s(Dr + slot * CHUNK_BYTES, src, CHUNK_BYTES, &dfull[slot]);
                    else if ((uint32_t)(j % NS) == rank)
                        bulk_g2s_mc(Dr + slot * CHUNK_BYTES, src, CHUNK_BYTES, &dfull[slot], MASK);
                }
                if (!T_FIRST) load_t(k, tile);
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer
        if (lane == 0) {
            constexpr uint32_t idesc_x = idesc_f16(128, 128, 0, 0);
            constexpr uint32_t idesc_w = idesc_f16(128, 128, 1, 1);
            const uint32_t wt = smem_u32(Wt), dr = smem_u32(Dr), tr = smem_u32(Tr);
            mbar_wait(wfull, 0);
            int dn = 0;
            for (int k = 0; k < nk; ++k) {
                const int b = k % XB, tb = k % NT;
                const int slot0 = dn % DS;
                B2_MMA_WAIT(&tfull[tb], (k / NT) & 1);
                BTRACE(k * 16 + 2);
                B2_MMA_WAIT(&xempty[b], ((k / XB) & 1) ^ 1);
                BTRACE(k * 16 + 7);
                tc_fence_after();
                const uint32_t accx = tmem + (uint32_t)(b * 128);
                // chunk pairs (2h, 2h+1): dX over those K chunks, then the dW^T N-half h, then release
                // the two ring slots -- the next tile's loads refill them mid-tile. Pairs sit in
                // consecutive slots (slot0 + 2h is even and <= DS - 2).
                auto dx_pair = [&](int h) {
                    const int sl = (slot0 + 2 * h) % DS;
                    for (int j = 2 * h; j < 2 * h + 2; ++j) {
                        B2_MMA_WAIT(OUTL ? &dready[sl + j - 2 * h] : &dfull[sl + j - 2 * h], ((dn + j) / DS) & 1);
                        BTRACE(k * 16 + 8 + j);
                        tc_fence_after();
#pragma unroll
                        for (int kq = 0; kq < 4; ++kq) {
                            const uint64_t ad = sdesc_sw128(dr + (sl + j - 2 * h) * CHUNK_BYTES + kq * 32, 16, 1024);
                            const uint64_t bd = sdesc_sw128(wt + j * CHUNK_BYTES + kq * 32, 16, 1024);
                            mma_f16(accx, ad, bd, idesc_x, (j | kq) != 0);
                        }
                    }
                };
                auto dw_half = [&](int h) {
                    const int sl = (slot0 + 2 * h) % DS;
#pragma unroll
                    for (int ks = 0; ks < 8; ++ks) {
                        const uint64_t ad = sdesc_sw128(tr + tb * 2 * CHUNK_BYTES + ks * 2048, CHUNK_BYTES, 1024);
                        const uint64_t bd = sdesc_sw128(dr + sl * CHUNK_BYTES + ks * 2048, CHUNK_BYTES, 1024);
                        mma_f16(tm_w + h * 128, ad, bd, idesc_w, (k | ks) != 0);
                    }
                    for (int j = 0; j < 2; ++j) {
                        if (NS == 1) mma_commit(&dempty[sl + j]);
                        else mma_commit_mc(&dempty[sl + j], MASK);
                    }
                };
                // all of dX first, committed before the dW MMAs: the epilogue drains it while dW runs
                for (int h = 0; h < KC / 2; ++h) dx_pair(h);
                mma_commit(&xfull[b]);
                for (int h = 0; h < KC / 2; ++h) dw_half(h);
                BTRACE(k * 16 + 3);
                mma_commit(&tempty[tb]);
                dn += KC;
            }
            mma_commit(wdone);
        }
    } else {
        // ---------------- epilogue warps: B2_EPI_WARPS, warp % 4 = TMEM lane quarter (rows); the
        // warps of a quarter split the CTA's 128 dX columns into CPW-wide slices
        constexpr int EWQ = B2_EPI_WARPS / 4;    // warps per lane quarter
        constexpr int CPW = 128 / EWQ;           // dX columns per warp (multiple of 32)
        constexpr int EPT = B2_EPI_THREADS;
        const int q = warp & 3;
        const int row = q * 32 + lane;
        const int wq = (warp - 2) >> 2;
        const int ep_tid = threadIdx.x - 64;
        const uint32_t t_lane = (uint32_t)(q * 32) << 16;
        const int N = a.N;
        float cs[CPW / 32], csx[CPW / 32], csy[CPW / 32];
        // column sums after the first butterfly level (lanes l, l^16), accumulated over all tiles;
        // the other four levels run once at the end (csdx/csdy: the g = 0 launch's x- and y-sums)
        float csd[CPW / 32][16], csdx[CPW / 32][16], csdy[CPW / 32][16];
#pragma unroll
        for (int g2 = 0; g2 < CPW / 32; ++g2)
#pragma unroll
            for (int i = 0; i < 16; ++i) csd[g2][i] = csdx[g2][i] = csdy[g2][i] = 0.f;
        auto level16 = [&](const float (&src)[32], float (&acc)[16], float scale) {
            const bool upper = (lane & 16) != 0;
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                const float send = (upper ? src[i] : src[i + 16]) * scale;
                const float keep = (upper ? src[i + 16] : src[i]) * scale;
                acc[i] += keep + __shfl_xor_sync(0xffffffffu, send, 16);
            }
        };
        auto finish16 = [&](float (&acc)[16]) {
#pragma unroll
            for (int st = 8; st >= 1; st >>= 1) {
                const bool upper = (lane & st) != 0;
#pragma unroll
                for (int i = 0; i < st; ++i) {
                    const float send = upper ? acc[i] : acc[i + st];
                    const float keep = upper ? acc[i + st] : acc[i];
                    acc[i] = keep + __shfl_xor_sync(0xffffffffu, send, st);
                }
            }
            return acc[0];
        };
#pragma unroll
        for (int g2 = 0; g2 < CPW / 32; ++g2) cs[g2] = csx[g2] = csy[g2] = 0.f;
        // output-layer transform state (outl). Thread -> granule lg (8 features) of every chunk,
        // rows orr + (EPT/8) m; chunks are transformed in order so the MMA can start on chunk 0
        // while later chunks are still being transformed. Delta_L is formed in half2 arithmetic
        // (it is stored in fp16 anyway); the output-layer column sums (dW_out = sum g t_L,
        // db_L = sum Delta_L) are fp32 and cover this CTA's own half of the features only.
        constexpr int ORG = EPT / 8;             // row groups of the transform
        constexpr int ORM = 128 / ORG;           // rows per thread and chunk
        const int olg = ep_tid & 7, orr = ep_tid >> 3;
        __half2 wo2[KC][4];
        float aw[2][8], ab[2][8], ag = 0.f;
        float s = 1.0f;
        float wboost = 1.0f;   // 2^ew: Delta_L = (s gbar 2^ew) (W_out 2^-ew) (1 - t_L^2), both factors fp16-safe
        if (OUTL) {
            float wm = 0.0f;
#pragma unroll
            for (int j = 0; j < KC; ++j)
#pragma unroll
                for (int e = 0; e < 8; ++e) wm = fmaxf(wm, fabsf(a.Wop[j * 64 + olg * 8 + e]));
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) wm = fmaxf(wm, __shfl_xor_sync(0xffffffffu, wm, o));   // lanes: all 8 granules
            const int ew = wout_exp(wm);
            wboost = exp2f((float)ew);
            s = grad_scale(a.st, ew);
            if (blockIdx.x == 0 && ep_tid == 0) {
                a.st->gscale = s;
                a.st->inv_gscale = 1.0f / s;
            }
            const float wsc = 1.0f / wboost;
#pragma unroll
            for (int j = 0; j < KC; ++j)
#pragma unroll
                for (int e = 0; e < 4; ++e)
                    wo2[j][e] = __floats2half2_rn(a.Wop[j * 64 + olg * 8 + 2 * e] * wsc,
                                                  a.Wop[j * 64 + olg * 8 + 2 * e + 1] * wsc);
#pragma unroll
            for (int jj = 0; jj < 2; ++jj)
#pragma unroll
                for (int e = 0; e < 8; ++e) aw[jj][e] = ab[jj][e] = 0.f;
        }
        const float kx = bwd_k(a.st, a.g);
        const f32x2_t K2 = pk2(kx, kx), NM2 = pk2(-kx * ACT_INV * ACT_INV, -kx * ACT_INV * ACT_INV);
        int dn = 0;
        for (int k = 0; k <= nk; ++k) {
            if (OUTL && k < nk) {
                // Delta_L = s gbar W_out (.) (1 - t_L^2), in place in this CTA's copy of the ring
                const int tile = pair + (a.rev ? nk - 1 - k : k) * a.npairs;
                if (warp == 2 && lane == 0) BTRACE(k * 16 + 12);
                float g[ORM];
                __half2 g2[ORM];
#pragma unroll
                for (int m = 0; m < ORM; ++m) {
                    g[m] = s * __ldg(a.gbar + (size_t)tile * 128 + orr + ORG * m);
                    g2[m] = __floats2half2_rn(g[m] * wboost, g[m] * wboost);
                    if (olg == 0) ag += g[m];
                }
                const __half2 one2 = __floats2half2_rn(1.0f, 1.0f);
                const __half2 tsc2 = __floats2half2_rn(ACT_INV, ACT_INV);
#pragma unroll
                for (int j = 0; j < KC; ++j) {
                    const int slot = (dn + j) % DS;
                    mbar_wait(&dfull[slot], ((dn + j) / DS) & 1);
                    const uint32_t blk = smem_u32(Dr + slot * CHUNK_BYTES);
                    const bool own = NS == 1 || (j >> 1) == (int)rank;
                    const int jj = NS == 1 ? j : (j & 1);
                    // the ORM rows of a granule column are first summed in half2 (g t and Delta_L are
                    // fp16 values already), then added to the fp32 sums once
                    __half2 haw[4], hab[4];
#pragma unroll
                    for (int e = 0; e < 4; ++e) haw[e] = hab[e] = __floats2half2_rn(0.0f, 0.0f);
#pragma unroll
                    for (int m = 0; m < ORM; ++m) {
                        const int r = orr + ORG * m;
                        const uint32_t off = (uint32_t)(r * 128 + ((olg ^ (r & 7)) << 4));
                        uint32_t w[4];
                        ld_shared_v4(blk + off, w[0], w[1], w[2], w[3]);
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            const __half2 t = __hmul2(*reinterpret_cast<__half2 *>(&w[e]), tsc2);   // t' -> t
                            const __half2 d = __hmul2(__hmul2(__hfma2(__hneg2(t), t, one2), wo2[j][e]), g2[m]);
                            if (a.outl_sums && own && jj < 2) {
                                haw[e] = __hfma2(g2[m], t, haw[e]);
                                hab[e] = __hadd2(hab[e], d);
                            }
                            w[e] = *reinterpret_cast<const uint32_t *>(&d);
                        }
                        st_shared_v4(blk + off, w[0], w[1], w[2], w[3]);
                    }
                    if (a.outl_sums && own && jj < 2) {
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            const float2 fw = __half22float2(haw[e]), fb = __half22float2(hab[e]);
                            aw[jj][2 * e] = fmaf(fw.x, 1.0f / wboost, aw[jj][2 * e]);   // haw is in g 2^ew units
                            aw[jj][2 * e + 1] = fmaf(fw.y, 1.0f / wboost, aw[jj][2 * e + 1]);
                            ab[jj][2 * e] += fb.x;
                            ab[jj][2 * e + 1] += fb.y;
                        }
                    }
                    fence_proxy_async_smem();
                    mbar_arrive(&dready[slot]);   // count = B2_EPI_THREADS
                    if (warp == 2 && lane == 0 && j == 0) BTRACE(k * 16 + 13);
                }
                if (warp == 2 && lane == 0) BTRACE(k * 16 + 14);
                dn += KC;
            }
            if (k == 0) continue;
            // ---- dX epilogue of tile k-1
            const int kk = k - 1, b = kk % XB, tb = kk % NT;
            const int tile = pair + (a.rev ? nk - 1 - kk : kk) * a.npairs;
            int pi, pj;
            point_ij(a.p0 + tile * 128 + row, N, pi, pj);
            const float x = (float)pi / (float)N, y = (float)pj / (float)N;
            if (warp == 2 && lane == 0) BTRACE(kk * 16 + 4);
            mbar_wait(&xfull[b], (kk / XB) & 1);
            if (warp == 2 && lane == 0) BTRACE(kk * 16 + 5);
            tc_fence_after();
            // EARLY_T: the dW MMAs of this tile are complete (xfull follows them): take this warp's t
            // values into registers and release the t slot now, so the next-but-one tile's t_in load
            // starts a whole epilogue earlier
            uint32_t tall[CPW / 32][4][4];
            if constexpr (EARLY_T) {
#pragma unroll
                for (int g2 = 0; g2 < CPW / 32; ++g2) {
                    const int col0 = wq * CPW + g2 * 32;
                    const uint32_t tsm = smem_u32(Tr) + (uint32_t)((tb * 2 + (col0 >> 6)) * CHUNK_BYTES + row * 128);
#pragma unroll
                    for (int j = 0; j < 4; ++j)
                        ld_shared_v4(tsm + (uint32_t)(((((col0 & 63) >> 3) + j) ^ (row & 7)) << 4), tall[g2][j][0],
                                     tall[g2][j][1], tall[g2][j][2], tall[g2][j][3]);
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&tempty[tb]);
            }
#pragma unroll
            for (int g2 = 0; g2 < CPW / 32; ++g2) {
                const int col0 = wq * CPW + g2 * 32;     // local dX column (i - 128 rank)
                const int hf = col0 >> 6;                // local t chunk
                const int lgb = (col0 & 63) >> 3;        // first logical granule in the chunk
                const uint32_t tsm = smem_u32(Tr) + (uint32_t)((tb * 2 + hf) * CHUNK_BYTES + row * 128);
                uint8_t *drow = (uint8_t *)a.din + ((size_t)tile * KC + 2 * rank + hf) * CHUNK_BYTES + row * 128;
                float v[32];
                tmem_ld32(tmem + t_lane + (uint32_t)(b * 128 + col0), v);
                uint32_t w[16];
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const int lg = lgb + j;
                    uint32_t tw[4];
                    if constexpr (EARLY_T) {
#pragma unroll
                        for (int q4 = 0; q4 < 4; ++q4) tw[q4] = tall[g2][j][q4];
                    } else {
                        ld_shared_v4(tsm + (uint32_t)((lg ^ (row & 7)) << 4), tw[0], tw[1], tw[2], tw[3]);
                    }
#pragma unroll
                    for (int mm = 0; mm < 4; ++mm) {
                        const float2 tf = __half22float2(*reinterpret_cast<const __half2 *>(&tw[mm]));
                        {   // k (1 - t^2) v for the pair in packed FFMA2s (t' = 2^14 t)
                            const f32x2_t T = pk2(tf.x, tf.y);
                            const f32x2_t V = pk2(v[8 * j + 2 * mm], v[8 * j + 2 * mm + 1]);
                            const f32x2_t NTV = ffma2(T, NM2, pk2(0.0f, 0.0f));   // -k 2^-28 t'
                            const f32x2_t G = ffma2(NTV, T, K2);                // k (1 - t^2)
                            upk2(ffma2(G, V, pk2(0.0f, 0.0f)), v[8 * j + 2 * mm], v[8 * j + 2 * mm + 1]);
                        }
                        w[4 * j + mm] = pack_half2(v[8 * j + 2 * mm], v[8 * j + 2 * mm + 1]);
                    }
                }
                if (!FIRST) {
                    // logical granules (2m, 2m+1) occupy one 32-byte sector, swapped when row is odd
#pragma unroll
                    for (int m = 0; m < 2; ++m) {
                        const int lg = lgb + 2 * m;
                        const int pos = (lg ^ (row & 7)) & ~1;
                        const uint32_t *g0 = &w[8 * m], *g1 = &w[8 * m + 4];
                        if (row & 1)
                            st_global_v8(drow + pos * 16, g1[0], g1[1], g1[2], g1[3], g0[0], g0[1], g0[2], g0[3]);
                        else
                            st_global_v8(drow + pos * 16, g0[0], g0[1], g0[2], g0[3], g1[0], g1[1], g1[2], g1[3]);
                    }
                }
                if (FIRST) {
                    if constexpr (DEFER_FIRST) {
                        level16(v, csdx[g2], x);
                        level16(v, csdy[g2], y);
                    } else
                    {
                        float vx[32], vy[32];
#pragma unroll
                        for (int e = 0; e < 32; ++e) { vx[e] = v[e] * x; vy[e] = v[e] * y; }
                        warp_reduce_scatter32(vx, lane);
                        warp_reduce_scatter32(vy, lane);
                        csx[g2] += vx[0];
                        csy[g2] += vy[0];
                    }
                }
                {   // bias sums (CUDA cores)
                    if (DEFER_CS && (!FIRST || DEFER_FIRST)) {
                        level16(v, csd[g2], 1.0f);
                    } else
                    {
                        warp_reduce_scatter32(v, lane);
                        cs[g2] += v[0];
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                if (warp == 2) BTRACE(kk * 16 + 6);
                mbar_arrive(&xempty[b]);
                if constexpr (!EARLY_T) mbar_arrive(&tempty[tb]);
            }
        }
        // remaining butterfly levels (8, 4, 2, 1) of the deferred column sums: column = lane
        if (DEFER_CS && (!FIRST || DEFER_FIRST)) {
#pragma unroll
            for (int g2 = 0; g2 < CPW / 32; ++g2) cs[g2] = finish16(csd[g2]);
        }
        if constexpr (DEFER_FIRST) {
#pragma unroll
            for (int g2 = 0; g2 < CPW / 32; ++g2) {
                csx[g2] = finish16(csdx[g2]);
                csy[g2] = finish16(csdy[g2]);
            }
        }
        // ---- end: all MMAs done -> the rings are free for the reductions
        if (nk > 0) mbar_wait(wdone, 0);
        tc_fence_after();
        named_bar(1, EPT);
        float *sred = (float *)Dr;   // [4 quarters][3][128]
#pragma unroll
        for (int g2 = 0; g2 < CPW / 32; ++g2) {
            const int col = wq * CPW + g2 * 32 + lane;
            sred[(q * 3 + 0) * 128 + col] = csx[g2];
            sred[(q * 3 + 1) * 128 + col] = csy[g2];
            sred[(q * 3 + 2) * 128 + col] = cs[g2];
        }
        // outl: pre-reduce the 4 row groups of a warp (lanes l, l^8, l^16, l^24 share olg) -> one
        // [2 kinds][128 own features] row per epilogue warp, then [EW] rows of g sums
        float *sob = sred + 12 * 128;
        if (OUTL && a.outl_sums) {
            const int ew = warp - 2;
#pragma unroll
            for (int jj = 0; jj < 2; ++jj)
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                    float x1 = aw[jj][e], x2 = ab[jj][e];
                    x1 += __shfl_xor_sync(0xffffffffu, x1, 8);
                    x1 += __shfl_xor_sync(0xffffffffu, x1, 16);
                    x2 += __shfl_xor_sync(0xffffffffu, x2, 8);
                    x2 += __shfl_xor_sync(0xffffffffu, x2, 16);
                    if (lane < 8) {
                        sob[(ew * 2 + 0) * 128 + jj * 64 + olg * 8 + e] = x1;
                        sob[(ew * 2 + 1) * 128 + jj * 64 + olg * 8 + e] = x2;
                    }
                }
            float gs = ag;
            gs += __shfl_xor_sync(0xffffffffu, gs, 8);
            gs += __shfl_xor_sync(0xffffffffu, gs, 16);
            if (lane == 0) sob[B2_EPI_WARPS * 2 * 128 + ew] = gs;
        }
        named_bar(1, EPT);
        if (ep_tid < 128) {
            const int col = ep_tid, ig = (int)rank * 128 + col;
            float sx = 0.f, sy = 0.f, sb = 0.f;
            for (int qq = 0; qq < 4; ++qq) {
                sx += sred[(qq * 3 + 0) * 128 + col];
                sy += sred[(qq * 3 + 1) * 128 + col];
                sb += sred[(qq * 3 + 2) * 128 + col];
            }
            float *pb = a.part_dx + (size_t)pair * 3 * WP;
            pb[2 * ig] = sx;
            pb[2 * ig + 1] = sy;
            pb[2 * WP + ig] = sb;
            if (OUTL && a.outl_sums) {
                float sw = 0.f, sbb = 0.f;
                for (int r = 0; r < B2_EPI_WARPS; ++r) {
                    sw += sob[(r * 2 + 0) * 128 + col];
                    sbb += sob[(r * 2 + 1) * 128 + col];
                }
                float *po = a.part_ob + (size_t)pair * (2 * WP + 1);
                po[ig] = sw;
                po[WP + ig] = sbb;
                if (rank == 0 && col == 0) {
                    float sg = 0.f;
                    for (int r = 0; r < B2_EPI_WARPS; ++r) sg += sob[B2_EPI_WARPS * 2 * 128 + r];
                    po[2 * WP] = sg;
                }
            }
        }
        // dW^T (rows i local = TMEM lanes, columns o) -> part_dw[pair][o][i], coalesced over i
        float *pw = a.part_dw + (size_t)pair * WP * WP + rank * 128 + row;
#pragma unroll 1
        for (int oc = wq * (WP / EWQ); oc < (wq + 1) * (WP / EWQ); oc += 32) {
            float v[32];
            if (nk > 0) {
                tmem_ld32(tm_w + t_lane + (uint32_t)oc, v);
            } else {
#pragma unroll
                for (int e = 0; e < 32; ++e) v[e] = 0.f;
            }
#pragma unroll
            for (int e = 0; e < 32; ++e) pw[(size_t)(oc + e) * WP] = v[e];
        }
    }
    tc_fence_before();
    if (NS > 1) cluster_sync_all();   // no CTA leaves while a peer may still multicast into it
    else __syncthreads();
    if (warp == 1) tmem_dealloc(tmem, 512);
}

// ================================================================ backward chain (WP >= 128)
// All hidden GEMMs of the backward in as few launches as possible, as a spatial pipeline: a
// cluster of S x NS CTAs holds S stages; stage s (CTAs [s NS, s NS + NS)) runs GEMM g0 - s like
// k_tc_bwd2 (W^T half resident, dX + dW^T per tile, Delta_out multicast to the stage's CTAs), and
// the clusters split the tile sequence. Delta_in of stage s goes to stage s+1 through a small
// per-cluster ring in global memory (BC_RS tiles per stage boundary, ~11 MB in total at C5, so it
// stays in L2) instead of a full HBM round trip per layer:
//   stage s epilogue  : wait oempty[slot] -> st.global its 64-column chunk -> proxy + gpu fence ->
//                       remote arrive on gfull[slot][chunk] of the stage-(s+1) CTA that loads it
//   stage s+1 producer: wait gfull -> multicast bulk load into the stage's Delta rings
//   stage s+1 MMA     : once the chunk pair of producer CTA h is consumed, commit (multicast) to
//                       oempty[slot] of that CTA -> the ring slot may be overwritten
// Bias gradients come from the tensor cores: each stage also accumulates 1^T Delta_out over its
// own half of the output features (an all-ones A operand: one 128-byte core matrix with zero
// strides), i.e. the bias gradient of theta layer g+1; only the last stage (g = 0) reduces its
// own output on the CUDA cores (bias and first-layer weights). The dX accumulator is single
// buffered to make room (its commit is issued before the second dW half, so the epilogue drains
// it under the remaining MMAs). The output-layer backward runs before the chain (k_tc_out_bwd).
constexpr int BC_RS = 3;   // global ring slots (tiles) per stage boundary
template <int WP>
struct BC {
    static constexpr uint32_t SMEM = B2<WP>::SMEM;   // includes the all-ones core matrix
};
struct BwdcArgs {
    int N, ntiles, nclus, S, g0;
    const __half *dsrc;   // stage 0 input: Delta_{g0+2}                    [ntiles][KC] blocks
    const __half *act;    // activations; t_{g+1} at act + g * lay
    __half *dout;         // Delta_{g0-S+2} of the last stage (HBM), unused when that stage has g = 0
    __half *ring;         // [nclus][S-1][BC_RS][KC] blocks
    const __half *WTf;    // [G][KC] blocks
    float *part_dx;       // [G][nclus][3*WP]  (only g = 0 is written: x, y and bias sums of Delta_1)
    float *part_dw;       // [G][nclus][WP*WP]
    float *part_cb;       // [G][nclus][WP]    1^T Delta_out of GEMM g (bias gradient of theta layer g+1)
    size_t lay;           // halves per activation layer
    long long *trace;     // debug timeline: CTAs 0..7 (cluster 0), 512 slots each; nullptr normally
    int p0;               // first MLP point of this shard
    const DevState *st;   // weight / Delta exponents per GEMM
};
#if CRV_TRACE
#define CTRACE(slot) do { if (a.trace && blockIdx.x < 8 && (slot) < 1024) a.trace[blockIdx.x * 1024 + (slot)] = clock64(); } while (0)
#else
#define CTRACE(slot) do { } while (0)
#endif

template <int WP>
__global__ void __launch_bounds__(B2_THREADS, 1) k_tc_bwdc(BwdcArgs a) {
    constexpr int NS = B2<WP>::NS, KC = B2<WP>::KC, DS = B2<WP>::DS, NT = B2<WP>::NT, RS = BC_RS;
    static_assert(B2_EPI_WARPS == 8, "chain epilogue: one 64-column chunk per warp");
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = align1024(smem_raw);
    uint8_t *Wt = smem;
    uint8_t *Dr = Wt + KC * CHUNK_BYTES;
    uint8_t *Tr = Dr + DS * CHUNK_BYTES;
    uint8_t *ones = Tr + 2 * NT * CHUNK_BYTES;   // 256 B of fp16 ones (A operand of the bias MMA)
    uint64_t *bars = (uint64_t *)(ones + 256);
    uint64_t *wfull = bars;
    uint64_t *dfull = bars + 1, *dempty = dfull + DS;
    uint64_t *tfull = dempty + DS, *tempty = tfull + NT, *xfull = tempty + NT, *xempty = xfull + 1;
    uint64_t *wdone = xempty + 1;
    uint64_t *gfull = wdone + 1;          // [RS][KC] (consumer side)
    uint64_t *oempty = gfull + RS * KC;   // [RS]     (producer side)
    uint32_t *tmem_slot = (uint32_t *)(oempty + RS);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t cr = cluster_rank();
    const int S = a.S;
    const int s = (int)cr / NS;
    const uint32_t rank = cr % NS;
    const int g = a.g0 - s;
    const bool first = g == 0;
    const bool to_ring = s < S - 1;
    const uint16_t smask = (uint16_t)(((1u << NS) - 1u) << (s * NS));
    const int cid = blockIdx.x / (S * NS);
    const int nk = cid < a.ntiles ? (a.ntiles - cid + a.nclus - 1) / a.nclus : 0;
    const __half *tin = a.act + (size_t)g * a.lay;
    auto ring_chunk = [&](int boundary, int gs, int j) -> __half * {
        return a.ring + ((((size_t)cid * (S - 1) + boundary) * RS + gs) * KC + j) * CHUNK_HALVES;
    };
    if (threadIdx.x < 64) reinterpret_cast<uint32_t *>(ones)[threadIdx.x] = 0x3C003C00u;   // fp16 1.0 pairs
    if (threadIdx.x == 0) {
        mbar_init(wfull, 1);
        for (int i = 0; i < DS; ++i) {
            mbar_init(&dfull[i], 1);
            mbar_init(&dempty[i], NS);
        }
        for (int i = 0; i < NT; ++i) {
            mbar_init(&tfull[i], 1);
            mbar_init(&tempty[i], 1 + B2_EPI_WARPS);
        }
        mbar_init(xfull, 1);
        mbar_init(xempty, B2_EPI_WARPS);
        mbar_init(wdone, 1);
        for (int i = 0; i < RS * KC; ++i) mbar_init(&gfull[i], 4);   // 4 warps (lane quarters) per chunk
        for (int i = 0; i < RS; ++i) mbar_init(&oempty[i], NS);      // one commit per consumer CTA
        fence_mbar_init();
    }
    fence_proxy_async_smem();   // the ones block is read by the tensor cores
    if (warp == 1) tmem_alloc(tmem_slot, 512);
    pdl_wait();
    pdl_trigger();
    tc_fence_before();
    cluster_sync_all();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const uint32_t tm_x = tmem, tm_c = tmem + 128, tm_w = tmem + 256;   // dX | 1^T Delta | dW^T

    if (warp == 0) {
        // ---------------- producer
        if (lane == 0) {
            mbar_arrive_expect_tx(wfull, KC * CHUNK_BYTES);
            for (int kc = 0; kc < KC; ++kc)
                bulk_g2s(Wt + kc * CHUNK_BYTES,
                         (const uint8_t *)a.WTf + ((size_t)g * KC * WP * 64 + (size_t)kc * WP * 64 + 128 * rank * 64) * 2,
                         CHUNK_BYTES, wfull);
            constexpr int PD = 3;
            auto prefetch = [&](int kp) {
                if (kp >= nk) return;
                const int tp = cid + kp * a.nclus;
                if (s == 0)
                    for (int j = (int)rank; j < KC; j += NS)
                        bulk_prefetch_l2((const uint8_t *)a.dsrc + ((size_t)tp * KC + j) * CHUNK_BYTES, CHUNK_BYTES);
                bulk_prefetch_l2((const uint8_t *)tin + ((size_t)tp * KC + 2 * rank) * CHUNK_BYTES, 2 * CHUNK_BYTES);
            };
            for (int kp = 1; kp < PD; ++kp) prefetch(kp);
            int dn = 0;
            auto load_t = [&](int k, int tile) {
                const int tb = k % NT;
                CTRACE(k * 16 + 0);
                mbar_wait_sleep(&tempty[tb], ((k / NT) & 1) ^ 1);
                CTRACE(k * 16 + 1);
                mbar_arrive_expect_tx(&tfull[tb], 2 * CHUNK_BYTES);
                bulk_g2s(Tr + tb * 2 * CHUNK_BYTES, (const uint8_t *)tin + ((size_t)tile * KC + 2 * rank) * CHUNK_BYTES,
                         2 * CHUNK_BYTES, &tfull[tb]);
            };
            for (int k = 0; k < nk; ++k) {
                const int tile = cid + k * a.nclus;
                const int gs = k % RS;
                prefetch(k + PD);
                load_t(k, tile);   // a tile's t_in before its Delta chunks
                for (int j = 0; j < KC; ++j, ++dn) {
                    const int slot = dn % DS;
                    mbar_wait_sleep(&dempty[slot], ((dn / DS) & 1) ^ 1);
                    mbar_arrive_expect_tx(&dfull[slot], CHUNK_BYTES);
                    if ((uint32_t)(j % NS) != rank) continue;   // the peer multicasts this chunk
                    const uint8_t *src;
                    if (s == 0) {
                        src = (const uint8_t *)a.dsrc + ((size_t)tile * KC + j) * CHUNK_BYTES;
                    } else {
                        if (j < 2) CTRACE(k * 16 + 11 + 2 * j);
                        mbar_wait_cluster(&gfull[gs * KC + j], (k / RS) & 1);
                        if (j < 2) CTRACE(k * 16 + 12 + 2 * j);
                        fence_proxy_async_global();
                        src = (const uint8_t *)ring_chunk(s - 1, gs, j);
                    }
                    if (NS == 1) bulk_g2s(Dr + slot * CHUNK_BYTES, src, CHUNK_BYTES, &dfull[slot]);
                    else bulk_g2s_mc(Dr + slot * CHUNK_BYTES, src, CHUNK_BYTES, &dfull[slot], smask);
                }
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer
        if (lane == 0) {
            constexpr uint32_t idesc_x = idesc_f16(128, 128, 0, 0);
            constexpr uint32_t idesc_w = idesc_f16(128, 128, 1, 1);
            constexpr uint32_t idesc_c = idesc_f16(128, 128, 0, 1);
            const uint32_t wt = smem_u32(Wt), dr = smem_u32(Dr), tr = smem_u32(Tr);
            const uint64_t d1 = sdesc_none(smem_u32(ones), 0, 0);
            mbar_wait_sleep(wfull, 0);
            int dn = 0;
            for (int k = 0; k < nk; ++k) {
                const int tb = k % NT, gs = k % RS;
                const int slot0 = dn % DS;
                mbar_wait_sleep(&tfull[tb], (k / NT) & 1);
                CTRACE(k * 16 + 2);
                mbar_wait_sleep(xempty, (k & 1) ^ 1);
                CTRACE(k * 16 + 7);
                tc_fence_after();
                for (int h = 0; h < KC / 2; ++h) {
                    const int sl = (slot0 + 2 * h) % DS;
                    for (int j = 2 * h; j < 2 * h + 2; ++j) {
                        mbar_wait_sleep(&dfull[sl + j - 2 * h], ((dn + j) / DS) & 1);
                        if (j == 0) CTRACE(k * 16 + 15);
                        tc_fence_after();
#pragma unroll
                        for (int kq = 0; kq < 4; ++kq) {
                            const uint64_t ad = sdesc_sw128(dr + (sl + j - 2 * h) * CHUNK_BYTES + kq * 32, 16, 1024);
                            const uint64_t bd = sdesc_sw128(wt + j * CHUNK_BYTES + kq * 32, 16, 1024);
                            mma_f16(tm_x, ad, bd, idesc_x, (j | kq) != 0);
                        }
                    }
                    if (h == KC / 2 - 1) {
                        mma_commit(xfull);   // dX complete: the epilogue drains it under the rest
                        CTRACE(k * 16 + 3);
                    }
#pragma unroll
                    for (int ks = 0; ks < 8; ++ks) {
                        const uint64_t ad = sdesc_sw128(tr + tb * 2 * CHUNK_BYTES + ks * 2048, CHUNK_BYTES, 1024);
                        const uint64_t bd = sdesc_sw128(dr + sl * CHUNK_BYTES + ks * 2048, CHUNK_BYTES, 1024);
                        mma_f16(tm_w + h * 128, ad, bd, idesc_w, (k | ks) != 0);
                    }
                    if (h == (int)rank) {
#pragma unroll
                        for (int ks = 0; ks < 8; ++ks) {
                            const uint64_t bd = sdesc_sw128(dr + sl * CHUNK_BYTES + ks * 2048, CHUNK_BYTES, 1024);
                            mma_f16(tm_c, d1, bd, idesc_c, (k | ks) != 0);
                        }
                    }
                    for (int j = 0; j < 2; ++j) {
                        if (NS == 1) mma_commit(&dempty[sl + j]);
                        else mma_commit_mc(&dempty[sl + j], smask);
                    }
                    // chunks (2h, 2h+1) came from CTA h of the previous stage: its ring slot is free
                    if (s > 0) mma_commit_mc(&oempty[gs], (uint16_t)(1u << ((s - 1) * NS + h)));
                }
                mma_commit(&tempty[tb]);
                dn += KC;
            }
            mma_commit(wdone);
        }
    } else {
        // ---------------- epilogue warps (8): warp % 4 = TMEM lane quarter, wq = which 64 columns
        constexpr int EPT = B2_EPI_THREADS;
        const int q = warp & 3;
        const int row = q * 32 + lane;
        const int wq = (warp - 2) >> 2;
        const int ep_tid = threadIdx.x - 64;
        const uint32_t t_lane = (uint32_t)(q * 32) << 16;
        const int N = a.N;
        float cs[2] = {0.f, 0.f}, csx[2] = {0.f, 0.f}, csy[2] = {0.f, 0.f};
        const float kx = bwd_k(a.st, g), mx = kx * (ACT_INV * ACT_INV);
        // hand this warp's chunk of a finished tile (ring slot pgs) to the next stage. Deferred by
        // one tile: by the time the next tile's dX is drained the stores are long complete, so the
        // gpu-scope fence does not stall the epilogue.
        int pgs = -1;
        auto handoff = [&]() {
            if (pgs < 0) return;
            fence_proxy_async_global();
            asm volatile("fence.acq_rel.cluster;" ::: "memory");
            __syncwarp();
            if (lane == 0) {
                const int j = 2 * (int)rank + wq;   // global chunk index within the tile
                mbar_arrive_cluster(mapa_shared(&gfull[pgs * KC + j], (uint32_t)((s + 1) * NS + (j % NS))));
            }
            pgs = -1;
        };
        for (int kk = 0; kk < nk; ++kk) {
            const int tb = kk % NT, gs = kk % RS;
            const int tile = cid + kk * a.nclus;
            if (warp == 2 && lane == 0) CTRACE(kk * 16 + 4);
            mbar_wait(xfull, kk & 1);
            if (warp == 2 && lane == 0) CTRACE(kk * 16 + 5);
            tc_fence_after();
            // this warp's 64 dX columns (local chunk wq) -> registers, then release the accumulator
            uint32_t r[4][16];
            const uint32_t tacc = tm_x + t_lane + (uint32_t)(wq * 64);
#pragma unroll
            for (int sl = 0; sl < 4; ++sl) tmem_ld16_async(tacc + (uint32_t)(16 * sl), r[sl]);
            tmem_wait_ld16(r[0]);
            tmem_wait_ld16(r[1]);
            tmem_wait_ld16(r[2]);
            tmem_wait_ld16(r[3]);
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(xempty);
            handoff();
            if (warp == 2 && lane == 0) CTRACE(kk * 16 + 8);
            if (to_ring && !first) mbar_wait(&oempty[gs], ((kk / RS) & 1) ^ 1);   // ring slot consumed
            if (warp == 2 && lane == 0) CTRACE(kk * 16 + 9);
            const uint32_t tsm = smem_u32(Tr) + (uint32_t)((tb * 2 + wq) * CHUNK_BYTES + row * 128);
            uint8_t *drow = to_ring ? (uint8_t *)ring_chunk(s, gs, 2 * (int)rank + wq) + row * 128
                                    : (uint8_t *)a.dout + ((size_t)tile * KC + 2 * rank + wq) * CHUNK_BYTES + row * 128;
            float x = 0.f, y = 0.f;
            if (first) {
                int pi, pj;
                point_ij(a.p0 + tile * 128 + row, N, pi, pj);
                x = (float)pi / (float)N;
                y = (float)pj / (float)N;
            }
#pragma unroll
            for (int hp = 0; hp < 2; ++hp) {          // slice pairs: columns wq*64 + 32 hp + [0, 32)
                float acc[32];
#pragma unroll
                for (int s2 = 0; s2 < 2; ++s2) {
                    const int sl = 2 * hp + s2;
                    uint32_t tw[8];
                    ld_shared_v4(tsm + (uint32_t)(((2 * sl) ^ (row & 7)) << 4), tw[0], tw[1], tw[2], tw[3]);
                    ld_shared_v4(tsm + (uint32_t)(((2 * sl + 1) ^ (row & 7)) << 4), tw[4], tw[5], tw[6], tw[7]);
                    uint32_t w[8];
#pragma unroll
                    for (int mm = 0; mm < 8; ++mm) {
                        const float2 tf = __half22float2(*reinterpret_cast<__half2 *>(&tw[mm]));
                        const float d0 = __uint_as_float(r[sl][2 * mm]) * fmaf(-mx * tf.x, tf.x, kx);
                        const float d1 = __uint_as_float(r[sl][2 * mm + 1]) * fmaf(-mx * tf.y, tf.y, kx);
                        acc[16 * s2 + 2 * mm] = d0;
                        acc[16 * s2 + 2 * mm + 1] = d1;
                        w[mm] = pack_half2(d0, d1);
                    }
                    if (!first) {
                        // logical granules (2 sl, 2 sl + 1) share one 32-byte sector, swapped on odd rows
                        const int pos = ((2 * sl) ^ (row & 7)) & ~1;
                        if (row & 1) st_global_v8(drow + pos * 16, w[4], w[5], w[6], w[7], w[0], w[1], w[2], w[3]);
                        else st_global_v8(drow + pos * 16, w[0], w[1], w[2], w[3], w[4], w[5], w[6], w[7]);
                    }
                }
                if (first) {
                    float tmp[32];
#pragma unroll
                    for (int e = 0; e < 32; ++e) tmp[e] = acc[e] * x;
                    warp_reduce_scatter32(tmp, lane);
                    csx[hp] += tmp[0];
#pragma unroll
                    for (int e = 0; e < 32; ++e) tmp[e] = acc[e] * y;
                    warp_reduce_scatter32(tmp, lane);
                    csy[hp] += tmp[0];
                    warp_reduce_scatter32(acc, lane);
                    cs[hp] += acc[0];
                }
            }
            if (warp == 2 && lane == 0) CTRACE(kk * 16 + 10);
            if (to_ring && !first) pgs = gs;
            __syncwarp();
            if (lane == 0) {
                if (warp == 2) CTRACE(kk * 16 + 6);
                mbar_arrive(&tempty[tb]);
            }
        }
        handoff();
        // ---- end: all MMAs done -> the rings are free for the reductions
        if (nk > 0) mbar_wait(wdone, 0);
        tc_fence_after();
        named_bar(1, EPT);
        float *sred = (float *)Dr;
        if (first) {
#pragma unroll
            for (int hp = 0; hp < 2; ++hp) {
                const int col = wq * 64 + hp * 32 + lane;
                sred[(q * 3 + 0) * 128 + col] = csx[hp];
                sred[(q * 3 + 1) * 128 + col] = csy[hp];
                sred[(q * 3 + 2) * 128 + col] = cs[hp];
            }
        }
        named_bar(1, EPT);
        if (first && ep_tid < 128) {
            const int col = ep_tid, ig = (int)rank * 128 + col;
            float sx = 0.f, sy = 0.f, sb = 0.f;
            for (int qq = 0; qq < 4; ++qq) {
                sx += sred[(qq * 3 + 0) * 128 + col];
                sy += sred[(qq * 3 + 1) * 128 + col];
                sb += sred[(qq * 3 + 2) * 128 + col];
            }
            float *pb = a.part_dx + ((size_t)g * a.nclus + cid) * 3 * WP;
            pb[2 * ig] = sx;
            pb[2 * ig + 1] = sy;
            pb[2 * WP + ig] = sb;
        }
        // 1^T Delta_out for the own output-feature half: every TMEM row holds the same sums
        if (q == 0) {
            float v[32];
            const int oc = wq * 64;
#pragma unroll
            for (int half = 0; half < 2; ++half) {
                if (nk > 0) {
                    tmem_ld32(tm_c + t_lane + (uint32_t)(oc + 32 * half), v);
                } else {
#pragma unroll
                    for (int e = 0; e < 32; ++e) v[e] = 0.f;
                }
                if (lane == 0) {
                    float *pc = a.part_cb + ((size_t)g * a.nclus + cid) * WP + (int)rank * 128 + oc + 32 * half;
#pragma unroll
                    for (int e = 0; e < 32; ++e) pc[e] = v[e];
                }
            }
        }
        // dW^T (rows i local = TMEM lanes, columns o) -> part_dw[g][cid][o][i], coalesced over i
        float *pw = a.part_dw + ((size_t)g * a.nclus + cid) * WP * WP + rank * 128 + row;
#pragma unroll 1
        for (int oc = wq * (WP / 2); oc < (wq + 1) * (WP / 2); oc += 32) {
            float v[32];
            if (nk > 0) {
                tmem_ld32(tm_w + t_lane + (uint32_t)oc, v);
            } else {
#pragma unroll
                for (int e = 0; e < 32; ++e) v[e] = 0.f;
            }
#pragma unroll
            for (int e = 0; e < 32; ++e) pw[(size_t)(oc + e) * WP] = v[e];
        }
    }
    tc_fence_before();
    cluster_sync_all();
    if (warp == 1) tmem_dealloc(tmem, 512);
}

// ================================================================ weight re-layout


// Per-layer scales and fp16 copies of the hidden weights, one block per hidden GEMM g:
// wexp[g] = ceil(log2(max|W_g| + margin)) - 14, so that |W_g 2^-wexp| <= 2^14 for the whole call
// (margin = 4 n lr bounds what n Adam steps can add to any weight: |m^/sqrt(v^)| < 4), and
// fexp[g] = round(log2(|W_g|_F / sqrt(fan_in))) (the typical gain of Delta through the layer, 0 for
// Xavier weights). Then the B-operand blocks (forward: rows = out features; backward-dX: rows = in
// features), zero padded to WP. Grid (G, nb): every block of layer g computes the layer's two sums
// in the same fixed order (identical results), block (g, 0) stores the exponents, and each block
// writes its 1/nb of the copies.
__global__ void __launch_bounds__(512) k_wscale(Net net, int WP, int KC, const float *__restrict__ theta,
                                                __half *__restrict__ Wf, __half *__restrict__ WTf, DevState *st,
                                                float margin) {
    __shared__ float smx[16], sss[16];
    __shared__ int se;
    const int g = blockIdx.x, l = g + 1;
    const int win = net.widths[l], wout = net.widths[l + 1];
    const float *W = theta + net.woff[l];
    const int n = win * wout;
    pdl_wait();
    float mx = 0.0f, ss = 0.0f;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const float w = W[i];
        mx = fmaxf(mx, fabsf(w));
        ss = fmaf(w, w, ss);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        ss += __shfl_xor_sync(0xffffffffu, ss, o);
    }
    if ((threadIdx.x & 31) == 0) { smx[threadIdx.x >> 5] = mx; sss[threadIdx.x >> 5] = ss; }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w) { mx = fmaxf(mx, smx[w]); ss += sss[w]; }
        int e = 0, f = 0;
        const float M = mx + margin;
        if (M > 0.0f && isfinite(M)) {
            int x;
            const float m = frexpf(M, &x);             // M = m 2^x, m in [0.5, 1)
            e = (m == 0.5f ? x - 1 : x) - 14;          // ceil(log2 M) - 14
        } else if (!isfinite(M)) {
            e = 100;                                   // non-finite weights: the next loss is non-finite
        }
        if (ss > 0.0f && isfinite(ss)) f = (int)rintf(0.5f * log2f(ss / (float)win));
        if (blockIdx.y == 0) {
            st->wexp[g] = e;
            st->fexp[g] = f;
        }
        se = e;
    }
    __syncthreads();
    const int e = se;
    for (int idx = blockIdx.y * blockDim.x + threadIdx.x; idx < WP * WP; idx += gridDim.y * blockDim.x) {
        const int nn = idx / WP, k = idx % WP;     // element (row nn, K index k) of the block set
        const float vf = (nn < wout && k < win) ? W[(long)nn * win + k] : 0.0f;   // W[nn][k]
        const float vt = (k < wout && nn < win) ? W[(long)k * win + nn] : 0.0f;   // W^T[nn][k]
        const size_t blk = ((size_t)g * KC + (k >> 6)) * (size_t)WP * 64;
        const uint32_t off = (uint32_t)(nn * 64 + ((((k & 63) >> 3) ^ (nn & 7)) << 3) + (k & 7));
        Wf[blk + off] = __float2half_rn(ldexpf(vf, -e));
        WTf[blk + off] = __float2half_rn(ldexpf(vt, -e));
    }
}

// fp32 operand copies: first layer and biases x 2 log2(e), output layer (zero padded to WP)
__global__ void k_tc_refresh(Net net, int WP, int L, const float *__restrict__ theta, float *__restrict__ W1p,
                             float *__restrict__ bp, float *__restrict__ Wop) {
    const long nsmall = 2L * WP + (long)L * WP + WP + 1;
    for (long s = (long)blockIdx.x * blockDim.x + threadIdx.x; s < nsmall; s += (long)gridDim.x * blockDim.x) {
        long e = s;
        if (e < 2L * WP) {
            const int r = (int)(e >> 1), d = (int)(e & 1);
            W1p[e] = r < net.widths[1] ? TANH_C * theta[net.woff[0] + 2 * r + d] : 0.0f;
        } else if ((e -= 2L * WP) < (long)L * WP) {
            const int l = (int)(e / WP), r = (int)(e % WP);
            bp[e] = r < net.widths[l + 1] ? TANH_C * theta[net.boff[l] + r] : 0.0f;
        } else {
            e -= (long)L * WP;
            if (e < WP) Wop[e] = e < net.widths[L] ? theta[net.woff[L] + e] : 0.0f;
            else Wop[WP] = theta[net.boff[L]];
        }
    }
}

// ================================================================ A8: Adam, fused into the reductions
// (adam_one in common.cuh: the thread that finishes gradient entry e updates theta[e], m[e], v[e]
// and the operand copies: hidden weights -> fp16 Wf / WTf with the call's exponent, first layer and
// biases -> fp32 x 2 log2(e), output layer -> fp32; padding entries keep the refresh's zeros)
AdamOp tc_adam_op(const Net &net, const TcBufs &b, float *theta, float *m, float *v, DevState *st, float lr,
                  float beta1, float beta2, float eps) {
    AdamOp A{};
    A.on = 1;
    A.theta = theta; A.m = m; A.v = v; A.st = st;
    A.lr = lr; A.beta1 = beta1; A.beta2 = beta2; A.eps = eps;
    A.net = net; A.WP = b.WP; A.KC = b.KC;
    A.Wf = b.Wf; A.WTf = b.WTf; A.W1p = b.W1p; A.bp = b.bp; A.Wop = b.Wop;
    return A;
}

// ================================================================ host side
template <int WP>
static void set_attrs(int L) {
    cudaFuncSetAttribute(k_tc_forward<WP>, cudaFuncAttributeMaxDynamicSharedMemorySize, fwd_smem_bytes<WP>(L));
    if constexpr (WP <= 128)
        cudaFuncSetAttribute(k_tc_forward<WP, false, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, fwd_smem_bytes<WP>(L));
    cudaFuncSetAttribute(k_tc_forward<WP, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, fwd_smem_bytes<WP>(L));
    if constexpr (WP >= 128) {
        cudaFuncSetAttribute(k_tc_bwd2<WP, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, B2<WP, 0>::SMEM);
        cudaFuncSetAttribute(k_tc_bwd2<WP, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, B2<WP, 1>::SMEM);
        cudaFuncSetAttribute(k_tc_bwd2<WP, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, B2<WP, 2>::SMEM);
        cudaFuncSetAttribute(k_tc_bwd2<WP, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, B2<WP, 3>::SMEM);
        cudaFuncSetAttribute(k_tc_bwdc<WP>, cudaFuncAttributeMaxDynamicSharedMemorySize, BC<WP>::SMEM);
    } else {
        cudaFuncSetAttribute(k_tc_bwd_layer<WP>, cudaFuncAttributeMaxDynamicSharedMemorySize, bwd_smem_bytes<WP>());
    }
}

// clusters of the backward chain (cluster size S x NS) that can be co-resident on the device
template <int WP>
static int chain_max_clusters(int csize) {
    if constexpr (WP >= 128) {
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = csize;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.gridDim = dim3(csize * 64);
        cfg.blockDim = dim3(B2_THREADS);
        cfg.dynamicSmemBytes = BC<WP>::SMEM;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        if (csize > 8) cudaFuncSetAttribute(k_tc_bwdc<WP>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        int n = 0;
        if (cudaOccupancyMaxActiveClusters(&n, k_tc_bwdc<WP>, &cfg) != cudaSuccess) {
            cudaGetLastError();
            return 0;
        }
        return n;
    } else {
        return 0;
    }
}

int tc_create(const Net &net, TcBufs &b, int tile0, int ntiles, std::string &err) {
    const int L = net.nl - 1;
    int w = net.widths[1];
    b.WP = ((w + 63) / 64) * 64;
    b.KC = b.WP / 64;
    b.L = L;
    b.G = L - 1;
    if (tile0 < 0 || ntiles < 1 || tile0 + ntiles > net.P / 128) {
        err = "shard tile range outside the MLP point set";
        return CRVPINN_EINVAL;
    }
    b.tile0 = tile0;
    b.ntiles = ntiles;
    const int WP = b.WP, KC = b.KC, G = b.G;
    if (fwd_smem_bytes<256>(L) > 232448 && WP == 256) {
        err = "too many layers for the shared-memory budget of the fused forward";
        return CRVPINN_EINVAL;
    }
    if (WP == 64) set_attrs<64>(L);
    else if (WP == 128) set_attrs<128>(L);
    else if (WP == 192) { err = "hidden width 160/192 not supported by the tensor path"; return CRVPINN_EINVAL; }
    else set_attrs<256>(L);
    int nsm = 148;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    // two CTAs (8 epilogue warps each) per SM when there are more tiles than SMs and both fit (WP = 128)
    b.fwd_ew = (WP == 128 && b.ntiles > nsm && 2 * fwd_smem_bytes<128>(L) <= 228 * 1024) ? 8 : 16;
    b.grid_fwd = b.ntiles < (b.fwd_ew == 8 ? 2 : 1) * nsm ? b.ntiles : (b.fwd_ew == 8 ? 2 : 1) * nsm;
    {
        // WP >= 128: clusters of NS = WP/128 CTAs (k_tc_bwd2); WP = 64: one CTA per "pair"
        const int NS = WP >= 128 ? WP / 128 : 1;
        int np_ = nsm / NS;
        if (np_ > b.ntiles) np_ = b.ntiles;
        b.npairs = np_;
        b.grid_dx = np_;              // rows of the column-sum partials
        b.grid_bwd = np_ * NS;        // CTAs per backward launch
        // backward chain (k_tc_bwdc): S stages of NS CTAs per cluster, clusters split the tiles
        // Default: on for small problems (<= 4 tiles per SM: C4 measured 0.100 vs 0.120 ms backward,
        // one launch instead of G amortises the per-launch fill/drain), off for large ones (C5:
        // 0.60 vs 0.49 ms). CRVPINN_BWD_CHAIN=0/1 forces it.
        const char *ce = getenv("CRVPINN_BWD_CHAIN");       // tuning knob: 0/1 = backward chain off/on
        const char *se = getenv("CRVPINN_BWD_STAGES");      // tuning knob: stages per cluster (implies chain)
        const bool small = b.ntiles <= 4 * nsm;
        const bool want = ce ? ce[0] == '1' : (se != nullptr || small);
        b.chain = 0;
        if (WP >= 128 && G >= 2 && want) {
            // more tiles than SMs: two stages per cluster (clusters of 2 CTAs with ~224 KB of shared memory
            // use all 148 SMs, clusters of 4 only 132): C4 145.0 vs 149.4 us per iteration with S = 4;
            // otherwise 8 / NS stages (C3: S = 2 and 4 measured equal)
            int S = se ? atoi(se) : (b.ntiles > nsm ? 2 : 8 / NS);
            if (S > G) S = G;
            if (S * NS > 8) S = 8 / NS;
            if (S < 1) S = 1;
            {
                int nc = WP == 128 ? chain_max_clusters<128>(S * NS) : chain_max_clusters<256>(S * NS);
                if (nc > b.ntiles) nc = b.ntiles;
                if (nc > 0) {
                    b.chain = 1;
                    b.chain_S = S;
                    b.npairs = b.grid_dx = nc;
                    b.grid_bwd = nc * S * NS;
                }
            }
        }
    }
    {
        // the output-layer backward is fused into the first backward GEMM (k_tc_bwd2); with the
        // chain it runs as its own bandwidth-bound pass (k_tc_out_bwd) so that it does not pace
        // every stage of the chain
        const char *e = getenv("CRVPINN_FUSE_OUTL");   // tuning knob: fused output-layer backward
        b.fuse_outl = WP >= 128 && !b.chain && !(e && e[0] == '0');
        b.grid_ob = WP >= 128 && b.fuse_outl ? b.npairs : (b.ntiles < 2 * nsm ? b.ntiles : 2 * nsm);
        const char *r = getenv("CRVPINN_BWD_REV");     // tuning knob: alternating tile-walk direction
        b.bwd_rev = !(r && r[0] == '0');
    }
    auto al = [&](void **p, size_t bytes) -> bool {
        if (cudaMalloc(p, bytes > 0 ? bytes : 16) != cudaSuccess) return false;
        cudaMemset(*p, 0, bytes > 0 ? bytes : 16);
        return true;
    };
    const size_t wblocks = (size_t)(G > 0 ? G : 1) * KC * WP * 64;
    const size_t actn = (size_t)L * b.ntiles * KC * CHUNK_HALVES;
    auto up64 = [](long v) { return (v + 63) / 64 * 64; };   // 256-byte aligned regions (float4 stores)
    b.off_ob = 0;
    b.off_dx = up64(b.off_ob + (long)b.grid_ob * (2 * WP + 1));
    b.off_dw = up64(b.off_dx + (long)(G > 0 ? G : 1) * b.grid_dx * 3 * WP);
    b.off_cb = up64(b.off_dw + (long)(G > 0 ? G * b.npairs : 1) * WP * WP);
    b.cb_bias = WP >= 128 && b.chain;   // hidden biases from the chain's tensor-core column sums
    const long ptotal = b.off_cb + (b.cb_bias ? (long)(G > 0 ? G : 1) * b.npairs * WP : 0);
    if (!al((void **)&b.Wf, wblocks * 2) || !al((void **)&b.WTf, wblocks * 2) ||
        !al((void **)&b.W1p, 2 * WP * 4) || !al((void **)&b.bp, (size_t)L * WP * 4) ||
        !al((void **)&b.Wop, (WP + 1) * 4) || !al((void **)&b.act, actn * 2) || !al((void **)&b.delta, actn * 2) ||
        !al((void **)&b.gbar, (size_t)net.P * 4) || !al((void **)&b.partial, ptotal * 4)) {
        err = "cudaMalloc failed for the tensor-core buffers";
        return CRVPINN_ENOMEM;
    }
    // reduction jobs (all partials are in gscale units -> scaled = 1)
    RedJob jobs[2 * CRV_MAX_LAYERS];
    int nj = 0;
    b.max_count = 0;
    b.groups = 0;
    // lev: the Delta level of the partials (activation layer a = 1..L; Delta_a carries the scale
    // s 2^-(fexp[a-1] + ... + fexp[G-1])), tsc: one stored activation factor t' = 2^14 t (dW)
    auto job = [&](long src, long dst, int count, int nsplit, long stride, int transposed, int cols, int ld,
                   int lev, int tsc) {
        RedJob &j = jobs[nj++];
        j.src = src; j.dst = dst; j.count = count; j.nsplit = nsplit; j.stride = stride;
        j.transposed = transposed; j.cols = cols; j.ld = ld; j.scaled = 1;
        j.g_lo = lev - 1; j.g_hi = G; j.tsc = tsc;
        if (count > b.max_count) b.max_count = count;
    };
    const int nl = net.nl;
    for (int l = 0; l < nl; ++l) {
        const int win = net.widths[l], wout = net.widths[l + 1];
        if (l == nl - 1) {   // output layer: from k_tc_out_bwd (WP = 64) / the outl launch of k_tc_bwd2
            job(b.off_ob, net.woff[l], win, b.grid_ob, 2 * WP + 1, 0, 1, 1, L, 0);
            job(b.off_ob + 2 * WP, net.boff[l], 1, b.grid_ob, 2 * WP + 1, 0, 1, 1, L, 0);
            continue;
        }
        // bias of theta layer l <-> Delta_{l+1}: from out_bwd (l = L-1) or dx(g = l); with the chain,
        // layers l >= 1 from the tensor-core sums 1^T Delta_out of GEMM l-1
        if (b.cb_bias && l >= 1)
            job(b.off_cb + (long)(l - 1) * b.npairs * WP, net.boff[l], wout, b.npairs, WP, 0, 1, 1, l + 1, 0);
        else if (l == L - 1) job(b.off_ob + WP, net.boff[l], wout, b.grid_ob, 2 * WP + 1, 0, 1, 1, l + 1, 0);
        else job(b.off_dx + (long)l * b.grid_dx * 3 * WP + 2 * WP, net.boff[l], wout, b.grid_dx, 3 * WP, 0, 1, 1,
                 l + 1, 0);
        if (l == 0) {
            if (G > 0) job(b.off_dx, net.woff[0], 2 * wout, b.grid_dx, 3 * WP, 0, 1, 1, 1, 0);
        }
    }
    // hidden-layer weight jobs: with WP >= 128 and a width that is a multiple of 4 they go to the
    // side-stream reduction (k_reduce_wide, float4 rows) launched right after GEMM g; the rest stay
    // in the table k_reduce walks after the last GEMM. Side jobs are appended after the deep ones.
    b.nsm = nsm;
    // Side-stream reductions: with the backward chain (its launches' dW reduced beside the next launch).
    // The per-GEMM path (k_tc_bwd2, C5) reduces every hidden layer after the last GEMM instead: its
    // side-stream reductions beside k_tc_bwd2 made C5's step(n) differ run to run in ~1 of 5 runs
    // (first in W0 / b0 / W1 / b1, scripts/det_steps.py, det_layers.py), and the
    // step time is the same without them (C5 793-801 vs 791-820 us per iteration).
    // CRVPINN_SIDE_REDUCE=0/1 forces it (A/B knob).
    const char *sre = getenv("CRVPINN_SIDE_REDUCE");
    const bool side_ok = sre ? sre[0] != '0' : b.chain != 0;
    for (int pass = 0; pass < 2; ++pass) {
        if (pass == 1) b.njobs_deep = nj;
        for (int l = 1; l < nl - 1; ++l) {
            const int win = net.widths[l], wout = net.widths[l + 1];
            const bool side = side_ok && WP >= 128 && win % 4 == 0;
            if (side != (pass == 1)) continue;
            job(b.off_dw + (long)(l - 1) * b.npairs * WP * WP, net.woff[l], wout * win, b.npairs, (long)WP * WP, 2,
                win, WP, l + 1, 1);
            b.wside[l - 1] = side;
            b.wjobs[l - 1] = jobs[nj - 1];
        }
    }
    if (G == 0) {
        err = "the tensor-core path needs at least two hidden layers";
        return CRVPINN_EINVAL;
    }
    b.njobs = nj;
    b.groups = reduce_groups(jobs, nj);
    b.groups_deep = reduce_groups(jobs, b.njobs_deep);
    if (cudaStreamCreateWithFlags(&b.side, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&b.ev_join, cudaEventDisableTiming) != cudaSuccess ||
        false) {
        err = "stream/event creation failed";
        return CRVPINN_ECUDA;
    }
    for (int g = 0; g < G; ++g)
        if (cudaEventCreateWithFlags(&b.ev_fork[g], cudaEventDisableTiming) != cudaSuccess) {
            err = "event creation failed";
            return CRVPINN_ECUDA;
        }
    if (!al((void **)&b.jobs, sizeof(RedJob) * nj)) {
        err = "cudaMalloc failed";
        return CRVPINN_ENOMEM;
    }
    cudaMemcpy(b.jobs, jobs, sizeof(RedJob) * nj, cudaMemcpyHostToDevice);
    if (b.chain) {
        const size_t rb = (size_t)b.npairs * (b.chain_S - 1) * BC_RS * KC * CHUNK_BYTES;
        if (!al((void **)&b.ring, rb)) {
            err = "cudaMalloc failed for the backward-chain ring";
            return CRVPINN_ENOMEM;
        }
    }
    b.ready = 1;
    return CRVPINN_OK;
}

void tc_destroy(TcBufs &b) {
    void *bufs[] = {b.Wf, b.WTf, b.W1p, b.bp, b.Wop, b.act, b.delta, b.gbar, b.partial, b.jobs, b.ring};
    for (void *p : bufs)
        if (p) cudaFree(p);
    b.Wf = b.WTf = nullptr;
    b.W1p = b.bp = b.Wop = b.gbar = b.partial = nullptr;
    b.act = b.delta = b.ring = nullptr;
    b.jobs = nullptr;
    for (auto &e : b.ev_fork)
        if (e) { cudaEventDestroy(e); e = nullptr; }
    if (b.ev_join) { cudaEventDestroy(b.ev_join); b.ev_join = nullptr; }
    if (b.side) { cudaStreamDestroy(b.side); b.side = nullptr; }
}

void tc_refresh_weights(const Net &net, const TcBufs &b, const float *theta, DevState *st, float margin,
                        cudaStream_t s) {
    launch_pdl(k_wscale, dim3(b.G, 16), dim3(512), 0, s, 1, net, b.WP, b.KC, theta, b.Wf, b.WTf, st, margin);
    const long nsmall = 2L * b.WP + (long)b.L * b.WP + b.WP + 1;
    k_tc_refresh<<<(unsigned)((nsmall + 255) / 256), 256, 0, s>>>(net, b.WP, b.L, theta, b.W1p, b.bp, b.Wop);
}

template <int WP>
static void fwd_launch(const Net &net, const TcBufs &b, float *u, cudaStream_t s) {
    static long long *trace = nullptr;
    const char *te = trace_env("CRVPINN_FWD_TRACE");   // debug: clock64 timeline of CTA 0 -> file
    if (te && !trace) { cudaMalloc(&trace, 4096 * 8); cudaMemset(trace, 0, 4096 * 8); }
    FwdArgs a{net.N, b.ntiles, b.L, b.G, b.Wf, b.W1p, b.bp, b.Wop, b.act, u, te ? trace : nullptr, nullptr, 0, b.tile0 * 128,
              b.st};
    if (te) {
        k_tc_forward<WP><<<b.grid_fwd, FWD_THREADS, fwd_smem_bytes<WP>(b.L), s>>>(a);
        cudaStreamSynchronize(s);
        static long long h[4096];
        cudaMemcpy(h, trace, sizeof(h), cudaMemcpyDeviceToHost);
        FILE *f = fopen(te, "wb");
        if (f) { fwrite(h, 8, 4096, f); fclose(f); }
        return;
    }
    if constexpr (WP <= 128) {
        if (b.fwd_ew == 8) {
            launch_pdl(k_tc_forward<WP, false, 8>, dim3(b.grid_fwd), dim3(fwd_threads<8>()), fwd_smem_bytes<WP>(b.L), s,
                       1, a);
            return;
        }
    }
    launch_pdl(k_tc_forward<WP>, dim3(b.grid_fwd), dim3(FWD_THREADS), fwd_smem_bytes<WP>(b.L), s, 1, a);
}

void tc_forward(const Net &net, const TcBufs &b, float *u, cudaStream_t s) {
    if (b.WP == 64) fwd_launch<64>(net, b, u, s);
    else if (b.WP == 128) fwd_launch<128>(net, b, u, s);
    else fwd_launch<256>(net, b, u, s);
}

template <int WP>
static void eval_launch(const Net &net, const TcBufs &b, const float *xy, int npts, float *out, cudaStream_t s) {
    const int ntiles = (npts + 127) / 128;
    const int grid = ntiles < b.nsm ? ntiles : b.nsm;
    FwdArgs a{net.N, ntiles, b.L, b.G, b.Wf, b.W1p, b.bp, b.Wop, nullptr, out, nullptr, xy, npts, 0, b.st};
    k_tc_forward<WP, true><<<grid, FWD_THREADS, fwd_smem_bytes<WP>(b.L), s>>>(a);
}

void tc_eval_points(const Net &net, const TcBufs &b, const float *xy, int npts, float *out, cudaStream_t s) {
    if (npts <= 0) return;
    if (b.WP == 64) eval_launch<64>(net, b, xy, npts, out, s);
    else if (b.WP == 128) eval_launch<128>(net, b, xy, npts, out, s);
    else eval_launch<256>(net, b, xy, npts, out, s);
}

template <int WP>
static void bwd_launch(const Net &net, const TcBufs &b, DevState *st, float *grad, cudaStream_t s,
                       const AdamOp *A) {
    const size_t lay = (size_t)b.ntiles * b.KC * CHUNK_HALVES;
    const int L = b.L;
    const int p0 = b.tile0 * 128;                    // this shard's first MLP point
    const float *gbar = b.gbar + p0;               // gbar covers every point (replicated field chain)
    if constexpr (WP >= 128) {
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute attr[2];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = B2<WP>::NS;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[1].val.programmaticStreamSerializationAllowed = 1;
        cfg.gridDim = dim3(b.grid_bwd);
        cfg.blockDim = dim3(B2_THREADS);
        cfg.dynamicSmemBytes = B2<WP>::SMEM;
        cfg.stream = s;
        cfg.attrs = attr;
        cfg.numAttrs = 2;
        if (!b.fuse_outl)
            k_tc_out_bwd<WP><<<b.grid_ob, OB_THREADS, 0, s>>>(b.ntiles, b.act + (size_t)(L - 1) * lay, gbar, b.Wop,
                                                              b.delta + (size_t)(L - 1) * lay, b.partial + b.off_ob,
                                                              st);
        int g_next = b.G - 1;   // GEMMs above g_next are done by the chain
        if (b.chain) {
            constexpr int NS = B2<WP>::NS;
            while (g_next >= 0) {
                const int g0 = g_next;
                const int Sl = b.chain_S < g0 + 1 ? b.chain_S : g0 + 1;
                attr[0].val.clusterDim.x = Sl * NS;
                cfg.gridDim = dim3(b.npairs * Sl * NS);
                cfg.dynamicSmemBytes = BC<WP>::SMEM;
                BwdcArgs a{net.N, b.ntiles, b.npairs, Sl, g0, b.delta + (size_t)(g0 + 1) * lay, b.act,
                           b.delta + (size_t)(g0 - Sl + 1) * lay, b.ring, b.WTf, b.partial + b.off_dx,
                           b.partial + b.off_dw, b.partial + b.off_cb, lay, nullptr, p0, st};
                static long long *ctrace = nullptr;
                const char *te = trace_env("CRVPINN_CHAIN_TRACE");   // debug: clock64 timeline -> file
                if (te && g0 == b.G - 1) {
                    if (!ctrace) cudaMalloc(&ctrace, 8 * 1024 * 8);
                    cudaMemset(ctrace, 0, 8 * 1024 * 8);
                    a.trace = ctrace;
                }
                cudaLaunchKernelEx(&cfg, k_tc_bwdc<WP>, a);
                if (te && g0 == b.G - 1) {
                    cudaStreamSynchronize(s);
                    static long long h[8 * 1024];
                    cudaMemcpy(h, ctrace, sizeof(h), cudaMemcpyDeviceToHost);
                    FILE *f = fopen(te, "wb");
                    if (f) { fwrite(h, 8, 8 * 1024, f); fclose(f); }
                }
                cudaEventRecord(b.ev_fork[g0], s);
                cudaStreamWaitEvent(b.side, b.ev_fork[g0], 0);
                // after the chain, nothing else shares the SMs: every layer's dW reduction in one launch
                RedJobSet js{};
                for (int g = g0; g > g0 - Sl; --g)
                    if (b.wside[g]) js.j[js.n++] = b.wjobs[g];
                launch_reduce_wide_set(b.partial, grad, js, st, 8 * b.nsm, b.side, A);
                g_next = g0 - Sl;
            }
            attr[0].val.clusterDim.x = NS;
            cfg.gridDim = dim3(b.npairs * NS);
            cfg.dynamicSmemBytes = B2<WP>::SMEM;
        }
        for (int g = g_next; g >= 0; --g) {
            const bool outl = g == b.G - 1 && b.fuse_outl;
            // Launches alternate the direction of their tile walk, starting backwards: the forward
            // and every launch leave the most recently written tiles (t_L, Delta_in) in L2, and the
            // next launch reads exactly those first.
            const int rev = ((b.G - 1 - g) & 1) == 0 ? b.bwd_rev : 0;
            Bwd2Args a{net.N, b.ntiles, b.npairs, g == 0 ? 1 : 0, outl ? 1 : 0, rev,
                       outl ? b.act + (size_t)(L - 1) * lay : b.delta + (size_t)(g + 1) * lay,
                       b.act + (size_t)g * lay, b.delta + (size_t)g * lay, b.WTf + (size_t)g * b.KC * WP * 64,
                       gbar, b.Wop, b.partial + b.off_ob,
                       b.partial + b.off_dx + (long)g * b.grid_dx * 3 * WP,
                       b.partial + b.off_dw + (long)g * b.npairs * WP * WP, st, nullptr,
                       b.partial + b.off_cb + (long)g * b.npairs * WP, 1, p0, g};
            static long long *trace = nullptr;
            const char *te = trace_env("CRVPINN_BWD_TRACE");
            const char *tg = getenv("CRVPINN_BWD_TRACE_G");
            const int trace_g = tg ? atoi(tg) : b.G - 1;
            if (te && g == trace_g) {
                if (!trace) cudaMalloc(&trace, 4096 * 8);
                cudaMemset(trace, 0, 4096 * 8);
                a.trace = trace;
            }
            const int mode = (outl ? 1 : 0) | (g == 0 ? 2 : 0);
            if (mode == 0) { cfg.dynamicSmemBytes = B2<WP, 0>::SMEM; cudaLaunchKernelEx(&cfg, k_tc_bwd2<WP, 0>, a); }
            else if (mode == 1) { cfg.dynamicSmemBytes = B2<WP, 1>::SMEM; cudaLaunchKernelEx(&cfg, k_tc_bwd2<WP, 1>, a); }
            else if (mode == 2) { cfg.dynamicSmemBytes = B2<WP, 2>::SMEM; cudaLaunchKernelEx(&cfg, k_tc_bwd2<WP, 2>, a); }
            else { cfg.dynamicSmemBytes = B2<WP, 3>::SMEM; cudaLaunchKernelEx(&cfg, k_tc_bwd2<WP, 3>, a); }
            // dW of GEMM g is final: reduce it on the side stream while GEMM g-1 runs
            cudaEventRecord(b.ev_fork[g], s);
            cudaStreamWaitEvent(b.side, b.ev_fork[g], 0);
            // (g > 0: beside the next GEMM, one small CTA per SM; g = 0: the SMs are free, four per SM;
            // the one-thread-per-output kernel measured ~6 us faster than the split-group one here)
            if (b.wside[g]) launch_reduce_wide(b.partial, grad, b.wjobs[g], st, g > 0 ? -b.nsm : -4 * b.nsm, b.side, A);
            if (te && g == trace_g) {
                cudaStreamSynchronize(s);
                static long long h[4096];
                cudaMemcpy(h, trace, sizeof(h), cudaMemcpyDeviceToHost);
                FILE *f = fopen(te, "wb");
                if (f) { fwrite(h, 8, 4096, f); fclose(f); }
            }
        }
    } else {
        k_tc_out_bwd<WP><<<b.grid_ob, OB_THREADS, 0, s>>>(b.ntiles, b.act + (size_t)(L - 1) * lay, gbar, b.Wop,
                                                          b.delta + (size_t)(L - 1) * lay, b.partial + b.off_ob, st);
        for (int g = b.G - 1; g >= 0; --g) {
            BwdArgs a{net.N, b.ntiles, g == 0 ? 1 : 0, b.npairs, b.delta + (size_t)(g + 1) * lay,
                      b.act + (size_t)g * lay, b.delta + (size_t)g * lay, b.WTf + (size_t)g * b.KC * WP * 64,
                      b.partial + b.off_dx + (long)g * b.grid_dx * 3 * WP,
                      b.partial + b.off_dw + (long)g * b.npairs * WP * WP, p0, st, g};
            k_tc_bwd_layer<WP><<<b.grid_dx, TC_THREADS, bwd_smem_bytes<WP>(), s>>>(a);
        }
    }
    if constexpr (WP >= 128) {
        launch_reduce(b.partial, grad, b.jobs, b.njobs_deep, b.groups_deep, st, s, A);   // column sums, W1, W_out
        cudaEventRecord(b.ev_join, b.side);
        cudaStreamWaitEvent(s, b.ev_join, 0);
    } else {
        launch_reduce(b.partial, grad, b.jobs, b.njobs, b.groups, st, s, A);
    }
}

void tc_backward(const Net &net, const TcBufs &b, DevState *st, float *grad, cudaStream_t s, const AdamOp *A) {
    if (b.WP == 64) bwd_launch<64>(net, b, st, grad, s, A);
    else if (b.WP == 128) bwd_launch<128>(net, b, st, grad, s, A);
    else bwd_launch<256>(net, b, st, grad, s, A);
}

int tc_launches(const Net &net, const TcBufs &b) {
    const int G = net.nl - 2;
    int bwd = G, side = 0;   // one launch per hidden GEMM, or the chain launches + remainder
    if (b.chain) {
        bwd = 0;
        int g = G - 1;
        while (g >= 0) {
            const int Sl = b.chain_S < g + 1 ? b.chain_S : g + 1;
            ++bwd;
            g -= Sl;
        }
    }
    for (int g = 0; g < G; ++g) side += b.wside[g] ? 1 : 0;
    if (b.chain) side = bwd;   // one batched reduction launch per chain launch
    return 1 /*fwd*/ + (b.WP < 128 || !b.fuse_outl ? 1 : 0) /*out_bwd*/ + bwd + side +
           1 /*reduce (+ Adam when training)*/;
}

}  // namespace crv
