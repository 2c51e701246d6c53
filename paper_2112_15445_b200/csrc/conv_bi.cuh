// conv_bi.cuh -- the batch-interleaved fp32 direct sparse conv kernel (sm_100a).
//
// Replaces the reference's hot loop kernels.sparse_conv_blocks
// (/root/reference/pkg/src/unsparse/kernels.py:57-100) for BINARY32.
//
// Layout: activations are batch-interleaved, IL = 32*SPL samples innermost
// ([n/IL][C][Hp][Wp][IL], zero halo): lane l of a warp holds samples SPL*l ..
// SPL*l+SPL-1, so for a given (pixel, tap) a warp's shared-memory load is SPL
// conflict-free 128-byte wavefronts and an output store is one coalesced line.
//   SPL = 1 (BI32): LDS.32, FMUL, FADD per MAC.
//   SPL = 2 (BI64): one LDS.64 feeds two samples; two FMUL then one packed FADD2
//   (add.rn.f32x2) -- 2 instructions per MAC instead of 3.  (mul.rn.f32x2 followed by
//   add.rn.f32x2 is contracted to FFMA2 by ptxas 12.9 even with --fmad=false, which
//   would break the reference's separately rounded multiply; FMUL + FADD2 is not.)
//
// Persistent, warp-specialised CTA of NWC compute warps + 1 producer warp:
//   * the producer's elected lane streams, for every tile this CTA owns and
//     every chunk of CC input channels, the input box [CC][HS][TWs][IL] with ONE
//     TMA tensor copy (cp.async.bulk.tensor.5d, out-of-range rows/columns/channels
//     zero-filled) plus that (group, chunk)'s entry block with one bulk copy into an
//     S-stage shared-memory ring, completing on full[s] and waiting on empty[s];
//   * compute warp w owns strip w % WS (a PR x PC output-pixel block) for the DW
//     output-channel slots of subgroup w / WS; DW*P accumulators per lane (SPL
//     samples each) live for the whole input-channel loop; after a stage each warp
//     arrives on empty[s] -- no CTA-wide barrier inside the loop;
//   * entry block of one (group, chunk): int2 hdr[NCLS][DT] (padded to 16 B) = {first, end} entry
//     index of every (pixel class, slot) run, then the runs, each starting 16-byte
//     aligned so two entries are one LDS.128 broadcast.  Slots map to output
//     channels through perm[] (the packer balances the warps' per-chunk work).  With
//     pixel classes (1x1 pixel blocks on small maps) a pixel's run omits the taps that
//     land on its zero halo: theta*0 adds +-0, a no-op for the never -0 accumulator;
//   * the register budget sets NWC: warps are spread over 4 SM sub-partitions, so
//     (NWC+1) warps leave 65536 / (4 * ceil((NWC+1)/4) * 32) registers per thread:
//     168 for NWC = 8, 128 for NWC = 12, 96 for NWC = 16.
//
// Per output element the arithmetic is the reference's: stored-order entries
// (ascending (c, kh, kw)), IEEE fp32 multiply then add, each rounded, so results
// are bit-identical to the reference for every tile configuration.
#pragma once
#include <cuda.h>

#include <type_traits>
#include <utility>

#include "common.cuh"

namespace usc_bi {
using namespace usc_dev;

// n / d for 0 <= n < 2^31 with one multiply-high (Granlund-Montgomery): m and s are
// set on the host (fdiv_make) so the per-item tile decode needs no integer division
struct FDiv {
    uint32_t d, m, s;
};
inline FDiv fdiv_make(uint32_t d) {
    uint32_t s = 0;
    while ((1ull << s) < d) ++s;
    return FDiv{d, static_cast<uint32_t>(((1ull << 32) * ((1ull << s) - d)) / d + 1), s};
}
__device__ __forceinline__ int fdiv(int n, const FDiv &f) {
    return static_cast<int>((__umulhi(static_cast<uint32_t>(n), f.m) + static_cast<uint32_t>(n)) >> f.s);
}

struct BiArgs {
    CUtensorMap xmap;        // x as 5-D [Nb][C][Hp][Wp][IL] (innermost first in the map)
    void *y;                 // fp32 (F32, I8) or binary16 (F16, CB4; I8 requantised codes) output
    const int *blk;          // byte offset of every (group, chunk) block, G*n_chunks+1
    const int *perm;         // output channel of every (group, warp, slot); -1 = empty
    const char *blocks;      // block base (16-byte aligned)
    const int *rowcls, *colcls;  // pixel class of every output row / column
    int ncls, ncls_c;        // classes (runs per slot), column classes
    int N, D, n_chunks, CC, DT;
    int HS, TWs, Yh, Yw, s_h;
    int WS, WC, SPRt, TH, row_tiles, col_tiles, G, tiles, S;
    int items, tfull, split;  // work items: tiles [0, tfull) whole, the rest split in `split` slot subsets
    int x_stage_bytes, stage_bytes;
    int fast;                 // store_tile_fast applies (see there)
    int i8shift;              // I8 fast requantisation: code = round(acc * 2^-i8shift) (see there)
    FDiv fG, fCT, fRT;        // divisions by G, col_tiles, row_tiles (tile decode)
    Epi ep;
};

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void tma_load_5d(void *dst, const CUtensorMap *map, int c0, int c1, int c2, int c3,
                                            int c4, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(smem_u32(bar))
        : "memory");
}

// ---------------------------------------------------------------------------
// lane value types and arithmetic per operand kind, SPL samples per lane
//   F32 (binary32 x, fp32 theta): FMUL then FADD (SPL 2: two FMUL + one FADD2).
//   F16 (binary16 x, binary16 theta): one FHFMA (fma.rn.f32.f16) per MAC -- the
//       binary16 x binary16 product is exact in fp32, so fma == FMUL+FADD bitwise.
//   CB4 (binary16 x, fp32 codebook centroid): products have up to 26 significant
//       bits, so FMUL then FADD (x widened with two conversions).
//   I8  (int8 codes staged as binary16, code weights): the F16 arithmetic, exact.

// shared-memory loads on 32-bit addresses with immediate offsets (LDS [R+imm]);
// not volatile: the address depends on an entry read after the stage's mbarrier
// wait, which keeps them behind it
template <int OFF>
__device__ __forceinline__ void lds_val(float &v, uint32_t a) {
    asm("ld.shared.f32 %0, [%1+%2];" : "=f"(v) : "r"(a), "n"(OFF));
}
template <int OFF>
__device__ __forceinline__ void lds_val(float2 &v, uint32_t a) {
    asm("ld.shared.v2.f32 {%0, %1}, [%2+%3];" : "=f"(v.x), "=f"(v.y) : "r"(a), "n"(OFF));
}
template <int OFF>
__device__ __forceinline__ void lds_val(uint32_t &v, uint32_t a) {
    asm("ld.shared.b32 %0, [%1+%2];" : "=r"(v) : "r"(a), "n"(OFF));
}
__device__ __forceinline__ int4 lds_v4(uint32_t a) {
    int4 v;
    asm("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
    return v;
}
__device__ __forceinline__ int2 lds_v2(uint32_t a) {
    int2 v;
    asm("ld.shared.v2.b32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a));
    return v;
}
__device__ __forceinline__ void fadd2(unsigned long long &acc, float lo, float hi) {
    unsigned long long q;
    asm("mov.b64 %0, {%1, %2};" : "=l"(q) : "f"(lo), "f"(hi));
    asm("add.rn.f32x2 %0, %0, %1;" : "+l"(acc) : "l"(q));
}
__device__ __forceinline__ void unpack2(unsigned long long a, float &lo, float &hi) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(a));
}
__device__ __forceinline__ float2 h2f2(uint32_t v) {
    float2 f;
    asm("{.reg .f16 l, h;\n mov.b32 {l, h}, %2;\n cvt.f32.f16 %0, l;\n cvt.f32.f16 %1, h;}"
        : "=f"(f.x), "=f"(f.y) : "r"(v));
    return f;
}

template <int KIND, int SPL> struct Ops;
template <> struct Ops<USC_F32, 1> {
    using V = float;
    using A = float;
    static constexpr int EB = 4;  // bytes per staged sample value
    __device__ static void zero(A &a) { a = 0.0f; }
    __device__ static V prod(uint32_t t, V v) { return __fmul_rn(__uint_as_float(t), v); }
    __device__ static void acc(A &a, V p) { a = __fadd_rn(a, p); }
    __device__ static void unpack(A a, float (&o)[1]) { o[0] = a; }
};
template <> struct Ops<USC_F32, 2> {
    using V = float2;
    using A = unsigned long long;  // packed (sample 2l, sample 2l+1) for FADD2
    static constexpr int EB = 4;
    __device__ static void zero(A &a) { a = 0ull; }  // (+0.0f, +0.0f)
    __device__ static V prod(uint32_t t, V v) {
        return make_float2(__fmul_rn(__uint_as_float(t), v.x), __fmul_rn(__uint_as_float(t), v.y));
    }
    __device__ static void acc(A &a, V p) { fadd2(a, p.x, p.y); }
    __device__ static void unpack(A a, float (&o)[2]) { unpack2(a, o[0], o[1]); }
};
template <> struct Ops<USC_CB4, 2> {
    using V = uint32_t;            // binary16 pair (sample 2l, 2l+1)
    using A = unsigned long long;
    static constexpr int EB = 2;
    __device__ static void zero(A &a) { a = 0ull; }
    __device__ static float2 prod(uint32_t t, V v) {
        const float2 x = h2f2(v);
        return make_float2(__fmul_rn(__uint_as_float(t), x.x), __fmul_rn(__uint_as_float(t), x.y));
    }
    __device__ static void acc(A &a, float2 p) { fadd2(a, p.x, p.y); }
    __device__ static void unpack(A a, float (&o)[2]) { unpack2(a, o[0], o[1]); }
};
template <> struct Ops<USC_F16, 2> {
    using V = uint32_t;  // binary16 pair
    using A = float2;
    static constexpr int EB = 2;
    __device__ static void zero(A &a) { a = make_float2(0.0f, 0.0f); }
    // theta: binary16 bits in the low half of t; fp32 += f16*f16, one rounding
    __device__ static void fma(A &a, uint32_t t, V v) {
        const unsigned short th = static_cast<unsigned short>(t), lo = static_cast<unsigned short>(v),
                             hi = static_cast<unsigned short>(v >> 16);
        asm("fma.rn.f32.f16 %0, %1, %2, %0;" : "+f"(a.x) : "h"(th), "h"(lo));
        asm("fma.rn.f32.f16 %0, %1, %2, %0;" : "+f"(a.y) : "h"(th), "h"(hi));
    }
    __device__ static void unpack(A a, float (&o)[2]) {
        o[0] = a.x;
        o[1] = a.y;
    }
};

// int8 codes staged as binary16 (exact): the F16 arithmetic; every product and partial
// sum is an integer below 2^24 (checked by the caller), so the fp32 accumulator equals
// the int32 sum exactly and the epilogue scales it by sigma_w*sigma_x
template <> struct Ops<USC_I8, 2> : Ops<USC_F16, 2> {};

// the P pixels of a thread for one tap: row 0 at a0, row 1 at a1 (bytes), columns
// SW pixels (SW*PXB bytes) apart
template <int PC, int PXB, int SW, typename V, int... I>
__device__ __forceinline__ void load_px_(V *v, uint32_t a0, uint32_t a1, std::integer_sequence<int, I...>) {
    ((I / PC == 0 ? lds_val<(I % PC) * SW * PXB>(v[I], a0) : lds_val<(I % PC) * SW * PXB>(v[I], a1)), ...);
}
template <int KIND, int PC, int PR, int SW, int SPL>
__device__ __forceinline__ void load_px(typename Ops<KIND, SPL>::V (&v)[PC * PR], uint32_t a0, uint32_t a1) {
    load_px_<PC, 32 * SPL * Ops<KIND, SPL>::EB, SW>(v, a0, a1, std::make_integer_sequence<int, PC * PR>{});
}

// acc[p] += t*v[p] for one entry (stored order: call in entry order)
template <int KIND, int SPL, int P>
__device__ __forceinline__ void mac_one(typename Ops<KIND, SPL>::A (&acc)[P], typename Ops<KIND, SPL>::V (&v)[P],
                                        uint32_t t) {
    using O = Ops<KIND, SPL>;
    if constexpr (KIND == USC_F16 || KIND == USC_I8) {
#pragma unroll
        for (int p = 0; p < P; ++p) O::fma(acc[p], t, v[p]);
    } else {
        decltype(O::prod(t, v[0])) q[P];
#pragma unroll
        for (int p = 0; p < P; ++p) q[p] = O::prod(t, v[p]);
#pragma unroll
        for (int p = 0; p < P; ++p) O::acc(acc[p], q[p]);
    }
}

// two entries n = {off0, t0, off1, t1}: products first, then the adds in stored order
template <int KIND, int SPL, int P>
__device__ __forceinline__ void mac_pair(typename Ops<KIND, SPL>::A (&acc)[P], typename Ops<KIND, SPL>::V (&v0)[P],
                                         typename Ops<KIND, SPL>::V (&v1)[P], const int4 &n) {
    using O = Ops<KIND, SPL>;
    if constexpr (KIND == USC_F16 || KIND == USC_I8) {
        mac_one<KIND, SPL, P>(acc, v0, static_cast<uint32_t>(n.y));
        mac_one<KIND, SPL, P>(acc, v1, static_cast<uint32_t>(n.w));
    } else {
        decltype(O::prod(0u, v0[0])) q0[P], q1[P];
#pragma unroll
        for (int p = 0; p < P; ++p) {
            q0[p] = O::prod(static_cast<uint32_t>(n.y), v0[p]);
            q1[p] = O::prod(static_cast<uint32_t>(n.w), v1[p]);
        }
#pragma unroll
        for (int p = 0; p < P; ++p) O::acc(acc[p], q0[p]);
#pragma unroll
        for (int p = 0; p < P; ++p) O::acc(acc[p], q1[p]);
    }
}

template <int KIND, int PC, int PR, int SW, int SPL>
__device__ __forceinline__ void load_pair(typename Ops<KIND, SPL>::V (&v0)[PC * PR],
                                          typename Ops<KIND, SPL>::V (&v1)[PC * PR], uint32_t xs, uint32_t rs,
                                          const int4 &n) {
    const uint32_t p0 = xs + n.x, p1 = xs + n.z;
    load_px<KIND, PC, PR, SW, SPL>(v0, p0, p0 + rs);
    load_px<KIND, PC, PR, SW, SPL>(v1, p1, p1 + rs);
}

// One slot's run of entries [ep, ee) (byte addresses, ep 16-B aligned), two entries
// (one LDS.128) per step.  PIPE: software pipelined -- the next pair's pixel loads
// are issued before this pair's math (ping-pong registers), so the shared-memory
// latency hides inside one warp.  Reads of the entry after a run stay inside the
// stage's 16-byte slack.
template <int KIND, int PC, int PR, int SW, int SPL, bool PIPE>
__device__ __forceinline__ void run_pairs(typename Ops<KIND, SPL>::A (&acc)[PC * PR], uint32_t xs, uint32_t rs,
                                          uint32_t ep, uint32_t ee) {
    constexpr int P = PC * PR;
    using V = typename Ops<KIND, SPL>::V;
    int4 nn = lds_v4(ep);
    if constexpr (PIPE) {
        if (ep + 16 <= ee) {
            V a0[P], a1[P], b0[P], b1[P];
            int4 n = nn;
            load_pair<KIND, PC, PR, SW, SPL>(a0, a1, xs, rs, n);
            ep += 16;
            nn = lds_v4(ep);
#pragma unroll 1
            while (true) {  // a* hold pair n; nn is the pair at ep
                if (ep + 16 > ee) {
                    mac_pair<KIND, SPL, P>(acc, a0, a1, n);
                    break;
                }
                load_pair<KIND, PC, PR, SW, SPL>(b0, b1, xs, rs, nn);
                int4 m = nn;
                ep += 16;
                nn = lds_v4(ep);
                mac_pair<KIND, SPL, P>(acc, a0, a1, n);
                n = m;
                if (ep + 16 > ee) {
                    mac_pair<KIND, SPL, P>(acc, b0, b1, n);
                    break;
                }
                load_pair<KIND, PC, PR, SW, SPL>(a0, a1, xs, rs, nn);
                m = nn;
                ep += 16;
                nn = lds_v4(ep);
                mac_pair<KIND, SPL, P>(acc, b0, b1, n);
                n = m;
            }
        }
    } else {
        // two pairs per iteration: the entry registers alternate instead of being moved
#pragma unroll 1
        for (; ep + 32 <= ee; ep += 32) {
            V v0[P], v1[P];
            load_pair<KIND, PC, PR, SW, SPL>(v0, v1, xs, rs, nn);
            const int4 n = lds_v4(ep + 16);
            mac_pair<KIND, SPL, P>(acc, v0, v1, nn);
            load_pair<KIND, PC, PR, SW, SPL>(v0, v1, xs, rs, n);
            nn = lds_v4(ep + 32);
            mac_pair<KIND, SPL, P>(acc, v0, v1, n);
        }
        if (ep + 16 <= ee) {
            V v0[P], v1[P];
            load_pair<KIND, PC, PR, SW, SPL>(v0, v1, xs, rs, nn);
            const int4 n = nn;
            ep += 16;
            nn = lds_v4(ep);
            mac_pair<KIND, SPL, P>(acc, v0, v1, n);
        }
    }
    if (ep < ee) {  // odd run: the last entry is nn.x, nn.y
        V v0[P];
        const uint32_t p0 = xs + nn.x;
        load_px<KIND, PC, PR, SW, SPL>(v0, p0, p0 + rs);
        mac_one<KIND, SPL, P>(acc, v0, static_cast<uint32_t>(nn.y));
    }
}

// output value of one accumulator (store_one semantics, common.cuh): F32 -> ReLU;
// F16/CB4 -> the _half_hook order of quantization.py:238-244 (saturate, binary16
// rounding, ReLU, saturate2 + rounding)
// shortcut value of the lane's j-th sample at (b, d, row, col) (residual epilogue)
template <int KIND>
__device__ __forceinline__ float res_value(const Epi &ep, long long b, int d, int row, int col) {
    const long long i = (b / ep.ril) * ep.r_sample_stride +
                        ((((long long)d * ep.rHp + row + ep.rph) * ep.rWs + col + ep.rpw) * ep.ril) + b % ep.ril;
    if constexpr (KIND == USC_F32)
        return static_cast<const float *>(ep.res)[i];
    else
        return __half2float(static_cast<const __half *>(ep.res)[i]);
}

template <int KIND>
__device__ __forceinline__ float epi_value(float v, const Epi &ep) {
    // ReLU is np.where(v > 0, v, 0) (nn.py:96-98): NaN -> 0
    if constexpr (KIND == USC_F32) {
        return ep.relu ? (v > 0.0f ? v : 0.0f) : v;
    } else if constexpr (KIND == USC_I8) {  // fp32 out = acc * sigma_w * sigma_x (power of two)
        v = __fmul_rn(v, ep.scale);
        if (ep.relu) v = v > 0.0f ? v : 0.0f;
        if (ep.requant) {  // next layer's codes (linear_quantize in fp64, quantization.py:61-76)
            const double q = static_cast<double>(v) * ep.rq_scale;
            double c = copysign(floor(fabs(q) + 0.5), q);
            c = c < -ep.rq_limit ? -ep.rq_limit : (c > ep.rq_limit ? ep.rq_limit : c);
            v = static_cast<float>(c);
        }
        return v;
    } else {
        if (ep.saturate) v = v > ep.cap ? ep.cap : v;  // np.minimum keeps NaN
        v = round16f(v);
        if (ep.relu) v = v > 0.0f ? v : 0.0f;
        if (ep.saturate2) {
            v = v > ep.cap2 ? ep.cap2 : v;
            v = round16f(v);
        }
        return v;
    }
}

// residual form (ResNet block output): F32 v = relu(acc + r); F16 v =
// relu(round16(round16(acc) + r)) -- the conv's binary16 hook, the add, the add's hook
template <int KIND>
__device__ __forceinline__ float epi_value_res(float v, const Epi &ep, float r) {
    if constexpr (KIND == USC_F32) {
        v = __fadd_rn(v, r);
    } else {
        v = __fadd_rn(round16f(v), r);
        v = round16f(v);
    }
    return ep.relu ? (v > 0.0f ? v : 0.0f) : v;
}

__device__ __forceinline__ uint32_t pack_h2(float lo, float hi) {  // exact: values on the binary16 grid
    const __half2 h = __halves2half2(__float2half_rn(lo), __float2half_rn(hi));
    return *reinterpret_cast<const uint32_t *>(&h);
}

// max-pool of a 2x2 window in np.argmax order (nn.py:124-135): first NaN, else
// first maximum
__device__ __forceinline__ float pool4(float w0, float w1, float w2, float w3) {
    const float w[4] = {w0, w1, w2, w3};
    float m = w[0];
    if (!isnan(m)) {
#pragma unroll
        for (int q = 1; q < 4; ++q) {
            if (isnan(w[q])) {
                m = w[q];
                break;
            }
            if (w[q] > m) m = w[q];
        }
    }
    return m;
}

// Work item -> (tile, slot part).  The last tiles of the schedule are split into
// `split` interleaved slot subsets (part p runs slots dw % split == p) so the final
// round of the persistent grid is not a partial wave of whole tiles.
__device__ __forceinline__ int item_tile(const BiArgs &a, int it, int &part) {
    if (it < a.tfull) {
        part = -1;
        return it;
    }
    const int j = it - a.tfull;
    part = j % a.split;
    return a.tfull + j / a.split;
}

// Epilogue of one tile for one warp: epi_value (ReLU, nn.py:96-98; binary16 hook for
// F16/CB4; int8 scale/requantise) then, if fused, the 2x2/2 max-pool (nn.py:124-135);
// element (b, d, row, col) of the output layout is obase + d*dstride + row*rstride +
// col*cstride (+ j*sstride for the lane's j-th sample)
template <int KIND, int PC, int PR, int DW, int SPL>
__device__ __forceinline__ void store_tile(const BiArgs &a, typename Ops<KIND, SPL>::A (&acc)[DW][PC * PR],
                                           int g, int wc, int sb, int r, int col0, int part, int lane) {
    using O = Ops<KIND, SPL>;
    constexpr int P = PC * PR;
    constexpr int IL = 32 * SPL;
    const int *pm = a.perm + g * a.DT + wc * DW;  // this warp's output channels (balanced)
    const bool pool = PR == 2 && a.ep.pool;
    const int orow = pool ? r / 2 : r, ocol = pool ? col0 / 2 : col0;
    const int b0 = sb * IL + lane * SPL;  // first sample of this lane
    const int oil = a.ep.out_padded ? a.ep.oil : 0;
    long long obase, dstride, sstride;
    int rstride, cstride;
    if (!a.ep.out_padded) {
        const int oh = pool ? a.Yh / 2 : a.Yh, ow = pool ? a.Yw / 2 : a.Yw;
        obase = ((long long)b0 * a.D * oh + orow) * ow + ocol;
        dstride = (long long)oh * ow;
        sstride = (long long)a.D * oh * ow;
        rstride = ow;
        cstride = 1;
    } else if (oil) {
        obase = (long long)(b0 / oil) * a.ep.o_sample_stride +
                (((long long)orow + a.ep.oph) * a.ep.oWs + ocol + a.ep.opw) * oil + b0 % oil;
        dstride = (long long)a.ep.oHp * a.ep.oWs * oil;
        sstride = 1;
        rstride = a.ep.oWs * oil;
        cstride = oil;
    } else {
        obase = (long long)b0 * a.ep.o_sample_stride + ((long long)orow + a.ep.oph) * a.ep.oWs + ocol + a.ep.opw;
        dstride = (long long)a.ep.oHp * a.ep.oWs;
        sstride = a.ep.o_sample_stride;
        rstride = a.ep.oWs;
        cstride = 1;
    }
    const bool vec = SPL == 2 && oil == IL;  // the lane's two samples adjacent: one vector store
    // residual shortcut (BI layout): element (b0, d, r + pr, col0 + pc) = rbase + d*rdst + pr*rrow + pc*ril
    long long rbase = 0, rdst = 0, rrow = 0;
    if (a.ep.residual) {
        rbase = (long long)(b0 / a.ep.ril) * a.ep.r_sample_stride +
                (((long long)r + a.ep.rph) * a.ep.rWs + col0 + a.ep.rpw) * a.ep.ril + b0 % a.ep.ril;
        rdst = (long long)a.ep.rHp * a.ep.rWs * a.ep.ril;
        rrow = (long long)a.ep.rWs * a.ep.ril;
    }
    const int ncol = min(PC, a.Yw - col0);
    const int nrow = min(PR, a.Yh - r);
#pragma unroll
    for (int dw = 0; dw < DW; ++dw) {
        if (part >= 0 && dw % a.split != part) continue;
        const int d = __ldg(pm + dw);
        if (d < 0) continue;
        const long long od = obase + d * dstride;
        float v[P][SPL];
#pragma unroll
        for (int p = 0; p < P; ++p) {
            O::unpack(acc[dw][p], v[p]);
            if constexpr (KIND == USC_F32 || KIND == USC_F16) {
                if (a.ep.residual) {
                    const int rr = r + p / PC, cc = col0 + p % PC;
                    if (rr < a.Yh && cc < a.Yw) {
                        float rv[SPL];
                        if (SPL == 2 && a.ep.ril == IL) {  // the lane's two samples adjacent: one load
                            const long long ri = rbase + (long long)d * rdst + (p / PC) * rrow + (p % PC) * IL;
                            if constexpr (KIND == USC_F32) {
                                const float2 q = *reinterpret_cast<const float2 *>(static_cast<const float *>(a.ep.res) + ri);
                                rv[0] = q.x;
                                rv[SPL - 1] = q.y;
                            } else {
                                const float2 q = __half22float2(
                                    *reinterpret_cast<const __half2 *>(static_cast<const __half *>(a.ep.res) + ri));
                                rv[0] = q.x;
                                rv[SPL - 1] = q.y;
                            }
                        } else {
#pragma unroll
                            for (int j = 0; j < SPL; ++j) rv[j] = b0 + j < a.N ? res_value<KIND>(a.ep, b0 + j, d, rr, cc) : 0.0f;
                        }
#pragma unroll
                        for (int j = 0; j < SPL; ++j) v[p][j] = epi_value_res<KIND>(v[p][j], a.ep, rv[j]);
                    }
                    continue;
                }
            }
#pragma unroll
            for (int j = 0; j < SPL; ++j) v[p][j] = epi_value<KIND>(v[p][j], a.ep);
        }
        // the thread's outputs: PC/2 pooled values of one row, or its P pixels
        float o[P][SPL];
        long long off[P];
        bool ok[P];
        int no = 0;
        if constexpr (PR == 2 && PC % 2 == 0) {
            if (pool) {
#pragma unroll
                for (int c2 = 0; c2 < PC / 2; ++c2) {
#pragma unroll
                    for (int j = 0; j < SPL; ++j)
                        o[c2][j] = pool4(v[2 * c2][j], v[2 * c2 + 1][j], v[PC + 2 * c2][j],
                                         v[PC + 2 * c2 + 1][j]);
                    off[c2] = od + c2 * cstride;
                    ok[c2] = 2 * c2 < ncol;
                }
                no = PC / 2;
            }
        }
        if (no == 0) {
#pragma unroll
            for (int p = 0; p < P; ++p) {
#pragma unroll
                for (int j = 0; j < SPL; ++j) o[p][j] = v[p][j];
                off[p] = od + (p / PC) * rstride + (p % PC) * cstride;
                ok[p] = (p / PC) < nrow && (p % PC) < ncol;
            }
            no = P;
        }
        const bool f32out = KIND == USC_F32 || (KIND == USC_I8 && !a.ep.requant);
        // sample-major layouts (plain NCHW / padded NCHW): a lane's pixels of one row are
        // contiguous, so full 4-pixel groups go out as one 16-byte (fp32) or 8-byte
        // (binary16) store per sample instead of four scalar ones
        if constexpr (PC % 4 == 0) {
            if (!vec && cstride == 1 && (sstride & 3) == 0 && (reinterpret_cast<uintptr_t>(a.y) & 15) == 0) {
                const int rows = no / PC > 0 ? no / PC : 1, per = no < PC ? no : PC;  // pooled: 1 row
#pragma unroll
                for (int rr = 0; rr < PR; ++rr) {
                    if (rr >= rows) break;
#pragma unroll
                    for (int q = 0; q < PC / 4; ++q) {
                        const int i = rr * per + 4 * q;
                        if (4 * q + 3 >= per || !ok[i] || !ok[i + 3] || (off[i] & 3)) continue;
#pragma unroll
                        for (int j = 0; j < SPL; ++j) {
                            if (b0 + j >= a.N) continue;
                            if (f32out)
                                *reinterpret_cast<float4 *>(static_cast<float *>(a.y) + off[i] + j * sstride) =
                                    make_float4(o[i][j], o[i + 1][j], o[i + 2][j], o[i + 3][j]);
                            else
                                *reinterpret_cast<uint2 *>(static_cast<__half *>(a.y) + off[i] + j * sstride) =
                                    make_uint2(pack_h2(o[i][j], o[i + 1][j]), pack_h2(o[i + 2][j], o[i + 3][j]));
                        }
#pragma unroll
                        for (int u = 0; u < 4; ++u) ok[i + u] = false;  // stored
                    }
                }
            }
        }
#pragma unroll
        for (int i = 0; i < P; ++i) {
            if (i >= no || !ok[i]) continue;
            if (f32out) {
                float *y = static_cast<float *>(a.y);
                if (vec) {
                    *reinterpret_cast<float2 *>(y + off[i]) = make_float2(o[i][0], o[i][SPL - 1]);
                } else {
#pragma unroll
                    for (int j = 0; j < SPL; ++j)
                        if (b0 + j < a.N) y[off[i] + j * sstride] = o[i][j];
                }
            } else {  // values are on the binary16 grid: the conversion is exact
                __half *y = static_cast<__half *>(a.y);
                if (vec) {
                    *reinterpret_cast<__half2 *>(y + off[i]) =
                        __halves2half2(__float2half_rn(o[i][0]), __float2half_rn(o[i][SPL - 1]));
                } else {
#pragma unroll
                    for (int j = 0; j < SPL; ++j)
                        if (b0 + j < a.N) y[off[i] + j * sstride] = __float2half_rn(o[i][j]);
                }
            }
        }
    }

}

// The common epilogue without the generic path's per-value flag tests: output (and
// residual shortcut, if any) in the padded BI layout of the kernel's interleave, no
// cap saturation / requantisation (launch_bi sets a.fast).  Per value:
//   F32: v = acc (+ r); ReLU
//   F16: v = sat16(acc) (+ r, sat16 again); ReLU; binary16 store
// The accumulator is never -0 (it starts at +0 and x + (-x) rounds to +0), so
// fmaxf(v, 0) is np.where(v > 0, v, 0) including NaN -> 0; ReLU commutes with the
// saturating binary16 rounding; ReLU'd values are NaN-free, so the fused 2x2 pool
// (only with ReLU) is a plain max (packed f16x2 for F16).
__device__ __forceinline__ float sat16_pre(float v) {  // finite |v| > 65504 -> +-65504 (sat_half)
    const float m = fabsf(v);
    return (m > 65504.0f && m != INFINITY) ? copysignf(65504.0f, v) : v;
}
__device__ __forceinline__ float relu_sat16_pre(float v) {  // sat16_pre(ReLU(v))
    v = fmaxf(v, 0.0f);
    const float c = fminf(v, 65504.0f);
    return v == INFINITY ? v : c;
}

// shortcut value type of one lane and pixel (SPL samples)
template <int KIND, int SPL>
using ResV = typename std::conditional<KIND == USC_F32, typename std::conditional<SPL == 1, float, float2>::type,
                                       __half2>::type;

// The fast epilogue's global loads -- the warp's output channels and, with a residual,
// the shortcut values of its DW x P outputs -- issued together so their latencies
// overlap (k_bi issues them before the input-channel loop when registers allow).
template <int KIND, int PC, int PR, int DW, int SPL, bool RES>
__device__ __forceinline__ void fast_loads(const BiArgs &a, int g, int wc, int sb, int r, int col0, int part,
                                           int lane, int (&dch)[DW], ResV<KIND, SPL> (&rv)[DW][PC * PR]) {
    constexpr int P = PC * PR;
    constexpr int IL = 32 * SPL;
    const int *pm = a.perm + g * a.DT + wc * DW;
#pragma unroll
    for (int dw = 0; dw < DW; ++dw) dch[dw] = (part >= 0 && dw % a.split != part) ? -1 : __ldg(pm + dw);
    if (!RES || !a.ep.residual) return;
    const int ncol = min(PC, a.Yw - col0), nrow = min(PR, a.Yh - r);
    const long long rbase = (long long)sb * a.ep.r_sample_stride +
                            (((long long)r + a.ep.rph) * a.ep.rWs + col0 + a.ep.rpw) * IL + lane * SPL;
    const long long rdst = (long long)a.ep.rHp * a.ep.rWs * IL;
    const int rrow = a.ep.rWs * IL;
    using RV = ResV<KIND, SPL>;
#pragma unroll
    for (int dw = 0; dw < DW; ++dw)
#pragma unroll
        for (int p = 0; p < P; ++p)
            if (dch[dw] >= 0 && p / PC < nrow && p % PC < ncol)
                rv[dw][p] = __ldg(reinterpret_cast<const RV *>(
                    static_cast<const char *>(a.ep.res) +
                    (rbase + dch[dw] * rdst + (p / PC) * rrow + (p % PC) * IL) * (KIND == USC_F32 ? 4 : 2)));
}

template <int KIND, int PC, int PR, int DW, int SPL, bool RES>
__device__ __forceinline__ void store_tile_fast(const BiArgs &a, typename Ops<KIND, SPL>::A (&acc)[DW][PC * PR],
                                                int sb, int r, int col0, int lane, const int (&dch)[DW],
                                                const ResV<KIND, SPL> (&rv)[DW][PC * PR]) {
    constexpr int P = PC * PR;
    constexpr int IL = 32 * SPL;
    constexpr bool POOLABLE = PR == 2 && PC % 2 == 0;
    const bool pool = POOLABLE && a.ep.pool, relu = a.ep.relu, res = RES && a.ep.residual;
    const int orow = pool ? r / 2 : r, ocol = pool ? col0 / 2 : col0;
    const long long obase = (long long)sb * a.ep.o_sample_stride +
                            (((long long)orow + a.ep.oph) * a.ep.oWs + ocol + a.ep.opw) * IL + lane * SPL;
    const long long dstride = (long long)a.ep.oHp * a.ep.oWs * IL;
    const int rstride = a.ep.oWs * IL;
    const int ncol = min(PC, a.Yw - col0), nrow = min(PR, a.Yh - r);
#pragma unroll
    for (int dw = 0; dw < DW; ++dw) {
        const int d = dch[dw];
        if (d < 0) continue;
        const long long od = obase + d * dstride;
        if constexpr (KIND == USC_F32) {
            float *y = static_cast<float *>(a.y) + od;
            float v[P][SPL];
#pragma unroll
            for (int p = 0; p < P; ++p) {
                if constexpr (SPL == 1) {
                    v[p][0] = acc[dw][p];
                } else {
                    Ops<KIND, SPL>::unpack(acc[dw][p], v[p]);
                }
                if (res && p / PC < nrow && p % PC < ncol) {
                    if constexpr (SPL == 1) {
                        v[p][0] = __fadd_rn(v[p][0], rv[dw][p]);
                    } else {
                        v[p][0] = __fadd_rn(v[p][0], rv[dw][p].x);
                        v[p][1] = __fadd_rn(v[p][1], rv[dw][p].y);
                    }
                }
                if (relu) {
#pragma unroll
                    for (int j = 0; j < SPL; ++j) v[p][j] = fmaxf(v[p][j], 0.0f);
                }
            }
            if (pool) {
                if constexpr (POOLABLE) {
#pragma unroll
                    for (int c2 = 0; c2 < PC / 2; ++c2) {
                        if (2 * c2 >= ncol) continue;
                        float o[SPL];
#pragma unroll
                        for (int j = 0; j < SPL; ++j)
                            o[j] = fmaxf(fmaxf(v[2 * c2][j], v[2 * c2 + 1][j]), fmaxf(v[PC + 2 * c2][j], v[PC + 2 * c2 + 1][j]));
                        if constexpr (SPL == 1)
                            y[c2 * IL] = o[0];
                        else
                            *reinterpret_cast<float2 *>(y + c2 * IL) = make_float2(o[0], o[SPL - 1]);
                    }
                }
            } else {
#pragma unroll
                for (int p = 0; p < P; ++p) {
                    if (p / PC >= nrow || p % PC >= ncol) continue;
                    float *q = y + (p / PC) * rstride + (p % PC) * IL;
                    if constexpr (SPL == 1)
                        *q = v[p][0];
                    else
                        *reinterpret_cast<float2 *>(q) = make_float2(v[p][0], v[p][SPL - 1]);
                }
            }
        } else if constexpr (KIND == USC_I8) {
            // int8 requantising epilogue with ReLU (quantization.py:61-76 on acc*sigma_w*sigma_x):
            // both scales are powers of two and acc is an exact integer, so the fp64
            // round-half-away-from-zero of acc*2^-s is (|acc| + 2^(s-1)) >> s, clamped
            // to +-limit -- integer ops, same codes (ReLU leaves no negative zero)
            __half *y = static_cast<__half *>(a.y) + od;
            const int sh = a.i8shift, lim = a.ep.rq_limit;
            auto code = [&](float v) -> int {
                const int m = max(__float2int_rn(v), 0);  // ReLU on the exact integer accumulator
                if (sh > 0) return min((m + (1 << (sh - 1))) >> sh, lim);
                return -sh >= 8 ? (m ? lim : 0) : min(m << -sh, lim);
            };
            int c[P][2];
#pragma unroll
            for (int p = 0; p < P; ++p) {
                c[p][0] = code(acc[dw][p].x);
                c[p][1] = code(acc[dw][p].y);
            }
            if (pool) {
                if constexpr (POOLABLE) {
#pragma unroll
                    for (int c2 = 0; c2 < PC / 2; ++c2) {
                        if (2 * c2 >= ncol) continue;
                        int o[2];
#pragma unroll
                        for (int j = 0; j < 2; ++j)
                            o[j] = max(max(c[2 * c2][j], c[2 * c2 + 1][j]), max(c[PC + 2 * c2][j], c[PC + 2 * c2 + 1][j]));
                        *reinterpret_cast<__half2 *>(y + c2 * IL) = __halves2half2(__int2half_rn(o[0]), __int2half_rn(o[1]));
                    }
                }
            } else {
#pragma unroll
                for (int p = 0; p < P; ++p) {
                    if (p / PC >= nrow || p % PC >= ncol) continue;
                    *reinterpret_cast<__half2 *>(y + (p / PC) * rstride + (p % PC) * IL) =
                        __halves2half2(__int2half_rn(c[p][0]), __int2half_rn(c[p][1]));
                }
            }
        } else if constexpr (KIND == USC_CB4) {
            // 4b/16b hook (quantization.py:238-244): round16(min(ReLU(round16(min(v, cap))), cap2)).
            // Tame tiles (every |v| < 65520, no NaN): one cvt per pixel, ReLU by sign bits,
            // and min with round16(cap2) -- equal to round16(min(x, cap2)) for x on the
            // binary16 grid (rounding is monotonic); otherwise the per-value epi_value.
            __half *y = static_cast<__half *>(a.y) + od;
            float v[P][2];
            uint32_t mx = 0;
#pragma unroll
            for (int p = 0; p < P; ++p) {
                Ops<KIND, SPL>::unpack(acc[dw][p], v[p]);
                mx = max(mx, max(__float_as_uint(v[p][0]) & 0x7fffffffu, __float_as_uint(v[p][1]) & 0x7fffffffu));
            }
            __half2 h[P];
            if (__all_sync(0xffffffffu, mx < 0x477FF000u)) {
                const float cap = a.ep.saturate ? a.ep.cap : INFINITY;
                const __half2 cap2 = a.ep.saturate2 ? __half2half2(sat_half(a.ep.cap2)) : __float2half2_rn(INFINITY);
#pragma unroll
                for (int p = 0; p < P; ++p) {
                    __half2 t = __floats2half2_rn(fminf(v[p][0], cap), fminf(v[p][1], cap));
                    if (relu) {
                        uint32_t b = *reinterpret_cast<uint32_t *>(&t), sg;
                        asm("prmt.b32 %0, %1, 0, 0xBB99;" : "=r"(sg) : "r"(b));
                        b &= ~sg;
                        t = *reinterpret_cast<__half2 *>(&b);
                    }
                    h[p] = __hmin2(t, cap2);
                }
            } else {
#pragma unroll
                for (int p = 0; p < P; ++p)
                    h[p] = __floats2half2_rn(epi_value<KIND>(v[p][0], a.ep), epi_value<KIND>(v[p][1], a.ep));
            }
            if (pool) {
                if constexpr (POOLABLE) {
#pragma unroll
                    for (int c2 = 0; c2 < PC / 2; ++c2) {
                        if (2 * c2 >= ncol) continue;
                        *reinterpret_cast<__half2 *>(y + c2 * IL) =
                            __hmax2(__hmax2(h[2 * c2], h[2 * c2 + 1]), __hmax2(h[PC + 2 * c2], h[PC + 2 * c2 + 1]));
                    }
                }
            } else {
#pragma unroll
                for (int p = 0; p < P; ++p) {
                    if (p / PC >= nrow || p % PC >= ncol) continue;
                    *reinterpret_cast<__half2 *>(y + (p / PC) * rstride + (p % PC) * IL) = h[p];
                }
            }
        } else {  // F16, SPL 2: one cvt.rn.f16x2 per pixel
            __half *y = static_cast<__half *>(a.y) + od;
            __half2 h[P];
            // "tame" tile (every |acc| < 65520, every shortcut finite -- the common case):
            // no saturation can trigger except on the residual sum, whose binary16 add
            // (HADD2, RN) equals round16 of the reference's fp32 add (fp32 has 24 >= 2*11+2
            // bits, so the double rounding is innocuous); overflow there is clamped to
            // 65504.  ReLU on the packed pair clears negative halves (and -0) by their
            // replicated sign bits.  Otherwise the per-value sat16 path below.
            uint32_t mx = 0, nf = 0;
#pragma unroll
            for (int p = 0; p < P; ++p) {
                mx = max(mx, max(__float_as_uint(acc[dw][p].x) & 0x7fffffffu, __float_as_uint(acc[dw][p].y) & 0x7fffffffu));
                if (res && p / PC < nrow && p % PC < ncol)
                    nf |= (*reinterpret_cast<const uint32_t *>(&rv[dw][p]) & 0x7c007c00u) + 0x04000400u;
            }
            const bool tame = mx < 0x477FF000u /* 65520.0f */ && !(nf & 0x80008000u);
            if (__all_sync(0xffffffffu, tame)) {
                const __half2 cap = __float2half2_rn(65504.0f), ncap = __float2half2_rn(-65504.0f);
#pragma unroll
                for (int p = 0; p < P; ++p) {
                    __half2 t = __floats2half2_rn(acc[dw][p].x, acc[dw][p].y);  // the conv's hook
                    if (res && p / PC < nrow && p % PC < ncol) t = __hadd2(t, rv[dw][p]);
                    if (relu) {
                        uint32_t b = *reinterpret_cast<uint32_t *>(&t), sg;
                        asm("prmt.b32 %0, %1, 0, 0xBB99;" : "=r"(sg) : "r"(b));  // sign of each half, replicated
                        b &= ~sg;
                        t = *reinterpret_cast<__half2 *>(&b);
                        if (res) t = __hmin2(t, cap);
                    } else if (res) {
                        t = __hmax2(__hmin2(t, cap), ncap);
                    }
                    h[p] = t;
                }
            } else {
#pragma unroll
                for (int p = 0; p < P; ++p) {
                    float2 v = acc[dw][p];
                    if (res) {
                        if (p / PC < nrow && p % PC < ncol) {
                            const float2 t = __half22float2(rv[dw][p]);
                            v = __half22float2(__floats2half2_rn(sat16_pre(v.x), sat16_pre(v.y)));  // the conv's hook
                            v.x = __fadd_rn(v.x, t.x);
                            v.y = __fadd_rn(v.y, t.y);
                        }
                    }
                    h[p] = relu ? __floats2half2_rn(relu_sat16_pre(v.x), relu_sat16_pre(v.y))
                                : __floats2half2_rn(sat16_pre(v.x), sat16_pre(v.y));
                }
            }
            if (pool) {
                if constexpr (POOLABLE) {
#pragma unroll
                    for (int c2 = 0; c2 < PC / 2; ++c2) {
                        if (2 * c2 >= ncol) continue;
                        *reinterpret_cast<__half2 *>(y + c2 * IL) =
                            __hmax2(__hmax2(h[2 * c2], h[2 * c2 + 1]), __hmax2(h[PC + 2 * c2], h[PC + 2 * c2 + 1]));
                    }
                }
            } else {
#pragma unroll
                for (int p = 0; p < P; ++p) {
                    if (p / PC >= nrow || p % PC >= ncol) continue;
                    *reinterpret_cast<__half2 *>(y + (p / PC) * rstride + (p % PC) * IL) = h[p];
                }
            }
        }
    }
}

// RES: the residual-epilogue variant (shortcut values prefetched before the channel
// loop when their registers fit); launch_inst selects it for fast residual epilogues
template <int KIND, int PC, int PR, int DW, int SW, int NWC, int SPL, bool RES>
__global__ void __launch_bounds__((NWC + 1) * 32, 1) k_bi(const __grid_constant__ BiArgs a) {
    using O = Ops<KIND, SPL>;
    using A = typename O::A;
    constexpr int P = PC * PR;          // a thread's pixel block: PR rows x PC cols
    constexpr int IL = 32 * SPL;        // samples per interleave block
    constexpr int PXB = O::EB * IL;     // bytes per staged pixel
    // software-pipeline the pair loop when the second value set fits the register cap
    constexpr int REGCAP = NWC <= 8 ? 168 : (NWC <= 12 ? 128 : 96);
    constexpr int VR = (KIND == USC_F32) ? SPL : 1;  // registers per staged value
    constexpr bool PIPE = SPL * DW * P + 4 * P * VR + (KIND == USC_F32 ? 40 : 56) <= REGCAP;
    constexpr int RVR = (KIND == USC_F32) ? SPL : 1;  // registers per shortcut value
    constexpr bool RPRE = RES && (KIND == USC_F32 || KIND == USC_F16) &&
                          SPL * DW * P + (PIPE ? 4 : 2) * P * VR + DW * P * RVR + 40 <= REGCAP;
    // otherwise the shortcut loads go out at the start of the last chunk, whose pair loop then
    // runs without software pipelining so the shortcut registers fit the cap
    constexpr bool LPRE = RES && !RPRE && (KIND == USC_F32 || KIND == USC_F16) &&
                          SPL * DW * P + 2 * P * VR + DW * P * RVR + 40 <= REGCAP;
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t *full = reinterpret_cast<uint64_t *>(smem);
    uint64_t *empty = full + 8;
    unsigned char *ring = smem + 128;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) {
        for (int s = 0; s < a.S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], NWC);
        }
        fence_mbar_init();
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&a.xmap)) : "memory");
    }
    __syncthreads();
    pdl_release();
    // every global access below waits for the previous kernel's output, except the producer's
    // entry blocks for the first S stages (the packed filter: constant data)
    if (warp != NWC) pdl_wait();

    if (warp == NWC) {
        // ---------------- producer warp ----------------
        if (lane == 0) {
            int s = 0;
            uint32_t ph = 1;
            const uint32_t xbytes = static_cast<uint32_t>(a.CC) * a.HS * a.TWs * PXB;  // full box
            int pre = 0;  // stages whose entry block went out before the wait
            for (int it = blockIdx.x; it < a.items && pre < a.S; it += gridDim.x) {
                int part;
                const int g = item_tile(a, it, part) % a.G;
                const int *blk_g = a.blk + g * a.n_chunks;
                for (int k = 0; k < a.n_chunks && pre < a.S; ++k, ++pre) {
                    const int lo = __ldg(blk_g + k), hi = __ldg(blk_g + k + 1);
                    const uint32_t eb = static_cast<uint32_t>(hi - lo);
                    mbar_expect_tx(&full[pre], xbytes + eb);
                    bulk_g2s(ring + pre * a.stage_bytes + a.x_stage_bytes, a.blocks + lo, eb, &full[pre]);
                }
            }
            pdl_wait();
            int n_st = 0;
            for (int it = blockIdx.x; it < a.items; it += gridDim.x) {
                int part;
                int q = item_tile(a, it, part);
                const int g = q % a.G;
                q /= a.G;
                const int ct = q % a.col_tiles;
                q /= a.col_tiles;
                const int rt = q % a.row_tiles;
                const int sb = q / a.row_tiles;
                const int y0 = rt * a.TH * a.s_h;
                const int x0 = ct * a.SPRt * PC * SW;
                const int *blk_g = a.blk + g * a.n_chunks;
                for (int k = 0; k < a.n_chunks; ++k, ++n_st) {
                    mbar_wait(&empty[s], ph);
                    unsigned char *st = ring + s * a.stage_bytes;
                    if (n_st >= pre) {  // (the first `pre` stages' entries are already in flight)
                        const int lo = __ldg(blk_g + k), hi = __ldg(blk_g + k + 1);
                        const uint32_t eb = static_cast<uint32_t>(hi - lo);
                        mbar_expect_tx(&full[s], xbytes + eb);
                        bulk_g2s(st + a.x_stage_bytes, a.blocks + lo, eb, &full[s]);
                    }
                    tma_load_5d(st, &a.xmap, 0, x0, y0, k * a.CC, sb, &full[s]);
                    if (++s == a.S) {
                        s = 0;
                        ph ^= 1;
                    }
                }
            }
        }
        return;
    }

    // ---------------- compute warps ----------------
    const int wsi = warp % a.WS, wc = warp / a.WS;
    const bool active = wc < a.WC;
    const int tr = wsi / a.SPRt, tcs = wsi - tr * a.SPRt;  // strip-row, strip within the tile
    const uint32_t base = ((tr * PR * a.s_h) * a.TWs + tcs * PC * SW) * PXB + lane * O::EB * SPL;
    const uint32_t rs = a.s_h * a.TWs * PXB;  // bytes between a thread's two pixel rows
    const int hdr_bytes = (a.ncls * a.DT * 8 + 15) & ~15;  // entries start 16-B aligned
    int s = 0;
    uint32_t ph = 0;
    for (int it = blockIdx.x; it < a.items; it += gridDim.x) {
        int part;
        int q = item_tile(a, it, part);
        int q2 = fdiv(q, a.fG);
        const int g = q - q2 * a.G;
        q = fdiv(q2, a.fCT);
        const int ct = q2 - q * a.col_tiles;
        const int sb = fdiv(q, a.fRT);
        const int rt = q - sb * a.row_tiles;
        const int r = rt * a.TH + tr * PR;
        const int col0 = (ct * a.SPRt + tcs) * PC;
        // pixel class (1x1 blocks): selects the runs without this pixel's halo taps
        const int cls = (a.ncls > 1 && r < a.Yh && col0 < a.Yw)
                            ? __ldg(a.rowcls + r) * a.ncls_c + __ldg(a.colcls + col0) : 0;

        // fast epilogue loads issued before the channel loop (latency hidden by it) when
        // the shortcut registers fit the cap, else right before the epilogue
        int dch[DW];
        ResV<KIND, SPL> rv[DW][P];
        if constexpr (RPRE) {
            if (a.fast && active && r < a.Yh) fast_loads<KIND, PC, PR, DW, SPL, RES>(a, g, wc, sb, r, col0, part, lane, dch, rv);
        }

        A acc[DW][P];
#pragma unroll
        for (int i = 0; i < DW; ++i)
#pragma unroll
            for (int p = 0; p < P; ++p) O::zero(acc[i][p]);

        for (int k = 0; k < a.n_chunks; ++k) {
            const uint32_t st = smem_u32(ring + s * a.stage_bytes);
            const bool late = LPRE && k == a.n_chunks - 1;
            if constexpr (LPRE) {
                if (late && a.fast && active && r < a.Yh)
                    fast_loads<KIND, PC, PR, DW, SPL, RES>(a, g, wc, sb, r, col0, part, lane, dch, rv);
            }
            mbar_wait(&full[s], ph);
            if (active) {
                const uint32_t xs = st + base;  // this thread's first pixel, tap (0,0,0)
                const uint32_t bp = st + a.x_stage_bytes;
                const uint32_t hdr = bp + (cls * a.DT + wc * DW) * 8, E = bp + hdr_bytes;
#pragma unroll
                for (int dw = 0; dw < DW; ++dw) {
                    const int2 h = lds_v2(hdr + dw * 8);  // run [h.x, h.y), h.x even
                    if (part >= 0 && dw % a.split != part) continue;
                    if (LPRE && late)
                        run_pairs<KIND, PC, PR, SW, SPL, false>(acc[dw], xs, rs, E + h.x * 8, E + h.y * 8);
                    else
                        run_pairs<KIND, PC, PR, SW, SPL, PIPE>(acc[dw], xs, rs, E + h.x * 8, E + h.y * 8);
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
            if (++s == a.S) {
                s = 0;
                ph ^= 1;
            }
        }

        if (active && r < a.Yh) {
            if constexpr (KIND == USC_F32 || KIND == USC_F16 || KIND == USC_I8 || KIND == USC_CB4) {
                if (a.fast) {
                    if constexpr (!RPRE && !LPRE)
                        fast_loads<KIND, PC, PR, DW, SPL, RES>(a, g, wc, sb, r, col0, part, lane, dch, rv);
                    store_tile_fast<KIND, PC, PR, DW, SPL, RES>(a, acc, sb, r, col0, lane, dch, rv);
                    continue;
                }
            }
            store_tile<KIND, PC, PR, DW, SPL>(a, acc, g, wc, sb, r, col0, part, lane);
        }
    }
}

template <int KIND, int PC, int PR, int DW, int SW, int NWC, int SPL>
int launch_inst(const usc_plan *pl, const BiArgs &a, cudaStream_t st) {
    constexpr bool HAS_RES = KIND == USC_F32 || KIND == USC_F16;
    const bool res = HAS_RES && a.fast && a.ep.residual;
    auto fn = res ? k_bi<KIND, PC, PR, DW, SW, NWC, SPL, HAS_RES> : k_bi<KIND, PC, PR, DW, SW, NWC, SPL, false>;
    static std::atomic<uint64_t> attr_res{0}, attr_plain{0};
    std::atomic<uint64_t> &attr = res ? attr_res : attr_plain;
    cudaError_t ae = ensure_smem_attr(fn, attr, 224 * 1024);
    if (ae != cudaSuccess) return usc::fail(USC_ERR_CUDA, "smem attribute: %s", cudaGetErrorString(ae));
    cudaError_t e = launch_pdl(fn, dim3(static_cast<unsigned>(pl->grid_x)), dim3((NWC + 1) * 32), pl->smem_bytes, st, a);
    if (e == cudaSuccess) e = cudaGetLastError();
    if (e != cudaSuccess) return usc::fail(USC_ERR_CUDA, "k_bi launch: %s", cudaGetErrorString(e));
    return USC_OK;
}

// fp32 instances with 8 (168 regs), 12 (128) and 16 (96) compute warps; binary16-input
// (F16, CB4) instances
int launch_w8(const usc_plan *pl, const BiArgs &a, cudaStream_t st);
int launch_w12(const usc_plan *pl, const BiArgs &a, cudaStream_t st);
int launch_w16(const usc_plan *pl, const BiArgs &a, cudaStream_t st);
int launch_h16(const usc_plan *pl, const BiArgs &a, cudaStream_t st);
int launch_hcb(const usc_plan *pl, const BiArgs &a, cudaStream_t st);
int launch_hi8(const usc_plan *pl, const BiArgs &a, cudaStream_t st);

}  // namespace usc_bi
