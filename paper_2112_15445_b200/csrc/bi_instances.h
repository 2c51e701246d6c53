// bi_instances.h -- the k_bi tile instances compiled into the library, one list
// per compute-warp count.  X(PC, PR, DW, SW, SPL): a thread's pixel block is PR rows
// x PC columns (column stride SW), DW output channels per warp, SPL samples per lane
// (1: BI32 layout, 2: BI64).  The planner (host.cpp) and the launchers
// (conv_bi_w*.cu) both expand these lists, so they cannot disagree.  SPL*DW*PC*PR
// accumulator registers must fit the register cap of the warp count: 168 (8 compute
// warps), 128 (12), 96 (16).
#pragma once

#define USC_BI_W8(X)                                                                                      \
    X(4, 2, 8, 1, 1) X(8, 2, 4, 1, 1) X(8, 1, 8, 1, 1) X(4, 2, 16, 1, 1) X(8, 2, 8, 1, 1) X(4, 1, 16, 1, 1) \
    X(2, 2, 16, 1, 1) X(8, 1, 16, 1, 1) X(2, 2, 8, 1, 1) X(1, 1, 16, 1, 1) X(2, 2, 4, 1, 1)                \
    X(2, 2, 2, 1, 1) X(2, 1, 4, 1, 1) X(1, 1, 4, 1, 1) X(4, 1, 8, 2, 1) X(8, 1, 8, 2, 1)                  \
    X(4, 2, 4, 1, 2) X(8, 1, 4, 1, 2) X(2, 2, 8, 1, 2) X(4, 2, 8, 1, 2) X(8, 2, 4, 1, 2) X(2, 2, 4, 1, 2)   \
    X(4, 1, 8, 1, 2) X(2, 1, 8, 1, 2) X(1, 1, 8, 1, 2) X(1, 1, 4, 1, 2) X(2, 2, 2, 1, 2) X(4, 1, 4, 2, 2)   \
    X(4, 2, 4, 2, 2) X(8, 1, 4, 2, 2)

#define USC_BI_W12(X)                                                                                     \
    X(4, 2, 8, 1, 1) X(8, 2, 4, 1, 1) X(8, 1, 8, 1, 1) X(2, 2, 16, 1, 1) X(4, 1, 16, 1, 1) X(2, 2, 8, 1, 1) \
    X(4, 2, 4, 1, 1) X(8, 1, 4, 1, 1) X(2, 1, 16, 1, 1) X(4, 1, 8, 2, 1)                                   \
    X(4, 2, 4, 1, 2) X(2, 2, 8, 1, 2) X(8, 1, 4, 1, 2) X(2, 2, 4, 1, 2) X(4, 1, 4, 1, 2)                   \
    X(4, 2, 4, 2, 2) X(4, 1, 4, 2, 2)

#define USC_BI_W16(X)                                                                                     \
    X(2, 2, 8, 1, 1) X(4, 2, 4, 1, 1) X(2, 2, 4, 1, 1) X(4, 1, 8, 1, 1) X(8, 1, 4, 1, 1) X(1, 1, 16, 1, 1) \
    X(2, 1, 16, 1, 1) X(1, 2, 16, 1, 1) X(2, 2, 2, 1, 1) X(4, 1, 4, 2, 1) X(2, 1, 8, 2, 1) X(1, 1, 8, 2, 1) \
    X(2, 2, 4, 1, 2) X(4, 1, 4, 1, 2) X(2, 2, 2, 1, 2) X(4, 2, 2, 1, 2) X(1, 1, 8, 1, 2) X(1, 1, 4, 1, 2)  \
    X(1, 1, 2, 1, 2) X(4, 2, 2, 2, 2) X(4, 1, 4, 2, 2) X(8, 1, 2, 2, 2)

// binary16-input kinds (F16: FHFMA; CB4: FMUL + FADD2), BI64 only (two samples per
// lane as one 32-bit half2 load).  X(NW, PC, PR, DW, SW), each built for F16 and CB4.
#define USC_BI_H(X)                                                                                  \
    X(8, 4, 2, 4, 1) X(8, 2, 2, 8, 1) X(8, 8, 1, 4, 1) X(8, 2, 2, 4, 1)               \
    X(8, 1, 1, 8, 1) X(8, 4, 1, 8, 2) X(12, 4, 2, 4, 1) X(12, 8, 1, 4, 1)            \
    X(12, 2, 2, 4, 1) X(16, 2, 2, 4, 1) X(16, 4, 1, 4, 1) X(16, 2, 2, 2, 1) X(16, 4, 2, 2, 1)          \
    X(16, 1, 1, 8, 1) X(16, 4, 1, 4, 2) X(12, 4, 2, 2, 1) X(12, 8, 1, 2, 1) X(12, 4, 1, 4, 1)           \
    X(8, 8, 2, 2, 1) X(16, 8, 1, 2, 1) X(16, 1, 1, 4, 1) X(8, 1, 1, 4, 1) X(16, 8, 2, 1, 1) X(12, 8, 2, 1, 1) \
    X(16, 4, 2, 2, 2) X(12, 4, 2, 4, 2) X(16, 8, 1, 2, 2)

// tensor-memory-fed fp32 BI64 kernel (kernel 4, conv_bt.cuh).  X(NW, PC, PR, DW),
// NW a multiple of 4 (the compute warps of each lane quarter fill its TMEM copy).
#define USC_BT(X)                                                                               \
    X(8, 2, 2, 8) X(8, 4, 2, 4) X(8, 4, 1, 8) X(8, 8, 1, 4) X(8, 2, 1, 16) X(12, 2, 2, 8) X(12, 4, 2, 4) \
    X(12, 4, 1, 8) X(12, 8, 1, 4) X(16, 2, 2, 4) X(16, 4, 1, 4) X(16, 2, 1, 8)

// register-window kernel (k_bw, conv_bw.cuh): X(FAMILY, NW, PC, DW, KW) -- FAMILY 0 =
// fp32 (F32), 1 = binary16 input (F16); a thread's block is one row of PC pixels, DW
// slots share the merged entry stream, KW = filter width (3 or 1), BI64, stride 1.
// Registers: 2*DW*PC accumulators + (PC+KW-1)*(FAMILY ? 1 : 2) window values under the
// cap of the warp count (168 for 8 compute warps, 128 for 12); DW*PC = 64 spills.
#define USC_BW(X)                                                                                    \
    X(0, 8, 4, 12, 3) X(0, 8, 4, 8, 3) X(0, 12, 4, 8, 3) X(0, 8, 4, 12, 1) X(0, 12, 4, 8, 1)           \
    X(1, 8, 4, 12, 3) X(1, 8, 4, 8, 3) X(1, 12, 4, 8, 3) X(1, 8, 4, 12, 1) X(1, 12, 4, 8, 1)
