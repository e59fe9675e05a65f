// k_tconv instantiation: which template instance serves a (MODE, precision, BN,
// swap, CTAs per SM, cluster kind) request.  Each MODE's instances are compiled
// in their own translation unit (inst_m<MODE>.cu, built in parallel) and reached
// through tconv_pick_mode (b2conv.cu's only entry into them).
#pragma once
#include "k_tma.cuh"

namespace b2c {

using TconvKernel = void (*)(const CUtensorMap, const CUtensorMap, TArgs);

struct TconvEntry {
    TconvKernel fn;
    int smem;
    int threads;
};

template <int BN, bool SWAP, int MODE, int OCC, int CL, int PREC = 0>
TconvEntry tconv_entry() {
    using C = TmaCfg<BN, SWAP, MODE, OCC, CL, PREC>;
    return TconvEntry{&k_tconv<BN, SWAP, MODE, OCC, CL, PREC>, C::SMEM, C::THREADS};
}

template <int MODE>
TconvEntry tconv_pick_bf16(int bn) {
    switch (bn) {
        case 32: return tconv_entry<32, false, MODE, 1, 1, 1>();
        case 64: return tconv_entry<64, false, MODE, 1, 1, 1>();
        case 128: return tconv_entry<128, false, MODE, 1, 1, 1>();
        case 192: return tconv_entry<192, false, MODE, 1, 1, 1>();
    }
    return TconvEntry{nullptr, 0, 0};
}

template <int MODE>
TconvEntry tconv_pick_fp8(int bn) {
    switch (bn) {
        case 32: return tconv_entry<32, false, MODE, 1, 1, 2>();
        case 64: return tconv_entry<64, false, MODE, 1, 1, 2>();
        case 128: return tconv_entry<128, false, MODE, 1, 1, 2>();
    }
    return TconvEntry{nullptr, 0, 0};
}

template <bool SWAP, int MODE>
TconvEntry tconv_pick_bn(int bn, int occ, int cl) {
    if (cl == 2) {
        if constexpr (!SWAP && MODE != 1 && MODE != 5 && MODE != 6) {
            switch (bn) {
                case 64: return tconv_entry<64, false, MODE, 1, 2>();
                case 96: return tconv_entry<96, false, MODE, 1, 2>();
                case 128: return tconv_entry<128, false, MODE, 1, 2>();
                case 192: return tconv_entry<192, false, MODE, 1, 2>();
            }
        }
        return TconvEntry{nullptr, 0, 0};
    }
    if (cl == 4) {  // split-K clusters (DSMEM fixup)
        if constexpr (!SWAP && (MODE == 0 || MODE == 5 || MODE == 6)) {
            switch (bn) {
                case 32: return tconv_entry<32, false, MODE, 1, 4>();
                case 64: return tconv_entry<64, false, MODE, 1, 4>();
            }
        }
        if constexpr (SWAP && MODE == 1) {
            if (bn == 32) return tconv_entry<32, true, 1, 1, 4>();
        }
        return TconvEntry{nullptr, 0, 0};
    }
    if (cl == 3) {  // 2-SM UMMA pairs
        if constexpr (!SWAP && MODE != 1 && MODE != 2 && MODE != 3) {
            switch (bn) {
                case 64: return tconv_entry<64, false, MODE, 1, 3>();
                case 96: return tconv_entry<96, false, MODE, 1, 3>();
                case 128: return tconv_entry<128, false, MODE, 1, 3>();
                case 192: return tconv_entry<192, false, MODE, 1, 3>();
            }
        }
        return TconvEntry{nullptr, 0, 0};
    }
    if constexpr (SWAP && MODE == 1) {  // fc weights on M, a 16-image pixel tile (batch <= 16)
        if (bn == 16 && cl == 1) return occ == 2 ? tconv_entry<16, true, 1, 2, 1>() : tconv_entry<16, true, 1, 1, 1>();
    }
    if (occ == 2) {
        switch (bn) {
            case 32: return tconv_entry<32, SWAP, MODE, 2, 1>();
            case 64: return tconv_entry<64, SWAP, MODE, 2, 1>();
        }
        return TconvEntry{nullptr, 0, 0};
    }
    switch (bn) {
        case 32: return tconv_entry<32, SWAP, MODE, 1, 1>();
        case 64: return tconv_entry<64, SWAP, MODE, 1, 1>();
        case 96: return tconv_entry<96, SWAP, MODE, 1, 1>();
        case 128: return tconv_entry<128, SWAP, MODE, 1, 1>();
        case 192: return tconv_entry<192, SWAP, MODE, 1, 1>();
    }
    return TconvEntry{nullptr, 0, 0};
}

template <int MODE>
TconvEntry tconv_pick_sw(int bn, int swap, int occ, int cl) {
    return swap ? tconv_pick_bn<true, MODE>(bn, occ, cl) : tconv_pick_bn<false, MODE>(bn, occ, cl);
}

// Winograd GEMMs (MODE 7): raw U / V matrices, either orientation
template <bool SWAP>
TconvEntry wino_pick(int bn) {
    switch (bn) {
        case 64: return tconv_entry<64, SWAP, 7, 1, 1>();
        case 128: return tconv_entry<128, SWAP, 7, 1, 1>();
        case 192: return tconv_entry<192, SWAP, 7, 1, 1>();
    }
    return TconvEntry{nullptr, 0, 0};
}

template <int MODE>
TconvEntry tconv_pick_impl(int prec, int bn, int swap, int occ, int cl) {
    constexpr bool has_bf16 = MODE == 0 || MODE == 2 || MODE == 4 || MODE == 5 || MODE == 6 || MODE == 8;
    constexpr bool has_fp8 = MODE == 0 || MODE == 4 || MODE == 5 || MODE == 6;
    if (prec == 1) {
        if constexpr (MODE == 8) {
            if (cl == 3)
                return bn == 128 ? tconv_entry<128, false, 8, 1, 3, 1>()
                       : bn == 192 ? tconv_entry<192, false, 8, 1, 3, 1>() : TconvEntry{nullptr, 0, 0};
        }
        if constexpr (has_bf16) return tconv_pick_bf16<MODE>(bn);
        return TconvEntry{nullptr, 0, 0};
    }
    if (prec == 2) {
        if constexpr (has_fp8) return tconv_pick_fp8<MODE>(bn);
        return TconvEntry{nullptr, 0, 0};
    }
    if constexpr (MODE == 8) {
        return TconvEntry{nullptr, 0, 0};
    } else if constexpr (MODE == 7) {
        return swap ? wino_pick<true>(bn) : wino_pick<false>(bn);
    } else if constexpr (MODE >= 4) {
        return swap ? TconvEntry{nullptr, 0, 0} : tconv_pick_bn<false, MODE>(bn, occ, cl);
    } else {
        return swap ? tconv_pick_bn<true, MODE>(bn, occ, cl) : tconv_pick_bn<false, MODE>(bn, occ, cl);
    }
}

#define B2C_DECLARE_PICK(M) TconvEntry tconv_pick_m##M(int prec, int bn, int swap, int occ, int cl);
B2C_DECLARE_PICK(0)
B2C_DECLARE_PICK(1)
B2C_DECLARE_PICK(2)
B2C_DECLARE_PICK(3)
B2C_DECLARE_PICK(4)
B2C_DECLARE_PICK(5)
B2C_DECLARE_PICK(6)
B2C_DECLARE_PICK(7)
B2C_DECLARE_PICK(8)
#undef B2C_DECLARE_PICK

#define B2C_DEFINE_PICK(M) \
    TconvEntry tconv_pick_m##M(int prec, int bn, int swap, int occ, int cl) { return tconv_pick_impl<M>(prec, bn, swap, occ, cl); }

inline TconvEntry tconv_pick_mode(int mode, int prec, int bn, int swap, int occ, int cl) {
    switch (mode) {
        case 0: return tconv_pick_m0(prec, bn, swap, occ, cl);
        case 1: return tconv_pick_m1(prec, bn, swap, occ, cl);
        case 2: return tconv_pick_m2(prec, bn, swap, occ, cl);
        case 3: return tconv_pick_m3(prec, bn, swap, occ, cl);
        case 4: return tconv_pick_m4(prec, bn, swap, occ, cl);
        case 5: return tconv_pick_m5(prec, bn, swap, occ, cl);
        case 6: return tconv_pick_m6(prec, bn, swap, occ, cl);
        case 7: return tconv_pick_m7(prec, bn, swap, occ, cl);
        case 8: return tconv_pick_m8(prec, bn, swap, occ, cl);
    }
    return TconvEntry{nullptr, 0, 0};
}

}  // namespace b2c
