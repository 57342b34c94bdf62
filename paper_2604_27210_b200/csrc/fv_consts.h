// fv_consts.h -- every FP64 constant of the device code that is not a
// high-word-only immediate, routed through one __constant__ block on the
// device.  sm_100a FP64 instructions take no 64-bit immediates: a literal
// such as 0x1.555555555543cp-3 costs two UMOV/IMAD.MOV issue slots per use,
// a __constant__ operand one LDC.64 (usually hoisted).  The host pass keeps
// the literal values (fv_tables.h).  Values are unchanged bit for bit.
#pragma once

// Divisors the reference divides by, with yh = RN(1/c) and yl = RN(1/c - yh)
// for fv_div_const (Markstein-corrected reciprocal product; see fv_libm.h).
#define FV_DIV_SQRT2_C 0x1.6a09e667f3bcdp+0
#define FV_DIV_SQRT2_YH 0x1.6a09e667f3bccp-1
#define FV_DIV_SQRT2_YL 0x1.08b2fb1366eaap-56
#define FV_DIV_6_YH 0x1.5555555555555p-3
#define FV_DIV_6_YL 0x1.5555555555555p-57
#define FV_DIV_120_YH 0x1.1111111111111p-7
#define FV_DIV_120_YL 0x1.1111111111111p-63
#define FV_DIV_5040_YH 0x1.a01a01a01a01ap-13
#define FV_DIV_5040_YL 0x1.a01a01a01a01ap-73
#define FV_DIV_362880_YH 0x1.71de3a556c734p-19
#define FV_DIV_362880_YL -0x1.c154f8ddc6c00p-73
#define FV_DIV_39916800_YH 0x1.ae64567f544e4p-26
#define FV_DIV_39916800_YL -0x1.c062e06d1f209p-80
#define FV_DIV_6227020800_YH 0x1.6124613a86d09p-33
#define FV_DIV_6227020800_YL 0x1.f28e0cc748ebep-87
#define FV_DIV_365_YH 0x1.6719f3601671ap-9
#define FV_DIV_365_YL -0x1.93fd31cc193fdp-66
#define FV_DIV_100_YH 0x1.47ae147ae147bp-7
#define FV_DIV_100_YL -0x1.eb851eb851eb8p-63

#define FV_K_1EM300 1e-300
#define FV_K_ONE_M_1EM15 (1.0 - 1e-15)
#define FV_K_1EM12 1e-12
#define FV_K_1EM14 1e-14
#define FV_K_1EM10 1e-10
#define FV_K_1EM9 1e-9
#define FV_K_1EM6 1e-6
#define FV_K_ONE_M_1EM6 (1.0 - 1e-6)
#define FV_K_ONE_P_1EM6 (1.0 + 1e-6)
#define FV_K_0P999 0.999
#define FV_K_MIN_SUB 5e-324
#define FV_K_0P425 0.425
#define FV_K_0P180625 0.180625
#define FV_K_1P6 1.6
#define FV_K_0P85 0.85
#define FV_K_0P05 0.05
#define FV_K_ISPI 0.56418958354775628694807945156
#define FV_K_M26P7 -26.7
#define FV_K_M6P1 -6.1
#define FV_K_TWO_M_TINY (2.0 - 1e-300)

struct FvK {
  double DIV_SQRT2_C;
  double DIV_SQRT2_YH;
  double DIV_SQRT2_YL;
  double DIV_6_YH;
  double DIV_6_YL;
  double DIV_120_YH;
  double DIV_120_YL;
  double DIV_5040_YH;
  double DIV_5040_YL;
  double DIV_362880_YH;
  double DIV_362880_YL;
  double DIV_39916800_YH;
  double DIV_39916800_YL;
  double DIV_6227020800_YH;
  double DIV_6227020800_YL;
  double DIV_365_YH;
  double DIV_365_YL;
  double DIV_100_YH;
  double DIV_100_YL;
  double ERFC_ERX;
  double ERFC_ONE_M_ERX;
  double ERFC_PA0;
  double ERFC_PA1;
  double ERFC_PA2;
  double ERFC_PA3;
  double ERFC_PA4;
  double ERFC_PA5;
  double ERFC_PA6;
  double ERFC_PP0;
  double ERFC_PP1;
  double ERFC_PP2;
  double ERFC_PP3;
  double ERFC_PP4;
  double ERFC_QA1;
  double ERFC_QA2;
  double ERFC_QA3;
  double ERFC_QA4;
  double ERFC_QA5;
  double ERFC_QA6;
  double ERFC_QQ1;
  double ERFC_QQ2;
  double ERFC_QQ3;
  double ERFC_QQ4;
  double ERFC_QQ5;
  double ERFC_RA0;
  double ERFC_RA1;
  double ERFC_RA2;
  double ERFC_RA3;
  double ERFC_RA4;
  double ERFC_RA5;
  double ERFC_RA6;
  double ERFC_RA7;
  double ERFC_RB0;
  double ERFC_RB1;
  double ERFC_RB2;
  double ERFC_RB3;
  double ERFC_RB4;
  double ERFC_RB5;
  double ERFC_RB6;
  double ERFC_SA1;
  double ERFC_SA2;
  double ERFC_SA3;
  double ERFC_SA4;
  double ERFC_SA5;
  double ERFC_SA6;
  double ERFC_SA7;
  double ERFC_SA8;
  double ERFC_SB1;
  double ERFC_SB2;
  double ERFC_SB3;
  double ERFC_SB4;
  double ERFC_SB5;
  double ERFC_SB6;
  double ERFC_SB7;
  double EXP_C2;
  double EXP_C3;
  double EXP_C4;
  double EXP_C5;
  double EXP_INVLN2N;
  double EXP_NEGLN2HIN;
  double EXP_NEGLN2LON;
  double HALF_ONE_MINUS_EPS;
  double HALF_SQRT_TWO_PI;
  double INV_SQRT_TWO_PI;
  double LOG_A0;
  double LOG_A1;
  double LOG_A2;
  double LOG_A3;
  double LOG_A4;
  double LOG_B1;
  double LOG_B10;
  double LOG_B2;
  double LOG_B3;
  double LOG_B4;
  double LOG_B5;
  double LOG_B6;
  double LOG_B7;
  double LOG_B8;
  double LOG_B9;
  double LOG_INV_SQRT_TWO_PI;
  double LOG_LN2HI;
  double LOG_LN2LO;
  double POW_A1;
  double POW_A2;
  double POW_A3;
  double POW_A4;
  double POW_A5;
  double POW_A6;
  double POW_LN2HI;
  double POW_LN2LO;
  double SMALL_T_THRESHOLD;
  double SQRT_TWO;
  double TWO_PI;
  double AS241_A0;
  double AS241_A1;
  double AS241_A2;
  double AS241_A3;
  double AS241_A4;
  double AS241_A5;
  double AS241_A6;
  double AS241_A7;
  double AS241_B0;
  double AS241_B1;
  double AS241_B2;
  double AS241_B3;
  double AS241_B4;
  double AS241_B5;
  double AS241_B6;
  double AS241_B7;
  double AS241_C0;
  double AS241_C1;
  double AS241_C2;
  double AS241_C3;
  double AS241_C4;
  double AS241_C5;
  double AS241_C6;
  double AS241_C7;
  double AS241_D0;
  double AS241_D1;
  double AS241_D2;
  double AS241_D3;
  double AS241_D4;
  double AS241_D5;
  double AS241_D6;
  double AS241_D7;
  double AS241_E0;
  double AS241_E1;
  double AS241_E2;
  double AS241_E3;
  double AS241_E4;
  double AS241_E5;
  double AS241_E6;
  double AS241_E7;
  double AS241_F0;
  double AS241_F1;
  double AS241_F2;
  double AS241_F3;
  double AS241_F4;
  double AS241_F5;
  double AS241_F6;
  double AS241_F7;
  double K_1EM300;
  double K_ONE_M_1EM15;
  double K_1EM12;
  double K_1EM14;
  double K_1EM10;
  double K_1EM9;
  double K_1EM6;
  double K_ONE_M_1EM6;
  double K_ONE_P_1EM6;
  double K_0P999;
  double K_MIN_SUB;
  double K_0P425;
  double K_0P180625;
  double K_1P6;
  double K_0P85;
  double K_0P05;
  double K_ISPI;
  double K_M26P7;
  double K_M6P1;
  double K_TWO_M_TINY;
};

#if defined(__CUDACC__)
static __constant__ FvK fv_kc = {
    FV_DIV_SQRT2_C,
    FV_DIV_SQRT2_YH,
    FV_DIV_SQRT2_YL,
    FV_DIV_6_YH,
    FV_DIV_6_YL,
    FV_DIV_120_YH,
    FV_DIV_120_YL,
    FV_DIV_5040_YH,
    FV_DIV_5040_YL,
    FV_DIV_362880_YH,
    FV_DIV_362880_YL,
    FV_DIV_39916800_YH,
    FV_DIV_39916800_YL,
    FV_DIV_6227020800_YH,
    FV_DIV_6227020800_YL,
    FV_DIV_365_YH,
    FV_DIV_365_YL,
    FV_DIV_100_YH,
    FV_DIV_100_YL,
    FV_ERFC_ERX,
    FV_ERFC_ONE_M_ERX,
    FV_ERFC_PA0,
    FV_ERFC_PA1,
    FV_ERFC_PA2,
    FV_ERFC_PA3,
    FV_ERFC_PA4,
    FV_ERFC_PA5,
    FV_ERFC_PA6,
    FV_ERFC_PP0,
    FV_ERFC_PP1,
    FV_ERFC_PP2,
    FV_ERFC_PP3,
    FV_ERFC_PP4,
    FV_ERFC_QA1,
    FV_ERFC_QA2,
    FV_ERFC_QA3,
    FV_ERFC_QA4,
    FV_ERFC_QA5,
    FV_ERFC_QA6,
    FV_ERFC_QQ1,
    FV_ERFC_QQ2,
    FV_ERFC_QQ3,
    FV_ERFC_QQ4,
    FV_ERFC_QQ5,
    FV_ERFC_RA0,
    FV_ERFC_RA1,
    FV_ERFC_RA2,
    FV_ERFC_RA3,
    FV_ERFC_RA4,
    FV_ERFC_RA5,
    FV_ERFC_RA6,
    FV_ERFC_RA7,
    FV_ERFC_RB0,
    FV_ERFC_RB1,
    FV_ERFC_RB2,
    FV_ERFC_RB3,
    FV_ERFC_RB4,
    FV_ERFC_RB5,
    FV_ERFC_RB6,
    FV_ERFC_SA1,
    FV_ERFC_SA2,
    FV_ERFC_SA3,
    FV_ERFC_SA4,
    FV_ERFC_SA5,
    FV_ERFC_SA6,
    FV_ERFC_SA7,
    FV_ERFC_SA8,
    FV_ERFC_SB1,
    FV_ERFC_SB2,
    FV_ERFC_SB3,
    FV_ERFC_SB4,
    FV_ERFC_SB5,
    FV_ERFC_SB6,
    FV_ERFC_SB7,
    FV_EXP_C2,
    FV_EXP_C3,
    FV_EXP_C4,
    FV_EXP_C5,
    FV_EXP_INVLN2N,
    FV_EXP_NEGLN2HIN,
    FV_EXP_NEGLN2LON,
    FV_HALF_ONE_MINUS_EPS,
    FV_HALF_SQRT_TWO_PI,
    FV_INV_SQRT_TWO_PI,
    FV_LOG_A0,
    FV_LOG_A1,
    FV_LOG_A2,
    FV_LOG_A3,
    FV_LOG_A4,
    FV_LOG_B1,
    FV_LOG_B10,
    FV_LOG_B2,
    FV_LOG_B3,
    FV_LOG_B4,
    FV_LOG_B5,
    FV_LOG_B6,
    FV_LOG_B7,
    FV_LOG_B8,
    FV_LOG_B9,
    FV_LOG_INV_SQRT_TWO_PI,
    FV_LOG_LN2HI,
    FV_LOG_LN2LO,
    FV_POW_A1,
    FV_POW_A2,
    FV_POW_A3,
    FV_POW_A4,
    FV_POW_A5,
    FV_POW_A6,
    FV_POW_LN2HI,
    FV_POW_LN2LO,
    FV_SMALL_T_THRESHOLD,
    FV_SQRT_TWO,
    FV_TWO_PI,
    FV_AS241_A0,
    FV_AS241_A1,
    FV_AS241_A2,
    FV_AS241_A3,
    FV_AS241_A4,
    FV_AS241_A5,
    FV_AS241_A6,
    FV_AS241_A7,
    FV_AS241_B0,
    FV_AS241_B1,
    FV_AS241_B2,
    FV_AS241_B3,
    FV_AS241_B4,
    FV_AS241_B5,
    FV_AS241_B6,
    FV_AS241_B7,
    FV_AS241_C0,
    FV_AS241_C1,
    FV_AS241_C2,
    FV_AS241_C3,
    FV_AS241_C4,
    FV_AS241_C5,
    FV_AS241_C6,
    FV_AS241_C7,
    FV_AS241_D0,
    FV_AS241_D1,
    FV_AS241_D2,
    FV_AS241_D3,
    FV_AS241_D4,
    FV_AS241_D5,
    FV_AS241_D6,
    FV_AS241_D7,
    FV_AS241_E0,
    FV_AS241_E1,
    FV_AS241_E2,
    FV_AS241_E3,
    FV_AS241_E4,
    FV_AS241_E5,
    FV_AS241_E6,
    FV_AS241_E7,
    FV_AS241_F0,
    FV_AS241_F1,
    FV_AS241_F2,
    FV_AS241_F3,
    FV_AS241_F4,
    FV_AS241_F5,
    FV_AS241_F6,
    FV_AS241_F7,
    FV_K_1EM300,
    FV_K_ONE_M_1EM15,
    FV_K_1EM12,
    FV_K_1EM14,
    FV_K_1EM10,
    FV_K_1EM9,
    FV_K_1EM6,
    FV_K_ONE_M_1EM6,
    FV_K_ONE_P_1EM6,
    FV_K_0P999,
    FV_K_MIN_SUB,
    FV_K_0P425,
    FV_K_0P180625,
    FV_K_1P6,
    FV_K_0P85,
    FV_K_0P05,
    FV_K_ISPI,
    FV_K_M26P7,
    FV_K_M6P1,
    FV_K_TWO_M_TINY,
};
#endif

#if defined(__CUDA_ARCH__)
#undef FV_DIV_SQRT2_C
#define FV_DIV_SQRT2_C (fv_kc.DIV_SQRT2_C)
#undef FV_DIV_SQRT2_YH
#define FV_DIV_SQRT2_YH (fv_kc.DIV_SQRT2_YH)
#undef FV_DIV_SQRT2_YL
#define FV_DIV_SQRT2_YL (fv_kc.DIV_SQRT2_YL)
#undef FV_DIV_6_YH
#define FV_DIV_6_YH (fv_kc.DIV_6_YH)
#undef FV_DIV_6_YL
#define FV_DIV_6_YL (fv_kc.DIV_6_YL)
#undef FV_DIV_120_YH
#define FV_DIV_120_YH (fv_kc.DIV_120_YH)
#undef FV_DIV_120_YL
#define FV_DIV_120_YL (fv_kc.DIV_120_YL)
#undef FV_DIV_5040_YH
#define FV_DIV_5040_YH (fv_kc.DIV_5040_YH)
#undef FV_DIV_5040_YL
#define FV_DIV_5040_YL (fv_kc.DIV_5040_YL)
#undef FV_DIV_362880_YH
#define FV_DIV_362880_YH (fv_kc.DIV_362880_YH)
#undef FV_DIV_362880_YL
#define FV_DIV_362880_YL (fv_kc.DIV_362880_YL)
#undef FV_DIV_39916800_YH
#define FV_DIV_39916800_YH (fv_kc.DIV_39916800_YH)
#undef FV_DIV_39916800_YL
#define FV_DIV_39916800_YL (fv_kc.DIV_39916800_YL)
#undef FV_DIV_6227020800_YH
#define FV_DIV_6227020800_YH (fv_kc.DIV_6227020800_YH)
#undef FV_DIV_6227020800_YL
#define FV_DIV_6227020800_YL (fv_kc.DIV_6227020800_YL)
#undef FV_DIV_365_YH
#define FV_DIV_365_YH (fv_kc.DIV_365_YH)
#undef FV_DIV_365_YL
#define FV_DIV_365_YL (fv_kc.DIV_365_YL)
#undef FV_DIV_100_YH
#define FV_DIV_100_YH (fv_kc.DIV_100_YH)
#undef FV_DIV_100_YL
#define FV_DIV_100_YL (fv_kc.DIV_100_YL)
#undef FV_ERFC_ERX
#define FV_ERFC_ERX (fv_kc.ERFC_ERX)
#undef FV_ERFC_ONE_M_ERX
#define FV_ERFC_ONE_M_ERX (fv_kc.ERFC_ONE_M_ERX)
#undef FV_ERFC_PA0
#define FV_ERFC_PA0 (fv_kc.ERFC_PA0)
#undef FV_ERFC_PA1
#define FV_ERFC_PA1 (fv_kc.ERFC_PA1)
#undef FV_ERFC_PA2
#define FV_ERFC_PA2 (fv_kc.ERFC_PA2)
#undef FV_ERFC_PA3
#define FV_ERFC_PA3 (fv_kc.ERFC_PA3)
#undef FV_ERFC_PA4
#define FV_ERFC_PA4 (fv_kc.ERFC_PA4)
#undef FV_ERFC_PA5
#define FV_ERFC_PA5 (fv_kc.ERFC_PA5)
#undef FV_ERFC_PA6
#define FV_ERFC_PA6 (fv_kc.ERFC_PA6)
#undef FV_ERFC_PP0
#define FV_ERFC_PP0 (fv_kc.ERFC_PP0)
#undef FV_ERFC_PP1
#define FV_ERFC_PP1 (fv_kc.ERFC_PP1)
#undef FV_ERFC_PP2
#define FV_ERFC_PP2 (fv_kc.ERFC_PP2)
#undef FV_ERFC_PP3
#define FV_ERFC_PP3 (fv_kc.ERFC_PP3)
#undef FV_ERFC_PP4
#define FV_ERFC_PP4 (fv_kc.ERFC_PP4)
#undef FV_ERFC_QA1
#define FV_ERFC_QA1 (fv_kc.ERFC_QA1)
#undef FV_ERFC_QA2
#define FV_ERFC_QA2 (fv_kc.ERFC_QA2)
#undef FV_ERFC_QA3
#define FV_ERFC_QA3 (fv_kc.ERFC_QA3)
#undef FV_ERFC_QA4
#define FV_ERFC_QA4 (fv_kc.ERFC_QA4)
#undef FV_ERFC_QA5
#define FV_ERFC_QA5 (fv_kc.ERFC_QA5)
#undef FV_ERFC_QA6
#define FV_ERFC_QA6 (fv_kc.ERFC_QA6)
#undef FV_ERFC_QQ1
#define FV_ERFC_QQ1 (fv_kc.ERFC_QQ1)
#undef FV_ERFC_QQ2
#define FV_ERFC_QQ2 (fv_kc.ERFC_QQ2)
#undef FV_ERFC_QQ3
#define FV_ERFC_QQ3 (fv_kc.ERFC_QQ3)
#undef FV_ERFC_QQ4
#define FV_ERFC_QQ4 (fv_kc.ERFC_QQ4)
#undef FV_ERFC_QQ5
#define FV_ERFC_QQ5 (fv_kc.ERFC_QQ5)
#undef FV_ERFC_RA0
#define FV_ERFC_RA0 (fv_kc.ERFC_RA0)
#undef FV_ERFC_RA1
#define FV_ERFC_RA1 (fv_kc.ERFC_RA1)
#undef FV_ERFC_RA2
#define FV_ERFC_RA2 (fv_kc.ERFC_RA2)
#undef FV_ERFC_RA3
#define FV_ERFC_RA3 (fv_kc.ERFC_RA3)
#undef FV_ERFC_RA4
#define FV_ERFC_RA4 (fv_kc.ERFC_RA4)
#undef FV_ERFC_RA5
#define FV_ERFC_RA5 (fv_kc.ERFC_RA5)
#undef FV_ERFC_RA6
#define FV_ERFC_RA6 (fv_kc.ERFC_RA6)
#undef FV_ERFC_RA7
#define FV_ERFC_RA7 (fv_kc.ERFC_RA7)
#undef FV_ERFC_RB0
#define FV_ERFC_RB0 (fv_kc.ERFC_RB0)
#undef FV_ERFC_RB1
#define FV_ERFC_RB1 (fv_kc.ERFC_RB1)
#undef FV_ERFC_RB2
#define FV_ERFC_RB2 (fv_kc.ERFC_RB2)
#undef FV_ERFC_RB3
#define FV_ERFC_RB3 (fv_kc.ERFC_RB3)
#undef FV_ERFC_RB4
#define FV_ERFC_RB4 (fv_kc.ERFC_RB4)
#undef FV_ERFC_RB5
#define FV_ERFC_RB5 (fv_kc.ERFC_RB5)
#undef FV_ERFC_RB6
#define FV_ERFC_RB6 (fv_kc.ERFC_RB6)
#undef FV_ERFC_SA1
#define FV_ERFC_SA1 (fv_kc.ERFC_SA1)
#undef FV_ERFC_SA2
#define FV_ERFC_SA2 (fv_kc.ERFC_SA2)
#undef FV_ERFC_SA3
#define FV_ERFC_SA3 (fv_kc.ERFC_SA3)
#undef FV_ERFC_SA4
#define FV_ERFC_SA4 (fv_kc.ERFC_SA4)
#undef FV_ERFC_SA5
#define FV_ERFC_SA5 (fv_kc.ERFC_SA5)
#undef FV_ERFC_SA6
#define FV_ERFC_SA6 (fv_kc.ERFC_SA6)
#undef FV_ERFC_SA7
#define FV_ERFC_SA7 (fv_kc.ERFC_SA7)
#undef FV_ERFC_SA8
#define FV_ERFC_SA8 (fv_kc.ERFC_SA8)
#undef FV_ERFC_SB1
#define FV_ERFC_SB1 (fv_kc.ERFC_SB1)
#undef FV_ERFC_SB2
#define FV_ERFC_SB2 (fv_kc.ERFC_SB2)
#undef FV_ERFC_SB3
#define FV_ERFC_SB3 (fv_kc.ERFC_SB3)
#undef FV_ERFC_SB4
#define FV_ERFC_SB4 (fv_kc.ERFC_SB4)
#undef FV_ERFC_SB5
#define FV_ERFC_SB5 (fv_kc.ERFC_SB5)
#undef FV_ERFC_SB6
#define FV_ERFC_SB6 (fv_kc.ERFC_SB6)
#undef FV_ERFC_SB7
#define FV_ERFC_SB7 (fv_kc.ERFC_SB7)
#undef FV_EXP_C2
#define FV_EXP_C2 (fv_kc.EXP_C2)
#undef FV_EXP_C3
#define FV_EXP_C3 (fv_kc.EXP_C3)
#undef FV_EXP_C4
#define FV_EXP_C4 (fv_kc.EXP_C4)
#undef FV_EXP_C5
#define FV_EXP_C5 (fv_kc.EXP_C5)
#undef FV_EXP_INVLN2N
#define FV_EXP_INVLN2N (fv_kc.EXP_INVLN2N)
#undef FV_EXP_NEGLN2HIN
#define FV_EXP_NEGLN2HIN (fv_kc.EXP_NEGLN2HIN)
#undef FV_EXP_NEGLN2LON
#define FV_EXP_NEGLN2LON (fv_kc.EXP_NEGLN2LON)
#undef FV_HALF_ONE_MINUS_EPS
#define FV_HALF_ONE_MINUS_EPS (fv_kc.HALF_ONE_MINUS_EPS)
#undef FV_HALF_SQRT_TWO_PI
#define FV_HALF_SQRT_TWO_PI (fv_kc.HALF_SQRT_TWO_PI)
#undef FV_INV_SQRT_TWO_PI
#define FV_INV_SQRT_TWO_PI (fv_kc.INV_SQRT_TWO_PI)
#undef FV_LOG_A0
#define FV_LOG_A0 (fv_kc.LOG_A0)
#undef FV_LOG_A1
#define FV_LOG_A1 (fv_kc.LOG_A1)
#undef FV_LOG_A2
#define FV_LOG_A2 (fv_kc.LOG_A2)
#undef FV_LOG_A3
#define FV_LOG_A3 (fv_kc.LOG_A3)
#undef FV_LOG_A4
#define FV_LOG_A4 (fv_kc.LOG_A4)
#undef FV_LOG_B1
#define FV_LOG_B1 (fv_kc.LOG_B1)
#undef FV_LOG_B10
#define FV_LOG_B10 (fv_kc.LOG_B10)
#undef FV_LOG_B2
#define FV_LOG_B2 (fv_kc.LOG_B2)
#undef FV_LOG_B3
#define FV_LOG_B3 (fv_kc.LOG_B3)
#undef FV_LOG_B4
#define FV_LOG_B4 (fv_kc.LOG_B4)
#undef FV_LOG_B5
#define FV_LOG_B5 (fv_kc.LOG_B5)
#undef FV_LOG_B6
#define FV_LOG_B6 (fv_kc.LOG_B6)
#undef FV_LOG_B7
#define FV_LOG_B7 (fv_kc.LOG_B7)
#undef FV_LOG_B8
#define FV_LOG_B8 (fv_kc.LOG_B8)
#undef FV_LOG_B9
#define FV_LOG_B9 (fv_kc.LOG_B9)
#undef FV_LOG_INV_SQRT_TWO_PI
#define FV_LOG_INV_SQRT_TWO_PI (fv_kc.LOG_INV_SQRT_TWO_PI)
#undef FV_LOG_LN2HI
#define FV_LOG_LN2HI (fv_kc.LOG_LN2HI)
#undef FV_LOG_LN2LO
#define FV_LOG_LN2LO (fv_kc.LOG_LN2LO)
#undef FV_POW_A1
#define FV_POW_A1 (fv_kc.POW_A1)
#undef FV_POW_A2
#define FV_POW_A2 (fv_kc.POW_A2)
#undef FV_POW_A3
#define FV_POW_A3 (fv_kc.POW_A3)
#undef FV_POW_A4
#define FV_POW_A4 (fv_kc.POW_A4)
#undef FV_POW_A5
#define FV_POW_A5 (fv_kc.POW_A5)
#undef FV_POW_A6
#define FV_POW_A6 (fv_kc.POW_A6)
#undef FV_POW_LN2HI
#define FV_POW_LN2HI (fv_kc.POW_LN2HI)
#undef FV_POW_LN2LO
#define FV_POW_LN2LO (fv_kc.POW_LN2LO)
#undef FV_SMALL_T_THRESHOLD
#define FV_SMALL_T_THRESHOLD (fv_kc.SMALL_T_THRESHOLD)
#undef FV_SQRT_TWO
#define FV_SQRT_TWO (fv_kc.SQRT_TWO)
#undef FV_TWO_PI
#define FV_TWO_PI (fv_kc.TWO_PI)
#undef FV_AS241_A0
#define FV_AS241_A0 (fv_kc.AS241_A0)
#undef FV_AS241_A1
#define FV_AS241_A1 (fv_kc.AS241_A1)
#undef FV_AS241_A2
#define FV_AS241_A2 (fv_kc.AS241_A2)
#undef FV_AS241_A3
#define FV_AS241_A3 (fv_kc.AS241_A3)
#undef FV_AS241_A4
#define FV_AS241_A4 (fv_kc.AS241_A4)
#undef FV_AS241_A5
#define FV_AS241_A5 (fv_kc.AS241_A5)
#undef FV_AS241_A6
#define FV_AS241_A6 (fv_kc.AS241_A6)
#undef FV_AS241_A7
#define FV_AS241_A7 (fv_kc.AS241_A7)
#undef FV_AS241_B0
#define FV_AS241_B0 (fv_kc.AS241_B0)
#undef FV_AS241_B1
#define FV_AS241_B1 (fv_kc.AS241_B1)
#undef FV_AS241_B2
#define FV_AS241_B2 (fv_kc.AS241_B2)
#undef FV_AS241_B3
#define FV_AS241_B3 (fv_kc.AS241_B3)
#undef FV_AS241_B4
#define FV_AS241_B4 (fv_kc.AS241_B4)
#undef FV_AS241_B5
#define FV_AS241_B5 (fv_kc.AS241_B5)
#undef FV_AS241_B6
#define FV_AS241_B6 (fv_kc.AS241_B6)
#undef FV_AS241_B7
#define FV_AS241_B7 (fv_kc.AS241_B7)
#undef FV_AS241_C0
#define FV_AS241_C0 (fv_kc.AS241_C0)
#undef FV_AS241_C1
#define FV_AS241_C1 (fv_kc.AS241_C1)
#undef FV_AS241_C2
#define FV_AS241_C2 (fv_kc.AS241_C2)
#undef FV_AS241_C3
#define FV_AS241_C3 (fv_kc.AS241_C3)
#undef FV_AS241_C4
#define FV_AS241_C4 (fv_kc.AS241_C4)
#undef FV_AS241_C5
#define FV_AS241_C5 (fv_kc.AS241_C5)
#undef FV_AS241_C6
#define FV_AS241_C6 (fv_kc.AS241_C6)
#undef FV_AS241_C7
#define FV_AS241_C7 (fv_kc.AS241_C7)
#undef FV_AS241_D0
#define FV_AS241_D0 (fv_kc.AS241_D0)
#undef FV_AS241_D1
#define FV_AS241_D1 (fv_kc.AS241_D1)
#undef FV_AS241_D2
#define FV_AS241_D2 (fv_kc.AS241_D2)
#undef FV_AS241_D3
#define FV_AS241_D3 (fv_kc.AS241_D3)
#undef FV_AS241_D4
#define FV_AS241_D4 (fv_kc.AS241_D4)
#undef FV_AS241_D5
#define FV_AS241_D5 (fv_kc.AS241_D5)
#undef FV_AS241_D6
#define FV_AS241_D6 (fv_kc.AS241_D6)
#undef FV_AS241_D7
#define FV_AS241_D7 (fv_kc.AS241_D7)
#undef FV_AS241_E0
#define FV_AS241_E0 (fv_kc.AS241_E0)
#undef FV_AS241_E1
#define FV_AS241_E1 (fv_kc.AS241_E1)
#undef FV_AS241_E2
#define FV_AS241_E2 (fv_kc.AS241_E2)
#undef FV_AS241_E3
#define FV_AS241_E3 (fv_kc.AS241_E3)
#undef FV_AS241_E4
#define FV_AS241_E4 (fv_kc.AS241_E4)
#undef FV_AS241_E5
#define FV_AS241_E5 (fv_kc.AS241_E5)
#undef FV_AS241_E6
#define FV_AS241_E6 (fv_kc.AS241_E6)
#undef FV_AS241_E7
#define FV_AS241_E7 (fv_kc.AS241_E7)
#undef FV_AS241_F0
#define FV_AS241_F0 (fv_kc.AS241_F0)
#undef FV_AS241_F1
#define FV_AS241_F1 (fv_kc.AS241_F1)
#undef FV_AS241_F2
#define FV_AS241_F2 (fv_kc.AS241_F2)
#undef FV_AS241_F3
#define FV_AS241_F3 (fv_kc.AS241_F3)
#undef FV_AS241_F4
#define FV_AS241_F4 (fv_kc.AS241_F4)
#undef FV_AS241_F5
#define FV_AS241_F5 (fv_kc.AS241_F5)
#undef FV_AS241_F6
#define FV_AS241_F6 (fv_kc.AS241_F6)
#undef FV_AS241_F7
#define FV_AS241_F7 (fv_kc.AS241_F7)
#undef FV_K_1EM300
#define FV_K_1EM300 (fv_kc.K_1EM300)
#undef FV_K_ONE_M_1EM15
#define FV_K_ONE_M_1EM15 (fv_kc.K_ONE_M_1EM15)
#undef FV_K_1EM12
#define FV_K_1EM12 (fv_kc.K_1EM12)
#undef FV_K_1EM14
#define FV_K_1EM14 (fv_kc.K_1EM14)
#undef FV_K_1EM10
#define FV_K_1EM10 (fv_kc.K_1EM10)
#undef FV_K_1EM9
#define FV_K_1EM9 (fv_kc.K_1EM9)
#undef FV_K_1EM6
#define FV_K_1EM6 (fv_kc.K_1EM6)
#undef FV_K_ONE_M_1EM6
#define FV_K_ONE_M_1EM6 (fv_kc.K_ONE_M_1EM6)
#undef FV_K_ONE_P_1EM6
#define FV_K_ONE_P_1EM6 (fv_kc.K_ONE_P_1EM6)
#undef FV_K_0P999
#define FV_K_0P999 (fv_kc.K_0P999)
#undef FV_K_MIN_SUB
#define FV_K_MIN_SUB (fv_kc.K_MIN_SUB)
#undef FV_K_0P425
#define FV_K_0P425 (fv_kc.K_0P425)
#undef FV_K_0P180625
#define FV_K_0P180625 (fv_kc.K_0P180625)
#undef FV_K_1P6
#define FV_K_1P6 (fv_kc.K_1P6)
#undef FV_K_0P85
#define FV_K_0P85 (fv_kc.K_0P85)
#undef FV_K_0P05
#define FV_K_0P05 (fv_kc.K_0P05)
#undef FV_K_ISPI
#define FV_K_ISPI (fv_kc.K_ISPI)
#undef FV_K_M26P7
#define FV_K_M26P7 (fv_kc.K_M26P7)
#undef FV_K_M6P1
#define FV_K_M6P1 (fv_kc.K_M6P1)
#undef FV_K_TWO_M_TINY
#define FV_K_TWO_M_TINY (fv_kc.K_TWO_M_TINY)
#endif
