#!/usr/bin/env python3
"""Generate ``paper_2604_27210_b200/csrc/fv_tables.h``: every numeric constant
the device restatement of the reference's arithmetic needs, emitted as exact
hex-float / hex-integer literals so nothing is retyped by hand.

Sources (all third-party numeric data or the reference's own computed module
constants -- no code is copied):

* glibc 2.39 libm (``/lib/x86_64-linux-gnu/libm-2.39.a``): the data objects
  ``__exp_data``, ``__log_data``, ``__pow_log_data`` (table-driven exp/log/pow
  of the ARM optimized-routines family that CPython's ``math.exp``,
  ``math.log`` and ``float.__pow__`` resolve to) and the fdlibm ``erfc``
  coefficients from ``s_erf.o``'s constant pool.
* scipy 1.18.1 ``scipy.special.erfcx`` = S. G. Johnson's Faddeeva ``erfcx``:
  the 100x7 Chebyshev table of ``erfcx_y100``, read from the bit-identical
  copy shipped in torch's ``ATen/native/Math.h`` (erfcx_y100).
* the reference's module-level constants, read from the imported modules:
  ``fastvol.lbr`` (_ASYM_FACTS, _ASYM_PASCAL, SMALL_T_THRESHOLD, ...) and
  ``fastvol.distributions`` (AS241 _A.._F, SQRT_TWO, INV_SQRT_TWO_PI).

Run here (needs /root/reference, libm-2.39.a and torch headers); the output is
committed and the GPU box only compiles it.
"""

import os
import re
import struct
import subprocess
import sys
import tempfile

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(REPO, "paper_2604_27210_b200", "csrc", "fv_tables.h")
LIBM_A = "/lib/x86_64-linux-gnu/libm-2.39.a"
REF_SRC = "/root/reference/pkg/src"


def torch_math_h():
    import torch  # noqa: F401  (only to locate the header tree)
    return os.path.join(os.path.dirname(torch.__file__), "include", "ATen",
                        "native", "Math.h")


def _section(obj, name):
    with tempfile.NamedTemporaryFile(suffix=".bin") as f:
        subprocess.run(["objcopy", "-O", "binary", "--only-section=" + name,
                        obj, f.name], check=True)
        return open(f.name, "rb").read()


def libm_objects(tmp):
    names = ["e_exp_data.o", "e_log_data.o", "e_pow_log_data.o", "s_erf.o"]
    subprocess.run(["ar", "x", LIBM_A] + names, cwd=tmp, check=True)
    return {n: os.path.join(tmp, n) for n in names}


def lc_constants(obj):
    """Map .LCn label -> double for an object's mergeable constant pools."""
    secs = {}
    out = subprocess.run(["readelf", "-S", "-W", obj], capture_output=True,
                         text=True, check=True).stdout
    for m in re.finditer(r"\[\s*(\d+)\]\s+(\.rodata\.cst(?:8|16))", out):
        secs[int(m.group(1))] = _section(obj, m.group(2))
    syms = subprocess.run(["readelf", "-s", "-W", obj], capture_output=True,
                          text=True, check=True).stdout
    vals = {}
    for m in re.finditer(r"([0-9a-f]{16})\s+0 NOTYPE\s+LOCAL\s+DEFAULT\s+(\d+)"
                         r" (\.LC\d+)", syms):
        off, sec, name = int(m.group(1), 16), int(m.group(2)), m.group(3)
        if sec in secs:
            vals[name] = struct.unpack_from("<d", secs[sec], off)[0]
    return vals


def hexd(v):
    if v != v:
        return "__builtin_nan(\"\")"
    if v == 0.0:
        return "-0.0" if struct.pack("<d", v)[7] & 0x80 else "0.0"
    return float.hex(v)


def u64(v):
    return "0x%016xull" % v


def emit_array(lines, ctype, name, values, fmt, per_line=4):
    lines.append("FV_TABLE(%s, %s, %d) = {" % (ctype, name, len(values)))
    for i in range(0, len(values), per_line):
        lines.append("    " + ", ".join(fmt(v) for v in values[i:i + per_line]) + ",")
    lines.append("};")


# fdlibm erfc coefficient name -> (.LC label in glibc 2.39 s_erf.o, sign).
# glibc's compiler folded ``c + x`` with a negative c into ``x - |c|``, so a few
# pool entries hold the negated coefficient (sign -1).  Approximate values are
# checked below so a different libm build fails loudly instead of silently.
ERFC_MAP = {
    "pp0": (".LC10", +1, 1.28379167095512558561e-01),
    "pp1": (".LC9", +1, -3.25042107247001499370e-01),
    "pp2": (".LC8", -1, -2.84817495755985104766e-02),
    "pp3": (".LC7", +1, -5.77027029648944159157e-03),
    "pp4": (".LC11", +1, -2.37630166566501626084e-05),
    "qq1": (".LC14", +1, 3.97917223959155352819e-01),
    "qq2": (".LC13", +1, 6.50222499887672944485e-02),
    "qq3": (".LC12", +1, 5.08130628187576562776e-03),
    "qq4": (".LC16", +1, 1.32494738004321644526e-04),
    "qq5": (".LC15", +1, -3.96022827877536812320e-06),
    "erx": (".LC30", +1, 8.45062911510467529297e-01),
    "pa0": (".LC20", -1, -2.36211856075265944077e-03),
    "pa1": (".LC19", +1, 4.14856118683748331666e-01),
    "pa2": (".LC18", -1, -3.72207876035701323847e-01),
    "pa3": (".LC17", +1, 3.18346619901161753674e-01),
    "pa4": (".LC22", -1, -1.10894694282396677476e-01),
    "pa5": (".LC21", +1, 3.54783043256182359371e-02),
    "pa6": (".LC23", +1, -2.16637559486879084300e-03),
    "qa1": (".LC26", +1, 1.06420880400844228286e-01),
    "qa2": (".LC25", +1, 5.40397917702171048937e-01),
    "qa3": (".LC24", +1, 7.18286544141962662868e-02),
    "qa4": (".LC28", +1, 1.26171219808761642112e-01),
    "qa5": (".LC27", +1, 1.36370839120290507362e-02),
    "qa6": (".LC29", +1, 1.19844998467991074170e-02),
    "ra0": (".LC36", -1, -9.86494403484714822705e-03),
    "ra1": (".LC35", +1, -6.93858572707181764372e-01),
    "ra2": (".LC34", -1, -1.05586262253232909814e+01),
    "ra3": (".LC33", +1, -6.23753324503260060396e+01),
    "ra4": (".LC38", -1, -1.62396669462573470355e+02),
    "ra5": (".LC37", +1, -1.84605092906711035994e+02),
    "ra6": (".LC40", -1, -8.12874355063065934246e+01),
    "ra7": (".LC39", +1, -9.81432934416914548592e+00),
    "sa1": (".LC43", +1, 1.96512716674392571292e+01),
    "sa2": (".LC42", +1, 1.37657754143519042600e+02),
    "sa3": (".LC41", +1, 4.34565877475229228821e+02),
    "sa4": (".LC45", +1, 6.45387271733267880336e+02),
    "sa5": (".LC44", +1, 4.29008140027567833386e+02),
    "sa6": (".LC47", +1, 1.08635005541779435134e+02),
    "sa7": (".LC46", +1, 6.57024977031928170135e+00),
    "sa8": (".LC48", +1, -6.04244152148580987438e-02),
    "rb0": (".LC52", -1, -9.86494292470009928597e-03),
    "rb1": (".LC51", +1, -7.99283237680523006574e-01),
    "rb2": (".LC50", -1, -1.77579549177547519889e+01),
    "rb3": (".LC49", +1, -1.60636384855821916062e+02),
    "rb4": (".LC54", -1, -6.37566443368389627722e+02),
    "rb5": (".LC53", +1, -1.02509513161107724954e+03),
    "rb6": (".LC55", +1, -4.83519191608651397019e+02),
    "sb1": (".LC58", +1, 3.03380607434824582924e+01),
    "sb2": (".LC57", +1, 3.25792512996573918826e+02),
    "sb3": (".LC56", +1, 1.53672958608443695994e+03),
    "sb4": (".LC60", +1, 3.19985821950859553908e+03),
    "sb5": (".LC59", +1, 2.55305040643316442583e+03),
    "sb6": (".LC62", +1, 4.74528541206955367215e+02),
    "sb7": (".LC61", +1, -2.24409524465858183362e+01),
    "one_m_erx": (".LC66", +1, 1.54937088489532470703e-01),
}


def erfcx_table(path):
    src = open(path).read()
    start = src.index("erfcx_y100(T y100)")
    end = src.index("calc_erfcx(T x)", start)
    body = src[start:end]
    rows = []
    for m in re.finditer(r"case (\d+): \{\s*T t = 2\*y100 - (\d+);\s*return ([^;]+);",
                         body):
        k, off, expr = int(m.group(1)), int(m.group(2)), m.group(3)
        assert off == 2 * k + 1, (k, off)
        nums = re.findall(r"[0-9]\.[0-9]+e[-+]?[0-9]+", expr)
        assert len(nums) == 7, (k, nums)
        rows.append((k, [float(n) for n in nums]))
    assert [k for k, _ in rows] == list(range(100))
    return [c for _, cs in rows for c in cs]


def main():
    sys.dont_write_bytecode = True
    sys.path.insert(0, REF_SRC)
    import fastvol.distributions as D
    import fastvol.lbr as L

    lines = [
        "// GENERATED by tools/gen_tables.py -- do not edit.",
        "// Exact constants for the bit-faithful device restatement of the",
        "// reference's arithmetic (glibc 2.39 libm data, scipy/Faddeeva erfcx",
        "// Chebyshev table, fastvol module constants).  See tools/gen_tables.py.",
        "// No include guard: fv_libm.h includes it once per table flavour (host",
        "// static arrays, device globals) with its own FV_TABLE definition.",
        "#include <stdint.h>",
        "#ifndef FV_TABLE_DEFINED_BY_INCLUDER",
        "#error \"define FV_TABLE(type, name, n) before including fv_tables.h\"",
        "#endif",
        "",
    ]
    with tempfile.TemporaryDirectory() as tmp:
        objs = libm_objects(tmp)
        exp_b = _section(objs["e_exp_data.o"], ".rodata")
        log_b = _section(objs["e_log_data.o"], ".rodata")
        pow_b = _section(objs["e_pow_log_data.o"], ".rodata")
        erf_lc = lc_constants(objs["s_erf.o"])

    # ---- glibc exp: struct exp_data (math_config.h, glibc 2.39) ------------
    assert len(exp_b) == 0x8b0
    hd = struct.unpack_from("<22d", exp_b, 0)
    names = ["INVLN2N", "SHIFT", "NEGLN2HIN", "NEGLN2LON", "C2", "C3", "C4", "C5"]
    lines.append("// glibc 2.39 __exp_data header (EXP_TABLE_BITS=7, EXP_POLY_ORDER=5)")
    for i, n in enumerate(names):
        lines.append("#define FV_EXP_%s %s" % (n, hexd(hd[i])))
    tab = struct.unpack_from("<256Q", exp_b, 22 * 8)
    lines.append("// __exp_data.tab: tab[2k] = asuint64(tail_k), tab[2k+1] = asuint64(2^(k/128)) - (k << 45)")
    emit_array(lines, "uint64_t", "fv_exp_tab", tab, u64)
    lines.append("")

    # ---- glibc log: struct log_data ----------------------------------------
    assert len(log_b) == 0x1090
    hd = struct.unpack_from("<18d", log_b, 0)
    lines.append("// glibc 2.39 __log_data (LOG_TABLE_BITS=7, LOG_POLY_ORDER=6, LOG_POLY1_ORDER=12)")
    lines.append("#define FV_LOG_LN2HI %s" % hexd(hd[0]))
    lines.append("#define FV_LOG_LN2LO %s" % hexd(hd[1]))
    for i in range(5):
        lines.append("#define FV_LOG_A%d %s" % (i, hexd(hd[2 + i])))
    for i in range(11):
        lines.append("#define FV_LOG_B%d %s" % (i, hexd(hd[7 + i])))
    tab = struct.unpack_from("<256d", log_b, 18 * 8)
    lines.append("// __log_data.tab: {invc, logc} x 128")
    emit_array(lines, "double", "fv_log_tab", tab, hexd)
    lines.append("")

    # ---- glibc pow: struct pow_log_data ------------------------------------
    assert len(pow_b) == 0x1048
    hd = struct.unpack_from("<9d", pow_b, 0)
    lines.append("// glibc 2.39 __pow_log_data (POW_LOG_TABLE_BITS=7, POW_LOG_POLY_ORDER=8)")
    lines.append("#define FV_POW_LN2HI %s" % hexd(hd[0]))
    lines.append("#define FV_POW_LN2LO %s" % hexd(hd[1]))
    for i in range(7):
        lines.append("#define FV_POW_A%d %s" % (i, hexd(hd[2 + i])))
    tab = struct.unpack_from("<512d", pow_b, 9 * 8)
    # keep {invc, logc, logctail} (drop the pad) -> 3 doubles per entry
    tab3 = []
    for i in range(128):
        tab3 += [tab[4 * i], tab[4 * i + 2], tab[4 * i + 3]]
    lines.append("// __pow_log_data.tab: {invc, logc, logctail} x 128")
    emit_array(lines, "double", "fv_powlog_tab", tab3, hexd, per_line=3)
    lines.append("")

    # ---- fdlibm erfc (glibc s_erf.c) ---------------------------------------
    lines.append("// fdlibm erfc coefficients as compiled into glibc 2.39 s_erf.o")
    for name, (lc, sign, approx) in ERFC_MAP.items():
        v = sign * erf_lc[lc]
        assert abs(v - approx) <= 1e-15 * abs(approx), (name, v, approx)
        lines.append("#define FV_ERFC_%s %s" % (name.upper(), hexd(v)))
    lines.append("")

    # erfc tail ranges [1.25, 1/0.35) and [1/0.35, 28) as one table so the
    # kernel evaluates one shared code path (no lane divergence between the
    # two): row 0 = ra0..ra7, sa1..sa8 ; row 1 = rb0..rb6, 0, sb1..sb7, 0.
    # The zero entries turn the missing terms into exact +0 additions.
    ev = {name: sign * erf_lc[lc] for name, (lc, sign, approx) in ERFC_MAP.items()}
    tail = ([ev["ra%d" % i] for i in range(8)] + [ev["sa%d" % i] for i in range(1, 9)]
            + [ev["rb%d" % i] for i in range(7)] + [0.0] + [ev["sb%d" % i] for i in range(1, 8)] + [0.0])
    lines.append("// fdlibm erfc tail coefficients, two rows of 16 (see tools/gen_tables.py)")
    emit_array(lines, "double", "fv_erfc_tail", tail, hexd)
    lines.append("")

    # erfc inner ranges |x| < 0.84375 (pp/qq in u = x^2) and [0.84375, 1.25)
    # (pa/qa in u = |x| - 1) as one rational form
    # ((n0 + u n1) + u^2 (n2 + u n3) + u^4 (n4 + u n5)) + u^6 n6 over
    # ((1 + u d1) + u^2 (d2 + u d3) + u^4 (d4 + u d5)) + u^6 d6, rows of 16:
    # n0..n6, d1..d6, pad.  Zero entries are exact +0 additions.
    mid = ([ev["pp%d" % i] for i in range(5)] + [0.0, 0.0] + [ev["qq%d" % i] for i in range(1, 6)] + [0.0]
           + [0.0, 0.0, 0.0]
           + [ev["pa%d" % i] for i in range(7)] + [ev["qa%d" % i] for i in range(1, 7)] + [0.0, 0.0, 0.0])
    assert len(mid) == 32
    lines.append("// fdlibm erfc inner-range coefficients, two rows of 16 (see tools/gen_tables.py)")
    emit_array(lines, "double", "fv_erfc_mid", mid, hexd)
    lines.append("")

    # all four erfc rational ranges in the tail's form, rows of 16:
    # P = ((c0 + s c1) + s^2 (c2 + s c3) + s^4 (c4 + s c5)) + s^6 (c6 + s c7),
    # Q = (((1 + s d1) + s^2 (d2 + s d3) + s^4 (d4 + s d5)) + s^6 (d6 + s d7)) + s^8 d8;
    # rows: |x| < 0.84375, [0.84375, 1.25), [1.25, 1/0.35), [1/0.35, 28).  The
    # inner rows' c7 = d7 = d8 = 0 add exact zeros (fx_erfc_u, fv_fast.h).
    uni = (mid[0:7] + [0.0] + mid[7:13] + [0.0, 0.0]
           + mid[16:23] + [0.0] + mid[23:29] + [0.0, 0.0] + tail)
    assert len(uni) == 64
    lines.append("// fdlibm erfc rationals of all four ranges in one form, rows of 16 (see tools/gen_tables.py)")
    emit_array(lines, "double", "fv_erfc_uni", uni, hexd)
    lines.append("")

    # ---- Faddeeva erfcx_y100 Chebyshev table -------------------------------
    cheb = erfcx_table(torch_math_h())
    lines.append("// Faddeeva erfcx_y100: 100 intervals x 7 coefficients (c0..c6),")
    lines.append("// t = 2*y100 - (2k+1), value = c0 + (c1 + (... + c6*t)*t)*t")
    emit_array(lines, "double", "fv_erfcx_tab", cheb, hexd, per_line=7)
    lines.append("")
    # the same rows padded to 8 (64-byte rows): four 16-byte loads per lookup
    cheb8 = []
    for k in range(100):
        cheb8 += list(cheb[7 * k:7 * k + 7]) + [0.0]
    lines.append("// fv_erfcx_tab padded to 8 per row (c0..c6, 0) for 16-byte loads")
    emit_array(lines, "double", "fv_erfcx_tab8", cheb8, hexd, per_line=8)
    lines.append("")

    # ---- fastvol constants --------------------------------------------------
    import math
    lines.append("// fastvol module constants (values read from the imported reference)")
    consts = {
        "SQRT_TWO": D.SQRT_TWO,                              # distributions.py:14
        "INV_SQRT_TWO_PI": D.INV_SQRT_TWO_PI,                # distributions.py:16
        "LOG_INV_SQRT_TWO_PI": math.log(D.INV_SQRT_TWO_PI),  # lbr.py:297, :366
        "HALF_SQRT_TWO_PI": 0.5 * math.sqrt(2.0 * math.pi),  # lbr.py:77
        "TWO_PI": 2.0 * math.pi,                             # solver.py:105
        "DBL_EPSILON": L.DBL_EPSILON,                        # lbr.py:37
        "SMALL_T_THRESHOLD": L.SMALL_T_THRESHOLD,            # lbr.py:40
        "HALF_ONE_MINUS_EPS": 0.5 * (1.0 - L.DBL_EPSILON),   # lbr.py:316
    }
    for k, v in consts.items():
        lines.append("#define FV_%s %s" % (k, hexd(v)))
    for nm in "ABCDEF":
        co = getattr(D, "_" + nm)
        assert len(co) == 8
        for i, v in enumerate(co):
            lines.append("#define FV_AS241_%s%d %s" % (nm, i, hexd(float(v))))
    facts = [float(v) for v in L._ASYM_FACTS]
    pas = [[float(L._ASYM_PASCAL[i, j]) for j in range(18)] for i in range(18)]
    for i in range(18):
        for j in range(18):
            assert (pas[i][j] != 0.0) == (i <= j)
    lines.append("// lbr.py:59-62 _ASYM_FACTS (18) and the upper triangle of _ASYM_PASCAL")
    lines.append("// (P[i][j] != 0 iff i <= j), stored column-major: col j holds P[0..j][j]")
    emit_array(lines, "double", "fv_asym_facts", facts, hexd)
    tri = [pas[i][j] for j in range(18) for i in range(j + 1)]
    emit_array(lines, "double", "fv_asym_pascal", tri, hexd)
    lines.append("")

    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    with open(OUT, "w") as f:
        f.write("\n".join(lines) + "\n")
    print("wrote", OUT, len(lines), "lines")


if __name__ == "__main__":
    main()
