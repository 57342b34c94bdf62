"""Repeat tests/test_price_iv.py::test_round_trip_exceptions_match_two_calls N times
(python tools/stress_roundtrip.py [N]) and count failures: the flake hunt behind the
broadcast-scalar ordering fix (profiles/README.md, r2f)."""
import sys, os, time
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import paper_2604_27210_b200 as fv
import test_price_iv as T
fails = 0
t0 = time.time()
for i in range(int(sys.argv[1]) if len(sys.argv) > 1 else 10):
    try:
        T.test_round_trip_exceptions_match_two_calls(fv)
    except AssertionError as e:
        fails += 1
        print("FAIL", i, str(e)[:600], flush=True)
print("done fails", fails, "in", round(time.time() - t0), "s")
