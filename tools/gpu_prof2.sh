cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
W=c3 KREGEX=k_price_greeks NCU_C=1 TAG=g0 bash tools/gpu_prof.sh
W=c2 KREGEX='k_halley_(iter|bracket)' NCU_C=2 TAG=h0 bash tools/gpu_prof.sh
for t in g0 h0; do
  for k in k_price_greeks k_halley_iter k_halley_bracket; do
    ncu -i gpurun_out/prof_$t.ncu-rep --page source --csv --print-source sass --kernel-name-base mangled -k regex:$k > gpurun_out/src_${t}_$k.csv 2>/dev/null
  done
done
ls -la gpurun_out
