#!/bin/bash
# Repeat the GPU suite with the in-tree library and each variants/lib_*.so;
# print one line per run (pass count / failures).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
N=${N:-6}
for i in $(seq 1 $N); do
  r=$(timeout 700 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -1)
  echo "default run $i: $r"
  for lib in variants/lib_*.so; do
    r=$(FV_LIB=$PWD/$lib timeout 700 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -1)
    echo "$(basename $lib) run $i: $r"
  done
done
