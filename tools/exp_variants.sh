#!/bin/bash
# compare library variants on the C5 bench (same binding); usage: tools/exp_variants.sh a.so b.so ...
for v in "$@"; do
  echo "== $v"
  LRBMS_LIB=$v python tools/exp_solver.py C5 100 '[{"rtol":1e-12}]' 2>&1 | tail -1
done
