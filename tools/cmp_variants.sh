#!/bin/bash
# stage times of library variants: tools/cmp_variants.sh CFG STEPS a.so b.so ...
cfg=$1; n=$2; shift 2
for v in "$@"; do
  echo "== $v $(LRBMS_LIB=$v timeout 120 python tools/exp_stages.py $cfg $n 2>&1 | tail -1)"
done
