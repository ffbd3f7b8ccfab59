#!/bin/bash
# CRN kernel variants: bash tools/tune_crn.sh OUT "name:flags" ...
out=$1; shift
for spec in "$@"; do
  name=${spec%%:*}; flags=${spec#*:}
  MC_EXTRA_FLAGS="$flags" MC_LIB_OUT=/tmp/mc_$name.so python -m paper_2005_10494_b200.build > /dev/null 2>&1 || { echo "{\"variant\": \"$name\", \"error\": \"build\"}" >> $out; continue; }
  for est in cond ind; do
    r=$(MC_LIB_PATH=/tmp/mc_$name.so timeout 300 python tools/time_fused.py --est $est --crn 2>/dev/null | tail -1)
    echo "{\"variant\": \"$name\", \"flags\": \"$flags\", \"result\": $r}" >> $out
  done
done
