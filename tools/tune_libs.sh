#!/bin/bash
# Time prebuilt library variants (tools/lib_<name>.so) with tools/time_fused.py on a GPU box.
# usage: bash tools/tune_libs.sh OUTFILE REPS name1 name2 ...   (extra time_fused args via TF_ARGS)
out=$1; reps=$2; shift 2
for r in $(seq $reps); do
  for name in "$@"; do
    res=$(MC_LIB_PATH=$PWD/tools/lib_$name.so timeout 300 python tools/time_fused.py $TF_ARGS 2>/dev/null | tail -1)
    echo "{\"variant\": \"$name\", \"rep\": $r, \"args\": \"$TF_ARGS\", \"result\": $res}" >> $out
  done
done
