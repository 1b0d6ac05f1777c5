#!/bin/bash
# Trace-serving sweep on this box's GPUs: designs x rates for one preset.
#   tools/trace_sweep.sh MODEL PRESET "RATES" "DESIGN P T;DESIGN P T" DURATION OUT [MAXOUT]
MODEL=$1; PRESET=$2; RATES=$3; DESIGNS=$4; DUR=$5; OUT=$6; MAXOUT=${7:-0}
IFS=';' read -ra DS <<< "$DESIGNS"
for R in $RATES; do
  for D in "${DS[@]}"; do
    set -- $D
    timeout 900 python tools/trace_serve.py --model $MODEL --design $1 --prompt-machines $2 \
      --token-machines $3 --preset $PRESET --rate $R --duration $DUR --max-output $MAXOUT \
      >> $OUT 2>> $OUT.err
  done
done
