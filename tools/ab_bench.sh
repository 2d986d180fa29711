#!/bin/bash
# A/B the train step of two library builds on the same box: tools/ab_bench.sh <libA> <libB> [rounds]
A=$1; B=$2; R=${3:-3}
for i in $(seq $R); do
  for L in $A $B; do
    ICE_LIB_PATH=$L python bench.py --no-autolabel --no-cpu --steps 20 > /tmp/ab.json 2>/dev/null
    python -c "import json,sys; d=json.load(open('/tmp/ab.json')); print(sys.argv[1][-40:], d['value'], d['ms_per_step'], d['clocks']['sm_mhz'])" $L
  done
done
