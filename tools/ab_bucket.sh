#!/bin/bash
# A/B of the single-GPU gradient bucket size (fused Adam per bucket on a side stream):
#   tools/ab_bucket.sh "4096 380 200" [rounds]
R=${2:-2}
for i in $(seq $R); do
  for mb in $1; do
    ICE_BUCKET_MB=$mb python bench.py --no-autolabel --no-cpu --no-config5 --steps 20 > /tmp/ab.json 2>/dev/null
    python -c "import json,sys; d=json.load(open('/tmp/ab.json')); print('bucket_mb', sys.argv[1], d['value'], d['ms_per_step'], d['clocks']['sm_mhz'])" $mb
  done
done
