#!/bin/bash
# A/B an environment toggle on the train step: tools/ab_env.sh VAR=value [rounds]
T=$1; R=${2:-3}
for i in $(seq $R); do
  for on in 0 1; do
    if [ $on = 1 ]; then export $T; else unset ${T%%=*}; fi
    python bench.py --no-autolabel --no-cpu --no-config5 --steps 20 > /tmp/ab.json 2>/dev/null
    python -c "import json,sys; d=json.load(open('/tmp/ab.json')); print(sys.argv[1], d['value'], d['ms_per_step'], d['clocks']['sm_mhz'])" "$([ $on = 1 ] && echo $T || echo default)"
  done
done
unset ${T%%=*}
