# A/B of the row-pair halo tiles (ICE_NO_PAIR) on the level-0/1 convolutions that use them
for rep in 1 2; do
for args in "fprop 32 256 256 64 64 64" "dgrad 32 128 128 64 0 128" "dgrad 32 256 256 64 64 64" "fprop 32 128 128 128 128 128" "dgrad 32 128 128 128 128 128" "fprop 32 128 128 128 0 128"; do
  a=$(python tools/time_conv.py $args 2>&1 | tail -1)
  b=$(ICE_NO_PAIR=1 python tools/time_conv.py $args 2>&1 | tail -1)
  echo "$args | pair: ${a##*]} | nopair: ${b##*]}"
done; done
