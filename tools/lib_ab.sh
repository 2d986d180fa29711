# per-shape A/B of the current library against paper_2403_13135_b200/_C/vbase (time_conv.py)
B=paper_2403_13135_b200/_C/vbase/libicelabel_b200.so
for args in "$@"; do
  a=$(python tools/time_conv.py $args 2>&1 | tail -1)
  b=$(ICE_LIB_PATH=$B python tools/time_conv.py $args 2>&1 | tail -1)
  echo "$args | new: ${a##*]} | base: ${b##*]}"
done
