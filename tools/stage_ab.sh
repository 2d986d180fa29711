# staged (TMA-store) vs direct epilogue stores on the level-0/1 halo kernels (ICE_NO_STAGE)
for args in "dgrad 32 256 256 64 64 64" "dgrad 32 256 256 64 0 64" "fprop 32 256 256 64 0 64" "dgrad 32 128 128 128 128 128" "fprop 32 128 128 128 0 128"; do
  a=$(python tools/time_conv.py $args 2>&1 | tail -1)
  b=$(ICE_NO_STAGE=1 python tools/time_conv.py $args 2>&1 | tail -1)
  c=$(ICE_LIB_PATH=paper_2403_13135_b200/_C/vnoepi/libicelabel_b200.so python tools/time_conv.py $args 2>&1 | tail -1)
  echo "$args | staged: ${a##*]} | direct: ${b##*]} | no epilogue: ${c##*]}"
done
