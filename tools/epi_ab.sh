# mainloop-only (ICE_EXP_NOEPI build in _C/vnoepi) vs full kernels: how much the epilogue costs per shape
for args in "fprop 32 256 256 64 0 64" "dgrad 32 256 256 64 0 64" "dgrad 32 256 256 64 64 64" "fprop 32 256 256 64 64 64" "dgrad 32 128 128 128 128 128" "fprop 32 128 128 128 0 128" "dgrad 32 128 128 64 0 128"; do
  a=$(python tools/time_conv.py $args 2>&1 | tail -1)
  b=$(ICE_LIB_PATH=paper_2403_13135_b200/_C/vnoepi/libicelabel_b200.so python tools/time_conv.py $args 2>&1 | tail -1)
  echo "$args | full: ${a##*]} | no epilogue: ${b##*]}"
done
