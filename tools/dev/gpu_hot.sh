# one --set full capture of one MD step of DPA3 2PTC (all 7 kernels), source-level
ncu --set full --import-source on --clock-control none --cache-control none -s 30 -c 7 \
    -o gpurun_out/hot_dpa3_2PTC python tools/ncu_target.py dpa3 2PTC 8 > gpurun_out/hot.log 2>&1
echo "ncu rc=$?"; ls -la gpurun_out/*.ncu-rep
