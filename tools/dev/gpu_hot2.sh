ncu --set full --import-source on --clock-control none --cache-control none -s 12 -c 3 \
    -o gpurun_out/hot_dpa2_2PTC python tools/ncu_target.py dpa2 2PTC 8 > gpurun_out/hot2.log 2>&1
echo "ncu rc=$?"
