# source-level stall hot spots of the DPA3 2PTC network kernels (one MD step captured)
ncu --set full --import-source on --clock-control none --cache-control none -s $((7*4+2)) -c 7 \
    -o gpurun_out/hot3 python tools/ncu_target.py dpa3 2PTC 8 > /dev/null 2>&1; echo "ncu rc=$?"
for k in "k_msg_fwd" "k_embed_bwd_pull" "k_msg_bwd_pull" "k_embed<"; do
  echo "=== $k"; python tools/ncu_hot.py gpurun_out/hot3.ncu-rep "$k" 14 2>&1 | cut -c1-230
done > gpurun_out/hot3.txt
python tools/ncu_hot.py gpurun_out/hot3.ncu-rep "k_msg_fwd" 14 1 2>&1 | cut -c1-230 > gpurun_out/hot3_last.txt
rm -f gpurun_out/hot3.ncu-rep
