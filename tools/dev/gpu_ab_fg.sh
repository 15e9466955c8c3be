# force-kernel lanes per atom: 8 (default at these sizes) vs 16 vs 4
timeout 600 python -m pytest tests/test_gpu_md.py -q -x -p no:cacheprovider 2>&1 | tail -1
HMDP_FORCE_FG=16 timeout 600 python -m pytest tests/test_gpu_md.py tests/test_gpu_skin.py -q -x -p no:cacheprovider 2>&1 | tail -1
HMDP_FORCE_FG=4 timeout 600 python -m pytest tests/test_gpu_md.py tests/test_gpu_skin.py -q -x -p no:cacheprovider 2>&1 | tail -1
AB_REPS=2 AB_CFGS="dpa3:2PTC dpa2:2PTC dpa3:3LZM dpa2:3LZM" timeout 1500 bash tools/ab_env.sh - HMDP_FORCE_FG=16 HMDP_FORCE_FG=4 2>&1 | tee gpurun_out/ab_fg.txt
