HMDP_SKIN=0 timeout 600 python -m pytest tests/test_dpfamily.py -q -x -p no:cacheprovider -m gpu 2>&1 | tail -2
timeout 600 python -m pytest tests/test_dpfamily.py -q -x -p no:cacheprovider -m gpu 2>&1 | tail -2
timeout 600 python -m pytest tests/test_dpfamily.py -q -x -p no:cacheprovider -m gpu 2>&1 | tail -2
HMDP_CGRAPH_MAPPED_IN=0 timeout 600 python -m pytest tests/test_dpfamily.py -q -x -p no:cacheprovider -m gpu 2>&1 | tail -2
