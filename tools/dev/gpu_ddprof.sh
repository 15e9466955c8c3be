ncu --metrics gpu__time_duration.sum --clock-control none -s 400 -c 120 --csv --log-file gpurun_out/dd_launches.csv python tools/dev/dd_compute_probe.py 4114 > /dev/null 2>&1
python tools/launches.py gpurun_out/dd_launches.csv
