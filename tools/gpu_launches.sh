# ncu launch list of one captured D121 step (per-kernel device time, serialized, cold-cache)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/profile_step.py --top 1 > gpurun_out/ncu_launch_run.log 2>&1
python tools/launch_summary.py gpurun_out/launches.csv > gpurun_out/launch_summary.txt; head -40 gpurun_out/launch_summary.txt
