timeout 900 python bench.py --dtype f32 --steps 5 --warmup 3 --no-cpu > gpurun_out/r2p_f32.json 2> gpurun_out/r2p_f32.err
tail -3 gpurun_out/r2p_f32.err
