# Round-2 decode-pass evidence: pass tests, the bench line, ncu DRAM traffic of the
# bench's pass, the launch list of a short bench run, one ncu --set full capture.
set -x
timeout 600 python -m pytest tests/test_gpu_pass.py -q -x -m gpu 2>&1 | tail -2
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r2c.json 2> gpurun_out/bench_r2c.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_decode_pass --csv python tools/prof_pass.py > gpurun_out/pass_traffic.csv 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launch_list_r2c.csv python bench.py --steps 2 --warmup 3 --no-shapes --no-70b --no-admm --no-cpu-baseline > gpurun_out/ncu_ll.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_decode_pass -s 2 -c 1 -o gpurun_out/prof_pass_r2c python tools/prof_pass.py > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/ncu_full.log
