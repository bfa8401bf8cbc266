mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kmap.py tests/test_gpu_configs.py -k "block or c5" -x -q > gpurun_out/kq_test.log 2>&1; echo rc=$? >> gpurun_out/kq_test.log
timeout 200 python tools/kmap_ab.py > gpurun_out/kq_ab.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/kq_launch.csv python tools/prof_kmap.py > gpurun_out/kq_ncu1.log 2>&1
