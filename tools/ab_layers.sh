# A/B helper: layer bench (lidar, C=32/64/96) + MinkUNet latency / 3-in-flight
mkdir -p gpurun_out
python tools/layer_bench.py --scan lidar --c 32 64 96 2>/dev/null | grep "implicit_gemm_s1\|implicit_gemm_s0\|dgrad" > gpurun_out/ab_layers_$1.txt
python tools/conc_probe.py --reps 2 2>&1 | grep "W=1 flush=1\|W=3 flush=1" >> gpurun_out/ab_layers_$1.txt
