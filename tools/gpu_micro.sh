cd tools/micro && ./ts_mma > ../../gpurun_out/r2_ts_mma.txt 2>&1; ./pipe_tp2 > ../../gpurun_out/r2_pipe_tp2.txt 2>&1; nvidia-smi --query-gpu=clocks.sm --format=csv >> ../../gpurun_out/r2_pipe_tp2.txt
