#!/bin/bash
# Multi-process rank-p2p on one B200 under MPS (nvidia-cuda-mps-control is in the image): with
# MPS the processes' kernels share the SMs concurrently, so the cross-process flag protocol
# (CUDA IPC peer pointers, acquire / release flags, fused halo stores) runs with writer and
# reader overlapping in time — without MPS they are time-sliced and a kernel boundary always
# separates them.  Runs the multi-process parity tests and the same-device multi-rank bench.
mkdir -p gpurun_out
export CUDA_MPS_PIPE_DIRECTORY=/tmp/ising_mps_pipe CUDA_MPS_LOG_DIRECTORY=/tmp/ising_mps_log
mkdir -p $CUDA_MPS_PIPE_DIRECTORY $CUDA_MPS_LOG_DIRECTORY
nvidia-cuda-mps-control -d && echo "MPS daemon started"
trap 'echo quit | nvidia-cuda-mps-control; echo "MPS daemon stopped"' EXIT
timeout 900 python -m pytest tests/test_gpu_multiprocess.py -q -s --timeout 600 > gpurun_out/mps_pytest.txt 2>&1
echo "pytest (MPS): $(tail -1 gpurun_out/mps_pytest.txt)"; grep -E "^world" gpurun_out/mps_pytest.txt
echo "MPS servers: $(echo get_server_list | nvidia-cuda-mps-control)"
for n in ${MPS_BENCH_N:-2 4}; do
  ISING_BENCH_SAME_DEVICE=1 timeout 900 python bench.py --gpus $n --steps 20 --warmup 5 ${MPS_BENCH_ARGS---no-legs} \
    > gpurun_out/mps_bench_n$n.json 2> gpurun_out/mps_bench_n$n.err
  echo "bench n=$n rc=$? $(python -c "import json,sys; d=json.load(open('gpurun_out/mps_bench_n$n.json')); print(d['value'], d['config']['transport'], d['invariance'])" 2>&1 | tail -1)"
done
tail -3 $CUDA_MPS_LOG_DIRECTORY/control.log 2>/dev/null
