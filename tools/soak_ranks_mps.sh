# Cross-process rank-p2p soaks under MPS (see tools/soak_ranks.py).
export CUDA_MPS_PIPE_DIRECTORY=/tmp/ising_mps_pipe CUDA_MPS_LOG_DIRECTORY=/tmp/ising_mps_log
mkdir -p $CUDA_MPS_PIPE_DIRECTORY $CUDA_MPS_LOG_DIRECTORY gpurun_out
nvidia-cuda-mps-control -d
trap 'echo quit | nvidia-cuda-mps-control' EXIT
for c in "4 32768 32768 3000" "8 16384 65536 1000" "2 4096 8192 50000"; do
  timeout 900 python tools/soak_ranks.py $c > gpurun_out/soak_ranks_case.out 2> gpurun_out/soak_ranks_case.err
  echo "case $c rc=$? $(tail -1 gpurun_out/soak_ranks_case.out)"
  grep -iE "error|exception|Traceback" gpurun_out/soak_ranks_case.err | head -3
done
