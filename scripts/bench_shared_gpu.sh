#!/bin/bash
# Functional check of bench.py's one-rank-per-process (N > 1) path on a single-GPU box:
# N processes on GPU 0 under a private MPS daemon (so their persistent kernels co-reside),
# gloo process group, AO_BENCH_SHARED_GPU=1.  usage: scripts/bench_shared_gpu.sh N [bench args]
N=${1:-2}; shift
D=$(mktemp -d)
export CUDA_MPS_PIPE_DIRECTORY=$D/pipe CUDA_MPS_LOG_DIRECTORY=$D/log
mkdir -p $CUDA_MPS_PIPE_DIRECTORY $CUDA_MPS_LOG_DIRECTORY
nvidia-cuda-mps-control -d || echo "no MPS: ranks time-slice the GPU"
sleep 0.5
AO_BENCH_SHARED_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N \
  --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus $N "$@"
rc=$?
echo quit | nvidia-cuda-mps-control
exit $rc
