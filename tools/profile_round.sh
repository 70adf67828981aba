#!/bin/bash
# Regenerates the profiles/ evidence of one source state on the GPU box (run under gpurun).
# Each step starts only after the previous one exited 0; nothing measured under ncu is a bench value.
set -e
mkdir -p gpurun_out/prof
python paper_1501_02946_b200/_build.py > /dev/null
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/prof/bench_cfg4.json 2> gpurun_out/prof/bench_cfg4.err
for c in cfg1 cfg2 cfg3 cfg5; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/prof/bench_$c.json 2>/dev/null
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof/launches_cfg4.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/prof/ncu_launch.log 2>&1
# (one warm-up reconstruction outside the capture: the first call of a plan has no sample-scale hint
#  and runs the gridding twice; the captured call is the steady state)
timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off -f -o gpurun_out/prof/full_cfg4 \
  python tools/profile_step.py --iters 1 --warm 1 > gpurun_out/prof/ncu_full.log 2>&1
python tools/ncu_summary.py gpurun_out/prof/full_cfg4.ncu-rep gpurun_out/prof/ncu_full_summary.json gpurun_out/prof/traffic.json cfg4
echo PROFILE_OK
# the sharded (multi-GPU) code path at world size 1 under torchrun, as the driver launches N > 1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 \
  bench.py --gpus 1 --sharded --steps 10 --warmup 3 > gpurun_out/prof/bench_cfg4_sharded_w1.json 2> gpurun_out/prof/sharded.err || tail -5 gpurun_out/prof/sharded.err
timeout 300 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/prof/bench_cfg4_reference.json 2> gpurun_out/prof/ref.err || tail -5 gpurun_out/prof/ref.err
echo PROFILE_DONE
