cd "${GRAFT_REPO_ROOT:-/root/repo}"; O=gpurun_out/x18; mkdir -p $O/timeline
timeout 1500 python tools/sweep_c3.py --out $O/c3.json > $O/c3.log 2>&1
timeout 900 python tools/timeline_run.py --out $O/timeline > $O/timeline.log 2>&1
GFS_BENCH_SHARE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 --total-gib 8 --quick > $O/bench_n2_shared.log 2>&1
timeout 600 python tools/preset_probe.py > $O/preset.log 2>&1
tail -3 $O/c3.log; tail -c 300 $O/bench_n2_shared.log
