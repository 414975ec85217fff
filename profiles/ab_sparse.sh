# A/B of sparse-kernel build variants on c4n (one box, interleaved): per-pass time from the bench line
cd $GRAFT_REPO_ROOT
for rep in 1 2; do
for v in "" _g1 _b16 _b4; do
  TSVD_LIB=$PWD/paper_2208_08410_b200/libtsvd$v.so python bench.py --config c4n --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab$v.log 2>&1
  tail -1 gpurun_out/ab$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', 'step_ms', round(d['ms_per_step'],1), 'pass_ms', round(d['roofline']['per_launch_ms'],2), 'frac', round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])"
done
done
