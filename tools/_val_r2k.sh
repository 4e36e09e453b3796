mkdir -p gpurun_out
python bench.py > gpurun_out/r2k_bench.json 2> gpurun_out/r2k_bench.err; echo "bench $?"
python bench.py --impl reference > gpurun_out/r2k_ref.json 2> gpurun_out/r2k_ref.err; echo "ref $?"
python -m pytest tests -m gpu -q > gpurun_out/r2k_pytest.log 2>&1; echo "pytest $?"; tail -2 gpurun_out/r2k_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2k_smoke.log 2>&1; echo "smoke $?"
bash tools/ncu_one.sh list r2k; echo "list done"
bash tools/ncu_one.sh pcg_kernel_h8s r2k_h8s; echo "h8s done"
BENCH_ARGS="--mode parity --steps 2 --warmup 3 --no-cpu-baseline --no-parity-pass" bash tools/ncu_one.sh pcg_kernel_h8p r2k_h8p; echo "h8p done"
BENCH_ARGS="--mode fp32 --steps 2 --warmup 3 --no-cpu-baseline --no-parity-pass" bash tools/ncu_one.sh pcg_kernel_h8x r2k_h8x; echo "h8x done"
python tools/sweep.py --T 16,100,128,191,256 --B 4096 --reps 2 --md gpurun_out/r2k_sweep_T.md > gpurun_out/r2k_sweep_T.jsonl 2>&1; echo "sweep $?"
python tools/sweep.py --T 16,100 --B 1048576 --reps 1 --md gpurun_out/r2k_sweep_1M.md > gpurun_out/r2k_sweep_1M.jsonl 2>&1; echo "sweep1M $?"
