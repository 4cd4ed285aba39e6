# A/B an environment switch of the library: GPU parity tests with it on, then the
# device-resident bench with and without it, interleaved.   usage: ab_env.sh VAR=value [VAR2=value ...]
cd "$(dirname "$0")/.."
env "$@" python -m pytest tests -m gpu -x -q > gpurun_out/t_ab.log 2>&1; echo "TESTS($*): $(tail -1 gpurun_out/t_ab.log)"
one() { python bench.py --no-e2e --no-cpu 2>gpurun_out/err_ab.log | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("'"$1"'", d["value"], d["ms_per_step"], "K1", d["roofline"]["avg_launch_ms"], d["stats"]["fixups"])'; }
for rep in 1 2; do one base; env "$@" bash -c "$(declare -f one); one '$*'"; done
