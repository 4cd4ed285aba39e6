# On the GPU box: device-resident bench of the in-tree library and every _variants/*/ build,
# interleaved twice (box drift), K1 event time and whole step.
cd "$(dirname "$0")/.."
one() {  # name libpath
  EF_LIB_OVERRIDE=$2 python bench.py --no-e2e --no-cpu "${@:3}" 2>gpurun_out/err_$1.log | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("'$1'", d["value"], d["ms_per_step"], "K1", d["roofline"]["avg_launch_ms"], d["clocks"]["sm_mhz"], d["stats"]["fixups"])'
}
for rep in 1 2; do
  one base paper_1710_07745_b200/libedgeforge_b200.so "$@"
  for v in _variants/*/; do n=$(basename $v); one $n $v/libedgeforge_b200.so "$@"; done
done
