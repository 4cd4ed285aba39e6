# device bench A/B: the in-tree library against every _variants/*/ build (twice, interleaved)
python -m paper_1710_07745_b200.build > /dev/null || { echo BUILD FAILED; exit 1; }
one() {  # name libpath [bench args]
  EF_LIB_OVERRIDE=$2 python bench.py --no-e2e --no-cpu "${@:3}" 2>gpurun_out/err_$1.log | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); x=d.get("extra") or {}; print("'$1'", d["value"], d["ms_per_step"], "K1", d["roofline"]["avg_launch_ms"], "C1", (x.get("c1") or {}).get("ms_per_step"), d["clocks"]["sm_mhz"])'
}
for rep in 1 2; do
  one base paper_1710_07745_b200/libedgeforge_b200.so "$@"
  for v in _variants/*/; do n=$(basename $v); one $n $v/libedgeforge_b200.so "$@"; done
done
