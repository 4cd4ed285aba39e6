# every config's device-resident bench value, with the default library and with an env switch
# usage: configs_ab.sh VAR=value ...
cd "$(dirname "$0")/.."
for c in 0 2 1; do
  for mode in base ab; do
    if [ $mode = ab ]; then pre="env $*"; else pre=""; fi
    $pre python bench.py --config $c --no-e2e --no-cpu 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("C'$c' '$mode'", d["value"], d["ms_per_step"])'
  done
done
