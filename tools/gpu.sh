#!/bin/bash
# One parameterized GPU job runner (run under gpurun from the repo root).  Every job writes
# into gpurun_out/<tag>/ so results of different jobs never overwrite each other; the
# summaries worth keeping are copied to profiles/ by hand, named per round.
#
#   tools/gpu.sh <tag> tests [pytest -k expr]         pytest -m gpu (+ smoke)
#   tools/gpu.sh <tag> bench [bench.py args]          default bench line (+ args)
#   tools/gpu.sh <tag> cfgs  [configs]                one bench line per config (device-resident)
#   tools/gpu.sh <tag> ncu   <kernel-regex> [bench.py args]   ncu --set full (+source) of one launch
#   tools/gpu.sh <tag> launches [bench.py args]       ncu launch list (gpu__time_duration per launch)
#   tools/gpu.sh <tag> ab    <defines-A> <defines-B> [bench.py args]
#                                                    same bench with two builds (-D lists, ',' separated)
#   tools/gpu.sh <tag> envs "A=1,B=2;A=3" [bench.py args]   the bench under each env setting
#   tools/gpu.sh <tag> sanitize                       compute-sanitizer memcheck/racecheck on small fills
# Several jobs can be chained:  tools/gpu.sh r02a tests ';' r02a bench --config C3
set -u
export PYTHONUNBUFFERED=1
run_job() {
  local tag=$1 job=$2; shift 2
  local out=gpurun_out/$tag
  mkdir -p "$out"
  case "$job" in
    tests)
      timeout 1500 python -m pytest tests -m gpu -x -q ${1:+-k "$1"} > "$out/pytest_gpu.log" 2>&1
      echo "pytest rc=$?"; tail -3 "$out/pytest_gpu.log"
      timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$out/smoke.log" 2>&1; echo "smoke rc=$?"; tail -2 "$out/smoke.log";;
    bench)
      timeout 900 python bench.py "$@" > "$out/bench.json" 2> "$out/bench.err"; echo "bench rc=$?"; tail -c 3000 "$out/bench.json";;
    cfgs)
      for c in ${1:-C1 C1S C2 C3 C3W C4 C4W C5}; do
        timeout 600 python bench.py --config "$c" --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 --secondary "" \
          >> "$out/cfgs.jsonl" 2>> "$out/cfgs.err"; echo "$c rc=$?"
      done
      python - "$out/cfgs.jsonl" <<'PY'
import json, sys
for l in open(sys.argv[1]):
    try: d = json.loads(l)
    except Exception: continue
    r = d.get("roofline", {})
    print(d["config"]["workload"][:40], "%.3e ev/s" % d["value"], "frac %.3f" % r.get("frac", 0), "ms %.3f" % d["ms_per_step"], r.get("kernel"))
PY
      ;;
    ncu)
      local rx=$1; shift
      timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$rx" -s 3 -c 1 -o "$out/prof" \
        python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 --secondary "" "$@" > "$out/ncu.log" 2>&1
      echo "ncu rc=$?"; tail -3 "$out/ncu.log";;
    launches)
      timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file "$out/launches.csv" \
        python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 "$@" > "$out/launches.log" 2>&1
      echo "launches rc=$?";;
    ab)
      local da=$1 db=$2; shift 2
      for v in A B; do
        local defs; [ $v = A ] && defs=$da || defs=$db
        BHIST_LIBRARY=$PWD/build_ab/libbhist_$v.so python -c "
import sys; from paper_2401_13310_b200 import _build
_build.build(force=True, defines=[d for d in sys.argv[1].split(',') if d])" "$defs" > "$out/build_$v.log" 2>&1 || { echo "build $v failed"; tail "$out/build_$v.log"; }
      done
      for rep in 1 2; do for v in A B; do
        BHIST_LIBRARY=$PWD/build_ab/libbhist_$v.so timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline \
          --e2e-steps 1 --secondary "" "$@" > "$out/ab_${v}_$rep.json" 2>> "$out/ab.err"
        python -c "import json,sys; d=json.load(open(sys.argv[1])); print(sys.argv[2], d['ms_per_step'], d['roofline']['frac'])" "$out/ab_${v}_$rep.json" "$v$rep"
      done; done;;
    envs)   # envs "A=1,B=2;A=3" [bench args]: the bench under each ';'-separated env setting
      local sets=$1; shift
      IFS=';' read -ra SETS <<< "$sets"
      for st in "${SETS[@]}"; do
        ( IFS=',' read -ra KV <<< "$st"; for kv in "${KV[@]}"; do [ -n "$kv" ] && export "$kv"; done
          timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 --secondary "" "$@" \
            > "$out/env.json" 2>> "$out/envs.err"
          python -c "import json,sys; d=json.load(open(sys.argv[1])); print(sys.argv[2], round(d['ms_per_step'],4), round(d['roofline']['frac'],4))" "$out/env.json" "[$st]" )
      done;;
    sanitize)
      for tool in memcheck racecheck synccheck; do
        echo "== compute-sanitizer --tool $tool" >> "$out/sanitize.log"
        timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_run.py >> "$out/sanitize.log" 2>&1
        echo "$tool rc=$?"; tail -2 "$out/sanitize.log"
      done;;
    *) echo "unknown job $job"; return 2;;
  esac
}
args=("$@"); cur=()
for a in "${args[@]}" ';'; do
  if [ "$a" = ";" ]; then [ ${#cur[@]} -gt 0 ] && run_job "${cur[@]}"; cur=(); else cur+=("$a"); fi
done
