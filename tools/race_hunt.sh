# race_hunt.sh LIB TUNE RUNS: how many of RUNS pair_stress runs (6 rounds of the
# four split-K configs each) show a mismatch or a launch failure
L=$1; T=$2; R=${3:-6}; bad=0
for r in $(seq 1 $R); do
  out=$(LQG_LIB_PATH=$L PS_TUNE=$T PS_SYNC=1 timeout 300 python tools/pair_stress.py 6 2>&1)
  if echo "$out" | grep -qE "MISMATCH|FAILED|Error"; then bad=$((bad+1)); fi
done
echo "$L [$T]: $bad of $R runs bad"
