# CNN A/B (env / library variants): conv_prof launch lists per setting; CFGS selects the configs
mkdir -p gpurun_out
i=0
for setting in "$@"; do
  i=$((i+1))
  for cfg in ${CFGS:-c3 c4}; do
    env $setting timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ab_${cfg}_$i.csv python tools/conv_prof.py $cfg > /dev/null 2>&1
    echo "== $setting $cfg"; python tools/launch_summary.py gpurun_out/ab_${cfg}_$i.csv ${TOP:-7} | grep -E "${PAT:-conv_tc|pool|total}"
  done
done
