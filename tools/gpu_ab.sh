# in-process A/B of library variants built by tools/build_variant.sh (args: settings for tools/tune_fwd.py)
python tools/tune_fwd.py "$@" > gpurun_out/ab.log 2>&1; tail -12 gpurun_out/ab.log
