MPK_VERBOSE=1 timeout 200 python tools/swf_check.py --env "MPK_SWEEP_PICK=swf" --env "MPK_SWEEP_PICK=swf SWF_FORCE_RERUN=1" --env "MPK_SWEEP_PICK=swf MPK_SWF_CL=8" --env "MPK_SWEEP_PICK=swf MPK_SWF_CL=1" cd9_97 cfg1 cd9_1000 cfg4 2>&1 | grep -v "^\[mpk\]"
for e in "MPK_SWF_CL=16" "MPK_SWF_CL=8" "MPK_SWF_CL=1"; do
echo "== $e"
env $e SWF_DBG=2 timeout 60 python tools/swf_probe.py cfg4 1
done
