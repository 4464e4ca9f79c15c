timeout 200 python tools/swf_check.py --env "MPK_SWEEP_PICK=swf" --env "MPK_SWEEP_PICK=swf SWF_FORCE_RERUN=1" cd9_97 cfg1 cd9_1000 cfg4
for e in "MPK_SWF_ONLY_G0=1" "MPK_SWF_PF=0"; do
echo "== $e"
env $e SWF_DBG=2 timeout 60 python tools/swf_probe.py cfg4 1
done
