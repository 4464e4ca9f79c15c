export MPK_SWEEP_PICK=swf SWF_ORACLE=0 MPK_SWF_ONLY_G0=1 MPK_SSWEEP_W=1 MPK_SWF_PF=0
timeout 300 ncu --set full --import-source on --clock-control none -k regex:swf_kernel -c 2 -f -o gpurun_out/swfg0 python tools/swf_probe.py child cfg4 > gpurun_out/ncu_g0.log 2>&1
ncu -i gpurun_out/swfg0.ncu-rep --page source --csv --print-source sass > gpurun_out/swfg0_src.csv 2>/dev/null
ncu -i gpurun_out/swfg0.ncu-rep --page details --csv > gpurun_out/swfg0_det.csv 2>/dev/null
