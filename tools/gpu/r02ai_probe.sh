mkdir -p gpurun_out
python tools/cold_only_probe.py > gpurun_out/probe_full.txt 2>&1; cat gpurun_out/probe_full.txt
TI64_VARIANT_LIB=$PWD/paper_2402_17580_b200/_lib/variants/lib_stub.so python tools/cold_only_probe.py > gpurun_out/probe_stub.txt 2>&1; cat gpurun_out/probe_stub.txt
python tools/cold_only_probe.py --amp 0 1 > gpurun_out/probe_base.txt 2>&1; cat gpurun_out/probe_base.txt
timeout 900 ncu --set full --import-source on --clock-control none -k regex:advance_kernel --launch-skip 2 -c 1 -o gpurun_out/prof_probe -f python tools/cold_only_probe.py --windows 3 > gpurun_out/ncu_probe.log 2>&1; tail -2 gpurun_out/ncu_probe.log
