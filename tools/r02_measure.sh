set -x
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r02b.json 2> gpurun_out/bench_r02b.err; echo bench_rc=$?
python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref_r02c.json 2>&1; echo ref_rc=$?
for v in main r1base; do if [ $v = main ]; then lib=paper_1609_01317_b200/_lib/libvoxelcast_b200.so; else lib=paper_1609_01317_b200/_lib/$v/libvoxelcast_b200.so; fi; echo "== $v" >> gpurun_out/ab_r1.log; VC_LIB=$lib python tools/kbench.py --variants volume,taps,volume+surface --frames 20 >> gpurun_out/ab_r1.log 2>&1; done
python bench.py --timed-only --steps 4 --warmup 3 > gpurun_out/timed_plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches.csv python bench.py --timed-only --steps 4 --warmup 3 > gpurun_out/ncu_launch.log 2>&1; echo launches_rc=$?
ncu --set full --clock-control none --import-source on -k regex:"shade_kernel|firsthit_kernel" -s 6 -c 2 -o gpurun_out/prof_r02_final python bench.py --timed-only --steps 2 --warmup 3 > gpurun_out/ncu_full.log 2>&1; echo full_rc=$?
