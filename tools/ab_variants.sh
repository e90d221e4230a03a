# A/B of library variants (built with paper_1609_01317_b200.build.build(defines=..., tag=...))
# on the C3 kbench scenes, after the parity tests of the main library.
#   bash tools/ab_variants.sh "legacy minb6" [kbench variants]
set -u
tags=${1:-}
kv=${2:-volume,volume+surface}
python -m pytest tests/test_gpu_parity.py tests/test_gpu_random.py tests/test_gpu_fullsize.py -x -q -k "not c5 and not c4" > gpurun_out/ab_pytest.log 2>&1; echo pytest_rc=$? >> gpurun_out/ab_pytest.log
: > gpurun_out/ab_kb.log
for v in main $tags; do
  if [ $v = main ]; then lib=paper_1609_01317_b200/_lib/libvoxelcast_b200.so; else lib=paper_1609_01317_b200/_lib/$v/libvoxelcast_b200.so; fi
  echo "== $v" >> gpurun_out/ab_kb.log
  VC_LIB=$lib python tools/kbench.py --variants $kv --frames 20 >> gpurun_out/ab_kb.log 2>&1
done
