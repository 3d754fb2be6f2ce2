# compute-sanitizer over the smoke path (tiny config, 6 batches, oracle-checked); every
# library buffer is its own cudaMalloc so memcheck sees out-of-bounds between buffers
set -o pipefail
mkdir -p gpurun_out
make -s || exit 1
for tool in memcheck initcheck racecheck synccheck; do
  echo "== $tool"
  TGS_CUDAMALLOC=1 timeout 900 compute-sanitizer --tool $tool --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/sanitize_$tool.txt 2>&1
  tail -4 gpurun_out/sanitize_$tool.txt
done
