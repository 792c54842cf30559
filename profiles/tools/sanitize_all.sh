set -x
CS=/usr/local/cuda/bin/compute-sanitizer
mkdir -p gpurun_out/san
for c in rows_static16 rows_static2 rows_inf16 rows_inf2 shard_fused shard3 entries patched fft recon draws; do
  for tool in memcheck racecheck synccheck; do
    timeout 600 $CS --tool $tool --print-limit 20 python profiles/tools/sanitize_cases.py $c > gpurun_out/san/${c}_${tool}.log 2>&1
    echo "$c $tool rc=$?" >> gpurun_out/san/summary.txt
  done
done
