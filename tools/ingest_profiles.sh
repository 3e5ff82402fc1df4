# Copy a round-end refresh (gpurun_out/${P}_*) into profiles/ and regenerate profiles/README.md.
#   P=f7 bash tools/ingest_profiles.sh
set -e
P=${P:-f7}
O=gpurun_out
tail -1 $O/${P}_bench.log > profiles/r1_bench_n1.json
cp $O/${P}_breakdown.txt profiles/r1_step_breakdown_mbs2_m32.txt
cp $O/${P}_launches.csv profiles/r1_launches_1p5b_zbh1_m8_mbs2.csv
{ echo "# ncu --metrics gpu__time_duration.sum --clock-control none -s 12000 -c 3200 python bench.py --steps 1 --warmup 3 --microbatches 8 --no-cpu-baseline"
  echo "# GPT-1.5B seq2048 zb-h1 d=1, m=8 x 2 sequences (T=4096), final round-1 kernels; cold-cache serialised launches: compare SHARES, not absolutes"
  python tests/ncu_summary.py $O/${P}_launches.csv; } > profiles/r1_launches_1p5b_zbh1_m8_mbs2.txt
{ echo "# ncu --set full --clock-control none --import-source on -k regex:'gemm_kernel|attn_' -c 7 python -m tests.prof_kernels"
  echo "# bench pass shapes at micro-batch 2 (T=4096, h=2048, 16 heads); final round-1 kernels (attention fwd v3, bwd v4)"
  echo; python tools/ncu_full_summary.py $O/${P}_full.ncu-rep; } > profiles/r1_ncu_full_t4096.md
python - <<PY
import json
rows = [json.loads(l) for l in open("$O/${P}_attn.log") if l.startswith("{")]
rows = [r for r in rows if "batch" in r]
keys = ("batch", "seq", "heads", "fwd_tcgen05_tflops", "bwd_tcgen05_tflops", "fwd_tcgen05_us", "bwd_tcgen05_us")
json.dump([{k: r[k] for k in keys} for r in rows], open("profiles/r1_attn_tflops.json", "w"), indent=1)
PY
cp $O/${P}_proj_1p5b_bal.json profiles/r1_projection_1p5b_balanced_mbs2.json
cp $O/${P}_proj_1p5b_even_p8.json profiles/r1_projection_1p5b_even_p8_mbs2.json
cp $O/${P}_proj_6b.json profiles/r1_projection_6b_p8_via_chunks.json
cp $O/${P}_proj_14b.json profiles/r1_projection_14b_p8_via_chunks.json
cp $O/${P}_proj_6b_l31.json profiles/r1_projection_6b_l31_p8_via_chunks.json
cp $O/${P}_proj_14b_l31.json profiles/r1_projection_14b_l31_p8_via_chunks.json
cp $O/${P}_proj_1p5b_l30_bal.json profiles/r1_projection_1p5b_l30_balanced_p8.json
python tools/profiles_readme.py
