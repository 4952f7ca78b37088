# Round-2 profile set (run on the GPU box from the repo root): per-CTA histogram, bench line,
# ncu launch list of the steady state, ncu --set full of one steady-state round of every lane
# (summarised on the box; the .ncu-rep of the three CTA-per-env kernels comes back for source
# inspection -- gpurun returns at most 64 MiB).
set -x
export GRIP_LIB=build/libgripipc_ctatime.so
timeout 600 python tools/cta_hist.py --rounds 64 --out gpurun_out/r2_cta_hist.json > gpurun_out/cta.log 2>&1
unset GRIP_LIB
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/b7.json 2> gpurun_out/b7.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"^k_" --launch-skip 12000 --launch-count 1500 --csv --log-file gpurun_out/r2_launches.csv python bench.py --no-cpu --steps 2 --warmup 3 > gpurun_out/ncu1.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_(linesearch|assemble_direct|candidates|tet_front|tet_jacobi2|tet_back|elements_w|begin|finalize|contact_K|tet_finish|eig_commit)" --launch-skip 12000 --launch-count 45 -o /tmp/r2_full python bench.py --no-cpu --steps 2 --warmup 3 > gpurun_out/ncu2.log 2>&1
python tools/ncu_summary.py /tmp/r2_full.ncu-rep gpurun_out/r2_ncu_full.json "ncu --set full of 45 steady-state launches of the bench's 3-lane layout (launch-skip 12000), every grip kernel of about one round of each lane" > gpurun_out/ncu_summary.log 2>&1
for k in k_linesearch k_assemble_direct k_candidates k_tet_jacobi2 k_begin; do python tools/ncu_lines.py /tmp/r2_full.ncu-rep "$k" 40 > gpurun_out/r2_lines_$k.txt 2>&1; done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_(linesearch|assemble_direct|candidates)" --launch-skip 2600 --launch-count 3 -o gpurun_out/r2_top3 python bench.py --no-cpu --steps 2 --warmup 3 > gpurun_out/ncu3.log 2>&1
ls -la gpurun_out
