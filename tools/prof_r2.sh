# Round-2 profile set (run on the GPU box from the repo root): per-CTA histogram, bench line,
# ncu launch list of the steady state, ncu --set full of one steady-state round of every lane
# (summarised on the box; the .ncu-rep of the three CTA-per-env kernels comes back for source
# inspection -- gpurun returns at most 64 MiB).  TAG names the output set.
set -x
TAG=${TAG:-v2}
export GRIP_LIB=build/libgripipc_ctatime.so
timeout 600 python tools/cta_hist.py --rounds 64 --out gpurun_out/r2_${TAG}_cta_hist.json > gpurun_out/cta.log 2>&1
unset GRIP_LIB
export GRIP_LIB=build/libgripipc_phase.so
timeout 600 python tests/diag_phase.py --steps 20 --warmup 5 > gpurun_out/r2_${TAG}_phase.txt 2>&1
unset GRIP_LIB
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r2_${TAG}_bench.json 2> gpurun_out/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"^k_" --launch-skip 20000 --launch-count 1500 --csv --log-file gpurun_out/r2_${TAG}_launches.csv python bench.py --no-cpu --steps 2 --warmup 3 > gpurun_out/ncu1.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_(linesearch|assemble_direct|candidates|tet_front|tet_jacobi2|tet_back|elements_w|bound|begin|finalize|contact_K|tet_finish|eig_commit|static|abd_w|tet_scan)" --launch-skip 20000 --launch-count 60 -o /tmp/r2_full python bench.py --no-cpu --steps 2 --warmup 3 > gpurun_out/ncu2.log 2>&1
python tools/ncu_summary.py /tmp/r2_full.ncu-rep gpurun_out/r2_ncu_full.json "ncu --set full of 60 steady-state launches of the bench's own layout (9 lanes: 3 per object kind, 44-45 envs each; launch-skip 20000): every grip kernel of about one round of a few lanes, all streams" > gpurun_out/ncu_summary.log 2>&1
for k in k_linesearch k_assemble_direct k_candidates k_tet_jacobi2 k_bound k_tet_front; do python tools/ncu_lines.py /tmp/r2_full.ncu-rep "$k" 40 > gpurun_out/r2_${TAG}_lines_$k.txt 2>&1; done
ls -la gpurun_out
