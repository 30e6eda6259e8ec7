#!/bin/bash
# Full evidence refresh on a B200 box (run under gpurun from the repo root):
#   gpurun --timeout 3000 -- 'bash scripts/refresh.sh r02'
# then, here: python scripts/update_profiles.py gpurun_out/<tag> <tag>
# GPU tests, the bench line, the reference arm, the ncu launch list of one bench step, and
# `ncu --set full` captures of one PCG iteration and of the one-time build kernels.
tag=${1:-r02}
out=gpurun_out/$tag
mkdir -p $out
python -m pytest tests -m gpu -q -x > $out/gputest.log 2>&1; echo "gpu tests exit $?" >> $out/gputest.log
python bench.py > $out/bench.json 2> $out/bench.err
python bench.py --impl reference --steps 3 --warmup 3 > $out/ref.json 2>&1
python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-extras > $out/plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file $out/launches.csv \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-extras > $out/ncu_launch.log 2>&1
python scripts/prof_pcg.py 6 > $out/plain2.log 2>&1 &&
ncu --set full --clock-control none --import-source on \
    -k regex:"k_spmv2|k_tree_lift|k_tree_coarse|k_tree_level0|k_hier_level0" -s 14 -c 5 \
    -o $out/${tag}_pcg_iteration python scripts/prof_pcg.py 6 > $out/ncu_full.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_bistoch -s 4 -c 2 \
    -o $out/${tag}_bistoch python scripts/prof_pcg.py 1 > $out/ncu_bs.log 2>&1
ncu --set full --clock-control none --import-source on \
    -k regex:"k_grid_sort|k_grid_neighbours|k_grid_write|k_splat|k_pyr_sort|k_slice" -c 16 \
    -o $out/${tag}_build_kernels python scripts/prof_pcg.py 1 > $out/ncu_build.log 2>&1
ls -la $out
