# session 5: slices per dynamic grab in the frontier sweeps (split single-slice 4 / light 2
# shipped vs 2/1 and 8/4), DF-P A/B
set -x
mkdir -p gpurun_out/r2s5g
timeout 1800 python profiles/r02/dfp_bisect_ab.py 24:1e-4,24:1e-6,26:1e-4,20:1e-4,20:1e-7,u20:1e-3 . _ab_g2 _ab_g8 > gpurun_out/r2s5g/grab_ab.txt 2>&1
cat gpurun_out/r2s5g/grab_ab.txt
