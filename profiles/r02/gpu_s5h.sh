# session 5: slices per dynamic grab of the frontier split single-slice sweep (4 shipped vs 8, 16)
set -x
mkdir -p gpurun_out/r2s5h
timeout 1800 python profiles/r02/dfp_bisect_ab.py 24:1e-4,24:1e-5,24:1e-6,24:1e-3,26:1e-4,22:1e-4 . _ab_s8 _ab_s16 > gpurun_out/r2s5h/split_grab_ab.txt 2>&1
cat gpurun_out/r2s5h/split_grab_ab.txt
