# session 5: slices per dynamic grab of the Static split single-slice sweep (4 shipped vs 2, 8)
set -x
mkdir -p gpurun_out/r2s5j
timeout 1800 python profiles/r02/bisect_ab.py 23,24,25,26 . _ab_st2 _ab_st8 > gpurun_out/r2s5j/static_grab_ab.txt 2>&1
cat gpurun_out/r2s5j/static_grab_ab.txt
