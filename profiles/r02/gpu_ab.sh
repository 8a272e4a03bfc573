python profiles/ab_static_layouts.py 24
rm paper_2404_08299_b200/csrc/_build/sweep.o
make -C paper_2404_08299_b200/csrc NVCC="/usr/local/cuda/bin/nvcc -DDYNPR_NO_FOLD" > /dev/null 2>&1
echo "--- no fold"
python profiles/ab_static_layouts.py 24
