for h in 0 2048 4096 8192 12288 16384 20480 24576 28800; do echo "hot=$h"; DYNPR_HOT=$h timeout 300 python profiles/prof_driver.py --scale 24 --static-iters 20; done
