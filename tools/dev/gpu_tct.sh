O=gpurun_out
cp paper_1506_06039_b200/libmoco.so /tmp/libmoco_keep.so
cp dev_so/libmoco_tct.so paper_1506_06039_b200/libmoco.so
for c in 2 3 1; do echo "== C$c" >> $O/tct.txt; MOCO_BATCH_WAVES=1 python tools/profile_run.py --config $c --frames 1184 --iters 2 2>&1 | grep TCT | tail -3 >> $O/tct.txt; done
cp /tmp/libmoco_keep.so paper_1506_06039_b200/libmoco.so
