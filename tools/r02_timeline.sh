# lattice launch timeline with exp_libs/tl.so (tools/build_exp_lib.sh, built before the gpurun call)
cp paper_2406_08186_b200/_lib/libqwb200.so /tmp/cur.so
cp exp_libs/tl.so paper_2406_08186_b200/_lib/libqwb200.so
for nx in 2048 4096; do python tools/r02_timeline.py $nx; done > gpurun_out/r02cy_timeline.txt 2>&1
cp /tmp/cur.so paper_2406_08186_b200/_lib/libqwb200.so
