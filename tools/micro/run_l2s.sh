B=tools/micro/l2_stream
( $B 2 5 388 2 4096; $B 2 5 388 2 8192; $B 2 5 388 2 16384; $B 2 6 388 2 16384; $B 1 12 388 1 16384 ) > gpurun_out/r02br_l2stream.txt 2>&1
