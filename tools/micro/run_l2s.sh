B=tools/micro/l2_stream
( $B 1 12 388 1; $B 1 12 388 2; $B 1 12 388 3; $B 1 12 388 4; $B 2 6 388 1; $B 2 6 388 2; $B 3 4 390 1; $B 3 4 390 2; $B 1 13 388 1; $B 1 13 388 2 ) > gpurun_out/r02bk_l2stream.txt 2>&1
