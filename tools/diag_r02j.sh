timeout 600 ncu -k regex:route3 --launch-skip 1 --launch-count 1 --set full --clock-control none -f -o gpurun_out/route3_batch python tools/prof_batched.py > gpurun_out/pb.log 2>&1
timeout 600 ncu -k regex:nsa_attend_batch --launch-skip 1 --launch-count 1 --set full --clock-control none -f -o gpurun_out/attend_batch python tools/prof_batched.py > gpurun_out/pb2.log 2>&1
ls -la gpurun_out/*batch*
