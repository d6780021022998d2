timeout -s KILL 60 ./scripts/micro/tmem_rate > gpurun_out/tmem_rate.log 2>&1
