for n in 256 1024; do
SVDK_JACOBI_DEVLOOP=0 timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/eig_launch_$n.csv python tools/eig_one.py $n > gpurun_out/eig_one_$n.log 2>&1; echo "n=$n rc=$?"
done
