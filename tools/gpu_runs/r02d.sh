mkdir -p gpurun_out
for g in 148 256 444; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_blind_rotate_v3 -s 1 -c 1 -o gpurun_out/r02d_br$g -f python tools/br_once.py $g > gpurun_out/r02d_ncu$g.log 2>&1
done
