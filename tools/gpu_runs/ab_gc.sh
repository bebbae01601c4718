# same-box A/B of variants/*.so; GCS (default "1 2 3") gates per SM at 148 / 256 / 444 gates, two passes
for rep in 1 2; do for v in $(ls variants/*.so); do
for gc in ${GCS:-1 2 3}; do n=$((148*gc)); [ $gc = 2 ] && n=256
echo "$v GC=$gc"; GATEWAVE_B200_LIB=$v GATEWAVE_BR_GC=$gc timeout 300 python tools/br_time.py $n; done; done; done
