M="--metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --csv"
for c in "0 1 16 4 1 2048 16 128" "0 1 16 4 1 2048 16 512" "0 1 16 4 1 2048 16 2048" "0 1 16 4 4 2048 16 2048" "0 1 16 4 16 2048 16 2048" "0 1 16 4 16 2048 16 256" "0 2 16 4 8 2048 16 2048" "0 2 16 4 8 7680 16 2560" "1 40 2 4 16 35 8457 2560" "1 40 2 4 16 35 8457 256" "1 40 2 4 1 35 8457 2560" "1 16 2 4 16 35 700 2048"; do
  echo "== $c"; ncu $M python profiles/skinny_one.py $c 3 2>&1 | grep -E "gpu__time|dram__bytes" | tail -2 | awk -F'","' '{print $(NF-1), $NF}'
done
