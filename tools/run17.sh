bash tools/run11.sh
bash tools/run16.sh
