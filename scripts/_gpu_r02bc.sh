# round-2 session-4 call C: exhaustive strip-width x row-block sweep under the two-lane chunk loop
python scripts/sweep_div.py 1024x64 256x64 512x64 1024x256 2048x64 4096x64 128x512
