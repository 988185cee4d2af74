g++ -std=c++17 -O1 -g -fsanitize=address -fno-omit-frame-pointer -Iinclude tests/cpp/dropin_test.cpp -o /tmp/dropin_asan -Lpaper_1703_04219_b200/lib -lp2g -Wl,-rpath,$PWD/paper_1703_04219_b200/lib
ASAN_OPTIONS=protect_shadow_gap=0:detect_leaks=0 /tmp/dropin_asan > gpurun_out/asan.log 2>&1; echo "asan rc=$?"
