// gtest_main.cpp -- TEST INFRASTRUCTURE: main() of the GTest shim (ref_shim/gtest/gtest.h).
#include <gtest/gtest.h>
int main(int argc, char** argv) { return ::testing::RunAllTests(argc, argv); }
