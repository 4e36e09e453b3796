// TEST INFRASTRUCTURE (oracle): entry point for the reference unit tests
// compiled against catch2_lite + eigen_lite.
#include <catch2/catch_amalgamated.hpp>
int main(int argc, char** argv) { return Catch::run_all(argc, argv); }
