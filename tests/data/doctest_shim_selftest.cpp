// Self-test of integration/doctest/doctest.h (tests/test_doctest_shim.py):
// SUBCASE traversal (each leaf once, nested), CHECK/REQUIRE semantics,
// Approx, CHECK_THROWS_AS.  Prints the visit log; the test compares it.
#define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
#include "doctest.h"

#include <cstdio>
#include <stdexcept>
#include <string>

static std::string visits;

TEST_CASE("subcases")
{
   visits += "[";
   SUBCASE("A")
   {
      visits += "A";
      SUBCASE("A1") { visits += "1"; }
      SUBCASE("A2") { visits += "2"; }
   }
   SUBCASE("B") { visits += "B"; }
   visits += "]";
}

TEST_CASE("checks")
{
   CHECK(1 + 1 == 2);
   CHECK(0.1 + 0.2 == doctest::Approx(0.3));
   CHECK(1.0 == doctest::Approx(1.0 + 1e-13).epsilon(1e-12));
   CHECK_FALSE(1.0 == doctest::Approx(1.1));
   CHECK_THROWS_AS(throw std::invalid_argument("x"), std::invalid_argument);
   CHECK_NOTHROW((void)0);
   REQUIRE(true);
}

TEST_CASE("report")
{
   std::printf("visits=%s\n", visits.c_str());
}
