#ifndef SELECT_TF32_TN_H
#define SELECT_TF32_TN_H

#include <stdint.h>

typedef struct {
    uint32_t acc;
    uint32_t row_tile;
    uint32_t col_tile;
    uint32_t wg_rows;
    uint32_t wg_cols;
} select_tf32_tn_config;

static inline select_tf32_tn_config select_tf32_tn(int64_t m, int64_t k, int64_t n) {
    (void)m;
    (void)k;
    (void)n;
    if (k < INT64_C(992)) {
        if (m < INT64_C(17740)) {
            if (n < INT64_C(287)) {
                if (k < INT64_C(544)) {
                    if (m < INT64_C(8870)) {
                        if (n < INT64_C(46)) {
                            if (m < INT64_C(2218)) {
                                if (m < INT64_C(1109)) {
                                    select_tf32_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    if (k < INT64_C(167)) {
                                        select_tf32_tn_config out = {1u, 1u, 4u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_tf32_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                }
                            } else {
                                if (m < INT64_C(4435)) {
                                    if (n < INT64_C(28)) {
                                        select_tf32_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (k < INT64_C(167)) {
                                            select_tf32_tn_config out = {8u, 1u, 4u, 16u, 16u};
                                            return out;
                                        } else {
                                            select_tf32_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    }
                                } else {
                                    select_tf32_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                    return out;
                                }
                            }
                        } else {
                            select_tf32_tn_config out = {4u, 1u, 1u, 8u, 8u};
                            return out;
                        }
                    } else {
                        if (n < INT64_C(91)) {
                            select_tf32_tn_config out = {4u, 1u, 1u, 8u, 8u};
                            return out;
                        } else {
                            select_tf32_tn_config out = {1u, 1u, 2u, 8u, 8u};
                            return out;
                        }
                    }
                } else {
                    if (m < INT64_C(555)) {
                        if (k < INT64_C(744)) {
                            select_tf32_tn_config out = {4u, 1u, 1u, 8u, 8u};
                            return out;
                        } else {
                            if (m < INT64_C(139)) {
                                select_tf32_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                if (m < INT64_C(278)) {
                                    select_tf32_tn_config out = {1u, 1u, 2u, 8u, 8u};
                                    return out;
                                } else {
                                    select_tf32_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                    return out;
                                }
                            }
                        }
                    } else {
                        if (n < INT64_C(111)) {
                            if (m < INT64_C(1109)) {
                                select_tf32_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                if (m < INT64_C(8870)) {
                                    if (m < INT64_C(2218)) {
                                        select_tf32_tn_config out = {1u, 1u, 2u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (m < INT64_C(4435)) {
                                            select_tf32_tn_config out = {1u, 1u, 4u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_tf32_tn_config out = {1u, 1u, 2u, 8u, 8u};
                                            return out;
                                        }
                                    }
                                } else {
                                    select_tf32_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                    return out;
                                }
                            }
                        } else {
                            select_tf32_tn_config out = {1u, 1u, 2u, 8u, 8u};
                            return out;
                        }
                    }
                }
            } else {
                if (m < INT64_C(2218)) {
                    if (k < INT64_C(405)) {
                        if (m < INT64_C(1109)) {
                            select_tf32_tn_config out = {4u, 1u, 1u, 8u, 8u};
                            return out;
                        } else {
                            if (n < INT64_C(768)) {
                                select_tf32_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                select_tf32_tn_config out = {1u, 1u, 2u, 8u, 8u};
                                return out;
                            }
                        }
                    } else {
                        if (m < INT64_C(634)) {
                            if (m < INT64_C(278)) {
                                if (m < INT64_C(70)) {
                                    if (k < INT64_C(702)) {
                                        select_tf32_tn_config out = {1u, 1u, 2u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_tf32_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                } else {
                                    select_tf32_tn_config out = {1u, 1u, 2u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                if (n < INT64_C(725)) {
                                    select_tf32_tn_config out = {1u, 1u, 2u, 8u, 8u};
                                    return out;
                                } else {
                                    select_tf32_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                    return out;
                                }
                            }
                        } else {
                            if (k < INT64_C(702)) {
                                select_tf32_tn_config out = {1u, 1u, 2u, 8u, 8u};
                                return out;
                            } else {
                                select_tf32_tn_config out = {1u, 1u, 4u, 8u, 8u};
                                return out;
                            }
                        }
                    }
                } else {
                    select_tf32_tn_config out = {1u, 1u, 2u, 8u, 8u};
                    return out;
                }
            }
        } else {
            if (n < INT64_C(28)) {
                if (m < INT64_C(70960)) {
                    select_tf32_tn_config out = {4u, 1u, 1u, 8u, 8u};
                    return out;
                } else {
                    select_tf32_tn_config out = {1u, 1u, 2u, 8u, 8u};
                    return out;
                }
            } else {
                if (k < INT64_C(97)) {
                    if (m < INT64_C(35480)) {
                        if (n < INT64_C(56)) {
                            select_tf32_tn_config out = {4u, 1u, 1u, 8u, 8u};
                            return out;
                        } else {
                            select_tf32_tn_config out = {1u, 1u, 2u, 8u, 8u};
                            return out;
                        }
                    } else {
                        select_tf32_tn_config out = {1u, 1u, 2u, 8u, 8u};
                        return out;
                    }
                } else {
                    if (n < INT64_C(91)) {
                        if (k < INT64_C(194)) {
                            if (m < INT64_C(100352)) {
                                select_tf32_tn_config out = {1u, 1u, 2u, 8u, 8u};
                                return out;
                            } else {
                                select_tf32_tn_config out = {8u, 1u, 4u, 16u, 16u};
                                return out;
                            }
                        } else {
                            select_tf32_tn_config out = {1u, 1u, 2u, 8u, 8u};
                            return out;
                        }
                    } else {
                        select_tf32_tn_config out = {8u, 1u, 4u, 16u, 16u};
                        return out;
                    }
                }
            }
        }
    } else {
        if (m < INT64_C(28)) {
            if (k < INT64_C(1620)) {
                if (m < INT64_C(3)) {
                    select_tf32_tn_config out = {1u, 1u, 4u, 8u, 8u};
                    return out;
                } else {
                    select_tf32_tn_config out = {1u, 1u, 2u, 8u, 8u};
                    return out;
                }
            } else {
                if (m < INT64_C(2)) {
                    if (n < INT64_C(2024)) {
                        select_tf32_tn_config out = {1u, 1u, 4u, 8u, 8u};
                        return out;
                    } else {
                        select_tf32_tn_config out = {8u, 1u, 4u, 16u, 16u};
                        return out;
                    }
                } else {
                    if (m < INT64_C(12)) {
                        select_tf32_tn_config out = {8u, 1u, 4u, 16u, 16u};
                        return out;
                    } else {
                        if (k < INT64_C(2897)) {
                            select_tf32_tn_config out = {1u, 1u, 2u, 8u, 8u};
                            return out;
                        } else {
                            select_tf32_tn_config out = {8u, 1u, 4u, 16u, 16u};
                            return out;
                        }
                    }
                }
            }
        } else {
            if (n < INT64_C(2509)) {
                if (m < INT64_C(278)) {
                    if (n < INT64_C(363)) {
                        select_tf32_tn_config out = {4u, 1u, 1u, 8u, 8u};
                        return out;
                    } else {
                        if (n < INT64_C(1025)) {
                            if (m < INT64_C(139)) {
                                if (k < INT64_C(3072)) {
                                    if (m < INT64_C(70)) {
                                        select_tf32_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (k < INT64_C(1449)) {
                                            select_tf32_tn_config out = {1u, 1u, 2u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_tf32_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    }
                                } else {
                                    select_tf32_tn_config out = {1u, 1u, 2u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                if (k < INT64_C(3072)) {
                                    select_tf32_tn_config out = {1u, 1u, 2u, 8u, 8u};
                                    return out;
                                } else {
                                    select_tf32_tn_config out = {8u, 1u, 4u, 16u, 16u};
                                    return out;
                                }
                            }
                        } else {
                            if (m < INT64_C(70)) {
                                select_tf32_tn_config out = {1u, 1u, 2u, 8u, 8u};
                                return out;
                            } else {
                                if (m < INT64_C(139)) {
                                    select_tf32_tn_config out = {8u, 1u, 4u, 16u, 16u};
                                    return out;
                                } else {
                                    select_tf32_tn_config out = {1u, 1u, 4u, 8u, 8u};
                                    return out;
                                }
                            }
                        }
                    }
                } else {
                    if (m < INT64_C(4435)) {
                        if (k < INT64_C(1537)) {
                            if (m < INT64_C(2218)) {
                                if (k < INT64_C(1087)) {
                                    if (m < INT64_C(1109)) {
                                        if (m < INT64_C(555)) {
                                            if (n < INT64_C(363)) {
                                                select_tf32_tn_config out = {1u, 1u, 2u, 8u, 8u};
                                                return out;
                                            } else {
                                                select_tf32_tn_config out = {1u, 1u, 4u, 8u, 8u};
                                                return out;
                                            }
                                        } else {
                                            select_tf32_tn_config out = {1u, 1u, 2u, 8u, 8u};
                                            return out;
                                        }
                                    } else {
                                        select_tf32_tn_config out = {1u, 1u, 4u, 8u, 8u};
                                        return out;
                                    }
                                } else {
                                    select_tf32_tn_config out = {1u, 1u, 2u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                select_tf32_tn_config out = {1u, 1u, 4u, 8u, 8u};
                                return out;
                            }
                        } else {
                            if (m < INT64_C(2535)) {
                                if (m < INT64_C(1109)) {
                                    if (k < INT64_C(2173)) {
                                        select_tf32_tn_config out = {8u, 1u, 4u, 16u, 16u};
                                        return out;
                                    } else {
                                        if (k < INT64_C(3259)) {
                                            select_tf32_tn_config out = {1u, 1u, 4u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_tf32_tn_config out = {8u, 1u, 4u, 16u, 16u};
                                            return out;
                                        }
                                    }
                                } else {
                                    select_tf32_tn_config out = {1u, 1u, 4u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                if (n < INT64_C(363)) {
                                    select_tf32_tn_config out = {8u, 1u, 4u, 16u, 16u};
                                    return out;
                                } else {
                                    select_tf32_tn_config out = {1u, 1u, 2u, 8u, 8u};
                                    return out;
                                }
                            }
                        }
                    } else {
                        if (m < INT64_C(35480)) {
                            if (k < INT64_C(1630)) {
                                if (m < INT64_C(8870)) {
                                    if (n < INT64_C(182)) {
                                        select_tf32_tn_config out = {8u, 1u, 4u, 16u, 16u};
                                        return out;
                                    } else {
                                        select_tf32_tn_config out = {1u, 1u, 2u, 8u, 8u};
                                        return out;
                                    }
                                } else {
                                    if (n < INT64_C(182)) {
                                        select_tf32_tn_config out = {1u, 1u, 2u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_tf32_tn_config out = {1u, 1u, 4u, 8u, 8u};
                                        return out;
                                    }
                                }
                            } else {
                                select_tf32_tn_config out = {1u, 1u, 2u, 8u, 8u};
                                return out;
                            }
                        } else {
                            if (m < INT64_C(141920)) {
                                if (m < INT64_C(70960)) {
                                    if (k < INT64_C(1630)) {
                                        select_tf32_tn_config out = {1u, 1u, 2u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_tf32_tn_config out = {1u, 1u, 4u, 8u, 8u};
                                        return out;
                                    }
                                } else {
                                    select_tf32_tn_config out = {1u, 1u, 4u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                select_tf32_tn_config out = {8u, 1u, 4u, 16u, 16u};
                                return out;
                            }
                        }
                    }
                }
            } else {
                select_tf32_tn_config out = {1u, 1u, 4u, 8u, 8u};
                return out;
            }
        }
    }
}

#endif /* SELECT_TF32_TN_H */
